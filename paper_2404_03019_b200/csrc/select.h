// select.h — H2 kernel selection (pure host code).
#pragma once

#include "../../include/geot.h"

namespace geot {

// Full configuration for a problem (§III-C: O(1) features
// Idx_size, avg = Idx_size / Idx_max, F -> configuration tuple).
// skew = max segment length / (nnz / S) when known (a caller hint), else <= 0.
geot_status select_config_impl(long long nnz, long long S, long long F, geot_reduce op, geot_dtype dt,
                               geot_itype it, int fused, double skew, geot_config* out);

// The pre-refit hand rules alone (the selector's comparison baseline).
geot_status select_hand_rules(long long nnz, long long S, long long F, geot_dtype dt, int fused, geot_config* out);

// Derive the lane shape (LPR, VPL) and rows-per-group for c->vec_elems.
void select_shape_for_vw(long long F, geot_dtype dt, geot_config* c);

// GEOT_VARIANT_STREAM: applicability, lane shape (16-byte lane vectors), the
// compiled pipelines, and switching a configuration to its default pipeline.
bool stream_eligible(long long nnz, long long F, geot_dtype dt, int fused);
bool stream_lane_shape(long long F, geot_dtype dt, int* lpr, int* vpl);
bool stream_pipe_compiled(int lpr, int vpl, geot_dtype dt, int w, int rs, int ns, int fused);
bool to_stream(long long F, geot_dtype dt, geot_config* c);
void stream_default_pipe(int lpr, int vpl, int* w, int* rs, int* ns);
bool narrow_eligible(long long nnz, long long F, geot_dtype dt, int fused);

// The generated tree itself (diagnostics / codegen-fidelity test) and its provenance.
void select_tree_raw(double log2_nnz, double avg, double skew, double F, double dtype, double fused, double op,
                     int out[4]);
const char* select_tree_provenance();

}  // namespace geot
