/*
 * geot.h — C ABI of the B200-native (sm_100a) GeoT segment-reduction library
 * (libgeot.so, built from paper_2404_03019_b200/csrc/).
 *
 * Operation (§II-B "Segment Reduction"): given a sorted
 * (non-decreasing) index Idx of length M = |E| and a row-major M x N matrix X
 * (N = F), produce Y (|V| x N) with
 *
 *      Y[s, :] = f over { X[e, :] : Idx[e] == s },   f in {sum, mean, max}
 *
 * (f varies per PAPER.md:76, Fig. 2(c); "mainly an engineering effort",
 * P:523-524).  The fused form (§IV, Listing 3,
 * `index_segment_reduce(edge_index[0], edge_index[1], x)`) reads
 * X[e, :] := x[src_idx[e], :] without materialising X; the weighted fused form
 * (`index_weight_segment_reduce`, SpMM on sorted COO) reads
 * X[e, :] := w[e] * x[src_idx[e], :].
 *
 * Conventions shared by every entry point:
 *  - Pointers named d_* / src / idx / x / out / workspace are DEVICE memory
 *    owned by the caller; the library never allocates, frees or retains them.
 *    Host pointers are named h_* / cfg.
 *  - Layout: every matrix is dense row-major with row stride F elements;
 *    `out` must not alias any input.
 *  - Values: GEOT_F32 (float) or GEOT_BF16 (bfloat16) inputs; accumulation is
 *    fp32; `out` has the input dtype (bf16: one round-to-nearest-even of the
 *    fp32 result).  Indices: GEOT_I32 or GEOT_I64 (all index arrays of one
 *    call share the type).
 *  - `out` is WRITE-ONLY: after a successful call every row [0, num_segments)
 *    is defined, empty segments included (0 for sum, mean and max — reading R1
 *    of DESIGN.md), so no pre-initialisation is needed.
 *  - Every call is asynchronous and stream-ordered on `stream`; none performs
 *    a hidden device->host synchronisation (the segment count is an argument,
 *    never read from Idx[M-1] as the paper's Python API implies).
 *  - Synchronous errors are returned immediately: a null pointer where data is
 *    needed, nnz < 0, num_segments < 0, F < 1, unknown enum, unsupported
 *    combination, workspace too small, or a CUDA launch error (GEOT_ERR_CUDA).
 *  - Data-dependent preconditions (Idx sorted, Idx in [seg_base,
 *    seg_base+num_segments), src_idx in [0, num_x_rows)) are NOT checked on the
 *    hot path (the paper's precondition "guaranteed by GNN frameworks",
 *    P:328); geot_validate_index() checks them.  On violating data the kernels
 *    stay memory-safe (out-of-range rows are skipped, nothing outside `out` is
 *    written) but the result is unspecified.
 *  - Determinism: for a fixed configuration the result is bitwise
 *    reproducible (tile-ordered carry combination, no floating-point atomics).
 *  - Thread safety: all entry points are re-entrant; the only global state is
 *    a lazily initialised per-device property cache and a launch counter.
 */
#ifndef GEOT_H
#define GEOT_H

#include <stddef.h>
#include <stdint.h>

#include <cuda_runtime_api.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GEOT_ABI_VERSION 1

typedef enum {
    GEOT_OK = 0,
    GEOT_ERR_INVALID_VALUE = 1,      /* bad scalar argument or null pointer      */
    GEOT_ERR_UNSUPPORTED = 2,        /* valid but unsupported combination        */
    GEOT_ERR_WORKSPACE_TOO_SMALL = 3,/* ws_bytes < geot_workspace_size(...)      */
    GEOT_ERR_UNSORTED_INDEX = 4,     /* reported by geot_validate_index only     */
    GEOT_ERR_INDEX_OUT_OF_RANGE = 5, /* reported by geot_validate_index only     */
    GEOT_ERR_SRC_OUT_OF_RANGE = 6,   /* reported by geot_validate_index only     */
    GEOT_ERR_CUDA = 7                /* a CUDA runtime error (launch, attribute) */
} geot_status;

typedef enum { GEOT_SUM = 0, GEOT_MEAN = 1, GEOT_MAX = 2 } geot_reduce;
typedef enum { GEOT_F32 = 0, GEOT_BF16 = 1 } geot_dtype;
typedef enum { GEOT_I32 = 0, GEOT_I64 = 1 } geot_itype;

/* Kernel variants (the B200 analog of the paper's SR / PR schedules, §III-B,
 * P:174-216). */
typedef enum {
    GEOT_VARIANT_AUTO = 0,      /* let geot_select_config() decide            */
    GEOT_VARIANT_EDGE_TILE = 1, /* edge-parallel tiles, lane-group sequential
                                   reduction (SR analog) + in-CTA segmented
                                   combine + deterministic tile carries        */
    GEOT_VARIANT_NARROW = 2,    /* small F: thread-sequential items + warp
                                   segmented scan via __shfl_sync (PR/Alg. 1
                                   analog)                                     */
    GEOT_VARIANT_STREAM = 3     /* rows >= 128 B, contiguous: persistent CTAs,
                                   per-warp TMA bulk-copy rings (cp.async.bulk
                                   + mbarrier), balanced contiguous edge ranges
                                   per lane group, agent-ordered carries;
                                   rows_per_group = rows per ring stage       */
} geot_variant;

/* Kernel configuration: the B200 analog of the paper's tunable tuple
 * <T_N, T_M, M_t, N_t, G_t> (Table I).  Zero fields mean "auto". */
typedef struct geot_config {
    int32_t variant;        /* geot_variant                                    */
    int32_t vec_elems;      /* elements per vector load (VW): f32 {4,1}, bf16 {8,1}  */
    int32_t lanes_per_row;  /* lanes of one row group (LPR): 1..32, power of 2 */
    int32_t vecs_per_lane;  /* vectors per lane per row (VPL): 1,2,4,8         */
    int32_t rows_per_group; /* sequential rows per lane group (R, M_t analog);
                               STREAM: rows per lane group per ring stage     */
    int32_t warps_per_cta;  /* EDGE_TILE: 8; STREAM: 8 or 16                   */
    int32_t ctas_per_sm;    /* persistent-grid multiplier; 0 = occupancy max   */
    int32_t stages;         /* STREAM: TMA ring stages per warp (4, 6, 8), or
                               1 = no ring: 128-bit LDG into a register double
                               buffer (2 CTAs per SM); 0 = auto              */
    int32_t reserved;       /* must be 0                                       */
} geot_config;

/* Human-readable status text (static storage). */
const char* geot_status_string(geot_status s);

/* Text of the CUDA error behind the calling thread's last GEOT_ERR_CUDA
 * ("" if none).  Static storage. */
const char* geot_last_cuda_error(void);

/* ABI version of the loaded library (== GEOT_ABI_VERSION). */
int geot_abi_version(void);

/* Number of kernels this process has launched through the library (all
 * devices, all threads) — used by bench.py to report gpu_launches. */
uint64_t geot_launch_count(void);

/* Measurement hook (bench.py roofline): the NEXT reduction call made by the
 * calling thread records `before` on its stream immediately before launching
 * its main reduction kernel and `after` immediately after it, so the caller
 * can time that kernel alone with CUDA events on the launching stream.
 * Either may be NULL to clear.  The pair is consumed by that one call. */
void geot_profile_events(cudaEvent_t before, cudaEvent_t after);

/* H2 kernel selection (P:301-315 data-aware config rules; the generated
 * decision tree of Listing 5, refit on B200 — DESIGN.md §5).
 * Pure host code: reads no device memory and launches nothing.
 * Features: nnz (Idx_size), num_segments (|V|; avg = nnz/num_segments),
 * F, op, dtype, itype, fused (0/1: index_segment_reduce form).
 * Writes a complete configuration to *cfg_out. */
geot_status geot_select_config(int64_t nnz, int64_t num_segments, int64_t F, geot_reduce op,
                               geot_dtype dtype, geot_itype itype, int fused, geot_config* cfg_out);

/* geot_select_config with the north_star's skew feature: skew = the longest
 * segment's length / (nnz / num_segments), e.g. from a plan computed once per
 * graph (Python: paper_2404_03019_b200.geot_plan); skew <= 0 = unknown (what
 * geot_select_config and the cfg = NULL reductions use).  NaN ->
 * GEOT_ERR_INVALID_VALUE.  Pure host code. */
geot_status geot_select_config_ex(int64_t nnz, int64_t num_segments, int64_t F, geot_reduce op,
                                  geot_dtype dtype, geot_itype itype, int fused, double skew, geot_config* cfg_out);

/* Diagnostics: the configuration the pre-refit hand rules pick (STREAM with the
 * lane shape's default pipeline when eligible, else NARROW when eligible, else
 * EDGE_TILE with ~128 KB tiles) — the baseline the refit tree is scored
 * against (the paper's Fig. 6 comparison).  Pure host code. */
geot_status geot_select_hand_rules(int64_t nnz, int64_t num_segments, int64_t F, geot_dtype dtype, int fused,
                                   geot_config* cfg_out);

/* The generated decision tree alone (select_tree.inc; Listing 5,
 * P:432-444), for diagnostics and the codegen-fidelity test: leaf tuple
 * (variant, rows_per_group, warps_per_cta, stages) for features
 * log2(nnz), avg = nnz/num_segments, skew = log2(max length / avg) or -1 when
 * unknown, F, dtype (0 f32 / 1 bf16), fused (0/1), op (0 sum / 1 mean / 2 max);
 * '<=' goes left at every threshold.  geot_select_config applies the leaf only
 * where it is valid for the input (else the hand rules). */
void geot_select_tree(double log2_nnz, double avg, double skew, double F, double dtype, double fused, double op,
                      int32_t out[4]);

/* Provenance text of the compiled tree (perf DB, split, quality). */
const char* geot_selector_provenance(void);

/* Workspace (device bytes) the reduction needs for the given problem under
 * configuration *cfg (NULL = the configuration geot_select_config picks).
 * The workspace holds per-agent carries plus a few control words: it must be
 * zero-filled ONCE before its first use (geot_workspace_init or any memset to
 * 0); every call leaves it ready for the next one, so it may then be reused by
 * any number of later calls, in stream order (never by two calls executing
 * concurrently). */
size_t geot_workspace_size(int64_t nnz, int64_t num_segments, int64_t F, geot_reduce op,
                           geot_dtype dtype, geot_itype itype, int fused, const geot_config* cfg);

/* Zero-fill a fresh workspace of ws_bytes device bytes on `stream`
 * (cudaMemsetAsync).  Needed once per workspace allocation. */
geot_status geot_workspace_init(void* workspace, size_t ws_bytes, cudaStream_t stream);

/* Health of a workspace (SYNCHRONOUS: reads its control words after
 * synchronising `stream`; a diagnostic, not for the hot path).  *h_status
 * (host) = 0 healthy; bit 1 = poisoned: some call drew an out-of-range ticket
 * because the workspace was not zero-filled before first use or was used by
 * two calls at once — such a call retires without writing its output (no trap,
 * no hang) and the flag stays set until geot_workspace_init; bit 2 = the
 * control words are not at rest (a call is in flight on another stream, or a
 * poisoned call left them so).  Recovery: geot_workspace_init, then repeat the
 * call.  NULL / tiny workspaces report 0. */
geot_status geot_workspace_status(const void* workspace, size_t ws_bytes, cudaStream_t stream, int32_t* h_status);

/* H4-H7: sorted-index segment reduction (Fig. 2; Alg. 1's result).
 *   src        [nnz, F] values (dtype), device
 *   idx        [nnz] non-decreasing segment ids (itype), device
 *   out        [num_segments, F] (dtype), device, write-only
 *   workspace  >= geot_workspace_size(..., fused=0, NULL) bytes, device (may be
 *              NULL when that size is 0)
 * Returns GEOT_OK or a synchronous error (see conventions). */
geot_status geot_segment_reduce(const void* src, const void* idx, int64_t nnz, int64_t num_segments,
                                int64_t F, geot_reduce op, geot_dtype dtype, geot_itype itype, void* out,
                                void* workspace, size_t ws_bytes, cudaStream_t stream);

/* Extended form used by the multi-GPU shard driver (H9) and by selector
 * sweeps: segment ids in idx lie in [seg_base, seg_base + num_segments) and
 * out row r holds segment seg_base + r; *cfg (nullable) overrides selection. */
geot_status geot_segment_reduce_ex(const void* src, const void* idx, int64_t nnz, int64_t seg_base,
                                   int64_t num_segments, int64_t F, geot_reduce op, geot_dtype dtype,
                                   geot_itype itype, void* out, void* workspace, size_t ws_bytes,
                                   const geot_config* cfg, cudaStream_t stream);

/* f4 (SURVEY §8(e), §8(f) "output all-gather fused into the epilogue"): the
 * H9 shard form of geot_segment_reduce_ex whose finished rows are stored
 * straight into EVERY rank's replica of the full output, so no separate
 * all-gather collective follows.
 *   outs     host array of nouts (1..8) device pointers, each a
 *            [total_segments, F] (dtype) buffer reachable from this GPU: its
 *            own replica and the peers' replicas mapped into this process
 *            (cudaDeviceEnablePeerAccess, CUDA IPC or symmetric memory); the
 *            stores to a peer travel over NVLink.
 *   rows [seg_base, seg_base + num_segments) of every replica are written
 *   (empty segments zero-filled); no other row is touched.  Ownership,
 *   workspace, stream and error behaviour as geot_segment_reduce_ex; nouts
 *   outside 1..8 or a NULL pointer -> GEOT_ERR_INVALID_VALUE.  Stream-ordered
 *   on THIS GPU only: the caller orders the peers' reads after it (e.g. a
 *   barrier after synchronising the stream). */
geot_status geot_segment_reduce_allgather(const void* src, const void* idx, int64_t nnz, int64_t seg_base,
                                          int64_t num_segments, int64_t F, geot_reduce op, geot_dtype dtype,
                                          geot_itype itype, void* const* outs, int nouts, void* workspace,
                                          size_t ws_bytes, const geot_config* cfg, cudaStream_t stream);

/* f4, NVLS form (not in the paper, which is single-GPU,
 * P:338): as geot_segment_reduce_allgather, but the peers' replicas are
 * reached through ONE multicast address: every finished row (and every
 * zero-filled empty row) is stored once into local_out with ordinary stores
 * and once through mc_out with multimem.st, which NVSwitch replicates into
 * every buffer bound to the multicast object (NVLink SHARP) — one store per
 * row instead of one per peer.
 *   local_out  this rank's [total_segments, F] replica (device).
 *   mc_out     the multicast virtual address of the replicas
 *              (cuMulticastCreate / cuMulticastBindMem / cuMemMap, or
 *              torch symmetric memory's multicast_ptr); it maps every rank's
 *              replica, including this one (its rows are written twice, with
 *              the same bits).
 *   Rows of a whole number of 4-byte words and 16-byte aligned buffers only
 *   (multimem.st has no 2-byte form), and no bf16 edge-tile shape (single
 *   bf16 elements): else GEOT_ERR_UNSUPPORTED.  NULL pointers, seg_base < 0 ->
 *   GEOT_ERR_INVALID_VALUE.  Ownership, workspace, stream, ordering and the
 *   other errors as geot_segment_reduce_allgather.  A plain device address
 *   passed as mc_out is written with multimem.st and faults: the caller
 *   checks that multicast is available (it is not on a single-GPU box). */
geot_status geot_segment_reduce_multicast(const void* src, const void* idx, int64_t nnz, int64_t seg_base,
                                          int64_t num_segments, int64_t F, geot_reduce op, geot_dtype dtype,
                                          geot_itype itype, void* local_out, void* mc_out, void* workspace,
                                          size_t ws_bytes, const geot_config* cfg, cudaStream_t stream);

/* H8: fused gather + segment reduction (P:293 index_segment_reduce):
 *   Y[s,:] = f over { x[src_idx[e], :] : dst_idx[e] == s }.
 *   x        [num_x_rows, F] node features (dtype), device
 *   src_idx  [nnz] arbitrary row ids into x (itype), device
 *   dst_idx  [nnz] non-decreasing segment ids (itype), device
 *   out      [num_segments, F], device, write-only. */
geot_status geot_gather_segment_reduce(const void* x, int64_t num_x_rows, const void* src_idx,
                                       const void* dst_idx, int64_t nnz, int64_t num_segments, int64_t F,
                                       geot_reduce op, geot_dtype dtype, geot_itype itype, void* out,
                                       void* workspace, size_t ws_bytes, cudaStream_t stream);

/* Weighted fused form (P:330 index_weight_segment_reduce; SpMM on sorted COO,
 * P:469): Y[s,:] = sum { w[e] * x[src_idx[e], :] : dst_idx[e] == s }.
 *   weight [nnz] fp32, device.  Only GEOT_SUM is supported (else
 *   GEOT_ERR_UNSUPPORTED), as in the paper. */
geot_status geot_gather_weight_segment_reduce(const void* x, int64_t num_x_rows, const void* src_idx,
                                              const void* dst_idx, const float* weight, int64_t nnz,
                                              int64_t num_segments, int64_t F, geot_dtype dtype,
                                              geot_itype itype, void* out, void* workspace,
                                              size_t ws_bytes, cudaStream_t stream);

/* Extended fused form: weight nullable (NULL = unweighted), seg_base, cfg. */
geot_status geot_gather_segment_reduce_ex(const void* x, int64_t num_x_rows, const void* src_idx,
                                          const void* dst_idx, const float* weight, int64_t nnz,
                                          int64_t seg_base, int64_t num_segments, int64_t F, geot_reduce op,
                                          geot_dtype dtype, geot_itype itype, void* out, void* workspace,
                                          size_t ws_bytes, const geot_config* cfg, cudaStream_t stream);

/* f3 (the paper defers autograd: P:497):
 * gradient of geot_segment_reduce (seg_base 0) w.r.t. src:
 *   grad_src[e,:] = g * grad_out[idx[e],:]  with g = 1 (sum), 1/count (mean),
 *   [src[e,f] == out[s,f]] / ties[s,f] (max; ties split evenly).
 *   grad_out  [num_segments, F] (dtype), device
 *   offsets   [num_segments+1] int64 from geot_segment_offsets (mean; else NULL)
 *   src, out  the forward input / output (max; else NULL)
 *   ties      [num_segments, F] fp32 scratch (max; else NULL)
 *   grad_src  [nnz, F] (dtype), device, write-only.  Deterministic. */
geot_status geot_segment_reduce_backward(const void* grad_out, const void* idx, int64_t nnz, int64_t num_segments,
                                         int64_t F, geot_reduce op, geot_dtype dtype, geot_itype itype,
                                         const int64_t* offsets, const void* src, const void* out, float* ties,
                                         void* grad_src, cudaStream_t stream);

/* f3: gradients of the (weighted) fused form, fp32, op sum or mean:
 *   grad_x[v,:]  = sum_{e: src[e]==v} w[e] * g(e) * grad_out[dst[e],:]   (scatter by the
 *                  unsorted source index: fp32 atomics, NOT bitwise reproducible)
 *   grad_w[e]    = g(e) * <x[src[e],:], grad_out[dst[e],:]>              (SDDMM)
 * with g = 1 (sum) or 1/count[dst[e]] (mean; offsets from geot_segment_offsets).
 * weight / grad_x / grad_w / x nullable (grad_w needs x). */
geot_status geot_gather_segment_reduce_backward(const float* grad_out, const void* src_idx, const void* dst_idx,
                                                const float* weight, int64_t nnz, int64_t num_segments,
                                                int64_t num_x_rows, int64_t F, geot_reduce op, geot_itype itype,
                                                const int64_t* offsets, const float* x, float* grad_x, float* grad_w,
                                                cudaStream_t stream);

/* H3: segment offsets (CSR row pointer) of a sorted index:
 *   offsets[s] = #{ e : idx[e] < s },  s = 0..num_segments  (int64, device,
 *   num_segments + 1 entries, write-only).  counts[s] = offsets[s+1]-offsets[s].
 * Bit-exact.  Not needed by geot_segment_reduce (boundaries are detected
 * inline, the is_seg test of Alg. 1). */
geot_status geot_segment_offsets(const void* idx, geot_itype itype, int64_t nnz, int64_t num_segments,
                                 int64_t* offsets, cudaStream_t stream);

/* Precondition check (P:85 sortedness):
 * writes to *d_status (device int32) a bit mask: 1 = idx not non-decreasing,
 * 2 = some idx outside [0, num_segments), 4 = some src_idx outside
 * [0, num_x_rows) (src_idx nullable).  0 = valid.  Asynchronous; the caller
 * reads *d_status after synchronising. */
geot_status geot_validate_index(const void* idx, geot_itype itype, int64_t nnz, int64_t num_segments,
                                const void* src_idx, int64_t num_x_rows, int32_t* d_status,
                                cudaStream_t stream);

/* H9: multi-GPU partition of the sorted edge stream at segment boundaries
 * (north_star; reading R18).  For p = 0..nparts:
 *   t_p = floor(p * nnz / nparts);  s_0 = 0;  s_nparts = num_segments;
 *   s_p = (t_p == 0) ? 0 : idx[t_p - 1] + 1;   e_p = #{ e : idx[e] < s_p }.
 * Part p owns output rows [s_p, s_{p+1}) and edges [e_p, e_{p+1}).
 *   seg_bounds, edge_bounds: int64 [nparts + 1], device, write-only.
 * Bit-exact. */
geot_status geot_partition(const void* idx, geot_itype itype, int64_t nnz, int64_t num_segments,
                           int nparts, int64_t* seg_bounds, int64_t* edge_bounds, cudaStream_t stream);

/* f4 / SURVEY §8(e) "Alternative partition (not default)": EXACT edge split
 * with a one-step exchange of the straddling partials.  For p = 0..nparts:
 *   t_p = floor(p * nnz / nparts)                       (edge_bounds: exact)
 *   s_0 = 0;  s_nparts = num_segments;  s_p = (t_p == 0) ? 0 : idx[t_p - 1] + 1
 *   boundary_keys[2p] = (t_p > 0) ? idx[t_p - 1] : -1;  boundary_keys[2p+1] = (t_p < nnz) ? idx[t_p] : -1
 * Part p reduces edges [t_p, t_{p+1}) and owns rows [s_p, s_{p+1}).  Where
 * idx[t_p - 1] == idx[t_p] the segment STRADDLES split p: it belongs to the
 * lower part (the one holding edge t_p - 1), and every higher part it reaches
 * contributes an fp32 partial (geot_segment_reduce_split) that the owner folds
 * in rank order (geot_combine_partials) — DESIGN.md reading R21.  Balance is
 * exact (|part| = floor or ceil of nnz/nparts) at the price of that exchange;
 * geot_partition (H9) needs no exchange but may be unbalanced by a hub.
 *   seg_bounds, edge_bounds  int64 [nparts + 1], device, write-only
 *   boundary_keys            int64 [2 * (nparts + 1)], device, write-only
 * Bit-exact.  nparts < 1, nnz < 0 or num_segments < 0 -> GEOT_ERR_INVALID_VALUE. */
geot_status geot_partition_exact(const void* idx, geot_itype itype, int64_t nnz, int64_t num_segments, int nparts,
                                 int64_t* seg_bounds, int64_t* edge_bounds, int64_t* boundary_keys,
                                 cudaStream_t stream);

/* Workspace of geot_segment_reduce_split (device bytes; zero-filled once, as
 * for geot_workspace_size, which it includes). */
size_t geot_split_workspace_size(int64_t nnz, int64_t num_segments, int64_t F, geot_reduce op, geot_dtype dtype,
                                 geot_itype itype, const geot_config* cfg);

/* One part of the exact split: geot_segment_reduce_ex over the part's edges
 * (rows [seg_base, seg_base + num_segments), the head segment's row, which
 * lies below seg_base when it straddles, is not written) PLUS the fp32
 * partials of
 *   slot 0: the head part, edges with key == idx[0]       (if head_open)
 *   slot 1: the tail part, edges with key == idx[nnz - 1] (if tail_open)
 * in partials[slot * F .. slot * F + F) (fp32, device) with their edge counts
 * in counts[slot] (int64, device); a closed slot gets count 0 and the op's
 * identity.  Each partial folds its rows in ascending order in chunks of 1024
 * and the chunks in order (deterministic).  When tail_open the tail key's row
 * holds only this part's edges until geot_combine_partials overwrites it.
 * head_open / tail_open come from geot_partition_exact's boundary keys
 * (idx[t_p - 1] == idx[t_p]); the part itself never reads past its edges. */
geot_status geot_segment_reduce_split(const void* src, const void* idx, int64_t nnz, int64_t seg_base,
                                      int64_t num_segments, int64_t F, geot_reduce op, geot_dtype dtype,
                                      geot_itype itype, int head_open, int tail_open, void* out, float* partials,
                                      int64_t* counts, void* workspace, size_t ws_bytes, const geot_config* cfg,
                                      cudaStream_t stream);

/* The owner's fold of a straddling segment: out_row[f] = finalize(fold over
 * k < nslots of partials[h_slots[k] * F + f]) with count = sum of
 * counts[h_slots[k]] (sum; mean = one fp32 division; max), stored in dtype.
 *   partials [*, F] fp32 and counts [*] int64: every part's two slots after
 *            the exchange (part q's head = slot 2q, tail = 2q + 1), device
 *   h_slots  host array of nslots (1..64) slot ids, folded in that order
 *   out_row  F elements (dtype), device.  Deterministic. */
geot_status geot_combine_partials(const float* partials, const int64_t* counts, const int32_t* h_slots, int nslots,
                                  int64_t F, geot_reduce op, geot_dtype dtype, void* out_row, cudaStream_t stream);

/* Self-test hook (tests only; nothing on the hot path calls it): runs the
 * narrow kernel's warp segmented scan (the warp pass of Alg. 1, P:199-205;
 * narrow.cuh warp_segscan) on nwarps x 32 (key, value) items, one item per
 * lane, a segment starting in lane l when l == 0 or keys[l] != keys[l-1].
 * Per lane: out_vals = fold (sum for GEOT_SUM / GEOT_MEAN, max for GEOT_MAX)
 * of the values from its segment's first lane through itself, out_flags = 1,
 * out_pos = that first lane's index (propagated for GEOT_MEAN only, else 0
 * except at starts).  All pointers device, [nwarps * 32]. */
geot_status geot_selftest_warp_segscan(const int32_t* keys, const float* vals, int64_t nwarps, geot_reduce op,
                                       float* out_vals, int32_t* out_flags, int64_t* out_pos, cudaStream_t stream);

#ifdef __cplusplus
}
#endif

#endif /* GEOT_H */
