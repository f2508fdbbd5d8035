// geot.cu — the C ABI of libgeot (include/geot.h): argument checking, kernel
// selection hand-off, workspace carving, launches; plus the small integer
// kernels (offsets H3, validation, partition H9, empty-output fill).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstring>

#include "../../include/geot.h"
#include "launch.cuh"
#include "narrow.cuh"
#include "select.h"

namespace geot {

std::atomic<unsigned long long> g_launches{0};
thread_local cudaEvent_t g_prof_before = nullptr, g_prof_after = nullptr;

// ----------------------------------------------------------- device cache
static int sm_count() {
    static std::atomic<int> cache[64];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
    int v = cache[dev].load(std::memory_order_relaxed);
    if (v > 0) return v;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
    cache[dev].store(v, std::memory_order_relaxed);
    return v;
}

// ----------------------------------------------------------- small kernels
// H3: offsets[s] = #{e : idx[e] < s}.  Thread e writes offsets[s] = e for the
// s in (idx[e-1], idx[e]] (the first edge at or past s); thread E writes E
// for s in (idx[E-1], S].  Each entry is written exactly once (sorted idx).
__global__ void offsets_kernel(const void* idx, int idx64, long long E, long long S, long long* offsets) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e <= E; e += stride) {
        const long long prev = (e == 0) ? -1 : load_index(idx, idx64, e - 1);
        const long long cur = (e == E) ? S : load_index(idx, idx64, e);
        long long lo = prev + 1, hi = cur;  // inclusive range of s
        if (lo < 0) lo = 0;
        if (hi > S) hi = S;
        for (long long s = lo; s <= hi; ++s) offsets[s] = e;
    }
}

// Precondition check: bit 1 unsorted, 2 idx out of [0,S), 4 src out of [0,V).
__global__ void validate_kernel(const void* idx, int idx64, long long E, long long S, const void* src,
                                long long V, int* status) {
    int bad = 0;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < E; e += stride) {
        const long long k = load_index(idx, idx64, e);
        if (k < 0 || k >= S) bad |= 2;
        if (e > 0 && load_index(idx, idx64, e - 1) > k) bad |= 1;
        if (src) {
            const long long r = load_index(src, idx64, e);
            if (r < 0 || r >= V) bad |= 4;
        }
    }
    bad = __reduce_or_sync(0xffffffffu, bad);
    if ((threadIdx.x & 31) == 0 && bad) atomicOr(status, bad);
}

// H9: one thread per bound p in [0, P].
__global__ void partition_kernel(const void* idx, int idx64, long long E, long long S, int P, long long* seg_b,
                                 long long* edge_b) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p > P) return;
    long long sp;
    if (p == 0)
        sp = 0;
    else if (p == P)
        sp = S;
    else {
        const long long tp = (long long)(((unsigned __int128)p * (unsigned __int128)E) / (unsigned __int128)P);
        sp = (tp == 0) ? 0 : load_index(idx, idx64, tp - 1) + 1;
    }
    // e_p = lower_bound(idx, sp)
    long long lo = 0, hi = E;
    while (lo < hi) {
        const long long mid = lo + ((hi - lo) >> 1);
        if (load_index(idx, idx64, mid) < sp)
            lo = mid + 1;
        else
            hi = mid;
    }
    seg_b[p] = sp;
    edge_b[p] = lo;
}

// E == 0: every output row is an empty segment -> zero bytes.
__global__ void zero_fill_kernel(unsigned char* out, long long bytes) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    const long long n16 = ((reinterpret_cast<uintptr_t>(out) & 15) == 0) ? bytes / 16 : 0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride)
        reinterpret_cast<uint4*>(out)[i] = make_uint4(0, 0, 0, 0);
    for (long long i = n16 * 16 + (long long)blockIdx.x * blockDim.x + threadIdx.x; i < bytes; i += stride) out[i] = 0;
}

// ------------------------------------------------------------ workspace
// Layout: [StreamCtrl | 256 B][stream flags: one u64 per possible agent][meta]
// [carry_h][carry_t].  The control words and flags sit at FIXED offsets for
// every call and variant, so stale bytes of other regions can never be read as
// a flag; they must be zero before the workspace's first use.
static int sm_count();
// one flag per agent: up to 16 warps x 8 agents per CTA, 2 CTAs per SM
static size_t ws_flag_bytes() { return align_up((size_t)sm_count() * 16 * 8 * 2 * sizeof(unsigned long long), 256); }
struct WsLayout {
    size_t ctrl = 0, flags = 0, meta = 0, carry_h = 0, carry_t = 0, total = 0;
};
static WsLayout ws_layout(long long ntiles, long long F) {
    WsLayout w;
    if (ntiles <= 1) return w;  // a single tile never carries
    w.ctrl = 0;
    w.flags = 256;
    w.meta = w.flags + ws_flag_bytes();
    w.carry_h = w.meta + align_up((size_t)ntiles * sizeof(TileMeta), 256);
    w.carry_t = w.carry_h + align_up((size_t)ntiles * (size_t)F * sizeof(float), 256);
    w.total = w.carry_t + align_up((size_t)ntiles * (size_t)F * sizeof(float), 256);
    return w;
}

long long stream_agents(long long nnz, int lpr, int warps, int nsm, int ctas_per_sm) {
    if (warps != 8 && warps != 16) return 0;
    const long long per_cta = (long long)warps * (32 / lpr);
    long long grid = nnz / per_cta;
    if (grid > (long long)nsm * ctas_per_sm) grid = (long long)nsm * ctas_per_sm;
    return grid >= 1 ? grid * per_cta : 0;
}

static long long tile_rows_of(const geot_config& c) { return (long long)(256 / c.lanes_per_row) * c.rows_per_group; }

static long long ntiles_of(long long nnz, const geot_config& c) {
    const long long tr = tile_rows_of(c);
    return (nnz + tr - 1) / tr;
}

static bool aligned(const void* p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

static thread_local cudaError_t g_last_cuda_error = cudaSuccess;
static geot_status from_cuda(cudaError_t e) {
    if (e == cudaSuccess) return GEOT_OK;
    g_last_cuda_error = e;
    return GEOT_ERR_CUDA;
}

// Complete / check a (possibly partial) configuration for a call.
static geot_status resolve_config(long long nnz, long long S, long long F, geot_reduce op, geot_dtype dt,
                                  geot_itype it, int fused, const geot_config* user, geot_config* out) {
    geot_config c;
    geot_status st = select_config_impl(nnz, S, F, op, dt, it, fused, 0.0, &c);
    if (st != GEOT_OK) return st;
    if (user) {
        if (user->reserved != 0) return GEOT_ERR_INVALID_VALUE;
        if (user->variant < 0 || user->variant > GEOT_VARIANT_STREAM) return GEOT_ERR_UNSUPPORTED;
        if (user->variant == GEOT_VARIANT_NARROW) {  // no tunables: the shape follows F
            if (!narrow_eligible(nnz, F, dt, fused)) return GEOT_ERR_UNSUPPORTED;
            c.variant = GEOT_VARIANT_NARROW;
            *out = c;
            return GEOT_OK;
        }
        const bool tile_fields = user->vec_elems || user->lanes_per_row || user->vecs_per_lane ||
                                 user->rows_per_group || user->ctas_per_sm;
        if (user->variant == GEOT_VARIANT_AUTO && c.variant == GEOT_VARIANT_NARROW && tile_fields) {
            c.variant = GEOT_VARIANT_EDGE_TILE;  // edge-tile fields given: tune the edge-tile kernel
            select_shape_for_vw(F, dt, &c);
            c.ctas_per_sm = 0;
        }
        if (user->variant == GEOT_VARIANT_EDGE_TILE && c.variant != GEOT_VARIANT_EDGE_TILE) {
            // back to the edge-tile defaults before applying the overrides
            c.variant = GEOT_VARIANT_EDGE_TILE;
            select_shape_for_vw(F, dt, &c);
            c.ctas_per_sm = 0;
        }
        if (user->variant == GEOT_VARIANT_STREAM && c.variant != GEOT_VARIANT_STREAM) {
            if (!stream_eligible(nnz, F, dt, fused) || !to_stream(F, dt, &c)) return GEOT_ERR_UNSUPPORTED;
        }
        if (c.variant == GEOT_VARIANT_STREAM) {  // lane shape fixed by F; pipeline shape tunable
            if (user->rows_per_group) c.rows_per_group = user->rows_per_group;
            if (user->warps_per_cta) c.warps_per_cta = user->warps_per_cta;
            if (user->stages) c.stages = user->stages;
            // (an uncompiled pipeline shape is refused at launch: GEOT_ERR_UNSUPPORTED)
            if ((user->vec_elems && user->vec_elems != c.vec_elems) ||
                (user->lanes_per_row && user->lanes_per_row != c.lanes_per_row) ||
                (user->vecs_per_lane && user->vecs_per_lane != c.vecs_per_lane))
                return GEOT_ERR_UNSUPPORTED;
            *out = c;
            return GEOT_OK;
        }
        if (user->vec_elems) c.vec_elems = user->vec_elems;
        if (user->lanes_per_row) c.lanes_per_row = user->lanes_per_row;
        if (user->vecs_per_lane) c.vecs_per_lane = user->vecs_per_lane;
        if (user->rows_per_group) c.rows_per_group = user->rows_per_group;
        if (user->warps_per_cta && user->warps_per_cta != 8) return GEOT_ERR_UNSUPPORTED;
        if (user->stages) return GEOT_ERR_UNSUPPORTED;
        c.ctas_per_sm = user->ctas_per_sm;
        const int wide = dt == GEOT_F32 ? 4 : 8;
        if (c.vec_elems != 1 && c.vec_elems != wide) return GEOT_ERR_UNSUPPORTED;
        if (F % c.vec_elems) return GEOT_ERR_UNSUPPORTED;
        const int l = c.lanes_per_row;
        if (l < 1 || l > 32 || (l & (l - 1))) return GEOT_ERR_UNSUPPORTED;
        const int v = c.vecs_per_lane;
        if (!(v == 1 || (l == 32 && (v == 2 || v == 4 || (v == 8 && dt == GEOT_F32))))) return GEOT_ERR_UNSUPPORTED;
        if (c.rows_per_group < 1 || c.rows_per_group > 1024) return GEOT_ERR_UNSUPPORTED;
        if (c.ctas_per_sm < 0) return GEOT_ERR_INVALID_VALUE;
    }
    *out = c;
    return GEOT_OK;
}

static geot_status check_enums(geot_reduce op, geot_dtype dt, geot_itype it) {
    if ((int)op < 0 || (int)op > 2) return GEOT_ERR_INVALID_VALUE;
    if ((int)dt < 0 || (int)dt > 1) return GEOT_ERR_INVALID_VALUE;
    if ((int)it < 0 || (int)it > 1) return GEOT_ERR_INVALID_VALUE;
    return GEOT_OK;
}

typedef cudaError_t (*edge_launcher)(const EdgeTileParams&, int, int, int, bool, int, int, cudaStream_t, LaunchInfo*);

static edge_launcher pick_launcher(geot_dtype dt, int mode) {
    static const edge_launcher table[2][3] = {
        {launch_edge_tile_f32_plain, launch_edge_tile_f32_gather, launch_edge_tile_f32_gatherw},
        {launch_edge_tile_bf16_plain, launch_edge_tile_bf16_gather, launch_edge_tile_bf16_gatherw}};
    return table[dt][mode];
}

// The shared body of every reduction entry point.
static OutSet single_out(void* out, long long seg_base) {
    OutSet os{};
    os.ptr[0] = out;
    os.n = 1;
    os.row_off = seg_base;
    return os;
}

static geot_status reduce_common(const void* X, long long V, const void* src_idx, const void* idx, const float* w,
                                 long long nnz, long long seg_base, long long S, long long F, geot_reduce op,
                                 geot_dtype dt, geot_itype it, const OutSet& os, void* ws, size_t ws_bytes,
                                 const geot_config* user_cfg, cudaStream_t stream, int mode) {
    void* out = os.ptr[0];
    geot_status st = check_enums(op, dt, it);
    if (st != GEOT_OK) return st;
    if (nnz < 0 || S < 0 || F < 1 || V < 0) return GEOT_ERR_INVALID_VALUE;
    if (F > (1LL << 30) || nnz > (1LL << 47)) return GEOT_ERR_UNSUPPORTED;
    if (mode == 2 && op != GEOT_SUM) return GEOT_ERR_UNSUPPORTED;
    if (S == 0) return GEOT_OK;
    for (int d = 0; d < os.n; ++d)
        if (!os.ptr[d]) return GEOT_ERR_INVALID_VALUE;
    if (nnz > 0 && (!X || !idx || (mode >= 1 && !src_idx) || (mode == 2 && !w))) return GEOT_ERR_INVALID_VALUE;
    const size_t esz = dt == GEOT_F32 ? 4 : 2;
    if (nnz == 0) {  // every segment is empty
        const long long bytes = S * F * (long long)esz;
        const int blocks = (int)std::min<long long>((bytes / 16 + 255) / 256 + 1, (long long)sm_count() * 8);
        for (int d = 0; d < os.n; ++d) {
            unsigned char* o = static_cast<unsigned char*>(os.ptr[d]) + (seg_base - os.row_off) * F * (long long)esz;
            zero_fill_kernel<<<blocks, 256, 0, stream>>>(o, bytes);
            g_launches.fetch_add(1, std::memory_order_relaxed);
        }
        return from_cuda(cudaGetLastError());
    }
    geot_config c;
    st = resolve_config(nnz, S, F, op, dt, it, mode >= 1, user_cfg, &c);
    if (st != GEOT_OK) return st;
    // vector path needs 16-byte aligned row starts of the value/output arrays
    bool outs_aligned = true;
    for (int d = 0; d < os.n; ++d) outs_aligned = outs_aligned && aligned(os.ptr[d], 16);
    if ((c.vec_elems > 1 || c.variant == GEOT_VARIANT_STREAM) && !(aligned(X, 16) && outs_aligned)) {
        if (user_cfg && (user_cfg->vec_elems > 1 || user_cfg->variant == GEOT_VARIANT_STREAM))
            return GEOT_ERR_UNSUPPORTED;
        c.variant = GEOT_VARIANT_EDGE_TILE;
        c.vec_elems = 1;
        c.ctas_per_sm = 0;
        select_shape_for_vw(F, dt, &c);
    }
    unsigned char* wsb = static_cast<unsigned char*>(ws);
    if (c.variant == GEOT_VARIANT_NARROW) {
        // narrow rows are stored whole (F * esz = 4..32 bytes, a power of two):
        // every destination must be aligned to the row-store width
        bool outs_row_aligned = true;
        for (int d = 0; d < os.n; ++d)
            outs_row_aligned = outs_row_aligned && aligned(os.ptr[d], (size_t)std::min<long long>(16, F * (long long)esz));
        if (mode == 0 && aligned(X, 16) && aligned(idx, 16) && outs_row_aligned &&
            (it == GEOT_I64 || seg_base + S < (long long)INT_MAX)) {  // 32-bit key arithmetic
            const int nsm = sm_count();
            const WsLayout L = ws_layout(narrow_agents_max(nsm), F);
            if (!ws) return GEOT_ERR_INVALID_VALUE;
            if (ws_bytes < L.total) return GEOT_ERR_WORKSPACE_TOO_SMALL;
            NarrowParams np{};
            np.X = X;
            np.idx = idx;
            np.out = out;
            np.outs = os;
            np.carry_h = reinterpret_cast<float*>(wsb + L.carry_h);
            np.carry_t = reinterpret_cast<float*>(wsb + L.carry_t);
            np.meta = reinterpret_cast<TileMeta*>(wsb + L.meta);
            np.flag = reinterpret_cast<unsigned long long*>(wsb + L.flags);
            np.ctrl = reinterpret_cast<StreamCtrl*>(wsb + L.ctrl);
            np.E = nnz;
            np.seg_base = seg_base;
            np.S = S;
            np.op = (int)op;
            cudaError_t e = launch_narrow(np, (int)F, dt == GEOT_BF16, op == GEOT_MAX, it == GEOT_I64, nsm, stream);
            if (e != cudaErrorNotSupported) return from_cuda(e);
        } else if (user_cfg && user_cfg->variant == GEOT_VARIANT_NARROW) {
            return GEOT_ERR_UNSUPPORTED;
        }
        c.variant = GEOT_VARIANT_EDGE_TILE;  // not applicable here: edge-tile kernel
    }
    if (c.variant == GEOT_VARIANT_STREAM) {
        const int nsm = sm_count();
        // f4 replicas launch the lane shape's default pipeline (launch.cuh): size
        // the agents for that pipeline, not for the selected one
        if (os.n > 1 && mode == 0) stream_default_pipe(c.lanes_per_row, c.vecs_per_lane, &c.warps_per_cta,
                                                       &c.rows_per_group, &c.stages);
        long long NA =
            stream_agents(nnz, c.lanes_per_row, c.warps_per_cta, nsm, c.stages == 1 ? 2 : 1);  // LDG mode: 2 CTAs/SM
        if (c.lanes_per_row <= 8 && S >= 0xFFFFFFFFLL) NA = 0;  // small-row path: 32-bit relative keys
        if (NA > 0) {
            const WsLayout L = ws_layout(NA, F);
            if (L.total > 0) {
                if (!ws) return GEOT_ERR_INVALID_VALUE;
                if (ws_bytes < L.total) return GEOT_ERR_WORKSPACE_TOO_SMALL;
            }
            StreamParams sp{};
            sp.X = X;
            sp.idx = idx;
            sp.out = out;
            sp.outs = os;
            sp.meta = L.total ? reinterpret_cast<TileMeta*>(wsb + L.meta) : nullptr;
            sp.carry_h = L.total ? reinterpret_cast<float*>(wsb + L.carry_h) : nullptr;
            sp.carry_t = L.total ? reinterpret_cast<float*>(wsb + L.carry_t) : nullptr;
            sp.flag = reinterpret_cast<unsigned long long*>(wsb + L.flags);
            sp.ctrl = reinterpret_cast<StreamCtrl*>(wsb + L.ctrl);
            if (NA * 8 > (long long)ws_flag_bytes()) return GEOT_ERR_UNSUPPORTED;
            sp.E = nnz;
            sp.seg_base = seg_base;
            sp.S = S;
            sp.NA = NA;
            // L rows per agent, a multiple of RS (stream.cuh: agent ranges, 4+ agents per warp)
            sp.L = ((nnz + NA - 1) / NA + c.rows_per_group - 1) / c.rows_per_group * c.rows_per_group;
            sp.NF = nnz / sp.L;
            sp.F = (int)F;
            sp.NV = (int)(F / c.vec_elems);
            sp.RS = c.rows_per_group;
            sp.row_bytes = (int)(F * (long long)esz);
            sp.op = (int)op;
            sp.idx64 = it == GEOT_I64;
            sp.src = src_idx;
            sp.w = w;
            sp.V = V;
            EdgeTileParams fx{};
            fx.out = out;
            fx.outs = os;
            fx.meta = sp.meta;
            fx.carry_h = sp.carry_h;
            fx.carry_t = sp.carry_t;
            fx.E = nnz;
            fx.seg_base = seg_base;
            fx.S = S;
            fx.ntiles = NA;
            fx.F = (int)F;
            fx.op = (int)op;
            const int ns = c.stages == 1 ? 0 : c.stages;
            cudaError_t e;
            if (mode >= 1)
                e = dt == GEOT_F32 ? launch_stream_gather_f32(sp, fx, c.lanes_per_row, c.vecs_per_lane, c.warps_per_cta,
                                                              c.rows_per_group, ns, op == GEOT_MAX, mode, nsm, stream)
                                   : launch_stream_gather_bf16(sp, fx, c.lanes_per_row, c.vecs_per_lane, c.warps_per_cta,
                                                               c.rows_per_group, ns, op == GEOT_MAX, mode, nsm, stream);
            else
                e = dt == GEOT_F32
                                ? launch_stream_f32(sp, fx, c.vec_elems, c.lanes_per_row, c.vecs_per_lane, c.warps_per_cta,
                                                    c.rows_per_group, c.stages == 1 ? 0 : c.stages, op == GEOT_MAX, nsm, stream)
                                : launch_stream_bf16(sp, fx, c.vec_elems, c.lanes_per_row, c.vecs_per_lane, c.warps_per_cta,
                                                     c.rows_per_group, c.stages == 1 ? 0 : c.stages, op == GEOT_MAX, nsm, stream);
            if (e == cudaErrorNotSupported) return GEOT_ERR_UNSUPPORTED;
            return from_cuda(e);
        }
        // too few rows for one per agent: edge-tile kernel with its own shape
        c.variant = GEOT_VARIANT_EDGE_TILE;
        c.ctas_per_sm = 0;
        const int wide = dt == GEOT_F32 ? 4 : 8;
        c.vec_elems = (F % wide == 0) ? wide : 1;  // the edge-tile kernel's vector widths
        select_shape_for_vw(F, dt, &c);
    }
    // the NVLS form has no 2-byte multicast store: bf16 edge tiles write single elements
    if (os.mc && dt == GEOT_BF16) return GEOT_ERR_UNSUPPORTED;
    const long long ntiles = ntiles_of(nnz, c);
    const WsLayout L = ws_layout(ntiles, F);
    if (L.total > 0) {
        if (!ws) return GEOT_ERR_INVALID_VALUE;
        if (ws_bytes < L.total) return GEOT_ERR_WORKSPACE_TOO_SMALL;
    }
    EdgeTileParams p{};
    p.X = X;
    p.idx = idx;
    p.src = src_idx;
    p.w = w;
    p.out = out;
    p.outs = os;
    p.meta = L.total ? reinterpret_cast<TileMeta*>(wsb + L.meta) : nullptr;
    p.carry_h = L.total ? reinterpret_cast<float*>(wsb + L.carry_h) : nullptr;
    p.carry_t = L.total ? reinterpret_cast<float*>(wsb + L.carry_t) : nullptr;
    p.E = nnz;
    p.seg_base = seg_base;
    p.S = S;
    p.V = V;
    p.ntiles = ntiles;
    p.F = (int)F;
    p.NV = (int)(F / c.vec_elems);
    p.R = c.rows_per_group;
    p.tile_rows = (int)tile_rows_of(c);
    p.op = (int)op;
    p.idx64 = it == GEOT_I64;
    edge_launcher fn = pick_launcher(dt, mode);
    cudaError_t e = fn(p, c.vec_elems, c.lanes_per_row, c.vecs_per_lane, op == GEOT_MAX, c.ctas_per_sm,
                       sm_count(), stream, nullptr);
    if (e == cudaErrorNotSupported) return GEOT_ERR_UNSUPPORTED;
    return from_cuda(e);
}

}  // namespace geot

using namespace geot;

extern "C" {

const char* geot_status_string(geot_status s) {
    switch (s) {
        case GEOT_OK: return "GEOT_OK";
        case GEOT_ERR_INVALID_VALUE: return "GEOT_ERR_INVALID_VALUE: bad scalar argument or null pointer";
        case GEOT_ERR_UNSUPPORTED: return "GEOT_ERR_UNSUPPORTED: valid but unsupported combination";
        case GEOT_ERR_WORKSPACE_TOO_SMALL: return "GEOT_ERR_WORKSPACE_TOO_SMALL";
        case GEOT_ERR_UNSORTED_INDEX: return "GEOT_ERR_UNSORTED_INDEX";
        case GEOT_ERR_INDEX_OUT_OF_RANGE: return "GEOT_ERR_INDEX_OUT_OF_RANGE";
        case GEOT_ERR_SRC_OUT_OF_RANGE: return "GEOT_ERR_SRC_OUT_OF_RANGE";
        case GEOT_ERR_CUDA: return "GEOT_ERR_CUDA: CUDA runtime error";
    }
    return "GEOT_ERR_UNKNOWN";
}

int geot_abi_version(void) { return GEOT_ABI_VERSION; }

uint64_t geot_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

void geot_select_tree(double log2_nnz, double avg, double skew, double F, double dtype, double fused, double op,
                      int32_t out[4]) {
    int o[4];
    select_tree_raw(log2_nnz, avg, skew, F, dtype, fused, op, o);
    for (int i = 0; i < 4; ++i) out[i] = o[i];
}

const char* geot_selector_provenance(void) { return select_tree_provenance(); }

const char* geot_last_cuda_error(void) {
    return g_last_cuda_error == cudaSuccess ? "" : cudaGetErrorString(g_last_cuda_error);
}

void geot_profile_events(cudaEvent_t before, cudaEvent_t after) {
    g_prof_before = before;
    g_prof_after = after;
}

geot_status geot_select_config(int64_t nnz, int64_t num_segments, int64_t F, geot_reduce op, geot_dtype dtype,
                               geot_itype itype, int fused, geot_config* cfg_out) {
    if (!cfg_out) return GEOT_ERR_INVALID_VALUE;
    geot_status st = check_enums(op, dtype, itype);
    if (st != GEOT_OK) return st;
    if (nnz < 0 || num_segments < 0 || F < 1) return GEOT_ERR_INVALID_VALUE;
    return select_config_impl(nnz, num_segments, F, op, dtype, itype, fused, 0.0, cfg_out);
}

geot_status geot_select_hand_rules(int64_t nnz, int64_t num_segments, int64_t F, geot_dtype dtype, int fused,
                                  geot_config* cfg_out) {
    if (!cfg_out || (int)dtype < 0 || (int)dtype > 1 || nnz < 0 || num_segments < 0 || F < 1)
        return GEOT_ERR_INVALID_VALUE;
    return select_hand_rules(nnz, num_segments, F, dtype, fused, cfg_out);
}

geot_status geot_select_config_ex(int64_t nnz, int64_t num_segments, int64_t F, geot_reduce op, geot_dtype dtype,
                                  geot_itype itype, int fused, double skew, geot_config* cfg_out) {
    if (!cfg_out) return GEOT_ERR_INVALID_VALUE;
    geot_status st = check_enums(op, dtype, itype);
    if (st != GEOT_OK) return st;
    if (nnz < 0 || num_segments < 0 || F < 1 || !(skew == skew)) return GEOT_ERR_INVALID_VALUE;
    return select_config_impl(nnz, num_segments, F, op, dtype, itype, fused, skew, cfg_out);
}

size_t geot_workspace_size(int64_t nnz, int64_t num_segments, int64_t F, geot_reduce op, geot_dtype dtype,
                           geot_itype itype, int fused, const geot_config* cfg) {
    if (nnz <= 0 || num_segments <= 0 || F < 1) return 0;
    if (check_enums(op, dtype, itype) != GEOT_OK) return 0;
    geot_config c;
    if (resolve_config(nnz, num_segments, F, op, dtype, itype, fused, cfg, &c) != GEOT_OK) return 0;
    // the misaligned fallback (VW = 1) never uses more tiles than the chosen shape:
    // size for the larger of the two so either path fits.
    geot_config c1 = c;
    c1.vec_elems = 1;
    select_shape_for_vw(F, dtype, &c1);
    long long nt = ntiles_of(nnz, c1);
    if (c.variant == GEOT_VARIANT_STREAM) {
        geot_config c2 = c;
        select_shape_for_vw(F, dtype, &c2);  // its edge-tile fallback shape
        nt = std::max(nt, ntiles_of(nnz, c2));
        nt = std::max(nt, stream_agents(nnz, c.lanes_per_row, 16, sm_count(), 2));  // upper bound on agents
    } else if (c.variant == GEOT_VARIANT_NARROW) {
        geot_config c2 = c;
        select_shape_for_vw(F, dtype, &c2);  // its edge-tile fallback shape
        nt = std::max(nt, ntiles_of(nnz, c2));
        nt = std::max(nt, narrow_agents_max(sm_count()));
    } else {
        nt = std::max(nt, ntiles_of(nnz, c));
    }
    return ws_layout(nt, F).total;
}

geot_status geot_workspace_init(void* workspace, size_t ws_bytes, cudaStream_t stream) {
    if (ws_bytes == 0) return GEOT_OK;
    if (!workspace) return GEOT_ERR_INVALID_VALUE;
    return from_cuda(cudaMemsetAsync(workspace, 0, ws_bytes, stream));
}

geot_status geot_workspace_status(const void* workspace, size_t ws_bytes, cudaStream_t stream, int32_t* h_status) {
    if (!h_status) return GEOT_ERR_INVALID_VALUE;
    *h_status = 0;
    if (!workspace || ws_bytes < sizeof(StreamCtrl)) return GEOT_OK;  // no control words
    StreamCtrl c;
    cudaError_t e = cudaMemcpyAsync(&c, workspace, sizeof(c), cudaMemcpyDeviceToHost, stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
    if (e != cudaSuccess) return from_cuda(e);
    *h_status = (c.poison ? 1 : 0) | ((c.ticket != 0 || c.done != 0) ? 2 : 0);
    return GEOT_OK;
}

geot_status geot_segment_reduce(const void* src, const void* idx, int64_t nnz, int64_t num_segments, int64_t F,
                                geot_reduce op, geot_dtype dtype, geot_itype itype, void* out, void* workspace,
                                size_t ws_bytes, cudaStream_t stream) {
    return reduce_common(src, nnz, nullptr, idx, nullptr, nnz, 0, num_segments, F, op, dtype, itype,
                         single_out(out, 0), workspace, ws_bytes, nullptr, stream, 0);
}

geot_status geot_segment_reduce_ex(const void* src, const void* idx, int64_t nnz, int64_t seg_base,
                                   int64_t num_segments, int64_t F, geot_reduce op, geot_dtype dtype,
                                   geot_itype itype, void* out, void* workspace, size_t ws_bytes,
                                   const geot_config* cfg, cudaStream_t stream) {
    return reduce_common(src, nnz, nullptr, idx, nullptr, nnz, seg_base, num_segments, F, op, dtype, itype,
                         single_out(out, seg_base), workspace, ws_bytes, cfg, stream, 0);
}

geot_status geot_gather_segment_reduce(const void* x, int64_t num_x_rows, const void* src_idx, const void* dst_idx,
                                       int64_t nnz, int64_t num_segments, int64_t F, geot_reduce op,
                                       geot_dtype dtype, geot_itype itype, void* out, void* workspace,
                                       size_t ws_bytes, cudaStream_t stream) {
    return reduce_common(x, num_x_rows, src_idx, dst_idx, nullptr, nnz, 0, num_segments, F, op, dtype, itype,
                         single_out(out, 0), workspace, ws_bytes, nullptr, stream, 1);
}

geot_status geot_gather_weight_segment_reduce(const void* x, int64_t num_x_rows, const void* src_idx,
                                              const void* dst_idx, const float* weight, int64_t nnz,
                                              int64_t num_segments, int64_t F, geot_dtype dtype, geot_itype itype,
                                              void* out, void* workspace, size_t ws_bytes, cudaStream_t stream) {
    return reduce_common(x, num_x_rows, src_idx, dst_idx, weight, nnz, 0, num_segments, F, GEOT_SUM, dtype, itype,
                         single_out(out, 0), workspace, ws_bytes, nullptr, stream, 2);
}

geot_status geot_gather_segment_reduce_ex(const void* x, int64_t num_x_rows, const void* src_idx,
                                          const void* dst_idx, const float* weight, int64_t nnz, int64_t seg_base,
                                          int64_t num_segments, int64_t F, geot_reduce op, geot_dtype dtype,
                                          geot_itype itype, void* out, void* workspace, size_t ws_bytes,
                                          const geot_config* cfg, cudaStream_t stream) {
    return reduce_common(x, num_x_rows, src_idx, dst_idx, weight, nnz, seg_base, num_segments, F, op, dtype, itype,
                         single_out(out, seg_base), workspace, ws_bytes, cfg, stream, weight ? 2 : 1);
}

geot_status geot_segment_reduce_allgather(const void* src, const void* idx, int64_t nnz, int64_t seg_base,
                                          int64_t num_segments, int64_t F, geot_reduce op, geot_dtype dtype,
                                          geot_itype itype, void* const* outs, int nouts, void* workspace,
                                          size_t ws_bytes, const geot_config* cfg, cudaStream_t stream) {
    if (!outs || nouts < 1 || nouts > kMaxOuts || seg_base < 0) return GEOT_ERR_INVALID_VALUE;
    OutSet os{};
    for (int d = 0; d < nouts; ++d) os.ptr[d] = outs[d];
    os.n = nouts;
    os.row_off = 0;  // every replica holds the full output: rows are global segment ids
    return reduce_common(src, nnz, nullptr, idx, nullptr, nnz, seg_base, num_segments, F, op, dtype, itype, os,
                         workspace, ws_bytes, cfg, stream, 0);
}

geot_status geot_segment_reduce_multicast(const void* src, const void* idx, int64_t nnz, int64_t seg_base,
                                          int64_t num_segments, int64_t F, geot_reduce op, geot_dtype dtype,
                                          geot_itype itype, void* local_out, void* mc_out, void* workspace,
                                          size_t ws_bytes, const geot_config* cfg, cudaStream_t stream) {
    if (!local_out || !mc_out || seg_base < 0) return GEOT_ERR_INVALID_VALUE;
    if (check_enums(op, dtype, itype) != GEOT_OK) return GEOT_ERR_INVALID_VALUE;
    const int esz = dtype == GEOT_F32 ? 4 : 2;
    // multimem.st moves whole 4/8/16-byte words: rows of whole words, word-aligned buffers
    if ((F * esz) % 4 != 0 || (reinterpret_cast<uintptr_t>(local_out) | reinterpret_cast<uintptr_t>(mc_out)) % 16 != 0)
        return GEOT_ERR_UNSUPPORTED;
    OutSet os{};
    os.ptr[0] = local_out;
    os.ptr[1] = mc_out;
    os.n = 2;
    os.mc = 1;
    os.row_off = 0;  // full-output replicas: rows are global segment ids
    return reduce_common(src, nnz, nullptr, idx, nullptr, nnz, seg_base, num_segments, F, op, dtype, itype, os,
                         workspace, ws_bytes, cfg, stream, 0);
}

geot_status geot_segment_reduce_backward(const void* grad_out, const void* idx, int64_t nnz, int64_t num_segments,
                                         int64_t F, geot_reduce op, geot_dtype dtype, geot_itype itype,
                                         const int64_t* offsets, const void* src, const void* out, float* ties,
                                         void* grad_src, cudaStream_t stream) {
    geot_status st = check_enums(op, dtype, itype);
    if (st != GEOT_OK) return st;
    if (nnz < 0 || num_segments < 0 || F < 1) return GEOT_ERR_INVALID_VALUE;
    if (nnz == 0) return GEOT_OK;
    if (!grad_out || !idx || !grad_src) return GEOT_ERR_INVALID_VALUE;
    if (op == GEOT_MEAN && !offsets) return GEOT_ERR_INVALID_VALUE;
    if (op == GEOT_MAX && (!src || !out || !ties)) return GEOT_ERR_INVALID_VALUE;
    cudaError_t e = launch_segment_backward(grad_out, idx, itype == GEOT_I64, nnz, 0, num_segments, (int)F, (int)op,
                                            dtype == GEOT_BF16, reinterpret_cast<const long long*>(offsets), src, out,
                                            ties, grad_src, stream);
    if (e == cudaSuccess) g_launches.fetch_add(op == GEOT_MAX ? 2 : 1, std::memory_order_relaxed);
    return from_cuda(e);
}

geot_status geot_gather_segment_reduce_backward(const float* grad_out, const void* src_idx, const void* dst_idx,
                                                const float* weight, int64_t nnz, int64_t num_segments,
                                                int64_t num_x_rows, int64_t F, geot_reduce op, geot_itype itype,
                                                const int64_t* offsets, const float* x, float* grad_x, float* grad_w,
                                                cudaStream_t stream) {
    if ((int)itype < 0 || (int)itype > 1) return GEOT_ERR_INVALID_VALUE;
    if (op != GEOT_SUM && op != GEOT_MEAN) return GEOT_ERR_UNSUPPORTED;
    if (nnz < 0 || num_segments < 0 || num_x_rows < 0 || F < 1) return GEOT_ERR_INVALID_VALUE;
    if (op == GEOT_MEAN && !offsets) return GEOT_ERR_INVALID_VALUE;
    if (grad_w && !x) return GEOT_ERR_INVALID_VALUE;
    const long long* off = reinterpret_cast<const long long*>(offsets);
    if (grad_x) {
        if (!grad_out || (nnz > 0 && (!src_idx || !dst_idx))) return GEOT_ERR_INVALID_VALUE;
        cudaError_t e = launch_gather_backward_x(grad_out, src_idx, dst_idx, itype == GEOT_I64, weight, nnz, 0,
                                                 num_segments, num_x_rows, (int)F, (int)op, off, grad_x, stream);
        if (e != cudaSuccess) return from_cuda(e);
        g_launches.fetch_add(1, std::memory_order_relaxed);
    }
    if (grad_w && nnz > 0) {
        cudaError_t e = launch_sddmm(x, grad_out, src_idx, dst_idx, itype == GEOT_I64, nnz, 0, num_segments,
                                     num_x_rows, (int)F, (int)op, off, grad_w, stream);
        if (e != cudaSuccess) return from_cuda(e);
        g_launches.fetch_add(1, std::memory_order_relaxed);
    }
    return GEOT_OK;
}

geot_status geot_segment_offsets(const void* idx, geot_itype itype, int64_t nnz, int64_t num_segments,
                                 int64_t* offsets, cudaStream_t stream) {
    if ((int)itype < 0 || (int)itype > 1) return GEOT_ERR_INVALID_VALUE;
    if (nnz < 0 || num_segments < 0 || !offsets || (nnz > 0 && !idx)) return GEOT_ERR_INVALID_VALUE;
    const long long work = nnz + 1;
    const int blocks = (int)std::min<long long>((work + 255) / 256, (long long)sm_count() * 16);
    offsets_kernel<<<blocks, 256, 0, stream>>>(idx, itype == GEOT_I64, nnz, num_segments,
                                               reinterpret_cast<long long*>(offsets));
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return from_cuda(cudaGetLastError());
}

geot_status geot_validate_index(const void* idx, geot_itype itype, int64_t nnz, int64_t num_segments,
                                const void* src_idx, int64_t num_x_rows, int32_t* d_status, cudaStream_t stream) {
    if ((int)itype < 0 || (int)itype > 1) return GEOT_ERR_INVALID_VALUE;
    if (nnz < 0 || num_segments < 0 || num_x_rows < 0 || !d_status || (nnz > 0 && !idx)) return GEOT_ERR_INVALID_VALUE;
    cudaError_t e = cudaMemsetAsync(d_status, 0, sizeof(int32_t), stream);
    if (e != cudaSuccess) return GEOT_ERR_CUDA;
    if (nnz == 0) return GEOT_OK;
    const int blocks = (int)std::min<long long>((nnz + 255) / 256, (long long)sm_count() * 16);
    validate_kernel<<<blocks, 256, 0, stream>>>(idx, itype == GEOT_I64, nnz, num_segments, src_idx, num_x_rows,
                                                reinterpret_cast<int*>(d_status));
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return from_cuda(cudaGetLastError());
}

geot_status geot_partition(const void* idx, geot_itype itype, int64_t nnz, int64_t num_segments, int nparts,
                           int64_t* seg_bounds, int64_t* edge_bounds, cudaStream_t stream) {
    if ((int)itype < 0 || (int)itype > 1) return GEOT_ERR_INVALID_VALUE;
    if (nnz < 0 || num_segments < 0 || nparts < 1 || nparts > (1 << 20) || !seg_bounds || !edge_bounds ||
        (nnz > 0 && !idx))
        return GEOT_ERR_INVALID_VALUE;
    const int threads = 128;
    const int blocks = (nparts + 1 + threads - 1) / threads;
    partition_kernel<<<blocks, threads, 0, stream>>>(idx, itype == GEOT_I64, nnz, num_segments, nparts,
                                                     reinterpret_cast<long long*>(seg_bounds),
                                                     reinterpret_cast<long long*>(edge_bounds));
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return from_cuda(cudaGetLastError());
}

}  // extern "C"
