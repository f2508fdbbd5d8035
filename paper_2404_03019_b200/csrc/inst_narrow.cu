// Instantiations + launcher of the small-F kernel family (narrow.cuh): the
// two 2-D TMA tensor maps (values / keys viewed as rows of one lane's chunk
// bytes, swizzled to the lane-row width) are encoded here, per call.
#include <cuda.h>

#include <mutex>

#include "launch.cuh"
#include "narrow.cuh"

namespace geot {

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(f);
    });
    return fn;
}

bool encode_tensor_map(CUtensorMap* m, CUtensorMapDataType dt, int rank, const void* base, const cuuint64_t* dims,
                       const cuuint64_t* strides, const cuuint32_t* box, CUtensorMapSwizzle sw) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    const cuuint32_t estr[5] = {1u, 1u, 1u, 1u, 1u};
    return fn(m, dt, (cuuint32_t)rank, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
              sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// rows of LB bytes over [base, base + nrows*LB), box = `boxrows` rows, swizzle = LB
// (rows over 256 bytes: 4-byte elements, the box's inner extent is <= 256 elements)
static bool encode_rows(CUtensorMap* m, const void* base, long long nrows, int lb, int boxrows) {
    EncodeTiledFn fn = encode_fn();
    if (!fn || nrows < boxrows || nrows > 0x7fffffffLL || lb > 1024) return false;
    const int esz = lb > 256 ? 4 : 1;
    const cuuint64_t dims[2] = {(cuuint64_t)(lb / esz), (cuuint64_t)nrows};
    const cuuint64_t strides[1] = {(cuuint64_t)lb};
    const cuuint32_t box[2] = {(cuuint32_t)(lb / esz), (cuuint32_t)boxrows};
    const cuuint32_t estr[2] = {1u, 1u};
    const CUtensorMapSwizzle sw = lb == 128  ? CU_TENSOR_MAP_SWIZZLE_128B
                                  : lb == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                  : lb == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                             : CU_TENSOR_MAP_SWIZZLE_NONE;
    return fn(m, esz == 4 ? CU_TENSOR_MAP_DATA_TYPE_UINT32 : CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base),
              dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// rows of more than 32 bytes: LPR lane groups holding 16-byte slices, 8 (bf16: 4) rows per group
template <typename T, int F>
constexpr int narrow_lpr() { return F * (int)sizeof(T) > 32 ? F * (int)sizeof(T) / 16 : 1; }

template <typename T, int F, int OP, bool I64, bool REP>
static cudaError_t run_narrow_r(NarrowParams p, int nsm, cudaStream_t st) {
    constexpr int KSZ = I64 ? 8 : 4;
    constexpr int LPR = narrow_lpr<T, F>();
    constexpr int NG = 32 / LPR;
// F = 1 with int32 keys: 32 rows per lane (128-byte lane rows of values and of
// keys, 1 CTA of 8 warps per SM): half the per-row share of the chunk's fixed
// work (A/B on one box, sweep E = 2^24: fp32 power-law 42.0 -> 38.9 us, uniform
// 36.9 -> 34.9; bf16 45.1 -> 38.9 / 40.5 -> 34.8)
// F = 1 with int64 keys: 16 rows per lane (128-byte lane rows of keys; the
// generic rule caps keys at 64 bytes per lane): A/B on one box, E = 2^24 fp32
// power-law 55.0 -> 41.9 us, uniform 55.6 -> 43.3 us
#ifndef GEOT_NARROW_F1_I64_ITEMS
#define GEOT_NARROW_F1_I64_ITEMS 16
#endif
#ifndef GEOT_NARROW_F1_ITEMS
#define GEOT_NARROW_F1_ITEMS 32
#endif
    constexpr int ITEMS = LPR > 1 ? (sizeof(T) == 2 ? 4 : 8)
                                  : ((F == 1 && !I64) ? GEOT_NARROW_F1_ITEMS
                                     : (F == 1 && I64)  ? GEOT_NARROW_F1_I64_ITEMS
                                                        : narrow_items(F, (int)sizeof(T), KSZ));
    constexpr int LBG = ITEMS * F * (int)sizeof(T), LBK = ITEMS * KSZ;
#ifndef GEOT_NARROW_F1_WARPS
#define GEOT_NARROW_F1_WARPS 12
#endif
    // fp32 F = 1 at 32 rows per lane: the 8 KB stages hold one CTA per SM, so the
    // CTA takes 12 warps (192 KB ring, 156 registers): the kernel is latency-bound
    // (issue-active 49 % at 8 warps), A/B on one box: power-law 36.9 -> 35.2 us,
    // uniform 33.4 -> 33.1 (8 warps with a third stage instead: 37.0 -> 37.6)
    constexpr int NW = (F == 1 && sizeof(T) == 4 && ITEMS == 32 && LPR == 1) ? GEOT_NARROW_F1_WARPS : kNarrowWarps;
    auto kern = narrow_kernel<T, F, ITEMS, OP, I64, REP, LPR, NW>;
    const size_t smem = narrow_smem_bytes(LBG, LBK, NG, NW);
    int occ = cached_occupancy(kern, NW * 32, smem);
    if (occ <= 0) return cudaErrorInvalidConfiguration;
    // every agent (warp) must own at least one chunk of NG*ITEMS rows
    long long grid = (long long)nsm * occ;
    const long long max_agents = p.E / ((long long)NG * ITEMS);
    if (grid * NW > max_agents) grid = max_agents / NW;
    if (grid < 1) return cudaErrorNotSupported;
    p.NA = grid * NW;
    // whole lane rows only: the tail (< one lane row) is read directly
    CUtensorMap tmv, tmk;
    memset(&tmv, 0, sizeof(tmv));
    memset(&tmk, 0, sizeof(tmk));
    const long long nrows = p.E / ITEMS;
    p.tma = (LBG >= 16 && LBK >= 16 && encode_rows(&tmv, p.X, nrows, LBG, NG) && encode_rows(&tmk, p.idx, nrows, LBK, NG))
                ? 1
                : 0;
    if (g_prof_before) cudaEventRecord(g_prof_before, st);
    kern<<<(unsigned)grid, NW * 32, smem, st>>>(tmv, tmk, p);
    if (g_prof_after) cudaEventRecord(g_prof_after, st);
    g_prof_before = g_prof_after = nullptr;
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) g_launches.fetch_add(1, std::memory_order_relaxed);
    return e;
}

// f4 replicas (outs.n > 1) get their own instantiations, so the single-output
// kernel carries no per-store replica loop (a branch region per item at F = 1)
template <typename T, int F, int OP, bool I64>
static cudaError_t run_narrow(const NarrowParams& p, int nsm, cudaStream_t st) {
    return p.outs.n > 1 ? run_narrow_r<T, F, OP, I64, true>(p, nsm, st) : run_narrow_r<T, F, OP, I64, false>(p, nsm, st);
}

template <typename T, int F>
static cudaError_t run_narrow_f(const NarrowParams& p, int op, bool i64, int nsm, cudaStream_t st) {
    if (op == OP_MAX) return i64 ? run_narrow<T, F, OP_MAX, true>(p, nsm, st) : run_narrow<T, F, OP_MAX, false>(p, nsm, st);
    if (op == OP_MEAN)
        return i64 ? run_narrow<T, F, OP_MEAN, true>(p, nsm, st) : run_narrow<T, F, OP_MEAN, false>(p, nsm, st);
    return i64 ? run_narrow<T, F, OP_SUM, true>(p, nsm, st) : run_narrow<T, F, OP_SUM, false>(p, nsm, st);
}

template <typename T>
static cudaError_t launch_narrow_t(const NarrowParams& p, int F, bool i64, int nsm, cudaStream_t st) {
    switch (F) {
        case 1: return run_narrow_f<T, 1>(p, p.op, i64, nsm, st);
        case 2: return run_narrow_f<T, 2>(p, p.op, i64, nsm, st);
        case 4: return run_narrow_f<T, 4>(p, p.op, i64, nsm, st);
        case 8: return run_narrow_f<T, 8>(p, p.op, i64, nsm, st);
        case 16:  // fp32: 4 lanes per row; bf16: one lane per row
            return run_narrow_f<T, 16>(p, p.op, i64, nsm, st);
        case 32:  // 8 (fp32) / 4 (bf16) lanes per row
            return run_narrow_f<T, 32>(p, p.op, i64, nsm, st);
        case 64:  // bf16: 8 lanes per row
            if constexpr (sizeof(T) == 2) return run_narrow_f<T, 64>(p, p.op, i64, nsm, st);
            return cudaErrorNotSupported;
        default: return cudaErrorNotSupported;
    }
}

// Agents the launcher will use (carry slots); 0 = not applicable.
long long narrow_agents_max(int nsm) { return (long long)nsm * 8 * kNarrowWarps; }  // >= every NW * CTAs/SM

cudaError_t launch_narrow(const NarrowParams& p, int F, bool bf16, bool ismax, bool i64, int nsm, cudaStream_t st) {
    (void)ismax;  // p.op carries the op
    return bf16 ? launch_narrow_t<__nv_bfloat16>(p, F, i64, nsm, st) : launch_narrow_t<float>(p, F, i64, nsm, st);
}

}  // namespace geot
