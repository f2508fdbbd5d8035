// Instantiations + launcher of the small-F kernel family (narrow.cuh).
#include "launch.cuh"
#include "narrow.cuh"

namespace geot {

// rows per lane: 32..64 value bytes per lane per chunk (2..16 rows)
__host__ __device__ constexpr int narrow_items(int F, int esz) {
    return (F * esz <= 8) ? 8 : ((F * esz <= 16) ? 4 : 2);
}

template <typename T, int F, bool ISMAX, bool I64>
static cudaError_t run_narrow(NarrowParams p, int nsm, cudaStream_t st) {
    constexpr int ITEMS = narrow_items(F, (int)sizeof(T));
    auto kern = narrow_kernel<T, F, ITEMS, ISMAX, I64>;
    int occ = cached_occupancy(kern, kNarrowWarps * 32, 0);
    if (occ <= 0) return cudaErrorInvalidConfiguration;
    // every agent (warp) must own at least one chunk of 32*ITEMS rows
    long long grid = (long long)nsm * occ;
    const long long max_agents = p.E / (32LL * ITEMS);
    if (grid * kNarrowWarps > max_agents) grid = max_agents / kNarrowWarps;
    if (grid < 1) return cudaErrorNotSupported;
    p.NA = grid * kNarrowWarps;
    if (g_prof_before) cudaEventRecord(g_prof_before, st);
    kern<<<(unsigned)grid, kNarrowWarps * 32, 0, st>>>(p);
    if (g_prof_after) cudaEventRecord(g_prof_after, st);
    g_prof_before = g_prof_after = nullptr;
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) g_launches.fetch_add(1, std::memory_order_relaxed);
    return e;
}

template <typename T>
static cudaError_t launch_narrow_t(const NarrowParams& p, int F, bool ismax, bool i64, int nsm, cudaStream_t st) {
#define GEOT_NSHAPE(F_)                                                                   \
    if (F == F_) {                                                                        \
        if (ismax)                                                                        \
            return i64 ? run_narrow<T, F_, true, true>(p, nsm, st) : run_narrow<T, F_, true, false>(p, nsm, st); \
        return i64 ? run_narrow<T, F_, false, true>(p, nsm, st) : run_narrow<T, F_, false, false>(p, nsm, st);  \
    }
    GEOT_NSHAPE(1)
    GEOT_NSHAPE(2)
    GEOT_NSHAPE(4)
    GEOT_NSHAPE(8)
    if constexpr (sizeof(T) == 2) {
        GEOT_NSHAPE(16)
    }
#undef GEOT_NSHAPE
    return cudaErrorNotSupported;
}

// Agents the launcher will use (carry slots); 0 = not applicable.
long long narrow_agents_max(int nsm) { return (long long)nsm * 8 * kNarrowWarps; }

cudaError_t launch_narrow(const NarrowParams& p, int F, bool bf16, bool ismax, bool i64, int nsm, cudaStream_t st) {
    return bf16 ? launch_narrow_t<__nv_bfloat16>(p, F, ismax, i64, nsm, st)
                : launch_narrow_t<float>(p, F, ismax, i64, nsm, st);
}

}  // namespace geot
