// Instantiations + launcher of the small-F kernel family (narrow.cuh).
#include "launch.cuh"
#include "narrow.cuh"

namespace geot {

template <typename T, int F, int OP, bool I64>
static cudaError_t run_narrow(NarrowParams p, int nsm, cudaStream_t st) {
    constexpr int ITEMS = narrow_items(F, (int)sizeof(T), I64 ? 8 : 4);
    auto kern = narrow_kernel<T, F, ITEMS, OP, I64>;
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
        case 16:
            if constexpr (sizeof(T) == 2) return run_narrow_f<T, 16>(p, p.op, i64, nsm, st);
            return cudaErrorNotSupported;
        default: return cudaErrorNotSupported;
    }
}

// Agents the launcher will use (carry slots); 0 = not applicable.
long long narrow_agents_max(int nsm) { return (long long)nsm * 8 * kNarrowWarps; }

cudaError_t launch_narrow(const NarrowParams& p, int F, bool bf16, bool ismax, bool i64, int nsm, cudaStream_t st) {
    (void)ismax;  // p.op carries the op
    return bf16 ? launch_narrow_t<__nv_bfloat16>(p, F, i64, nsm, st) : launch_narrow_t<float>(p, F, i64, nsm, st);
}

}  // namespace geot
