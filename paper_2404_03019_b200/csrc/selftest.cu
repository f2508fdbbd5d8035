// selftest.cu — device self-test of the warp segmented scan that the narrow
// kernel's warp pass runs (narrow.cuh warp_segscan, the Alg. 1 doubling loop,
// P:199-205), exposed for the exhaustive test SPEC.md asks of the warp
// primitive (all 6,435 non-decreasing length-8 key sequences; S:457:
// random 16- and 32-lane cases).  Test hook only: nothing on the hot path
// calls it.
#include <cuda_runtime.h>

#include <atomic>

#include "../../include/geot.h"
#include "narrow.cuh"

namespace geot {

extern std::atomic<unsigned long long> g_launches;

namespace {

// One warp per 32 (key, value) items: lane l holds item l; a segment starts in
// lane l when l == 0 or its key differs from lane l-1's; the scan's inputs are
// exactly the narrow kernel's (sv = value, sf = start flag, spos = l if a
// segment starts here).
template <int OP>
__global__ void segscan_selftest_kernel(const int* __restrict__ keys, const float* __restrict__ vals, long long nwarps,
                                        float* out_v, int* out_sf, long long* out_pos) {
    const long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= nwarps) return;  // warp-uniform
    const long long i = w * 32 + lane;
    const int k = keys[i];
    const int kp = __shfl_up_sync(0xffffffffu, k, 1);
    bool sf = lane == 0 || k != kp;
    float sv[1] = {vals[i]};
    long long spos = sf ? lane : 0;
    warp_segscan<1, OP>(sv, sf, spos, lane);
    out_v[i] = sv[0];
    out_sf[i] = sf ? 1 : 0;
    out_pos[i] = spos;
}

}  // namespace
}  // namespace geot

using namespace geot;

extern "C" geot_status geot_selftest_warp_segscan(const int32_t* keys, const float* vals, int64_t nwarps, geot_reduce op,
                                                  float* out_vals, int32_t* out_flags, int64_t* out_pos,
                                                  cudaStream_t stream) {
    if (nwarps < 0 || (int)op < 0 || (int)op > 2) return GEOT_ERR_INVALID_VALUE;
    if (nwarps == 0) return GEOT_OK;
    if (!keys || !vals || !out_vals || !out_flags || !out_pos) return GEOT_ERR_INVALID_VALUE;
    const long long threads = nwarps * 32;
    const int blocks = (int)((threads + 255) / 256);
    long long* pos = reinterpret_cast<long long*>(out_pos);
    if (op == GEOT_MAX)
        segscan_selftest_kernel<OP_MAX><<<blocks, 256, 0, stream>>>(keys, vals, nwarps, out_vals, out_flags, pos);
    else if (op == GEOT_MEAN)
        segscan_selftest_kernel<OP_MEAN><<<blocks, 256, 0, stream>>>(keys, vals, nwarps, out_vals, out_flags, pos);
    else
        segscan_selftest_kernel<OP_SUM><<<blocks, 256, 0, stream>>>(keys, vals, nwarps, out_vals, out_flags, pos);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cudaGetLastError() == cudaSuccess ? GEOT_OK : GEOT_ERR_CUDA;
}
