// backward.cu — gradients of the segment reductions (the paper
// leaves autograd as future work, naming SDDMM as the
// operation the fused form's backward needs).
//
//  * segment_reduce_backward:  dX[e,:] = g(e) * dY[idx[e]-seg_base, :]  where
//      sum : g = 1;  mean: g = 1/count[s];  max: g = [X[e,f] == Y[s,f]] / ties[s,f]
//    (ties split evenly — the convention of torch.scatter_reduce 'amax').
//    One thread per 16-byte output vector; rows of dY are re-read by every edge
//    of their segment (consecutive edges → L1/L2 hits).  Counts come from the
//    offsets (geot_segment_offsets); max ties from one extra pass.
//  * gather backward w.r.t. x (fused sum/mean, optional weights):
//      dx[src[e],:] += w[e] * g(e) * dY[dst[e],:]  — a scatter by the UNSORTED
//    source index: fp32 red.global.add (not bitwise reproducible; documented).
//  * SDDMM for the edge-weight gradient: dw[e] = <x[src[e],:], dY[dst[e],:]> (mean:
//    / count), one warp per edge, fp32 accumulation.
#include <cuda_runtime.h>

#include "common.cuh"

namespace geot {

template <typename T>
__device__ __forceinline__ float ldf(const T* p) {
    if constexpr (sizeof(T) == 4)
        return __ldg(reinterpret_cast<const float*>(p));
    else
        return __uint_as_float((uint32_t)__ldg(reinterpret_cast<const unsigned short*>(p)) << 16);
}
template <typename T>
__device__ __forceinline__ void stf(T* p, float v) {
    if constexpr (sizeof(T) == 4)
        *reinterpret_cast<float*>(p) = v;
    else
        *reinterpret_cast<uint16_t*>(p) = f2bf_bits(v);
}

// ties[s,f] = #{e in s : X[e,f] == Y[s,f]}  (max backward); ties must be zeroed
template <typename T>
__global__ void max_ties_kernel(const T* X, const T* Y, const void* idx, int idx64, long long E, long long seg_base,
                                long long S, int F, float* ties) {
    const long long n = E * (long long)F;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const long long e = i / F;
        const int f = (int)(i - e * F);
        const long long s = load_index(idx, idx64, e) - seg_base;
        if (s < 0 || s >= S) continue;
        if (ldf(X + i) == ldf(Y + s * F + f)) atomicAdd(ties + s * F + f, 1.0f);
    }
}

template <typename T>
__global__ void segment_backward_kernel(const T* dY, const void* idx, int idx64, long long E, long long seg_base,
                                        long long S, int F, int op, const long long* offsets, const T* X, const T* Y,
                                        const float* ties, T* dX) {
    const long long n = E * (long long)F;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const long long e = i / F;
        const int f = (int)(i - e * F);
        const long long s = load_index(idx, idx64, e) - seg_base;
        float g = 0.f;
        if (s >= 0 && s < S) {
            g = ldf(dY + s * F + f);
            if (op == OP_MEAN) {
                const long long c = offsets[s + 1] - offsets[s];
                g = c > 0 ? __fdiv_rn(g, (float)c) : 0.f;
            } else if (op == OP_MAX) {
                const float yv = ldf(Y + s * F + f);
                g = (ldf(X + i) == yv) ? __fdiv_rn(g, ties[s * F + f]) : 0.f;
            }
        }
        stf(dX + i, g);
    }
}

// dx must be zeroed; fp32 only
__global__ void gather_backward_x_kernel(const float* dY, const void* src, const void* dst, int idx64, const float* w,
                                         long long E, long long seg_base, long long S, long long V, int F, int op,
                                         const long long* offsets, float* dx) {
    const long long n = E * (long long)F;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const long long e = i / F;
        const int f = (int)(i - e * F);
        const long long s = load_index(dst, idx64, e) - seg_base;
        const long long r = load_index(src, idx64, e);
        if (s < 0 || s >= S || r < 0 || r >= V) continue;
        float g = __ldg(dY + s * F + f);
        if (w) g *= __ldg(w + e);
        if (op == OP_MEAN) {
            const long long c = offsets[s + 1] - offsets[s];
            g = __fdiv_rn(g, (float)c);
        }
        atomicAdd(dx + r * F + f, g);
    }
}

// dw[e] = sum_f x[src[e], f] * dY[dst[e], f]  (/ count for mean); one warp per edge
__global__ void sddmm_kernel(const float* x, const float* dY, const void* src, const void* dst, int idx64, long long E,
                             long long seg_base, long long S, long long V, int F, int op, const long long* offsets,
                             float* dw) {
    const int lane = threadIdx.x & 31;
    const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
    for (long long e = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); e < E; e += warps) {
        const long long s = load_index(dst, idx64, e) - seg_base;
        const long long r = load_index(src, idx64, e);
        float acc = 0.f;
        if (s >= 0 && s < S && r >= 0 && r < V)
            for (int f = lane; f < F; f += 32) acc = fmaf(__ldg(x + r * F + f), __ldg(dY + s * F + f), acc);
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) {
            if (op == OP_MEAN && s >= 0 && s < S) {
                const long long c = offsets[s + 1] - offsets[s];
                acc = __fdiv_rn(acc, (float)c);
            }
            dw[e] = acc;
        }
    }
}

static int grid_for(long long n) {
    long long b = (n + 255) / 256;
    if (b > 148LL * 16) b = 148LL * 16;
    return (int)(b < 1 ? 1 : b);
}

cudaError_t launch_segment_backward(const void* dY, const void* idx, int idx64, long long E, long long seg_base,
                                    long long S, int F, int op, int bf16, const long long* offsets, const void* X,
                                    const void* Y, float* ties, void* dX, cudaStream_t st) {
    const long long n = E * (long long)F;
    if (n == 0) return cudaSuccess;
    if (op == OP_MAX) {
        cudaError_t e = cudaMemsetAsync(ties, 0, sizeof(float) * (size_t)S * F, st);
        if (e != cudaSuccess) return e;
        if (bf16)
            max_ties_kernel<__nv_bfloat16><<<grid_for(n), 256, 0, st>>>(
                (const __nv_bfloat16*)X, (const __nv_bfloat16*)Y, idx, idx64, E, seg_base, S, F, ties);
        else
            max_ties_kernel<float><<<grid_for(n), 256, 0, st>>>((const float*)X, (const float*)Y, idx, idx64, E,
                                                                seg_base, S, F, ties);
    }
    if (bf16)
        segment_backward_kernel<__nv_bfloat16><<<grid_for(n), 256, 0, st>>>(
            (const __nv_bfloat16*)dY, idx, idx64, E, seg_base, S, F, op, offsets, (const __nv_bfloat16*)X,
            (const __nv_bfloat16*)Y, ties, (__nv_bfloat16*)dX);
    else
        segment_backward_kernel<float><<<grid_for(n), 256, 0, st>>>((const float*)dY, idx, idx64, E, seg_base, S, F,
                                                                    op, offsets, (const float*)X, (const float*)Y,
                                                                    ties, (float*)dX);
    return cudaGetLastError();
}

cudaError_t launch_gather_backward_x(const float* dY, const void* src, const void* dst, int idx64, const float* w,
                                     long long E, long long seg_base, long long S, long long V, int F, int op,
                                     const long long* offsets, float* dx, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(dx, 0, sizeof(float) * (size_t)V * F, st);
    if (e != cudaSuccess) return e;
    const long long n = E * (long long)F;
    if (n == 0) return cudaSuccess;
    gather_backward_x_kernel<<<grid_for(n), 256, 0, st>>>(dY, src, dst, idx64, w, E, seg_base, S, V, F, op, offsets,
                                                          dx);
    return cudaGetLastError();
}

cudaError_t launch_sddmm(const float* x, const float* dY, const void* src, const void* dst, int idx64, long long E,
                         long long seg_base, long long S, long long V, int F, int op, const long long* offsets,
                         float* dw, cudaStream_t st) {
    if (E == 0) return cudaSuccess;
    sddmm_kernel<<<grid_for(E * 32), 256, 0, st>>>(x, dY, src, dst, idx64, E, seg_base, S, V, F, op, offsets, dw);
    return cudaGetLastError();
}

}  // namespace geot
