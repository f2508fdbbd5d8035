// backward.cu — gradients of the segment reductions (the paper
// leaves autograd as future work, naming SDDMM as the
// operation the fused form's backward needs).
//
//  * segment_reduce_backward:  dX[e,:] = g(e) * dY[idx[e]-seg_base, :]  where
//      sum : g = 1;  mean: g = 1/count[s];  max: g = [X[e,f] == Y[s,f]] / ties[s,f]
//    (ties split evenly — the convention of torch.scatter_reduce 'amax').
//    Counts come from the offsets (geot_segment_offsets); max ties from one
//    extra pass.
//  * gather backward w.r.t. x (fused sum/mean, optional weights):
//      dx[src[e],:] += w[e] * g(e) * dY[dst[e],:]  — a scatter by the UNSORTED
//    source index: fp32 vector reductions (red.global.add.v4.f32); not bitwise
//    reproducible (documented, reading R20).
//  * SDDMM for the edge-weight gradient: dw[e] = <x[src[e],:], dY[dst[e],:]> (mean:
//    / count), fp32 accumulation.
//
// Layout of every kernel: a lane GROUP per row (LPR = pow2ceil(row vectors),
// at most 32 lanes), the group loads the row's index (and count / weight) once
// and its lanes walk the row's 16-byte vectors (4-byte scalars when the row is
// not a whole number of aligned vectors); rows are taken grid-stride.  No
// per-element index load or 64-bit division.  dX / dx are written (or reduced)
// once per element: the HBM-bound part; dY rows are re-read by every edge of
// their segment (consecutive edges: L1/L2 hits).
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

// VW elements (a 16-byte vector when VW = 16 / sizeof(T), else one scalar)
template <typename T, int VW>
struct Vec {
    float v[VW];
    __device__ __forceinline__ void load(const T* p) {
        if constexpr (VW == 1) {
            v[0] = ldf(p);
        } else {
            const uint4 r = __ldg(reinterpret_cast<const uint4*>(p));
            const uint32_t w[4] = {r.x, r.y, r.z, r.w};
            if constexpr (sizeof(T) == 4) {
#pragma unroll
                for (int q = 0; q < 4; ++q) v[q] = __uint_as_float(w[q]);
            } else {
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    v[2 * q] = __uint_as_float(w[q] << 16);
                    v[2 * q + 1] = __uint_as_float(w[q] & 0xFFFF0000u);
                }
            }
        }
    }
    __device__ __forceinline__ void store(T* p) const {
        if constexpr (VW == 1) {
            if constexpr (sizeof(T) == 4)
                *reinterpret_cast<float*>(p) = v[0];
            else
                *reinterpret_cast<uint16_t*>(p) = f2bf_bits(v[0]);
        } else if constexpr (sizeof(T) == 4) {
            *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
        } else {
            uint32_t w[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) w[q] = (uint32_t)f2bf_bits(v[2 * q]) | ((uint32_t)f2bf_bits(v[2 * q + 1]) << 16);
            *reinterpret_cast<uint4*>(p) = make_uint4(w[0], w[1], w[2], w[3]);
        }
    }
};

struct RowGrid {  // lane group of one row, grid-stride over rows
    int li, lpr;
    long long row0, rstride;
    __device__ __forceinline__ RowGrid(int lpr_) : lpr(lpr_) {
        const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
        li = (int)(tid % lpr_);
        row0 = tid / lpr_;
        rstride = (long long)gridDim.x * blockDim.x / lpr_;
    }
};

// ties[s,f] = #{e in s : X[e,f] == Y[s,f]}  (max backward); ties must be zeroed
template <typename T, int VW>
__global__ void max_ties_kernel(const T* X, const T* Y, const void* idx, int idx64, long long E, long long seg_base,
                                long long S, int F, int lpr, float* ties) {
    const RowGrid g(lpr);
    const int NV = F / VW;
    for (long long e = g.row0; e < E; e += g.rstride) {
        const long long s = load_index(idx, idx64, e) - seg_base;
        if (s < 0 || s >= S) continue;
        for (int v = g.li; v < NV; v += lpr) {
            Vec<T, VW> x, y;
            x.load(X + e * F + v * VW);
            y.load(Y + s * F + v * VW);
#pragma unroll
            for (int q = 0; q < VW; ++q)
                if (x.v[q] == y.v[q]) atomicAdd(ties + s * F + v * VW + q, 1.0f);
        }
    }
}

template <typename T, int VW, int OP>
__global__ void segment_backward_kernel(const T* dY, const void* idx, int idx64, long long E, long long seg_base,
                                        long long S, int F, int lpr, const long long* offsets, const T* X, const T* Y,
                                        const float* ties, T* dX) {
    const RowGrid g(lpr);
    const int NV = F / VW;
    for (long long e = g.row0; e < E; e += g.rstride) {
        const long long s = load_index(idx, idx64, e) - seg_base;
        const bool ok = s >= 0 && s < S;
        float cnt = 1.f;
        if constexpr (OP == OP_MEAN)
            if (ok) cnt = (float)(offsets[s + 1] - offsets[s]);
        for (int v = g.li; v < NV; v += lpr) {
            Vec<T, VW> o;
            if (ok) {
                o.load(dY + s * F + v * VW);
                if constexpr (OP == OP_MEAN) {
#pragma unroll
                    for (int q = 0; q < VW; ++q) o.v[q] = __fdiv_rn(o.v[q], cnt);  // cnt >= 1: e is in s
                } else if constexpr (OP == OP_MAX) {
                    Vec<T, VW> x, y;
                    x.load(X + e * F + v * VW);
                    y.load(Y + s * F + v * VW);
#pragma unroll
                    for (int q = 0; q < VW; ++q)
                        o.v[q] = (x.v[q] == y.v[q]) ? __fdiv_rn(o.v[q], __ldg(ties + s * F + v * VW + q)) : 0.f;
                }
            } else {
#pragma unroll
                for (int q = 0; q < VW; ++q) o.v[q] = 0.f;
            }
            o.store(dX + e * F + v * VW);
        }
    }
}

__device__ __forceinline__ void red_add_v4(float* p, float a, float b, float c, float d) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d)
                 : "memory");
}

// dx must be zeroed; fp32 only
template <int VW, int OP>
__global__ void gather_backward_x_kernel(const float* dY, const void* src, const void* dst, int idx64, const float* w,
                                         long long E, long long seg_base, long long S, long long V, int F, int lpr,
                                         const long long* offsets, float* dx) {
    const RowGrid g(lpr);
    const int NV = F / VW;
    for (long long e = g.row0; e < E; e += g.rstride) {
        const long long s = load_index(dst, idx64, e) - seg_base;
        const long long r = load_index(src, idx64, e);
        if (s < 0 || s >= S || r < 0 || r >= V) continue;
        float scale = w ? __ldg(w + e) : 1.f;
        float cnt = 1.f;
        if constexpr (OP == OP_MEAN) cnt = (float)(offsets[s + 1] - offsets[s]);
        for (int v = g.li; v < NV; v += lpr) {
            Vec<float, VW> d;
            d.load(dY + s * F + v * VW);
#pragma unroll
            for (int q = 0; q < VW; ++q) {
                d.v[q] *= scale;
                if constexpr (OP == OP_MEAN) d.v[q] = __fdiv_rn(d.v[q], cnt);
            }
            float* p = dx + r * F + v * VW;
            if constexpr (VW == 4)
                red_add_v4(p, d.v[0], d.v[1], d.v[2], d.v[3]);
            else
                atomicAdd(p, d.v[0]);
        }
    }
}

// dw[e] = sum_f x[src[e], f] * dY[dst[e], f]  (/ count for mean); a lane group per edge
template <int VW, int OP>
__global__ void sddmm_kernel(const float* x, const float* dY, const void* src, const void* dst, int idx64, long long E,
                             long long seg_base, long long S, long long V, int F, int lpr, const long long* offsets,
                             float* dw) {
    const RowGrid g(lpr);
    const int NV = F / VW;
    const int lane = threadIdx.x & 31;
    const unsigned gmask = lpr == 32 ? 0xffffffffu : (((1u << lpr) - 1u) << (lane & ~(lpr - 1)));
    // the row (edge) is uniform within a group, so the group's shuffles below
    // always see all of its lanes
    for (long long e = g.row0; e < E; e += g.rstride) {
        const long long s = load_index(dst, idx64, e) - seg_base;
        const long long r = load_index(src, idx64, e);
        const bool ok = s >= 0 && s < S && r >= 0 && r < V;
        float acc = 0.f;
        if (ok)
            for (int v = g.li; v < NV; v += lpr) {
                Vec<float, VW> a, b;
                a.load(x + r * F + v * VW);
                b.load(dY + s * F + v * VW);
#pragma unroll
                for (int q = 0; q < VW; ++q) acc = fmaf(a.v[q], b.v[q], acc);
            }
        for (int o = lpr >> 1; o; o >>= 1) acc += __shfl_xor_sync(gmask, acc, o);
        if (g.li == 0) {
            if (OP == OP_MEAN && s >= 0 && s < S) acc = __fdiv_rn(acc, (float)(offsets[s + 1] - offsets[s]));
            dw[e] = acc;
        }
    }
}

static int pow2ceil_i(int x) {
    int p = 1;
    while (p < x) p <<= 1;
    return p;
}
// lanes per row: the row's vectors, rounded up to a power of two, <= 32
static int lanes_for(int nv) { return nv >= 32 ? 32 : pow2ceil_i(nv < 1 ? 1 : nv); }
// grid: enough threads for every row once, capped at 148 SMs x 8 CTAs of 256 threads
static int grid_rows(long long rows, int lpr) {
    long long b = (rows * lpr + 255) / 256;
    if (b > 148LL * 8) b = 148LL * 8;
    return (int)(b < 1 ? 1 : b);
}
static bool al16(const void* p) { return p == nullptr || (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

template <typename T, int VW>
static cudaError_t seg_bwd(const void* dY, const void* idx, int idx64, long long E, long long seg_base, long long S,
                           int F, int op, const long long* offsets, const void* X, const void* Y, float* ties, void* dX,
                           cudaStream_t st) {
    const int lpr = lanes_for(F / VW);
    const int grid = grid_rows(E, lpr);
    if (op == OP_MAX) {
        cudaError_t e = cudaMemsetAsync(ties, 0, sizeof(float) * (size_t)S * F, st);
        if (e != cudaSuccess) return e;
        max_ties_kernel<T, VW><<<grid, 256, 0, st>>>((const T*)X, (const T*)Y, idx, idx64, E, seg_base, S, F, lpr, ties);
        segment_backward_kernel<T, VW, OP_MAX><<<grid, 256, 0, st>>>((const T*)dY, idx, idx64, E, seg_base, S, F, lpr,
                                                                      offsets, (const T*)X, (const T*)Y, ties, (T*)dX);
    } else if (op == OP_MEAN) {
        segment_backward_kernel<T, VW, OP_MEAN><<<grid, 256, 0, st>>>((const T*)dY, idx, idx64, E, seg_base, S, F, lpr,
                                                                       offsets, nullptr, nullptr, nullptr, (T*)dX);
    } else {
        segment_backward_kernel<T, VW, OP_SUM><<<grid, 256, 0, st>>>((const T*)dY, idx, idx64, E, seg_base, S, F, lpr,
                                                                      offsets, nullptr, nullptr, nullptr, (T*)dX);
    }
    return cudaGetLastError();
}

cudaError_t launch_segment_backward(const void* dY, const void* idx, int idx64, long long E, long long seg_base,
                                    long long S, int F, int op, int bf16, const long long* offsets, const void* X,
                                    const void* Y, float* ties, void* dX, cudaStream_t st) {
    if (E == 0 || F == 0) return cudaSuccess;
    const int wide = bf16 ? 8 : 4;
    const bool vec = F % wide == 0 && al16(dY) && al16(dX) && (op != OP_MAX || (al16(X) && al16(Y)));
    if (bf16)
        return vec ? seg_bwd<__nv_bfloat16, 8>(dY, idx, idx64, E, seg_base, S, F, op, offsets, X, Y, ties, dX, st)
                   : seg_bwd<__nv_bfloat16, 1>(dY, idx, idx64, E, seg_base, S, F, op, offsets, X, Y, ties, dX, st);
    return vec ? seg_bwd<float, 4>(dY, idx, idx64, E, seg_base, S, F, op, offsets, X, Y, ties, dX, st)
               : seg_bwd<float, 1>(dY, idx, idx64, E, seg_base, S, F, op, offsets, X, Y, ties, dX, st);
}

cudaError_t launch_gather_backward_x(const float* dY, const void* src, const void* dst, int idx64, const float* w,
                                     long long E, long long seg_base, long long S, long long V, int F, int op,
                                     const long long* offsets, float* dx, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(dx, 0, sizeof(float) * (size_t)V * F, st);
    if (e != cudaSuccess) return e;
    if (E == 0 || F == 0) return cudaSuccess;
    const bool vec = F % 4 == 0 && al16(dY) && al16(dx);
    const int lpr = lanes_for(vec ? F / 4 : F);
    const int grid = grid_rows(E, lpr);
#define GEOT_GBX(VW_, OP_)                                                                                      \
    gather_backward_x_kernel<VW_, OP_><<<grid, 256, 0, st>>>(dY, src, dst, idx64, w, E, seg_base, S, V, F, lpr, \
                                                              offsets, dx)
    if (vec) {
        if (op == OP_MEAN) GEOT_GBX(4, OP_MEAN); else GEOT_GBX(4, OP_SUM);
    } else {
        if (op == OP_MEAN) GEOT_GBX(1, OP_MEAN); else GEOT_GBX(1, OP_SUM);
    }
#undef GEOT_GBX
    return cudaGetLastError();
}

cudaError_t launch_sddmm(const float* x, const float* dY, const void* src, const void* dst, int idx64, long long E,
                         long long seg_base, long long S, long long V, int F, int op, const long long* offsets,
                         float* dw, cudaStream_t st) {
    if (E == 0) return cudaSuccess;
    const bool vec = F % 4 == 0 && al16(x) && al16(dY);
    const int lpr = lanes_for(vec ? F / 4 : F);
    const int grid = grid_rows(E, lpr);
#define GEOT_SDDMM(VW_, OP_)                                                                                        \
    sddmm_kernel<VW_, OP_><<<grid, 256, 0, st>>>(x, dY, src, dst, idx64, E, seg_base, S, V, F, lpr, offsets, dw)
    if (vec) {
        if (op == OP_MEAN) GEOT_SDDMM(4, OP_MEAN); else GEOT_SDDMM(4, OP_SUM);
    } else {
        if (op == OP_MEAN) GEOT_SDDMM(1, OP_MEAN); else GEOT_SDDMM(1, OP_SUM);
    }
#undef GEOT_SDDMM
    return cudaGetLastError();
}

}  // namespace geot
