// common.cuh — shared device helpers of libgeot (sm_100a).
// Vector I/O of fp32 / bf16 rows, index loads, op folding.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <climits>

namespace geot {

enum : int { OP_SUM = 0, OP_MEAN = 1, OP_MAX = 2 };

// Sentinel keys for the rows just outside [0, E): never equal to a real key.
constexpr long long KEY_BEFORE = LLONG_MIN;
constexpr long long KEY_AFTER = LLONG_MAX;

// ---------------------------------------------------------------- raw loads
// X rows are read exactly once: keep them out of L1 (streaming).  Node rows of
// the fused gather (x) are re-read by many edges: default read-only caching.
__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
    uint4 r;
    asm("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
        : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
        : "l"(p));
    return r;
}
__device__ __forceinline__ uint32_t ld_stream(const uint32_t* p) {
    uint32_t r;
    asm("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(p));
    return r;
}
__device__ __forceinline__ uint16_t ld_stream(const uint16_t* p) {
    uint16_t r;
    asm("ld.global.nc.L1::no_allocate.u16 %0, [%1];" : "=h"(r) : "l"(p));
    return r;
}
__device__ __forceinline__ uint4 ld_cached(const uint4* p) { return __ldg(p); }
__device__ __forceinline__ uint32_t ld_cached(const uint32_t* p) { return __ldg(p); }
__device__ __forceinline__ uint16_t ld_cached(const uint16_t* p) { return __ldg(p); }

__device__ __forceinline__ void st_vec(uint4* p, uint4 v) { *p = v; }
__device__ __forceinline__ void st_vec(uint32_t* p, uint32_t v) { *p = v; }
__device__ __forceinline__ void st_vec(uint16_t* p, uint16_t v) { *p = v; }

__device__ __forceinline__ long long load_index(const void* p, int idx64, long long i) {
    return idx64 ? __ldg(static_cast<const long long*>(p) + i)
                 : (long long)__ldg(static_cast<const int*>(p) + i);
}

__device__ __forceinline__ uint16_t f2bf_bits(float f) {
    __nv_bfloat16 b = __float2bfloat16_rn(f);  // round-to-nearest-even
    return *reinterpret_cast<uint16_t*>(&b);
}

// ------------------------------------------------------- typed vector views
// Conv<T, VW>: a vector of VW elements of T moved as one raw word.
template <typename T, int VW>
struct Conv;

template <>
struct Conv<float, 4> {
    using Raw = uint4;
    __device__ __forceinline__ static void unpack(const Raw& r, float (&f)[4]) {
        f[0] = __uint_as_float(r.x);
        f[1] = __uint_as_float(r.y);
        f[2] = __uint_as_float(r.z);
        f[3] = __uint_as_float(r.w);
    }
    __device__ __forceinline__ static Raw pack(const float (&f)[4]) {
        return make_uint4(__float_as_uint(f[0]), __float_as_uint(f[1]), __float_as_uint(f[2]),
                          __float_as_uint(f[3]));
    }
};
template <>
struct Conv<float, 1> {
    using Raw = uint32_t;
    __device__ __forceinline__ static void unpack(const Raw& r, float (&f)[1]) { f[0] = __uint_as_float(r); }
    __device__ __forceinline__ static Raw pack(const float (&f)[1]) { return __float_as_uint(f[0]); }
};
template <>
struct Conv<__nv_bfloat16, 8> {
    using Raw = uint4;
    __device__ __forceinline__ static void unpack(const Raw& r, float (&f)[8]) {
        const uint32_t w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            f[2 * i] = __uint_as_float(w[i] << 16);
            f[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
        }
    }
    __device__ __forceinline__ static Raw pack(const float (&f)[8]) {
        uint32_t w[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) w[i] = (uint32_t)f2bf_bits(f[2 * i]) | ((uint32_t)f2bf_bits(f[2 * i + 1]) << 16);
        return make_uint4(w[0], w[1], w[2], w[3]);
    }
};
template <>
struct Conv<__nv_bfloat16, 1> {
    using Raw = uint16_t;
    __device__ __forceinline__ static void unpack(const Raw& r, float (&f)[1]) {
        f[0] = __uint_as_float((uint32_t)r << 16);
    }
    __device__ __forceinline__ static Raw pack(const float (&f)[1]) { return f2bf_bits(f[0]); }
};

// Final value of an output element (H7): sum as accumulated; mean = one IEEE
// fp32 division by the count (never fast-math, reading R6); max as folded.
__device__ __forceinline__ float finalize(float acc, int op, long long count) {
    return op == OP_MEAN ? __fdiv_rn(acc, (float)count) : acc;
}

template <bool ISMAX>
__device__ __forceinline__ float fold(float a, float b) {
    if constexpr (ISMAX)
        return fmaxf(a, b);
    else
        return a + b;
}

template <bool ISMAX>
__device__ __forceinline__ float identity() {
    if constexpr (ISMAX)
        return __int_as_float(0xff800000);  // -inf
    else
        return 0.0f;
}

// Per-tile carry metadata written by the reduction kernel on EVERY call (so
// the workspace needs no initialisation) and read by the fix-up kernel.
struct TileMeta {
    long long head_key;    // key of the tile's first row
    long long head_end;    // one past the last row of the head segment (global)
    long long tail_start;  // first row of the tail segment (global), if carried
    int flags;             // TM_* bits
    int pad;
};
enum : int { TM_HEAD_OPEN = 1, TM_TAIL_OPEN = 2, TM_MIDDLE = 4 };

struct EdgeTileParams {
    const void* X;       // [E, F] values, or [V, F] node rows (fused)
    const void* idx;     // [E] sorted segment ids
    const void* src;     // [E] gather rows (fused), else null
    const float* w;      // [E] weights (weighted fused), else null
    void* out;           // [S, F]
    float* carry_h;      // [ntiles, F] tile-head partials
    float* carry_t;      // [ntiles, F] tile-tail partials
    TileMeta* meta;      // [ntiles]
    long long E, seg_base, S, V;
    long long ntiles;
    int F, NV;           // elements / vectors per row
    int R;               // rows per lane group
    int tile_rows;       // rows per tile
    int op;
    int idx64;
};

}  // namespace geot
