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
__device__ __forceinline__ uint2 ld_stream(const uint2* p) {
    uint2 r;
    asm("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
    return r;
}
__device__ __forceinline__ uint4 ld_cached(const uint4* p) { return __ldg(p); }
__device__ __forceinline__ uint2 ld_cached(const uint2* p) { return __ldg(p); }
__device__ __forceinline__ uint32_t ld_cached(const uint32_t* p) { return __ldg(p); }
__device__ __forceinline__ uint16_t ld_cached(const uint16_t* p) { return __ldg(p); }

__device__ __forceinline__ void st_vec(uint4* p, uint4 v) { *p = v; }
__device__ __forceinline__ void st_vec(uint2* p, uint2 v) { *p = v; }
__device__ __forceinline__ void st_vec(uint32_t* p, uint32_t v) { *p = v; }
__device__ __forceinline__ void st_vec(uint16_t* p, uint16_t v) { *p = v; }
// f4, NVLS form: a store through a multicast address (multimem.st; NVSwitch
// writes it into every replica bound to the multicast object).  4/8/16 bytes —
// the host rejects rows that are not whole 4-byte words for this form.
__device__ __forceinline__ void st_mc(uint4* p, uint4 v) {
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w)
                 : "memory");
}
__device__ __forceinline__ void st_mc(uint2* p, uint2 v) {
    asm volatile("multimem.st.relaxed.sys.global.v2.f32 [%0], {%1,%2};" ::"l"(p), "r"(v.x), "r"(v.y) : "memory");
}
__device__ __forceinline__ void st_mc(uint32_t* p, uint32_t v) {
    asm volatile("multimem.st.relaxed.sys.global.f32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_mc(uint16_t* p, uint16_t v) { *p = v; }  // unreachable (host check)
template <typename V>
__device__ __forceinline__ void st_vec_mc(V* p, V v, bool mc) {
    if (mc)
        st_mc(p, v);
    else
        st_vec(p, v);
}

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
struct Conv<float, 2> {
    using Raw = uint2;
    __device__ __forceinline__ static void unpack(const Raw& r, float (&f)[2]) {
        f[0] = __uint_as_float(r.x);
        f[1] = __uint_as_float(r.y);
    }
    __device__ __forceinline__ static Raw pack(const float (&f)[2]) {
        return make_uint2(__float_as_uint(f[0]), __float_as_uint(f[1]));
    }
};
template <>
struct Conv<__nv_bfloat16, 4> {
    using Raw = uint2;
    __device__ __forceinline__ static void unpack(const Raw& r, float (&f)[4]) {
        f[0] = __uint_as_float(r.x << 16);
        f[1] = __uint_as_float(r.x & 0xFFFF0000u);
        f[2] = __uint_as_float(r.y << 16);
        f[3] = __uint_as_float(r.y & 0xFFFF0000u);
    }
    __device__ __forceinline__ static Raw pack(const float (&f)[4]) {
        return make_uint2((uint32_t)f2bf_bits(f[0]) | ((uint32_t)f2bf_bits(f[1]) << 16),
                          (uint32_t)f2bf_bits(f[2]) | ((uint32_t)f2bf_bits(f[3]) << 16));
    }
};
template <>
struct Conv<__nv_bfloat16, 2> {
    using Raw = uint32_t;
    __device__ __forceinline__ static void unpack(const Raw& r, float (&f)[2]) {
        f[0] = __uint_as_float(r << 16);
        f[1] = __uint_as_float(r & 0xFFFF0000u);
    }
    __device__ __forceinline__ static Raw pack(const float (&f)[2]) {
        return (uint32_t)f2bf_bits(f[0]) | ((uint32_t)f2bf_bits(f[1]) << 16);
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

// ------------------------------------------------ mbarrier + TMA bulk copies
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
// TMA bulk copy global -> shared (1-D, 16-byte aligned, size % 16 == 0),
// completing `bytes` transactions on `bar`; X is streamed once: evict-first.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}
// ------------------------------------ inter-CTA publication (release/acquire)
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ int ld_volatile_i32(const int* p) { return *reinterpret_cast<const volatile int*>(p); }
__device__ __forceinline__ long long ld_volatile_i64(const long long* p) {
    return *reinterpret_cast<const volatile long long*>(p);
}
__device__ __forceinline__ float ld_cg_f32(const float* p) { return __ldcg(p); }  // L2, never a stale L1 line

// Ampere-style async copies of 4 / 8 bytes (keys) into shared memory, tracked
// by an mbarrier: the arrive fires when all of this thread's prior cp.async
// operations have completed (.noinc: counted in the barrier's init count).
__device__ __forceinline__ void cp_async_4(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_8(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// 16-byte shared-memory load from a 32-bit shared address (volatile: never
// hoisted above the mbarrier wait that publishes the data)
template <typename V>
__device__ __forceinline__ V lds_vec(uint32_t addr);
template <>
__device__ __forceinline__ uint4 lds_vec<uint4>(uint32_t addr) {
    uint4 r;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(addr));
    return r;
}
template <>
__device__ __forceinline__ uint2 lds_vec<uint2>(uint32_t addr) {
    uint2 r;
    asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "r"(addr));
    return r;
}
template <>
__device__ __forceinline__ uint32_t lds_vec<uint32_t>(uint32_t addr) {
    uint32_t r;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(r) : "r"(addr));
    return r;
}
template <>
__device__ __forceinline__ uint16_t lds_vec<uint16_t>(uint32_t addr) {
    uint16_t r;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(r) : "r"(addr));
    return r;
}

// Output destinations (f4, fused all-gather epilogue): every finished row
// `key` is stored to ptr[q] + (key - row_off) * F for q < n.  A plain call has
// n = 1, ptr[0] = out, row_off = seg_base; the all-gather form has one full
// [S_total, F] buffer per rank (peer / IPC-mapped pointers reached over
// NVLink) and row_off = 0, so each rank writes its rows into every replica.
constexpr int kMaxOuts = 8;
struct OutSet {
    void* ptr[kMaxOuts];
    int n;
    int mc;  // 1: ptr[1] is a multicast address (NVLS form): stores to it use multimem.st
    long long row_off;
};
// destination d of an OutSet: multimem.st for the multicast address
__device__ __forceinline__ bool out_is_mc(const OutSet& os, int d) { return os.mc && d == 1; }

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
    void* out;           // [S, F]  (== outs.ptr[0])
    OutSet outs;         // every destination of a finished row
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
