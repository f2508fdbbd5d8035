// narrow.cuh — the small-F segment-reduction kernel (GEOT_VARIANT_NARROW):
// rows of 4..32 bytes (fp32 F in {1,2,4,8}, bf16 F in {1,2,4,8,16}).
//
// The paper's PR schedule (Alg. 1) and its F=1 weakness (P:407-422:
// cooperative-group overhead, lanes walking the M-loop uncoalesced) motivate
// this B200 design.  At F = 1 the whole budget is ~8 bytes of HBM per row, so
// the kernel is built around instruction count and bytes in flight:
//  * agents are whole warps with contiguous, ITEMS-aligned edge ranges
//    (balanced), one persistent grid, in-kernel carry resolution exactly as in
//    stream.cuh (ticketed CTAs, epoch-published agent carries);
//  * a warp processes chunks of 32*ITEMS rows; lane l owns ITEMS consecutive
//    rows.  A chunk's values and keys are two 2-D TMA tensor tiles (32 lane
//    rows of LB bytes each) landing in a per-warp NS-stage shared-memory ring
//    with the 32/64/128-byte swizzle, so that every lane reading its own LB
//    contiguous bytes with 128-bit LDS is bank-conflict free.  One elected lane
//    issues two TMA copies per chunk; nothing is double-buffered in registers;
//  * lane pass (SR within the lane): is_seg of every item (Alg. 1:
//    key != previous key) as one bit mask, then a predicated sequential
//    accumulation that restarts at heads.  Every segment that STARTS and ENDS
//    inside the lane is stored right there (predicated store, 32-bit keys and
//    address arithmetic for int32 indices);
//  * warp pass (the shfl doubling loop of Alg. 1): a segmented
//    inclusive scan of the lanes' tail partials with __shfl_up_sync, "a
//    segment starts in this lane" as the reset flag; it gives each lane the
//    carry of the segment that continues into it from the left, which the lane
//    folds into that segment's in-lane prefix (read back from a per-warp
//    shared-memory copy of the lane's partials: one dynamic index, no select
//    chain) and stores once where it ends.  A segment ending exactly at a
//    chunk boundary is stored by the next chunk's lane 0 (no look-ahead load);
//  * empty segments: a lane whose key span (last key - key before its first
//    row) differs from its number of segment heads has a gap (or unsorted
//    data) and zero-fills it (rare path, keys re-read from the ring).
#pragma once

#include <cuda.h>

#include "common.cuh"
#include "stream.cuh"

namespace geot {

struct NarrowParams {
    const void* X;
    const void* idx;
    void* out;      // == outs.ptr[0]
    OutSet outs;    // every destination of a finished row (f4)
    float* carry_h;
    float* carry_t;
    TileMeta* meta;
    unsigned long long* flag;
    StreamCtrl* ctrl;
    long long E, seg_base, S;
    long long NA;  // agents = warps of the grid
    int op;
    int tma;       // 1: full chunks come through the TMA ring (tensor maps valid)
};

constexpr int kNarrowWarps = 8;

// rows per lane per chunk: at most 128 value bytes, 64 key bytes, 32 fp32
// partials and 16 rows per lane (power of two)
__host__ __device__ constexpr int narrow_items(int F, int esz, int ksz) {
    int r = 16;
    while (r > 2 && (r * F * esz > 128 || r * ksz > 64 || r * F > 32)) r /= 2;
    return r;
}
// one ring area (values or keys tile of 32 lane rows), 1024-byte aligned (swizzle atom)
__host__ __device__ constexpr int narrow_area(int lb, int ng = 32) { return ((ng * lb + 1023) / 1024) * 1024; }
__host__ __device__ constexpr int narrow_stage_bytes(int lbv, int lbk, int ng = 32) {
    return narrow_area(lbv, ng) + narrow_area(lbk, ng);
}
// ring depth: 3 stages of <= 4 KB, else 2 (two 8-warp CTAs per SM fit either way;
// F = 1 at 32 rows per lane, 8 KB stages, 1 CTA/SM: a third stage measured
// 37.0 -> 37.6 us, the kernel is not bound by bytes in flight)
__host__ __device__ constexpr int narrow_stages(int lbv, int lbk, int ng = 32) {
    return narrow_stage_bytes(lbv, lbk, ng) <= 4096 ? 3 : 2;
}
__host__ __device__ constexpr size_t narrow_smem_bytes(int lbv, int lbk, int ng = 32, int nw = kNarrowWarps) {
    return (size_t)nw * narrow_stages(lbv, lbk, ng) * narrow_stage_bytes(lbv, lbk, ng)  // rings
           + (size_t)nw * narrow_stages(lbv, lbk, ng) * 8                              // mbarriers
           + 1024;                                                             // alignment slack
}

// physical offset of logical byte o of a tile written by TMA with the swizzle
// matching a lane row of LB bytes (16B chunk bits [4,4+b) ^= bits [7,7+b))
template <int LB>
__device__ __forceinline__ uint32_t swz(uint32_t o) {
    if constexpr (LB == 32) return o ^ (((o >> 7) & 1u) << 4);
    if constexpr (LB == 64) return o ^ (((o >> 7) & 3u) << 4);
    if constexpr (LB == 128) return o ^ (((o >> 7) & 7u) << 4);
    return o;
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar,
                                            uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

// 32-bit words of LB bytes of a lane row from the (swizzled) ring
template <int LB>
__device__ __forceinline__ void lds_row(uint32_t base, int lane, uint32_t (&w)[LB / 4]) {
    static_assert(LB % 8 == 0, "8-byte granularity");
    if constexpr (LB % 16 == 0) {
#pragma unroll
        for (int q = 0; q < LB / 16; ++q) {
            const uint4 v = lds_vec<uint4>(base + swz<LB>((uint32_t)(lane * LB + q * 16)));
            w[4 * q] = v.x;
            w[4 * q + 1] = v.y;
            w[4 * q + 2] = v.z;
            w[4 * q + 3] = v.w;
        }
    } else {  // LB == 8 (two int32 keys): unswizzled 8-byte rows
        uint32_t x, y;
        asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(x), "=r"(y) : "r"(base + lane * 8));
        w[0] = x;
        w[1] = y;
    }
}

template <typename T>
__device__ __forceinline__ float elem_from_words(const uint32_t* w, int i) {
    if constexpr (sizeof(T) == 4)
        return __uint_as_float(w[i]);
    else
        return __uint_as_float((i & 1) ? (w[i >> 1] & 0xFFFF0000u) : (w[i >> 1] << 16));
}

template <typename T>
__device__ __forceinline__ float ld_elem(const T* p) {
    if constexpr (sizeof(T) == 4)
        return __ldg(reinterpret_cast<const float*>(p));
    else
        return __uint_as_float((uint32_t)__ldg(reinterpret_cast<const unsigned short*>(p)) << 16);
}

// one output row of F elements from fp32 values (vector stores when they fit)
template <typename T, int F>
__device__ __forceinline__ void st_row(T* row, const float (&v)[F], bool mc = false) {
    // (mc: the multicast destination of the f4 NVLS form, multimem.st)
    if constexpr (sizeof(T) == 4) {
        if constexpr (F % 4 == 0) {
#pragma unroll
            for (int f = 0; f < F; f += 4)
                st_vec_mc(reinterpret_cast<uint4*>(row + f),
                          make_uint4(__float_as_uint(v[f]), __float_as_uint(v[f + 1]), __float_as_uint(v[f + 2]),
                                     __float_as_uint(v[f + 3])),
                          mc);
        } else if constexpr (F == 2) {
            st_vec_mc(reinterpret_cast<uint2*>(row), make_uint2(__float_as_uint(v[0]), __float_as_uint(v[1])), mc);
        } else {
            st_vec_mc(reinterpret_cast<uint32_t*>(row), __float_as_uint(v[0]), mc);
        }
    } else {
        if constexpr (F == 1) {
            *reinterpret_cast<uint16_t*>(row) = f2bf_bits(v[0]);  // (no multicast form: 2-byte rows)
        } else {
            uint32_t w[F / 2];
#pragma unroll
            for (int i = 0; i < F / 2; ++i)
                w[i] = (uint32_t)f2bf_bits(v[2 * i]) | ((uint32_t)f2bf_bits(v[2 * i + 1]) << 16);
            if constexpr (F == 2) {
                st_vec_mc(reinterpret_cast<uint32_t*>(row), w[0], mc);
            } else if constexpr (F == 4) {
                st_vec_mc(reinterpret_cast<uint2*>(row), make_uint2(w[0], w[1]), mc);
            } else {
#pragma unroll
                for (int i = 0; i < F / 2; i += 4)
                    st_vec_mc(reinterpret_cast<uint4*>(row + 2 * i), make_uint4(w[i], w[i + 1], w[i + 2], w[i + 3]), mc);
            }
        }
    }
}

template <int OP>
__device__ __forceinline__ float nfold(float a, float b) {
    return fold<OP == OP_MAX>(a, b);
}
template <int OP>
__device__ __forceinline__ float nident() {
    return identity<OP == OP_MAX>();
}

// The warp pass of Alg. 1 (the __shfl doubling loop): a segmented
// inclusive scan over the 32 lanes.  In: sv = the lane's value, sf = "a segment
// starts in this lane" (reset flag), spos = that start's position (mean only).
// Out: sv = fold of the values from the nearest lane <= this one whose flag is
// set (or from lane 0) through this lane; sf = whether such a lane exists;
// spos = its position.  log2(32) = 5 steps; lane l takes lane l-d's partial
// only while its own chain has not reached a segment start.  (Checked on every
// non-decreasing 8-key sequence and on random 16/32-lane sequences by
// geot_selftest_warp_segscan.)
template <int F, int OP, int LPR = 1>
__device__ __forceinline__ void warp_segscan(float (&sv)[F], bool& sf, long long& spos, int lane) {
#pragma unroll
    for (int d = LPR; d < 32; d <<= 1) {  // LPR lanes per row: a scan over the lane groups
        float ov[F];
#pragma unroll
        for (int f = 0; f < F; ++f) ov[f] = __shfl_up_sync(0xffffffffu, sv[f], d);
        const bool of = __shfl_up_sync(0xffffffffu, (int)sf, d) != 0;
        long long op_ = 0;
        if constexpr (OP == OP_MEAN) op_ = __shfl_up_sync(0xffffffffu, spos, d);
        if (lane >= d && !sf) {
#pragma unroll
            for (int f = 0; f < F; ++f) sv[f] = nfold<OP>(ov[f], sv[f]);
            sf = of;
            if constexpr (OP == OP_MEAN) spos = op_;
        }
    }
}

// LPR > 1 (rows of 64 / 128 bytes): a row is LPR 16-byte lane slices and the
// roles of a lane above are played by a group of LPR lanes: group g owns rows
// g*ITEMS .. of the chunk, each lane its slice of them; the warp pass scans the
// 32/LPR groups.  F is then the slice width (elements per lane), FR the row.
// CTAs per SM the kernel is compiled for: 2, or 1 when two rings do not fit
template <typename T, int FR, int ITEMS, bool I64, int LPR, int NW = kNarrowWarps>
__host__ __device__ constexpr int narrow_min_ctas() {
    return narrow_smem_bytes(ITEMS * FR * (int)sizeof(T), ITEMS * (I64 ? 8 : 4), 32 / LPR, NW) > 113 * 1024 ? 1 : 2;
}

// NW warps (agents) per CTA: 8, or 12 where one CTA per SM holds the ring anyway
template <typename T, int FR, int ITEMS, int OP, bool I64, bool REP = false, int LPR = 1, int NW = kNarrowWarps>
__global__ void __launch_bounds__(NW * 32, (narrow_min_ctas<T, FR, ITEMS, I64, LPR, NW>()))
    narrow_kernel(const __grid_constant__ CUtensorMap tmv, const __grid_constant__ CUtensorMap tmk,
                  const NarrowParams p) {
    static_assert(FR % LPR == 0 && 32 % LPR == 0, "lane groups");
    constexpr int F = FR / LPR;            // elements per lane of a row (a 16-byte slice when LPR > 1)
    constexpr int NG = 32 / LPR;           // lane groups (row owners) per warp
    constexpr int CH = NG * ITEMS;         // rows per chunk
    constexpr int ESZ = sizeof(T);
    constexpr int KSZ = I64 ? 8 : 4;
    constexpr int LBV = ITEMS * F * ESZ;   // value bytes per lane per chunk
    constexpr int LBG = ITEMS * FR * ESZ;  // value bytes per group per chunk (a TMA tile row)
    constexpr int LBK = ITEMS * KSZ;       // key bytes per group per chunk
    constexpr int VWORDS = LBV / 4, KWORDS = LBK / 4;
    constexpr int NS = narrow_stages(LBG, LBK, NG);
    constexpr int AREA_V = narrow_area(LBG, NG);
    constexpr int STAGE = narrow_stage_bytes(LBG, LBK, NG);
    static_assert(LPR == 1 || F * ESZ == 16, "lane groups hold 16-byte slices");
    using KT = typename std::conditional<I64, long long, int>::type;
    constexpr int RB = FR * ESZ;              // output row bytes
    constexpr int WROWS = STAGE / RB;         // output-window rows (a stage buffer; >= CH + 1)
    static_assert(WROWS >= CH + 1, "the output window must cover a chunk's rows");
    // window mode for rows of <= 8 bytes and fp32 F = 4 (A/B on the F = 1..8
    // sweep: F=1 power-law 59 -> 43 us, fp32 F=4 -2 %, bf16 F=8 +16 % -> off;
    // 32-byte rows: few segments per chunk, and the extra live row spills)
    constexpr bool WIN = RB <= 8 || (RB == 16 && ESZ == 4);

    extern __shared__ __align__(16) unsigned char smem_dyn[];
    // the swizzle pattern is a function of the shared address: 1024-byte align the rings
    unsigned char* smem_raw = smem_dyn + ((1024u - (smem_u32(smem_dyn) & 1023u)) & 1023u);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int grp = lane / LPR, li = lane % LPR;  // row-owner group, slice within the row
    const uint32_t ring = smem_u32(smem_raw) + (uint32_t)(warp * NS * STAGE);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + (size_t)NW * NS * STAGE) + warp * NS;

    const T* __restrict__ X = static_cast<const T*>(p.X);
    const KT* __restrict__ I = static_cast<const KT*>(p.idx);
    const long long seg_lo = p.seg_base, seg_hi = p.seg_base + p.S;
    // row of key seg_lo, this lane's slice
    T* __restrict__ out0 = static_cast<T*>(p.outs.ptr[0]) + (seg_lo - p.outs.row_off) * FR + li * F;
    const long long E = p.E;

    __shared__ unsigned s_ticket;
    __shared__ unsigned long long s_epoch;
    if (!draw_ticket(p.ctrl, &s_ticket, &s_epoch)) {  // poisoned workspace: retire (stream.cuh)
        retire_cta(p.ctrl);
        return;
    }
    const unsigned long long pub = s_epoch + 1;
    const long long a = (long long)s_ticket * NW + warp;
    auto agent_lo = [&](long long x) -> long long {
        if (x >= p.NA) return E;
        return ((x * E) / p.NA) / ITEMS * ITEMS;
    };
    const long long e_lo = agent_lo(a), e_hi = agent_lo(a + 1);
    const int nchunks = (int)((e_hi - e_lo + CH - 1) / CH);
    // every chunk comes through the TMA ring (rows past the tensor are zero-filled
    // by TMA; the global tail lane row, if partial, is read directly)
    const int nring = p.tma ? nchunks : 0;

    const uint64_t pol = policy_evict_first();
    if (lane == 0) {
        for (int s = 0; s < NS; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
    }
    __syncwarp();
    auto issue = [&](int s) {  // lane 0: chunk s into stage s % NS
        const int b = s % NS;
        const int row = (int)((e_lo + (long long)s * CH) / ITEMS);  // lane-row coordinate
        mbar_arrive_expect_tx(&bars[b], (uint32_t)NG * (LBG + LBK));
        tma_load_2d(ring + b * STAGE, &tmv, 0, row, &bars[b], pol);
        tma_load_2d(ring + b * STAGE + AREA_V, &tmk, 0, row, &bars[b], pol);
    };
    if (lane == 0)
        for (int s = 0; s < NS && s < nring; ++s) issue(s);

    auto key_at = [&](long long e) -> long long { return (long long)__ldg(I + e); };
    // zero rows strictly between keys lo_k and hi_k, clamped to [seg_lo, seg_hi)
    auto gap_fill = [&](long long lo_k, long long hi_k) {
        long long r0 = (lo_k < seg_lo) ? seg_lo : lo_k + 1;
        long long r1 = (hi_k > seg_hi) ? seg_hi : hi_k;
        float z[F];
#pragma unroll
        for (int f = 0; f < F; ++f) z[f] = 0.0f;
        if constexpr (REP) {
            for (int d = 0; d < p.outs.n; ++d)
                for (long long r = r0; r < r1; ++r)
                    st_row<T, F>(static_cast<T*>(p.outs.ptr[d]) + (r - p.outs.row_off) * FR + li * F, z,
                                 out_is_mc(p.outs, d));
        } else {
            for (long long r = r0; r < r1; ++r) st_row<T, F>(out0 + (r - seg_lo) * FR, z);
        }
    };
    // a store at key k (32-bit relative arithmetic for int32 keys; memory-safe)
    const KT kseg_lo = (KT)seg_lo;
    const unsigned long long nseg = (unsigned long long)p.S;
    auto store_at = [&](bool pred, KT k, const float (&v)[F], int count) {
        bool ok;
        unsigned long long rel;
        if constexpr (I64) {
            rel = (unsigned long long)(k - kseg_lo);
            ok = pred && rel < nseg;
        } else {
            const unsigned r32 = (unsigned)k - (unsigned)kseg_lo;  // wraps for keys < seg_lo
            ok = pred && r32 < (unsigned)nseg;                      // S < 2^31 on this path
            rel = r32;
        }
        float o[F];
#pragma unroll
        for (int f = 0; f < F; ++f) o[f] = (OP == OP_MEAN) ? __fdiv_rn(v[f], (float)count) : v[f];
        if (ok) {
            st_row<T, F>(out0 + rel * FR, o);
            if constexpr (REP)  // replicas (f4): global row index
                for (int d = 1; d < p.outs.n; ++d)
                    st_row<T, F>(static_cast<T*>(p.outs.ptr[d]) + ((long long)rel + seg_lo - p.outs.row_off) * FR + li * F,
                                 o, out_is_mc(p.outs, d));
        }
    };

    const bool active = e_lo < e_hi;
    const long long prevk = (active && e_lo > 0) ? key_at(e_lo - 1) : KEY_BEFORE;
    const long long nextk = (active && e_hi < E) ? key_at(e_hi) : KEY_AFTER;
    const long long first_key = active ? key_at(e_lo) : KEY_AFTER;
    const bool head_open = active && prevk == first_key;
    // virtual neighbours: the rows before the first / after the last edge carry
    // keys seg_lo-1 / seg_hi, so leading / trailing empty rows are ordinary gaps
    const KT kprev0 = (KT)((e_lo > 0) ? prevk : seg_lo - 1);
    const KT knext_end = (KT)((e_hi < E) ? nextk : seg_hi);

    // running segment across chunks (identical in every lane)
    float rc[F];  // value of the open segment (from its start, or from e_lo for the head segment)
#pragma unroll
    for (int f = 0; f < F; ++f) rc[f] = nident<OP>();
    KT rkey = kprev0;        // key of the last row before the current chunk
    long long rpos = 0;      // start row (relative to e_lo) of the open segment (mean counts)
    bool rhead = head_open;  // the open segment began in an earlier agent
    float hacc[F];           // this agent's partial of that head segment, once it ends here
#pragma unroll
    for (int f = 0; f < F; ++f) hacc[f] = nident<OP>();
    long long head_end = -1;

#pragma unroll 1
    for (int s = 0; s < nchunks; ++s) {
        const long long c0 = e_lo + (long long)s * CH;
        const long long r0 = c0 + (long long)grp * ITEMS;  // this lane's (group's) first row
        const bool last_chunk = s == nchunks - 1;  // warp-uniform
        const long long nvl = e_hi - r0;
        const int nv = nvl <= 0 ? 0 : (nvl >= ITEMS ? ITEMS : (int)nvl);  // valid items of the lane
        // a lane whose row is not in the ring: the global tail row, or no tensor maps
        const bool direct = !p.tma || (nv > 0 && r0 + ITEMS > E);
        float acc[ITEMS][F];
        KT k[ITEMS];
        const int b = s % NS;
        if (p.tma) {
            mbar_wait(&bars[b], (uint32_t)((s / NS) & 1));
            uint32_t vw[VWORDS], kw[KWORDS];
            if constexpr (LPR == 1) {
                lds_row<LBV>(ring + b * STAGE, lane, vw);
            } else {  // the lane's 16-byte slice of each of its group's rows
#pragma unroll
                for (int i = 0; i < ITEMS; ++i) {
                    const uint4 v = lds_vec<uint4>(ring + b * STAGE + swz<LBG>((uint32_t)(grp * LBG + i * RB + li * 16)));
                    vw[4 * i] = v.x;
                    vw[4 * i + 1] = v.y;
                    vw[4 * i + 2] = v.z;
                    vw[4 * i + 3] = v.w;
                }
            }
            lds_row<LBK>(ring + b * STAGE + AREA_V, grp, kw);
#pragma unroll
            for (int i = 0; i < ITEMS; ++i) {
#pragma unroll
                for (int f = 0; f < F; ++f) acc[i][f] = elem_from_words<T>(vw, i * F + f);
                if constexpr (I64)
                    k[i] = (long long)(((unsigned long long)kw[2 * i + 1] << 32) | kw[2 * i]);
                else
                    k[i] = (int)kw[i];
            }
        }
        if (__any_sync(0xffffffffu, direct)) {
            if (direct) {
#pragma unroll
                for (int i = 0; i < ITEMS; ++i) {
                    const bool ok = i < nv;
#pragma unroll
                    for (int f = 0; f < F; ++f) acc[i][f] = ok ? ld_elem<T>(X + (r0 + i) * FR + li * F + f) : 0.f;
                    k[i] = ok ? __ldg(I + r0 + i) : (KT)0;
                }
            }
        }
        if (last_chunk) {  // lanes past the agent's end: padding never starts a segment
            if (nv == 0) k[0] = 0;
#pragma unroll
            for (int i = 0; i < ITEMS; ++i) {
                if (i >= nv) {
                    if (i > 0) k[i] = k[i - 1];
#pragma unroll
                    for (int f = 0; f < F; ++f) acc[i][f] = nident<OP>();
                }
            }
        }
        // neighbours: the key before the lane's first row and after its last row
        // (lane 31 of a chunk that is not the agent's last: unknown -> "continues";
        // a segment ending there is stored by the next chunk's lane 0)
        KT kp = __shfl_up_sync(0xffffffffu, k[ITEMS - 1], LPR);
        if (grp == 0) kp = rkey;
        KT kn = __shfl_down_sync(0xffffffffu, k[0], LPR);
        if (grp == NG - 1) kn = k[ITEMS - 1];
        if (last_chunk && nv > 0 && r0 + nv >= e_hi) kn = knext_end;  // the agent's last row

        // ---- lane pass: heads (is_seg), sequential accumulation with restarts
        unsigned hm = (nv > 0 && k[0] != kp) ? 1u : 0u;
#pragma unroll
        for (int i = 1; i < ITEMS; ++i) hm |= (unsigned)(k[i] != k[i - 1]) << i;  // padding repeats the last key
#ifndef GEOT_NARROW_FMA_CHAIN
#define GEOT_NARROW_FMA_CHAIN 0
#endif
#pragma unroll
        for (int i = 1; i < ITEMS; ++i) {
            const bool h = (hm >> i) & 1u;
            if constexpr (OP != OP_MAX && GEOT_NARROW_FMA_CHAIN) {
                // the restart folded into the add: acc[i] = m * acc[i-1] + acc[i] with
                // m = 0 at a head, 1 elsewhere (fma(1, a, x) rounds exactly like a + x,
                // fma(0, a, x) = x for finite a) — ONE dependent instruction per item
                // on the lane's chain instead of an add and a select
                const float m = h ? 0.f : 1.f;
                if constexpr (F % 2 == 0) {
#pragma unroll
                    for (int f = 0; f < F; f += 2) {
                        const float2 t = __ffma2_rn(make_float2(m, m), make_float2(acc[i - 1][f], acc[i - 1][f + 1]),
                                                    make_float2(acc[i][f], acc[i][f + 1]));
                        acc[i][f] = t.x;
                        acc[i][f + 1] = t.y;
                    }
                } else {
#pragma unroll
                    for (int f = 0; f < F; ++f) acc[i][f] = __fmaf_rn(m, acc[i - 1][f], acc[i][f]);
                }
            } else if constexpr (OP != OP_MAX && F % 2 == 0) {  // packed fp32x2 adds (FADD2)
#pragma unroll
                for (int f = 0; f < F; f += 2) {
                    const float2 t = __fadd2_rn(make_float2(acc[i - 1][f], acc[i - 1][f + 1]),
                                                make_float2(acc[i][f], acc[i][f + 1]));
                    acc[i][f] = h ? acc[i][f] : t.x;
                    acc[i][f + 1] = h ? acc[i][f + 1] : t.y;
                }
            } else {
#pragma unroll
                for (int f = 0; f < F; ++f) acc[i][f] = h ? acc[i][f] : nfold<OP>(acc[i - 1][f], acc[i][f]);
            }
        }
        const KT klast = k[ITEMS - 1];  // padded: the last valid key
        const bool last_ends = nv > 0 && klast != kn;
        const unsigned em = (hm >> 1) | ((unsigned)last_ends << (nv > 0 ? nv - 1 : 0));  // items ending a segment
        // segments that start and end inside the lane
        const unsigned smk = em & ~((hm & (0u - hm)) - 1u);
        // the chunk's last valid row and its key (the running key of the next chunk)
        const unsigned vmask = __ballot_sync(0xffffffffu, nv > 0);
        const int ll = 31 - __clz(vmask);
        const KT kl = __shfl_sync(0xffffffffu, klast, ll);
        // Output window (warp-uniform choice): every row this chunk finalises
        // lies in [rkey, kl] — finished segments and the empty rows between
        // them.  When that span fits in the stage buffer the chunk writes its
        // finished rows into a zeroed shared-memory window (slot = key - rkey)
        // and copies the window out with coalesced stores: empty segments cost
        // nothing extra and no per-row global address is formed.  Otherwise
        // (very sparse keys, all-singleton chunks at F >= 2, unsorted data) the
        // rows are stored directly and gaps zero-filled lane by lane.
        const bool win = WIN && (unsigned long long)((long long)kl - (long long)rkey) < (unsigned long long)WROWS;
        T* const wrow = reinterpret_cast<T*>(smem_raw + (size_t)(warp * NS + b) * STAGE);  // window slot 0 = row rkey
        const int llg = ll / LPR;  // the chunk's last valid group
        const uint32_t wkey = (uint32_t)rkey;
        auto wput = [&](bool pred, KT key, const float (&v)[F], int count) {
            // clamped slot: memory-safe whatever the keys (the span test covers sorted data)
            uint32_t slot = (uint32_t)key - wkey;
            slot = slot < (uint32_t)WROWS ? slot : (uint32_t)(WROWS - 1);
            float o[F];
#pragma unroll
            for (int f = 0; f < F; ++f) o[f] = (OP == OP_MEAN) ? __fdiv_rn(v[f], (float)count) : v[f];
            if (pred) st_row<T, F>(wrow + (size_t)slot * FR + li * F, o);
        };
        bool wr_lo = false, wr_hi = false;  // this lane finalised row rkey / row kl (window mode)

        if (!win) {
#pragma unroll
            for (int i = 0; i < ITEMS; ++i) {
                int cnt = 1;
                if constexpr (OP == OP_MEAN) cnt = i + 1 - (31 - __clz(hm & ((2u << i) - 1u)));
                store_at((smk >> i) & 1u, k[i], acc[i], cnt);  // predicated, no branch
            }
        }
        // the running segment ended exactly at the previous chunk's end
        if (grp == 0 && s > 0 && (hm & 1u)) {
            if (rhead) {
#pragma unroll
                for (int f = 0; f < F; ++f) hacc[f] = rc[f];
                head_end = c0;
            } else if (!win) {
                store_at(true, rkey, rc, (int)((c0 - e_lo) - rpos));
            }
        }

        // gaps (empty segments) or unsorted keys outside window mode: a lane
        // whose key span differs from its number of heads.  Such a lane finds
        // its gap items from the keys in its registers (bit i: k[i] - k[i-1] > 1,
        // k[-1] = kp) and zero-fills each gap, reading the two keys of a gap back
        // from its ring slot (a dynamic item index; no local memory).
        if (!win) {
            const bool gap = nv > 0 && (long long)klast - (long long)kp != (long long)__popc(hm);
            if (__any_sync(0xffffffffu, gap) && gap) {
                unsigned gm = 0;
#pragma unroll
                for (int i = 0; i < ITEMS; ++i) {
                    const long long kq = i == 0 ? (long long)kp : (long long)k[i - 1];
                    gm |= (unsigned)(i < nv && (long long)k[i] - kq > 1) << i;
                }
                const uint32_t kb = ring + b * STAGE + AREA_V;
                auto key_item = [&](int i) -> long long {
                    if (direct) return key_at(r0 + i);
                    if constexpr (I64) {
                        unsigned long long t;
                        asm volatile("ld.shared.u64 %0, [%1];" : "=l"(t) : "r"(kb + swz<LBK>((uint32_t)(grp * LBK + i * 8))));
                        return (long long)t;
                    } else {
                        int t;
                        asm volatile("ld.shared.s32 %0, [%1];" : "=r"(t) : "r"(kb + swz<LBK>((uint32_t)(grp * LBK + i * 4))));
                        return t;
                    }
                };
                while (gm) {
                    const int i = __ffs(gm) - 1;
                    gm &= gm - 1;
                    gap_fill(i == 0 ? (long long)kp : key_item(i - 1), key_item(i));
                }
            }
        }

        // ---- warp pass: segmented inclusive scan of the lane tails (Alg. 1 analog)
        float sv[F];
#pragma unroll
        for (int f = 0; f < F; ++f) sv[f] = acc[ITEMS - 1][f];
        bool sf = hm != 0;  // a segment starts in this lane (reset flag)
        long long spos = hm ? (r0 - e_lo) + (31 - __clz(hm)) : 0;  // start row of the lane's tail segment
        warp_segscan<F, OP, LPR>(sv, sf, spos, lane);
        const bool reach = !sf;  // this lane's chain reaches back to the open segment
        if (reach) {
#pragma unroll
            for (int f = 0; f < F; ++f) sv[f] = nfold<OP>(rc[f], sv[f]);
            spos = rpos;
        }
        // carry into this lane: the previous lane's inclusive value
        float cin[F];
#pragma unroll
        for (int f = 0; f < F; ++f) cin[f] = __shfl_up_sync(0xffffffffu, sv[f], LPR);
        long long cpos = 0;
        if constexpr (OP == OP_MEAN) cpos = __shfl_up_sync(0xffffffffu, spos, LPR);
        bool creach = __shfl_up_sync(0xffffffffu, (int)reach, LPR) != 0;
        if (grp == 0) {
#pragma unroll
            for (int f = 0; f < F; ++f) cin[f] = rc[f];
            cpos = rpos;
            creach = true;
        }

        // ---- the segment continuing into the lane from the left: ends at item j
        const bool cont = nv > 0 && !(hm & 1u);
        const int j = hm ? (__ffs(hm) - 2) : (last_ends ? nv - 1 : -1);
        bool cput = false;  // window mode: this lane finalises row k[0] with ctot
        float ctot[F];
        int ccnt = 1;
        if (cont && j >= 0) {
            // the lane's partial at item j (a dynamic index)
            float tot[F];
            if constexpr (ESZ == 4) {
                // fp32: the lane's partials have exactly the shape of its value row,
                // whose ring slot it has already consumed: write them there (same
                // swizzled layout, conflict-free) and read item j back
                const uint32_t vb = ring + b * STAGE;
                // byte offset of the lane's element f of item i in the stage's value tile
                auto voff = [&](int i, int f) -> uint32_t {
                    if constexpr (LPR == 1)
                        return swz<LBV>((uint32_t)(lane * LBV + (i * F + f) * 4));
                    else
                        return swz<LBG>((uint32_t)(grp * LBG + i * RB + li * 16 + f * 4));
                };
#pragma unroll
                for (int q = 0; q < LBV / 16; ++q) {
                    const int e0 = 4 * q;  // the lane's elements e0 .. e0+3 (item e0 / F)
                    asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(vb + voff(e0 / F, e0 % F)),
                                 "f"(acc[(e0 + 0) / F][(e0 + 0) % F]), "f"(acc[(e0 + 1) / F][(e0 + 1) % F]),
                                 "f"(acc[(e0 + 2) / F][(e0 + 2) % F]), "f"(acc[(e0 + 3) / F][(e0 + 3) % F])
                                 : "memory");
                }
#pragma unroll
                for (int f = 0; f < F; ++f) {
                    float t;
                    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(t) : "r"(vb + voff(j, f)) : "memory");
                    tot[f] = nfold<OP>(cin[f], t);
                }
            } else {  // bf16: the partials are twice the row; select chain
#pragma unroll
                for (int f = 0; f < F; ++f) tot[f] = acc[0][f];
#pragma unroll
                for (int i = 1; i < ITEMS; ++i)
#pragma unroll
                    for (int f = 0; f < F; ++f) tot[f] = (i == j) ? acc[i][f] : tot[f];
#pragma unroll
                for (int f = 0; f < F; ++f) tot[f] = nfold<OP>(cin[f], tot[f]);
            }
            if (creach && rhead) {  // the agent's head segment: resolved below
#pragma unroll
                for (int f = 0; f < F; ++f) hacc[f] = tot[f];
                head_end = r0 + j + 1;
            } else if (!win) {
                store_at(true, k[0], tot, (int)((r0 - e_lo) + j + 1 - cpos));
            } else {
                cput = true;
#pragma unroll
                for (int f = 0; f < F; ++f) ctot[f] = tot[f];
                ccnt = (int)((r0 - e_lo) + j + 1 - cpos);
            }
        }

        if (win) {
            // rows finalised here: (rkey, kl) always; rkey if its segment (not the
            // agent's head) ended in this chunk; kl if its segment ended at the
            // agent's last row
            const bool put0 = grp == 0 && s > 0 && (hm & 1u) && !rhead;  // running segment, ended at c0
            wr_lo = put0 || (cput && k[0] == rkey);
            wr_hi = (cput && k[0] == kl) || (grp == llg && nv > 0 && ((smk >> (nv - 1)) & 1u));
            long long lo = (long long)rkey + (__any_sync(0xffffffffu, wr_lo) ? 0 : 1);
            long long hi = (long long)kl - (__any_sync(0xffffffffu, wr_hi) ? 0 : 1);
            if (lo < seg_lo) lo = seg_lo;
            if (hi > seg_hi - 1) hi = seg_hi - 1;
            using U = typename std::conditional<
                RB >= 16, uint4,
                typename std::conditional<RB == 8, uint2,
                                          typename std::conditional<RB == 4, uint32_t, uint16_t>::type>::type>::type;
            constexpr int UPR = RB / (int)sizeof(U);  // units per row
            const int nunits = hi >= lo ? (int)(hi - lo + 1) * UPR : 0;
            U* const wu = reinterpret_cast<U*>(wrow + (size_t)((uint32_t)lo - wkey) * FR);
            __syncwarp();  // every lane is done reading the stage (keys, values, partials)
            for (int u = lane; u < nunits; u += 32) wu[u] = U{};
            __syncwarp();
#pragma unroll
            for (int i = 0; i < ITEMS; ++i) {
                int cnt = 1;
                if constexpr (OP == OP_MEAN) cnt = i + 1 - (31 - __clz(hm & ((2u << i) - 1u)));
                wput((smk >> i) & 1u, k[i], acc[i], cnt);
            }
            if (put0) wput(true, rkey, rc, (int)((c0 - e_lo) - rpos));
            if (cput) wput(true, k[0], ctot, ccnt);
            __syncwarp();
            if constexpr (REP) {
                for (int d = 0; d < p.outs.n; ++d) {
                    U* const g = reinterpret_cast<U*>(static_cast<T*>(p.outs.ptr[d]) + (lo - p.outs.row_off) * FR);
                    const bool mc = out_is_mc(p.outs, d);
                    for (int u = lane; u < nunits; u += 32) st_vec_mc(g + u, wu[u], mc);
                }
            } else {
                U* const g = reinterpret_cast<U*>(out0 - li * F + (lo - seg_lo) * FR);
                for (int u = lane; u < nunits; u += 32) g[u] = wu[u];
            }
        }

        // ---- release the stage (all lanes are done with it) and refill it: the
        // proxy fence orders this chunk's shared-memory accesses before the refill
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0 && s + NS < nring) issue(s + NS);

        // ---- running segment for the next chunk: the last valid lane's state
#pragma unroll
        for (int f = 0; f < F; ++f) rc[f] = __shfl_sync(0xffffffffu, sv[f], llg * LPR + li);
        rkey = kl;
        if constexpr (OP == OP_MEAN) rpos = __shfl_sync(0xffffffffu, spos, ll);
        if (__any_sync(0xffffffffu, hm != 0)) rhead = false;
    }
    // owner-lane broadcast of the head partial (at most one lane set it)
    const unsigned hmk = __ballot_sync(0xffffffffu, head_end >= 0);
    if (hmk) {
        const int hl = __ffs(hmk) - 1;
#pragma unroll
        for (int f = 0; f < F; ++f) hacc[f] = __shfl_sync(0xffffffffu, hacc[f], (hl / LPR) * LPR + li);
        head_end = __shfl_sync(0xffffffffu, head_end, hl);
    }

    // ---- agent end: publish the open tail (H5), then resolve an owned head
    int flags = 0;
    if (active) {
        const bool tail_open = nextk == (long long)rkey;
        if (head_open) flags |= TM_HEAD_OPEN;
        if (e_hi == E && grp == 0 && (long long)rkey + 1 < seg_hi) gap_fill((long long)rkey, KEY_AFTER);
        if (tail_open) {
            flags |= TM_TAIL_OPEN;
            if (rhead) flags |= TM_MIDDLE;  // the whole range lies inside one segment
            if (grp == 0) {  // each lane of the first group writes its slice of the carry row
                float* c = (rhead ? p.carry_h : p.carry_t) + a * FR + li * F;
#pragma unroll
                for (int f = 0; f < F; ++f) c[f] = rc[f];
                if (lane == 0) {
                    p.meta[a].flags = flags;
                    p.meta[a].tail_start = e_lo + rpos;
                }
                __threadfence();
            }
            __syncwarp();
            if (lane == 0) st_release_u64(&p.flag[a], pub);
        }
    }
    __syncwarp();
    if (active && head_open && !(flags & TM_MIDDLE) && grp == 0) {
        long long u = a - 1;
        bool ok = true;
        for (; u >= 0; --u) {
            if (!wait_flag_or_poison(&p.flag[u], pub, p.ctrl)) {
                ok = false;
                break;
            }
            if (!(ld_volatile_i32(&p.meta[u].flags) & TM_MIDDLE)) break;
        }
        if (u < 0) u = 0;
        if (ok) {
            float tot[F];
#pragma unroll
            for (int f = 0; f < F; ++f) tot[f] = ld_cg_f32(p.carry_t + u * FR + li * F + f);
            for (long long m = u + 1; m < a; ++m)
#pragma unroll
                for (int f = 0; f < F; ++f) tot[f] = nfold<OP>(tot[f], ld_cg_f32(p.carry_h + m * FR + li * F + f));
#pragma unroll
            for (int f = 0; f < F; ++f) tot[f] = nfold<OP>(tot[f], hacc[f]);
            store_at(true, (KT)first_key, tot, (int)(head_end - ld_volatile_i64(&p.meta[u].tail_start)));
        }
    }
    retire_cta(p.ctrl);
}

}  // namespace geot
