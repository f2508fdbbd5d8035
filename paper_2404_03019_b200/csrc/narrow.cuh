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
//    rows (64 bytes of values), fetched with 128-bit loads of values and keys
//    one chunk ahead (register double buffer; the lane-contiguous 16-byte
//    pieces of one sector are merged in L1, so DRAM sees every byte once);
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
//    chain) and stores once where it ends;
//  * empty segments: a lane whose key span (last key - key before its first
//    row) differs from its number of segment heads has a gap (or unsorted
//    data) and zero-fills it item by item (rare path).
#pragma once

#include "common.cuh"
#include "stream.cuh"

namespace geot {

struct NarrowParams {
    const void* X;
    const void* idx;
    void* out;
    float* carry_h;
    float* carry_t;
    TileMeta* meta;
    unsigned long long* flag;
    StreamCtrl* ctrl;
    long long E, seg_base, S;
    long long NA;  // agents = warps of the grid
    int op;
};

constexpr int kNarrowWarps = 8;

// rows per lane per chunk: at most 64 value bytes, 128 value + key bytes and
// 16 rows per lane (register budget of the double buffer)
__host__ __device__ constexpr int narrow_items(int F, int esz, int ksz) {
    int r = 64 / (F * esz) < 16 ? 64 / (F * esz) : 16;
    while (r > 2 && r * (F * esz + ksz) > 128) r /= 2;
    return r;
}

// raw 32-bit words of NB bytes at p (NB multiple of 8; 16-byte pieces when
// possible).  L1-allocating loads: the lanes' 16-byte pieces of one sector
// arrive in separate instructions and are merged in L1.
template <int NB>
__device__ __forceinline__ void ld_words(const void* p, uint32_t (&w)[NB / 4]) {
    static_assert(NB % 8 == 0, "8-byte granularity");
    if constexpr (NB % 16 == 0) {
#pragma unroll
        for (int i = 0; i < NB / 16; ++i) {
            const uint4 v = ld_cached(reinterpret_cast<const uint4*>(p) + i);
            w[4 * i] = v.x;
            w[4 * i + 1] = v.y;
            w[4 * i + 2] = v.z;
            w[4 * i + 3] = v.w;
        }
    } else {
#pragma unroll
        for (int i = 0; i < NB / 8; ++i) {
            const uint2 v = __ldg(reinterpret_cast<const uint2*>(p) + i);
            w[2 * i] = v.x;
            w[2 * i + 1] = v.y;
        }
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
__device__ __forceinline__ void st_row(T* row, const float (&v)[F]) {
    if constexpr (sizeof(T) == 4) {
        if constexpr (F % 4 == 0) {
#pragma unroll
            for (int f = 0; f < F; f += 4)
                *reinterpret_cast<float4*>(row + f) = make_float4(v[f], v[f + 1], v[f + 2], v[f + 3]);
        } else if constexpr (F == 2) {
            *reinterpret_cast<float2*>(row) = make_float2(v[0], v[1]);
        } else {
            *reinterpret_cast<float*>(row) = v[0];
        }
    } else {
        if constexpr (F == 1) {
            *reinterpret_cast<uint16_t*>(row) = f2bf_bits(v[0]);
        } else {
            uint32_t w[F / 2];
#pragma unroll
            for (int i = 0; i < F / 2; ++i)
                w[i] = (uint32_t)f2bf_bits(v[2 * i]) | ((uint32_t)f2bf_bits(v[2 * i + 1]) << 16);
            if constexpr (F == 2) {
                *reinterpret_cast<uint32_t*>(row) = w[0];
            } else if constexpr (F == 4) {
                *reinterpret_cast<uint2*>(row) = make_uint2(w[0], w[1]);
            } else {
#pragma unroll
                for (int i = 0; i < F / 2; i += 4)
                    *reinterpret_cast<uint4*>(row + 2 * i) = make_uint4(w[i], w[i + 1], w[i + 2], w[i + 3]);
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

// Rows per CTA for the occupancy target: the register double buffer holds
// 2 x 64 value bytes + 2 x ITEMS keys per lane.
template <typename T, int F, int ITEMS, int OP, bool I64>
__global__ void __launch_bounds__(kNarrowWarps * 32, 2) narrow_kernel(const NarrowParams p) {
    constexpr int CH = 32 * ITEMS;             // rows per chunk
    constexpr int ESZ = sizeof(T);
    constexpr int VB = ITEMS * F * ESZ;        // value bytes per lane per chunk
    constexpr int KB = ITEMS * (I64 ? 8 : 4);  // key bytes per lane per chunk
    constexpr int VWORDS = VB / 4, KWORDS = KB / 4;
    constexpr int NACC = ITEMS * F;            // fp32 partials per lane
    static_assert(NACC % 4 == 0 || NACC < 4, "partials are spilled in 16-byte pieces");
    constexpr int NQ = (NACC + 3) / 4;         // 16-byte pieces of partials per lane
    using KT = typename std::conditional<I64, long long, int>::type;
    constexpr bool ISMAX = OP == OP_MAX;

    // per-warp copy of every lane's partials, piece-major [q][lane] (conflict-free)
    __shared__ float4 s_acc[kNarrowWarps][NQ][32];

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const T* __restrict__ X = static_cast<const T*>(p.X);
    const KT* __restrict__ I = static_cast<const KT*>(p.idx);
    T* __restrict__ out = static_cast<T*>(p.out);
    const long long seg_lo = p.seg_base, seg_hi = p.seg_base + p.S;
    const long long E = p.E;

    __shared__ unsigned s_ticket;
    __shared__ unsigned long long s_epoch;
    if (threadIdx.x == 0) {
        s_ticket = atomicAdd(&p.ctrl->ticket, 1u);
        s_epoch = ld_acquire_u64(&p.ctrl->epoch);
        if (s_ticket >= gridDim.x) __trap();  // workspace not zero-filled before first use
    }
    __syncthreads();
    const unsigned long long pub = s_epoch + 1;
    const long long a = (long long)s_ticket * kNarrowWarps + warp;
    auto agent_lo = [&](long long x) -> long long {
        if (x >= p.NA) return E;
        return ((x * E) / p.NA) / ITEMS * ITEMS;
    };
    const long long e_lo = agent_lo(a), e_hi = agent_lo(a + 1);

    auto key_at = [&](long long e) -> long long { return (long long)__ldg(I + e); };
    // zero rows strictly between keys lo_k and hi_k, clamped to [seg_lo, seg_hi)
    auto gap_fill = [&](long long lo_k, long long hi_k) {
        long long r0 = (lo_k < seg_lo) ? seg_lo : lo_k + 1;
        long long r1 = (hi_k > seg_hi) ? seg_hi : hi_k;
        float z[F];
#pragma unroll
        for (int f = 0; f < F; ++f) z[f] = 0.0f;
        for (long long r = r0; r < r1; ++r) st_row<T, F>(out + (r - seg_lo) * F, z);
    };
    // a store at key k (32-bit relative arithmetic for int32 keys; memory-safe)
    const KT kseg_lo = (KT)seg_lo;
    const unsigned long long nseg = (unsigned long long)p.S;
    auto store_at = [&](KT k, const float (&v)[F], int count) {
        unsigned long long rel;
        if constexpr (I64)
            rel = (unsigned long long)(k - kseg_lo);
        else
            rel = (unsigned long long)((unsigned)k - (unsigned)kseg_lo);  // wraps for keys < seg_lo
        if (rel < nseg) {
            float o[F];
#pragma unroll
            for (int f = 0; f < F; ++f) o[f] = (OP == OP_MEAN) ? __fdiv_rn(v[f], (float)count) : v[f];
            st_row<T, F>(out + rel * F, o);
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
    KT rkey = kprev0;     // key of the last row before the current chunk
    long long rpos = 0;   // start row (relative to e_lo) of the open segment (mean counts)
    bool rhead = head_open;  // the open segment began in an earlier agent
    float hacc[F];        // this agent's partial of that head segment, once it ends here
#pragma unroll
    for (int f = 0; f < F; ++f) hacc[f] = nident<OP>();
    long long head_end = -1;

    uint32_t nvw[VWORDS], nkw[KWORDS];  // next chunk (full lanes only)
    auto prefetch = [&](long long c) {
        const long long r = c + (long long)lane * ITEMS;
        if (r + ITEMS <= e_hi) {
            ld_words<VB>(X + r * F, nvw);
            ld_words<KB>(I + r, nkw);
        }
    };
    prefetch(e_lo);
#pragma unroll 1
    for (long long c0 = e_lo; c0 < e_hi; c0 += CH) {
        const long long r0 = c0 + (long long)lane * ITEMS;  // this lane's first row
        long long nvl = e_hi - r0;
        const int nv = nvl <= 0 ? 0 : (nvl >= ITEMS ? ITEMS : (int)nvl);  // valid items
        const bool full_chunk = c0 + CH <= e_hi;                           // warp-uniform
        float acc[ITEMS][F];
        KT k[ITEMS];
        if (nv == ITEMS) {
            uint32_t vw[VWORDS], kw[KWORDS];
#pragma unroll
            for (int i = 0; i < VWORDS; ++i) vw[i] = nvw[i];
#pragma unroll
            for (int i = 0; i < KWORDS; ++i) kw[i] = nkw[i];
            prefetch(c0 + CH);
#pragma unroll
            for (int i = 0; i < ITEMS; ++i) {
#pragma unroll
                for (int f = 0; f < F; ++f) acc[i][f] = elem_from_words<T>(vw, i * F + f);
                if constexpr (I64)
                    k[i] = (long long)(((unsigned long long)kw[2 * i + 1] << 32) | kw[2 * i]);
                else
                    k[i] = (int)kw[i];
            }
        } else {  // the agent's last chunk: partial lanes
#pragma unroll
            for (int i = 0; i < ITEMS; ++i) {
                const bool ok = i < nv;
#pragma unroll
                for (int f = 0; f < F; ++f) acc[i][f] = ok ? ld_elem<T>(X + (r0 + i) * F + f) : nident<OP>();
                k[i] = ok ? __ldg(I + r0 + i) : (KT)0;
            }
#pragma unroll
            for (int i = 1; i < ITEMS; ++i)
                if (i >= nv) k[i] = k[i - 1];  // padding never starts a segment
        }
        // neighbours: the key before the lane's first row and after its last row
        KT kp = __shfl_up_sync(0xffffffffu, k[ITEMS - 1], 1);
        if (lane == 0) kp = rkey;
        KT kn = __shfl_down_sync(0xffffffffu, k[0], 1);
        {
            // lane 31 of a full chunk: the next chunk's first key (lane 0's prefetch)
            KT pf;
            if constexpr (I64)
                pf = (long long)(((unsigned long long)nkw[1] << 32) | nkw[0]);
            else
                pf = (int)nkw[0];
            pf = __shfl_sync(0xffffffffu, pf, 0);
            if (lane == 31 && full_chunk) kn = (c0 + CH + ITEMS <= e_hi) ? pf : (KT)((c0 + CH < e_hi) ? key_at(c0 + CH) : (long long)knext_end);
            if (nv > 0 && r0 + nv >= e_hi) kn = knext_end;  // the agent's last row
        }

        // ---- lane pass: heads (is_seg), sequential accumulation with restarts
        unsigned hm = (nv > 0 && k[0] != kp) ? 1u : 0u;
#pragma unroll
        for (int i = 1; i < ITEMS; ++i) hm |= (unsigned)(k[i] != k[i - 1]) << i;  // padding repeats the last key
#pragma unroll
        for (int i = 1; i < ITEMS; ++i) {
            const bool h = (hm >> i) & 1u;
#pragma unroll
            for (int f = 0; f < F; ++f) acc[i][f] = h ? acc[i][f] : nfold<OP>(acc[i - 1][f], acc[i][f]);
        }
        const KT klast = k[ITEMS - 1];  // padded: the last valid key
        const bool last_ends = nv > 0 && klast != kn;
        const unsigned em = (hm >> 1) | ((unsigned)last_ends << (nv > 0 ? nv - 1 : 0));  // items ending a segment

        // segments that start and end inside the lane: store now
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            const unsigned upto = (2u << i) - 1u;
            if (((em >> i) & 1u) && (hm & upto)) {
                int cnt = 1;
                if constexpr (OP == OP_MEAN) cnt = i + 1 - (31 - __clz(hm & upto));
                store_at(k[i], acc[i], cnt);
            }
        }

        // gaps (empty segments) or unsorted keys: key span != number of heads
        if (nv > 0 && (long long)klast - (long long)kp != (long long)__popc(hm)) {
            long long pk = (long long)kp;
#pragma unroll
            for (int i = 0; i < ITEMS; ++i)
                if ((hm >> i) & 1u) {
                    if ((long long)k[i] != pk + 1) gap_fill(pk, (long long)k[i]);
                    pk = (long long)k[i];
                }
        }

        // ---- warp pass: segmented inclusive scan of the lane tails (Alg. 1 analog)
        float sv[F];
#pragma unroll
        for (int f = 0; f < F; ++f) sv[f] = acc[ITEMS - 1][f];
        bool sf = hm != 0;  // a segment starts in this lane (reset flag)
        long long spos = hm ? (r0 - e_lo) + (31 - __clz(hm)) : 0;  // start row of the lane's tail segment
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
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
        const bool reach = !sf;  // this lane's chain reaches back to the open segment
        if (reach) {
#pragma unroll
            for (int f = 0; f < F; ++f) sv[f] = nfold<OP>(rc[f], sv[f]);
            spos = rpos;
        }
        // carry into this lane: the previous lane's inclusive value
        float cin[F];
#pragma unroll
        for (int f = 0; f < F; ++f) cin[f] = __shfl_up_sync(0xffffffffu, sv[f], 1);
        long long cpos = 0;
        if constexpr (OP == OP_MEAN) cpos = __shfl_up_sync(0xffffffffu, spos, 1);
        bool creach = __shfl_up_sync(0xffffffffu, (int)reach, 1) != 0;
        if (lane == 0) {
#pragma unroll
            for (int f = 0; f < F; ++f) cin[f] = rc[f];
            cpos = rpos;
            creach = true;
        }

        // ---- the segment continuing into the lane from the left: ends at item j
        const bool cont = nv > 0 && !(hm & 1u);
        const int j = hm ? (__ffs(hm) - 2) : (last_ends ? nv - 1 : -1);
        if (cont && j >= 0) {
            // the lane's partial at item j, via the per-warp shared-memory copy
            float4* mine = &s_acc[warp][0][lane];
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                float4 t;
                t.x = acc[(4 * q + 0) / F][(4 * q + 0) % F];
                t.y = (4 * q + 1 < NACC) ? acc[(4 * q + 1) / F][(4 * q + 1) % F] : 0.f;
                t.z = (4 * q + 2 < NACC) ? acc[(4 * q + 2) / F][(4 * q + 2) % F] : 0.f;
                t.w = (4 * q + 3 < NACC) ? acc[(4 * q + 3) / F][(4 * q + 3) % F] : 0.f;
                mine[q * 32] = t;
            }
            const float* sp = reinterpret_cast<const float*>(&s_acc[warp][0][0]);
            float tot[F];
#pragma unroll
            for (int f = 0; f < F; ++f) {
                const int e = j * F + f;  // element e of the lane's partials: piece e/4, word e%4
                tot[f] = nfold<OP>(cin[f], sp[((e >> 2) * 32 + lane) * 4 + (e & 3)]);
            }
            if (creach && rhead) {  // the agent's head segment: resolved below
#pragma unroll
                for (int f = 0; f < F; ++f) hacc[f] = tot[f];
                head_end = r0 + j + 1;
            } else {
                store_at(k[0], tot, (int)((r0 - e_lo) + j + 1 - cpos));
            }
        }

        // ---- running segment for the next chunk: the last valid lane's state
        const unsigned vmask = __ballot_sync(0xffffffffu, nv > 0);
        const int ll = 31 - __clz(vmask);
#pragma unroll
        for (int f = 0; f < F; ++f) rc[f] = __shfl_sync(0xffffffffu, sv[f], ll);
        rkey = __shfl_sync(0xffffffffu, klast, ll);
        if constexpr (OP == OP_MEAN) rpos = __shfl_sync(0xffffffffu, spos, ll);
        if (__any_sync(0xffffffffu, hm != 0)) rhead = false;
    }
    // owner-lane broadcast of the head partial (at most one lane set it)
    const unsigned hmk = __ballot_sync(0xffffffffu, head_end >= 0);
    if (hmk) {
        const int hl = __ffs(hmk) - 1;
#pragma unroll
        for (int f = 0; f < F; ++f) hacc[f] = __shfl_sync(0xffffffffu, hacc[f], hl);
        head_end = __shfl_sync(0xffffffffu, head_end, hl);
    }

    // ---- agent end: publish the open tail (H5), then resolve an owned head
    int flags = 0;
    if (active) {
        const bool tail_open = nextk == (long long)rkey;
        if (head_open) flags |= TM_HEAD_OPEN;
        if (e_hi == E && lane == 0 && (long long)rkey + 1 < seg_hi) gap_fill((long long)rkey, KEY_AFTER);
        if (tail_open) {
            flags |= TM_TAIL_OPEN;
            if (rhead) flags |= TM_MIDDLE;  // the whole range lies inside one segment
            if (lane == 0) {
                float* c = (rhead ? p.carry_h : p.carry_t) + a * F;
#pragma unroll
                for (int f = 0; f < F; ++f) c[f] = rc[f];
                p.meta[a].flags = flags;
                p.meta[a].tail_start = e_lo + rpos;
                __threadfence();
                st_release_u64(&p.flag[a], pub);
            }
        }
    }
    __syncwarp();
    if (active && head_open && !(flags & TM_MIDDLE) && lane == 0) {
        long long u = a - 1;
        for (; u >= 0; --u) {
            while (ld_acquire_u64(&p.flag[u]) != pub) {
            }
            if (!(ld_volatile_i32(&p.meta[u].flags) & TM_MIDDLE)) break;
        }
        if (u < 0) u = 0;
        float tot[F];
#pragma unroll
        for (int f = 0; f < F; ++f) tot[f] = ld_cg_f32(p.carry_t + u * F + f);
        for (long long m = u + 1; m < a; ++m)
#pragma unroll
            for (int f = 0; f < F; ++f) tot[f] = nfold<OP>(tot[f], ld_cg_f32(p.carry_h + m * F + f));
#pragma unroll
        for (int f = 0; f < F; ++f) tot[f] = nfold<OP>(tot[f], hacc[f]);
        store_at((KT)first_key, tot, (int)(head_end - ld_volatile_i64(&p.meta[u].tail_start)));
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned done = atomicAdd(&p.ctrl->done, 1u);
        if (done == gridDim.x - 1) {
            p.ctrl->done = 0;
            p.ctrl->ticket = 0;
            __threadfence();
            atomicAdd(&p.ctrl->epoch, 1ull);
        }
    }
}

}  // namespace geot
