// narrow.cuh — the small-F segment-reduction kernel (GEOT_VARIANT_NARROW):
// rows of 4..32 bytes (fp32 F in {1,2,4,8}, bf16 F in {1,2,4,8,16}).
//
// The paper's PR schedule (Alg. 1) and its F=1 weakness (P:407-422:
// cooperative-group overhead, lanes walking the M-loop uncoalesced) motivate
// this B200 design:
//  * agents are whole warps with contiguous, ITEMS-aligned edge ranges
//    (balanced), one persistent grid, in-kernel carry resolution exactly as in
//    stream.cuh (ticketed CTAs, epoch-published agent carries);
//  * a warp processes chunks of 32*ITEMS rows; lane l owns ITEMS consecutive
//    rows, fetched with 128-bit vector loads of values and keys (coalesced:
//    the chunk is one contiguous byte range), and reduces them sequentially
//    in registers (SR within the lane);
//  * lanes are then combined by a warp-level SEGMENTED inclusive scan of the
//    lanes' tail partials with __shfl_up_sync (the shfl_down doubling loop of
//    Alg. 1, with "a segment starts in this lane" as the reset flag instead of
//    key comparison), carrying the segment start position for mean counts;
//  * each segment is written once, by the lane holding its last row; gaps are
//    zero-filled by the lane that observes them.
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

// raw 32-bit words of NB bytes at p (NB multiple of 8; 16-byte pieces when possible)
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

template <typename T>
__device__ __forceinline__ void st_elem(T* p, float v) {
    if constexpr (sizeof(T) == 4)
        *reinterpret_cast<float*>(p) = v;
    else
        *reinterpret_cast<uint16_t*>(p) = f2bf_bits(v);
}

template <typename T, int F, int ITEMS, bool ISMAX, bool I64>
__global__ void __launch_bounds__(kNarrowWarps * 32) narrow_kernel(const NarrowParams p) {
    constexpr int CH = 32 * ITEMS;           // rows per chunk
    constexpr int ESZ = sizeof(T);
    constexpr int VB = ITEMS * F * ESZ;      // value bytes per lane per chunk
    constexpr int KB = ITEMS * (I64 ? 8 : 4);  // key bytes per lane per chunk
    constexpr int VWORDS = VB / 4, KWORDS = KB / 4;
    using IdxT = typename std::conditional<I64, long long, int>::type;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const T* __restrict__ X = static_cast<const T*>(p.X);
    const IdxT* __restrict__ I = static_cast<const IdxT*>(p.idx);
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
    auto write_seg = [&](long long key, const float (&v)[F], long long count) {
        if (key < seg_lo || key >= seg_hi) return;
        T* row = out + (key - seg_lo) * F;
#pragma unroll
        for (int f = 0; f < F; ++f) st_elem<T>(row + f, finalize(v[f], p.op, count));
    };
    auto gap_fill = [&](long long lo_k, long long hi_k) {  // rows strictly between two keys
        if (hi_k <= lo_k + 1) return;  // the common case: adjacent (or unsorted) keys, no gap
        long long r0 = (lo_k < seg_lo) ? seg_lo : lo_k + 1;
        long long r1 = (hi_k > seg_hi) ? seg_hi : hi_k;
        for (long long r = r0; r < r1; ++r)
#pragma unroll
            for (int f = 0; f < F; ++f) st_elem<T>(out + (r - seg_lo) * F + f, 0.0f);
    };
    auto ident = [&](float (&v)[F]) {
#pragma unroll
        for (int f = 0; f < F; ++f) v[f] = identity<ISMAX>();
    };

    const bool active = e_lo < e_hi;
    const long long prevk = (active && e_lo > 0) ? key_at(e_lo - 1) : KEY_BEFORE;
    const long long nextk = (active && e_hi < E) ? key_at(e_hi) : KEY_AFTER;
    const long long first_key = active ? key_at(e_lo) : KEY_AFTER;
    const bool head_open = active && prevk == first_key;
    // (the gap before the first row is filled by chunk 0's lane 0 below)

    // running segment across chunks (identical in every lane)
    float rc[F];  // value of the open segment from its start (or from e_lo if it began earlier)
    ident(rc);
    long long rkey = prevk;                    // key of the open segment (prevk before the first row)
    int rstart = head_open ? -1 : 0;  // its first row - e_lo; -1: began in an earlier agent
    // head partial of a segment that began in an earlier agent and ends here
    float hacc[F];
    ident(hacc);
    long long head_end = -1;

    // software pipeline: the raw words of a full lane's NEXT chunk are in flight
    // while the current chunk is reduced (two chunks of loads per warp)
    uint32_t nvw[VWORDS], nkw[KWORDS];
    auto prefetch = [&](long long c) {
        const long long r = c + (long long)lane * ITEMS;
        if (c < e_hi && r + ITEMS <= e_hi) {
            ld_words<VB>(X + r * F, nvw);
            ld_words<KB>(I + r, nkw);
        }
    };
    prefetch(e_lo);
    for (long long c0 = e_lo; c0 < e_hi; c0 += CH) {
        const long long r0 = c0 + (long long)lane * ITEMS;  // this lane's first row
        int nv = (int)min((long long)ITEMS, e_hi - r0);     // valid items (may be <= 0)
        if (nv < 0) nv = 0;
        float v[ITEMS][F];
        IdxT k[ITEMS];  // 32-bit keys for int32 indices (cheaper compares)
        if (nv == ITEMS) {  // full lane: vector loads (ITEMS-aligned rows => aligned bytes)
            uint32_t vw[VWORDS], kw[KWORDS];
#pragma unroll
            for (int i = 0; i < VWORDS; ++i) vw[i] = nvw[i];
#pragma unroll
            for (int i = 0; i < KWORDS; ++i) kw[i] = nkw[i];
            prefetch(c0 + CH);
#pragma unroll
            for (int i = 0; i < ITEMS; ++i) {
#pragma unroll
                for (int f = 0; f < F; ++f) v[i][f] = elem_from_words<T>(vw, i * F + f);
                if constexpr (I64)
                    k[i] = (long long)(((unsigned long long)kw[2 * i + 1] << 32) | kw[2 * i]);
                else
                    k[i] = (int)kw[i];
            }
        } else {
#pragma unroll
            for (int i = 0; i < ITEMS; ++i) {
                const bool ok = i < nv;
#pragma unroll
                for (int f = 0; f < F; ++f) v[i][f] = ok ? ld_elem<T>(X + (r0 + i) * F + f) : identity<ISMAX>();
                k[i] = ok ? __ldg(I + r0 + i) : (IdxT)0;  // items >= nv are never read
            }
        }
        // neighbours: last key of the previous lane (lane 0: the open segment's key)
        // and first key of the next lane (lane 31 / beyond: next chunk's first key)
        long long my_last = KEY_AFTER;  // static indexing only (no local-memory arrays)
#pragma unroll
        for (int i = 0; i < ITEMS; ++i)
            if (i < nv) my_last = k[i];
        long long prev_last = __shfl_up_sync(0xffffffffu, my_last, 1);
        if (lane == 0) prev_last = rkey;
        long long next_first = __shfl_down_sync(0xffffffffu, k[0], 1);
        // lane 31: the next chunk's first key, from lane 0's prefetched words when available
        long long pf_first = KEY_AFTER;
        if constexpr (I64)
            pf_first = (long long)(((unsigned long long)nkw[1] << 32) | nkw[0]);
        else
            pf_first = (long long)(int)nkw[0];
        const bool pf_ok = (c0 + CH) + ITEMS <= e_hi;  // lane 0's next rows were prefetched
        const long long nxt_chunk_first = __shfl_sync(0xffffffffu, pf_first, 0);
        if (lane == 31 || r0 + ITEMS >= e_hi) {
            const long long nr = r0 + (nv > 0 ? nv : 0);
            if (lane == 31 && nv == ITEMS && pf_ok)
                next_first = nxt_chunk_first;
            else
                next_first = (nr < e_hi) ? key_at(nr) : nextk;
        }

        // ---- lane pass (SR): an inclusive segmented scan over the lane's items,
        // predicated (no per-item divergent branches): acc[i] = value of the
        // segment containing item i from its start (or from the lane start if
        // it began further left), st[i] = its start row relative to e_lo (-2:
        // began left of this lane).  is_seg (Alg. 1): key differs from the left.
        const int lane_rel = (int)(r0 - e_lo);
        float acc[ITEMS][F];
        int st[ITEMS];
        bool head[ITEMS];
        bool any_head = false;
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            head[i] = (i < nv) && ((i == 0) ? ((long long)k[0] != prev_last) : (k[i] != k[i - 1]));
            any_head = any_head || head[i];
#pragma unroll
            for (int f = 0; f < F; ++f)
                acc[i][f] = (i == 0 || head[i]) ? v[i][f] : fold<ISMAX>(acc[i - 1][f], v[i][f]);
            st[i] = head[i] ? lane_rel + i : ((i == 0) ? -2 : st[i - 1]);
        }
        const bool cont = nv > 0 && !head[0];  // the first segment continues from the left
        // gaps: rows strictly between a key and the next different one (rare:
        // only where segments are empty) — filled by the lane holding the head
        unsigned gaps = 0;  // heads whose key is not the previous key + 1
#pragma unroll
        for (int i = 0; i < ITEMS; ++i)
            if (head[i] && (i == 0 ? (long long)k[0] != prev_last + 1 : (long long)k[i] != (long long)k[i - 1] + 1))
                gaps |= 1u << i;
        if (__any_sync(0xffffffffu, gaps != 0)) {
#pragma unroll
            for (int i = 0; i < ITEMS; ++i)
                if ((gaps >> i) & 1u) gap_fill((i == 0) ? prev_last : (long long)k[i - 1], (long long)k[i]);
        }

        // ---- warp segmented inclusive scan of the lane tails (Alg. 1 analog)
        float sv[F];
#pragma unroll
        for (int f = 0; f < F; ++f) sv[f] = acc[ITEMS - 1][f];
        // -2 = "inherit from the left" doubles as the scan's reset flag
        int sst = (nv > 0) ? st[ITEMS - 1] : -2;
        (void)any_head;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            float ov[F];
#pragma unroll
            for (int f = 0; f < F; ++f) ov[f] = __shfl_up_sync(0xffffffffu, sv[f], d);
            const int ost = __shfl_up_sync(0xffffffffu, sst, d);
            if (lane >= d && sst == -2) {
#pragma unroll
                for (int f = 0; f < F; ++f) sv[f] = fold<ISMAX>(ov[f], sv[f]);
                sst = ost;
            }
        }
        // lanes whose chain reaches lane 0 unreset inherit the running segment
        if (sst == -2) {
#pragma unroll
            for (int f = 0; f < F; ++f) sv[f] = fold<ISMAX>(rc[f], sv[f]);
            sst = rstart;
        }
        // exclusive value for the first segment: previous lane's inclusive value
        float cin[F];
#pragma unroll
        for (int f = 0; f < F; ++f) cin[f] = __shfl_up_sync(0xffffffffu, sv[f], 1);
        int cst = __shfl_up_sync(0xffffffffu, sst, 1);
        if (lane == 0) {
#pragma unroll
            for (int f = 0; f < F; ++f) cin[f] = rc[f];
            cst = rstart;
        }

        // ---- items before the lane's first head continue the segment from the left
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            if (cont && st[i] == -2) {
#pragma unroll
                for (int f = 0; f < F; ++f) acc[i][f] = fold<ISMAX>(cin[f], acc[i][f]);
                st[i] = cst;
            }
        }
        // ---- writes: every item that ends a segment stores it (predicated, once)
        const bool last_ends = nv > 0 && next_first != my_last;
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            const bool ends = (i < nv) && ((i + 1 < nv) ? head[i + 1] : (i == nv - 1 && last_ends));
            if (ends && st[i] == -1) {  // began in an earlier agent: this agent owns it (below)
#pragma unroll
                for (int f = 0; f < F; ++f) hacc[f] = acc[i][f];
                head_end = r0 + i + 1;
            }
            const long long key = (long long)k[i];
            if (ends && st[i] != -1 && key >= seg_lo && key < seg_hi) {  // predicated store
                T* row = out + (key - seg_lo) * F;
                const int cnt = lane_rel + i + 1 - st[i];
#pragma unroll
                for (int f = 0; f < F; ++f) st_elem<T>(row + f, finalize(acc[i][f], p.op, cnt));
            }
        }
        // ---- running segment for the next chunk: the last valid lane's scan value
        const unsigned vmask = __ballot_sync(0xffffffffu, nv > 0);
        const int ll = 31 - __clz(vmask);
#pragma unroll
        for (int f = 0; f < F; ++f) rc[f] = __shfl_sync(0xffffffffu, sv[f], ll);
        rkey = __shfl_sync(0xffffffffu, my_last, ll);
        rstart = __shfl_sync(0xffffffffu, sst, ll);
        // a segment that ended exactly at the chunk end restarts the running value
        if (__shfl_sync(0xffffffffu, (int)last_ends, ll)) {
            ident(rc);
            rstart = -3;  // no open segment (next chunk's first row starts a new one)
        }
    }
    // owner-lane broadcast of the head partial (at most one lane set it)
    const unsigned hm = __ballot_sync(0xffffffffu, head_end >= 0);
    if (hm) {
        const int hl = __ffs(hm) - 1;
#pragma unroll
        for (int f = 0; f < F; ++f) hacc[f] = __shfl_sync(0xffffffffu, hacc[f], hl);
        head_end = __shfl_sync(0xffffffffu, head_end, hl);
    }

    // ---- agent end: publish the open tail (H5), then resolve an owned head
    int flags = 0;
    if (active) {
        const bool tail_open = (nextk == rkey) && rstart != -3;
        if (head_open) flags |= TM_HEAD_OPEN;
        if (e_hi == E && lane == 0) gap_fill(rkey, KEY_AFTER);
        if (tail_open) {
            flags |= TM_TAIL_OPEN;
            if (rstart == -1) flags |= TM_MIDDLE;  // the whole range lies inside one segment
            if (lane == 0) {
                float* c = (rstart == -1 ? p.carry_h : p.carry_t) + a * F;
#pragma unroll
                for (int f = 0; f < F; ++f) c[f] = rc[f];
                p.meta[a].flags = flags;
                p.meta[a].tail_start = e_lo + rstart;
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
            for (int f = 0; f < F; ++f) tot[f] = fold<ISMAX>(tot[f], ld_cg_f32(p.carry_h + m * F + f));
#pragma unroll
        for (int f = 0; f < F; ++f) tot[f] = fold<ISMAX>(tot[f], hacc[f]);
        write_seg(first_key, tot, head_end - ld_volatile_i64(&p.meta[u].tail_start));
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
