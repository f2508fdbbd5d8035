// stream.cuh — the TMA-streaming segment-reduction kernel (H4-H7) for rows of
// >= 128 bytes with contiguous, 16-byte aligned storage: the B200 hot path.
//
// Decomposition (the paper's tiling space, re-derived for B200):
//  * one persistent CTA per SM, W warps; each warp holds G = 32/LPR lane
//    groups ("agents").  Agent a owns the contiguous row range
//    [a*E/NA, (a+1)*E/NA) — a perfectly balanced split of the edge stream, so
//    hub segments never unbalance the grid (the reason for edge-parallel
//    tiling, SURVEY §7 hard part (b)).
//  * every warp runs its own NSTAGE-deep ring of shared-memory stages; one
//    elected lane issues 1-D TMA bulk copies (cp.async.bulk, evict-first) of
//    each group's next RS rows and arms the stage's mbarrier with the byte
//    count, while the group's lanes fetch the stage's keys with 4/8-byte
//    cp.async tracked by the same mbarrier.  The warp consumes a stage once
//    that mbarrier phase completes.  No block-wide barrier on the hot path.
//  * each agent reduces its rows sequentially in fp32 registers (SR),
//    detects the segment heads of a whole stage at once with the is_seg test
//    of Alg. 1 (key != previous key, one ballot), stores each
//    complete segment once, zero-fills gaps, and hands its head / tail partial
//    segments to per-agent carries combined in agent order by
//    carry_fixup_kernel (edge_tile.cuh).
#pragma once

#include <cuda.h>

#include <type_traits>

#include "common.cuh"
#include "edge_tile.cuh"

namespace geot {

// Default pipeline shape per lane shape (the selector may pick another compiled
// one, see launch.cuh): W warps per CTA (16 hides shared-memory latency
// better; 8 when a lane holds >= 4 vectors per row — register budget), RS rows
// per lane group per stage, NS stages: NS x W x stage <= ~192 KB of ring.
__host__ __device__ constexpr int stream_warps(int vpl) { return vpl >= 4 ? 8 : 16; }
__host__ __device__ constexpr int stream_rs(int vpl) { return vpl == 1 ? 6 : (vpl == 8 ? 1 : 3); }
__host__ __device__ constexpr int stream_stages(int vpl) { return 4 + 0 * vpl; }

// Rows per unrolled sub-chunk of a stage: the largest divisor of RS <= 8.
__host__ __device__ constexpr int stream_sub(int rs) {
    int d = rs < 8 ? rs : 8;
    while (rs % d) --d;
    return d;
}

// Control words in the workspace (zero-filled once before first use; the last
// CTA of every call re-arms ticket/done and advances the epoch, so per-agent
// flags published in a call (value epoch+1) never need clearing).
struct StreamCtrl {
    unsigned ticket;
    unsigned done;
    unsigned long long epoch;
    unsigned poison;  // sticky: set when a CTA drew a ticket >= gridDim.x (a workspace
                      // not zero-filled before first use, or used by two calls at
                      // once); cleared only by geot_workspace_init
    unsigned pad;
};

// CTA start: draw the ticket.  A ticket outside [0, gridDim.x) means the control
// words were not in their rest state: flag the workspace (geot_workspace_status
// reports it) and let the CTA retire without touching the output.  Agents that
// wait on carries poll the flag, so nothing spins on agents that never run.
__device__ __forceinline__ bool draw_ticket(StreamCtrl* ctrl, unsigned* s_ticket, unsigned long long* s_epoch) {
    if (threadIdx.x == 0) {
        *s_ticket = atomicAdd(&ctrl->ticket, 1u);
        *s_epoch = ld_acquire_u64(&ctrl->epoch);
        if (*s_ticket >= gridDim.x) atomicOr(&ctrl->poison, 1u);
    }
    __syncthreads();
    return *s_ticket < gridDim.x;
}

// wait_flag_acquire that gives up (false) once the workspace is flagged poisoned
__device__ __forceinline__ bool wait_flag_or_poison(const unsigned long long* p, unsigned long long v,
                                                    const StreamCtrl* ctrl) {
    unsigned long long x;
    for (unsigned n = 0;; ++n) {
        asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(x) : "l"(p) : "memory");
        if (x == v) break;
        if ((n & 255u) == 255u && *reinterpret_cast<const volatile unsigned*>(&ctrl->poison)) return false;
    }
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    return true;
}

#ifdef GEOT_TRACE
// experiments only (-DGEOT_TRACE, tools/trace_stream.py): per-CTA start / end
// and per-agent loop-end %globaltimer stamps, read back by geot_debug_trace
__device__ unsigned long long g_trace_cta[4096 * 4];
__device__ unsigned long long g_trace_agent[65536];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ unsigned smid() {
    unsigned r;
    asm volatile("mov.u32 %0, %smid;" : "=r"(r));
    return r;
}
#endif

// CTA end: the last CTA out re-arms ticket / done and advances the epoch.
__device__ __forceinline__ void retire_cta(StreamCtrl* ctrl) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned done = atomicAdd(&ctrl->done, 1u);
        if (done == gridDim.x - 1) {
            ctrl->done = 0;
            ctrl->ticket = 0;
            __threadfence();
            atomicAdd(&ctrl->epoch, 1ull);
        }
    }
}

struct StreamParams {
    const void* X;
    const void* idx;
    void* out;        // == outs.ptr[0]
    OutSet outs;      // every destination of a finished row (f4)
    float* carry_h;   // [NA, F] partial of an agent lying wholly inside one segment
    float* carry_t;   // [NA, F] tail partial of a segment continuing past the agent
    TileMeta* meta;   // [NA] flags / tail_start of publishing agents
    unsigned long long* flag;  // [NA] == epoch+1 once the agent's carry is published
    StreamCtrl* ctrl;
    long long E, seg_base, S;
    long long NA;      // agents (= carry slots)
    long long L;       // rows per agent (a multiple of RS): agent a owns [a*L, min((a+1)*L, E))
    long long NF;      // agents whose range is full (a*L + L <= E)
    int tma3;          // 1: `tmx` is a valid 3-D tensor map of X as [agent][stage][RS rows]
    int F, NV;         // elements / 16-byte vectors per row
    int RS;            // rows per group per stage (== the kernel's RS)
    int row_bytes;     // F * sizeof(T)
    int op;
    int idx64;
    // fused forms (MODE 1/2): row e's data is x[src[e], :] (x has V rows), times w[e]
    const void* src;
    const float* w;
    long long V;
};

__host__ __device__ inline size_t stream_smem_bytes(int W, int NS, int G, int RS, int row_bytes, int mode = 0) {
    return (size_t)W * NS * G * RS * row_bytes       // row ring
           + (size_t)W * NS * G * RS * 8             // key ring
           + (size_t)W * NS * 8                      // mbarriers
           + (mode == 2 ? (size_t)W * NS * G * RS * 4 : 0)   // weight ring
           + (mode >= 1 ? (size_t)W * NS * G * RS * 8 : 0);  // src-id ring (NS stages ahead)
}

// 3-D tensor TMA (box {c0, c1, c2}) global -> shared, completing on `bar`
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

// cp.async of 16 bytes; src_bytes 0 zero-fills the destination (no global read)
__device__ __forceinline__ void cp_async_16_zfill(uint32_t dst, const void* src, uint32_t src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}


// NS > 0: TMA bulk-copy ring of NS stages per warp (one CTA per SM).
// NS == 0: the same agents and carries, rows streamed with 128-bit LDG into a
//          register double buffer (several CTAs per SM, no shared ring).
//
// MODE 1/2 (fused gather, H8): the same agents, ring, keys and carries, but a
// stage's rows are GATHERED: every lane cp.async-copies its 16-byte slices of
// the rows x[src[e]] into the ring.  The src ids travel one ring cycle ahead:
// issuing stage s also cp.async-loads the ids of stage s + NS into the same
// buffer's id slots, so they have landed when stage s is consumed and its
// buffer is refilled.  MODE 2 also stages w[e] and folds w[e] * x[src[e]].  An
// out-of-range src id gathers a zero row (memory-safe; results for bad data
// are unspecified).
template <typename T, int VW, int LPR, int VPL, bool ISMAX, int W, int RS, int NS, int MODE = 0, bool SRC64 = false,
          bool REP = false>
__global__ void __launch_bounds__(W * 32, NS > 0 ? 1 : 2)
    stream_kernel(const StreamParams p, const __grid_constant__ CUtensorMap tmx) {
    constexpr bool TMA = NS > 0;
    static_assert(MODE == 0 || NS > 0, "the fused forms use the shared-memory ring");
    constexpr int NSX = TMA ? NS : 1;
    constexpr int G = 32 / LPR;
    using Cv = Conv<T, VW>;
    using Raw = typename Cv::Raw;
    constexpr int SUB = stream_sub(RS);  // rows per unrolled sub-chunk (LDG path: RS <= 8)
    static_assert(NS > 0 || SUB == RS, "the LDG pipeline holds whole stages in registers");
    constexpr int VB = (int)sizeof(Raw);  // bytes per lane vector (2..16; one agent per warp below 16)
    static_assert(RS <= LPR, "one key per lane per stage");
    static_assert(VB == 16 || LPR == 32, "narrow lane vectors: one agent per warp");

    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gi = lane / LPR, li = lane % LPR;
    const unsigned gmask = (LPR == 32) ? 0xffffffffu : (((1u << LPR) - 1u) << (gi * LPR));
    const int row_bytes = p.row_bytes;
    const int stage_bytes = G * RS * row_bytes;
    unsigned char* wbuf = smem_raw + (size_t)warp * NS * stage_bytes;
    unsigned long long* wkey =
        reinterpret_cast<unsigned long long*>(smem_raw + (size_t)W * NS * stage_bytes) + warp * NS * G * RS;
    uint64_t* bars =
        reinterpret_cast<uint64_t*>(smem_raw + (size_t)W * NS * stage_bytes + (size_t)W * NS * G * RS * 8) + warp * NS;
    float* wring = reinterpret_cast<float*>(smem_raw + (size_t)W * NS * stage_bytes + (size_t)W * NS * G * RS * 8 +
                                            (size_t)W * NS * 8) +
                   warp * NS * G * RS;
    unsigned long long* sring =
        reinterpret_cast<unsigned long long*>(smem_raw + (size_t)W * NS * stage_bytes + (size_t)W * NS * G * RS * 8 +
                                              (size_t)W * NS * 8 + (MODE == 2 ? (size_t)W * NS * G * RS * 4 : 0)) +
        warp * NS * G * RS;

    const long long seg_lo = p.seg_base, seg_hi = p.seg_base + p.S;
    const int F = p.F;
    const T* __restrict__ X = static_cast<const T*>(p.X);
    // destination 0 addressed by key - seg_lo (row of key seg_lo); replicas (f4) below
    T* __restrict__ out = static_cast<T*>(p.outs.ptr[0]) + (seg_lo - p.outs.row_off) * (long long)F;
    const int isz = p.idx64 ? 8 : 4;
    const unsigned char* idxb = static_cast<const unsigned char*>(p.idx);

    // CTA ticket: agents are numbered in CTA start order, so an agent only
    // ever waits on agents of CTAs that started before it (forward progress).
    __shared__ unsigned s_ticket;
    __shared__ unsigned long long s_epoch;
    if (!draw_ticket(p.ctrl, &s_ticket, &s_epoch)) {
        retire_cta(p.ctrl);
        return;
    }
    const unsigned long long pub = s_epoch + 1;  // "published in this call" flag value
#ifdef GEOT_TRACE
    if (threadIdx.x == 0 && s_ticket < 4096) {
        g_trace_cta[s_ticket * 4 + 0] = gtimer();
        g_trace_cta[s_ticket * 4 + 2] = smid();
    }
#endif

    // agent ranges.  4+ agents per warp (EQL): L rows each (L = ceil(E / NA)
    // rounded up to RS), so every stage of a full agent holds RS rows and the G
    // agents of a warp sit at a constant stride in X (one 3-D TMA copy per stage,
    // below); the last agents may be short or empty (empty ones only at the end:
    // no agent ever waits on one).  Otherwise [a*E/NA, (a+1)*E/NA) (A/B: the
    // equal-length split with per-agent copies cost products bf16 ~10 %).
    constexpr bool EQL = TMA && MODE == 0 && G >= 4;
    const long long a = ((long long)s_ticket * W + warp) * G + gi;
    long long e_lo, e_hi;
    if constexpr (EQL) {
        e_lo = (a * p.L < p.E) ? a * p.L : p.E;
        e_hi = (e_lo + p.L < p.E) ? e_lo + p.L : p.E;
    } else {
        e_lo = (a * p.E) / p.NA;
        e_hi = ((a + 1) * p.E) / p.NA;
    }
    const int nrows = (int)(e_hi - e_lo);
    const int nst = (nrows + RS - 1) / RS;
    const int nst_w = __reduce_max_sync(0xffffffffu, nst);
    const int nfull_w = __reduce_min_sync(0xffffffffu, nrows / RS);  // stages full in every group
    // every group's range, for the producer lane: held in registers for 1-2
    // agents per warp; recomputed where used for EQL (4G registers otherwise)
    const long long wa0 = ((long long)s_ticket * W + warp) * G;
    constexpr int GH = EQL ? 1 : G;
    long long glo_r[GH], ghi_r[GH];
    const unsigned char* xg_r[GH];
#pragma unroll
    for (int g = 0; g < GH; ++g) {
        glo_r[g] = __shfl_sync(0xffffffffu, e_lo, g * LPR);
        ghi_r[g] = __shfl_sync(0xffffffffu, e_hi, g * LPR);
        xg_r[g] = reinterpret_cast<const unsigned char*>(X) + glo_r[g] * (long long)row_bytes;
    }
    auto glo = [&](int g) -> long long {
        if constexpr (EQL)
            return (wa0 + g) * p.L < p.E ? (wa0 + g) * p.L : p.E;
        else
            return glo_r[g];
    };
    auto ghi = [&](int g) -> long long {
        if constexpr (EQL)
            return glo(g) + p.L < p.E ? glo(g) + p.L : p.E;
        else
            return ghi_r[g];
    };
    auto xg = [&](int g) -> const unsigned char* {
        if constexpr (EQL)
            return reinterpret_cast<const unsigned char*>(X) + glo(g) * (long long)row_bytes;
        else
            return xg_r[g];
    };

    if constexpr (TMA) {
        // int32 keys land in the low half of 8-byte slots: zero the ring once
        for (int i = lane; i < NS * G * RS; i += 32) wkey[i] = 0ull;
        if (lane == 0) {
            for (int s = 0; s < NS; ++s)
                mbar_init(&bars[s], MODE == 0 ? 1 + 32 : 32);  // (TMA producer +) 32 cp.async arrivals
            fence_mbar_init();
        }
        __syncwarp();
    }
    const uint64_t pol = policy_evict_first();
    // 3-D TMA for the warp's value stages (G >= 2 agents per warp, plain form):
    // every agent of the warp full, stage buffers 128-byte aligned
    const long long a0 = wa0;  // the warp's first agent
    bool use3d = false;
    if constexpr (EQL)
        use3d = p.tma3 && a0 + G <= p.NF && ((smem_u32(wbuf) | (uint32_t)stage_bytes) & 127u) == 0;

    const bool col_ok0 = li < p.NV;  // (fused forms: one 16-byte vector per lane)
    const unsigned long long xrows = (unsigned long long)p.V;
    const unsigned xrows32 = p.V < 0xFFFFFFFFLL ? (unsigned)p.V : 0xFFFFFFFFu;
    const unsigned xrow_bytes = (unsigned)p.row_bytes;
    const unsigned char* xlane = reinterpret_cast<const unsigned char*>(X) + li * 16;  // this lane's column
    // fused forms: the src ids of stage s + NS are cp.async-loaded into the id
    // slot of buffer s % NS by issue(s) (so they land with stage s), and read
    // back by the refill that issues stage s + NS (same lane, same slot)
    auto id_copy = [&](int s) {  // src ids of stage s into the slots of buffer s % NS
        const long long e = e_lo + (long long)s * RS + li;
        if (li < RS && e < e_hi) {
            void* dst = sring + ((s % NSX) * G + gi) * RS + li;
            if (isz == 4)
                cp_async_4(dst, static_cast<const unsigned char*>(p.src) + e * 4);
            else
                cp_async_8(dst, static_cast<const unsigned char*>(p.src) + e * 8);
        }
    };

    // all lanes: fill stage s of every group of the warp into buffer s % NS
    auto issue = [&](int s, long long sq) {
        const int b = s % NSX;
        if constexpr (MODE >= 1) {
            // gather: lane li copies its 16-byte slices of each of the stage's rows
            // x[src] (cp.async, L2 only); the ids come from this buffer's id slots
            long long cl = e_hi - (e_lo + (long long)s * RS);
            int c = cl < 0 ? 0 : (cl > RS ? RS : (int)cl);
            c = col_ok0 ? c : 0;
            asm volatile("" : "+r"(c));  // a 32-bit row count (no 64-bit compare per row)
            const unsigned long long* ids = sring + (b * G + gi) * RS;
            const uint32_t gbase = smem_u32(wbuf) + (uint32_t)(b * stage_bytes + gi * RS * row_bytes + li * 16);
#pragma unroll
            for (int r = 0; r < RS; ++r) {
                if (r < c) {
                    const unsigned long long raw = ids[r];  // broadcast within the group
                    if constexpr (SRC64) {
                        const bool ok = raw < xrows;
                        const size_t off = (size_t)(ok ? raw : 0ull) * xrow_bytes;  // byte offset of row src in x
                        cp_async_16_zfill(gbase + (uint32_t)(r * row_bytes), xlane + off, ok ? 16u : 0u);
                    } else {
                        // int32 ids (V < 2^31): the row address is ONE wide multiply-add
                        const unsigned sid = (unsigned)raw;
                        const bool ok = sid < xrows32;
                        unsigned long long addr;
                        asm("mad.wide.u32 %0, %1, %2, %3;"
                            : "=l"(addr)
                            : "r"(ok ? sid : 0u), "r"(xrow_bytes), "l"(reinterpret_cast<unsigned long long>(xlane)));
                        cp_async_16_zfill(gbase + (uint32_t)(r * row_bytes), reinterpret_cast<const void*>(addr),
                                          ok ? 16u : 0u);
                    }
                }
            }
            __syncwarp();  // every lane has read the id slots before they are refilled
            id_copy(s + NSX);
            if constexpr (MODE == 2) {
                const long long e = e_lo + (long long)s * RS + li;
                if (li < RS && e < e_hi) cp_async_4(wring + (b * G + gi) * RS + li, p.w + e);
            }
        } else if (lane == 0 && s < nfull_w && use3d) {
            // all G agents of the warp are full: their stage-s rows are ONE box of
            // the 3-D view [agent][stage][RS rows] of X (one TMA instead of G copies)
            mbar_arrive_expect_tx(&bars[b], (uint32_t)stage_bytes);
            tma_load_3d(smem_u32(wbuf + b * stage_bytes), &tmx, 0, s, (int)a0, &bars[b], pol);
        } else if (lane == 0 && s < nfull_w) {
            // every group has RS rows in this stage (all but the last stage or two)
            unsigned char* buf = wbuf + b * stage_bytes;
            const uint32_t gb = (uint32_t)(RS * row_bytes);
            mbar_arrive_expect_tx(&bars[b], G * gb);
            const size_t soff = (size_t)s * gb;
#pragma unroll
            for (int g = 0; g < G; ++g)
                bulk_g2s(buf + g * gb, xg(g) + soff, gb, &bars[b], pol);
        } else if (lane == 0) {
            unsigned char* buf = wbuf + b * stage_bytes;
            uint32_t total = 0;
            int cnt[G];
#pragma unroll
            for (int g = 0; g < G; ++g) {
                long long c = ghi(g) - (glo(g) + (long long)s * RS);
                c = c < 0 ? 0 : (c > RS ? RS : c);
                cnt[g] = (int)c;
                total += (uint32_t)c * row_bytes;
            }
            mbar_arrive_expect_tx(&bars[b], total);
#pragma unroll
            for (int g = 0; g < G; ++g)
                if (cnt[g] > 0)
                    bulk_g2s(buf + g * RS * row_bytes, X + (glo(g) + (long long)s * RS) * F,
                             (uint32_t)cnt[g] * row_bytes, &bars[b], pol);
        }
        const long long e = e_lo + (long long)s * RS + li;
        if (li < RS && e < e_hi) {
            void* dst = wkey + (b * G + gi) * RS + li;
            if (isz == 4)
                cp_async_4(dst, idxb + e * 4);
            else
                cp_async_8(dst, idxb + e * 8);
        }
        cp_async_mbar_arrive(&bars[b]);
    };
    if constexpr (MODE >= 1) {
        // the ids of the first NS stages: loaded and waited for here (cp.async group)
        for (int s = 0; s < NS && s < nst_w; ++s) id_copy(s);
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncwarp();
        for (int s = 0; s < NS && s < nst_w; ++s) issue(s, 0);
    } else if constexpr (TMA) {
        for (int s = 0; s < NS && s < nst_w; ++s) issue(s, 0);
    }

    // Every key is read the way the key ring holds it: int32 keys ZERO-extended
    // (they land in the low half of zeroed 8-byte slots).  Keys must compare the
    // same wherever they were read — the carry chain's head/tail tests pair a
    // ring copy with these direct loads (a sign/zero mismatch on a negative key
    // once deadlocked it).  Negative int32 keys thus read as values >= 2^31, i.e.
    // out of range, skipped like any other (results for bad data unspecified).
    auto key_ld = [&](long long e) -> long long {
        return p.idx64 ? __ldg(static_cast<const long long*>(p.idx) + e)
                       : (long long)(unsigned)__ldg(static_cast<const int*>(p.idx) + e);
    };
    const long long prevk = (e_lo > 0) ? key_ld(e_lo - 1) : KEY_BEFORE;
    const long long nextk = (e_hi < p.E) ? key_ld(e_hi) : KEY_AFTER;
    const long long first_key = (nrows > 0) ? key_ld(e_lo) : KEY_AFTER;

    auto vec_col = [&](int j) { return li + j * LPR; };
    auto write_row = [&](long long key, const float (&acc)[VPL][VW], long long count) {
        if (key < seg_lo || key >= seg_hi) return;
        Raw packed[VPL];
#pragma unroll
        for (int j = 0; j < VPL; ++j) {
            float o[VW];
#pragma unroll
            for (int q = 0; q < VW; ++q) o[q] = finalize(acc[j][q], p.op, count);
            packed[j] = Cv::pack(o);
        }
        {
            T* rowp = out + (key - seg_lo) * (long long)F;
#pragma unroll
            for (int j = 0; j < VPL; ++j)
                if (vec_col(j) < p.NV) st_vec(reinterpret_cast<Raw*>(rowp + vec_col(j) * VW), packed[j]);
        }
        if constexpr (REP) {  // f4: the same row into every replica
            for (int d = 1; d < p.outs.n; ++d) {
                T* rp = static_cast<T*>(p.outs.ptr[d]) + (key - p.outs.row_off) * (long long)F;
                for (int j = 0; j < VPL; ++j)
                    if (vec_col(j) < p.NV) st_vec_mc(reinterpret_cast<Raw*>(rp + vec_col(j) * VW), packed[j], out_is_mc(p.outs, d));
            }
        }
    };
    // predicated form of write_row (no branch around the store)
    auto write_row_pred = [&](bool pred, long long key, const float (&acc)[VPL][VW], long long count) {
        const bool ok = pred && key >= seg_lo && key < seg_hi;
        Raw packed[VPL];
#pragma unroll
        for (int j = 0; j < VPL; ++j) {
            float o[VW];
#pragma unroll
            for (int q = 0; q < VW; ++q) o[q] = finalize(acc[j][q], p.op, count);
            packed[j] = Cv::pack(o);
        }
        T* rowp = out + (key - seg_lo) * (long long)F;
#pragma unroll
        for (int j = 0; j < VPL; ++j)
            if (ok && vec_col(j) < p.NV) st_vec(reinterpret_cast<Raw*>(rowp + vec_col(j) * VW), packed[j]);
        if constexpr (REP) {
            if (ok)
                for (int d = 1; d < p.outs.n; ++d) {
                    T* rp = static_cast<T*>(p.outs.ptr[d]) + (key - p.outs.row_off) * (long long)F;
                    for (int j = 0; j < VPL; ++j)
                        if (vec_col(j) < p.NV) st_vec_mc(reinterpret_cast<Raw*>(rp + vec_col(j) * VW), packed[j], out_is_mc(p.outs, d));
                }
        }
    };
    auto gap_fill = [&](long long lo_k, long long hi_k) {
        long long r0 = (lo_k < seg_lo) ? seg_lo : lo_k + 1;
        long long r1 = (hi_k > seg_hi) ? seg_hi : hi_k;
        float z[VW];
#pragma unroll
        for (int q = 0; q < VW; ++q) z[q] = 0.0f;
        const Raw zr = Cv::pack(z);
        for (long long r = r0; r < r1; ++r) {
            T* rowp = out + (r - seg_lo) * (long long)F;
#pragma unroll
            for (int j = 0; j < VPL; ++j) {
                const int v = vec_col(j);
                if (v < p.NV) st_vec(reinterpret_cast<Raw*>(rowp + v * VW), zr);
            }
        }
        if constexpr (REP) {
            for (int d = 1; d < p.outs.n; ++d) {
                for (long long r = r0; r < r1; ++r) {
                    T* rp = static_cast<T*>(p.outs.ptr[d]) + (r - p.outs.row_off) * (long long)F;
                    for (int j = 0; j < VPL; ++j)
                        if (vec_col(j) < p.NV) st_vec_mc(reinterpret_cast<Raw*>(rp + vec_col(j) * VW), zr, out_is_mc(p.outs, d));
                }
            }
        }
    };
    auto carry_store = [&](float* carry, const float (&acc)[VPL][VW]) {
        float* c = carry + a * (long long)F;
#pragma unroll
        for (int j = 0; j < VPL; ++j) {
            const int v = vec_col(j);
            if (v < p.NV)
#pragma unroll
                for (int q = 0; q < VW; ++q) c[v * VW + q] = acc[j][q];
        }
    };
    float acc[VPL][VW];
#pragma unroll
    for (int j = 0; j < VPL; ++j)
#pragma unroll
        for (int q = 0; q < VW; ++q) acc[j][q] = identity<ISMAX>();
    // bf16 max (branchy path): fold packed bf16 pairs with HMNMX2 (exact: the max is
    // one of the inputs) and widen to the fp32 acc only where a segment ends
    constexpr bool PKMAX = ISMAX && sizeof(T) == 2 && MODE == 0 && G < 4;
    // the lean row loop (process_small below) for 4+ agents per warp.  (Also
    // tried for every one-vector-per-lane shape: A/B on one box, products bf16
    // 2810 -> 3482 us, arxiv 167 -> 191, Reddit fused 3693 -> 5495, fp32 F=64
    // 850 -> 790: with 1-2 agents per warp the branchy end-of-segment path is
    // cheaper than a predicated store + selects on every row.)
    constexpr bool LEAN = G >= 4;
    constexpr int PKW = PKMAX ? VW / 2 : 1;
    uint32_t pk[VPL][PKW];
#pragma unroll
    for (int j = 0; j < VPL; ++j)
#pragma unroll
        for (int w = 0; w < PKW; ++w) pk[j][w] = 0xFF80FF80u;  // bf16 -inf, -inf
    auto sync_acc = [&]() {
        if constexpr (PKMAX) {
#pragma unroll
            for (int j = 0; j < VPL; ++j)
#pragma unroll
                for (int w = 0; w < PKW; ++w) {
                    acc[j][2 * w] = __uint_as_float(pk[j][w] << 16);
                    acc[j][2 * w + 1] = __uint_as_float(pk[j][w] & 0xFFFF0000u);
                }
        }
    };

    long long cur = first_key;
    const bool head_open = nrows > 0 && prevk == cur;
    if (nrows > 0 && !head_open) gap_fill(prevk, cur);
    long long seg_start = e_lo;
    bool first = true;
    int flags = 0;
    long long head_end = 0;
    float hacc[VPL][VW];  // head partial of a segment that began in an earlier agent
    bool col_ok[VPL];
#pragma unroll
    for (int j = 0; j < VPL; ++j) col_ok[j] = vec_col(j) < p.NV;
    // one stage of RS rows (already in registers) + this lane's key (row li)
    // SUB rows at a time (code size: the segment-end path is inlined once per
    // row of a sub-chunk); `heads` bit r = row r starts a segment; the key of
    // row r is held by lane (koff + r) of the group
    // wst[r]: the weight of row r (MODE 2), read from the ring by every lane of
    // the group (broadcast) before the stage's buffer is refilled — a shuffle
    // with a group mask would cost a WARPSYNC loop per row
    auto process = [&](const Raw (&rows)[SUB][VPL], unsigned heads, long long kmine, int koff, int cnt,
                       long long r_base, const float (&wst)[SUB]) {
#pragma unroll
        for (int r = 0; r < SUB; ++r) {
            // (G >= 4: no early exit — the warp-wide votes below need every lane)
            if constexpr (G < 4) {
                if (r >= cnt) break;
            }
            const bool valid = r < cnt;
            const Raw (&raw)[VPL] = rows[r];
            if constexpr (G >= 4) {
                // small rows, 4+ agents per warp: their segment ends rarely coincide, so
                // a branch per end would serialise the warp — the end of a segment is
                // handled branch-free (predicated store, selects); only the rare
                // events (head-partial capture, gaps) take warp-uniform branches
                const bool h = valid && ((heads >> r) & 1u);
                const long long k = __shfl_sync(0xffffffffu, kmine, (koff + r) & (LPR - 1), LPR);
                const long long e = r_base + r;
                const bool hf = h && first && head_open;
                if (__any_sync(0xffffffffu, hf)) {
                    if (hf) {
#pragma unroll
                        for (int j = 0; j < VPL; ++j)
#pragma unroll
                            for (int q = 0; q < VW; ++q) hacc[j][q] = acc[j][q];
                        flags |= TM_HEAD_OPEN;
                        head_end = e;
                    }
                }
                write_row_pred(h && !hf, cur, acc, e - seg_start);
                const bool gp = h && k != cur + 1;
                if (__any_sync(0xffffffffu, gp)) {
                    if (gp) gap_fill(cur, k);
                }
                first = first && !h;
                cur = h ? k : cur;
                seg_start = h ? e : seg_start;
#pragma unroll
                for (int j = 0; j < VPL; ++j)
#pragma unroll
                    for (int q = 0; q < VW; ++q) acc[j][q] = h ? identity<ISMAX>() : acc[j][q];
            } else if ((heads >> r) & 1u) {  // segment `cur` ended at the previous row
                const long long k = __shfl_sync(gmask, kmine, koff + r, LPR);
                const long long e = r_base + r;
                sync_acc();
                if (first && head_open) {
#pragma unroll
                    for (int j = 0; j < VPL; ++j)
#pragma unroll
                        for (int q = 0; q < VW; ++q) hacc[j][q] = acc[j][q];
                    flags |= TM_HEAD_OPEN;
                    head_end = e;
                } else {
                    write_row(cur, acc, e - seg_start);
                }
                first = false;
                gap_fill(cur, k);
                cur = k;
                seg_start = e;
#pragma unroll
                for (int j = 0; j < VPL; ++j)
#pragma unroll
                    for (int q = 0; q < VW; ++q) acc[j][q] = identity<ISMAX>();
                if constexpr (PKMAX) {
#pragma unroll
                    for (int j = 0; j < VPL; ++j)
#pragma unroll
                        for (int w = 0; w < PKW; ++w) pk[j][w] = 0xFF80FF80u;
                }
            }
            if constexpr (G >= 4) {
                if (!valid) continue;  // (no collective below this point)
            }
            float wr = 1.0f;
            if constexpr (MODE == 2) wr = wst[r];
            if constexpr (PKMAX) {
#pragma unroll
                for (int j = 0; j < VPL; ++j) {
                    const uint32_t* rw = reinterpret_cast<const uint32_t*>(&raw[j]);
#pragma unroll
                    for (int w = 0; w < PKW; ++w) {
                        __nv_bfloat162 a = *reinterpret_cast<const __nv_bfloat162*>(&pk[j][w]);
                        const __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162*>(&rw[w]);
                        a = __hmax2(a, b);
                        pk[j][w] = *reinterpret_cast<const uint32_t*>(&a);
                    }
                }
                continue;
            }
#pragma unroll
            for (int j = 0; j < VPL; ++j) {
                float f[VW];
                Cv::unpack(raw[j], f);
#pragma unroll
                for (int q = 0; q < VW; ++q)
                    if constexpr (MODE == 2) f[q] = wr * f[q];
                if constexpr (!ISMAX && VW % 2 == 0) {
                    // packed fp32x2 adds (sm_100 FADD2): two IEEE RN adds per instruction
#pragma unroll
                    for (int q = 0; q < VW; q += 2) {
                        const float2 t = __fadd2_rn(make_float2(acc[j][q], acc[j][q + 1]), make_float2(f[q], f[q + 1]));
                        acc[j][q] = t.x;
                        acc[j][q + 1] = t.y;
                    }
                } else {
#pragma unroll
                    for (int q = 0; q < VW; ++q) acc[j][q] = fold<ISMAX>(acc[j][q], f[q]);
                }
            }
        }
    };

    // ---- small rows (G >= 4 agents per warp, one 16-byte vector per lane): the
    // per-row work of every agent is one predicated vector store of the segment
    // that ended, selects and a packed fold; everything else is per stage —
    // relative 32-bit keys, the gap test of every row (rare zero-fill), and the
    // capture of the agent's head partial (at most once per agent)
    // rows[r] is row koff + r of the stage (a sub-chunk of SUB rows; the stage's
    // keys sit one per lane: lane li holds row li); heads_w is the group's head
    // mask shifted by koff, cnt the group's valid rows counted from koff
    auto process_small = [&](const Raw (&rows)[SUB][VPL], unsigned heads_w, long long kmine, long long kprev,
                             int koff, int cnt, long long r_base, const float (&wst)[SUB]) {
        // this sub-chunk's head bits (the shifted ballot still holds later rows and groups)
        const unsigned heads = heads_w & ((1u << SUB) - 1u);
        const unsigned long long nseg = (unsigned long long)p.S;  // < 2^32 - 1 (host check)
        const int rb = (int)(r_base - e_lo);                      // agent-relative row of row 0
        unsigned crel = (unsigned long long)(cur - seg_lo) < nseg ? (unsigned)(cur - seg_lo) : 0xFFFFFFFFu;
        const unsigned krl = (unsigned long long)(kmine - seg_lo) < nseg ? (unsigned)(kmine - seg_lo) : 0xFFFFFFFFu;
        int sst = (int)(seg_start - e_lo);
        // empty segments before a head row (its key is not the previous key + 1),
        // for the whole stage at its first sub-chunk
        const bool gpl = koff == 0 && li < cnt && kmine != kprev && kmine != kprev + 1;
        if (__any_sync(0xffffffffu, gpl)) {
#pragma unroll 1
            for (int r = 0; r < RS; ++r) {
                const long long kp_ = __shfl_sync(0xffffffffu, kprev, r, LPR);
                const long long k_ = __shfl_sync(0xffffffffu, kmine, r, LPR);
                const bool g_ = __shfl_sync(0xffffffffu, (int)gpl, r, LPR) != 0;
                if (g_) gap_fill(kp_, k_);
            }
        }
        unsigned char* const out_lane = reinterpret_cast<unsigned char*>(out + li * VW);
        const unsigned rowb = (unsigned)row_bytes;
        auto rows_loop = [&](auto capc) {
            constexpr bool CAP = decltype(capc)::value;
            bool capp = first && head_open;  // the agent's head segment not closed yet
#pragma unroll
            for (int r = 0; r < SUB; ++r) {
                const bool h = (heads >> r) & 1u;
                const unsigned kr = __shfl_sync(0xffffffffu, krl, koff + r, LPR);
                bool st = h && crel != 0xFFFFFFFFu && col_ok0;
                if constexpr (CAP) {
                    const bool hf = h && capp;
                    if (hf) {
#pragma unroll
                        for (int q = 0; q < VW; ++q) hacc[0][q] = acc[0][q];
                        flags |= TM_HEAD_OPEN;
                        head_end = r_base + r;
                    }
                    st = st && !hf;
                    capp = capp && !h;
                }
                {  // the segment crel ended at row r - 1: one predicated store
                    float o[VW];
#pragma unroll
                    for (int q = 0; q < VW; ++q) o[q] = finalize(acc[0][q], p.op, rb + r - sst);
                    const Raw pk = Cv::pack(o);
                    if (st) st_vec(reinterpret_cast<Raw*>(out_lane + (size_t)crel * rowb), pk);
                    if constexpr (REP) {
                        if (st)
                            for (int d = 1; d < p.outs.n; ++d) {
                                T* rp = static_cast<T*>(p.outs.ptr[d]) +
                                        ((long long)crel + seg_lo - p.outs.row_off) * (long long)F + li * VW;
                                st_vec_mc(reinterpret_cast<Raw*>(rp), pk, out_is_mc(p.outs, d));
                            }
                    }
                }
                crel = h ? kr : crel;
                sst = h ? rb + r : sst;
                float f[VW];
                Cv::unpack(rows[r][0], f);
                if constexpr (MODE == 2) {
#pragma unroll
                    for (int q = 0; q < VW; ++q) f[q] = (r < cnt ? wst[r] : 0.f) * f[q];  // stale weight slots past cnt
                }
                if constexpr (ISMAX) {
                    const bool valid = r < cnt;
#pragma unroll
                    for (int q = 0; q < VW; ++q) acc[0][q] = h ? f[q] : (valid ? fmaxf(acc[0][q], f[q]) : acc[0][q]);
                } else {  // rows past cnt are zero vectors (no head): adding them is exact
#pragma unroll
                    for (int q = 0; q < VW; q += 2) {
                        const float2 t = __fadd2_rn(make_float2(h ? 0.f : acc[0][q], h ? 0.f : acc[0][q + 1]),
                                                    make_float2(f[q], f[q + 1]));
                        acc[0][q] = t.x;
                        acc[0][q + 1] = t.y;
                    }
                }
            }
        };
        if (__any_sync(0xffffffffu, first && head_open && heads != 0))
            rows_loop(std::true_type{});
        else
            rows_loop(std::false_type{});
        // running segment after the stage: the key of the group's last row
        const int nv = cnt < SUB ? cnt : SUB;
        const long long klast = __shfl_sync(0xffffffffu, kmine, koff + (nv > 0 ? nv - 1 : 0), LPR);
        if (nv > 0) cur = klast;
        seg_start = e_lo + sst;
        first = first && heads == 0;
    };

    if constexpr (TMA) {
        // refill the buffer of stage s with stage s + NS (fused: src ids from the queue)
        auto refill = [&](int s) {
            if (s + NSX < nst_w) issue(s + NSX, 0);
        };
        // 32-bit shared address of this lane's first vector in group gi's rows of buffer 0
        const uint32_t lane_s0 = smem_u32(wbuf) + gi * RS * row_bytes + li * VB;
#pragma unroll 1
        for (int s = 0; s < nst_w; ++s) {
            const int b = s % NSX;
            mbar_wait(&bars[b], (uint32_t)((s / NSX) & 1));
            const uint32_t sbase = lane_s0 + b * stage_bytes;
            const long long* gkey = reinterpret_cast<const long long*>(wkey + (b * G + gi) * RS);
            const long long r_base = e_lo + (long long)s * RS;
            int cnt = (int)(e_hi - r_base);
            cnt = cnt < 0 ? 0 : (cnt > RS ? RS : cnt);
            const long long kmine = (li < cnt) ? gkey[li] : KEY_AFTER;
            const long long kprev = (li == 0) ? cur : ((li <= cnt) ? gkey[li - 1] : KEY_AFTER);
            const float* wslots = MODE == 2 ? wring + (b * G + gi) * RS : nullptr;
            // is_seg of the whole stage (Alg. 1): row r starts a segment iff its
            // key differs from row r-1's (row -1: `cur`); every lane of the warp
            // is here (full-warp ballot: a group mask costs a WARPSYNC loop)
            const unsigned heads = __ballot_sync(0xffffffffu, li < cnt && kmine != kprev) >> (gi * LPR);
            if constexpr (SUB == RS) {
                // the whole stage's rows into registers at once, then hand the buffer
                // back to the TMA producer right away (the proxy fence orders these
                // shared-memory reads before the async-proxy writes of the refill)
                Raw rows[SUB][VPL];
#pragma unroll
                for (int r = 0; r < SUB; ++r)
#pragma unroll
                    for (int j = 0; j < VPL; ++j)
                        // (fused forms, 1-2 agents per warp: rows past cnt are never
                        // folded — the row loop stops at cnt — so no zero default and
                        // no predicate: Reddit-shaped 3601 -> 3261 us; the plain form
                        // measured 1-2 % slower without them, kept)
                        rows[r][j] = ((LEAN || MODE == 0) ? (r < cnt && col_ok[j]) : true)
                                         ? lds_vec<Raw>(sbase + r * row_bytes + j * LPR * VB)
                                         : Raw{};
                float wst[SUB];
#pragma unroll
                for (int r = 0; r < SUB; ++r) wst[r] = MODE == 2 ? wslots[r] : 1.0f;
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                refill(s);
                if constexpr (LEAN)
                    process_small(rows, heads, kmine, kprev, 0, cnt, r_base, wst);
                else
                    process(rows, heads, kmine, 0, cnt, r_base, wst);
            } else {
                // large stages of small rows: SUB rows at a time, buffer released after
                // (the lean loop holds full-warp collectives: a warp-uniform bound)
                const int cnt_loop = LEAN ? __reduce_max_sync(0xffffffffu, cnt) : cnt;
#pragma unroll 1
                for (int r0 = 0; r0 < cnt_loop; r0 += SUB) {
                    Raw rows[SUB][VPL];
#pragma unroll
                    for (int r = 0; r < SUB; ++r)
#pragma unroll
                        for (int j = 0; j < VPL; ++j)
                            rows[r][j] = ((LEAN || MODE == 0) ? (r0 + r < cnt && col_ok[j]) : true)
                                             ? lds_vec<Raw>(sbase + (r0 + r) * row_bytes + j * LPR * VB)
                                             : Raw{};
                    float wst[SUB];
#pragma unroll
                    for (int r = 0; r < SUB; ++r) wst[r] = (MODE == 2 && r0 + r < RS) ? wslots[r0 + r] : 1.0f;
                    if constexpr (LEAN)
                        process_small(rows, heads >> r0, kmine, kprev, r0, cnt - r0, r_base + r0, wst);
                    else
                        process(rows, heads >> r0, kmine, r0, cnt - r0, r_base + r0, wst);
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                refill(s);
            }
        }
    } else {
        // LDG path: the next stage's rows and key are loaded into registers
        // (128-bit ld.global.nc.L1::no_allocate) while the current one is reduced
        Raw nxt[RS][VPL];
        long long nkey = KEY_AFTER;
        auto fetch = [&](int s) {
            const long long rb = e_lo + (long long)s * RS;
            int c = (int)(e_hi - rb);
            c = c < 0 ? 0 : (c > RS ? RS : c);
            const T* base = X + rb * (long long)F;
#pragma unroll
            for (int r = 0; r < RS; ++r)
#pragma unroll
                for (int j = 0; j < VPL; ++j)
                    nxt[r][j] = (r < c && col_ok[j])
                                    ? ld_stream(reinterpret_cast<const Raw*>(base + (long long)r * F + vec_col(j) * VW))
                                    : Raw{};
            nkey = (li < c) ? key_ld(rb + li) : KEY_AFTER;
        };
        if (nst_w > 0) fetch(0);
#pragma unroll 1
        for (int s = 0; s < nst_w; ++s) {  // warp-uniform trip count (groups past their range idle)
            Raw rows[RS][VPL];
#pragma unroll
            for (int r = 0; r < RS; ++r)
#pragma unroll
                for (int j = 0; j < VPL; ++j) rows[r][j] = nxt[r][j];
            const long long kmine = nkey;
            if (s + 1 < nst_w) fetch(s + 1);
            const long long r_base = e_lo + (long long)s * RS;
            int cnt = (int)(e_hi - r_base);
            cnt = cnt < 0 ? 0 : (cnt > RS ? RS : cnt);
            long long kprev = __shfl_up_sync(0xffffffffu, kmine, 1, LPR);
            if (li == 0) kprev = cur;
            const unsigned heads = __ballot_sync(0xffffffffu, li < cnt && kmine != kprev) >> (gi * LPR);
            const float wst[SUB] = {};
            if constexpr (LEAN)
                process_small(rows, heads, kmine, kprev, 0, cnt, r_base, wst);
            else
                process(rows, heads, kmine, 0, cnt, r_base, wst);
        }
    }

#ifdef GEOT_TRACE
    if (li == 0 && a < 65536) g_trace_agent[a] = gtimer();
#endif
    // ---- agent end: publish the carries later agents need (H5) ...
    sync_acc();
    if (nrows > 0) {
        const bool tail_open = (nextk == cur);
        if (first && head_open) {
            flags |= TM_HEAD_OPEN;
            head_end = e_hi;
            if (tail_open) {  // the whole range lies inside one segment
                flags |= TM_TAIL_OPEN | TM_MIDDLE;
                carry_store(p.carry_h, acc);
            } else {
#pragma unroll
                for (int j = 0; j < VPL; ++j)
#pragma unroll
                    for (int q = 0; q < VW; ++q) hacc[j][q] = acc[j][q];
            }
        } else if (tail_open) {
            carry_store(p.carry_t, acc);
            flags |= TM_TAIL_OPEN;
        } else {
            write_row(cur, acc, e_hi - seg_start);
        }
        if (e_hi == p.E) gap_fill(cur, KEY_AFTER);
        if (tail_open) {  // some later agent owns this segment: publish (release)
            if (li == 0) {
                p.meta[a].flags = flags;
                p.meta[a].tail_start = seg_start;
            }
            __syncwarp(gmask);
            __threadfence();
            if (li == 0) st_release_u64(&p.flag[a], pub);
        }
    }
    __syncwarp();
    // ---- ... and own the segments that end here but began earlier: combine the
    // start agent's tail carry, the wholly-covered agents' carries and this
    // agent's head partial, in agent order (deterministic), write the row once.
    if (nrows > 0 && (flags & TM_HEAD_OPEN) && !(flags & TM_MIDDLE)) {
        long long u = a - 1;
        bool ok = true;
        for (; u >= 0; --u) {  // predecessors are consistent by construction: agent
                               // u's tail test and agent u+1's head test compare the same keys
            if (!wait_flag_or_poison(&p.flag[u], pub, p.ctrl)) {
                ok = false;
                break;
            }
            if (!(ld_volatile_i32(&p.meta[u].flags) & TM_MIDDLE)) break;
        }
        if (u < 0) u = 0;  // unreachable (agent 0 never has an open head)
        if (ok) {
            const long long count = head_end - ld_volatile_i64(&p.meta[u].tail_start);
            float tot[VPL][VW];
#pragma unroll
            for (int j = 0; j < VPL; ++j) {
                const int v = vec_col(j);
#pragma unroll
                for (int q = 0; q < VW; ++q) tot[j][q] = (v < p.NV) ? ld_cg_f32(p.carry_t + u * (long long)F + v * VW + q) : 0.f;
            }
            for (long long m = u + 1; m < a; ++m) {
#pragma unroll
                for (int j = 0; j < VPL; ++j) {
                    const int v = vec_col(j);
#pragma unroll
                    for (int q = 0; q < VW; ++q)
                        if (v < p.NV) tot[j][q] = fold<ISMAX>(tot[j][q], ld_cg_f32(p.carry_h + m * (long long)F + v * VW + q));
                }
            }
#pragma unroll
            for (int j = 0; j < VPL; ++j)
#pragma unroll
                for (int q = 0; q < VW; ++q) tot[j][q] = fold<ISMAX>(tot[j][q], hacc[j][q]);
            write_row(first_key, tot, count);
        }
    }
    // ---- last CTA out re-arms the control words for the next call
#ifdef GEOT_TRACE
    __syncthreads();
    if (threadIdx.x == 0 && s_ticket < 4096) g_trace_cta[s_ticket * 4 + 1] = gtimer();
#endif
    retire_cta(p.ctrl);
}

}  // namespace geot
