// edge_tile.cuh — the edge-parallel segment-reduction kernel (H4-H7, H8) and
// its deterministic tile-carry fix-up (H5).
//
// Paper mapping (§III):
//  * block tiling / thread-group tiling: a CTA owns a tile of
//    `tile_rows` consecutive edges (the M_b analog) for one feature tile of
//    LPR*VPL vectors (the N_b analog, grid.y); inside it NG = 8*32/LPR lane
//    groups each own R consecutive rows (M_t) x the feature tile (N_t).
//  * sequential reduction SR (Fig. 3 b.1): each lane group walks its R
//    rows in order, accumulating in fp32 registers, and commits at segment
//    ends — but with a plain exactly-once vector store instead of the paper's
//    atomicAdd, because every complete segment has exactly one owner.
//  * segment detection is the is_seg test of Alg. 1: a row starts
//    a segment iff its key differs from the previous row's key.
//  * partial segments at lane-group edges are combined in shared memory in
//    group order; partial segments at tile edges go to per-tile carries that
//    the fix-up kernel combines in tile order (no floating-point atomics:
//    bitwise reproducible; reading R8).
//  * empty segments (H6) are zero-filled by the group that owns the gap, so
//    `out` needs no memset (reading R1).
// Unlike the paper, the index (and the gathered row ids / weights of
// the fused form) of a tile is staged in shared memory: it is a contiguous
// stream, independent of where segments fall.
#pragma once

#include "common.cuh"

namespace geot {

template <int LPR, int VPL, int VW>
struct TileShape {
    static constexpr int kWarps = 8;
    static constexpr int G = 32 / LPR;         // lane groups per warp
    static constexpr int NG = kWarps * G;      // lane groups per CTA
    static constexpr int FTV = LPR * VPL;      // vectors per feature tile
    static constexpr int FTE = FTV * VW;       // elements per feature tile
    // rows in flight per lane group (loads issued before any is consumed)
    static constexpr int U = (VPL * VW >= 32) ? 2 : ((VPL * VW >= 16) ? 4 : 8);
};

__host__ __device__ inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Shared-memory bytes of one CTA for a tile of `tile_rows` rows.
template <int LPR, int VPL, int VW>
__host__ __device__ inline size_t edge_tile_smem_bytes(int tile_rows, int mode) {
    using S = TileShape<LPR, VPL, VW>;
    size_t b = 2ull * S::NG * S::FTE * sizeof(float);  // sH, sT
    b += 2ull * S::NG * sizeof(long long);              // head_end, tail_start
    b += S::NG * sizeof(int);                           // flags
    b = align_up(b, 16);
    b += (size_t)(tile_rows + 2) * sizeof(long long);   // keys
    if (mode >= 1) b += (size_t)tile_rows * sizeof(long long);  // gather rows
    if (mode >= 2) b += (size_t)tile_rows * sizeof(float);      // weights
    return b;
}

template <typename T, int VW, int LPR, int VPL, int MODE, bool ISMAX>
__global__ void __launch_bounds__(256) edge_tile_kernel(const EdgeTileParams p) {
    using Sh = TileShape<LPR, VPL, VW>;
    using Cv = Conv<T, VW>;
    using Raw = typename Cv::Raw;
    constexpr int G = Sh::G, NG = Sh::NG, FTV = Sh::FTV, FTE = Sh::FTE, U = Sh::U;

    extern __shared__ __align__(16) unsigned char smem_raw[];
    float* sH = reinterpret_cast<float*>(smem_raw);
    float* sT = sH + NG * FTE;
    long long* gHeadEnd = reinterpret_cast<long long*>(sT + NG * FTE);
    long long* gTailStart = gHeadEnd + NG;
    int* gFlags = reinterpret_cast<int*>(gTailStart + NG);
    long long* skey = reinterpret_cast<long long*>(
        smem_raw + align_up(2ull * NG * FTE * sizeof(float) + 2ull * NG * sizeof(long long) + NG * sizeof(int), 16));
    long long* ssrc = skey + p.tile_rows + 2;
    float* sw = reinterpret_cast<float*>(ssrc + p.tile_rows);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gi = lane / LPR;  // group within warp
    const int li = lane % LPR;  // lane within group
    const int g = warp * G + gi;
    const int fv0 = blockIdx.y * FTV;
    const long long seg_lo = p.seg_base, seg_hi = p.seg_base + p.S;  // valid keys [lo, hi)
    const int F = p.F;
    const T* __restrict__ X = static_cast<const T*>(p.X);

    auto vec_col = [&](int j) { return fv0 + li + j * LPR; };

    // exactly-once store of a finished segment row (H7 epilogue)
    auto write_row = [&](long long key, const float (&acc)[VPL][VW], long long count) {
        if (key < seg_lo || key >= seg_hi) return;
        for (int d = 0; d < p.outs.n; ++d) {
            T* rowp = static_cast<T*>(p.outs.ptr[d]) + (key - p.outs.row_off) * (long long)F;
#pragma unroll
            for (int j = 0; j < VPL; ++j) {
                const int v = vec_col(j);
                if (v < p.NV) {
                    float o[VW];
#pragma unroll
                    for (int q = 0; q < VW; ++q) o[q] = finalize(acc[j][q], p.op, count);
                    st_vec_mc(reinterpret_cast<Raw*>(rowp + (long long)v * VW), Cv::pack(o), out_is_mc(p.outs, d));
                }
            }
        }
    };
    // zero rows strictly between keys a and b (H6), clamped to [lo, hi)
    auto gap_fill = [&](long long a, long long b) {
        long long r0 = (a < seg_lo) ? seg_lo : a + 1;
        long long r1 = (b > seg_hi) ? seg_hi : b;  // exclusive
        float z[VW];
#pragma unroll
        for (int q = 0; q < VW; ++q) z[q] = 0.0f;
        const Raw zr = Cv::pack(z);
        for (int d = 0; d < p.outs.n; ++d)
            for (long long r = r0; r < r1; ++r) {
                T* rowp = static_cast<T*>(p.outs.ptr[d]) + (r - p.outs.row_off) * (long long)F;
#pragma unroll
                for (int j = 0; j < VPL; ++j) {
                    const int v = vec_col(j);
                    if (v < p.NV) st_vec_mc(reinterpret_cast<Raw*>(rowp + (long long)v * VW), zr, out_is_mc(p.outs, d));
                }
            }
    };
    auto slot_store = [&](float* base, int grp, const float (&acc)[VPL][VW]) {
#pragma unroll
        for (int j = 0; j < VPL; ++j)
#pragma unroll
            for (int q = 0; q < VW; ++q) base[(size_t)grp * FTE + (li + j * LPR) * VW + q] = acc[j][q];
    };
    auto slot_fold = [&](const float* base, int grp, float (&acc)[VPL][VW]) {
#pragma unroll
        for (int j = 0; j < VPL; ++j)
#pragma unroll
            for (int q = 0; q < VW; ++q)
                acc[j][q] = fold<ISMAX>(acc[j][q], base[(size_t)grp * FTE + (li + j * LPR) * VW + q]);
    };
    auto set_ident = [&](float (&acc)[VPL][VW]) {
#pragma unroll
        for (int j = 0; j < VPL; ++j)
#pragma unroll
            for (int q = 0; q < VW; ++q) acc[j][q] = identity<ISMAX>();
    };
    auto carry_store = [&](float* carry, long long tile, const float (&acc)[VPL][VW]) {
        float* c = carry + tile * (long long)F;
#pragma unroll
        for (int j = 0; j < VPL; ++j) {
            const int v = vec_col(j);
            if (v < p.NV)
#pragma unroll
                for (int q = 0; q < VW; ++q) c[(long long)v * VW + q] = acc[j][q];
        }
    };

    asm volatile("griddepcontrol.launch_dependents;");  // let the fix-up grid launch early (PDL)
    for (long long tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x) {
        const long long A = tile * p.tile_rows;
        const int n = (int)min((long long)p.tile_rows, p.E - A);

        // ---- stage the tile's keys (rows A-1 .. A+n) and gather metadata
        for (int i = threadIdx.x; i < n + 2; i += blockDim.x) {
            const long long e = A - 1 + i;
            long long k;
            if (e < 0)
                k = KEY_BEFORE;
            else if (e >= p.E)
                k = KEY_AFTER;
            else
                k = load_index(p.idx, p.idx64, e);
            skey[i] = k;
            if (MODE >= 1 && i >= 1 && i <= n) {
                ssrc[i - 1] = load_index(p.src, p.idx64, e);
                if (MODE == 2) sw[i - 1] = __ldg(p.w + e);
            }
        }
        __syncthreads();

        // ---- per-group sequential walk (SR analog)
        const int la = g * p.R;
        const int lb = min(la + p.R, n);
        const int glast = (n - 1) / p.R;
        if (la < lb) {
            int myflags = 0;
            long long headEnd = 0, tailStart = 0;
            long long cur = skey[la + 1];
            const long long prevk = skey[la];
            const bool head_open = (prevk == cur);
            if (!head_open) gap_fill(prevk, cur);
            int seg_start = la;
            bool first = true;
            float acc[VPL][VW];
            set_ident(acc);

            // per-lane column offsets (elements) and validity, loop invariant
            int coff[VPL];
            bool cok[VPL];
#pragma unroll
            for (int j = 0; j < VPL; ++j) {
                coff[j] = vec_col(j) * VW;
                cok[j] = vec_col(j) < p.NV;
            }
            // MODE 0: rows are contiguous; the row pointer advances by F per row
            const T* xbase = X + (MODE == 0 ? (A + la) * (long long)F : 0);

            auto fetch = [&](int l, const T* rowp, Raw (&r)[VPL], float& wt, bool& ok) {
                ok = true;
                wt = 1.0f;
                if constexpr (MODE != 0) {
                    const long long rr = ssrc[l];
                    ok = (rr >= 0 && rr < p.V);  // memory safety on bad data
                    rowp = X + (ok ? rr : 0) * (long long)F;
                    if constexpr (MODE == 2) wt = sw[l];
                }
#pragma unroll
                for (int j = 0; j < VPL; ++j) {
                    if (ok && cok[j]) {
                        const Raw* vp = reinterpret_cast<const Raw*>(rowp + coff[j]);
                        r[j] = (MODE == 0) ? ld_stream(vp) : ld_cached(vp);
                    } else {
                        r[j] = Raw{};
                    }
                }
            };
            auto consume = [&](int l, const Raw (&r)[VPL], float wt, bool ok) {
                const long long k = skey[l + 1];
                if (k != cur) {  // is_seg: segment `cur` ended at row l-1
                    if (first && head_open) {
                        slot_store(sH, g, acc);
                        myflags |= TM_HEAD_OPEN;
                        headEnd = A + l;
                    } else {
                        write_row(cur, acc, l - seg_start);
                    }
                    first = false;
                    gap_fill(cur, k);
                    cur = k;
                    seg_start = l;
                    set_ident(acc);
                }
                if (ok) {
#pragma unroll
                    for (int j = 0; j < VPL; ++j) {
                        float f[VW];
                        Cv::unpack(r[j], f);
#pragma unroll
                        for (int q = 0; q < VW; ++q)
                            if constexpr (MODE == 2) f[q] = wt * f[q];
                        if constexpr (!ISMAX && VW % 2 == 0) {  // packed fp32x2 adds (FADD2)
#pragma unroll
                            for (int q = 0; q < VW; q += 2) {
                                const float2 t =
                                    __fadd2_rn(make_float2(acc[j][q], acc[j][q + 1]), make_float2(f[q], f[q + 1]));
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

            int l0 = la;
            for (; l0 + U <= lb; l0 += U) {  // full groups of U rows: no bounds checks
                Raw raw[U][VPL];
                float wt[U];
                bool ok[U];
                const T* xl = xbase + (long long)(l0 - la) * F;
#pragma unroll
                for (int u = 0; u < U; ++u) fetch(l0 + u, xl + u * F, raw[u], wt[u], ok[u]);
#pragma unroll
                for (int u = 0; u < U; ++u) consume(l0 + u, raw[u], wt[u], ok[u]);
            }
            for (; l0 < lb; ++l0) {  // ragged remainder
                Raw raw[VPL];
                float wt;
                bool ok;
                fetch(l0, xbase + (long long)(l0 - la) * F, raw, wt, ok);
                consume(l0, raw, wt, ok);
            }
            const bool tail_open = (skey[lb + 1] == cur);
            if (first && head_open) {
                slot_store(sH, g, acc);
                myflags |= TM_HEAD_OPEN;
                headEnd = A + lb;
                if (tail_open) myflags |= TM_TAIL_OPEN | TM_MIDDLE;
            } else if (tail_open) {
                slot_store(sT, g, acc);
                myflags |= TM_TAIL_OPEN;
                tailStart = A + seg_start;
            } else {
                write_row(cur, acc, lb - seg_start);
            }
            if (A + lb == p.E) gap_fill(cur, KEY_AFTER);  // trailing empty segments
            if (li == 0) {
                gFlags[g] = myflags;
                gHeadEnd[g] = headEnd;
                gTailStart[g] = tailStart;
            }
        }
        __syncthreads();

        // ---- in-CTA combination of partial segments, in group order
        if (la < lb) {
            const int f = gFlags[g];
            if ((f & TM_HEAD_OPEN) && !(f & TM_MIDDLE)) {
                // head segment of group g ends inside g and began in an earlier group
                int u = g - 1;
                while (u >= 0 && (gFlags[u] & TM_MIDDLE)) --u;
                float acc[VPL][VW];
                set_ident(acc);
                if (u >= 0) slot_fold(sT, u, acc);
                for (int v = u + 1; v <= g; ++v) slot_fold(sH, v, acc);
                if (u >= 0) {
                    write_row(skey[la + 1], acc, gHeadEnd[g] - gTailStart[u]);
                } else {  // began before the tile: tile-head carry
                    carry_store(p.carry_h, tile, acc);
                    if (li == 0 && blockIdx.y == 0) p.meta[tile].head_end = gHeadEnd[g];
                }
            }
            if (g == glast && (f & TM_TAIL_OPEN)) {
                int u = g;
                while (u >= 0 && (gFlags[u] & TM_MIDDLE)) --u;
                float acc[VPL][VW];
                set_ident(acc);
                if (u >= 0) {
                    slot_fold(sT, u, acc);
                    for (int v = u + 1; v <= g; ++v) slot_fold(sH, v, acc);
                    carry_store(p.carry_t, tile, acc);
                    if (li == 0 && blockIdx.y == 0) p.meta[tile].tail_start = gTailStart[u];
                } else {  // the whole tile lies inside one segment
                    for (int v = 0; v <= g; ++v) slot_fold(sH, v, acc);
                    carry_store(p.carry_h, tile, acc);
                }
            }
        }
        if (threadIdx.x == 0 && blockIdx.y == 0 && p.meta) {  // a lone tile never carries
            int fl = 0;
            if (gFlags[0] & TM_HEAD_OPEN) fl |= TM_HEAD_OPEN;
            if (gFlags[glast] & TM_TAIL_OPEN) fl |= TM_TAIL_OPEN;
            bool mid = true;
            for (int v = 0; v <= glast; ++v) mid = mid && (gFlags[v] & TM_MIDDLE);
            if (mid) fl |= TM_MIDDLE;
            p.meta[tile].flags = fl;
            p.meta[tile].head_key = skey[1];
        }
        __syncthreads();
    }
}

// Fix-up (H5): one warp per tile whose head segment began in an earlier tile
// and ends in this one.  Combines, in tile order, the start tile's tail carry,
// the carries of the tiles lying wholly inside the segment, and this tile's
// head carry, in fp64, and writes the output row once.
template <typename T, bool ISMAX>
__global__ void __launch_bounds__(256) carry_fixup_kernel(const EdgeTileParams p) {
    asm volatile("griddepcontrol.wait;" ::: "memory");  // the reduction kernel's carries are complete
    const int lane = threadIdx.x & 31;
    const long long t = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (t >= p.ntiles) return;
    const TileMeta m = p.meta[t];
    if (!(m.flags & TM_HEAD_OPEN) || (m.flags & TM_MIDDLE)) return;
    // find the start tile u < t: the nearest earlier tile that is not MIDDLE
    long long u = -1;
    for (long long base = t - 1; base >= 0; base -= 32) {
        const long long c = base - lane;
        const bool stop = (c >= 0) && !(p.meta[c].flags & TM_MIDDLE);
        const unsigned bal = __ballot_sync(0xffffffffu, stop || c < 0);
        if (bal) {
            const int first = __ffs(bal) - 1;
            u = base - first;
            break;
        }
    }
    if (u < 0) return;
    const TileMeta mu = p.meta[u];
    if (!(mu.flags & TM_TAIL_OPEN)) return;  // inconsistent (unsorted) input
    const long long key = m.head_key;
    if (key < p.seg_base || key >= p.seg_base + p.S) return;
    const long long count = m.head_end - mu.tail_start;
    for (int f = lane; f < p.F; f += 32) {
        double acc = (double)p.carry_t[u * (long long)p.F + f];
        for (long long v = u + 1; v <= t; ++v) {
            const double x = (double)p.carry_h[v * (long long)p.F + f];
            acc = ISMAX ? fmax(acc, x) : acc + x;
        }
        float r = (float)acc;
        r = finalize(r, p.op, count);
        for (int d = 0; d < p.outs.n; ++d) {
            T* orow = static_cast<T*>(p.outs.ptr[d]) + (key - p.outs.row_off) * (long long)p.F;
            if constexpr (sizeof(T) == 4)
                st_vec_mc(reinterpret_cast<uint32_t*>(orow) + f, __float_as_uint(r), out_is_mc(p.outs, d));
            else  // (no multicast form for bf16 edge tiles: the host rejects it)
                reinterpret_cast<uint16_t*>(orow)[f] = f2bf_bits(r);
        }
    }
}

}  // namespace geot
