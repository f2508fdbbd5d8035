// split.cu — f4 "Alternative partition": the EXACT edge split
// of the sorted edge stream with a one-step exchange of the straddling
// partials (include/geot.h: geot_partition_exact, geot_segment_reduce_split,
// geot_combine_partials; reading R21).
//
// H9 (geot_partition) moves every split to a segment boundary, so parts never
// share a segment but a hub can unbalance them.  Here part p takes exactly
// edges [floor(pE/P), floor((p+1)E/P)); a segment cut by a split is reduced
// piecewise: each part reduces its own rows as usual, and additionally emits
// the fp32 partials of its head piece (the segment continuing from the left)
// and its tail piece (continuing to the right).  After an all-gather of those
// 2F floats per part (the exchange, shard.py), the part that holds the
// segment's FIRST edge folds the pieces in rank order and writes the row once
// — deterministic, no atomics.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>

#include "../../include/geot.h"
#include "common.cuh"

namespace geot {

extern std::atomic<unsigned long long> g_launches;

namespace {

constexpr int kSplitChunk = 1024;  // rows per sequentially folded chunk of a piece

__global__ void partition_exact_kernel(const void* idx, int idx64, long long E, long long S, int P, long long* seg_b,
                                       long long* edge_b, long long* keys) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p > P) return;
    const long long tp = (long long)(((unsigned __int128)p * (unsigned __int128)E) / (unsigned __int128)P);
    const long long before = tp > 0 ? load_index(idx, idx64, tp - 1) : -1;
    const long long at = tp < E ? load_index(idx, idx64, tp) : -1;
    long long sp;
    if (p == 0)
        sp = 0;
    else if (p == P)
        sp = S;
    else
        sp = tp == 0 ? 0 : before + 1;
    seg_b[p] = sp;
    edge_b[p] = tp;
    keys[2 * p] = before;
    keys[2 * p + 1] = at;
}

// first e in [lo, hi) with idx[e] > key (idx sorted; memory-safe otherwise)
__device__ long long upper_bound_key(const void* idx, int idx64, long long lo, long long hi, long long key) {
    while (lo < hi) {
        const long long mid = lo + ((hi - lo) >> 1);
        if (load_index(idx, idx64, mid) <= key)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}
// first e in [lo, hi) with idx[e] >= key
__device__ long long lower_bound_key(const void* idx, int idx64, long long lo, long long hi, long long key) {
    while (lo < hi) {
        const long long mid = lo + ((hi - lo) >> 1);
        if (load_index(idx, idx64, mid) < key)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

template <typename T>
__device__ __forceinline__ float ld_val(const T* p) {
    if constexpr (sizeof(T) == 4)
        return __ldg(reinterpret_cast<const float*>(p));
    else
        return __uint_as_float((uint32_t)__ldg(reinterpret_cast<const unsigned short*>(p)) << 16);
}

// The two pieces of this part: head = [0, h_end) (rows with idx[0]'s key),
// tail = [t_beg, E) (rows with idx[E-1]'s key); each cut into chunks of
// kSplitChunk rows, every chunk folded sequentially per column into
// chunk_part[(slot * maxch + c) * F + f].
template <typename T, bool ISMAX>
__global__ void split_chunk_kernel(const T* __restrict__ X, const void* idx, int idx64, long long E, int F,
                                   int head_open, int tail_open, float* __restrict__ chunk_part, long long maxch) {
    const long long k0 = load_index(idx, idx64, 0), kl = load_index(idx, idx64, E - 1);
    const long long h_end = head_open ? upper_bound_key(idx, idx64, 0, E, k0) : 0;
    const long long t_beg = tail_open ? lower_bound_key(idx, idx64, 0, E, kl) : E;
    const long long nh = (h_end + kSplitChunk - 1) / kSplitChunk;
    const long long nt = (E - t_beg + kSplitChunk - 1) / kSplitChunk;
    for (long long c = blockIdx.x; c < nh + nt; c += gridDim.x) {
        const int slot = c < nh ? 0 : 1;
        const long long cc = slot ? c - nh : c;
        const long long lo = (slot ? t_beg : 0) + cc * kSplitChunk;
        const long long hi = std::min(lo + kSplitChunk, slot ? E : h_end);
        for (int f = threadIdx.x; f < F; f += blockDim.x) {
            float acc = identity<ISMAX>();
            for (long long e = lo; e < hi; ++e) acc = fold<ISMAX>(acc, ld_val<T>(X + e * F + f));
            chunk_part[(slot * maxch + cc) * F + f] = acc;
        }
    }
}

// Block `slot` folds its piece's chunks in chunk order: partials[slot], counts[slot].
template <bool ISMAX>
__global__ void split_finish_kernel(const void* idx, int idx64, long long E, int F, int head_open, int tail_open,
                                    const float* __restrict__ chunk_part, long long maxch, float* partials,
                                    long long* counts) {
    const int slot = blockIdx.x;
    const bool open = slot == 0 ? head_open : tail_open;
    long long len = 0;
    if (open) {
        const long long k = load_index(idx, idx64, slot == 0 ? 0 : E - 1);
        len = slot == 0 ? upper_bound_key(idx, idx64, 0, E, k) : E - lower_bound_key(idx, idx64, 0, E, k);
    }
    const long long nch = (len + kSplitChunk - 1) / kSplitChunk;
    for (int f = threadIdx.x; f < F; f += blockDim.x) {
        float tot = open ? identity<ISMAX>() : 0.0f;
        for (long long c = 0; c < nch; ++c) tot = fold<ISMAX>(tot, chunk_part[(slot * maxch + c) * F + f]);
        partials[slot * (long long)F + f] = tot;
    }
    if (threadIdx.x == 0) counts[slot] = len;
}

constexpr int kMaxSlots = 64;
struct SlotList {
    int n;
    int s[kMaxSlots];
};

template <typename T, bool ISMAX>
__global__ void combine_kernel(const float* __restrict__ partials, const long long* __restrict__ counts, SlotList sl,
                               int F, int op, T* __restrict__ out_row) {
    long long count = 0;
    for (int k = 0; k < sl.n; ++k) count += counts[sl.s[k]];
    for (int f = threadIdx.x; f < F; f += blockDim.x) {
        float tot = identity<ISMAX>();
        for (int k = 0; k < sl.n; ++k) tot = fold<ISMAX>(tot, partials[(long long)sl.s[k] * F + f]);
        const float o[1] = {count > 0 ? finalize(tot, op, count) : 0.0f};
        reinterpret_cast<typename Conv<T, 1>::Raw*>(out_row)[f] = Conv<T, 1>::pack(o);
    }
}

geot_status cuda_status(cudaError_t e) { return e == cudaSuccess ? GEOT_OK : GEOT_ERR_CUDA; }

size_t split_extra_bytes(long long nnz, long long F) {
    const long long maxch = (nnz + kSplitChunk - 1) / kSplitChunk;
    return (size_t)(2 * maxch * F) * sizeof(float);
}

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }
// The piece partials go after the reduction's own workspace — and never below
// its first 256 bytes, the control words of the stream / narrow kernels (ticket,
// done, epoch, poison), even when this part needs no reduction workspace (a
// part inside one segment has num_segments = 0 and workspace size 0: placing the
// partials at offset 0 overwrote the control words of the cached workspace and
// poisoned every later call on it).
size_t split_chunk_offset(size_t red) { return align256(red < 256 ? 256 : red); }

}  // namespace
}  // namespace geot

using namespace geot;

extern "C" {

geot_status geot_partition_exact(const void* idx, geot_itype itype, int64_t nnz, int64_t num_segments, int nparts,
                                 int64_t* seg_bounds, int64_t* edge_bounds, int64_t* boundary_keys,
                                 cudaStream_t stream) {
    if ((int)itype < 0 || (int)itype > 1) return GEOT_ERR_INVALID_VALUE;
    if (nnz < 0 || num_segments < 0 || nparts < 1 || nparts > (1 << 20) || !seg_bounds || !edge_bounds ||
        !boundary_keys || (nnz > 0 && !idx))
        return GEOT_ERR_INVALID_VALUE;
    const int threads = 128;
    const int blocks = (nparts + 1 + threads - 1) / threads;
    partition_exact_kernel<<<blocks, threads, 0, stream>>>(idx, itype == GEOT_I64, nnz, num_segments, nparts,
                                                           reinterpret_cast<long long*>(seg_bounds),
                                                           reinterpret_cast<long long*>(edge_bounds),
                                                           reinterpret_cast<long long*>(boundary_keys));
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cuda_status(cudaGetLastError());
}

size_t geot_split_workspace_size(int64_t nnz, int64_t num_segments, int64_t F, geot_reduce op, geot_dtype dtype,
                                 geot_itype itype, const geot_config* cfg) {
    if (nnz <= 0 || F < 1) return 0;
    return split_chunk_offset(geot_workspace_size(nnz, num_segments, F, op, dtype, itype, 0, cfg)) +
           split_extra_bytes(nnz, F);
}

geot_status geot_segment_reduce_split(const void* src, const void* idx, int64_t nnz, int64_t seg_base,
                                      int64_t num_segments, int64_t F, geot_reduce op, geot_dtype dtype,
                                      geot_itype itype, int head_open, int tail_open, void* out, float* partials,
                                      int64_t* counts, void* workspace, size_t ws_bytes, const geot_config* cfg,
                                      cudaStream_t stream) {
    if ((int)op < 0 || (int)op > 2 || (int)dtype < 0 || (int)dtype > 1 || (int)itype < 0 || (int)itype > 1)
        return GEOT_ERR_INVALID_VALUE;
    if (nnz < 0 || num_segments < 0 || F < 1 || !partials || !counts) return GEOT_ERR_INVALID_VALUE;
    if (nnz == 0) {
        head_open = tail_open = 0;
    } else if (!src || !idx) {
        return GEOT_ERR_INVALID_VALUE;
    }
    const size_t red = nnz > 0 ? geot_workspace_size(nnz, num_segments, F, op, dtype, itype, 0, cfg) : 0;
    const size_t need = nnz > 0 ? split_chunk_offset(red) + split_extra_bytes(nnz, F) : 0;
    if (ws_bytes < need) return GEOT_ERR_WORKSPACE_TOO_SMALL;
    if (need > 0 && !workspace) return GEOT_ERR_INVALID_VALUE;
    // the part's own rows (a straddling head's row lies below seg_base: not written)
    geot_status st = geot_segment_reduce_ex(src, idx, nnz, seg_base, num_segments, F, op, dtype, itype, out,
                                            red ? workspace : nullptr, red, cfg, stream);
    if (st != GEOT_OK) return st;
    float* chunk = reinterpret_cast<float*>(static_cast<unsigned char*>(workspace) + split_chunk_offset(red));
    const long long maxch = (nnz + kSplitChunk - 1) / kSplitChunk;
    const bool ismax = op == GEOT_MAX;
    const int threads = F >= 256 ? 256 : (F >= 128 ? 128 : 64);
    if (head_open || tail_open) {
        int dev = 0, blocks = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&blocks, cudaDevAttrMultiProcessorCount, dev);
        blocks = (int)std::min<long long>(std::max(blocks, 1) * 4LL, 2 * maxch);
        const int i64 = itype == GEOT_I64;
        if (dtype == GEOT_F32) {
            if (ismax)
                split_chunk_kernel<float, true><<<blocks, threads, 0, stream>>>(
                    static_cast<const float*>(src), idx, i64, nnz, (int)F, head_open, tail_open, chunk, maxch);
            else
                split_chunk_kernel<float, false><<<blocks, threads, 0, stream>>>(
                    static_cast<const float*>(src), idx, i64, nnz, (int)F, head_open, tail_open, chunk, maxch);
        } else {
            if (ismax)
                split_chunk_kernel<__nv_bfloat16, true><<<blocks, threads, 0, stream>>>(
                    static_cast<const __nv_bfloat16*>(src), idx, i64, nnz, (int)F, head_open, tail_open, chunk, maxch);
            else
                split_chunk_kernel<__nv_bfloat16, false><<<blocks, threads, 0, stream>>>(
                    static_cast<const __nv_bfloat16*>(src), idx, i64, nnz, (int)F, head_open, tail_open, chunk, maxch);
        }
        g_launches.fetch_add(1, std::memory_order_relaxed);
    }
    if (ismax)
        split_finish_kernel<true><<<2, threads, 0, stream>>>(idx, itype == GEOT_I64, nnz, (int)F, head_open,
                                                             tail_open, chunk, maxch, partials,
                                                             reinterpret_cast<long long*>(counts));
    else
        split_finish_kernel<false><<<2, threads, 0, stream>>>(idx, itype == GEOT_I64, nnz, (int)F, head_open,
                                                              tail_open, chunk, maxch, partials,
                                                              reinterpret_cast<long long*>(counts));
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cuda_status(cudaGetLastError());
}

geot_status geot_combine_partials(const float* partials, const int64_t* counts, const int32_t* h_slots, int nslots,
                                  int64_t F, geot_reduce op, geot_dtype dtype, void* out_row, cudaStream_t stream) {
    if ((int)op < 0 || (int)op > 2 || (int)dtype < 0 || (int)dtype > 1) return GEOT_ERR_INVALID_VALUE;
    if (!partials || !counts || !h_slots || !out_row || nslots < 1 || nslots > kMaxSlots || F < 1)
        return GEOT_ERR_INVALID_VALUE;
    SlotList sl{};
    sl.n = nslots;
    for (int k = 0; k < nslots; ++k) {
        if (h_slots[k] < 0) return GEOT_ERR_INVALID_VALUE;
        sl.s[k] = h_slots[k];
    }
    const int threads = F >= 256 ? 256 : 128;
    const long long* cnt = reinterpret_cast<const long long*>(counts);
    if (dtype == GEOT_F32) {
        if (op == GEOT_MAX)
            combine_kernel<float, true><<<1, threads, 0, stream>>>(partials, cnt, sl, (int)F, (int)op,
                                                                   static_cast<float*>(out_row));
        else
            combine_kernel<float, false><<<1, threads, 0, stream>>>(partials, cnt, sl, (int)F, (int)op,
                                                                    static_cast<float*>(out_row));
    } else {
        if (op == GEOT_MAX)
            combine_kernel<__nv_bfloat16, true><<<1, threads, 0, stream>>>(partials, cnt, sl, (int)F, (int)op,
                                                                           static_cast<__nv_bfloat16*>(out_row));
        else
            combine_kernel<__nv_bfloat16, false><<<1, threads, 0, stream>>>(partials, cnt, sl, (int)F, (int)op,
                                                                            static_cast<__nv_bfloat16*>(out_row));
    }
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cuda_status(cudaGetLastError());
}

}  // extern "C"
