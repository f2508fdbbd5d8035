// launch.cuh — host-side launchers of the kernel family (internal to libgeot).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unordered_map>

#include "edge_tile.cuh"
#include "stream.cuh"

namespace geot {

// Incremented once per kernel launch issued by the library (geot_launch_count).
extern std::atomic<unsigned long long> g_launches;
// geot_profile_events(): events bracketing the next main reduction kernel.
extern thread_local cudaEvent_t g_prof_before, g_prof_after;

struct LaunchInfo {
    int grid_x = 0, grid_y = 0, smem = 0;
};

// Occupancy (CTAs per SM) of one kernel instantiation at a given dynamic smem
// size; cached per (kernel, smem) because the query costs microseconds.
struct OccKey {
    const void* fn;
    size_t smem;
    int dev;
    bool operator==(const OccKey& o) const { return fn == o.fn && smem == o.smem && dev == o.dev; }
};
struct OccKeyHash {
    size_t operator()(const OccKey& k) const {
        return std::hash<const void*>()(k.fn) ^ (k.smem * 0x9E3779B97F4A7C15ull) ^ ((size_t)k.dev << 48);
    }
};

// The kernel's max-dynamic-smem attribute is ONE value per (function, device):
// it is only ever raised (to the largest size seen), never lowered, so a
// cached smaller size can never leave it below a later launch's need.
template <typename K>
int cached_occupancy(K kernel, int threads, size_t smem) {
    static std::mutex mu;
    static std::unordered_map<OccKey, int, OccKeyHash> cache;
    static std::unordered_map<OccKey, size_t, OccKeyHash> attr_set;  // smem field unused (0)
    int dev = 0;
    cudaGetDevice(&dev);
    const OccKey key{reinterpret_cast<const void*>(kernel), smem, dev};
    const OccKey fkey{reinterpret_cast<const void*>(kernel), 0, dev};
    std::lock_guard<std::mutex> lk(mu);
    if (smem > 48 * 1024) {
        size_t& cur = attr_set[fkey];
        if (smem > cur) {
            if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
                return 0;
            cur = smem;
        }
    }
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, threads, smem) != cudaSuccess) occ = 0;
    cache[key] = occ;
    return occ;
}

// H5 fix-up launch: programmatic dependent launch, so its launch overlaps the
// reduction kernel's tail (the kernel itself waits with griddepcontrol.wait).
template <typename T, bool ISMAX>
cudaError_t launch_fixup(const EdgeTileParams& p, cudaStream_t st) {
    if (p.ntiles <= 1) return cudaSuccess;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)((p.ntiles + 7) / 8));
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, carry_fixup_kernel<T, ISMAX>, p);
    if (e != cudaSuccess) return e;
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cudaSuccess;
}

template <typename T, int VW, int LPR, int VPL, int MODE, bool ISMAX>
cudaError_t run_edge_tile(const EdgeTileParams& p, int ctas_per_sm, int nsm, cudaStream_t st, LaunchInfo* li) {
    using Sh = TileShape<LPR, VPL, VW>;
    auto kern = edge_tile_kernel<T, VW, LPR, VPL, MODE, ISMAX>;
    const size_t smem = edge_tile_smem_bytes<LPR, VPL, VW>(p.tile_rows, MODE);
    if (smem > 227 * 1024) return cudaErrorInvalidValue;
    int occ = cached_occupancy(kern, 256, smem);
    if (occ <= 0) return cudaErrorInvalidConfiguration;
    if (ctas_per_sm > 0 && ctas_per_sm < occ) occ = ctas_per_sm;
    long long gx = (long long)nsm * occ;
    if (gx > p.ntiles) gx = p.ntiles;
    const int gy = (p.NV + Sh::FTV - 1) / Sh::FTV;
    dim3 grid((unsigned)gx, (unsigned)gy);
    if (g_prof_before) cudaEventRecord(g_prof_before, st);
    kern<<<grid, 256, smem, st>>>(p);
    if (g_prof_after) cudaEventRecord(g_prof_after, st);
    g_prof_before = g_prof_after = nullptr;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    g_launches.fetch_add(1, std::memory_order_relaxed);
    if (li) {
        li->grid_x = (int)gx;
        li->grid_y = gy;
        li->smem = (int)smem;
    }
    return launch_fixup<T, ISMAX>(p, st);
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no swizzle
// unless given, no interleave, 256-byte L2 promotion); false if unavailable.
bool encode_tensor_map(CUtensorMap* m, CUtensorMapDataType dt, int rank, const void* base, const cuuint64_t* dims,
                       const cuuint64_t* strides, const cuuint32_t* box, CUtensorMapSwizzle sw);

// Stream kernel: one persistent CTA per SM (fewer when nnz is small so every
// agent owns >= 1 row).  Agent count = carry slots.
long long stream_agents(long long nnz, int lpr, int warps, int nsm, int ctas_per_sm);

template <typename T, int VW, int LPR, int VPL, bool ISMAX, int W, int RS, int NS, int MODE = 0, bool SRC64 = false,
          bool REP = false>
cudaError_t run_stream(const StreamParams& p, const EdgeTileParams& fix, int nsm, cudaStream_t st) {
    constexpr int G = 32 / LPR;
    auto kern = stream_kernel<T, VW, LPR, VPL, ISMAX, W, RS, NS, MODE, SRC64, REP>;
    const size_t smem = stream_smem_bytes(W, NS, G, RS, p.row_bytes, MODE);
    if (smem > 227 * 1024) return cudaErrorNotSupported;
    const int occ = cached_occupancy(kern, W * 32, smem);
    if (occ < (NS > 0 ? 1 : 2)) return cudaErrorInvalidConfiguration;  // agents assume this many CTAs/SM
    const long long grid = p.NA / ((long long)W * G);
    if (grid < 1 || grid * W * G != p.NA) return cudaErrorInvalidValue;
    // the warp's value stages as one 3-D box: X viewed as [agent][stage][RS rows]
    // (uint64 elements: the box's inner extent RS * row_bytes <= 2048 bytes)
    StreamParams q = p;
    CUtensorMap tmx;
    std::memset(&tmx, 0, sizeof(tmx));
    q.tma3 = 0;
    static const bool no_tma3 = [] {  // experiments: GEOT_NO_TMA3=1 keeps the per-agent bulk copies
        const char* e = std::getenv("GEOT_NO_TMA3");
        return e && e[0] == '1';
    }();
    if constexpr (NS > 0 && MODE == 0 && G >= 4) {  // (stream.cuh EQL: equal-length agents)
        const long long sb = (long long)RS * p.row_bytes;
        if (!no_tma3 && p.NF >= 1 && sb % 16 == 0 && sb <= 2048 && p.L % RS == 0) {
            const cuuint64_t dims[3] = {(cuuint64_t)(sb / 8), (cuuint64_t)(p.L / RS), (cuuint64_t)p.NF};
            const cuuint64_t strides[2] = {(cuuint64_t)sb, (cuuint64_t)(p.L * p.row_bytes)};
            const cuuint32_t box[3] = {(cuuint32_t)(sb / 8), 1u, (cuuint32_t)G};
            q.tma3 = encode_tensor_map(&tmx, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, p.X, dims, strides, box,
                                       CU_TENSOR_MAP_SWIZZLE_NONE)
                         ? 1
                         : 0;
        }
    }
    if (g_prof_before) cudaEventRecord(g_prof_before, st);
    kern<<<(unsigned)grid, W * 32, smem, st>>>(q, tmx);
    if (g_prof_after) cudaEventRecord(g_prof_after, st);
    g_prof_before = g_prof_after = nullptr;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    g_launches.fetch_add(1, std::memory_order_relaxed);
    (void)fix;  // carries are resolved inside the stream kernel (no fix-up launch)
    return cudaSuccess;
}

// Compiled (lane shape) x (pipeline shape W warps / RS rows per stage / NS
// stages).  Lane shapes: 16-byte lane vectors, LPR lanes per row (32/LPR
// agents per warp), VPL vectors per lane; the first pipeline listed for a lane
// shape is its default (stream_default_pipe in select.cpp mirrors it).
template <typename T>
cudaError_t launch_stream(const StreamParams& p, const EdgeTileParams& fix, int vw, int lpr, int vpl, int w, int rs,
                          int ns, bool ismax, int nsm, cudaStream_t st) {
    constexpr int WIDE = 16 / (int)sizeof(T);
    if (vw != WIDE) return cudaErrorNotSupported;
    if (p.outs.n > 1) {  // f4 replicas: the default pipeline of each lane shape
#define GEOT_RSHAPE(LPR_, VPL_, W_, RS_, NS_)                                                              \
    if (lpr == LPR_ && vpl == VPL_)                                                                        \
        return ismax ? run_stream<T, WIDE, LPR_, VPL_, true, W_, RS_, NS_, 0, false, true>(p, fix, nsm, st)  \
                     : run_stream<T, WIDE, LPR_, VPL_, false, W_, RS_, NS_, 0, false, true>(p, fix, nsm, st);
        GEOT_RSHAPE(4, 1, 16, 4, 4)
        GEOT_RSHAPE(8, 1, 16, 6, 4)
        GEOT_RSHAPE(16, 1, 16, 6, 4)
        GEOT_RSHAPE(32, 1, 16, 6, 4)
        GEOT_RSHAPE(32, 2, 16, 3, 4)
        GEOT_RSHAPE(32, 4, 8, 3, 4)
        if constexpr (sizeof(T) == 4) {
            GEOT_RSHAPE(32, 8, 8, 1, 4)
        }
#undef GEOT_RSHAPE
        return cudaErrorNotSupported;
    }
#define GEOT_SSHAPE(LPR_, VPL_, W_, RS_, NS_)                                                        \
    if (lpr == LPR_ && vpl == VPL_ && w == W_ && rs == RS_ && ns == NS_)                             \
        return ismax ? run_stream<T, WIDE, LPR_, VPL_, true, W_, RS_, NS_>(p, fix, nsm, st)          \
                     : run_stream<T, WIDE, LPR_, VPL_, false, W_, RS_, NS_>(p, fix, nsm, st);
#define GEOT_SSHAPE_V1(LPR_)         \
    GEOT_SSHAPE(LPR_, 1, 16, 6, 4)   \
    GEOT_SSHAPE(LPR_, 1, 8, 6, 8)    \
    GEOT_SSHAPE(LPR_, 1, 16, 3, 8)   \
    GEOT_SSHAPE(LPR_, 1, 8, 8, 6)    \
    GEOT_SSHAPE(LPR_, 1, 8, 4, 0)    \
    GEOT_SSHAPE(LPR_, 1, 8, 8, 0)
    GEOT_SSHAPE(4, 1, 16, 4, 4) /* 64-byte rows: 8 agents per warp */
    GEOT_SSHAPE(4, 1, 8, 4, 8)
    GEOT_SSHAPE(4, 1, 8, 4, 0)
    GEOT_SSHAPE_V1(8)
    GEOT_SSHAPE_V1(16)
    GEOT_SSHAPE(16, 1, 16, 12, 2) /* 256-byte rows: deeper stages */
    GEOT_SSHAPE(16, 1, 16, 8, 3)
    GEOT_SSHAPE_V1(32)
    GEOT_SSHAPE(32, 1, 16, 12, 2) /* 512-byte rows: deeper stages (fewer per-stage overheads) */
    GEOT_SSHAPE(32, 1, 16, 8, 3)
    GEOT_SSHAPE(32, 2, 16, 3, 4)
    GEOT_SSHAPE(32, 2, 8, 3, 8)
    GEOT_SSHAPE(32, 2, 8, 4, 0)
    GEOT_SSHAPE(32, 4, 8, 3, 4)
    GEOT_SSHAPE(32, 4, 8, 2, 0)
    if constexpr (sizeof(T) == 4) {
        GEOT_SSHAPE(32, 8, 8, 1, 4)
        GEOT_SSHAPE(32, 8, 8, 1, 6)
        GEOT_SSHAPE(32, 8, 8, 1, 0)
    }
#undef GEOT_SSHAPE_V1
#undef GEOT_SSHAPE
    return cudaErrorNotSupported;
}
// Fused gather forms through the stream kernel (MODE 1: x[src[e]], 2: w[e] *
// x[src[e]]): 16-byte lane vectors, one vector per lane, two pipelines per lane shape.
template <typename T>
cudaError_t launch_stream_gather(const StreamParams& p, const EdgeTileParams& fix, int lpr, int vpl, int w, int rs,
                                 int ns, bool ismax, int mode, int nsm, cudaStream_t st) {
    constexpr int WIDE = 16 / (int)sizeof(T);
    if (vpl != 1 || (mode != 1 && mode != 2)) return cudaErrorNotSupported;
#define GEOT_GSHAPE_I(LPR_, W_, RS_, NS_, I64_)                                                                \
    if (mode == 2) return run_stream<T, WIDE, LPR_, 1, false, W_, RS_, NS_, 2, I64_>(p, fix, nsm, st);          \
    return ismax ? run_stream<T, WIDE, LPR_, 1, true, W_, RS_, NS_, 1, I64_>(p, fix, nsm, st)                   \
                 : run_stream<T, WIDE, LPR_, 1, false, W_, RS_, NS_, 1, I64_>(p, fix, nsm, st);
#define GEOT_GSHAPE(LPR_, W_, RS_, NS_)                                                                        \
    if (lpr == LPR_ && w == W_ && rs == RS_ && ns == NS_) {                                                    \
        if (p.idx64) {                                                                                         \
            GEOT_GSHAPE_I(LPR_, W_, RS_, NS_, true)                                                            \
        } else {                                                                                               \
            GEOT_GSHAPE_I(LPR_, W_, RS_, NS_, false)                                                           \
        }                                                                                                      \
    }
    GEOT_GSHAPE(4, 16, 4, 4)
    GEOT_GSHAPE(8, 16, 6, 4)
    GEOT_GSHAPE(16, 16, 6, 4)
    GEOT_GSHAPE(16, 16, 8, 3)
    GEOT_GSHAPE(16, 16, 12, 2)
    GEOT_GSHAPE(8, 16, 8, 3)
    GEOT_GSHAPE(32, 16, 8, 3)
    GEOT_GSHAPE(32, 16, 12, 2)
    GEOT_GSHAPE(32, 16, 6, 4)
#undef GEOT_GSHAPE_I
#undef GEOT_GSHAPE
    return cudaErrorNotSupported;
}
cudaError_t launch_stream_gather_f32(const StreamParams&, const EdgeTileParams&, int, int, int, int, int, bool, int,
                                     int, cudaStream_t);
cudaError_t launch_stream_gather_bf16(const StreamParams&, const EdgeTileParams&, int, int, int, int, int, bool, int,
                                      int, cudaStream_t);

// gradients (backward.cu)
cudaError_t launch_segment_backward(const void* dY, const void* idx, int idx64, long long E, long long seg_base,
                                    long long S, int F, int op, int bf16, const long long* offsets, const void* X,
                                    const void* Y, float* ties, void* dX, cudaStream_t st);
cudaError_t launch_gather_backward_x(const float* dY, const void* src, const void* dst, int idx64, const float* w,
                                     long long E, long long seg_base, long long S, long long V, int F, int op,
                                     const long long* offsets, float* dx, cudaStream_t st);
cudaError_t launch_sddmm(const float* x, const float* dY, const void* src, const void* dst, int idx64, long long E,
                         long long seg_base, long long S, long long V, int F, int op, const long long* offsets,
                         float* dw, cudaStream_t st);

// small-F kernel family (inst_narrow.cu)
struct NarrowParams;
cudaError_t launch_narrow(const NarrowParams& p, int F, bool bf16, bool ismax, bool i64, int nsm, cudaStream_t st);
long long narrow_agents_max(int nsm);

cudaError_t launch_stream_f32(const StreamParams&, const EdgeTileParams&, int, int, int, int, int, int, bool, int,
                              cudaStream_t);
cudaError_t launch_stream_bf16(const StreamParams&, const EdgeTileParams&, int, int, int, int, int, int, bool, int,
                               cudaStream_t);

// Switch over the compiled (VW, LPR, VPL, ISMAX) set for one (T, MODE).
// Compiled shapes: LPR in {1,2,4,8,16,32} with VPL = 1, and LPR = 32 with
// VPL in {2,4,8} (bf16 wide vectors: VPL <= 4).
template <typename T, int MODE>
cudaError_t launch_edge_tile(const EdgeTileParams& p, int vw, int lpr, int vpl, bool ismax, int ctas_per_sm,
                             int nsm, cudaStream_t st, LaunchInfo* li) {
    constexpr int WIDE = 16 / (int)sizeof(T);
#define GEOT_SHAPE(VW_, LPR_, VPL_)                                                                  \
    if (vw == VW_ && lpr == LPR_ && vpl == VPL_) {                                                   \
        return ismax ? run_edge_tile<T, VW_, LPR_, VPL_, MODE, true>(p, ctas_per_sm, nsm, st, li)    \
                     : run_edge_tile<T, VW_, LPR_, VPL_, MODE, false>(p, ctas_per_sm, nsm, st, li);  \
    }
#define GEOT_SHAPES_FOR_VW(VW_)  \
    GEOT_SHAPE(VW_, 1, 1)        \
    GEOT_SHAPE(VW_, 2, 1)        \
    GEOT_SHAPE(VW_, 4, 1)        \
    GEOT_SHAPE(VW_, 8, 1)        \
    GEOT_SHAPE(VW_, 16, 1)       \
    GEOT_SHAPE(VW_, 32, 1)       \
    GEOT_SHAPE(VW_, 32, 2)       \
    GEOT_SHAPE(VW_, 32, 4)
    GEOT_SHAPES_FOR_VW(WIDE)
    GEOT_SHAPES_FOR_VW(1)
    if constexpr (sizeof(T) == 4) {
        GEOT_SHAPE(WIDE, 32, 8)
        GEOT_SHAPE(1, 32, 8)
    }
#undef GEOT_SHAPES_FOR_VW
#undef GEOT_SHAPE
    return cudaErrorNotSupported;
}

// Explicit instantiation entry points (one translation unit each, compiled in
// parallel): inst_<dtype>_<mode>.cu
cudaError_t launch_edge_tile_f32_plain(const EdgeTileParams&, int, int, int, bool, int, int, cudaStream_t, LaunchInfo*);
cudaError_t launch_edge_tile_f32_gather(const EdgeTileParams&, int, int, int, bool, int, int, cudaStream_t, LaunchInfo*);
cudaError_t launch_edge_tile_f32_gatherw(const EdgeTileParams&, int, int, int, bool, int, int, cudaStream_t, LaunchInfo*);
cudaError_t launch_edge_tile_bf16_plain(const EdgeTileParams&, int, int, int, bool, int, int, cudaStream_t, LaunchInfo*);
cudaError_t launch_edge_tile_bf16_gather(const EdgeTileParams&, int, int, int, bool, int, int, cudaStream_t, LaunchInfo*);
cudaError_t launch_edge_tile_bf16_gatherw(const EdgeTileParams&, int, int, int, bool, int, int, cudaStream_t, LaunchInfo*);

}  // namespace geot
