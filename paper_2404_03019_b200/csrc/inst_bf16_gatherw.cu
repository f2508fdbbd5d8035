// Instantiations of the edge-tile kernel family for dtype=bf16, mode=gatherw
// (split per translation unit so nvcc can compile them in parallel).
#include "launch.cuh"

namespace geot {
cudaError_t launch_edge_tile_bf16_gatherw(const EdgeTileParams& p, int vw, int lpr, int vpl, bool ismax,
                                       int ctas_per_sm, int nsm, cudaStream_t st, LaunchInfo* li) {
    return launch_edge_tile<__nv_bfloat16, 2>(p, vw, lpr, vpl, ismax, ctas_per_sm, nsm, st, li);
}
}  // namespace geot
