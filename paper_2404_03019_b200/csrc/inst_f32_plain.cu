// Instantiations of the edge-tile kernel family for dtype=f32, mode=plain
// (split per translation unit so nvcc can compile them in parallel).
#include "launch.cuh"

namespace geot {
cudaError_t launch_edge_tile_f32_plain(const EdgeTileParams& p, int vw, int lpr, int vpl, bool ismax,
                                       int ctas_per_sm, int nsm, cudaStream_t st, LaunchInfo* li) {
    return launch_edge_tile<float, 0>(p, vw, lpr, vpl, ismax, ctas_per_sm, nsm, st, li);
}
}  // namespace geot
