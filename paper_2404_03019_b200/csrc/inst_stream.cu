// Instantiations of the TMA-streaming kernel family (fp32 and bf16).
#include "launch.cuh"

namespace geot {
cudaError_t launch_stream_f32(const StreamParams& p, const EdgeTileParams& fix, int vw, int lpr, int vpl, int w, int rs,
                              int ns, bool ismax, int nsm, cudaStream_t st) {
    return launch_stream<float>(p, fix, vw, lpr, vpl, w, rs, ns, ismax, nsm, st);
}
cudaError_t launch_stream_bf16(const StreamParams& p, const EdgeTileParams& fix, int vw, int lpr, int vpl, int w,
                               int rs, int ns, bool ismax, int nsm, cudaStream_t st) {
    return launch_stream<__nv_bfloat16>(p, fix, vw, lpr, vpl, w, rs, ns, ismax, nsm, st);
}
}  // namespace geot
