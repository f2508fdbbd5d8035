// Instantiations of the fused-gather forms of the stream kernel (fp32 and bf16).
#include "launch.cuh"

namespace geot {
cudaError_t launch_stream_gather_f32(const StreamParams& p, const EdgeTileParams& fix, int lpr, int vpl, int w, int rs,
                                     int ns, bool ismax, int mode, int nsm, cudaStream_t st) {
    return launch_stream_gather<float>(p, fix, lpr, vpl, w, rs, ns, ismax, mode, nsm, st);
}
cudaError_t launch_stream_gather_bf16(const StreamParams& p, const EdgeTileParams& fix, int lpr, int vpl, int w,
                                      int rs, int ns, bool ismax, int mode, int nsm, cudaStream_t st) {
    return launch_stream_gather<__nv_bfloat16>(p, fix, lpr, vpl, w, rs, ns, ismax, mode, nsm, st);
}
}  // namespace geot
