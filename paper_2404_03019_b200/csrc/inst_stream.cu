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

#ifdef GEOT_TRACE
// experiments only: copy the trace stamps of the last stream-kernel launch to the host
extern "C" int geot_debug_trace(unsigned long long* cta, int ncta4, unsigned long long* agents, int nagents) {
    if (cudaMemcpyFromSymbol(cta, geot::g_trace_cta, sizeof(unsigned long long) * ncta4) != cudaSuccess) return 1;
    if (cudaMemcpyFromSymbol(agents, geot::g_trace_agent, sizeof(unsigned long long) * nagents) != cudaSuccess) return 1;
    return 0;
}
#endif
