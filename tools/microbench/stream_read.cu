// stream_read.cu — read-bandwidth ceiling experiments on B200 (tooling only).
//
// Measures, for a 4 GB buffer, the achieved HBM read bandwidth of
//   (a) per-warp TMA bulk-copy rings (cp.async.bulk + mbarrier) with W warps per
//       CTA, copy size C bytes, NS stages, consumer summing the stage from smem;
//   (b) plain 128-bit ld.global.nc loads with U loads in flight per thread.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_read stream_read.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int NS>
__global__ void tma_ring(const char* __restrict__ src, size_t bytes, int W, int C, float* sink) {
    extern __shared__ __align__(128) unsigned char sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char* buf = sm + (size_t)warp * NS * C;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + (size_t)W * NS * C) + warp * NS;
    const long long nw = (long long)gridDim.x * W;
    const long long w = (long long)blockIdx.x * W + warp;
    const long long chunks = bytes / C;
    const long long c0 = chunks * w / nw, c1 = chunks * (w + 1) / nw;
    const int n = (int)(c1 - c0);
    if (lane == 0) {
        for (int s = 0; s < NS; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[s])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncwarp();
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    auto issue = [&](int s) {
        const int b = s % NS;
        asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bars[b])),
                     "r"(C));
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
                "r"(smem_u32(buf + (size_t)b * C)),
            "l"(src + (c0 + s) * (long long)C), "r"(C), "r"(smem_u32(&bars[b])), "l"(pol)
            : "memory");
    };
    if (lane == 0)
        for (int s = 0; s < NS && s < n; ++s) issue(s);
    float acc = 0.f;
    for (int s = 0; s < n; ++s) {
        const int b = s % NS;
        uint32_t ok = 0;
        while (!ok)
            asm volatile(
                "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                : "=r"(ok)
                : "r"(smem_u32(&bars[b])), "r"((uint32_t)((s / NS) & 1))
                : "memory");
        const float4* f = reinterpret_cast<const float4*>(buf + (size_t)b * C);
        for (int i = lane; i < C / 16; i += 32) {
            float4 v = f[i];
            acc += v.x + v.y + v.z + v.w;
        }
        __syncwarp();
        if (lane == 0 && s + NS < n) issue(s + NS);
    }
    if (acc == 12345.f) sink[0] = acc;
}

template <int U>
__global__ void ldg_read(const float4* __restrict__ src, size_t n16, float* sink) {
    float acc = 0.f;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + (U - 1) * stride < n16; i += U * stride) {
        float4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const float4* p = src + i + u * stride;
            asm("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                : "=f"(v[u].x), "=f"(v[u].y), "=f"(v[u].z), "=f"(v[u].w)
                : "l"(p));
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
    }
    for (; i < n16; i += stride) acc += src[i].x;
    if (acc == 12345.f) sink[0] = acc;
}

int main() {
    const size_t bytes = 4ull << 30;
    char* src;
    float* sink;
    cudaMalloc(&src, bytes);
    cudaMalloc(&sink, 64);
    cudaMemset(src, 0, bytes);
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto timeit = [&](auto launch) {
        launch();
        cudaDeviceSynchronize();
        float best = 1e30f;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(a);
            launch();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
        }
        return bytes / (best * 1e-3) / 1e9;
    };
    struct P {
        int W, C, NS;
    };
    std::vector<P> ps = {{16, 3072, 4}, {16, 1536, 8}, {8, 6144, 4}, {8, 3072, 8}, {16, 2048, 6}, {8, 4096, 6},
                         {4, 12288, 4}, {4, 6144, 8}, {16, 1024, 8}, {32, 1536, 4}, {8, 12288, 2}, {2, 24576, 4}};
    for (auto p : ps) {
        const size_t smem = (size_t)p.W * p.NS * p.C + p.W * p.NS * 8;
        double gbs = -1;
        auto run = [&](auto kern) {
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            gbs = timeit([&] { kern<<<nsm, p.W * 32, smem>>>(src, bytes, p.W, p.C, sink); });
        };
        if (p.NS == 2) run(tma_ring<2>);
        if (p.NS == 4) run(tma_ring<4>);
        if (p.NS == 6) run(tma_ring<6>);
        if (p.NS == 8) run(tma_ring<8>);
        printf("TMA ring W=%2d C=%6d NS=%d smem=%6zu : %7.1f GB/s  %s\n", p.W, p.C, p.NS, smem, gbs,
               cudaGetErrorString(cudaGetLastError()));
    }
    for (int blocks_per_sm : {4, 8}) {
        const size_t n16 = bytes / 16;
        double g2 = timeit([&] { ldg_read<2><<<nsm * blocks_per_sm, 256>>>((const float4*)src, n16, sink); });
        double g4 = timeit([&] { ldg_read<4><<<nsm * blocks_per_sm, 256>>>((const float4*)src, n16, sink); });
        double g8 = timeit([&] { ldg_read<8><<<nsm * blocks_per_sm, 256>>>((const float4*)src, n16, sink); });
        printf("LDG.128 %d CTAs/SM x256: U=2 %7.1f  U=4 %7.1f  U=8 %7.1f GB/s\n", blocks_per_sm, g2, g4, g8);
    }
    return 0;
}
