// l2_gather.cu — ceiling of L2-resident random row gathers on this GPU (the
// roofline of the fused gather + segment-reduce path, H8; SURVEY §8(d):
// "Fused (Reddit-shaped) is bounded by L2/gather throughput").
//
// x: V rows of ROW bytes (Reddit-shaped: V = 232,965, ROW = 256 B -> 59.6 MB,
// L2-resident after the first touch).  N row ids drawn uniformly (splitmix64,
// the same recipe as the workload's src_idx).  Every warp gathers rows with
// 16-byte lane slices (ROW/16 lanes per row, as the stream kernel does) and
// folds them into registers; U rows per lane group in flight.  Two index
// sources: "hash" (ids computed in registers: a pure gather ceiling) and
// "stream" (ids read from an int32 array in HBM, 4 B per row, as the kernel
// does).  Reports gathered GB/s = N * ROW / t (best of reps, CUDA events).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_gather l2_gather.cu
//   ./l2_gather [V] [N]
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

__host__ __device__ inline uint64_t splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__global__ void make_ids(int* ids, long long n, unsigned V, uint64_t seed) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        ids[i] = (int)(splitmix64(seed + (uint64_t)i) % V);
}

__global__ void fill(float* x, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        x[i] = (float)(i & 1023) * 0.001f;
}

// LPR lanes per row (16-byte slices), G = 32/LPR rows per warp step, U steps in flight
template <int LPR, int U, bool STREAM_IDS>
__global__ void __launch_bounds__(512) gather(const uint4* __restrict__ x, const int* __restrict__ ids, long long n,
                                             unsigned V, uint64_t seed, float* sink) {
    constexpr int G = 32 / LPR;
    const int lane = threadIdx.x & 31, gi = lane / LPR, li = lane % LPR;
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    float acc0 = 0.f, acc1 = 0.f, acc2 = 0.f, acc3 = 0.f;
    // contiguous row ranges per warp (as the kernel's agents): rows r = base + step*G + gi
    const long long per = (n + nwarps - 1) / nwarps;
    const long long r0 = warp * per, r1 = min(n, r0 + per);
    for (long long r = r0 + gi; r < r1; r += (long long)G * U) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long rr = r + (long long)u * G;
            unsigned id;
            if constexpr (STREAM_IDS)
                id = rr < r1 ? (unsigned)__ldg(ids + rr) : 0u;
            else
                id = (unsigned)(splitmix64(seed + (uint64_t)rr) % V);
            const uint4* p = x + (size_t)id * LPR + li;
            asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                         : "l"(p));
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            acc0 += __uint_as_float(v[u].x);
            acc1 += __uint_as_float(v[u].y);
            acc2 += __uint_as_float(v[u].z);
            acc3 += __uint_as_float(v[u].w);
        }
    }
    if (acc0 + acc1 + acc2 + acc3 == 12345.678f) sink[0] = acc0;  // keep the loads alive
}

template <int LPR, int U, bool S>
float run(const uint4* x, const int* ids, long long n, unsigned V, float* sink, int blocks_per_sm, int nsm) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int grid = nsm * blocks_per_sm;
    gather<LPR, U, S><<<grid, 512>>>(x, ids, n, V, 7, sink);  // warm (x into L2)
    float best = 1e30f;
    for (int rep = 0; rep < 10; ++rep) {
        cudaEventRecord(a);
        gather<LPR, U, S><<<grid, 512>>>(x, ids, n, V, 7, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return best;
}

int main(int argc, char** argv) {
    const unsigned V = argc > 1 ? (unsigned)atol(argv[1]) : 232965u;
    const long long N = argc > 2 ? atoll(argv[2]) : 114615892LL;
    constexpr int ROW = 256;  // bytes (F = 64 fp32)
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    float* x;
    int* ids;
    float* sink;
    cudaMalloc(&x, (size_t)V * ROW);
    cudaMalloc(&ids, (size_t)N * 4);
    cudaMalloc(&sink, 4);
    fill<<<nsm * 8, 256>>>(x, (long long)V * ROW / 4);
    make_ids<<<nsm * 8, 256>>>(ids, N, V, 7);
    cudaDeviceSynchronize();
    const double bytes = (double)N * ROW;
    double best = 0;
    const char* best_name = "";
    auto report = [&](const char* name, float ms) {
        const double gbs = bytes / (ms * 1e-3) / 1e9;
        printf("{\"variant\": \"%s\", \"ms\": %.4f, \"gathered_GBps\": %.1f}\n", name, ms, gbs);
        if (gbs > best) {
            best = gbs;
            best_name = name;
        }
    };
    report("hash LPR16 U4 1cta", run<16, 4, false>((const uint4*)x, ids, N, V, sink, 1, nsm));
    report("hash LPR16 U8 1cta", run<16, 8, false>((const uint4*)x, ids, N, V, sink, 1, nsm));
    report("hash LPR16 U8 2cta", run<16, 8, false>((const uint4*)x, ids, N, V, sink, 2, nsm));
    report("hash LPR16 U16 2cta", run<16, 16, false>((const uint4*)x, ids, N, V, sink, 2, nsm));
    report("hash LPR16 U16 4cta", run<16, 16, false>((const uint4*)x, ids, N, V, sink, 4, nsm));
    report("stream LPR16 U8 2cta", run<16, 8, true>((const uint4*)x, ids, N, V, sink, 2, nsm));
    report("stream LPR16 U16 2cta", run<16, 16, true>((const uint4*)x, ids, N, V, sink, 2, nsm));
    report("stream LPR16 U16 4cta", run<16, 16, true>((const uint4*)x, ids, N, V, sink, 4, nsm));
    cudaError_t e = cudaGetLastError();
    printf("{\"best\": \"%s\", \"gbs\": %.1f, \"V\": %u, \"N\": %lld, \"row_bytes\": %d, \"err\": \"%s\"}\n", best_name, best,
           V, N, ROW, cudaGetErrorString(e));
    return e == cudaSuccess ? 0 : 1;
}
