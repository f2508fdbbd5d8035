// synth.cu — device side of the shared seeded input generator (synth/__init__.py
// is the host side; the two are checked bit-for-bit by the GPU tests).
// Holds none of the method's arithmetic: it only draws inputs.
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// mode 0 real, 1 signed, 2 int; dtype 0 f32, 1 bf16 (see synth/__init__.py)
__device__ __forceinline__ float value_of(uint64_t h, int dtype, int mode) {
    if (mode == 2) return (float)((long long)(h % 17ull) - 8);
    if (dtype == 0) {
        const double k = (double)(h >> 40);
        return mode == 0 ? (float)(k * 0x1p-24) : (float)(k * 0x1p-23 - 1.0);
    }
    const double k = (double)(h >> 56);
    return mode == 0 ? (float)(k * 0x1p-8) : (float)(k * 0x1p-7 - 1.0);
}

__global__ void fill_values_kernel(void* out, int dtype, uint64_t base, long long e_begin, long long n_rows,
                                   long long F, int mode) {
    const long long total = n_rows * F;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
        const long long r = i / F, f = i - r * F;
        const uint64_t ctr = base + (uint64_t)(e_begin + r) * (uint64_t)F + (uint64_t)f;
        const float v = value_of(splitmix64(ctr), dtype, mode);
        if (dtype == 0)
            static_cast<float*>(out)[i] = v;
        else
            static_cast<uint16_t*>(out)[i] = (uint16_t)(__float_as_uint(v) >> 16);  // exact in bf16
    }
}

// idx[i] = s such that bounds[s] <= e_begin + i < bounds[s+1] (+ key_offset)
__global__ void expand_index_kernel(const long long* bounds, long long S, long long e_begin, long long n, void* out,
                                    int itype, long long key_offset) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const long long e = e_begin + i;
        long long lo = 0, hi = S;  // largest s with bounds[s] <= e
        while (hi - lo > 1) {
            const long long mid = (lo + hi) >> 1;
            if (bounds[mid] <= e)
                lo = mid;
            else
                hi = mid;
        }
        const long long k = lo + key_offset;
        if (itype == 0)
            static_cast<int*>(out)[i] = (int)k;
        else
            static_cast<long long*>(out)[i] = k;
    }
}

__global__ void src_index_kernel(void* out, int itype, uint64_t seed2, long long e_begin, long long n, long long V) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const long long r = (long long)(splitmix64(seed2 + (uint64_t)(e_begin + i)) % (uint64_t)V);
        if (itype == 0)
            static_cast<int*>(out)[i] = (int)r;
        else
            static_cast<long long*>(out)[i] = r;
    }
}

int grid_for(long long n) {
    long long b = (n + 255) / 256;
    if (b > 148 * 32) b = 148 * 32;
    if (b < 1) b = 1;
    return (int)b;
}

}  // namespace

extern "C" {

int synth_fill_values(void* out, int dtype, uint64_t seed, long long e_begin, long long n_rows, long long F, int mode,
                      cudaStream_t st) {
    if (n_rows <= 0) return 0;
    const uint64_t base = seed * 0x9E3779B97F4A7C15ull;
    fill_values_kernel<<<grid_for(n_rows * F), 256, 0, st>>>(out, dtype, base, e_begin, n_rows, F, mode);
    return (int)cudaGetLastError();
}

int synth_expand_index(const long long* bounds, long long S, long long e_begin, long long n, void* out, int itype,
                       long long key_offset, cudaStream_t st) {
    if (n <= 0) return 0;
    expand_index_kernel<<<grid_for(n), 256, 0, st>>>(bounds, S, e_begin, n, out, itype, key_offset);
    return (int)cudaGetLastError();
}

int synth_src_index(void* out, int itype, uint64_t seed2, long long e_begin, long long n, long long V,
                    cudaStream_t st) {
    if (n <= 0) return 0;
    src_index_kernel<<<grid_for(n), 256, 0, st>>>(out, itype, seed2, e_begin, n, V);
    return (int)cudaGetLastError();
}

}  // extern "C"
