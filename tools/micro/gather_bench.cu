// Random-gather ceiling on B200: sum of b[idx[k]] over 64M random indices into a 4M-entry
// (32 MB fp64) vector, idx streamed once.  Reports time and gathers/s for several
// loads-in-flight depths.  nvcc -O3 -gencode arch=compute_100a,code=sm_100a gather_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int U>
__global__ void gather_sum(const int *__restrict__ idx, const double *__restrict__ b, int64_t n, double *out) {
    double acc = 0.0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += stride * U) {
        int c[U];
        double g[U];
#pragma unroll
        for (int u = 0; u < U; ++u) c[u] = k + u * stride < n ? __ldcs(idx + k + u * stride) : 0;
#pragma unroll
        for (int u = 0; u < U; ++u) g[u] = __ldg(b + c[u]);
#pragma unroll
        for (int u = 0; u < U; ++u) acc += (k + u * stride < n) ? g[u] : 0.0;
    }
    if (acc == 12345.0) *out = acc;
}

__global__ void init_idx(int *idx, int64_t n, int m, uint64_t seed) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
        uint64_t z = (k + 1) * 0x9E3779B97F4A7C15ull ^ seed;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
        idx[k] = (int)(z % (uint64_t)m);
    }
}

template <int U>
void run(const int *idx, const double *b, int64_t n, double *out, int grid, int block) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    gather_sum<U><<<grid, block>>>(idx, b, n, out);
    cudaEventRecord(e0);
    const int reps = 10;
    for (int r = 0; r < reps; ++r) gather_sum<U><<<grid, block>>>(idx, b, n, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double us = ms * 1e3 / reps;
    printf("U=%2d grid=%6d block=%4d: %8.1f us  %6.1f G gathers/s  idx stream %6.1f GB/s\n", U, grid, block, us,
           n / us * 1e-3, n * 4.0 / us * 1e-3);
}

int main(int argc, char **argv) {
    const int64_t n = 64000000;
    int m = argc > 1 ? atoi(argv[1]) : 4000000;
    int *idx;
    double *b, *out;
    cudaMalloc(&idx, n * 4);
    cudaMalloc(&b, (size_t)m * 8);
    cudaMalloc(&out, 8);
    cudaMemset(b, 0, (size_t)m * 8);
    init_idx<<<4096, 256>>>(idx, n, m, 12345);
    cudaDeviceSynchronize();
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    printf("vector %d entries (%.1f MB), %lld gathers\n", m, m * 8e-6, (long long)n);
    for (int occ : {4, 8}) {
        run<1>(idx, b, n, out, sms * occ, 256);
        run<4>(idx, b, n, out, sms * occ, 256);
        run<8>(idx, b, n, out, sms * occ, 256);
        run<16>(idx, b, n, out, sms * occ, 256);
    }
    return 0;
}
