// Microbenchmark: HBM bandwidth of 128-byte row traffic in a permuted order
// (the pattern of the sweeps' b reads and x' writes when the matrix rows are
// Morton-ordered but the vectors keep the reference numbering) vs in order.
// y[p[i]] = x[p[i]] + 1 for rows of 16 doubles, 4 threads per row, 256-bit
// accesses. p = identity, random, or random within aligned blocks of B rows.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bench_perm bench_perm.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <random>
#include <vector>

__global__ void __launch_bounds__(256) k_copy(int n, const int* __restrict__ p, const double* __restrict__ x,
                                              double* __restrict__ y) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t r = t / 4;
    if (r >= n) return;
    const int64_t o = static_cast<int64_t>(p[r]) * 16 + (t % 4) * 4;
    double a, b, c, d;
    asm volatile("ld.global.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(x + o));
    asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(y + o), "d"(a + 1), "d"(b + 1), "d"(c + 1),
                 "d"(d + 1)
                 : "memory");
}

int main(int argc, char** argv) {
    const int n = argc > 1 ? std::atoi(argv[1]) : 10485762;
    double *x, *y;
    int* dp;
    cudaMalloc(&x, sizeof(double) * 16 * n);
    cudaMalloc(&y, sizeof(double) * 16 * n);
    cudaMalloc(&dp, sizeof(int) * n);
    cudaMemset(x, 0, sizeof(double) * 16 * n);
    std::vector<int> p(n);
    std::mt19937_64 rng(7);
    const int blocks[] = {0, 1, 8, 64, 512, 4096, 1 << 30};
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int B : blocks) {
        std::iota(p.begin(), p.end(), 0);
        if (B > 1) {
            for (int s = 0; s < n; s += B) std::shuffle(p.begin() + s, p.begin() + std::min(n, s + B), rng);
        }
        cudaMemcpy(dp, p.data(), sizeof(int) * n, cudaMemcpyHostToDevice);
        const unsigned g = static_cast<unsigned>((4LL * n + 255) / 256);
        for (int w = 0; w < 3; ++w) k_copy<<<g, 256>>>(n, dp, x, y);
        cudaEventRecord(a);
        const int it = 20;
        for (int i = 0; i < it; ++i) k_copy<<<g, 256>>>(n, dp, x, y);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        ms /= it;
        const double bytes = static_cast<double>(n) * (256.0 + 4.0);
        std::printf("shuffle block %10d rows: %.3f ms  %.0f GB/s\n", B, ms, bytes / ms / 1e6);
    }
    return 0;
}
