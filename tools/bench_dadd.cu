// Microbenchmark: latency of a dependent fp64 add chain (DADD) on one warp,
// the floor of the projection's reference-order mean chain (k_project_sums):
// (1) operands in registers, (2) operands streamed from shared memory with
// LDS.64 (stride 16 doubles, the [rows][16] stage layout), (3) with LDS.128
// from a lane-contiguous layout.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -o bench_dadd bench_dadd.cu
#include <cstdio>

__global__ void k_chain(int n, const double* __restrict__ p, double* out, long long* cyc) {
    double s = 0.0;
    const double a = p[threadIdx.x], b = p[threadIdx.x + 32];
    const long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        s = __dadd_rn(s, a);
        s = __dadd_rn(s, b);
    }
    const long long t1 = clock64();
    out[threadIdx.x] = s;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}

__global__ void k_chain_lds(int reps, double* out, long long* cyc) {
    __shared__ double sm[256 * 16];
    for (int i = threadIdx.x; i < 256 * 16; i += 32) sm[i] = 1e-3 * i;
    __syncwarp();
    const int lane = threadIdx.x & 15;
    double s = 0.0;
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll 32
        for (int i = 0; i < 256; ++i) s = __dadd_rn(s, sm[i * 16 + lane]);
    }
    const long long t1 = clock64();
    out[threadIdx.x] = s;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}

__global__ void k_chain_lds128(int reps, double* out, long long* cyc) {
    __shared__ double sm[16 * 258];
    for (int i = threadIdx.x; i < 16 * 258; i += 32) sm[i] = 1e-3 * i;
    __syncwarp();
    const int lane = threadIdx.x & 15;
    const double2* row = reinterpret_cast<const double2*>(sm + lane * 258);
    double s = 0.0;
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll 16
        for (int i = 0; i < 128; ++i) {
            const double2 v = row[i];
            s = __dadd_rn(s, v.x);
            s = __dadd_rn(s, v.y);
        }
    }
    const long long t1 = clock64();
    out[threadIdx.x] = s;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
    double *p, *o;
    long long* c;
    cudaMalloc(&p, 64 * sizeof(double));
    cudaMalloc(&o, 32 * sizeof(double));
    cudaMalloc(&c, sizeof(long long));
    cudaMemset(p, 0, 64 * sizeof(double));
    long long h = 0;
    const int n = 1 << 20;
    for (int w = 0; w < 2; ++w) k_chain<<<1, 32>>>(n, p, o, c);
    cudaMemcpy(&h, c, sizeof h, cudaMemcpyDeviceToHost);
    std::printf("dependent DADD, register operands: %.2f cycles per add\n", static_cast<double>(h) / (2.0 * n));
    const int reps = 2048;
    cudaFuncSetAttribute(k_chain_lds, cudaFuncAttributeMaxDynamicSharedMemorySize, 0);
    for (int w = 0; w < 2; ++w) k_chain_lds<<<1, 32>>>(reps, o, c);
    cudaMemcpy(&h, c, sizeof h, cudaMemcpyDeviceToHost);
    std::printf("dependent DADD, LDS.64 operands:   %.2f cycles per add\n", static_cast<double>(h) / (256.0 * reps));
    for (int w = 0; w < 2; ++w) k_chain_lds128<<<1, 32>>>(reps, o, c);
    cudaMemcpy(&h, c, sizeof h, cudaMemcpyDeviceToHost);
    std::printf("dependent DADD, LDS.128 operands:  %.2f cycles per add\n", static_cast<double>(h) / (256.0 * reps));
    std::printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
