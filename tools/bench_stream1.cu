// Microbenchmark: how fast can ONE SM stream a [n][16] fp64 array from HBM
// (the projection chain's input)? Variants: TMA bulk ring (S stages x T
// bytes), plain 256-bit loads by W warps, and the same with the fp64 add
// chain of warp 0 consuming every value (the k_project_sums structure).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bench_stream1 bench_stream1.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mb_init(uint64_t* b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void mb_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t par) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(
            su32(b)),
        "r"(par)
        : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     su32(dst)),
                 "l"(src), "r"(bytes), "r"(su32(b))
                 : "memory");
}

// TMA ring; CHAIN: warp 0 lanes 0..15 add every value in row order
template <int CHAIN>
__global__ void k_tma(int64_t n_doubles, int stages, int tile_bytes, const double* __restrict__ src, double* out) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) uint64_t full[16], empty[16];
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            mb_init(&full[s], 1);
            mb_init(&empty[s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int per = tile_bytes / 8;
    const int64_t ntiles = n_doubles / per;
    if (threadIdx.x == 32) {
        for (int64_t c = 0; c < ntiles; ++c) {
            const int s = static_cast<int>(c % stages);
            if (c >= stages) mb_wait(&empty[s], static_cast<uint32_t>(((c / stages) - 1) & 1));
            mb_tx(&full[s], tile_bytes);
            bulk(sm + static_cast<size_t>(s) * tile_bytes, src + c * per, tile_bytes, &full[s]);
        }
    } else if (threadIdx.x < 32) {
        double acc = 0.0;
        const int lane = threadIdx.x;
        for (int64_t c = 0; c < ntiles; ++c) {
            const int s = static_cast<int>(c % stages);
            mb_wait(&full[s], static_cast<uint32_t>((c / stages) & 1));
            const double* t = reinterpret_cast<const double*>(sm + static_cast<size_t>(s) * tile_bytes);
            if (CHAIN == 1) {
                if (lane < 16)
                    for (int i = 0; i < per / 16; ++i) acc = __dadd_rn(acc, t[i * 16 + lane]);
            } else if (CHAIN == 2) {  // next 16 loaded while adding the current 16
                if (lane < 16) {
                    const double* pt = t + lane;
                    const int rows = per / 16;
                    double p[16], q[16];
#pragma unroll
                    for (int u = 0; u < 16; ++u) p[u] = pt[u * 16];
                    for (int i0 = 0; i0 < rows; i0 += 16) {
                        if (i0 + 16 < rows) {
#pragma unroll
                            for (int u = 0; u < 16; ++u) q[u] = pt[(i0 + 16 + u) * 16];
                        }
#pragma unroll
                        for (int u = 0; u < 16; ++u) acc = __dadd_rn(acc, p[u]);
#pragma unroll
                        for (int u = 0; u < 16; ++u) p[u] = q[u];
                    }
                }
            } else if (CHAIN == 3) {  // unroll 32, compiler-scheduled
                if (lane < 16) {
                    const int rows = per / 16;
#pragma unroll 32
                    for (int i = 0; i < rows; ++i) acc = __dadd_rn(acc, t[i * 16 + lane]);
                }
            } else {
                acc += t[lane];
            }
            __syncwarp();
            if (lane == 0) mb_arrive(&empty[s]);
        }
        out[threadIdx.x] = acc;
    }
}

// plain loads: all threads of the CTA stream 256-bit chunks, no consumer
__global__ void k_ldg(int64_t n_doubles, const double* __restrict__ src, double* out) {
    double acc = 0.0;
    for (int64_t i = threadIdx.x * 4; i < n_doubles; i += blockDim.x * 4 * 4) {
        double v[4][4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t j = i + u * blockDim.x * 4;
            if (j < n_doubles)
                asm volatile("ld.global.v4.f64 {%0, %1, %2, %3}, [%4];"
                             : "=d"(v[u][0]), "=d"(v[u][1]), "=d"(v[u][2]), "=d"(v[u][3])
                             : "l"(src + j));
            else
                v[u][0] = v[u][1] = v[u][2] = v[u][3] = 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) acc += v[u][0] + v[u][1] + v[u][2] + v[u][3];
    }
    out[threadIdx.x] = acc;
}

int main() {
    const int64_t n = 10485762LL * 16 / 8;  // 1/8 of config 4's 16-RHS vector: 168 MB
    double *src, *out;
    cudaMalloc(&src, sizeof(double) * n);
    cudaMalloc(&out, sizeof(double) * 1024);
    cudaMemset(src, 0, sizeof(double) * n);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto report = [&](const char* what) {
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        std::printf("%-44s %8.2f ms  %6.1f GB/s  %s\n", what, ms, 8.0 * n / ms / 1e6,
                    cudaGetErrorString(cudaGetLastError()));
    };
    const int cfg[][2] = {{8, 16384}, {6, 32768}, {3, 65536}, {2, 98304}};
    for (int chain : {0, 1, 2, 3}) {
        for (auto& c : cfg) {
            const size_t smem = static_cast<size_t>(c[0]) * c[1];
            auto k = chain == 0 ? k_tma<0> : chain == 1 ? k_tma<1> : chain == 2 ? k_tma<2> : k_tma<3>;
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
            k<<<1, 64, smem>>>(n, c[0], c[1], src, out);
            cudaEventRecord(a);
            k<<<1, 64, smem>>>(n, c[0], c[1], src, out);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            char buf[96];
            std::snprintf(buf, sizeof buf, "TMA chain%d stages=%d tile=%d", chain, c[0], c[1]);
            report(buf);
        }
    }
    for (int threads : {128, 256, 512, 1024}) {
        k_ldg<<<1, threads>>>(n, src, out);
        cudaEventRecord(a);
        k_ldg<<<1, threads>>>(n, src, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        char buf[96];
        std::snprintf(buf, sizeof buf, "LDG.256 threads=%d", threads);
        report(buf);
    }
    return 0;
}
