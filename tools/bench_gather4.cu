// Microbenchmark: gather 7 rows of x[n][16] (fp64, 128 B rows) per output row
// and write their sum -- the access pattern of the level-0 sweep -- with
// (A) register gathers (256-bit LDG per 4 lanes, as k_rowop_pipe does) and
// (B) TMA tile::gather4 into a shared-memory ring fed by a producer warp.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bench_gather4 bench_gather4.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                             \
    do {                                                                                  \
        cudaError_t e = (x);                                                              \
        if (e != cudaSuccess) {                                                           \
            std::printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
            std::exit(1);                                                                 \
        }                                                                                 \
    } while (0)

constexpr int W = 7;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// (A) register gathers: 4 threads per row, 4 doubles each (256-bit)
__global__ void __launch_bounds__(256) k_regs(int n, const int* __restrict__ idx, const double* __restrict__ x,
                                              double* __restrict__ y) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t r = t / 4;
    const int l0 = static_cast<int>(t % 4) * 4;
    if (r >= n) return;
    double xv[W][4];
#pragma unroll
    for (int j = 0; j < W; ++j) {
        const int c = idx[r * W + j];
        asm volatile("ld.global.v4.f64 {%0, %1, %2, %3}, [%4];"
                     : "=d"(xv[j][0]), "=d"(xv[j][1]), "=d"(xv[j][2]), "=d"(xv[j][3])
                     : "l"(x + static_cast<int64_t>(c) * 16 + l0));
    }
    double s[4] = {0, 0, 0, 0};
#pragma unroll
    for (int j = 0; j < W; ++j)
#pragma unroll
        for (int l = 0; l < 4; ++l) s[l] += xv[j][l];
    asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(y + r * 16 + l0), "d"(s[0]), "d"(s[1]), "d"(s[2]),
                 "d"(s[3])
                 : "memory");
}

// (B) TMA gather4: tile = ROWS rows x W entries; producer lane issues
// ROWS*W/4 gather4 ops per tile into stage s; 224 consumers (56 rows x 4).
constexpr int ROWS = 56, STAGES = 3, CONS = 224;
constexpr int STAGE_BYTES = ROWS * W * 128;

__global__ void __launch_bounds__(CONS + 32, 1) k_tma(int n, const int* __restrict__ idx,
                                                       const __grid_constant__ CUtensorMap tmap,
                                                       double* __restrict__ y) {
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
    const int tid = threadIdx.x;
    const int ntiles = (n + ROWS - 1) / ROWS;
    const int per = (ntiles + gridDim.x - 1) / gridDim.x;
    const int t0 = blockIdx.x * per, t1 = min(t0 + per, ntiles);
    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&full[s])), "r"(1));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&empty[s])), "r"(CONS / 32));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto wait = [](uint64_t* bar, uint32_t par) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(
                smem_u32(bar)),
            "r"(par)
            : "memory");
    };
    if (tid == CONS) {
        int i = 0;
        for (int t = t0; t < t1; ++t, ++i) {
            const int s = i % STAGES;
            if (i >= STAGES) wait(&empty[s], ((i / STAGES) - 1) & 1);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])),
                         "r"(STAGE_BYTES)
                         : "memory");
            unsigned char* st = smem + static_cast<size_t>(s) * STAGE_BYTES;
            const int* ti = idx + static_cast<int64_t>(t) * ROWS * W;
            for (int q = 0; q < ROWS * W; q += 4) {
                int c0 = ti[q], c1 = ti[q + 1], c2 = ti[q + 2], c3 = ti[q + 3];
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                    " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(st + q * 128)),
                    "l"(&tmap), "r"(smem_u32(&full[s])), "r"(0), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
                    : "memory");
            }
        }
    } else if (tid < CONS) {
        const int q = tid / 4, l0 = (tid % 4) * 4;
        int i = 0;
        for (int t = t0; t < t1; ++t, ++i) {
            const int s = i % STAGES;
            wait(&full[s], (i / STAGES) & 1);
            const double* st = reinterpret_cast<const double*>(smem + static_cast<size_t>(s) * STAGE_BYTES);
            double sum[4] = {0, 0, 0, 0};
#pragma unroll
            for (int j = 0; j < W; ++j) {
                const double4 v = *reinterpret_cast<const double4*>(st + (q * W + j) * 16 + l0);
                sum[0] += v.x;
                sum[1] += v.y;
                sum[2] += v.z;
                sum[3] += v.w;
            }
            __syncwarp();
            if ((tid & 31) == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s])) : "memory");
            const int64_t r = static_cast<int64_t>(t) * ROWS + q;
            if (r < n)
                asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(y + r * 16 + l0), "d"(sum[0]),
                             "d"(sum[1]), "d"(sum[2]), "d"(sum[3])
                             : "memory");
        }
    }
}

int main(int argc, char** argv) {
    const int n = argc > 1 ? std::atoi(argv[1]) : 10485762;
    const int spread = argc > 2 ? std::atoi(argv[2]) : 3000;  // neighbour index distance (Morton-like locality)
    const int ntiles = (n + ROWS - 1) / ROWS;
    const int npad = ntiles * ROWS;
    std::vector<int> idx(static_cast<size_t>(npad) * W);
    const int off[W] = {0, -1, 1, -spread, spread, -spread - 1, spread + 1};
    for (int64_t r = 0; r < npad; ++r)
        for (int j = 0; j < W; ++j) {
            int64_t c = r + off[j];
            if (c < 0) c = 0;
            if (c >= n) c = n - 1;
            idx[r * W + j] = static_cast<int>(c);
        }
    double *x, *y;
    int* d_idx;
    CK(cudaMalloc(&x, sizeof(double) * 16 * n));
    CK(cudaMalloc(&y, sizeof(double) * 16 * npad));
    CK(cudaMalloc(&d_idx, sizeof(int) * idx.size()));
    CK(cudaMemcpy(d_idx, idx.data(), sizeof(int) * idx.size(), cudaMemcpyHostToDevice));
    CK(cudaMemset(x, 0, sizeof(double) * 16 * n));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    CUtensorMap tmap;
    cuuint64_t gdim[2] = {16, static_cast<cuuint64_t>(n)};
    cuuint64_t gstride[1] = {16 * sizeof(double)};
    cuuint32_t box[2] = {16, 1};
    cuuint32_t estr[2] = {1, 1};
    CUresult cr = cuTensorMapEncodeTiled(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, x, gdim, gstride, box, estr,
                                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                         CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) {
        std::printf("encode failed %d\n", static_cast<int>(cr));
        return 1;
    }
    const size_t smem = static_cast<size_t>(STAGES) * STAGE_BYTES;
    CK(cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    const double bytes = static_cast<double>(n) * (128.0 /*x once*/ + 128.0 /*y*/ + 4.0 * W);
    for (int rep = 0; rep < 2; ++rep) {
        for (int mode = 0; mode < 2; ++mode) {
            for (int w = 0; w < 2; ++w) {
                if (mode == 0)
                    k_regs<<<static_cast<unsigned>((4LL * n + 255) / 256), 256>>>(n, d_idx, x, y);
                else
                    k_tma<<<sms, CONS + 32, smem>>>(n, d_idx, tmap, y);
            }
            CK(cudaEventRecord(a));
            const int iters = 10;
            for (int it = 0; it < iters; ++it) {
                if (mode == 0)
                    k_regs<<<static_cast<unsigned>((4LL * n + 255) / 256), 256>>>(n, d_idx, x, y);
                else
                    k_tma<<<sms, CONS + 32, smem>>>(n, d_idx, tmap, y);
            }
            CK(cudaEventRecord(b));
            CK(cudaEventSynchronize(b));
            CK(cudaGetLastError());
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, a, b));
            ms /= iters;
            std::printf("%s n=%d spread=%d: %.3f ms  %.0f GB/s (unique bytes)  %.0f GB/s (gathered bytes)\n",
                        mode == 0 ? "regs  " : "gather4", n, spread, ms, bytes / ms / 1e6,
                        static_cast<double>(n) * (128.0 * W + 128 + 4.0 * W) / ms / 1e6);
        }
    }
    return 0;
}
