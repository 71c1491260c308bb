// Cost of one grid-wide barrier (cooperative_groups grid.sync) vs a cluster
// barrier and a block barrier on the B200, 148 x k CTAs of 256 threads.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bench_gridsync tools/bench_gridsync.cu
#include <cooperative_groups.h>
#include <cstdio>

namespace cg = cooperative_groups;

__global__ void k_grid(int iters, int* sink) {
    cg::grid_group g = cg::this_grid();
    int v = 0;
    for (int i = 0; i < iters; ++i) {
        v += threadIdx.x;
        g.sync();
    }
    if (v == -1) *sink = v;
}
__global__ void __cluster_dims__(8, 1, 1) k_cluster(int iters, int* sink) {
    cg::cluster_group c = cg::this_cluster();
    int v = 0;
    for (int i = 0; i < iters; ++i) {
        v += threadIdx.x;
        c.sync();
    }
    if (v == -1) *sink = v;
}
__global__ void k_block(int iters, int* sink) {
    int v = 0;
    for (int i = 0; i < iters; ++i) {
        v += threadIdx.x;
        __syncthreads();
    }
    if (v == -1) *sink = v;
}

int main() {
    int* sink;
    cudaMalloc(&sink, 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 2000;
    for (int per_sm : {1, 2, 4}) {
        void* args[] = {(void*)&iters, (void*)&sink};
        cudaLaunchCooperativeKernel((void*)k_grid, 148 * per_sm, 256, args, 0, 0);
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((void*)k_grid, 148 * per_sm, 256, args, 0, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("grid.sync  %3d CTAs: %.3f us per barrier (%s)\n", 148 * per_sm, 1e3 * ms / iters,
               cudaGetErrorString(cudaGetLastError()));
    }
    k_cluster<<<144, 256>>>(iters, sink);
    cudaEventRecord(a);
    k_cluster<<<144, 256>>>(iters, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("cluster.sync (8 CTAs): %.3f us per barrier (%s)\n", 1e3 * ms / iters, cudaGetErrorString(cudaGetLastError()));
    k_block<<<1, 256>>>(iters, sink);
    cudaEventRecord(a);
    k_block<<<1, 256>>>(iters, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("__syncthreads (1 CTA): %.3f us per barrier\n", 1e3 * ms / iters);
    return 0;
}
