// Microbenchmark of the exact parallel projection chain (csrc/seqsum.cuh):
// config-4-sized input (10,485,762 rows x 16 RHS, p = w*b with w ~ dual areas
// and b ~ U(-1,1)), per-kernel CUDA-event times over the 2^20-row passes, the
// walk's cycle split (tree build / tries / literal chains, -DSEQ_PROFILE) and a
// bitwise check against the host's sequential loop.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -std=c++17 -DSEQ_PROFILE \
//        -o tools/bench_seqwalk tools/bench_seqwalk.cu
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

#include "../paper_2508_12501_b200/csrc/seqsum.cuh"

using namespace decmg_gpu;

int main(int argc, char** argv) {
    const int n = argc > 1 ? std::atoi(argv[1]) : 10485762;
    const int nrhs = argc > 2 ? std::atoi(argv[2]) : 16;
    std::vector<double> w(n), b(static_cast<size_t>(n) * nrhs);
    std::mt19937_64 rng(7);
    std::uniform_real_distribution<double> u(0.0, 1.0);
    for (int i = 0; i < n; ++i) w[i] = (0.8 + 0.4 * u(rng)) * (4.0 * 3.141592653589793 / n);
    for (auto& v : b) v = 2.0 * u(rng) - 1.0;
    std::vector<double> ref(nrhs, 0.0);
    for (int i = 0; i < n; ++i)
        for (int l = 0; l < nrhs; ++l) ref[l] = ref[l] + w[i] * b[static_cast<size_t>(i) * nrhs + l];
    double *dw, *db, *dbuf, *dstate, *dmean;
    int* dfb;
    const size_t per = static_cast<size_t>(kSeqPassRecs) * nrhs;
    const size_t pstride = static_cast<size_t>((std::min(kSeqPassRows, n) + 3) & ~1);
    const size_t nodes_d = static_cast<size_t>(nrhs) * kSeqPassGrps * kGrpNodes * sizeof(SeqNode) / sizeof(double);
    cudaMalloc(&dw, sizeof(double) * n);
    cudaMalloc(&db, sizeof(double) * b.size());
    cudaMalloc(&dbuf, sizeof(double) * (2 * per + pstride * nrhs + nodes_d));
    cudaMalloc(&dstate, sizeof(double) * 32);
    cudaMalloc(&dmean, sizeof(double) * 32);
    cudaMalloc(&dfb, sizeof(int));
    cudaMemcpy(dw, w.data(), sizeof(double) * n, cudaMemcpyHostToDevice);
    cudaMemcpy(db, b.data(), sizeof(double) * b.size(), cudaMemcpyHostToDevice);
    double* approx = dbuf;
    double* guess = approx + per;
    double* prodT = guess + per;
    SeqNode* nodes = reinterpret_cast<SeqNode*>(prodT + pstride * nrhs);
    const int smax = kTileRows * 33 * static_cast<int>(sizeof(double));
    cudaFuncSetAttribute(k_seq_prod, cudaFuncAttributeMaxDynamicSharedMemorySize, smax);
    cudaFuncSetAttribute(k_seq_walk, cudaFuncAttributeMaxDynamicSharedMemorySize, kWalkSmem);
    const size_t smem = static_cast<size_t>(kTileRows) * (nrhs + 1) * sizeof(double);
    cudaEvent_t ev[5];
    for (auto& e : ev) cudaEventCreate(&e);
    for (int rep = 0; rep < 3; ++rep) {
        float tk[4] = {0, 0, 0, 0};
        cudaMemset(dstate, 0, sizeof(double) * 32);
        cudaMemset(dfb, 0, sizeof(int));
#ifdef SEQ_PROFILE
        unsigned long long z[6] = {0, 0, 0, 0, 0, 0};
        cudaMemcpyToSymbol(g_seq_prof, z, sizeof z);
#endif
        for (int a = 0; a < n; a += kSeqPassRows) {
            const int e = std::min(n, a + kSeqPassRows);
            const int ntile = (e - a + kTileRows - 1) / kTileRows;
            const int nrec = (e - a + kRecRows - 1) / kRecRows;
            const int ngrp = (e - a + kGrpRows - 1) / kGrpRows;
            const int stride = (e - a + 1) & ~1;
            cudaEventRecord(ev[0]);
            k_seq_prod<<<ntile, 256, smem>>>(a, e, nrhs, stride, dw, db, prodT, approx);
            cudaEventRecord(ev[1]);
            k_seq_guess<<<nrhs, 1024>>>(nrec, approx, dstate, guess);
            cudaEventRecord(ev[2]);
            k_seq_tree<<<dim3(ngrp, (nrhs + 3) / 4), 128>>>(a, e, nrhs, stride, prodT, guess, nodes);
            cudaEventRecord(ev[3]);
            k_seq_walk<<<nrhs, 32, kWalkSmem>>>(a, e, stride, prodT, nodes, dstate, 1.0, e >= n ? dmean : nullptr, dfb);
            cudaEventRecord(ev[4]);
            cudaEventSynchronize(ev[4]);
            for (int k = 0; k < 4; ++k) {
                float ms;
                cudaEventElapsedTime(&ms, ev[k], ev[k + 1]);
                tk[k] += ms;
            }
        }
        std::vector<double> got(nrhs);
        int fb = 0;
        cudaMemcpy(got.data(), dmean, sizeof(double) * nrhs, cudaMemcpyDeviceToHost);
        cudaMemcpy(&fb, dfb, sizeof(int), cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int l = 0; l < nrhs; ++l) bad += std::memcmp(&got[l], &ref[l], 8) != 0;
        std::printf("prod %.3f ms  guess %.3f ms  tree %.3f ms  walk %.3f ms  | fallback records %d of %lld | %s (%s)\n",
                    tk[0], tk[1], tk[2], tk[3], fb, static_cast<long long>((n + kRecRows - 1) / kRecRows) * nrhs,
                    bad ? "MISMATCH" : "bit-identical to the sequential loop", cudaGetErrorString(cudaGetLastError()));
#ifdef SEQ_PROFILE
        unsigned long long pr[6];
        cudaMemcpyFromSymbol(pr, g_seq_prof, sizeof pr);
        std::printf("  walk cycles summed over lanes: wait %.3g  tries %.3g (%llu tries)  literal %.3g  issue %.3g  total %.3g\n",
                    static_cast<double>(pr[0]), static_cast<double>(pr[1]), pr[3], static_cast<double>(pr[2]),
                    static_cast<double>(pr[5]), static_cast<double>(pr[4]));
#endif
    }
    return 0;
}
