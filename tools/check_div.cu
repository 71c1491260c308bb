// GPU check: div_rn(a, d, div_seed(d)) (rowkernels.cuh, the sweeps' shared-
// divisor division) returns the bits of __ddiv_rn(a, d) for every input.
// Inputs: uniformly random 64-bit patterns (all exponents, NaN/Inf/denormal
// included), the value ranges of the V-cycle (|a| in [1e-30, 1e30], d in
// [1e-8, 1e8]), and a table of special values crossed with each other.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a --fmad=false -O3 -std=c++17 -o check_div check_div.cu
// Prints "mismatches N of M" and exits 1 when N > 0.
#include "../paper_2508_12501_b200/csrc/rowkernels.cuh"

#include <cstdio>
#include <cstring>

namespace {

__device__ uint64_t mix(uint64_t z) {
    z += 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

__device__ double special(int k) {
    const double t[] = {0.0, -0.0, 1.0, -1.0, 3.0, 0.1, 1e-310, -1e-310, 4.9e-324, 2.2250738585072014e-308,
                        1.7976931348623157e308, -1.7976931348623157e308, __longlong_as_double(0x7ff0000000000000LL),
                        __longlong_as_double(0xfff0000000000000LL), __longlong_as_double(0x7ff8000000000000LL),
                        1e-300, 1e300, 2.0, 0.5, 6.0, 7.0, 1.0000000000000002, 0.9999999999999999};
    return t[k % 23];
}

__global__ void k_check(int64_t n, uint64_t seed, unsigned long long* bad, double* ex) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        const uint64_t r1 = mix(seed ^ (2 * i)), r2 = mix(seed ^ (2 * i + 1));
        double a, d;
        const int mode = static_cast<int>(i % 4);
        if (mode == 0) {  // any bit pattern
            a = __longlong_as_double(static_cast<long long>(r1));
            d = __longlong_as_double(static_cast<long long>(r2));
        } else if (mode == 1) {  // the V-cycle's ranges
            const double ua = (r1 >> 11) * (1.0 / 9007199254740992.0), ud = (r2 >> 11) * (1.0 / 9007199254740992.0);
            a = ((r1 & 1) ? -1.0 : 1.0) * exp10(-30.0 + 60.0 * ua);
            d = exp10(-8.0 + 16.0 * ud);
        } else if (mode == 2) {  // random mantissas, nearby exponents
            a = __longlong_as_double(static_cast<long long>((r1 & 0x800fffffffffffffULL) | (0x3ffULL << 52)));
            d = __longlong_as_double(static_cast<long long>((r2 & 0x000fffffffffffffULL) | (0x3feULL << 52)));
        } else {  // specials crossed, perturbed in the last bits
            a = special(static_cast<int>(r1 % 23));
            d = special(static_cast<int>(r2 % 23));
            if (r1 & 0x100) a = __longlong_as_double(__double_as_longlong(a) ^ static_cast<long long>((r1 >> 20) & 3));
        }
        const double ref = __ddiv_rn(a, d);
        const double got = decmg_gpu::div_rn(a, d, decmg_gpu::div_seed(d));
        if (__double_as_longlong(ref) != __double_as_longlong(got)) {
            const unsigned long long k = atomicAdd(bad, 1ULL);
            if (k < 4) {
                ex[4 * k] = a;
                ex[4 * k + 1] = d;
                ex[4 * k + 2] = ref;
                ex[4 * k + 3] = got;
            }
        }
    }
}

}  // namespace

int main(int argc, char** argv) {
    const int64_t n = argc > 1 ? std::atoll(argv[1]) : (1LL << 32);
    unsigned long long* bad;
    double* ex;
    cudaMalloc(&bad, sizeof(unsigned long long));
    cudaMalloc(&ex, 16 * sizeof(double));
    cudaMemset(bad, 0, sizeof(unsigned long long));
    k_check<<<148 * 8, 256>>>(n, 0x5eed5eedULL, bad, ex);
    unsigned long long h = 0;
    double hex[16];
    if (cudaMemcpy(&h, bad, sizeof(h), cudaMemcpyDeviceToHost) != cudaSuccess) {
        std::printf("CUDA error: %s\n", cudaGetErrorString(cudaGetLastError()));
        return 2;
    }
    cudaMemcpy(hex, ex, sizeof(hex), cudaMemcpyDeviceToHost);
    std::printf("mismatches %llu of %lld\n", h, static_cast<long long>(n));
    for (unsigned long long k = 0; k < h && k < 4; ++k)
        std::printf("  a=%.17g d=%.17g ddiv=%.17g div_rn=%.17g\n", hex[4 * k], hex[4 * k + 1], hex[4 * k + 2],
                    hex[4 * k + 3]);
    return h ? 1 : 0;
}
