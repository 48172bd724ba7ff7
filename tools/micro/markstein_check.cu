// markstein_check.cu -- exhaustive-ish check that the pixel normaliser's
// reciprocal + one-correction quotient equals __ddiv_rn (pixels.cuh).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mk markstein_check.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ uint64_t mix(uint64_t z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

__global__ void check(uint64_t seed, int per, unsigned long long *bad) {
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long nb = 0;
    for (int i = 0; i < per; ++i) {
        const uint64_t h = mix(seed ^ (t * 1315423911ull + i));
        const uint64_t g = mix(h);
        // a: [-2^40, 2^40] with random exponents; sd: (2^-60, 2^60)
        const int ea = (int)(h >> 52) % 80 - 60, eb = (int)(g >> 52) % 120 - 60;
        const double a = ldexp((double)(int64_t)(h & 0xfffffffffffffull) / 4503599627370496.0 *
                                   ((h >> 63) ? -1.0 : 1.0) + ((h >> 63) ? -1.0 : 1.0), ea);
        double sd = ldexp(1.0 + (double)(g & 0xfffffffffffffull) / 4503599627370496.0, eb);
        if ((i & 15) == 0)  // significands next to all ones (1/sd next to a power of two)
            sd = ldexp(2.0 - ldexp((double)(1 + (g & 0xff)), -52), eb);
        const double r = __ddiv_rn(1.0, sd);
        const double q0 = __dmul_rn(a, r);
        const double q = __fma_rn(__fma_rn(-q0, sd, a), r, q0);
        if (q != __ddiv_rn(a, sd)) ++nb;
    }
    atomicAdd(bad, nb);
}

int main() {
    unsigned long long *bad, h = 0;
    cudaMalloc(&bad, 8);
    cudaMemset(bad, 0, 8);
    const int blocks = 148 * 16, threads = 256, per = 1024;
    for (int rep = 0; rep < 8; ++rep) check<<<blocks, threads>>>(rep * 7919ull + 1, per, bad);
    cudaMemcpy(&h, bad, 8, cudaMemcpyDeviceToHost);
    printf("markstein: %llu mismatches of %llu quotients (%s)\n", h,
           8ull * blocks * threads * per, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
