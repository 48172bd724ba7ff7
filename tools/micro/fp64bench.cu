// fp64bench.cu -- B200 FP64 latency / throughput probes for the pixel
// normaliser's sequential float64 chains (clock64 per warp).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64bench fp64bench.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>  // CH independent DADD chains per lane
__global__ void dadd_chain(int iters, double *out, long long *cyc) {
    double a[CH];
    for (int c = 0; c < CH; ++c) a[c] = threadIdx.x * 1e-3 + c;
    const double b = out[0] * 1e-30 + 1.0000001;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) a[c] = __dadd_rn(a[c], b);
    }
    long long t1 = clock64();
    double s = 0;
    for (int c = 0; c < CH; ++c) s += a[c];
    out[1 + blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int CH>  // F2F.F64.F32 throughput: independent conversions summed in float64
__global__ void f2f_tp(int iters, const float *in, double *out, long long *cyc) {
    double a[CH];
    for (int c = 0; c < CH; ++c) a[c] = 0;
    float v = in[threadIdx.x & 31];
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            a[c] = __dadd_rn(a[c], (double)v);
            v = __fadd_rn(v, 1.0f);
        }
    }
    long long t1 = clock64();
    double s = 0;
    for (int c = 0; c < CH; ++c) s += a[c];
    out[1 + blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <typename K>
void run(const char *name, K kern, int blocks, int threads, int iters, int ops_per_iter) {
    double *out;
    long long *cyc;
    float *in;
    cudaMalloc(&out, sizeof(double) * (1 + blocks * threads));
    cudaMemset(out, 0, sizeof(double) * (1 + blocks * threads));
    cudaMalloc(&cyc, sizeof(long long) * blocks);
    cudaMalloc(&in, 128);
    cudaMemset(in, 0, 128);
    kern(blocks, threads, iters, out, cyc, in);
    cudaDeviceSynchronize();
    kern(blocks, threads, iters, out, cyc, in);
    cudaDeviceSynchronize();
    long long c;
    cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
    printf("%-34s blocks %4d x %4d: %.2f cycles per iter (%d ops/lane/iter) err=%s\n", name, blocks,
           threads, (double)c / iters, ops_per_iter, cudaGetErrorString(cudaGetLastError()));
    cudaFree(out);
    cudaFree(cyc);
    cudaFree(in);
}

int main() {
    const int it = 1 << 14;
#define CHAIN(CH, B, T)                                                                      \
    run("dadd chains=" #CH, [](int b, int t, int i, double *o, long long *c, float *) {    \
        dadd_chain<CH><<<b, t>>>(i, o, c);                                                   \
    }, B, T, it, CH)
#define F2F(CH, B, T)                                                                        \
    run("f2f+dadd chains=" #CH, [](int b, int t, int i, double *o, long long *c, float *in) { \
        f2f_tp<CH><<<b, t>>>(i, in, o, c);                                                   \
    }, B, T, it, CH)
    CHAIN(1, 1, 32);
    CHAIN(2, 1, 32);
    CHAIN(4, 1, 32);
    CHAIN(8, 1, 32);
    CHAIN(1, 148, 128);
    CHAIN(4, 148, 128);
    CHAIN(4, 148, 256);
    CHAIN(8, 148, 512);
    F2F(1, 1, 32);
    F2F(4, 1, 32);
    F2F(8, 1, 32);
    F2F(4, 148, 128);
    F2F(8, 148, 512);
    return 0;
}
