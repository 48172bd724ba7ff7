// Latency of the float64 cartpole step chain (the bit-exact path: --fmad=false,
// IEEE division, libdevice sin/cos) in one warp.  Build with --fmad=false.
#include <cstdio>
#include "../../paper_2502_08844_b200/csrc/tasks.cuh"

using namespace dk;

template <int V>
__global__ void chain(double *out, long long *cyc, int steps, Params<double> p) {
    Cartpole<double>::W w;
    w.x = 0.1 * threadIdx.x / 32.; w.th = 0.05; w.xd = 0.; w.thd = 0.01;
    Cartpole<double>::refresh(w);
    long long t0 = clock64();
    for (int k = 0; k < steps; ++k) {
        double u[1] = {(k & 1) ? 3. : -3.};
        if (V == 0) {
            Cartpole<double>::step_u(w, u, p);
        } else if (V == 1) {
            double s, c;
            sincos(w.th, &s, &c);
            w.th = w.th + 0.01 * s + 1e-3 * c;
        } else {
            w.th = w.th / (1.0000001 + w.th * 1e-9);  // one IEEE division per step
        }
    }
    asm volatile("mov.f64 %0, %0;" : "+d"(w.th) :: "memory");
    long long t1 = clock64();
    out[threadIdx.x] = w.th + w.x;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
    double *out; long long *cyc;
    cudaMalloc(&out, 128 * sizeof(double));
    cudaMalloc(&cyc, sizeof(long long));
    Params<double> p{0.01, 9.81, 1., .5, .05, 2.5, 1., .1, .5, 1.8, 10., 1., 1., 1., 1., 0., 8., 1.};
    const int steps = 20000;
    const char *names[3] = {"f64 cartpole step_u", "f64 sincos chain", "f64 division chain"};
    for (int v = 0; v < 3; ++v) {
        for (int rep = 0; rep < 2; ++rep) {
            if (v == 0) chain<0><<<1, 32>>>(out, cyc, steps, p);
            if (v == 1) chain<1><<<1, 32>>>(out, cyc, steps, p);
            if (v == 2) chain<2><<<1, 32>>>(out, cyc, steps, p);
            cudaDeviceSynchronize();
        }
        long long c;
        cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
        printf("%-24s %.1f cycles/step\n", names[v], (double)c / steps);
    }
    return 0;
}
