// Microbenchmark: latency of the cartpole f32 step chain in one warp (no memory
// traffic, no barriers), timed with clock64.  Variants isolate sincos and the
// 2x2 solve.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I.. chainbench.cu
#include <cstdio>
#include "../../paper_2502_08844_b200/csrc/tasks.cuh"

using namespace dk;

// V = 4..7: the producer's fast-group body (8 steps unrolled) with its
// shared-memory traffic: 4 = u from smem, 5 = + 6 STS per step (world_to_slot),
// 6 = registers only but unrolled by 8, 7 = 5 with u loaded at the group start.
template <int V>
__global__ void group_body(float *out, long long *cyc, int steps, Params<float> p) {
    __shared__ float ring[8][6][32];
    __shared__ float act[8][32];
    const int lane = threadIdx.x;
    for (int s = 0; s < 8; ++s) act[s][lane] = (s & 1) ? 3.f : -3.f;
    __syncwarp();
    Cartpole<float>::W w;
    w.x = 0.1f * lane / 32.f; w.th = 0.05f; w.xd = 0.f; w.thd = 0.01f;
    Cartpole<float>::refresh(w);
    long long t0 = clock64();
    for (int g = 0; g < steps / 8; ++g) {
        float ua[8];
        if (V == 7) {
#pragma unroll
            for (int s = 0; s < 8; ++s) ua[s] = act[s][lane];
        }
#pragma unroll
        for (int s = 0; s < 8; ++s) {
            float u[1];
            if (V == 6) u[0] = (s & 1) ? 3.f : -3.f;
            else if (V == 7) u[0] = ua[s];
            else u[0] = act[s][lane];
            Cartpole<float>::step_u(w, u, p);
            if (V == 5 || V == 7) {
                const float *f = reinterpret_cast<const float *>(&w);
#pragma unroll
                for (int j = 0; j < 6; ++j) ring[s][j][lane] = f[j];
            }
        }
        __syncwarp();
    }
    asm volatile("mov.f32 %0, %0;" : "+f"(w.th) :: "memory");
    long long t1 = clock64();
    out[lane] = w.th + w.thd + w.c + ring[lane & 7][lane % 6][lane];
    if (lane == 0) cyc[0] = t1 - t0;
}

// two independent worlds per lane (the TL = 2 producer): does the second chain
// fill the first one's latency?
__global__ void chain2(float *out, long long *cyc, int steps, Params<float> p) {
    Cartpole<float>::W w[2];
    for (int t = 0; t < 2; ++t) {
        w[t].x = 0.1f * threadIdx.x / 32.f + t; w[t].th = 0.05f + 0.1f * t; w[t].xd = 0.f;
        w[t].thd = 0.01f;
        Cartpole<float>::refresh(w[t]);
    }
    float acc = 0.f;
    long long t0 = clock64();
    for (int k = 0; k < steps; ++k) {
        float u[1] = {(k & 1) ? 3.f : -3.f};
#pragma unroll
        for (int t = 0; t < 2; ++t) Cartpole<float>::step_u(w[t], u, p);
        acc += w[0].x + w[1].x;
    }
    asm volatile("mov.f32 %0, %0;" : "+f"(acc) :: "memory");
    long long t1 = clock64();
    out[threadIdx.x] = acc + w[0].th + w[1].th;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

template <int V>
__global__ void chain(float *out, long long *cyc, int steps, Params<float> p) {
    Cartpole<float>::W w;
    w.x = 0.1f * threadIdx.x / 32.f; w.th = 0.05f; w.xd = 0.f; w.thd = 0.01f;
    Cartpole<float>::refresh(w);
    float u[1] = {0.3f};
    float acc = 0.f;
    long long t0 = clock64();
    for (int k = 0; k < steps; ++k) {
        u[0] = (k & 1) ? 3.f : -3.f;
        if (V == 0) {
            Cartpole<float>::step_u(w, u, p);            // full step
        } else if (V == 1) {
            float s, c;
            sincosf_fast(w.th, &s, &c);                  // sincos chain only
            w.th = w.th + 0.01f * s + 1e-3f * c;
        } else if (V == 2) {
            // 2x2 solve + Euler without trig (s, c fixed)
            const float m12 = p.pole_mass * p.pole_length * w.c;
            const float det = (p.cart_mass + p.pole_mass) * (p.pole_mass * p.pole_length * p.pole_length) - m12 * m12;
            const float thdd = RealOps<float>::div_(u[0] - m12 * w.thd, det);
            w.thd = w.thd + p.dt * thdd;
            w.c = w.c + p.dt * w.thd * 1e-3f;
        } else {
            w.th = fmaf(w.th, 1.0000001f, 1e-7f);       // 1 dependent FFMA per step
        }
        acc += w.x;
    }
    asm volatile("mov.f32 %0, %0;" : "+f"(w.th) :: "memory");  // loop result before t1
    long long t1 = clock64();
    out[threadIdx.x] = acc + w.th + w.thd + w.c;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
    float *out; long long *cyc;
    cudaMalloc(&out, 128 * sizeof(float));
    cudaMalloc(&cyc, sizeof(long long));
    Params<float> p{0.01f, 9.81f, 1.f, .5f, .05f, 2.5f, 1.f, .1f, .5f, 1.8f, 10.f, 1.f, 1.f, 1.f, 1.f, 0.f, 8.f, 1.f};
    const int steps = 100000;
    const char *names[8] = {"full cartpole step_u", "sincosf_fast chain", "2x2 solve + euler", "1 FFMA/step",
                            "group: u from smem", "group: u smem + 6 STS", "group: regs, unroll 8",
                            "group: u preload + 6 STS"};
    for (int v = 0; v < 8; ++v) {
        for (int rep = 0; rep < 2; ++rep) {
            if (v == 0) chain<0><<<1, 32>>>(out, cyc, steps, p);
            if (v == 1) chain<1><<<1, 32>>>(out, cyc, steps, p);
            if (v == 2) chain<2><<<1, 32>>>(out, cyc, steps, p);
            if (v == 3) chain<3><<<1, 32>>>(out, cyc, steps, p);
            if (v == 4) group_body<4><<<1, 32>>>(out, cyc, steps, p);
            if (v == 5) group_body<5><<<1, 32>>>(out, cyc, steps, p);
            if (v == 6) group_body<6><<<1, 32>>>(out, cyc, steps, p);
            if (v == 7) group_body<7><<<1, 32>>>(out, cyc, steps, p);
            cudaDeviceSynchronize();
        }
        long long c;
        cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
        printf("%-24s %.1f cycles/step\n", names[v], (double)c / steps);
    }
    for (int rep = 0; rep < 2; ++rep) {
        chain2<<<1, 32>>>(out, cyc, steps, p);
        cudaDeviceSynchronize();
    }
    long long c;
    cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
    printf("%-24s %.1f cycles/step (both worlds)\n", "two chains per lane", (double)c / steps);
    return 0;
}
