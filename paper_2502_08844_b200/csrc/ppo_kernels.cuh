// ppo_kernels.cuh -- the rollout-side PPO math that follows the env step
// (SURVEY.md §8f rank 1): generalized advantage estimation and the running
// observation normaliser, on device.
//
//   compute_gae        ppo.py:80-102
//   normalizer_update  mathcore.py:234-251
//   normalizer_apply   mathcore.py:254-265 / normalizer_invert 268-272
//
// float64 arithmetic is written with explicit _rn intrinsics, one rounding per
// Python / NumPy operation in the reference's order, so the f64 results match
// the reference bit for bit where the reference's own order is sequential
// (GAE, apply / invert) and to a few ulps where NumPy sums columns
// sequentially and the device sums them as a fixed-order tree (update).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace dk {

__device__ __forceinline__ double to_f64(float v) { return (double)v; }
__device__ __forceinline__ double to_f64(double v) { return v; }

// delta_t = r_t + gamma (1 - done_t) V_{t+1} - V_t;  A_t = delta_t + gamma lam (1 - done_t) A_{t+1}
// One thread per world walks t = T-1 .. 0 (coalesced [T, N] rows).  Inputs are
// read as float64 (the reference converts with np.asarray(dtype=float64)).
template <typename T>
__global__ void gae_kernel(int64_t Tn, int64_t n, const T *__restrict__ rewards,
                           const T *__restrict__ values, const T *__restrict__ dones,
                           const T *__restrict__ bootstrap, double gamma, double lam,
                           T *__restrict__ adv, T *__restrict__ ret) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double gl = __dmul_rn(gamma, lam);  // gamma * lam * nonterm * last: left to right
    double next_v = to_f64(bootstrap[i]);
    double last = 0.0;
    auto step = [&](int64_t e, double r, double v, double d) {
        const double nonterm = __dsub_rn(1.0, d);
        const double delta = __dsub_rn(__dadd_rn(r, __dmul_rn(__dmul_rn(gamma, nonterm), next_v)), v);
        last = __dadd_rn(delta, __dmul_rn(__dmul_rn(gl, nonterm), last));
        adv[e] = (T)last;
        ret[e] = (T)__dadd_rn(last, v);  // advantages + values
        next_v = v;
    };
    // CH time steps of loads in flight per thread before the serial recurrence
    // consumes them (one world per thread leaves few warps per SM: without
    // this, every step waited a full DRAM round trip)
    // ... double-buffered (two register buffers with static indices, so nothing
    // spills to local memory): the next chunk's loads are issued before this
    // chunk's recurrence runs
    constexpr int CH = 16;
    int64_t t = Tn - 1;
    T ra[CH], va[CH], da[CH], rb[CH], vb[CH], db[CH];
    auto load = [&](T *r, T *v, T *d, int64_t t0) {
#pragma unroll
        for (int k = 0; k < CH; ++k) {
            const int64_t e = (t0 - k) * n + i;
            r[k] = rewards[e]; v[k] = values[e]; d[k] = dones[e];
        }
    };
    auto run = [&](const T *r, const T *v, const T *d, int64_t t0) {
#pragma unroll
        for (int k = 0; k < CH; ++k)
            step((t0 - k) * n + i, to_f64(r[k]), to_f64(v[k]), to_f64(d[k]));
    };
    if (t + 1 >= CH) load(ra, va, da, t);
    while (t + 1 >= CH) {
        if (t + 1 >= 2 * CH) load(rb, vb, db, t - CH);
        run(ra, va, da, t);
        t -= CH;
        if (t + 1 < CH) break;
        if (t + 1 >= 2 * CH) load(ra, va, da, t - CH);
        run(rb, vb, db, t);
        t -= CH;
    }
    for (; t >= 0; --t) {
        const int64_t e = t * n + i;
        step(e, to_f64(rewards[e]), to_f64(values[e]), to_f64(dones[e]));
    }
}

// Column sums of a row-major [rows, dim] batch in float64, deterministic:
// thread k = l * dim + j (l < lanes) adds rows l, l + lanes, ... of column j
// (consecutive threads read consecutive addresses) into partial[k]; with
// `center`, it sums (x - center[j])^2 instead (NumPy's var: mean of squared
// deviations from the batch mean).
template <typename T>
__global__ void colsum_kernel(int64_t rows, int dim, int64_t lanes, const T *__restrict__ batch,
                              const double *__restrict__ center, double *__restrict__ partial) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= lanes * dim) return;
    const int64_t l = k / dim;
    const int j = (int)(k - l * dim);
    const double c = center ? center[j] : 0.0;
    double s = 0.0;
#pragma unroll 8
    for (int64_t r = l; r < rows; r += lanes) {  // (loads run ahead; the sum stays in order)
        const double x = to_f64(batch[r * dim + j]);
        if (center) {
            const double d = __dsub_rn(x, c);
            s = __dadd_rn(s, __dmul_rn(d, d));
        } else {
            s = __dadd_rn(s, x);
        }
    }
    partial[k] = s;
}

// One 256-thread block per column: each thread sums the partials l = t, t + 256,
// ... in order (eight loads in flight), then a fixed shared-memory / shuffle tree
// (deterministic).  out[j] = sum / rows (a mean, NumPy's true_divide by the
// count).  (One warp per column, one dependent L2 round trip per partial, took
// ~40 us per call at 30 x 8192 rows.)
constexpr int kColReduceThreads = 256;
static __global__ void __launch_bounds__(kColReduceThreads)
colreduce_kernel(int dim, int64_t lanes, int64_t rows, const double *__restrict__ partial,
                 double *__restrict__ out) {
    __shared__ double red[kColReduceThreads / 32];
    const int j = blockIdx.x;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    double s = 0.0;
    int64_t l = t;
    constexpr int64_t S = kColReduceThreads;
    for (; l + 7 * S < lanes; l += 8 * S) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = partial[(l + u * S) * dim + j];
#pragma unroll
        for (int u = 0; u < 8; ++u) s = __dadd_rn(s, v[u]);
    }
    for (; l < lanes; l += S) s = __dadd_rn(s, partial[l * dim + j]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s = __dadd_rn(s, __shfl_down_sync(0xffffffffu, s, o));
    if (lane == 0) red[warp] = s;
    __syncthreads();
    if (t == 0) {
        double tot = red[0];
        for (int w = 1; w < kColReduceThreads / 32; ++w) tot = __dadd_rn(tot, red[w]);
        out[j] = __ddiv_rn(tot, (double)rows);
    }
}

// mathcore.py:245-251, per column, in the reference's operation order.
static __global__ void norm_merge_kernel(int dim, double count, double b_count,
                                         const double *__restrict__ b_mean,
                                         const double *__restrict__ b_var, double *mean,
                                         double *var) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= dim) return;
    const double total = __dadd_rn(count, b_count);
    const double delta = __dsub_rn(b_mean[j], mean[j]);
    const double m = __dadd_rn(mean[j], __dmul_rn(delta, __ddiv_rn(b_count, total)));
    const double m_a = __dmul_rn(var[j], count);
    const double m_b = __dmul_rn(b_var[j], b_count);
    // delta**2 * n.count * b_count / total: ((delta^2 * count) * b_count) / total
    const double cross =
        __ddiv_rn(__dmul_rn(__dmul_rn(__dmul_rn(delta, delta), count), b_count), total);
    const double v = __ddiv_rn(__dadd_rn(__dadd_rn(m_a, m_b), cross), total);
    mean[j] = m;
    var[j] = v > 0.0 ? v : (v == v ? 0.0 : v);  // np.maximum(var, 0.0) (NaN propagates)
}

// normalizer_apply: clip((x - mean) / sqrt(var + eps), -10, 10); invert:
// x * sqrt(var + eps) + mean.  count == 0 copies (the reference's early return).
template <typename T>
__global__ void norm_apply_kernel(int64_t total, int dim, const T *__restrict__ batch,
                                  const double *__restrict__ mean, const double *__restrict__ var,
                                  double eps, int copy, int invert, T *__restrict__ out) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= total) return;
    const int j = (int)(k % dim);
    const double x = to_f64(batch[k]);
    if (copy) {
        out[k] = (T)x;
        return;
    }
    const double sd = __dsqrt_rn(__dadd_rn(var[j], eps));
    double y;
    if (invert) {
        y = __dadd_rn(__dmul_rn(x, sd), mean[j]);
    } else {
        y = __ddiv_rn(__dsub_rn(x, mean[j]), sd);
        y = y < -10.0 ? -10.0 : (y > 10.0 ? 10.0 : y);  // np.clip (NaN passes through)
    }
    out[k] = (T)y;
}

}  // namespace dk
