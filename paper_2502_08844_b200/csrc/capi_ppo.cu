// capi_ppo.cu -- extern "C" entry points of the rollout-side PPO math
// (include/deskrl_b200.h): GAE and the running
// observation normaliser.
#include <cstdio>

#include "../../include/deskrl_b200.h"
#include "ppo_kernels.cuh"

#include "devguard.h"
#include "pdl.h"

extern "C" int dk_internal_fail(int code, const char *msg);  // capi.cu

namespace {

int cuda_rc(cudaError_t e, const char *what) {
    if (e == cudaSuccess) return DK_OK;
    char buf[256];
    snprintf(buf, sizeof(buf), "%s: %s", what, cudaGetErrorString(e));
    return dk_internal_fail(DK_ERR_CUDA, buf);
}

unsigned blocks(int64_t n, int bs) { return (unsigned)((n + bs - 1) / bs); }

// rows are spread over `lanes` strided accumulators per column: enough threads
// to fill the GPU, each still summing >= 16 rows
int64_t pick_lanes(int64_t rows, int dim) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int64_t lanes = ((int64_t)sms * 2048 + dim - 1) / dim;
    const int64_t cap = (rows + 15) / 16;
    if (lanes > cap) lanes = cap;
    return lanes < 1 ? 1 : lanes;
}

size_t ws_bytes(int64_t rows, int dim) {
    return sizeof(double) * ((size_t)pick_lanes(rows, dim) * dim + 2 * (size_t)dim);
}

// caller workspace (>= ws_bytes) or a stream-ordered allocation
struct Workspace {
    double *p = nullptr;
    bool owned = false;
    cudaStream_t st;
    cudaError_t init(void *ws, size_t ws_size, size_t need, cudaStream_t s) {
        st = s;
        if (ws && ws_size >= need) {
            p = (double *)ws;
            return cudaSuccess;
        }
        owned = true;
        return cudaMallocAsync((void **)&p, need, st);
    }
    ~Workspace() {
        if (owned && p) cudaFreeAsync(p, st);
    }
};

template <typename T>
int norm_update(int64_t rows, int dim, const T *batch, double count, double *mean, double *var,
                void *ws, size_t ws_size, cudaStream_t st) {
    const int64_t lanes = pick_lanes(rows, dim);
    Workspace w;
    cudaError_t e = w.init(ws, ws_size, ws_bytes(rows, dim), st);
    if (e != cudaSuccess) return cuda_rc(e, "normalizer workspace");
    double *partial = w.p, *b_mean = w.p + lanes * dim, *b_var = b_mean + dim;
    const int64_t P = lanes * dim;
    dk::colsum_kernel<T><<<blocks(P, 256), 256, 0, st>>>(rows, dim, lanes, batch, nullptr, partial);
    dk::colreduce_kernel<<<(unsigned)dim, dk::kColReduceThreads, 0, st>>>(dim, lanes, rows, partial, b_mean);
    dk::colsum_kernel<T><<<blocks(P, 256), 256, 0, st>>>(rows, dim, lanes, batch, b_mean, partial);
    dk::colreduce_kernel<<<(unsigned)dim, dk::kColReduceThreads, 0, st>>>(dim, lanes, rows, partial, b_var);
    dk::norm_merge_kernel<<<blocks(dim, 128), 128, 0, st>>>(dim, count, (double)rows, b_mean,
                                                           b_var, mean, var);
    return cuda_rc(cudaGetLastError(), "normalizer update launch");
}

}  // namespace


// tanh-Gaussian sampling + log-prob (ppo.policy_forward / tanh_gaussian_log_prob,
// ppo.py:185-217) fused: one thread per row; float32 in torch's eager operation
// order (this translation unit is built with --fmad=false, like the separate
// elementwise kernels it replaces); the NaN-mean check as a sticky flag.
__global__ void ppo_sample_kernel(int64_t n, int A, const float *mean, const float *log_std,
                                  int64_t ls_stride, const float *eps, float *pre, float *act,
                                  float *lp, int *nan_flag) {
    dk::pdl_wait();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float kHalfLog2Pi = 0.91893853320467274178f;  // 0.5 * log(2 pi) as float32
    const float kLog2 = 0.69314718055994530942f;
    float s = 0.0f;
    bool bad = false;
    for (int a = 0; a < A; ++a) {
        const float m = mean[i * A + a], l = log_std[i * ls_stride + a];
        bad |= isnan(m);
        const float sd = expf(l);
        const float u = m + sd * eps[i * A + a];
        const float z = (u - m) / sd;
        const float base = ((-0.5f * (z * z)) - l) - kHalfLog2Pi;
        const float x = -2.0f * u;
        const float sp = x > 20.0f ? x : log1pf(expf(x));
        const float corr = 2.0f * ((kLog2 - u) - sp);
        s = s + (base - corr);
        pre[i * A + a] = u;
        act[i * A + a] = tanhf(u);
    }
    lp[i] = s;
    if (bad) atomicOr(nan_flag, 1);
}

// ---------------------------------------------------------------------------
// The per-step bookkeeping of collect_rollout (ppo.py:295-378) in three
// kernels around the policy call, the env step and the value call (the torch
// version was ~25 small elementwise / copy / reduction launches per step).
// Every value is computed exactly as the separate torch ops did: normaliser
// apply in float64 (norm_apply_kernel's expression), conversions to float64,
// the reward target reward * scale + discount * term_value with two roundings.

__device__ __forceinline__ float norm_f32(float x, const dk_ppo_norm &nm, int j) {
    if (!nm.present || nm.copy) return x;
    const double sd = __dsqrt_rn(__dadd_rn(nm.var[j], nm.epsilon));
    double y = __ddiv_rn(__dsub_rn((double)x, nm.mean[j]), sd);
    y = y < -10.0 ? -10.0 : (y > 10.0 ? 10.0 : y);  // np.clip (NaN passes through)
    return (float)y;
}

// obs_p [n, dp] / obs_v [n, dv] -> raw copies (nullable), the normalised policy
// input pol [n, dp], the value input val [n, dv] and its copy val2 (nullable)
__global__ void ppo_inputs_kernel(int64_t n, int dp, int dv, const float *obs_p,
                                  const float *obs_v, dk_ppo_norm np_, dk_ppo_norm nv_,
                                  float *raw_p, float *raw_v, float *pol, float *val, float *val2) {
    dk::pdl_wait();
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t tp = n * dp;
    if (e < tp) {
        const float x = obs_p[e];
        if (raw_p) raw_p[e] = x;
        pol[e] = norm_f32(x, np_, (int)(e % dp));
    }
    if (e < n * dv) {
        const float x = obs_v[e];
        if (raw_v) raw_v[e] = x;
        const float y = norm_f32(x, nv_, (int)(e % dv));
        val[e] = y;
        if (val2) val2[e] = y;
    }
}

// after the env step: boot = trunc & ~done & terminal_mask (ppo.py:327-341),
// dones = float64(done | trunc), and the boot rows' normalised terminal
// observations compacted into val_term[0, *count) (pos[i] = the row's slot, -1
// if not a boot row).  Only those rows need a value: every other world's
// bootstrap term is masked to 0, so the value call runs on *count rows instead
// of n (a truncation is one step in episode_length).  The slot order follows
// the atomics; each world's value does not depend on it (rows are independent).
__global__ void ppo_bootstrap_kernel(int64_t n, int dv, const uint8_t *done, const uint8_t *trunc,
                                     const uint8_t *tmask, const float *term_obs,
                                     dk_ppo_norm nv_, float *val_term, int64_t *count,
                                     int32_t *pos, double *dones) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const bool b = trunc[i] && !done[i] && tmask[i];
    dones[i] = (done[i] || trunc[i]) ? 1.0 : 0.0;
    int32_t slot = -1;
    if (b) {
        slot = (int32_t)atomicAdd(reinterpret_cast<unsigned long long *>(count), 1ull);
        for (int j = 0; j < dv; ++j)
            val_term[(int64_t)slot * dv + j] = norm_f32(term_obs[i * dv + j], nv_, j);
    }
    pos[i] = slot;
}

// after the value calls (values [n] of the step's inputs, nullable when the
// caller evaluates the phase's values in one launch after it; term_values[pos[i]]
// of the boot rows' terminal observations): the reward target, the value, the
// float64 action, and per-block float64 reward sums (summed in a fixed order by
// the caller: deterministic)
constexpr int kRecordThreads = 256;
__global__ void __launch_bounds__(kRecordThreads)
ppo_record_kernel(int64_t n, int A, const float *reward, const int32_t *pos, const float *values,
                  const float *term_values, const float *action, double scale, double discount,
                  double *rew_out, double *val_out, double *act_out, double *reward_partial) {
    __shared__ double red[kRecordThreads];
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    double r = 0.0;
    if (i < n) {
        r = (double)reward[i];
        const int32_t p = pos[i];
        if (!term_values && p >= 0) {
            // boot row, its terminal value added after the phase
            // (ppo_boot_fixup_kernel: the same two roundings)
            rew_out[i] = __dmul_rn(r, scale);
        } else {
            const double tv = p >= 0 ? (double)term_values[p] : 0.0;
            rew_out[i] = __dadd_rn(__dmul_rn(r, scale), __dmul_rn(discount, tv));
        }
        if (values) val_out[i] = (double)values[i];
        for (int a = 0; a < A; ++a) act_out[i * A + a] = (double)action[i * A + a];
    }
    red[threadIdx.x] = r;
    __syncthreads();
    for (int s = kRecordThreads / 2; s > 0; s >>= 1) {
        if ((int)threadIdx.x < s) red[threadIdx.x] = red[threadIdx.x] + red[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) reward_partial[blockIdx.x] = red[0];
}

static_assert(sizeof(dk_ppo_post) == 192, "dk_ppo_post layout (paper_2502_08844_b200/_native.py PpoPostC)");

// dk_ppo_step_post: one thread per element of the next step's inputs (the
// first n threads also do world i's bootstrap and record; the first
// dk_ppo_record_blocks(n) blocks hold the worlds, so the per-block reward sums
// cover the same 256-world ranges as ppo_record_kernel's)
__global__ void __launch_bounds__(kRecordThreads)
ppo_post_kernel(dk_ppo_post a, dk_ppo_norm np_, dk_ppo_norm nv_) {
    dk::pdl_wait();
    __shared__ double red[kRecordThreads];
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t n = a.n;
    double r = 0.0;
    if (e < n) {
        const int64_t i = e;
        // bootstrap (ppo_bootstrap_kernel, slots accumulating over the phase)
        const bool b = a.trunc[i] && !a.done[i] && a.terminal_mask[i];
        a.dones[i] = (a.done[i] || a.trunc[i]) ? 1.0 : 0.0;
        int32_t slot = -1;
        if (b) {
            slot = (int32_t)atomicAdd(reinterpret_cast<unsigned long long *>(a.count), 1ull);
            for (int j = 0; j < a.dv; ++j)
                a.val_term[(int64_t)slot * a.dv + j] = norm_f32(a.terminal_obs[i * a.dv + j], nv_, j);
        }
        a.pos[i] = slot;
        // record (ppo_record_kernel with values / term_values NULL)
        r = (double)a.reward[i];
        const double rs = __dmul_rn(r, a.reward_scaling);
        a.rewards_out[i] = slot >= 0 ? rs : __dadd_rn(rs, __dmul_rn(a.discounting, 0.0));
        for (int k = 0; k < a.action_dim; ++k)
            a.actions_out[i * a.action_dim + k] = (double)a.action[i * a.action_dim + k];
    }
    if ((int64_t)blockIdx.x * blockDim.x < n) {  // block-uniform
        red[threadIdx.x] = r;
        __syncthreads();
        for (int s2 = kRecordThreads / 2; s2 > 0; s2 >>= 1) {
            if ((int)threadIdx.x < s2) red[threadIdx.x] = red[threadIdx.x] + red[threadIdx.x + s2];
            __syncthreads();
        }
        if (threadIdx.x == 0) a.reward_partial[blockIdx.x] = red[0];
    }
    if (a.next_obs_p) {  // the next step's inputs (ppo_inputs_kernel)
        if (e < n * a.dp) {
            const float x = a.next_obs_p[e];
            if (a.next_raw_p) a.next_raw_p[e] = x;
            a.next_pol[e] = norm_f32(x, np_, (int)(e % a.dp));
        }
        if (e < n * a.dv) {
            const float x = a.next_obs_v[e];
            if (a.next_raw_v) a.next_raw_v[e] = x;
            a.next_val[e] = norm_f32(x, nv_, (int)(e % a.dv));
        }
    }
}

// after a phase whose terminal values were evaluated in one call: the boot
// rows' reward targets get discount * term_values[pos] (pos [T * n])
__global__ void ppo_boot_fixup_kernel(int64_t tn, const int32_t *pos, const float *term_values,
                                      double discount, double *rew) {
    dk::pdl_wait();
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= tn) return;
    const int32_t p = pos[e];
    if (p >= 0) rew[e] = __dadd_rn(rew[e], __dmul_rn(discount, (double)term_values[p]));
}

extern "C" {

int dk_ppo_sample(int64_t n, int action_dim, const float *mean, const float *log_std,
                  int64_t log_std_stride, const float *eps, float *pre_tanh, float *action,
                  float *log_prob, int *nan_flag, void *stream) {
    dk::PtrDeviceGuard dg_(mean);
    if (n < 0 || action_dim < 1 || !mean || !log_std || !eps || !pre_tanh || !action ||
        !log_prob || !nan_flag)
        return dk_internal_fail(DK_ERR_INVALID_INPUT, "dk_ppo_sample: bad arguments");
    if (n == 0) return DK_OK;
    cudaError_t e = dk::launch_pdl(ppo_sample_kernel, dim3((unsigned)((n + 255) / 256)), dim3(256),
                                   0, (cudaStream_t)stream, n, action_dim, mean, log_std,
                                   log_std_stride, eps, pre_tanh, action, log_prob, nan_flag);
    if (e == cudaSuccess) e = cudaGetLastError();
    return e == cudaSuccess ? DK_OK : dk_internal_fail(DK_ERR_CUDA, cudaGetErrorString(e));
}

int dk_ppo_gae(int dtype, int64_t num_steps, int64_t num_worlds, const void *rewards,
               const void *values, const void *dones, const void *bootstrap, double gamma,
               double lam, void *advantages, void *returns, void *stream) {
    dk::PtrDeviceGuard dg_(rewards);  // launch on the buffers' device
    if (!rewards || !values || !dones || !bootstrap || !advantages || !returns)
        return dk_internal_fail(DK_ERR_INVALID_INPUT, "compute_gae: missing argument");
    if (num_steps < 0 || num_worlds < 0)
        return dk_internal_fail(DK_ERR_INVALID_INPUT, "compute_gae: mismatched shapes");
    if (num_steps == 0 || num_worlds == 0) return DK_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const unsigned g = blocks(num_worlds, 128);
    if (dtype == DK_F64)
        dk::gae_kernel<double><<<g, 128, 0, st>>>(
            num_steps, num_worlds, (const double *)rewards, (const double *)values,
            (const double *)dones, (const double *)bootstrap, gamma, lam, (double *)advantages,
            (double *)returns);
    else
        dk::gae_kernel<float><<<g, 128, 0, st>>>(
            num_steps, num_worlds, (const float *)rewards, (const float *)values,
            (const float *)dones, (const float *)bootstrap, gamma, lam, (float *)advantages,
            (float *)returns);
    return cuda_rc(cudaGetLastError(), "gae launch");
}

size_t dk_norm_workspace_bytes(int64_t rows, int dim) {
    return rows > 0 && dim > 0 ? ws_bytes(rows, dim) : 0;
}

int dk_norm_update(int dtype, int64_t rows, int dim, const void *batch, double count,
                   double *mean, double *var, void *workspace, size_t workspace_bytes,
                   void *stream) {
    dk::PtrDeviceGuard dg_(batch);  // launch on the buffers' device
    if (!batch || !mean || !var)
        return dk_internal_fail(DK_ERR_INVALID_INPUT, "normalizer_update: missing argument");
    if (dim <= 0 || rows < 0)
        return dk_internal_fail(DK_ERR_INVALID_INPUT, "normalizer dim mismatch");
    if (rows == 0) return DK_OK;  // (NumPy: mean of an empty batch is NaN; callers pass rows)
    cudaStream_t st = (cudaStream_t)stream;
    if (dtype == DK_F64)
        return norm_update<double>(rows, dim, (const double *)batch, count, mean, var, workspace,
                                   workspace_bytes, st);
    return norm_update<float>(rows, dim, (const float *)batch, count, mean, var, workspace,
                              workspace_bytes, st);
}

int dk_norm_colsum(int dtype, int64_t rows, int dim, const void *batch, const double *center,
                   double *sums, void *workspace, size_t workspace_bytes, void *stream) {
    dk::PtrDeviceGuard dg_(batch);  // launch on the buffers' device
    if (!batch || !sums)
        return dk_internal_fail(DK_ERR_INVALID_INPUT, "normalizer colsum: missing argument");
    if (dim <= 0 || rows < 0)
        return dk_internal_fail(DK_ERR_INVALID_INPUT, "normalizer dim mismatch");
    cudaStream_t st = (cudaStream_t)stream;
    if (rows == 0) return cuda_rc(cudaMemsetAsync(sums, 0, sizeof(double) * dim, st), "memset");
    const int64_t lanes = pick_lanes(rows, dim);
    Workspace w;
    cudaError_t e = w.init(workspace, workspace_bytes, ws_bytes(rows, dim), st);
    if (e != cudaSuccess) return cuda_rc(e, "normalizer workspace");
    double *partial = w.p;
    const int64_t P = lanes * dim;
    if (dtype == DK_F64)
        dk::colsum_kernel<double><<<blocks(P, 256), 256, 0, st>>>(rows, dim, lanes,
                                                                 (const double *)batch, center,
                                                                 partial);
    else
        dk::colsum_kernel<float><<<blocks(P, 256), 256, 0, st>>>(rows, dim, lanes,
                                                                (const float *)batch, center,
                                                                partial);
    // rows = 1: colreduce divides by it, so out = the plain column sums
    dk::colreduce_kernel<<<(unsigned)dim, dk::kColReduceThreads, 0, st>>>(dim, lanes, 1, partial, sums);
    return cuda_rc(cudaGetLastError(), "normalizer colsum launch");
}

int dk_norm_merge(int dim, double count, double batch_count, const double *batch_mean,
                  const double *batch_var, double *mean, double *var, void *stream) {
    dk::PtrDeviceGuard dg_(mean);  // launch on the buffers' device
    if (!batch_mean || !batch_var || !mean || !var)
        return dk_internal_fail(DK_ERR_INVALID_INPUT, "normalizer merge: missing argument");
    if (dim <= 0) return dk_internal_fail(DK_ERR_INVALID_INPUT, "normalizer dim mismatch");
    dk::norm_merge_kernel<<<blocks(dim, 128), 128, 0, (cudaStream_t)stream>>>(
        dim, count, batch_count, batch_mean, batch_var, mean, var);
    return cuda_rc(cudaGetLastError(), "normalizer merge launch");
}

int dk_norm_apply(int dtype, int64_t rows, int dim, const void *batch, double count,
                  const double *mean, const double *var, double epsilon, int invert, void *out,
                  void *stream) {
    dk::PtrDeviceGuard dg_(batch);  // launch on the buffers' device
    if (!batch || !mean || !var || !out)
        return dk_internal_fail(DK_ERR_INVALID_INPUT, "normalizer_apply: missing argument");
    if (dim <= 0 || rows < 0)
        return dk_internal_fail(DK_ERR_INVALID_INPUT, "normalizer dim mismatch");
    const int64_t total = rows * dim;
    if (total == 0) return DK_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const int copy = count == 0.0 ? 1 : 0;
    if (dtype == DK_F64)
        dk::norm_apply_kernel<double><<<blocks(total, 256), 256, 0, st>>>(
            total, dim, (const double *)batch, mean, var, epsilon, copy, invert, (double *)out);
    else
        dk::norm_apply_kernel<float><<<blocks(total, 256), 256, 0, st>>>(
            total, dim, (const float *)batch, mean, var, epsilon, copy, invert, (float *)out);
    return cuda_rc(cudaGetLastError(), "normalizer apply launch");
}


int dk_ppo_step_inputs(int64_t n, int dp, int dv, const float *obs_p, const float *obs_v,
                       const dk_ppo_norm *norm_p, const dk_ppo_norm *norm_v, float *raw_p,
                       float *raw_v, float *pol, float *val, float *val2, void *stream) {
    dk::PtrDeviceGuard dg_(obs_p);
    if (n < 0 || dp < 1 || dv < 1 || !obs_p || !obs_v || !pol || !val)
        return dk_internal_fail(DK_ERR_INVALID_INPUT, "dk_ppo_step_inputs: bad arguments");
    if (n == 0) return DK_OK;
    dk_ppo_norm off = {};
    const int64_t tot = n * (dp > dv ? dp : dv);
    const cudaError_t e = dk::launch_pdl(
        ppo_inputs_kernel, dim3(blocks(tot, 256)), dim3(256), 0, (cudaStream_t)stream, n, dp, dv,
        obs_p, obs_v, norm_p ? *norm_p : off, norm_v ? *norm_v : off, raw_p, raw_v, pol, val, val2);
    return cuda_rc(e != cudaSuccess ? e : cudaGetLastError(), "dk_ppo_step_inputs launch");
}

namespace {
int step_bootstrap(int64_t n, int dv, const uint8_t *done, const uint8_t *trunc,
                   const uint8_t *terminal_mask, const float *terminal_obs,
                   const dk_ppo_norm *norm_v, float *val_term, int64_t *count, int32_t *pos,
                   double *dones, bool accumulate, void *stream) {
    dk::PtrDeviceGuard dg_(done);
    if (n < 0 || dv < 1 || !done || !trunc || !terminal_mask || !terminal_obs || !val_term ||
        !count || !pos || !dones)
        return dk_internal_fail(DK_ERR_INVALID_INPUT, "dk_ppo_step_bootstrap: bad arguments");
    cudaStream_t st = (cudaStream_t)stream;
    if (!accumulate) {
        cudaError_t e = cudaMemsetAsync(count, 0, sizeof(int64_t), st);
        if (e != cudaSuccess) return cuda_rc(e, "dk_ppo_step_bootstrap count");
    }
    if (n == 0) return DK_OK;
    dk_ppo_norm off = {};
    ppo_bootstrap_kernel<<<blocks(n, 256), 256, 0, st>>>(n, dv, done, trunc, terminal_mask,
                                                         terminal_obs, norm_v ? *norm_v : off,
                                                         val_term, count, pos, dones);
    return cuda_rc(cudaGetLastError(), "dk_ppo_step_bootstrap launch");
}
}  // namespace

int dk_ppo_step_bootstrap(int64_t n, int dv, const uint8_t *done, const uint8_t *trunc,
                          const uint8_t *terminal_mask, const float *terminal_obs,
                          const dk_ppo_norm *norm_v, float *val_term, int64_t *count,
                          int32_t *pos, double *dones, void *stream) {
    return step_bootstrap(n, dv, done, trunc, terminal_mask, terminal_obs, norm_v, val_term,
                          count, pos, dones, false, stream);
}

int dk_ppo_step_bootstrap_acc(int64_t n, int dv, const uint8_t *done, const uint8_t *trunc,
                              const uint8_t *terminal_mask, const float *terminal_obs,
                              const dk_ppo_norm *norm_v, float *val_term, int64_t *count,
                              int32_t *pos, double *dones, void *stream) {
    return step_bootstrap(n, dv, done, trunc, terminal_mask, terminal_obs, norm_v, val_term,
                          count, pos, dones, true, stream);
}

int dk_ppo_step_post(const dk_ppo_post *a, const dk_ppo_norm *norm_p,
                     const dk_ppo_norm *norm_v, void *stream) {
    if (!a || !a->done) return dk_internal_fail(DK_ERR_INVALID_INPUT, "dk_ppo_step_post: null");
    dk::PtrDeviceGuard dg_(a->done);
    const bool next = a->next_obs_p != nullptr;
    if (a->n < 0 || a->dv < 1 || a->action_dim < 1 || !a->trunc || !a->terminal_mask ||
        !a->terminal_obs || !a->val_term || !a->count || !a->pos || !a->dones || !a->reward ||
        !a->action || !a->rewards_out || !a->actions_out || !a->reward_partial ||
        (next && (a->dp < 1 || !a->next_obs_v || !a->next_pol || !a->next_val)))
        return dk_internal_fail(DK_ERR_INVALID_INPUT, "dk_ppo_step_post: bad arguments");
    if (a->n == 0) return DK_OK;
    dk_ppo_norm off = {};
    int64_t tot = a->n;
    if (next) {
        const int64_t m = a->n * (a->dp > a->dv ? a->dp : a->dv);
        tot = m > tot ? m : tot;
    }
    const cudaError_t e = dk::launch_pdl(ppo_post_kernel, dim3(blocks(tot, kRecordThreads)),
                                         dim3(kRecordThreads), 0, (cudaStream_t)stream, *a,
                                         norm_p ? *norm_p : off, norm_v ? *norm_v : off);
    return cuda_rc(e != cudaSuccess ? e : cudaGetLastError(), "dk_ppo_step_post launch");
}

int dk_ppo_boot_fixup(int64_t tn, const int32_t *pos, const float *term_values,
                      double discounting, double *rewards, void *stream) {
    dk::PtrDeviceGuard dg_(pos);
    if (tn < 0 || !pos || !term_values || !rewards)
        return dk_internal_fail(DK_ERR_INVALID_INPUT, "dk_ppo_boot_fixup: bad arguments");
    if (tn == 0) return DK_OK;
    const cudaError_t e = dk::launch_pdl(ppo_boot_fixup_kernel, dim3(blocks(tn, 256)), dim3(256),
                                         0, (cudaStream_t)stream, tn, pos, term_values,
                                         discounting, rewards);
    return cuda_rc(e != cudaSuccess ? e : cudaGetLastError(), "dk_ppo_boot_fixup launch");
}

int64_t dk_ppo_record_blocks(int64_t n) { return (n + kRecordThreads - 1) / kRecordThreads; }

int dk_ppo_step_record(int64_t n, int action_dim, const float *reward, const int32_t *pos,
                       const float *values, const float *term_values, const float *action,
                       double reward_scaling, double discounting, double *rewards_out,
                       double *values_out, double *actions_out, double *reward_partial,
                       void *stream) {
    dk::PtrDeviceGuard dg_(reward);
    if (n < 0 || action_dim < 1 || !reward || !pos || !action ||
        !rewards_out || (values && !values_out) || !actions_out || !reward_partial)
        return dk_internal_fail(DK_ERR_INVALID_INPUT, "dk_ppo_step_record: bad arguments");
    if (n == 0) return DK_OK;
    ppo_record_kernel<<<blocks(n, kRecordThreads), kRecordThreads, 0, (cudaStream_t)stream>>>(
        n, action_dim, reward, pos, values, term_values, action, reward_scaling, discounting,
        rewards_out, values_out, actions_out, reward_partial);
    return cuda_rc(cudaGetLastError(), "dk_ppo_step_record launch");
}
}  // extern "C"
