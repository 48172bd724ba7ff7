// capi_ppo.cu -- extern "C" entry points of the rollout-side PPO math
// (include/deskrl_b200.h): GAE and the running
// observation normaliser.
#include <cstdio>

#include "../../include/deskrl_b200.h"
#include "ppo_kernels.cuh"

#include "devguard.h"

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
    dk::colreduce_kernel<<<blocks(dim, 8), 256, 0, st>>>(dim, lanes, rows, partial, b_mean);
    dk::colsum_kernel<T><<<blocks(P, 256), 256, 0, st>>>(rows, dim, lanes, batch, b_mean, partial);
    dk::colreduce_kernel<<<blocks(dim, 8), 256, 0, st>>>(dim, lanes, rows, partial, b_var);
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

extern "C" {

int dk_ppo_sample(int64_t n, int action_dim, const float *mean, const float *log_std,
                  int64_t log_std_stride, const float *eps, float *pre_tanh, float *action,
                  float *log_prob, int *nan_flag, void *stream) {
    dk::PtrDeviceGuard dg_(mean);
    if (n < 0 || action_dim < 1 || !mean || !log_std || !eps || !pre_tanh || !action ||
        !log_prob || !nan_flag)
        return dk_internal_fail(DK_ERR_INVALID_INPUT, "dk_ppo_sample: bad arguments");
    if (n == 0) return DK_OK;
    ppo_sample_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        n, action_dim, mean, log_std, log_std_stride, eps, pre_tanh, action, log_prob, nan_flag);
    cudaError_t e = cudaGetLastError();
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
    dk::colreduce_kernel<<<blocks(dim, 8), 256, 0, st>>>(dim, lanes, 1, partial, sums);
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

}  // extern "C"
