// capi_mlp.cu -- extern "C" entry points of the tensor-core MLP forward
// (mlp_tc.cuh; include/deskrl_b200.h "PPO networks on the tensor cores").
#include <cstdio>

#include "../../include/deskrl_b200.h"
#include "devguard.h"
#include "mlp_tc.cuh"

extern "C" int dk_internal_fail(int code, const char *msg);  // capi.cu

namespace {
int cuda_rc(cudaError_t e, const char *what) {
    if (e == cudaSuccess) return DK_OK;
    char buf[256];
    snprintf(buf, sizeof(buf), "%s: %s", what, cudaGetErrorString(e));
    return dk_internal_fail(DK_ERR_CUDA, buf);
}
}  // namespace

extern "C" {

int dk_mlp_pack(const float *w, int n, int k, void *w_hi, void *w_lo, void *stream) {
    dk::PtrDeviceGuard dg_(w);
    if (!w || !w_hi || !w_lo) return dk_internal_fail(DK_ERR_INVALID_INPUT, "dk_mlp_pack: null");
    if (n <= 0 || k <= 0 || n % 8 || k % dk::mlp::KC)
        return dk_internal_fail(DK_ERR_INVALID_INPUT,
                                "dk_mlp_pack: n must be a multiple of 8 and k of 32");
    const int total = n * k;
    dk::mlp::pack_weights_kernel<<<(total + 255) / 256, 256, 0, (cudaStream_t)stream>>>(
        w, n, k, (__nv_bfloat16 *)w_hi, (__nv_bfloat16 *)w_lo);
    return cuda_rc(cudaGetLastError(), "dk_mlp_pack");
}

namespace {
int mlp_forward(const dk_mlp *net, int64_t rows, const int64_t *rows_dev, const float *x,
                int64_t x_stride, float *y, int64_t y_stride, int desc_swap, void *stream);
}

int dk_mlp_forward_dbg(const dk_mlp *net, int64_t rows, const float *x, int64_t x_stride,
                       float *y, int64_t y_stride, int desc_swap, void *stream) {
    return mlp_forward(net, rows, nullptr, x, x_stride, y, y_stride, desc_swap, stream);
}

int dk_mlp_forward_count(const dk_mlp *net, int64_t max_rows, const int64_t *rows_dev,
                         const float *x, int64_t x_stride, float *y, int64_t y_stride,
                         void *stream) {
    if (!rows_dev) return dk_internal_fail(DK_ERR_INVALID_INPUT, "dk_mlp_forward_count: null");
    return mlp_forward(net, max_rows, rows_dev, x, x_stride, y, y_stride, 0, stream);
}

}  // extern "C"

namespace {
int mlp_forward(const dk_mlp *net, int64_t rows, const int64_t *rows_dev, const float *x,
                int64_t x_stride, float *y, int64_t y_stride, int desc_swap, void *stream) {
    if (!net || !x || !y) return dk_internal_fail(DK_ERR_INVALID_INPUT, "dk_mlp_forward: null");
    dk::PtrDeviceGuard dg_(x);
    const int H = net->hidden;
    if (!(H == 128 || H == 256) || net->d_in < 1 || net->d_in > 16 || net->n_out < 1 ||
        net->n_out > 4 || net->n_tc < 1)
        return dk_internal_fail(DK_ERR_INVALID_INPUT,
                                "dk_mlp_forward: hidden must be 128 or 256, d_in <= 16, "
                                "1 <= n_out <= 4, at least one hidden x hidden layer");
    if (rows <= 0) return DK_OK;
    dk::mlp::MlpArgs a;
    a.x = x;
    a.rows = rows;
    a.x_stride = x_stride;
    a.d_in = net->d_in;
    a.H = H;
    a.n_tc = net->n_tc;
    a.n_out = net->n_out;
    a.w0 = net->w0;
    a.b0 = net->b0;
    a.whi = (const __nv_bfloat16 *)net->w_hi;
    a.wlo = (const __nv_bfloat16 *)net->w_lo;
    a.bh = net->b_hidden;
    a.wout = net->w_out;
    a.bout = net->b_out;
    a.y = y;
    a.y_stride = y_stride;
    a.desc_swap = desc_swap;
    a.rows_dev = rows_dev;
    const size_t smem = dk::mlp::mlp_smem_bytes(H, net->d_in, net->n_tc, net->n_out);
    if (smem > 227 * 1024)
        return dk_internal_fail(DK_ERR_INVALID_INPUT, "dk_mlp_forward: network too large");
    static size_t attr = 0;
    if (smem > attr) {
        cudaError_t e = cudaFuncSetAttribute(dk::mlp::mlp_tc_kernel,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return cuda_rc(e, "dk_mlp_forward attribute");
        attr = smem;
    }
    const unsigned grid = (unsigned)((rows + dk::mlp::M - 1) / dk::mlp::M);
    dk::mlp::mlp_tc_kernel<<<grid, dk::mlp::THREADS, smem, (cudaStream_t)stream>>>(a);
    return cuda_rc(cudaGetLastError(), "mlp_tc_kernel");
}
}  // namespace

extern "C" {

int dk_mlp_forward(const dk_mlp *net, int64_t rows, const float *x, int64_t x_stride, float *y,
                   int64_t y_stride, void *stream) {
    return dk_mlp_forward_dbg(net, rows, x, x_stride, y, y_stride, 0, stream);
}

}  // extern "C"
