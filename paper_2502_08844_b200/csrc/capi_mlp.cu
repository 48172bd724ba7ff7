// capi_mlp.cu -- extern "C" entry points of the tensor-core MLP forward
// (mlp_tc.cuh; include/deskrl_b200.h "PPO networks on the tensor cores").
#include <cstdio>

#include "../../include/deskrl_b200.h"
#include "devguard.h"
#include "pdl.h"
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

namespace {
// validated kernel arguments of one network call (DK_OK or an error code)
int mlp_args(const dk_mlp *net, int64_t rows, const int64_t *rows_dev, const float *x,
             int64_t x_stride, float *y, int64_t y_stride, int desc_swap, dk::mlp::MlpArgs &a,
             size_t &smem) {
    if (!net || !x || !y) return dk_internal_fail(DK_ERR_INVALID_INPUT, "dk_mlp_forward: null");
    const int H = net->hidden;
    if (!(H == 128 || H == 256) || net->d_in < 1 || net->d_in > dk::mlp::MAXDIN ||
        net->n_out < 1 || net->n_out > dk::mlp::MAXOUT || net->n_tc < 1)
        return dk_internal_fail(DK_ERR_INVALID_INPUT,
                                "dk_mlp_forward: hidden must be 128 or 256, d_in <= 128, "
                                "1 <= n_out <= 16, at least one hidden x hidden layer");
    if (dk::mlp::tc_layer0(net->d_in) && (!net->w0_hi || !net->w0_lo))
        return dk_internal_fail(DK_ERR_INVALID_INPUT,
                                "dk_mlp_forward: d_in > 16 needs the packed layer-0 weights");
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
    a.w0hi = (const __nv_bfloat16 *)net->w0_hi;
    a.w0lo = (const __nv_bfloat16 *)net->w0_lo;
    a.y = y;
    a.y_stride = y_stride;
    a.desc_swap = desc_swap;
    a.rows_dev = rows_dev;
    a.ns = dk::mlp::mlp_stages(H, net->d_in, net->n_out);
    if (a.ns < 2)
        return dk_internal_fail(DK_ERR_INVALID_INPUT, "dk_mlp_forward: network too large");
    smem = dk::mlp::mlp_smem_bytes(H, net->d_in, net->n_out, a.ns);
    return DK_OK;
}

int64_t tiles(int64_t rows) { return rows > 0 ? (rows + dk::mlp::M - 1) / dk::mlp::M : 0; }

int mlp_launch(const dk::mlp::MlpArgs &a0, int64_t t0, const dk::mlp::MlpArgs &a1, int64_t t1,
               size_t smem, void *stream) {
    if (t0 + t1 == 0) return DK_OK;
    const bool wide = a0.n_out > 4 || (t1 > 0 && a1.n_out > 4);
    const void *fn = wide ? (const void *)dk::mlp::mlp_tc_kernel<dk::mlp::MAXOUT>
                          : (const void *)dk::mlp::mlp_tc_kernel<4>;
    static dk::SmemOptIn optin[2];
    cudaError_t e = optin[wide ? 1 : 0].ensure(fn, smem);
    if (e != cudaSuccess) return cuda_rc(e, "dk_mlp_forward attribute");
    // programmatic dependent launch: the grid is placed while the previous kernel
    // of the PPO step drains (the kernel waits before touching its data)
    e = dk::launch_pdl(wide ? dk::mlp::mlp_tc_kernel<dk::mlp::MAXOUT> : dk::mlp::mlp_tc_kernel<4>,
                       dim3((unsigned)(t0 + t1)), dim3(dk::mlp::THREADS), smem,
                       (cudaStream_t)stream, a0, a1, t0);
    return cuda_rc(e != cudaSuccess ? e : cudaGetLastError(), "mlp_tc_kernel");
}

int mlp_forward(const dk_mlp *net, int64_t rows, const int64_t *rows_dev, const float *x,
                int64_t x_stride, float *y, int64_t y_stride, int desc_swap, void *stream) {
    if (!x) return dk_internal_fail(DK_ERR_INVALID_INPUT, "dk_mlp_forward: null");
    dk::PtrDeviceGuard dg_(x);
    dk::mlp::MlpArgs a;
    size_t smem = 0;
    const int rc = mlp_args(net, rows, rows_dev, x, x_stride, y, y_stride, desc_swap, a, smem);
    if (rc != DK_OK) return rc;
    if (rows <= 0) return DK_OK;
    return mlp_launch(a, tiles(rows), a, 0, smem, stream);
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

int dk_mlp_forward(const dk_mlp *net, int64_t rows, const float *x, int64_t x_stride, float *y,
                   int64_t y_stride, void *stream) {
    return dk_mlp_forward_dbg(net, rows, x, x_stride, y, y_stride, 0, stream);
}

int dk_mlp_forward_pair(const dk_mlp *net0, int64_t rows0, const float *x0, int64_t x0_stride,
                        float *y0, int64_t y0_stride, const dk_mlp *net1, int64_t rows1,
                        const float *x1, int64_t x1_stride, float *y1, int64_t y1_stride,
                        void *stream) {
    if (!x0 || !x1) return dk_internal_fail(DK_ERR_INVALID_INPUT, "dk_mlp_forward_pair: null");
    dk::PtrDeviceGuard dg_(x0);
    dk::mlp::MlpArgs a0, a1;
    size_t s0 = 0, s1 = 0;
    int rc = mlp_args(net0, rows0, nullptr, x0, x0_stride, y0, y0_stride, 0, a0, s0);
    if (rc != DK_OK) return rc;
    rc = mlp_args(net1, rows1, nullptr, x1, x1_stride, y1, y1_stride, 0, a1, s1);
    if (rc != DK_OK) return rc;
    return mlp_launch(a0, tiles(rows0), a1, tiles(rows1), s0 > s1 ? s0 : s1, stream);
}

}  // extern "C"
