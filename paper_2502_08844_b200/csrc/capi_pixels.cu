// capi_pixels.cu -- extern "C" entry points of the cartpole pixel observation
// path (include/deskrl_b200.h).
#include <cstdio>

#include "../../include/deskrl_b200.h"
#include "pixels.cuh"

#include "devguard.h"

extern "C" int dk_internal_fail(int code, const char *msg);  // capi.cu

namespace {

int cuda_rc(cudaError_t e, const char *what) {
    if (e == cudaSuccess) return DK_OK;
    char buf[256];
    snprintf(buf, sizeof(buf), "%s: %s", what, cudaGetErrorString(e));
    return dk_internal_fail(DK_ERR_CUDA, buf);
}

int check_view(int w, int h) {
    if (w <= 0 || h <= 0)
        return dk_internal_fail(DK_ERR_INVALID_INPUT, "viewport must have positive area");
    if (w > dk::kMaxView || h > dk::kMaxView)
        return dk_internal_fail(DK_ERR_INVALID_INPUT, "viewport larger than 512 pixels");
    return DK_OK;
}

}  // namespace

extern "C" {

int dk_pixels_render_rgb(int64_t n, int w, int h, double pole_length, const double *frames,
                         const double *visuals, int brightness, uint8_t *out, void *stream) {
    dk::PtrDeviceGuard dg_(out);  // launch on the buffers' device
    if (int rc = check_view(w, h)) return rc;
    if (!frames || !visuals || !out)
        return dk_internal_fail(DK_ERR_INVALID_INPUT, "render: missing argument");
    if (n == 0) return DK_OK;
    dk::pixel_rgb_kernel<<<(unsigned)n, 256, 0, (cudaStream_t)stream>>>(
        n, w, h, pole_length, (const dk::PixFrame *)frames, visuals, brightness, out);
    return cuda_rc(cudaGetLastError(), "render launch");
}

int dk_pixels_advance(int dtype, int64_t n, int obs_dim, const void *obs,
                      const uint8_t *reset_mask, int first, double *history, double *visuals,
                      uint32_t *episode, int randomize, const dk_visual_bounds *bounds,
                      uint64_t seed, int64_t env_index_offset, int skip_words, void *stream) {
    dk::PtrDeviceGuard dg_(history);  // launch on the buffers' device
    if (!obs || !history || !visuals || !episode || !bounds)
        return dk_internal_fail(DK_ERR_INVALID_INPUT, "pixels advance: missing argument");
    if (obs_dim < 3)
        return dk_internal_fail(DK_ERR_INVALID_INPUT, "pixels need [x, cos, sin, ...] rows");
    if (n == 0) return DK_OK;
    dk::VisualBoundsC b;
    for (int k = 0; k < dk::kVis; ++k) b.nominal[k] = bounds->nominal[k];
    b.color_jitter = bounds->color_jitter;
    b.camera_offset_range = bounds->camera_offset_range;
    b.zoom_lo = bounds->zoom_range[0];
    b.zoom_hi = bounds->zoom_range[1];
    b.bright_lo = bounds->brightness_range[0];
    b.bright_hi = bounds->brightness_range[1];
    const unsigned g = (unsigned)((n + 127) / 128);
    cudaStream_t st = (cudaStream_t)stream;
    if (dtype == DK_F64)
        dk::pixel_advance_kernel<double><<<g, 128, 0, st>>>(
            n, obs_dim, (const double *)obs, reset_mask, first, (dk::PixFrame *)history, visuals,
            episode, randomize, b, seed, env_index_offset, skip_words);
    else
        dk::pixel_advance_kernel<float><<<g, 128, 0, st>>>(
            n, obs_dim, (const float *)obs, reset_mask, first, (dk::PixFrame *)history, visuals,
            episode, randomize, b, seed, env_index_offset, skip_words);
    return cuda_rc(cudaGetLastError(), "pixels advance launch");
}

int dk_pixels_stack(int dtype, int64_t n, int w, int h, double pole_length,
                    const double *history, const double *visuals, void *out, void *stream) {
    dk::PtrDeviceGuard dg_(out);  // launch on the buffers' device
    if (int rc = check_view(w, h)) return rc;
    if (!history || !visuals || !out)
        return dk_internal_fail(DK_ERR_INVALID_INPUT, "pixels stack: missing argument");
    if (n == 0) return DK_OK;
    cudaStream_t st = (cudaStream_t)stream;
    if (dtype == DK_F64)
        dk::pixel_stack_kernel<double><<<(unsigned)n, dk::kPixStackThreads, 0, st>>>(
            n, w, h, pole_length, (const dk::PixFrame *)history, visuals, (double *)out);
    else
        dk::pixel_stack_kernel<float><<<(unsigned)n, dk::kPixStackThreads, 0, st>>>(
            n, w, h, pole_length, (const dk::PixFrame *)history, visuals, (float *)out);
    return cuda_rc(cudaGetLastError(), "pixels stack launch");
}

int dk_pixels_terminal(int dtype, int64_t n, int w, int h, double pole_length, int obs_dim,
                       const void *term_obs, const uint8_t *mask, const double *history,
                       const double *visuals, void *out, void *stream) {
    dk::PtrDeviceGuard dg_(out);  // launch on the buffers' device
    if (int rc = check_view(w, h)) return rc;
    if (!term_obs || !mask || !history || !visuals || !out)
        return dk_internal_fail(DK_ERR_INVALID_INPUT, "pixels terminal: missing argument");
    if (n == 0) return DK_OK;
    cudaStream_t st = (cudaStream_t)stream;
    if (dtype == DK_F64)
        dk::pixel_terminal_kernel<double><<<(unsigned)n, 256, 0, st>>>(
            n, w, h, pole_length, obs_dim, (const double *)term_obs, mask,
            (const dk::PixFrame *)history, visuals, (double *)out);
    else
        dk::pixel_terminal_kernel<float><<<(unsigned)n, 256, 0, st>>>(
            n, w, h, pole_length, obs_dim, (const float *)term_obs, mask,
            (const dk::PixFrame *)history, visuals, (float *)out);
    return cuda_rc(cudaGetLastError(), "pixels terminal launch");
}

int dk_pixels_normalize(int in_dtype, int out_dtype, int64_t n, int h, int w, int c,
                        const void *x, int channels_first, double *stats, void *out,
                        void *stream) {
    dk::PtrDeviceGuard dg_(x);  // launch on the buffers' device
    // any positive image size (not the renderer's viewport limit), overflow-safe
    if (c <= 0 || n < 0 || h <= 0 || w <= 0 || (int64_t)h * w > (1LL << 30) / c)
        return dk_internal_fail(DK_ERR_INVALID_INPUT, "pixel_normalize: shape");
    if (n == 0) return DK_OK;
    if (!x || !stats || !out)
        return dk_internal_fail(DK_ERR_INVALID_INPUT, "pixel_normalize: missing argument");
    cudaStream_t st = (cudaStream_t)stream;
    const int hw = h * w;
    const unsigned gs = (unsigned)((n * c + 127) / 128);
    if (in_dtype == DK_F32 && c == 3 && hw % dk::pixnorm::PN == 0 && ((uintptr_t)x & 15) == 0 &&
        ((uintptr_t)out & 15) == 0) {
        static unsigned long long attr_set = 0;  // per device (bit = ordinal)
        int dev = 0;
        cudaGetDevice(&dev);
        if (dev >= 64 || !((attr_set >> dev) & 1ull)) {
            cudaError_t e = cudaFuncSetAttribute(dk::pixnorm_stats3_kernel,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 dk::pixnorm::SMEM);
            if (e != cudaSuccess) return cuda_rc(e, "pixel_normalize attribute");
            if (dev < 64) __atomic_fetch_or(&attr_set, 1ull << dev, __ATOMIC_RELAXED);
        }
        // samples per CTA: spread the batch over every SM's two CTA slots (the
        // stage reads are bound per SM), at most one warp of samples
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        int64_t spc = (n + 2 * (int64_t)sms - 1) / (2 * (int64_t)sms);
#ifdef DK_PIXNORM_SPC
        spc = DK_PIXNORM_SPC;
#endif
        spc = spc < 1 ? 1 : (spc > 32 ? 32 : spc);
        dk::pixnorm_stats3_kernel<<<(unsigned)((n + spc - 1) / spc), 96, dk::pixnorm::SMEM, st>>>(
            n, hw, (int)spc, (const float *)x, stats);
        const dim3 g((unsigned)((hw / 4 + 255) / 256), (unsigned)(n < 65535 ? n : 65535));
        const float *xf = (const float *)x;
        if (out_dtype == DK_F64) {
            if (channels_first)
                dk::pixnorm_apply3_kernel<double, true><<<g, 256, 0, st>>>(n, hw, xf, stats, (double *)out);
            else
                dk::pixnorm_apply3_kernel<double, false><<<g, 256, 0, st>>>(n, hw, xf, stats, (double *)out);
        } else {
            if (channels_first)
                dk::pixnorm_apply3_kernel<float, true><<<g, 256, 0, st>>>(n, hw, xf, stats, (float *)out);
            else
                dk::pixnorm_apply3_kernel<float, false><<<g, 256, 0, st>>>(n, hw, xf, stats, (float *)out);
        }
        return cuda_rc(cudaGetLastError(), "pixel_normalize launch");
    }
    if (in_dtype == DK_F64)
        dk::pixnorm_stats_kernel<double><<<gs, 128, 0, st>>>(n, hw, c, (const double *)x, stats);
    else
        dk::pixnorm_stats_kernel<float><<<gs, 128, 0, st>>>(n, hw, c, (const float *)x, stats);
    const int64_t total = n * (int64_t)hw * c;
    const unsigned ga = (unsigned)((total + 255) / 256);
    if (in_dtype == DK_F64 && out_dtype == DK_F64)
        dk::pixnorm_apply_kernel<double, double><<<ga, 256, 0, st>>>(
            n, hw, c, (const double *)x, stats, channels_first, (double *)out);
    else if (in_dtype == DK_F64)
        dk::pixnorm_apply_kernel<double, float><<<ga, 256, 0, st>>>(
            n, hw, c, (const double *)x, stats, channels_first, (float *)out);
    else if (out_dtype == DK_F64)
        dk::pixnorm_apply_kernel<float, double><<<ga, 256, 0, st>>>(
            n, hw, c, (const float *)x, stats, channels_first, (double *)out);
    else
        dk::pixnorm_apply_kernel<float, float><<<ga, 256, 0, st>>>(
            n, hw, c, (const float *)x, stats, channels_first, (float *)out);
    return cuda_rc(cudaGetLastError(), "pixel_normalize launch");
}

}  // extern "C"
