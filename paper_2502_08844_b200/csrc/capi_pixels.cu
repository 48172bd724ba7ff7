// capi_pixels.cu -- extern "C" entry points of the cartpole pixel observation
// path (include/deskrl_b200.h).
#include <cstdio>

#include "../../include/deskrl_b200.h"
#include "pixels.cuh"

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
    if (int rc = check_view(w, h)) return rc;
    if (!history || !visuals || !out)
        return dk_internal_fail(DK_ERR_INVALID_INPUT, "pixels stack: missing argument");
    if (n == 0) return DK_OK;
    cudaStream_t st = (cudaStream_t)stream;
    if (dtype == DK_F64)
        dk::pixel_stack_kernel<double><<<(unsigned)n, 256, 0, st>>>(
            n, w, h, pole_length, (const dk::PixFrame *)history, visuals, (double *)out);
    else
        dk::pixel_stack_kernel<float><<<(unsigned)n, 256, 0, st>>>(
            n, w, h, pole_length, (const dk::PixFrame *)history, visuals, (float *)out);
    return cuda_rc(cudaGetLastError(), "pixels stack launch");
}

int dk_pixels_terminal(int dtype, int64_t n, int w, int h, double pole_length, int obs_dim,
                       const void *term_obs, const uint8_t *mask, const double *history,
                       const double *visuals, void *out, void *stream) {
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

}  // extern "C"
