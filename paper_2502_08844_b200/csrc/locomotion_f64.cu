// float64 instantiation of the locomotion step-tail kernels (--fmad=false:
// the reference's two-rounding arithmetic).
#include "locomotion.cuh"
namespace dk {
DK_LOCO_LAUNCHERS(, double)

// curriculum_update is integer-only; it lives in this unit once.
cudaError_t launch_curriculum(int64_t n, int64_t *state, const uint8_t *success,
                              int64_t max_level, int64_t threshold, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    curriculum_kernel<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(n, state, success, max_level,
                                                                  threshold);
    return cudaGetLastError();
}

// randomize_params and the delay-line reset are f64 / integer-only: this unit once.
cudaError_t launch_randomize_params(int64_t n, int nf, const double *nominal, int nr,
                                    const int *field, const int *dist, const double *lo,
                                    const double *hi, uint64_t seed, int64_t env0,
                                    const uint32_t *episode, uint64_t step, double *out,
                                    unsigned long long *fail, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    randomize_params_kernel<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(
        n, nf, nominal, nr, field, dist, lo, hi, seed, env0, episode, step, out, fail);
    return cudaGetLastError();
}

cudaError_t launch_delay_reset(int64_t n, int min_delay, int max_delay, uint64_t seed,
                               int64_t env0, const uint32_t *episode, uint64_t step,
                               int32_t *delay, int32_t *count, int32_t *head, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    delay_reset_kernel<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(
        n, min_delay, max_delay, seed, env0, episode, step, delay, count, head);
    return cudaGetLastError();
}
}
