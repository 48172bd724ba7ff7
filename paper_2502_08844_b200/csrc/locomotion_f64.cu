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
}
