// envstep_launch.cuh -- host-side launchers, explicitly instantiated per real
// type in envstep_f32.cu / envstep_f64.cu (the f64 TU is compiled with
// --fmad=false to keep the reference's two-rounding arithmetic).
#pragma once
#include "envstep_kernels.cuh"
#include "devguard.h"

namespace dk {

// SM count of the current device (148 on B200), queried once per device
inline int sm_count() {
    static int cached[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return 148;
    if (!cached[dev]) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        cached[dev] = v > 0 ? v : 148;
    }
    return cached[dev];
}
#ifdef DK_NO_PDL
constexpr bool kUsePdl = false;
#else
constexpr bool kUsePdl = true;
#endif
#ifndef DK_MIN_ROLLOUT_SMEM
#define DK_MIN_ROLLOUT_SMEM (80 * 1024)
#endif
constexpr size_t kMinRolloutSmem = DK_MIN_ROLLOUT_SMEM;

inline int pick_block(int64_t n) {
    // Few worlds per GPU (1K-8K) is a latency-bound regime: spread warps over
    // all 148 SMs before stacking them on one SM.
    int bs = 256;
    const int sms = sm_count();
    while (bs > 32 && (n + bs - 1) / bs < 2 * sms) bs /= 2;
    return bs;
}

// Dynamic shared memory requested per rollout CTA: at least 80 KB so that at
// most two CTAs share an SM.  With programmatic dependent launch the next
// rollout's CTAs are placed while this one drains; a third 57 KB CTA would fit
// and leave some SMs with three chains (measured 17% slower at 8192 worlds).
template <class S>
constexpr size_t launch_smem() {
    return S::SMEM > kMinRolloutSmem ? S::SMEM : kMinRolloutSmem;
}

template <class Task, typename T, int TL>
inline cudaError_t launch_task_rollout_tl(const T *actions, int64_t K, const EnvScalars &sc,
                                          const Params<T> &p, const Worlds<T> &w,
                                          const StepOut<T> &out, unsigned long long *err,
                                          cudaStream_t st) {
    using S = RolloutShape<Task, T, TL>;
    static SmemOptIn optin[2];  // per device and instantiation; opt in above 48 KB
    {
        cudaError_t e = optin[0].ensure((const void *)rollout_kernel<Task, T, true, TL>,
                                        launch_smem<S>());
        if (e == cudaSuccess)
            e = optin[1].ensure((const void *)rollout_kernel<Task, T, false, TL>, launch_smem<S>());
        if (e != cudaSuccess) return e;
    }
    auto kern = sc.action_repeat == 1 ? rollout_kernel<Task, T, true, TL>
                                      : rollout_kernel<Task, T, false, TL>;
    const int64_t grid = (sc.n + S::WPC - 1) / S::WPC;  // one block per CTA tile
    // Programmatic dependent launch: back-to-back rollouts overlap this launch
    // (and its CTAs' set-up) with the previous rollout's drain; the kernel
    // waits (griddepcontrol.wait) before touching anything the previous grid
    // wrote, and each CTA releases its dependents once its producer is done.
    EnvScalars scl = sc;
    scl.solo_sm = grid <= sm_count() ? 1 : 0;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(S::THREADS);
    cfg.dynamicSmemBytes = launch_smem<S>();
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = kUsePdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, actions, K, scl, p, w, out, err);
}

// K = 1: one thread per world (step1_kernel), 64-thread blocks so that even a
// few thousand worlds spread over the SMs; programmatic dependent launch as
// the rollout kernel
template <class Task, typename T>
inline cudaError_t launch_task_step1(const T *actions, const EnvScalars &sc, const Params<T> &p,
                                     const Worlds<T> &w, const StepOut<T> &out,
                                     unsigned long long *err, cudaStream_t st) {
    auto kern = sc.action_repeat == 1 ? step1_kernel<Task, T, true> : step1_kernel<Task, T, false>;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)((sc.n + 63) / 64));
    cfg.blockDim = dim3(64);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = kUsePdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, actions, sc, p, w, out, err);
}

template <class Task, typename T>
inline cudaError_t launch_task_rollout(const T *actions, int64_t K, const EnvScalars &sc,
                                       const Params<T> &p, const Worlds<T> &w,
                                       const StepOut<T> &out, unsigned long long *err,
                                       cudaStream_t st, int64_t *launches) {
    *launches += 1;
#ifndef DK_NO_STEP1
    if (K == 1 && sc.n > 0) return launch_task_step1<Task, T>(actions, sc, p, w, out, err, st);
#endif
    return launch_task_rollout_tl<Task, T, 1>(actions, K, sc, p, w, out, err, st);
}

template <typename T>
cudaError_t launch_rollout(int task, const T *actions, int64_t K, const EnvScalars &sc,
                           const Params<T> &p, const Worlds<T> &w, const StepOut<T> &out,
                           unsigned long long *err, cudaStream_t st, int64_t *launches) {
    switch (task) {
    case 0: return launch_task_rollout<Pendulum<T>, T>(actions, K, sc, p, w, out, err, st, launches);
    case 1: return launch_task_rollout<Cartpole<T>, T>(actions, K, sc, p, w, out, err, st, launches);
    case 2: return launch_task_rollout<Acrobot<T>, T>(actions, K, sc, p, w, out, err, st, launches);
    default: return launch_task_rollout<Reacher<T>, T>(actions, K, sc, p, w, out, err, st, launches);
    }
}

template <class Task, typename T>
inline cudaError_t launch_task_reset(const EnvScalars &sc, const Params<T> &p, const Worlds<T> &w,
                                     int rewind, T *obs, cudaStream_t st, int64_t *launches) {
    const int bs = pick_block(sc.n);
    const int64_t grid = (sc.n + bs - 1) / bs;
    reset_kernel<Task, T><<<(unsigned)grid, bs, bs * Task::O * sizeof(T), st>>>(sc, p, w, rewind,
                                                                               obs);
    *launches += 1;
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_reset(int task, const EnvScalars &sc, const Params<T> &p, const Worlds<T> &w,
                         int rewind, T *obs, cudaStream_t st, int64_t *launches) {
    switch (task) {
    case 0: return launch_task_reset<Pendulum<T>, T>(sc, p, w, rewind, obs, st, launches);
    case 1: return launch_task_reset<Cartpole<T>, T>(sc, p, w, rewind, obs, st, launches);
    case 2: return launch_task_reset<Acrobot<T>, T>(sc, p, w, rewind, obs, st, launches);
    default: return launch_task_reset<Reacher<T>, T>(sc, p, w, rewind, obs, st, launches);
    }
}

template <typename T>
cudaError_t launch_get_state(int task, const EnvScalars &sc, const Worlds<T> &w, double *s4,
                             double *t2, cudaStream_t st) {
    const int bs = 128;
    const unsigned grid = (unsigned)((sc.n + bs - 1) / bs);
    switch (task) {
    case 0: get_state_kernel<Pendulum<T>, T><<<grid, bs, 0, st>>>(sc, w, s4, t2); break;
    case 1: get_state_kernel<Cartpole<T>, T><<<grid, bs, 0, st>>>(sc, w, s4, t2); break;
    case 2: get_state_kernel<Acrobot<T>, T><<<grid, bs, 0, st>>>(sc, w, s4, t2); break;
    default: get_state_kernel<Reacher<T>, T><<<grid, bs, 0, st>>>(sc, w, s4, t2); break;
    }
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_set_state(int task, const EnvScalars &sc, const Worlds<T> &w, const double *s4,
                             const double *t2, cudaStream_t st) {
    const int bs = 128;
    const unsigned grid = (unsigned)((sc.n + bs - 1) / bs);
    switch (task) {
    case 0: set_state_kernel<Pendulum<T>, T><<<grid, bs, 0, st>>>(sc, w, s4, t2); break;
    case 1: set_state_kernel<Cartpole<T>, T><<<grid, bs, 0, st>>>(sc, w, s4, t2); break;
    case 2: set_state_kernel<Acrobot<T>, T><<<grid, bs, 0, st>>>(sc, w, s4, t2); break;
    default: set_state_kernel<Reacher<T>, T><<<grid, bs, 0, st>>>(sc, w, s4, t2); break;
    }
    return cudaGetLastError();
}

// Explicit instantiation declarations (definitions in envstep_f32.cu / _f64.cu).
#define DK_DECLARE_LAUNCHERS(T)                                                                  \
    extern template cudaError_t launch_rollout<T>(int, const T *, int64_t, const EnvScalars &,   \
                                                  const Params<T> &, const Worlds<T> &,          \
                                                  const StepOut<T> &, unsigned long long *,      \
                                                  cudaStream_t, int64_t *);                      \
    extern template cudaError_t launch_reset<T>(int, const EnvScalars &, const Params<T> &,      \
                                                const Worlds<T> &, int, T *, cudaStream_t,       \
                                                int64_t *);                                      \
    extern template cudaError_t launch_get_state<T>(int, const EnvScalars &, const Worlds<T> &,  \
                                                    double *, double *, cudaStream_t);           \
    extern template cudaError_t launch_set_state<T>(int, const EnvScalars &, const Worlds<T> &,  \
                                                    const double *, const double *, cudaStream_t);

#define DK_INSTANTIATE_LAUNCHERS(T)                                                              \
    template cudaError_t launch_rollout<T>(int, const T *, int64_t, const EnvScalars &,          \
                                           const Params<T> &, const Worlds<T> &,                 \
                                           const StepOut<T> &, unsigned long long *,             \
                                           cudaStream_t, int64_t *);                             \
    template cudaError_t launch_reset<T>(int, const EnvScalars &, const Params<T> &,             \
                                         const Worlds<T> &, int, T *, cudaStream_t, int64_t *);  \
    template cudaError_t launch_get_state<T>(int, const EnvScalars &, const Worlds<T> &,         \
                                             double *, double *, cudaStream_t);                  \
    template cudaError_t launch_set_state<T>(int, const EnvScalars &, const Worlds<T> &,         \
                                             const double *, const double *, cudaStream_t);

}  // namespace dk
