// capi_loco.cu -- extern "C" entry points of the locomotion step tail
// (include/deskrl_b200.h).
#include <cstdio>
#include <string>

#include "../../include/deskrl_b200.h"
#include "locomotion.cuh"

namespace dk {
DK_LOCO_LAUNCHERS(extern, float)
DK_LOCO_LAUNCHERS(extern, double)
cudaError_t launch_curriculum(int64_t n, int64_t *state, const uint8_t *success,
                              int64_t max_level, int64_t threshold, cudaStream_t st);
cudaError_t launch_randomize_params(int64_t n, int nf, const double *nominal, int nr,
                                    const int *field, const int *dist, const double *lo,
                                    const double *hi, uint64_t seed, int64_t env0,
                                    const uint32_t *episode, uint64_t step, double *out,
                                    unsigned long long *fail, cudaStream_t st);
cudaError_t launch_delay_reset(int64_t n, int min_delay, int max_delay, uint64_t seed,
                               int64_t env0, const uint32_t *episode, uint64_t step,
                               int32_t *delay, int32_t *count, int32_t *head, cudaStream_t st);
}  // namespace dk

extern "C" int dk_internal_fail(int code, const char *msg);  // capi.cu

namespace {

int cuda_rc(cudaError_t e, const char *what) {
    if (e == cudaSuccess) return DK_OK;
    char buf[256];
    snprintf(buf, sizeof(buf), "%s: %s", what, cudaGetErrorString(e));
    return dk_internal_fail(DK_ERR_CUDA, buf);
}

template <typename T>
dk::RewardCfg<T> reward_cfg(const dk_reward_config &c) {
    dk::RewardCfg<T> r;
    const double w[16] = {c.w_lin_vel, c.w_ang_vel, c.w_airtime, c.w_clearance, c.w_phase,
                          c.w_slip, c.w_orientation, c.w_torque, c.w_joint_pos,
                          c.w_action_rate, c.w_energy, c.w_pose, c.w_termination,
                          c.w_standstill, c.w_lin_vel_z, c.w_ang_vel_xy};
    for (int k = 0; k < 16; ++k) r.w[k] = (T)w[k];
    r.sigma_lin = (T)c.sigma_lin_vel;
    r.sigma_ang = (T)c.sigma_ang_vel;
    r.airtime_min = (T)c.airtime_min;
    r.airtime_max = (T)c.airtime_max;
    r.sigma_phase = (T)c.sigma_phase;
    r.swing_height = (T)c.swing_height;
    r.gated = c.standstill_gated != 0;
    return r;
}

template <typename T>
dk::LocoFrames<T> frames_of(const dk_loco_frames &f) {
    dk::LocoFrames<T> o;
    o.q = (const T *)f.base_orientation; o.lin = (const T *)f.base_lin_vel;
    o.ang = (const T *)f.base_ang_vel; o.jpos = (const T *)f.joint_pos;
    o.jvel = (const T *)f.joint_vel; o.jtau = (const T *)f.joint_torque;
    o.fh = (const T *)f.foot_height; o.fhd = (const T *)f.foot_height_des;
    o.fvel = (const T *)f.foot_vel_xy; o.contact = f.foot_contact;
    o.air = (const T *)f.airtime; o.touchdown = f.touchdown; o.phase = (const T *)f.phase;
    o.cmd = (const T *)f.command; o.act = (const T *)f.action;
    o.pact = (const T *)f.prev_action; o.nom = (const T *)f.joint_nominal;
    o.def = (const T *)f.joint_default; o.done = f.done;
    o.nom_stride = f.nominal_stride;
    o.def_stride = f.default_stride;
    return o;
}

template <typename T>
int tail(int64_t K, int64_t N, int nj, int nf, const dk_reward_config *cfg,
         const dk_loco_frames *fr, const void *pa, const void *cmd, const double *noise,
         const dk_noise_key *key, const void *pert, const dk_loco_outputs *out,
         unsigned long long *bad, cudaStream_t st) {
    dk::LocoArgs a;
    a.K = K; a.N = N; a.nj = nj; a.nf = nf;
    a.seed = key ? key->seed : 0;
    a.env0 = key ? key->env_index_offset : 0;
    a.step0 = key ? key->step : 0;
    a.episode = key ? key->episode : nullptr;
    a.has_noise = noise != nullptr;
    for (int k = 0; k < 5; ++k) a.noise[k] = noise ? noise[k] : 0.0;
    dk::LocoOut<T> o{(T *)out->total, (T *)out->unclipped, (T *)out->terms, (T *)out->state_obs,
                     (T *)out->privileged_obs};
    return cuda_rc(dk::launch_loco_tail<T>(frames_of<T>(*fr), (const T *)pa, (const T *)cmd,
                                           (const T *)pert, reward_cfg<T>(*cfg), a, o, bad, st),
                   "loco tail launch");
}

}  // namespace

extern "C" {

int dk_loco_tail(int dtype, int64_t K, int64_t N, int nj, int nf, const dk_reward_config *cfg,
                 const dk_loco_frames *frames, const void *prev_action, const void *command,
                 const double *noise, const dk_noise_key *key, const void *pert,
                 const dk_loco_outputs *out, unsigned long long *bad_row, void *stream) {
    if (!cfg || !frames || !out || !out->total || !out->unclipped || !bad_row)
        return dk_internal_fail(DK_ERR_INVALID_INPUT, "dk_loco_tail: missing argument");
    if (nj < 1 || nf < 1 || nj > 256 || nf > 64 || K < 0 || N < 0)
        return dk_internal_fail(DK_ERR_INVALID_INPUT, "dk_loco_tail: bad dimensions");
    if (cfg->sigma_lin_vel <= 0 || cfg->sigma_ang_vel <= 0 || cfg->sigma_phase <= 0)
        return dk_internal_fail(DK_ERR_CONFIG, "kernel scales must be positive");
    if (cfg->airtime_min > cfg->airtime_max)
        return dk_internal_fail(DK_ERR_CONFIG, "airtime_min must not exceed airtime_max");
    cudaStream_t st = (cudaStream_t)stream;
    if (dtype == DK_F64)
        return tail<double>(K, N, nj, nf, cfg, frames, prev_action, command, noise, key, pert,
                            out, bad_row, st);
    return tail<float>(K, N, nj, nf, cfg, frames, prev_action, command, noise, key, pert, out,
                       bad_row, st);
}

int dk_loco_pd(int dtype, int64_t n, int nj, const double *pp, const void *qdef, const void *a,
               const void *prev, const void *q, const void *qd, void *target, void *torque,
               void *stream) {
    if (!pp || !qdef || !a || !q || !qd || !torque)
        return dk_internal_fail(DK_ERR_INVALID_INPUT, "dk_loco_pd: missing argument");
    if (pp[0] < 0 || pp[1] < 0)
        return dk_internal_fail(DK_ERR_INVALID_INPUT, "PD gains must be non-negative");
    if (pp[2] <= 0) return dk_internal_fail(DK_ERR_INVALID_INPUT, "action scale must be positive");
    const int rel = pp[6] != 0.0;
    if (rel && !prev)
        return dk_internal_fail(DK_ERR_INVALID_INPUT, "relative PD mode needs prev_target");
    cudaStream_t st = (cudaStream_t)stream;
    if (dtype == DK_F64)
        return cuda_rc(dk::launch_pd<double>(n, nj, pp[0], pp[1], pp[2], pp[3], pp[4], pp[5], rel,
                                             (const double *)qdef, (const double *)a,
                                             (const double *)prev, (const double *)q,
                                             (const double *)qd, (double *)target,
                                             (double *)torque, st),
                       "pd launch");
    return cuda_rc(dk::launch_pd<float>(n, nj, (float)pp[0], (float)pp[1], (float)pp[2],
                                        (float)pp[3], (float)pp[4], (float)pp[5], rel,
                                        (const float *)qdef, (const float *)a,
                                        (const float *)prev, (const float *)q, (const float *)qd,
                                        (float *)target, (float *)torque, st),
                   "pd launch");
}

int dk_loco_phase(int dtype, int64_t n, int nf, const void *phi, const void *freq, const void *dt,
                  void *phi_out, void *cs_out, void *stream) {
    if (!phi || !freq || !dt)
        return dk_internal_fail(DK_ERR_INVALID_INPUT, "dk_loco_phase: missing argument");
    cudaStream_t st = (cudaStream_t)stream;
    if (dtype == DK_F64)
        return cuda_rc(dk::launch_phase<double>(n, nf, (const double *)phi, (const double *)freq,
                                                (const double *)dt, (double *)phi_out,
                                                (double *)cs_out, st),
                       "phase launch");
    return cuda_rc(dk::launch_phase<float>(n, nf, (const float *)phi, (const float *)freq,
                                           (const float *)dt, (float *)phi_out, (float *)cs_out,
                                           st),
                   "phase launch");
}

int dk_loco_progress_clip(int dtype, int64_t n, const void *raw, void *hist, void *reward,
                          void *stream) {
    if (!raw || !hist || !reward)
        return dk_internal_fail(DK_ERR_INVALID_INPUT, "dk_loco_progress_clip: missing argument");
    cudaStream_t st = (cudaStream_t)stream;
    if (dtype == DK_F64)
        return cuda_rc(dk::launch_progress<double>(n, (const double *)raw, (double *)hist,
                                                   (double *)reward, st),
                       "progress launch");
    return cuda_rc(dk::launch_progress<float>(n, (const float *)raw, (float *)hist,
                                              (float *)reward, st),
                   "progress launch");
}

int dk_dr_sensor_noise(int dtype, int64_t n, int dim, void *obs, int nspec, const int32_t *off,
                       const int32_t *len, const double *scale, const int32_t *kind,
                       const dk_noise_key *key, void *stream) {
    if (!obs || !key || (nspec > 0 && (!off || !len || !scale)))
        return dk_internal_fail(DK_ERR_INVALID_INPUT, "dk_dr_sensor_noise: missing argument");
    cudaStream_t st = (cudaStream_t)stream;
    if (dtype == DK_F64)
        return cuda_rc(dk::launch_sensor_noise<double>(n, dim, (double *)obs, nspec, off, len, scale,
                                                       kind, key->seed, key->env_index_offset,
                                                       key->episode, key->step, st),
                       "sensor noise launch");
    return cuda_rc(dk::launch_sensor_noise<float>(n, dim, (float *)obs, nspec, off, len, scale,
                                                  kind, key->seed, key->env_index_offset,
                                                  key->episode, key->step, st),
                   "sensor noise launch");
}

int dk_dr_randomize_params(int64_t n, int num_fields, const double *nominal, int num_ranges,
                           const int32_t *field, const int32_t *distribution, const double *low,
                           const double *high, const dk_noise_key *key, double *out,
                           unsigned long long *fail_world, void *stream) {
    if (!nominal || !out || !key || !fail_world ||
        (num_ranges > 0 && (!field || !distribution || !low || !high)))
        return dk_internal_fail(DK_ERR_INVALID_INPUT, "dk_dr_randomize_params: missing argument");
    if (num_fields <= 0 || num_ranges < 0)
        return dk_internal_fail(DK_ERR_INVALID_INPUT, "dk_dr_randomize_params: bad sizes");
    return cuda_rc(dk::launch_randomize_params(n, num_fields, nominal, num_ranges, field,
                                               distribution, low, high, key->seed,
                                               key->env_index_offset, key->episode, key->step,
                                               out, fail_world, (cudaStream_t)stream),
                   "randomize_params launch");
}

int dk_dr_delay_reset(int64_t n, int min_delay, int max_delay, const dk_noise_key *key,
                      int32_t *delay, int32_t *count, int32_t *head, void *stream) {
    if (!key || !delay || !count || !head)
        return dk_internal_fail(DK_ERR_INVALID_INPUT, "dk_dr_delay_reset: missing argument");
    if (min_delay < 0 || max_delay < min_delay)
        return dk_internal_fail(DK_ERR_CONFIG, "delay bounds must satisfy 0 <= min <= max");
    return cuda_rc(dk::launch_delay_reset(n, min_delay, max_delay, key->seed,
                                          key->env_index_offset, key->episode, key->step, delay,
                                          count, head, (cudaStream_t)stream),
                   "delay reset launch");
}

int dk_dr_delay_push_pop(int dtype, int64_t n, int dim, int min_delay, int max_delay,
                         int per_step, void *ring, int32_t *head, int32_t *count,
                         const int32_t *delay, const dk_noise_key *key, const void *value,
                         void *out, void *stream) {
    if (!ring || !head || !count || !delay || !key || !value || !out)
        return dk_internal_fail(DK_ERR_INVALID_INPUT, "dk_dr_delay_push_pop: missing argument");
    if (min_delay < 0 || max_delay < min_delay)
        return dk_internal_fail(DK_ERR_CONFIG, "delay bounds must satisfy 0 <= min <= max");
    cudaStream_t st = (cudaStream_t)stream;
    if (dtype == DK_F64)
        return cuda_rc(dk::launch_delay_push_pop<double>(
                           n, dim, min_delay, max_delay, per_step, (double *)ring, head, count,
                           delay, key->seed, key->env_index_offset, key->episode, key->step,
                           (const double *)value, (double *)out, st),
                       "delay push_pop launch");
    return cuda_rc(dk::launch_delay_push_pop<float>(
                       n, dim, min_delay, max_delay, per_step, (float *)ring, head, count, delay,
                       key->seed, key->env_index_offset, key->episode, key->step,
                       (const float *)value, (float *)out, st),
                   "delay push_pop launch");
}

int dk_dr_pose_injection(int dtype, int64_t n, int dim, void *pose, const double *bounds,
                         double prob, const dk_noise_key *key, uint8_t *injected, void *stream) {
    if (!pose || !bounds || !key)
        return dk_internal_fail(DK_ERR_INVALID_INPUT, "dk_dr_pose_injection: missing argument");
    if (!(prob >= 0.0 && prob <= 1.0))
        return dk_internal_fail(DK_ERR_INVALID_INPUT, "prob must lie in [0, 1]");
    cudaStream_t st = (cudaStream_t)stream;
    if (dtype == DK_F64)
        return cuda_rc(dk::launch_pose_injection<double>(n, dim, (double *)pose, bounds, prob,
                                                         key->seed, key->env_index_offset,
                                                         key->episode, key->step, injected, st),
                       "pose injection launch");
    return cuda_rc(dk::launch_pose_injection<float>(n, dim, (float *)pose, bounds, prob,
                                                    key->seed, key->env_index_offset,
                                                    key->episode, key->step, injected, st),
                   "pose injection launch");
}

int dk_dr_curriculum(int64_t n, int64_t *state, const uint8_t *success, int64_t max_level,
                     int64_t threshold, void *stream) {
    if (!state || !success)
        return dk_internal_fail(DK_ERR_INVALID_INPUT, "dk_dr_curriculum: missing argument");
    return cuda_rc(dk::launch_curriculum(n, state, success, max_level, threshold,
                                         (cudaStream_t)stream),
                   "curriculum launch");
}

}  // extern "C"
