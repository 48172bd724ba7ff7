/*
 * deskrl_b200.h -- C ABI of the B200-native batched env step.
 *
 * This is the drop-in boundary for the reference's hot path, the batched
 * env reset/step of deskrl (/root/reference/pkg/src/deskrl/envkit.py:595-650).
 * The reference has no native layer; its specified native boundary is the
 * "bindings" BoundEnvHandle (make_env / reset / step with
 * contiguous arrays, single-writer handle), realised there as JSON over stdio
 * (serve.py:48-108).  Each entry point below names the reference interface it
 * replaces.  INTEGRATION.md shows the ctypes binding a maintainer would add.
 *
 * Conventions
 *  - Plain C types only.  Buffers are caller-owned.  Functions without the
 *    _host suffix take DEVICE pointers and enqueue work on `stream`
 *    (a cudaStream_t passed as void*, NULL = legacy default stream) without
 *    synchronising.  The _host variants take host pointers (pinned for full
 *    speed), copy in/out internally and return after the results are in the
 *    host buffers, like the reference's synchronous numpy call.
 *  - Element type of every floating-point buffer is the env's dtype
 *    (DK_F32 -> float, DK_F64 -> double).  Flags are uint8 (0/1).
 *  - Layouts are row-major: actions [N, A]; obs [N, O]; rewards [N];
 *    info [N, I].  Rollouts are time-major: [K, N, ...].
 *  - Return value: DK_OK or a DK_ERR_* code; dk_last_error() holds the
 *    message (thread-local).
 *  - A handle is single-writer: do not drive one handle from
 *    two host threads at once.
 */
#ifndef DESKRL_B200_H
#define DESKRL_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DK_ABI_VERSION 7  /* 2: DR kinds / params / delays; 3: PPO math; 4: pixels; 5-6: normaliser halves, workspace; 7: pixel_normalize */

/* Status codes.  The Python host maps them to the reference's exception
 * classes: ConfigError (randomization.py:19), InvalidInputError
 * (mathcore.py:22), UsageError (envkit.py:37). */
enum {
    DK_OK = 0,
    DK_ERR_CONFIG = 1,
    DK_ERR_INVALID_INPUT = 2,
    DK_ERR_USAGE = 3,
    DK_ERR_CUDA = 4,
};

/* Task ids; names as registered_tasks() (envkit.py:456-462). */
enum {
    DK_TASK_PENDULUM_SWINGUP = 0, /* "pendulum-swingup"  envkit.py:255-294 */
    DK_TASK_CARTPOLE_BALANCE = 1, /* "cartpole-balance"  envkit.py:297-349 */
    DK_TASK_ACROBOT_SWINGUP = 2,  /* "acrobot-swingup"   envkit.py:383-409 */
    DK_TASK_REACHER_EASY = 3,     /* "reacher-easy"      envkit.py:412-453 */
};

enum { DK_F32 = 0, DK_F64 = 1 };

/* Model: DynamicsParams (dynamics.py:36-60), same fields, same order.
 * dt is the effective step (EnvConfig.dt or the task default,
 * envkit.py:485-487). */
typedef struct dk_dynamics_params {
    double dt, gravity;
    double pend_mass, pend_length, pend_damping, pend_torque_limit;
    double cart_mass, pole_mass, pole_length, rail_limit, cart_force_limit;
    double link1_mass, link2_mass, link1_length, link2_length, link_damping;
    double elbow_torque_limit, reacher_torque_limit;
} dk_dynamics_params;

/* EnvConfig fields on the step path (envkit.py:56-75). */
typedef struct dk_env_config {
    int32_t task;           /* DK_TASK_* */
    int32_t dtype;          /* DK_F32 or DK_F64: arithmetic and buffer type */
    int64_t episode_length; /* control steps, 1 .. 2^31-1 */
    int64_t action_repeat;  /* >= 1 */
    int32_t wide_init;      /* pendulum full-circle starts (envkit.py:263-268) */
    int32_t reserved;
    uint64_t seed;          /* EnvConfig.seed; reset() may replace it */
} dk_env_config;

typedef struct dk_env dk_env;

/* Task name -> DK_TASK_* (or -1); dimensions of a task. */
int dk_task_id(const char *name);
int dk_task_dims(int task, int *action_dim, int *obs_dim, int *info_dim);

/* BatchEnv.__init__ (envkit.py:598-609) + Environment.__init__ (472-495).
 * Allocates the per-world state (structure of arrays) on `device`.
 * env_index_offset is the global index of world 0 (multi-GPU sharding:
 * rank r passes r*num_envs so Philox streams match a single-device run). */
int dk_env_create(const dk_env_config *cfg, const dk_dynamics_params *params,
                  int64_t num_envs, int64_t env_index_offset, int device, dk_env **out);

/* BatchEnv.close (envkit.py:648-650); frees device memory. */
int dk_env_destroy(dk_env *env);

/* BatchEnv.reset (envkit.py:616-623).  has_seed != 0 models reset(seed=s):
 * seed replaced, episode counters rewound; otherwise every world starts its
 * next episode.  Clears a pending sticky error.  obs_out: [N, O] device. */
int dk_env_reset(dk_env *env, int has_seed, uint64_t seed, void *obs_out, void *stream);

/* BatchEnv.step (envkit.py:625-646) on device buffers.
 *   actions        [N, A]  in
 *   obs_out        [N, O]  observation after the step (post-reset obs where
 *                          a world auto-reset), == "state" == "privileged_state"
 *   reward_out     [N]
 *   done_out       [N]     u8 (always 0 for these tasks, envkit.py:543)
 *   trunc_out      [N]     u8
 *   terminal_obs   [N, O]  written only where terminal_mask is 1 (may be NULL)
 *   terminal_mask  [N]     u8, infos[i]["terminal_observation"] present (may be NULL)
 *   info_out       [N, I]  reward terms of infos[i] (may be NULL)
 * Validation is batch-atomic: a non-finite action or a world that needs a
 * reset makes the whole call a no-op and leaves a sticky error that
 * dk_env_check_error() reports (the reference raises after having stepped
 * the worlds before the offending one, envkit.py:527-531, 630-637). */
int dk_env_step(dk_env *env, const void *actions, int autoreset, void *obs_out, void *reward_out,
                uint8_t *done_out, uint8_t *trunc_out, void *terminal_obs_out,
                uint8_t *terminal_mask_out, void *info_out, void *stream);

/* K consecutive BatchEnv.step(autoreset=True) calls fused into one launch
 * (the unroll loop of ppo.collect_rollout, ppo.py:308-322, and of
 * bench.measure_stage, bench.py:122-125).  actions [K, N, A]; outputs
 * [K, N, ...] time-major, same meaning as dk_env_step. */
int dk_env_rollout(dk_env *env, int64_t num_steps, const void *actions, void *obs_out,
                   void *reward_out, uint8_t *done_out, uint8_t *trunc_out,
                   void *terminal_obs_out, uint8_t *terminal_mask_out, void *info_out,
                   void *stream);

/* Host-buffer variants (synchronous).  dk_env_rollout_host pipelines the
 * host<->device copies of chunks of `chunk_steps` steps against the compute
 * of neighbouring chunks on internal streams. */
int dk_env_reset_host(dk_env *env, int has_seed, uint64_t seed, void *obs_out);
int dk_env_step_host(dk_env *env, const void *actions, int autoreset, void *obs_out,
                     void *reward_out, uint8_t *done_out, uint8_t *trunc_out,
                     void *terminal_obs_out, uint8_t *terminal_mask_out, void *info_out);
int dk_env_rollout_host(dk_env *env, int64_t num_steps, int64_t chunk_steps, const void *actions,
                        void *obs_out, void *reward_out, uint8_t *done_out, uint8_t *trunc_out,
                        void *terminal_obs_out, uint8_t *terminal_mask_out, void *info_out);

/* Synchronises `stream` and reports (then clears) the sticky error left by
 * dk_env_step / dk_env_rollout: returns DK_OK, DK_ERR_INVALID_INPUT
 * (non-finite action) or DK_ERR_USAGE (world needs reset); *step_index and
 * *env_index locate the first offending (step, world) in reference order. */
int dk_env_check_error(dk_env *env, void *stream, int64_t *step_index, int64_t *env_index);

/* Per-world state as float64 host arrays (Environment.state / steps /
 * _episode / _needs_reset / _target, envkit.py:490-513): state [N, 4],
 * target [N, 2], steps [N], episode [N], needs_reset [N].  Any may be NULL.
 * Synchronous.  set_state writes them back (tests, render-preview). */
int dk_env_get_state(dk_env *env, double *state, double *target, int64_t *steps,
                     int64_t *episode, uint8_t *needs_reset);
int dk_env_set_state(dk_env *env, const double *state, const double *target,
                     const int64_t *steps, const int64_t *episode, const uint8_t *needs_reset);

/* Number of kernels this handle has launched (evidence for bench.py). */
int64_t dk_env_kernel_launches(const dk_env *env);

/* ------------------------------------------------------------------------ */
/* Locomotion step tail.  These replace per-frame */
/* pure functions of the reference that the north_star fuses into the step  */
/* tail; all pointers are DEVICE pointers, element type = dtype (DK_F32 /    */
/* DK_F64), rows row-major.  Noise draws come from the Philox stream         */
/* stream_rng(key.seed, key.env_index_offset + world, episode[world], step)  */
/* (envkit.py:41-49), so they are bit-compatible with the reference given    */
/* the same generator.                                                       */

/* RewardTermConfig (rewards.py:51-75), same fields, same order. */
typedef struct dk_reward_config {
    double w_lin_vel, sigma_lin_vel, w_ang_vel, sigma_ang_vel, w_airtime, airtime_min,
        airtime_max, w_clearance, w_phase, sigma_phase, swing_height, w_slip, w_orientation,
        w_torque, w_joint_pos, w_action_rate, w_energy, w_pose, w_termination, w_standstill,
        w_lin_vel_z, w_ang_vel_xy;
    int32_t standstill_gated;
    int32_t reserved;
} dk_reward_config;

/* A batch of LocomotionFrame (rewards.py:17-44): every field [R, dim] with
 * R = num_steps * num_worlds rows (step-major).  Flags are uint8.
 * joint_nominal / joint_default may be one broadcast [J] row (stride 0). */
typedef struct dk_loco_frames {
    const void *base_orientation, *base_lin_vel, *base_ang_vel, *joint_pos, *joint_vel,
        *joint_torque, *foot_height, *foot_height_des, *foot_vel_xy;
    const uint8_t *foot_contact;
    const void *airtime;
    const uint8_t *touchdown;
    const void *phase, *command, *action, *prev_action, *joint_nominal, *joint_default;
    const uint8_t *done;
    int64_t nominal_stride, default_stride;
} dk_loco_frames;

/* total_reward's RewardBreakdown (rewards.py:84-89, 201-211) and the two
 * observation slots of build_locomotion_observation (envkit.py:147-193).
 * terms [R,16] (TERM_REGISTRY order), state_obs [R, 9+3J+3+2F],
 * privileged_obs [R, 9+3J+3+2F + F+J+3]; terms / obs pointers may be NULL. */
typedef struct dk_loco_outputs {
    void *total, *unclipped, *terms, *state_obs, *privileged_obs;
} dk_loco_outputs;

typedef struct dk_noise_key {
    uint64_t seed;
    int64_t env_index_offset;
    const uint32_t *episode; /* [num_worlds] device, or NULL for episode 0 */
    uint64_t step;           /* step of row block 0; block k uses step + k */
} dk_noise_key;

/* rewards.total_reward + envkit.build_locomotion_observation fused.
 * prev_action [R,J] / command [R,3] default to the frame's fields when NULL;
 * obs_noise: host double[5] ObservationNoise (gravity, lin_vel, ang_vel,
 * joint_pos, joint_vel) or NULL; perturbation [R,3] or NULL.
 * bad_row: device u64 the caller initialises to ~0; receives the first row
 * whose quaternion is not unit (InvalidInputError, mathcore.py:46-47). */
int dk_loco_tail(int dtype, int64_t num_steps, int64_t num_worlds, int num_joints, int num_feet,
                 const dk_reward_config *cfg, const dk_loco_frames *frames,
                 const void *prev_action, const void *command, const double *obs_noise,
                 const dk_noise_key *key, const void *perturbation, const dk_loco_outputs *out,
                 unsigned long long *bad_row, void *stream);

/* action_to_target + pd_torque (envkit.py:111-131).  pd_params (host):
 * kp, kd, action_scale, torque_limit, range_lo, range_hi, relative(0/1). */
int dk_loco_pd(int dtype, int64_t n, int num_joints, const double *pd_params,
               const void *q_default, const void *action, const void *prev_target, const void *q,
               const void *qd, void *target, void *torque, void *stream);

/* advance_phase + phase_encode (mathcore.py:143-177): phi [n,F], freq/dt [n];
 * phi_out [n,F] and/or cos_sin_out [n,F,2]. */
int dk_loco_phase(int dtype, int64_t n, int num_feet, const void *phi, const void *freq,
                  const void *dt, void *phi_out, void *cos_sin_out, void *stream);

/* progress_clip_reward (envkit.py:196-202); history_max updated in place. */
int dk_loco_progress_clip(int dtype, int64_t n, const void *raw, void *history_max, void *reward,
                          void *stream);

/* apply_sensor_noise (randomization.py:88-108), in place on obs [n, dim];
 * specs as device arrays (offset, length, scale, kind) in spec order; kind 0 =
 * uniform U(-scale, scale), 1 = gaussian Generator.normal(0, scale) (NumPy's
 * ziggurat, bit-compatible); kind may be NULL (all uniform).  Each world draws
 * from stream_rng(seed, env_index_offset + world, episode, step). */
int dk_dr_sensor_noise(int dtype, int64_t n, int dim, void *obs, int num_specs,
                       const int32_t *spec_offset, const int32_t *spec_length,
                       const double *spec_scale, const int32_t *spec_kind,
                       const dk_noise_key *key, void *stream);

/* randomize_params (randomization.py:156-181) for n worlds, float64: out
 * [n, num_fields] = nominal [num_fields] with ranges r (device arrays, spec
 * order) applied to field[r]: distribution 0 uniform_additive, 1
 * uniform_multiplicative, 2 log_uniform (low/high already log()ed by the
 * caller); a positive nominal is redrawn while non-positive, up to 100 tries.
 * fail_world: device u64 the caller initialises to ~0; receives
 * world * num_ranges + range of the first world (then range) that could not
 * be drawn (ConfigError, randomization.py:179). */
int dk_dr_randomize_params(int64_t n, int num_fields, const double *nominal, int num_ranges,
                           const int32_t *field, const int32_t *distribution, const double *low,
                           const double *high, const dk_noise_key *key, double *out,
                           unsigned long long *fail_world, void *stream);

/* DelayLine (randomization.py:27-62) for n worlds.  State (device): ring
 * [n, max_delay + 1, dim] of dtype, head / count / delay [n] int32.
 * reset: empties every line and draws its episode delay
 * Generator.integers(min_delay, max_delay + 1) from the world's stream.
 * push_pop: appends value [n, dim] and writes out [n, dim] = the value aged
 * d steps (d = episode delay, or a fresh per-step draw when per_step), the
 * oldest held value during warm-up. */
int dk_dr_delay_reset(int64_t n, int min_delay, int max_delay, const dk_noise_key *key,
                      int32_t *delay, int32_t *count, int32_t *head, void *stream);
int dk_dr_delay_push_pop(int dtype, int64_t n, int dim, int min_delay, int max_delay,
                         int per_step, void *ring, int32_t *head, int32_t *count,
                         const int32_t *delay, const dk_noise_key *key, const void *value,
                         void *out, void *stream);

/* pose_injection (randomization.py:188-199), in place on pose [n, dim];
 * bounds device double [dim, 2]; injected [n] u8 (may be NULL). */
int dk_dr_pose_injection(int dtype, int64_t n, int dim, void *pose, const double *bounds,
                         double prob, const dk_noise_key *key, uint8_t *injected, void *stream);

/* curriculum_update (randomization.py:224-238), in place on state [n,4] i64 =
 * (level, successes_at_level, episodes, total_successes). */
int dk_dr_curriculum(int64_t n, int64_t *state, const uint8_t *success, int64_t max_level,
                     int64_t promotion_threshold, void *stream);

/* ---------------------------------------------------------------------------
 * Rollout-side PPO math, device pointers, float64
 * arithmetic whatever the storage dtype (the reference converts to float64).
 *
 * compute_gae (ppo.py:80-102): rewards / values / dones [T, N], bootstrap [N]
 * -> advantages, returns (= advantages + values) [T, N]. */
/* ppo.policy_forward sampling (ppo.py:204-217) + tanh_gaussian_log_prob
 * (ppo.py:185-192), fused, float32: pre_tanh = mean + exp(log_std) * eps,
 * action = tanh(pre_tanh), log_prob [n] summed over the action dims;
 * log_std rows of log_std_stride (0 = one shared row); *nan_flag |= 1 if a mean
 * is NaN (the reference raises RuntimeError). */
int dk_ppo_sample(int64_t n, int action_dim, const float *mean, const float *log_std,
                  int64_t log_std_stride, const float *eps, float *pre_tanh, float *action,
                  float *log_prob, int *nan_flag, void *stream);
/* The per-step bookkeeping of ppo.collect_rollout (ppo.py:295-378) around the
 * policy call, the env step and the value call, float32 observations / float64
 * batch fields, each value computed as the reference's separate ops do.
 * dk_ppo_norm: a RunningNormalizer's device statistics for normalizer_apply
 * (mathcore.py:254-262: clip((x - mean) / sqrt(var + eps), -10, 10); copy = 1
 * while count == 0; present = 0: no normaliser, the identity). */
typedef struct {
    const double *mean, *var;
    double epsilon;
    int32_t copy, present;
} dk_ppo_norm;
/* obs_p [n, dp] / obs_v [n, dv] -> raw copies raw_p / raw_v (nullable), the
 * normalised policy input pol [n, dp], the normalised value input val [n, dv]
 * and its copy val2 (nullable; e.g. the first half of the value call's input). */
int dk_ppo_step_inputs(int64_t n, int dp, int dv, const float *obs_p, const float *obs_v,
                       const dk_ppo_norm *norm_p, const dk_ppo_norm *norm_v, float *raw_p,
                       float *raw_v, float *pol, float *val, float *val2, void *stream);
/* after the env step: boot = trunc & ~done & terminal_mask (the truncation
 * bootstrap, ppo.py:327-341), dones [n] = float64(done | trunc), and the boot
 * rows' normalised terminal observations compacted into val_term[0, *count)
 * (pos[i] = the row's slot, -1 for the other rows, whose bootstrap term is 0):
 * the value of the terminal observations is needed for those rows only. */
int dk_ppo_step_bootstrap(int64_t n, int dv, const uint8_t *done, const uint8_t *trunc,
                          const uint8_t *terminal_mask, const float *terminal_obs,
                          const dk_ppo_norm *norm_v, float *val_term, int64_t *count,
                          int32_t *pos, double *dones, void *stream);
/* the same without resetting *count: slots keep counting across the steps of a
 * phase (val_term holds the whole phase's terminal rows), for one value call
 * and dk_ppo_boot_fixup after the phase */
int dk_ppo_step_bootstrap_acc(int64_t n, int dv, const uint8_t *done, const uint8_t *trunc,
                              const uint8_t *terminal_mask, const float *terminal_obs,
                              const dk_ppo_norm *norm_v, float *val_term, int64_t *count,
                              int32_t *pos, double *dones, void *stream);
/* after the value calls (values [n] of the step's inputs, term_values[pos[i]]
 * of the compacted terminal rows): rewards_out = reward * reward_scaling +
 * discounting * (pos[i] >= 0 ? term_values[pos[i]] : 0), values_out =
 * float64(values) (values NULL: values_out not written -- the caller evaluates
 * the phase's values in one call after it), actions_out = float64(action)
 * [n, action_dim], and
 * reward_partial[dk_ppo_record_blocks(n)] = float64 reward sums per block.
 * term_values NULL: the boot rows' rewards_out = reward * reward_scaling, their
 * terminal values added by dk_ppo_boot_fixup after the phase. */
int64_t dk_ppo_record_blocks(int64_t n);
int dk_ppo_step_record(int64_t n, int action_dim, const float *reward, const int32_t *pos,
                       const float *values, const float *term_values, const float *action,
                       double reward_scaling, double discounting, double *rewards_out,
                       double *values_out, double *actions_out, double *reward_partial,
                       void *stream);
/* one launch after the env step of a phase whose values and terminal values are
 * evaluated after it: dk_ppo_step_bootstrap_acc + dk_ppo_step_record (values and
 * term_values NULL) for this step, and dk_ppo_step_inputs for the next step's
 * observations (next_obs_p NULL: the phase's last step) */
typedef struct {
    int64_t n;
    int32_t dp, dv, action_dim, reserved;
    /* this step: env outputs and the bootstrap / record buffers */
    const uint8_t *done, *trunc, *terminal_mask;
    const float *terminal_obs; /* [n, dv] the critic's terminal rows */
    float *val_term;           /* compacted boot rows, slots from *count on */
    int64_t *count;
    int32_t *pos;              /* [n] slot or -1 */
    double *dones;             /* [n] */
    const float *reward, *action;
    double reward_scaling, discounting;
    double *rewards_out, *actions_out, *reward_partial;
    /* the next step's inputs (dk_ppo_step_inputs), nullable */
    const float *next_obs_p, *next_obs_v;
    float *next_raw_p, *next_raw_v, *next_pol, *next_val;
} dk_ppo_post;
int dk_ppo_step_post(const dk_ppo_post *args, const dk_ppo_norm *norm_p,
                     const dk_ppo_norm *norm_v, void *stream);
/* rewards [tn] += discounting * term_values[pos[e]] where pos[e] >= 0 (pos [tn]:
 * the phase's dk_ppo_step_bootstrap_acc slots): the reward targets of the boot
 * rows, rounded as dk_ppo_step_record would */
int dk_ppo_boot_fixup(int64_t tn, const int32_t *pos, const float *term_values,
                      double discounting, double *rewards, void *stream);
int dk_ppo_gae(int dtype, int64_t num_steps, int64_t num_worlds, const void *rewards,
               const void *values, const void *dones, const void *bootstrap, double gamma,
               double lam, void *advantages, void *returns, void *stream);

/* normalizer_update (mathcore.py:234-251): merges batch [rows, dim] into the
 * running statistics mean / var (device float64 [dim], updated in place);
 * count is the statistics' count before the update (the caller adds rows). */
int dk_norm_update(int dtype, int64_t rows, int dim, const void *batch, double count,
                   double *mean, double *var, void *workspace, size_t workspace_bytes,
                   void *stream);
/* Device scratch dk_norm_update / dk_norm_colsum use for [rows, dim]; a
 * smaller (or NULL) workspace makes them allocate stream-ordered scratch. */
size_t dk_norm_workspace_bytes(int64_t rows, int dim);

/* The two halves of normalizer_update for data-parallel ranks: column sums
 * (or, with center [dim], sums of squared deviations) of the local batch in
 * float64 -- all-reduce them across ranks -- then the reference's merge of
 * the global batch mean / var (mathcore.py:245-251) into mean / var. */
int dk_norm_colsum(int dtype, int64_t rows, int dim, const void *batch, const double *center,
                   double *sums, void *workspace, size_t workspace_bytes, void *stream);
int dk_norm_merge(int dim, double count, double batch_count, const double *batch_mean,
                  const double *batch_var, double *mean, double *var, void *stream);

/* normalizer_apply (mathcore.py:254-265) or, with invert, normalizer_invert
 * (268-272) of batch [rows, dim] into out (same dtype); count == 0 copies. */
int dk_norm_apply(int dtype, int64_t rows, int dim, const void *batch, double count,
                  const double *mean, const double *var, double epsilon, int invert, void *out,
                  void *stream);

/* ---------------------------------------------------------------------------
 * Cartpole pixel observations: pixelrender.py's
 * rasteriser, brightness post-process, luma and 3-frame stack.
 * A frame is drawn from (cart x, cos th, sin th) -- the first three entries
 * of a cartpole state_obs row -- and 13 visual doubles per world: background,
 * cart and pole RGB, camera offset x / y, zoom, brightness. */
typedef struct dk_visual_bounds { /* VisualBounds, pixelrender.py:44-51 */
    double nominal[13];
    double color_jitter, camera_offset_range;
    double zoom_range[2], brightness_range[2];
} dk_visual_bounds;

/* batch_render (+ brightness_postprocess when brightness != 0): frames
 * [n, 3] (x, cos, sin) f64, visuals [n, 13] -> RGB out [n, h, w, 3] u8. */
int dk_pixels_render_rgb(int64_t n, int w, int h, double pole_length, const double *frames,
                         const double *visuals, int brightness, uint8_t *out, void *stream);

/* Per-world stack bookkeeping after a reset (first != 0) or a step: history
 * [n, 3, 3] f64 (three frames, oldest first), visuals [n, 13] f64, episode
 * [n] u32.  Worlds reset this step (reset_mask [n] u8, or all when first)
 * draw new visuals -- randomize_visuals from stream_rng(seed, env, episode, 0)
 * after skip_words sample_initial draws, or bounds->nominal -- and refill the
 * history with the new frame; the others shift it. */
int dk_pixels_advance(int dtype, int64_t n, int obs_dim, const void *obs,
                      const uint8_t *reset_mask, int first, double *history, double *visuals,
                      uint32_t *episode, int randomize, const dk_visual_bounds *bounds,
                      uint64_t seed, int64_t env_index_offset, int skip_words, void *stream);

/* The stacked grayscale observation [n, h, w, 3] (dtype) of the history. */
int dk_pixels_stack(int dtype, int64_t n, int w, int h, double pole_length,
                    const double *history, const double *visuals, void *out, void *stream);

/* Terminal stacks of autoreset worlds (mask [n] u8): [h1, h2, term_obs frame]
 * with the pre-reset visuals; call before dk_pixels_advance. */
int dk_pixels_terminal(int dtype, int64_t n, int w, int h, double pole_length, int obs_dim,
                       const void *term_obs, const uint8_t *mask, const double *history,
                       const double *visuals, void *out, void *stream);

/* ppo.pixel_normalize (ppo.py:232-238): per-sample, per-channel
 * standardisation of x [n, h, w, c] (in_dtype) into out (out_dtype), laid out
 * [n, h, w, c] or, with channels_first, [n, c, h, w]; stats: device float64
 * scratch [n, c, 2] (receives mean, std). */
int dk_pixels_normalize(int in_dtype, int out_dtype, int64_t n, int h, int w, int c,
                        const void *x, int channels_first, double *stats, void *out,
                        void *stream);

/* ------------------------------------------------------------------------
 * Articulated contact physics: SURVEY.md §8a rows G1-G4 (north_star
 * subsystems 2-5).  The reference has NO such code (SPEC.md:8 puts the
 * MJX/MuJoCo contact solver out of scope; PAPER.md:580 fixes feet-only
 * collision for the joystick tasks), so parity is against the repo's own
 * independent fp64 oracle (oracle/physics.c) and is labelled UNPINNED.
 *
 * The model is a Go1-shaped quadruped: a floating trunk (free joint: 7 qpos,
 * 6 qvel; linear velocity in the world frame, angular velocity in the trunk
 * frame, MuJoCo's convention) and DK_PHYS_LIMBS serial limbs of DK_PHYS_LJ
 * hinges (hip abduction, hip, knee), bodies aligned with their parent at q=0.
 * qpos = [trunk pos 3, trunk quat (w,x,y,z) 4, joints 12];
 * qvel = [trunk lin vel (world) 3, trunk ang vel (trunk frame) 3, joints 12].
 * Geoms (ids): 0 floor plane z=0, 1 trunk box, 2+2l thigh capsule of limb l
 * (body 1 origin -> body 2 origin), 3+2l foot sphere of limb l.  Contacts are
 * listed in geom order (box corners in corner order, capsule ends, foot).
 * Dynamics per step (timestep h): FK, composite-rigid-body mass matrix + armature + h*damping
 * (implicit joint damping), recursive Newton-Euler bias, position actuators
 * tau = clip(kp (ctrl - q) - kd qd, +-limit), soft constraints (MuJoCo-style:
 * solref (timeconst, dampratio), constant impedance solimp) for pyramidal
 * friction cones (4 edges per contact) and joint limits, a primal Newton
 * solver with exact line search, semi-implicit Euler (velocity first,
 * quaternion exponential map).  DESIGN.md §3 "Go1 physics" has the details.
 * ------------------------------------------------------------------------ */
#define DK_PHYS_LIMBS 4
#define DK_PHYS_LJ 3
#define DK_PHYS_NQ 19
#define DK_PHYS_NV 18
#define DK_PHYS_NU 12
#define DK_PHYS_NBODY 13
#define DK_PHYS_MAXCON 16 /* 4 box corners + 4 x (2 capsule ends + 1 foot) */
#define DK_PHYS_NSENSOR 46 /* framequat 4, gyro 3, velocimeter 3, jointpos 12, jointvel 12, foot pos 12 */

typedef struct dk_phys_model {
    double timestep;            /* physics step h (s) */
    double gravity[3];
    double friction;            /* pyramidal cone coefficient mu */
    double solref[2];           /* timeconst, dampratio */
    double solimp;              /* constant impedance in (0, 1) */
    double base_mass;
    double base_ipos[3];        /* trunk com in the trunk frame */
    double base_inertia[3];     /* principal inertia (trunk frame axes) */
    double base_box[3];         /* trunk box half sizes */
    double body_pos[4][3][3];   /* body origin in its parent's frame */
    double jnt_axis[4][3][3];   /* hinge axis (unit) in the body frame */
    double body_mass[4][3];
    double body_ipos[4][3][3];  /* com in the body frame */
    double body_inertia[4][3][3];
    double jnt_range[4][3][2];
    double dof_damping[4][3];
    double dof_armature[4][3];
    double torque_limit[4][3];
    double kp, kd;              /* position actuators */
    double foot_pos[4][3];      /* foot sphere centre in the last body's frame */
    double foot_radius;
    double thigh_radius;        /* capsule radius */
    int32_t iterations;         /* max Newton iterations */
    int32_t ls_iterations;      /* max line-search iterations */
    int32_t collide_box;        /* trunk box vs floor (0 = feet-only) */
    int32_t collide_thigh;      /* thigh capsules vs floor */
} dk_phys_model;

typedef struct dk_phys dk_phys;

/* Outputs of the LAST physics step of a dk_phys_step call (every pointer
 * nullable; device buffers in the handle's dtype unless int32). */
typedef struct dk_phys_diag {
    void *qacc;              /* [N, NV] constrained acceleration */
    void *qfrc_bias;         /* [N, NV] Coriolis/centrifugal + gravity */
    void *qfrc_constraint;   /* [N, NV] */
    void *act_force;         /* [N, NU] actuator torques */
    int32_t *ncon;           /* [N] */
    int32_t *contact_geom;   /* [N, MAXCON, 2] (0 = floor, geom id) */
    void *contact_dist;      /* [N, MAXCON] signed distance (< 0: penetration) */
    void *contact_pos;       /* [N, MAXCON, 3] world */
    void *contact_force;     /* [N, MAXCON, 3] normal, tangent x, tangent y */
    int32_t *solver_iter;    /* [N] Newton iterations used */
    void *sensordata;        /* [N, NSENSOR] of the post-step state */
} dk_phys_diag;

/* Go1-shaped defaults (Menagerie unitree_go1-like masses and offsets,
 * Playground Go1 joystick solver/actuator settings: h = 0.004, kp 35, kd 0.5). */
int dk_phys_default_model(dk_phys_model *model);
int dk_phys_create(const dk_phys_model *model, int dtype, int64_t num_worlds, int device,
                   dk_phys **out);
int dk_phys_destroy(dk_phys *phys);
/* device buffers, row-major [N, NQ] / [N, NV], handle dtype */
int dk_phys_set_state(dk_phys *phys, const void *qpos, const void *qvel, void *stream);
int dk_phys_get_state(dk_phys *phys, void *qpos, void *qvel, void *stream);
/* num_steps physics steps of every world with ctrl [N, NU] (joint position
 * targets) held; diag (nullable) receives the last step's outputs. */
int dk_phys_step(dk_phys *phys, int64_t num_steps, const void *ctrl, const dk_phys_diag *diag,
                 void *stream);
/* G1 inspection at the current state: M (mass matrix incl. armature, without
 * the implicit-damping term) [N, NV, NV], qfrc_bias [N, NV], body positions
 * xpos [N, NBODY, 3] and com positions xipos [N, NBODY, 3] (all nullable). */
int dk_phys_inspect(dk_phys *phys, void *mass_matrix, void *qfrc_bias, void *xpos, void *xipos,
                    void *stream);
/* Synchronising check of the sticky "matrix not positive definite" flag a
 * step sets for a non-finite state / control (DK_ERR_INVALID_INPUT). */
int dk_phys_check(dk_phys *phys);
int64_t dk_phys_kernel_launches(const dk_phys *phys);

/* ------------------------------------------------------------------------
 * Go1 joystick environment (north_star subsystem 6): the physics step above
 * with the locomotion tail (rows B1-B7) fused into the same kernel --
 * action -> PD targets (envkit.action_to_target, absolute), ctrl_dt/timestep
 * physics steps, foot kinematics, airtime / touchdown / advance_phase,
 * rewards.total_reward, build_locomotion_observation with Philox sensor
 * noise, termination (trunk upside down or below term_height), truncation,
 * Philox-keyed auto-reset.  No reference counterpart: UNPINNED.
 * Observations: state [N, 56], privileged_state [N, 75] (Go1 shape of
 * build_locomotion_observation); reward f[N]; done / trunc u8[N].
 * ------------------------------------------------------------------------ */
typedef struct dk_go1_config {
    int64_t episode_length;      /* control steps per episode */
    double ctrl_dt;              /* control period (s); physics steps = ctrl_dt / timestep */
    double action_scale;         /* PD target = q_default + action_scale * clip(a, -1, 1) */
    double gait_freq;            /* advance_phase frequency (Hz) */
    double term_height;          /* terminate below this trunk height (m) */
    double cmd_lo[3], cmd_hi[3]; /* joystick command ranges (vx, vy, yaw rate) */
    double joint_noise;          /* reset joint offsets U(-x, x) */
    double yaw_range;            /* reset heading U(-x, x) */
    double obs_noise[5];         /* ObservationNoise: gravity, lin_vel, ang_vel, joint_pos, joint_vel */
    uint64_t seed;
    dk_reward_config reward;
    /* domain randomisation drawn per world at every reset (randomization.py:156-181
     * additive / multiplicative kinds): foot friction U(lo, hi), trunk payload
     * U(lo, hi) kg added to the trunk mass, PD stiffness scale U(lo, hi) x kp;
     * lo == hi fixes the value */
    double dr_friction[2], dr_payload[2], dr_kp_scale[2];
} dk_go1_config;

typedef struct dk_go1_env dk_go1_env;

int dk_go1_default_config(dk_go1_config *cfg);
int dk_go1_create(const dk_phys_model *model, const dk_go1_config *cfg, int dtype,
                  int64_t num_worlds, int64_t env_index_offset, int device, dk_go1_env **out);
int dk_go1_destroy(dk_go1_env *env);
/* reset every world (episode 0; has_seed: replace the config seed); obs [N,56],
 * priv [N,75] (nullable) device buffers */
int dk_go1_reset(dk_go1_env *env, int has_seed, uint64_t seed, void *obs, void *priv,
                 void *stream);
/* K control steps; actions [K,N,12]; obs [K,N,56]; priv [K,N,75] | NULL; reward [K,N];
 * done / trunc u8 [K,N]; terms [K,N,16] | NULL; terminal_obs [K,N,56] | NULL;
 * terminal_mask u8 [K,N] | NULL (device buffers, handle dtype) */
int dk_go1_step(dk_go1_env *env, int64_t num_steps, const void *actions, void *obs, void *priv,
                void *reward, uint8_t *done, uint8_t *trunc, void *terms, void *terminal_obs,
                uint8_t *terminal_mask, void *stream);
/* the same with the auto-reset worlds' terminal PRIVILEGED rows too
 * (terminal_priv [K, N, 75], nullable: the clean last observation of an episode
 * for an asymmetric critic's truncation bootstrap) */
int dk_go1_step_ex(dk_go1_env *env, int64_t num_steps, const void *actions, void *obs,
                   void *priv, void *reward, uint8_t *done, uint8_t *trunc, void *terms,
                   void *terminal_obs, void *terminal_priv, uint8_t *terminal_mask,
                   void *stream);
/* state as row-major device buffers (each nullable): qpos [N,19], qvel [N,18],
 * command [N,3], phase [N,4], airtime [N,4], last_contact u8 [N,4],
 * prev_action [N,12], steps i32 [N], episode u32 [N] */
int dk_go1_get_state(dk_go1_env *env, void *qpos, void *qvel, void *command, void *phase,
                     void *airtime, uint8_t *last_contact, void *prev_action, int32_t *steps,
                     uint32_t *episode, void *stream);
/* synchronising error check: non-finite actions (DK_ERR_INVALID_INPUT, with
 * the first step / world), non-positive-definite physics matrices */
int dk_go1_check(dk_go1_env *env, int64_t *step_index, int64_t *env_index);
/* the worlds' current physical parameters [N, 3]: friction, trunk mass, kp */
int dk_go1_get_params(dk_go1_env *env, void *params, void *stream);
int64_t dk_go1_kernel_launches(const dk_go1_env *env);

/* ------------------------------------------------------------------------
 * PPO networks on the tensor cores (ppo.py:109-141
 * _mlp / MLPPolicy / MLPValue): y = W_out silu(... silu(W_0 x + b_0) ...) + b_out.
 * Layer 0 (d_in <= 16) and the output layer (n_out <= 4) run in float32 on the
 * CUDA cores; the n_tc hidden x hidden layers (hidden 128 or 256) on tcgen05
 * tensor cores with a BF16x3 split and float32 accumulation.  Weights are
 * float32 torch Linear layouts [out, in]; hidden weights pre-packed by
 * dk_mlp_pack (bf16 hi / lo, hidden*hidden elements each per layer).
 * ------------------------------------------------------------------------ */
typedef struct dk_mlp {
    int32_t d_in, hidden, n_tc, n_out;
    const float *w0, *b0;        /* [hidden, d_in], [hidden] */
    const void *w_hi, *w_lo;     /* packed [n_tc][hidden * hidden] bf16 */
    const float *b_hidden;       /* [n_tc][hidden] */
    const float *w_out, *b_out;  /* [n_out, hidden], [n_out] */
    const void *w0_hi, *w0_lo;   /* d_in > 16: layer 0 packed [hidden * K0] bf16, K0 = d_in
                                    rounded up to 32 (zero columns), on the tensor cores */
} dk_mlp;

int dk_mlp_pack(const float *w, int n, int k, void *w_hi, void *w_lo, void *stream);
int dk_mlp_forward(const dk_mlp *net, int64_t rows, const float *x, int64_t x_stride, float *y,
                   int64_t y_stride, void *stream);
/* developer hook: desc_swap = 1 swaps the descriptors' LBO / SBO (layout check) */
/* two networks in one launch (their row tiles share the GPU: e.g. the PPO
 * policy and value on the same observations), each as dk_mlp_forward. */
int dk_mlp_forward_pair(const dk_mlp *net0, int64_t rows0, const float *x0, int64_t x0_stride,
                        float *y0, int64_t y0_stride, const dk_mlp *net1, int64_t rows1,
                        const float *x1, int64_t x1_stride, float *y1, int64_t y1_stride,
                        void *stream);
/* the same forward with the row count read on the device (*rows_dev <=
 * max_rows; e.g. a count produced by an earlier kernel on the stream). */
int dk_mlp_forward_count(const dk_mlp *net, int64_t max_rows, const int64_t *rows_dev,
                         const float *x, int64_t x_stride, float *y, int64_t y_stride,
                         void *stream);
int dk_mlp_forward_dbg(const dk_mlp *net, int64_t rows, const float *x, int64_t x_stride,
                       float *y, int64_t y_stride, int desc_swap, void *stream);

/* Benchmark/timing helper (no reference counterpart): enqueue on `stream` a
 * one-thread kernel that waits until *host_flag (pinned host memory) becomes
 * non-zero, or max_spins polls have elapsed (0 = no limit).  Lets a caller
 * queue a timed region behind it and release it once the whole region is
 * submitted. */
int dk_stream_gate(const int32_t *host_flag, int64_t max_spins, void *stream);

int dk_abi_version(void);
const char *dk_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* DESKRL_B200_H */
