// capi_go1.cu -- extern "C" entry points of the fused Go1 joystick env
// (include/deskrl_b200.h "Go1 joystick environment"; go1env.cuh).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <type_traits>
#include <vector>

#include "../../include/deskrl_b200.h"
#include "go1env.cuh"

namespace dk {
namespace go1 {
DK_GO1_DECLARE(float)
DK_GO1_DECLARE(double)
}  // namespace go1
namespace phys {
DK_PHYS_DECLARE(float)
DK_PHYS_DECLARE(double)
}  // namespace phys
}  // namespace dk

extern "C" int dk_internal_fail(int code, const char *msg);  // capi.cu

struct dk_go1_env {
    dk_phys_model model;
    dk_go1_config cfg;
    int dtype = DK_F32, device = 0;
    int64_t n = 0, env0 = 0;
    void *qpos = nullptr, *qvel = nullptr, *cmd = nullptr, *phase = nullptr, *air = nullptr,
         *prev = nullptr, *dr = nullptr;
    uint8_t *lastc = nullptr;
    int32_t *steps = nullptr;
    uint32_t *episode = nullptr;
    unsigned long long *err = nullptr;
    int32_t *bad = nullptr;
    int64_t launches = 0;
    bool was_reset = false;
};

namespace {

int cuda_rc(cudaError_t e, const char *what) {
    if (e == cudaSuccess) return DK_OK;
    char buf[256];
    snprintf(buf, sizeof(buf), "%s: %s", what, cudaGetErrorString(e));
    return dk_internal_fail(DK_ERR_CUDA, buf);
}

struct Guard {
    int prev = -1;
    explicit Guard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~Guard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

const double kHome[12] = {0, 0.9, -1.8, 0, 0.9, -1.8, 0, 0.9, -1.8, 0, 0.9, -1.8};
const double kPhase0[4] = {0.0, 3.141592653589793, 3.141592653589793, 0.0};  // trot

template <typename T>
dk::phys::PhysConst<T> phys_const(const dk_phys_model &m) {
    dk::phys::PhysConst<T> c;
    memset(&c, 0, sizeof(c));
    c.h = (T)m.timestep;
    for (int i = 0; i < 3; ++i) {
        c.g[i] = (T)m.gravity[i];
        c.base_ipos[i] = (T)m.base_ipos[i];
        c.base_inertia[i] = (T)m.base_inertia[i];
        c.base_box[i] = (T)m.base_box[i];
    }
    c.mu = (T)m.friction;
    const double imp = m.solimp, tc = m.solref[0], dr = m.solref[1];
    c.imp = (T)imp;
    c.kstiff = (T)(1.0 / (imp * imp * tc * tc * dr * dr));
    c.bdamp = (T)(2.0 / (imp * tc));
    c.rscale = (T)((1.0 - imp) / imp);
    c.base_mass = (T)m.base_mass;
    c.kp = (T)m.kp;
    c.kd = (T)m.kd;
    c.foot_radius = (T)m.foot_radius;
    c.thigh_radius = (T)m.thigh_radius;
    c.iterations = m.iterations;
    c.ls_iterations = m.ls_iterations;
    c.collide_box = m.collide_box != 0;
    c.collide_thigh = m.collide_thigh != 0;
    c.rows_per_lane = 4 * c.collide_box + 4 * (2 * c.collide_thigh + 1) + 3;
    for (int l = 0; l < 4; ++l) {
        auto &L = c.limb[l];
        for (int j = 0; j < 3; ++j) {
            for (int i = 0; i < 3; ++i) {
                L.body_pos[j][i] = (T)m.body_pos[l][j][i];
                L.axis[j][i] = (T)m.jnt_axis[l][j][i];
                L.ipos[j][i] = (T)m.body_ipos[l][j][i];
                L.inertia[j][i] = (T)m.body_inertia[l][j][i];
            }
            L.mass[j] = (T)m.body_mass[l][j];
            L.range[j][0] = (T)m.jnt_range[l][j][0];
            L.range[j][1] = (T)m.jnt_range[l][j][1];
            L.damping[j] = (T)m.dof_damping[l][j];
            L.armature[j] = (T)m.dof_armature[l][j];
            L.tlim[j] = (T)m.torque_limit[l][j];
        }
        for (int i = 0; i < 3; ++i) L.foot_pos[i] = (T)m.foot_pos[l][i];
    }
    return c;
}

template <typename T>
dk::go1::EnvConst<T> env_const(const dk_go1_env *e) {
    dk::go1::EnvConst<T> c;
    memset(&c, 0, sizeof(c));
    const dk_go1_config &g = e->cfg;
    c.substeps = (int)std::lround(g.ctrl_dt / e->model.timestep);
    c.episode_length = g.episode_length;
    c.seed = g.seed;
    c.env0 = e->env0;
    c.ctrl_dt = (T)g.ctrl_dt;
    c.action_scale = (T)g.action_scale;
    c.gait_freq = (T)g.gait_freq;
    c.term_height = (T)g.term_height;
    c.home_height = (T)0.278;
    for (int j = 0; j < 12; ++j) c.q_default[j] = (T)kHome[j];
    for (int f = 0; f < 4; ++f) c.phase0[f] = (T)kPhase0[f];
    for (int k = 0; k < 3; ++k) {
        c.cmd_lo[k] = g.cmd_lo[k];
        c.cmd_hi[k] = g.cmd_hi[k];
    }
    c.joint_noise = g.joint_noise;
    c.yaw_range = g.yaw_range;
    for (int k = 0; k < 2; ++k) {
        (k == 0 ? c.dr_lo : c.dr_hi)[0] = g.dr_friction[k];
        (k == 0 ? c.dr_lo : c.dr_hi)[1] = g.dr_payload[k];
        (k == 0 ? c.dr_lo : c.dr_hi)[2] = g.dr_kp_scale[k];
    }
    c.has_noise = 0;
    for (int k = 0; k < 5; ++k) {
        c.noise[k] = g.obs_noise[k];
        if (g.obs_noise[k] > 0) c.has_noise = 1;
    }
    const dk_reward_config &r = g.reward;
    const double w[16] = {r.w_lin_vel, r.w_ang_vel, r.w_airtime, r.w_clearance, r.w_phase,
                          r.w_slip, r.w_orientation, r.w_torque, r.w_joint_pos,
                          r.w_action_rate, r.w_energy, r.w_pose, r.w_termination,
                          r.w_standstill, r.w_lin_vel_z, r.w_ang_vel_xy};
    for (int k = 0; k < 16; ++k) c.rc.w[k] = (T)w[k];
    c.rc.sigma_lin = (T)r.sigma_lin_vel;
    c.rc.sigma_ang = (T)r.sigma_ang_vel;
    c.rc.airtime_min = (T)r.airtime_min;
    c.rc.airtime_max = (T)r.airtime_max;
    c.rc.sigma_phase = (T)r.sigma_phase;
    c.rc.swing_height = (T)r.swing_height;
    c.rc.gated = r.standstill_gated != 0;
    return c;
}

template <typename T>
int launch(dk_go1_env *e, dk::go1::EnvIO<T> io, cudaStream_t st) {
    dk::go1::EnvState<T> s;
    s.qpos = (T *)e->qpos;
    s.qvel = (T *)e->qvel;
    s.cmd = (T *)e->cmd;
    s.phase = (T *)e->phase;
    s.air = (T *)e->air;
    s.prev_action = (T *)e->prev;
    s.dr = (T *)e->dr;
    s.last_contact = e->lastc;
    s.steps = e->steps;
    s.episode = e->episode;
    io.n = e->n;
    io.err = e->err;
    io.bad = e->bad;
    e->launches += 1;
    return cuda_rc(dk::go1::launch_env<T>(phys_const<T>(e->model), env_const<T>(e), s, io, st),
                   "go1_env_kernel");
}

template <typename T>
cudaError_t rows_out(const void *soa, void *rows, int64_t n, int width, cudaStream_t st) {
    return dk::phys::launch_transpose<T>((const T *)soa, (T *)rows, n, width, false, st);
}

}  // namespace

extern "C" {

int dk_go1_default_config(dk_go1_config *c) {
    if (!c) return dk_internal_fail(DK_ERR_INVALID_INPUT, "null config");
    memset(c, 0, sizeof(*c));
    c->episode_length = 1000;
    c->ctrl_dt = 0.02;
    c->action_scale = 0.5;
    c->gait_freq = 1.5;
    c->term_height = 0.12;
    const double lo[3] = {-1.5, -0.8, -1.2}, hi[3] = {1.5, 0.8, 1.2};
    for (int k = 0; k < 3; ++k) {
        c->cmd_lo[k] = lo[k];
        c->cmd_hi[k] = hi[k];
    }
    c->joint_noise = 0.1;
    c->yaw_range = 3.141592653589793;
    const double nz[5] = {0.05, 0.1, 0.2, 0.01, 1.5};  // ObservationNoise defaults
    for (int k = 0; k < 5; ++k) c->obs_noise[k] = nz[k];
    c->seed = 0;
    c->dr_friction[0] = 0.4;  // Playground-like Go1 randomisation ranges
    c->dr_friction[1] = 1.0;
    c->dr_payload[0] = -0.5;
    c->dr_payload[1] = 1.5;
    c->dr_kp_scale[0] = 0.9;
    c->dr_kp_scale[1] = 1.1;
    dk_reward_config &r = c->reward;  // RewardTermConfig defaults (rewards.py:51-75)
    r.w_lin_vel = 1.0; r.sigma_lin_vel = 0.25; r.w_ang_vel = 0.5; r.sigma_ang_vel = 0.25;
    r.w_airtime = 1.0; r.airtime_min = 0.1; r.airtime_max = 0.5; r.w_clearance = -1.0;
    r.w_phase = 1.0; r.sigma_phase = 0.001; r.swing_height = 0.08; r.w_slip = -0.1;
    r.w_orientation = -1.0; r.w_torque = -1e-4; r.w_joint_pos = -0.1; r.w_action_rate = -0.01;
    r.w_energy = -1e-3; r.w_pose = 0.5; r.w_termination = -1.0; r.w_standstill = -0.1;
    r.w_lin_vel_z = -0.5; r.w_ang_vel_xy = -0.05; r.standstill_gated = 0;
    return DK_OK;
}

int dk_go1_create(const dk_phys_model *model, const dk_go1_config *cfg, int dtype, int64_t n,
                  int64_t env0, int device, dk_go1_env **out) {
    if (!model || !cfg || !out) return dk_internal_fail(DK_ERR_INVALID_INPUT, "null argument");
    *out = nullptr;
    if (dtype != DK_F32 && dtype != DK_F64)
        return dk_internal_fail(DK_ERR_CONFIG, "dtype must be DK_F32 or DK_F64");
    if (n < 1) return dk_internal_fail(DK_ERR_CONFIG, "num_worlds must be >= 1");
    if (cfg->episode_length < 1 || cfg->episode_length >= (1LL << 31))
        return dk_internal_fail(DK_ERR_CONFIG, "episode_length must be in [1, 2^31)");
    const double ratio = cfg->ctrl_dt / model->timestep;
    if (!(ratio >= 0.5) || std::fabs(ratio - std::lround(ratio)) > 1e-9)
        return dk_internal_fail(DK_ERR_CONFIG, "ctrl_dt must be a positive multiple of timestep");
    if (!(model->timestep > 0) || model->iterations < 1 || model->ls_iterations < 1 ||
        !(model->solimp > 0 && model->solimp < 1))
        return dk_internal_fail(DK_ERR_CONFIG, "invalid physics model");
    for (int k = 0; k < 3; ++k)
        if (!(cfg->cmd_lo[k] <= cfg->cmd_hi[k]))
            return dk_internal_fail(DK_ERR_CONFIG, "command range lower > upper");
    if (!(cfg->dr_friction[0] <= cfg->dr_friction[1] && cfg->dr_friction[0] >= 0 &&
          cfg->dr_payload[0] <= cfg->dr_payload[1] &&
          model->base_mass + cfg->dr_payload[0] > 0 && cfg->dr_kp_scale[0] <= cfg->dr_kp_scale[1] &&
          cfg->dr_kp_scale[0] >= 0))
        return dk_internal_fail(DK_ERR_CONFIG, "invalid domain randomisation range");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev)
        return dk_internal_fail(DK_ERR_CUDA, "no such CUDA device");
    Guard g(device);
    dk_go1_env *e = new dk_go1_env;
    e->model = *model;
    e->cfg = *cfg;
    e->dtype = dtype;
    e->device = device;
    e->n = n;
    e->env0 = env0;
    const size_t es = dtype == DK_F64 ? 8 : 4;
    cudaError_t r = cudaSuccess;
    auto alloc = [&](void **p, size_t bytes) {
        if (r == cudaSuccess) r = cudaMalloc(p, bytes);
        if (r == cudaSuccess) r = cudaMemset(*p, 0, bytes);
    };
    alloc(&e->qpos, es * DK_PHYS_NQ * n);
    alloc(&e->qvel, es * DK_PHYS_NV * n);
    alloc(&e->cmd, es * 3 * n);
    alloc(&e->phase, es * 4 * n);
    alloc(&e->air, es * 4 * n);
    alloc(&e->prev, es * 12 * n);
    alloc(&e->dr, es * 3 * n);
    alloc((void **)&e->lastc, 4 * n);
    alloc((void **)&e->steps, 4 * n);
    alloc((void **)&e->episode, 4 * n);
    alloc((void **)&e->err, sizeof(unsigned long long));
    alloc((void **)&e->bad, sizeof(int32_t));
    if (r == cudaSuccess) r = cudaMemset(e->err, 0xff, sizeof(unsigned long long));
    if (r != cudaSuccess) {
        dk_go1_destroy(e);
        return cuda_rc(r, "dk_go1_create");
    }
    *out = e;
    return DK_OK;
}

int dk_go1_destroy(dk_go1_env *e) {
    if (!e) return DK_OK;
    Guard g(e->device);
    for (void *p : {e->qpos, e->qvel, e->cmd, e->phase, e->air, e->prev, e->dr, (void *)e->lastc,
                    (void *)e->steps, (void *)e->episode, (void *)e->err, (void *)e->bad})
        cudaFree(p);
    delete e;
    return DK_OK;
}

int dk_go1_reset(dk_go1_env *e, int has_seed, uint64_t seed, void *obs, void *priv, void *stream) {
    if (!e) return dk_internal_fail(DK_ERR_INVALID_INPUT, "null handle");
    if (!obs) return dk_internal_fail(DK_ERR_INVALID_INPUT, "null obs");
    if (has_seed) e->cfg.seed = seed;
    Guard g(e->device);
    e->was_reset = true;
    if (e->dtype == DK_F64) {
        dk::go1::EnvIO<double> io{};
        io.reset_all = 1;
        io.obs = (double *)obs;
        io.priv = (double *)priv;
        return launch<double>(e, io, (cudaStream_t)stream);
    }
    dk::go1::EnvIO<float> io{};
    io.reset_all = 1;
    io.obs = (float *)obs;
    io.priv = (float *)priv;
    return launch<float>(e, io, (cudaStream_t)stream);
}

int dk_go1_step(dk_go1_env *e, int64_t K, const void *actions, void *obs, void *priv,
                void *reward, uint8_t *done, uint8_t *trunc, void *terms, void *terminal_obs,
                uint8_t *terminal_mask, void *stream) {
    return dk_go1_step_ex(e, K, actions, obs, priv, reward, done, trunc, terms, terminal_obs,
                          nullptr, terminal_mask, stream);
}

int dk_go1_step_ex(dk_go1_env *e, int64_t K, const void *actions, void *obs, void *priv,
                   void *reward, uint8_t *done, uint8_t *trunc, void *terms, void *terminal_obs,
                   void *terminal_priv, uint8_t *terminal_mask, void *stream) {
    if (!e) return dk_internal_fail(DK_ERR_INVALID_INPUT, "null handle");
    if (!e->was_reset) return dk_internal_fail(DK_ERR_USAGE, "call reset() before step()");
    if (K < 0) return dk_internal_fail(DK_ERR_INVALID_INPUT, "num_steps must be >= 0");
    if (K == 0) return DK_OK;
    if (!actions || !obs || !reward || !done || !trunc)
        return dk_internal_fail(DK_ERR_INVALID_INPUT, "null output buffer");
    Guard g(e->device);
    auto fill = [&](auto &io) {
        using T = std::remove_pointer_t<decltype(io.obs)>;
        io.K = K;
        io.actions = (const T *)actions;
        io.obs = (T *)obs;
        io.priv = (T *)priv;
        io.reward = (T *)reward;
        io.done = done;
        io.trunc = trunc;
        io.terms = (T *)terms;
        io.terminal_obs = (T *)terminal_obs;
        io.terminal_priv = (T *)terminal_priv;
        io.terminal_mask = terminal_mask;
    };
    if (e->dtype == DK_F64) {
        dk::go1::EnvIO<double> io{};
        fill(io);
        return launch<double>(e, io, (cudaStream_t)stream);
    }
    dk::go1::EnvIO<float> io{};
    fill(io);
    return launch<float>(e, io, (cudaStream_t)stream);
}

int dk_go1_get_state(dk_go1_env *e, void *qpos, void *qvel, void *command, void *phase,
                     void *airtime, uint8_t *last_contact, void *prev_action, int32_t *steps,
                     uint32_t *episode, void *stream) {
    if (!e) return dk_internal_fail(DK_ERR_INVALID_INPUT, "null handle");
    Guard g(e->device);
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t r = cudaSuccess;
    const int64_t n = e->n;
    auto T2 = [&](const void *src, void *dst, int width) {
        if (!dst || r != cudaSuccess) return;
        r = e->dtype == DK_F64 ? rows_out<double>(src, dst, n, width, st)
                               : rows_out<float>(src, dst, n, width, st);
    };
    T2(e->qpos, qpos, DK_PHYS_NQ);
    T2(e->qvel, qvel, DK_PHYS_NV);
    T2(e->cmd, command, 3);
    T2(e->phase, phase, 4);
    T2(e->air, airtime, 4);
    T2(e->prev, prev_action, 12);
    if (last_contact && r == cudaSuccess) {
        // u8 SoA [4][n] -> rows [n][4] on the host (small)
        std::vector<uint8_t> h(4 * n), o(4 * n);
        r = cudaMemcpyAsync(h.data(), e->lastc, 4 * n, cudaMemcpyDeviceToHost, st);
        if (r == cudaSuccess) r = cudaStreamSynchronize(st);
        for (int64_t i = 0; i < n; ++i)
            for (int f = 0; f < 4; ++f) o[4 * i + f] = h[f * n + i];
        if (r == cudaSuccess)
            r = cudaMemcpyAsync(last_contact, o.data(), 4 * n, cudaMemcpyHostToDevice, st);
        if (r == cudaSuccess) r = cudaStreamSynchronize(st);
    }
    if (steps && r == cudaSuccess)
        r = cudaMemcpyAsync(steps, e->steps, 4 * n, cudaMemcpyDeviceToDevice, st);
    if (episode && r == cudaSuccess)
        r = cudaMemcpyAsync(episode, e->episode, 4 * n, cudaMemcpyDeviceToDevice, st);
    return cuda_rc(r, "dk_go1_get_state");
}

int dk_go1_check(dk_go1_env *e, int64_t *step_index, int64_t *env_index) {
    if (!e) return dk_internal_fail(DK_ERR_INVALID_INPUT, "null handle");
    Guard g(e->device);
    unsigned long long err = 0;
    int32_t bad = 0;
    cudaError_t r = cudaMemcpy(&err, e->err, sizeof(err), cudaMemcpyDeviceToHost);
    if (r == cudaSuccess) r = cudaMemcpy(&bad, e->bad, sizeof(bad), cudaMemcpyDeviceToHost);
    if (r != cudaSuccess) return cuda_rc(r, "dk_go1_check");
    if (err != ~0ull) {
        if (step_index) *step_index = (int64_t)(err / (unsigned long long)e->n);
        if (env_index) *env_index = (int64_t)(err % (unsigned long long)e->n);
        cudaMemset(e->err, 0xff, sizeof(unsigned long long));
        return dk_internal_fail(DK_ERR_INVALID_INPUT, "action contains non-finite values");
    }
    if (bad) {
        cudaMemset(e->bad, 0, sizeof(int32_t));
        return dk_internal_fail(DK_ERR_INVALID_INPUT,
                                "physics step: mass or Hessian matrix not positive definite");
    }
    return DK_OK;
}

int dk_go1_get_params(dk_go1_env *e, void *params, void *stream) {
    if (!e || !params) return dk_internal_fail(DK_ERR_INVALID_INPUT, "null argument");
    Guard g(e->device);
    cudaStream_t st = (cudaStream_t)stream;
    return cuda_rc(e->dtype == DK_F64 ? rows_out<double>(e->dr, params, e->n, 3, st)
                                      : rows_out<float>(e->dr, params, e->n, 3, st),
                   "dk_go1_get_params");
}

int64_t dk_go1_kernel_launches(const dk_go1_env *e) { return e ? e->launches : 0; }

}  // extern "C"
