// go1env.cuh -- the Go1 joystick environment step, fused (north_star
// subsystem 6: reward, observation, termination, auto-reset and domain
// randomisation in the step kernel's tail, one HBM round trip per control step).
//
// One launch advances every world K control steps.  Per control step and
// world (one lane quad, lane = limb, as in physics.cuh):
//   action -> PD targets      envkit.action_to_target, absolute mode (envkit.py:111-131)
//   `substeps` physics steps  physics.cuh phys_step (PD torque clip = envkit.pd_torque)
//   foot kinematics           foot height / velocity, contact = sphere below the floor
//   gait bookkeeping          airtime, touchdown, advance_phase (mathcore.py:143-171),
//                             swing_height_profile (rewards.py:92-94)
//   reward                    rewards.total_reward, 16 terms (rewards.py:97-211)
//   observation               envkit.build_locomotion_observation with Philox-keyed
//                             uniform sensor noise (envkit.py:147-193; randomization
//                             B7 sensor noise)
//   termination / truncation  upside-down trunk or trunk below term_height; episode_length
//   auto-reset                Philox-keyed reset draw (stream_rng(seed, env, episode, 0),
//                             envkit.py:41-49), terminal observation kept
// The frame of the reward/observation row is assembled in shared memory by the
// four lanes, the four lanes evaluate the reward and observation row together
// (loco_row's math, locomotion.cuh, split by joint / foot and quad-reduced) and
// draw the sensor noise together (each lane its Philox blocks), and the CTA
// stores its 32 worlds' contiguous output rows cooperatively.  The reference has no Go1 env: the physics is
// checked against oracle/physics.c, the tail against oracle/locomotion.c, and
// the glue against oracle/go1env.py (tests/test_gpu_go1env.py) -- UNPINNED.
#pragma once
#include "locomotion.cuh"
#include "physics.cuh"

namespace dk {
namespace go1 {

using phys::Lane;
using phys::PhysConst;
using phys::Rows;

constexpr int NJ = 12, NF = 4;
constexpr int S = 9 + 3 * NJ + 3 + 2 * NF;  // 56: state slot
constexpr int P = S + NF + NJ + 3;          // 75: privileged slot
constexpr int FR = 112;                     // frame scratch per world (T)

template <typename T>
struct EnvConst {
    int substeps;
    int has_noise;
    int64_t episode_length;
    uint64_t seed;
    int64_t env0;
    T ctrl_dt, action_scale, gait_freq, term_height, home_height;
    T q_default[NJ];
    T phase0[NF];
    double cmd_lo[3], cmd_hi[3], joint_noise, yaw_range;
    double dr_lo[3], dr_hi[3];  // domain randomisation: friction, payload (kg), kp scale
    double noise[5];
    RewardCfg<T> rc;
};

template <typename T>
struct EnvState {  // structure of arrays, [field][n]
    T *qpos, *qvel, *cmd, *phase, *air, *prev_action;
    T *dr;  // [3][n]: friction, trunk mass, kp of the world's current episode
    uint8_t *last_contact;
    int32_t *steps;
    uint32_t *episode;
};

template <typename T>
struct EnvIO {
    int64_t n, K;
    int reset_all;          // 1: reset every world (episode = 0) and write its obs (K ignored)
    const T *actions;       // [K][n][12]
    T *obs, *priv;          // [K][n][56] / [K][n][75] (priv nullable)
    T *reward;              // [K][n]
    uint8_t *done, *trunc;  // [K][n]
    T *terms;               // [K][n][16] nullable
    T *terminal_obs;        // [K][n][56] nullable (rows of auto-reset worlds)
    T *terminal_priv;       // [K][n][75] nullable: their privileged rows (asymmetric critics)
    uint8_t *terminal_mask; // [K][n] nullable
    unsigned long long *err;  // first (step * n + world) with a non-finite action
    int32_t *bad;             // set when a physics factorisation broke down
};

// frame scratch offsets (T units)
enum {
    O_Q = 0, O_LIN = 4, O_ANG = 7, O_CMD = 10, O_JPOS = 13, O_JVEL = 25, O_JTAU = 37,
    O_ACT = 49, O_FPA = 61, O_AIR = 73, O_FH = 77, O_FHD = 81, O_FVEL = 85, O_PHASE = 93,
    O_FLAGS = 97  // 8 bytes: touchdown[4], contact[4] (as raw bytes)
};

// foot position and world velocity of the lane's limb (point on the last body)
template <typename T>
__device__ __forceinline__ void foot_kin(const PhysConst<T> &P, const Lane<T> &L, int l, T *fpos,
                                         T *fvel) {
    const auto &lm = P.limb[l];
    T R0[9];
    phys::quat2mat(L.quat, R0);
    T w[3];
    phys::mat_vec3(R0, L.wb, w);
    T vel[6] = {w[0], w[1], w[2], L.vlin[0], L.vlin[1], L.vlin[2]};
    T Rp[9], pp[3];
#pragma unroll
    for (int i = 0; i < 9; ++i) Rp[i] = R0[i];
#pragma unroll
    for (int i = 0; i < 3; ++i) pp[i] = L.pos[i];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        T off[3], a[3], Rq[9], Rj[9], rel[3], lin[3];
        phys::mat_vec3(Rp, lm.body_pos[j], off);
#pragma unroll
        for (int i = 0; i < 3; ++i) pp[i] = pp[i] + off[i];
        phys::mat_vec3(Rp, lm.axis[j], a);
        phys::axis_rot(lm.axis[j], L.q[j], Rq);
        phys::mat_mul3(Rp, Rq, Rj);
#pragma unroll
        for (int i = 0; i < 9; ++i) Rp[i] = Rj[i];
#pragma unroll
        for (int i = 0; i < 3; ++i) rel[i] = L.pos[i] - pp[i];
        phys::cross3(a, rel, lin);
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            vel[i] = vel[i] + a[i] * L.qd[j];
            vel[3 + i] = vel[3 + i] + lin[i] * L.qd[j];
        }
    }
    T foff[3];
    phys::mat_vec3(Rp, lm.foot_pos, foff);
#pragma unroll
    for (int i = 0; i < 3; ++i) fpos[i] = pp[i] + foff[i];
    T r[3], wr[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) r[i] = fpos[i] - L.pos[i];
    phys::cross3(vel, r, wr);
#pragma unroll
    for (int i = 0; i < 3; ++i) fvel[i] = vel[3 + i] + wr[i];
}

// per-world reset draw from stream_rng(seed, env, episode, 0): yaw, the 12
// joint offsets, the 3 command components, then the episode's physical
// parameters (friction, payload, kp scale) -- Generator.uniform order; the
// parameters follow randomization.randomize_params' additive / multiplicative
// kinds (randomization.py:156-181)
template <typename T>
__device__ __noinline__ void reset_world(const PhysConst<T> &P, const EnvConst<T> &E, Lane<T> &L, int l,
                            uint64_t env, uint32_t episode, T *cmd, T &phase, T &air,
                            T *prev_action) {
    Philox4x64 rng;
    rng.init(E.seed, env, episode, 0);
    // 19 draws in Generator.uniform order: yaw, 12 joint offsets, 3 commands,
    // 3 physical parameters (one rolled loop: a single copy of the Philox code)
    double u[19];
#pragma unroll 1
    for (int i = 0; i < 19; ++i) {
        double lo, hi;
        if (i == 0) {
            lo = -E.yaw_range; hi = E.yaw_range;
        } else if (i < 13) {
            lo = -E.joint_noise; hi = E.joint_noise;
        } else if (i < 16) {
            lo = E.cmd_lo[i - 13]; hi = E.cmd_hi[i - 13];
        } else {
            lo = E.dr_lo[i - 16]; hi = E.dr_hi[i - 16];
        }
        u[i] = rng.uniform(lo, hi);
    }
    L.mu = (T)u[16];
    L.base_mass = (T)((double)P.base_mass + u[17]);
    L.kp = (T)((double)P.kp * u[18]);
    const double yaw = u[0];
    const double *jn = u + 1;
#pragma unroll
    for (int k = 0; k < 3; ++k) cmd[k] = (T)u[13 + k];
    double sh, ch;
    sincos(0.5 * yaw, &sh, &ch);
    L.pos[0] = T(0);
    L.pos[1] = T(0);
    L.pos[2] = E.home_height;
    L.quat[0] = (T)ch;
    L.quat[1] = T(0);
    L.quat[2] = T(0);
    L.quat[3] = (T)sh;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        L.vlin[i] = T(0);
        L.wb[i] = T(0);
        L.qd[i] = T(0);
        L.q[i] = (T)((double)E.q_default[3 * l + i] + jn[3 * l + i]);
        prev_action[i] = T(0);
    }
    phase = E.phase0[l];
    air = T(0);
}

// Observation noise into the row, quad-parallel: the draws of
// stream_rng(seed, env, episode, step) in build_locomotion_observation's group
// order (gravity, lin vel, ang vel, joint pos, joint vel; a group with scale 0
// draws nothing, envkit.py:176-180).  Word q of the stream is word q % 4 of
// Philox block q / 4 (philox_seek); lane l computes the blocks b with b % 4 == l
// and adds the draws of their words, so every element is touched by one lane.
template <typename T>
__device__ __noinline__ void go1_noise_quad(T *row, uint64_t seed, uint64_t env,
                                            uint32_t episode, uint64_t step,
                                            const double *noise, int l) {
    const int start[5] = {0, 3, 6, 9, 9 + NJ}, len[5] = {3, 3, 3, NJ, NJ};
    int total = 0;  // words drawn: the enabled groups' elements
#pragma unroll
    for (int gi = 0; gi < 5; ++gi)
        if (noise[gi] > 0) total += len[gi];
    // the lanes' blocks side by side (block b on lane b % 4; a block-at-a-time
    // walk over the words made the quad's lanes take turns)
    for (int b = l; 4 * b < total; b += 4) {
        Philox4x64 r;
        philox_seek(r, seed, env, episode, step, (uint64_t)b << 2);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int q = 4 * b + j;
            if (q >= total) break;
            // word q -> row slot of its element and its group's scale (unrolled:
            // the group tables stay in registers)
            int slot = 0, f = 0;
            double sc = 0.0;
#pragma unroll
            for (int gi = 0; gi < 5; ++gi) {
                const double g_sc = noise[gi];
                if (g_sc > 0) {
                    if (q >= f && q < f + len[gi]) {
                        slot = start[gi] + (q - f);
                        sc = g_sc;
                    }
                    f += len[gi];
                }
            }
            const uint64_t w = j == 0 ? r.buf[0] : j == 1 ? r.buf[1] : j == 2 ? r.buf[2] : r.buf[3];
            const double range = __dsub_rn(sc, -sc);
            const double u = __dmul_rn((double)(w >> 11), 1.0 / 9007199254740992.0);
            row[slot] = row[slot] + (T)__dadd_rn(-sc, __dmul_rn(range, u));
        }
    }
}

// rewards.total_reward + the clean observation row (loco_row's math,
// locomotion.cuh), quad-parallel: lane l takes joints 3l..3l+2 and foot l, the
// ten per-joint / per-foot sums are quad-reduced, lane 0 adds the trunk terms.
// Returns the unclipped total in every lane; terms16 filled by lane 0.
template <typename T>
__device__ __noinline__ T go1_row_quad(const EnvConst<T> &E, const T *fr, const uint8_t *flags,
                                       bool done, T *row, T *terms16, int l) {
    const RewardCfg<T> &c = E.rc;
    const int o_jp = 9, o_jv = 9 + NJ, o_pa = 9 + 2 * NJ, o_cmd = 9 + 3 * NJ;
    const int o_ph = o_cmd + 3, o_con = S, o_tau = S + NF, o_pert = S + NF + NJ;
    T tt = 0, jp = 0, ar = 0, en = 0, pose = 0, vv = 0;
#pragma unroll
    for (int jj = 0; jj < 3; ++jj) {
        const int j = 3 * l + jj;
        const T qj = fr[O_JPOS + j], vj = fr[O_JVEL + j], tj = fr[O_JTAU + j];
        tt = tt + tj * tj;
        const T d1 = qj - E.q_default[j];
        jp = jp + d1 * d1;
        const T d2 = fr[O_ACT + j] - fr[O_FPA + j];
        ar = ar + d2 * d2;
        en = en + fabs(vj * tj);
        pose = pose + d1 * d1;  // joint_default == joint_nominal == q_default here
        vv = vv + vj * vj;
        row[o_jp + j] = qj;
        row[o_jv + j] = vj;
        row[o_pa + j] = fr[O_ACT + j];
        row[o_tau + j] = tj;
    }
    T air_s, clr, ph, slip;
    {
        const int k = l;
        const T span = c.airtime_max - c.airtime_min;
        T gain = (fr[O_AIR + k] - c.airtime_min) * (flags[k] ? T(1) : T(0));
        air_s = gain < T(0) ? T(0) : (gain > span ? span : gain);
        const T hk = fr[O_FH + k], err_h = hk - fr[O_FHD + k];
        const T vx = fr[O_FVEL + 2 * k], vy = fr[O_FVEL + 2 * k + 1];
        const T sp = RealOps<T>::sqrt_(vx * vx + vy * vy);
        clr = err_h * err_h * RealOps<T>::sqrt_(sp);
        T sn, cs;
        RealOps<T>::sincos_(fr[O_PHASE + k], &sn, &cs);
        const T tgt = c.swing_height * (sn > T(0) ? sn : T(0));
        const T dz = hk - tgt;
        ph = dz * dz;
        const T m = flags[4 + k] ? T(1) : T(0);
        const T cx = vx * m, cy = vy * m;
        slip = cx * cx + cy * cy;
        row[o_ph + 2 * k] = cs;
        row[o_ph + 2 * k + 1] = sn;
        row[o_con + k] = m;
    }
    tt = phys::qsum(tt); jp = phys::qsum(jp); ar = phys::qsum(ar); en = phys::qsum(en);
    pose = phys::qsum(pose); vv = phys::qsum(vv); air_s = phys::qsum(air_s);
    clr = phys::qsum(clr); ph = phys::qsum(ph); slip = phys::qsum(slip);
    T t[16];
    const T *lin = fr + O_LIN, *ang = fr + O_ANG, *fcmd = fr + O_CMD;
    const T e0 = fcmd[0] - lin[0], e1 = fcmd[1] - lin[1];
    t[0] = rexp(-(e0 * e0 + e1 * e1) / c.sigma_lin);
    const T ea = fcmd[2] - ang[2];
    t[1] = rexp(-(ea * ea) / c.sigma_ang);
    T g[3];
    if (!project_gravity(fr + O_Q, g)) g[0] = g[1] = g[2] = T(NAN);
    t[6] = g[0] * g[0] + g[1] * g[1];
    t[7] = tt; t[8] = jp; t[9] = ar; t[10] = en;
    t[11] = rexp(-pose);
    t[2] = air_s; t[3] = clr; t[4] = rexp(-ph / c.sigma_phase); t[5] = slip;
    t[12] = done ? T(1) : T(0);
    const T cn = RealOps<T>::sqrt_(fcmd[0] * fcmd[0] + fcmd[1] * fcmd[1]);
    t[13] = !c.gated ? cn : (cn > T(0.1) ? T(0) : RealOps<T>::sqrt_(vv));
    t[14] = lin[2] * lin[2];
    t[15] = ang[0] * ang[0] + ang[1] * ang[1];
    T u = T(0);
#pragma unroll
    for (int k = 0; k < 16; ++k) u = u + c.w[k] * t[k];
    if (l == 0) {
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            row[i] = g[i];
            row[3 + i] = lin[i];
            row[6 + i] = ang[i];
            row[o_cmd + i] = fcmd[i];
            row[o_pert + i] = T(0);
        }
        if (terms16)
#pragma unroll
            for (int k = 0; k < 16; ++k) terms16[k] = t[k];
    }
    return u;
}

// lane-parallel part of the frame of the current state (each lane its limb,
// lane 0 the trunk); returns the lane's foot contact.  noinline: one copy for
// the step and the two reset paths (instruction-cache footprint).
template <typename T>
__device__ __noinline__ bool fill_frame(const PhysConst<T> &Pc, const EnvConst<T> &E,
                                        const Lane<T> &L, int l, T *fr, uint8_t *flags,
                                        const T *act3, const T *tau3, const T *prev,
                                        const T *cmd, bool reset_frame, uint8_t lastc, T &phase,
                                        T &air) {
    T fpos[3], fvel[3];
    foot_kin(Pc, L, l, fpos, fvel);
    const bool contact = fpos[2] - Pc.foot_radius < T(0);
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        fr[O_JPOS + 3 * l + j] = L.q[j];
        fr[O_JVEL + 3 * l + j] = L.qd[j];
        fr[O_JTAU + 3 * l + j] = tau3[j];
        fr[O_ACT + 3 * l + j] = act3[j];
        fr[O_FPA + 3 * l + j] = prev[j];
    }
    if (!reset_frame) {
        air = air + E.ctrl_dt;
        phase = wrap_angle_dev(phase + T(6.283185307179586) * E.gait_freq * E.ctrl_dt);
    }
    const bool td = reset_frame ? false : (contact && !lastc);
    fr[O_AIR + l] = air;
    fr[O_FH + l] = fpos[2] - Pc.foot_radius;
    T sn, cs;
    RealOps<T>::sincos_(phase, &sn, &cs);
    fr[O_FHD + l] = E.rc.swing_height * (sn > T(0) ? sn : T(0));
    fr[O_FVEL + 2 * l] = fvel[0];
    fr[O_FVEL + 2 * l + 1] = fvel[1];
    fr[O_PHASE + l] = phase;
    flags[l] = td ? 1 : 0;
    flags[4 + l] = contact ? 1 : 0;
    if (l == 0) {
        T R0[9], vl[3];
        phys::quat2mat(L.quat, R0);
        phys::mat_tvec3(R0, L.vlin, vl);
#pragma unroll
        for (int i = 0; i < 4; ++i) fr[O_Q + i] = L.quat[i];
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            fr[O_LIN + i] = vl[i];
            fr[O_ANG + i] = L.wb[i];
            fr[O_CMD + i] = cmd[i];
        }
    }
    return contact;
}

template <typename T>
__global__ void __launch_bounds__(phys::THREADS)
go1_env_kernel(PhysConst<T> pc, EnvConst<T> ec, EnvState<T> st, EnvIO<T> io) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const size_t pc_b = (sizeof(PhysConst<T>) + 15) & ~size_t(15);
    const size_t ec_b = (sizeof(EnvConst<T>) + 15) & ~size_t(15);
    PhysConst<T> &Pc = *reinterpret_cast<PhysConst<T> *>(smem_raw);
    EnvConst<T> &E = *reinterpret_cast<EnvConst<T> *>(smem_raw + pc_b);
    const int nt = blockDim.x, wpc = nt >> 2;
    T *rowbuf = reinterpret_cast<T *>(smem_raw + pc_b + ec_b);
    T *frames = rowbuf + (size_t)pc.rows_per_lane * phys::RF * nt;  // [wpc][FR]
    T *tile = frames + (size_t)wpc * FR;                             // [wpc][P]
    {
        const uint32_t *s1 = reinterpret_cast<const uint32_t *>(&pc);
        uint32_t *d1 = reinterpret_cast<uint32_t *>(smem_raw);
        for (int i = threadIdx.x; i < (int)(sizeof(PhysConst<T>) / 4); i += nt) d1[i] = s1[i];
        const uint32_t *s2 = reinterpret_cast<const uint32_t *>(&ec);
        uint32_t *d2 = reinterpret_cast<uint32_t *>(smem_raw + pc_b);
        for (int i = threadIdx.x; i < (int)(sizeof(EnvConst<T>) / 4); i += nt) d2[i] = s2[i];
    }
    __syncthreads();
    const int tid = threadIdx.x, l = tid & 3, wl = tid >> 2;
    const int64_t n = io.n;
    const int64_t w0 = (int64_t)blockIdx.x * wpc;
    const int64_t w = w0 + wl;
    const bool live = w < n;
    const int nlive = (int)(n - w0 < wpc ? n - w0 : wpc);
    T *fr = frames + (size_t)wl * FR;
    T *row = tile + (size_t)wl * P;
    uint8_t *flags = reinterpret_cast<uint8_t *>(fr + O_FLAGS);
    Rows<T> rows{rowbuf + (size_t)tid * pc.rows_per_lane * phys::RF};
    const uint64_t env = (uint64_t)(E.env0 + w);

    // ---- load the world
    Lane<T> L;
    T cmd[3] = {T(0), T(0), T(0)}, phase = T(0), air = T(0), prev[3] = {T(0), T(0), T(0)};
    uint8_t lastc = 1;
    int32_t steps = 0;
    uint32_t episode = 0;
    if (live) {
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            L.pos[i] = st.qpos[i * n + w];
            L.vlin[i] = st.qvel[i * n + w];
            L.wb[i] = st.qvel[(3 + i) * n + w];
            L.q[i] = st.qpos[(7 + 3 * l + i) * n + w];
            L.qd[i] = st.qvel[(6 + 3 * l + i) * n + w];
            cmd[i] = st.cmd[i * n + w];
            prev[i] = st.prev_action[(3 * l + i) * n + w];
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) L.quat[i] = st.qpos[(3 + i) * n + w];
        phase = st.phase[l * n + w];
        air = st.air[l * n + w];
        L.mu = st.dr[w];
        L.base_mass = st.dr[n + w];
        L.kp = st.dr[2 * n + w];
        lastc = st.last_contact[l * n + w];
        steps = st.steps[w];
        episode = st.episode[w];
    }

    auto build = [&](bool done, T *reward, T *terms16) {  // all four lanes of the quad
        const T u = go1_row_quad(E, fr, flags, done, row, terms16, l);
        if (reward) *reward = T(0) > u ? T(0) : u;
    };
    // cooperative, coalesced store of the CTA's rows [nlive][cols] (tile pitch P)
    auto store_rows = [&](T *dst, int cols) {
        for (int e = tid; e < nlive * cols; e += nt) {
            const int r = e / cols, c = e - r * cols;
            dst[(w0 + r) * cols + c] = tile[r * P + c];
        }
    };
    const unsigned qm = phys::quad_mask();

    // observation noise key: stream_rng(seed, env, episode, steps + 1) -- step 0
    // of an episode's stream belongs to its reset draw
    auto add_noise = [&]() {  // all four lanes of the quad
        if (E.has_noise) go1_noise_quad(row, E.seed, env, episode, (uint64_t)steps + 1, E.noise, l);
    };
    auto do_reset = [&]() {
        reset_world(Pc, E, L, l, env, episode, cmd, phase, air, prev);
        const T zero3[3] = {T(0), T(0), T(0)};
        const bool c = fill_frame(Pc, E, L, l, fr, flags, zero3, zero3, prev, cmd, true, lastc,
                                  phase, air);
        lastc = c ? 1 : 0;
        __syncwarp(qm);
        build(false, nullptr, nullptr);
        __syncwarp(qm);
    };

    if (io.reset_all) {
        if (live) {
            episode = 0;
            steps = 0;
            do_reset();
        }
        __syncthreads();
        if (io.priv) store_rows(io.priv, P);
        __syncthreads();
        if (live) add_noise();
        __syncthreads();
        store_rows(io.obs, S);
    }

    for (int64_t k = 0; k < (io.reset_all ? 0 : io.K); ++k) {
        T a[3] = {T(0), T(0), T(0)}, tau[3] = {T(0), T(0), T(0)};
        bool done = false, trunc = false;
        T rw = T(0);
        T t16[16];
        if (live) {
            // action -> clipped [-1, 1] -> absolute joint targets
            bool finite = true;
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                T v = io.actions[(k * n + w) * NJ + 3 * l + j];
                finite &= isfinite(v);
                v = isfinite(v) ? (v < T(-1) ? T(-1) : (v > T(1) ? T(1) : v)) : T(0);
                a[j] = v;
                L.ctrl[j] = E.q_default[3 * l + j] + E.action_scale * v;
            }
            if (!phys::qall(finite) && l == 0 && io.err)
                atomicMin(io.err, (unsigned long long)(k * n + w));
            bool okp = true;
            // (a full CTA: every thread steps, so the step's CTA barriers are safe)
            for (int s = 0; s < E.substeps; ++s)
                okp &= phys::phys_step(Pc, L, rows, l,
                                       static_cast<const phys::PhysArgs<T> *>(nullptr), w,
                                       static_cast<const phys::PhysInspect<T> *>(nullptr),
                                       s + 1 == E.substeps ? tau : nullptr, nlive == wpc);
            if (!okp && l == 0 && io.bad) *io.bad = 1;
            const bool c = fill_frame(Pc, E, L, l, fr, flags, a, tau, prev, cmd, false, lastc,
                                      phase, air);
            // termination: trunk upside down (its z axis points down) or below term_height
            T R0[9];
            phys::quat2mat(L.quat, R0);
            done = R0[8] < T(0) || L.pos[2] < E.term_height;
            steps += 1;
            trunc = steps >= E.episode_length;
            __syncwarp(qm);
            build(done, &rw, t16);
            __syncwarp(qm);
            // post-reward bookkeeping (the frame used the pre-step values)
            air = c ? T(0) : air;
            lastc = c ? 1 : 0;
#pragma unroll
            for (int j = 0; j < 3; ++j) prev[j] = a[j];
            if (l == 0) {
                io.reward[k * n + w] = rw;
                io.done[k * n + w] = done ? 1 : 0;
                io.trunc[k * n + w] = trunc ? 1 : 0;
                if (io.terms)
#pragma unroll
                    for (int q = 0; q < 16; ++q) io.terms[(k * n + w) * 16 + q] = t16[q];
                if (io.terminal_mask) io.terminal_mask[k * n + w] = (done || trunc) ? 1 : 0;
            }
            // auto-reset: emit the terminal observation, start the next episode
            if (done || trunc) {
                if (io.terminal_priv) {  // the clean row, before the sensor noise
                    __syncwarp(qm);
                    for (int c2 = l; c2 < P; c2 += 4) io.terminal_priv[(k * n + w) * P + c2] = row[c2];
                    __syncwarp(qm);
                }
                add_noise();
                __syncwarp(qm);
                if (io.terminal_obs)
                    for (int c2 = l; c2 < S; c2 += 4) io.terminal_obs[(k * n + w) * S + c2] = row[c2];
                __syncwarp(qm);
                episode += 1;
                steps = 0;
                do_reset();
            }
        }
        __syncthreads();
        if (io.priv) store_rows(io.priv + k * n * P, P);
        __syncthreads();
        if (live) add_noise();
        __syncthreads();
        store_rows(io.obs + k * n * S, S);
        __syncthreads();
    }

    // ---- store the world
    if (live) {
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            if (l == 0) {
                st.qpos[i * n + w] = L.pos[i];
                st.qvel[i * n + w] = L.vlin[i];
                st.qvel[(3 + i) * n + w] = L.wb[i];
                st.cmd[i * n + w] = cmd[i];
            }
            st.qpos[(7 + 3 * l + i) * n + w] = L.q[i];
            st.qvel[(6 + 3 * l + i) * n + w] = L.qd[i];
            st.prev_action[(3 * l + i) * n + w] = prev[i];
        }
        if (l == 0) {
#pragma unroll
            for (int i = 0; i < 4; ++i) st.qpos[(3 + i) * n + w] = L.quat[i];
            st.steps[w] = steps;
            st.episode[w] = episode;
        }
        st.phase[l * n + w] = phase;
        st.air[l * n + w] = air;
        if (l == 0) {
            st.dr[w] = L.mu;
            st.dr[n + w] = L.base_mass;
            st.dr[2 * n + w] = L.kp;
        }
        st.last_contact[l * n + w] = lastc;
    }
}

}  // namespace go1
}  // namespace dk

namespace dk {
namespace go1 {

template <typename T>
size_t env_smem_bytes(const PhysConst<T> &pc, int threads) {
    return ((sizeof(PhysConst<T>) + 15) & ~size_t(15)) + ((sizeof(EnvConst<T>) + 15) & ~size_t(15)) +
           (size_t)pc.rows_per_lane * phys::RF * threads * sizeof(T) +
           (size_t)(threads / 4) * (FR + P) * sizeof(T);
}

template <typename T>
cudaError_t launch_env(const PhysConst<T> &pc, const EnvConst<T> &ec, const EnvState<T> &st,
                       const EnvIO<T> &io, cudaStream_t s) {
    const int threads = phys::pick_threads(io.n, [&](int t) { return env_smem_bytes(pc, t); });
    const size_t smem = env_smem_bytes(pc, threads);
    static SmemOptIn optin;  // per device
    cudaError_t e = optin.ensure((const void *)go1_env_kernel<T>, smem);
    if (e != cudaSuccess) return e;
    const int wpc = threads / 4;
    const unsigned grid = (unsigned)((io.n + wpc - 1) / wpc);
    go1_env_kernel<T><<<grid, threads, smem, s>>>(pc, ec, st, io);
    return cudaGetLastError();
}

#define DK_GO1_DECLARE(T)                                                                     \
    extern template cudaError_t launch_env<T>(const PhysConst<T> &, const EnvConst<T> &,     \
                                              const EnvState<T> &, const EnvIO<T> &,         \
                                              cudaStream_t);
#define DK_GO1_INSTANTIATE(T)                                                                 \
    template cudaError_t launch_env<T>(const PhysConst<T> &, const EnvConst<T> &,            \
                                       const EnvState<T> &, const EnvIO<T> &, cudaStream_t);

}  // namespace go1
}  // namespace dk
