// locomotion.cuh -- the locomotion step tail at Go1 shape.
//
// loco_tail_kernel fuses, per world and step, the reward table
// (rewards.total_reward + the 16 terms, rewards.py:97-211) with the observation
// builder (envkit.build_locomotion_observation, envkit.py:147-193: projected
// gravity, phase encoding, Philox-keyed uniform sensor noise, privileged slot),
// so each frame is read from HBM once and every output is written once.
// One thread owns one (step, world) row; per-warp shared-memory tiles turn the
// row-major outputs into contiguous row stores.  The joint / foot loops are
// runtime-sized (Go1: 12 joints, 4 feet; bipeds; hands), accumulating in
// registers in the reference's term order.
#pragma once
#include "envmath.cuh"

// Unroll factors of the runtime-sized joint / foot loops (development hooks;
// unset = the compiler's choice).
#define DK_PRAGMA_(x) _Pragma(#x)
#define DK_UNROLL_(n) DK_PRAGMA_(unroll n)
#ifdef DK_TAIL_UNROLL_J
#define DK_UNROLL_J DK_UNROLL_(DK_TAIL_UNROLL_J)
#else
#define DK_UNROLL_J
#endif
#ifdef DK_TAIL_UNROLL_F
#define DK_UNROLL_F DK_UNROLL_(DK_TAIL_UNROLL_F)
#else
#define DK_UNROLL_F
#endif

namespace dk {

template <typename T>
struct LocoFrames {  // rows [K*N, dim]; nominal / default: stride 0 = broadcast [dim]
    const T *q, *lin, *ang, *jpos, *jvel, *jtau, *fh, *fhd, *fvel;
    const uint8_t *contact;
    const T *air;
    const uint8_t *touchdown;
    const T *phase, *cmd, *act, *pact, *nom, *def;
    const uint8_t *done;
    int64_t nom_stride, def_stride;
};

template <typename T>
struct RewardCfg {  // RewardTermConfig (rewards.py:51-75)
    T w[16];        // weights in TERM_REGISTRY order (rewards.py:181-198)
    T sigma_lin, sigma_ang, airtime_min, airtime_max, sigma_phase, swing_height;
    int gated;
};

template <typename T>
struct LocoOut {
    T *total, *unclipped, *terms, *state, *priv;  // terms / state / priv may be null
};

struct LocoArgs {
    int64_t K, N;       // steps x worlds rows
    int nj, nf;
    uint64_t seed;
    int64_t env0;
    uint64_t step0;
    const uint32_t *episode;  // [N] or null (episode 0)
    double noise[5];          // gravity, lin_vel, ang_vel, joint_pos, joint_vel
    int has_noise;
};

// mathcore.project_gravity (mathcore.py:93-97) incl. quat_check_unit (42-48);
// returns false for a non-unit quaternion.
template <typename T>
__device__ __forceinline__ bool project_gravity(const T *q4, T *g) {
    const T w = q4[0], x = q4[1], y = q4[2], z = q4[3];
    const T nrm = RealOps<T>::sqrt_(w * w + x * x + y * y + z * z);
    if (fabs(nrm - T(1)) > T(1e-6)) return false;  // (NaN passes, as in the reference)
    // quat_rotate(conj(q), (0,0,-1)) written out like quat_mul(quat_mul(c, p), conj(c))
    const T c0 = w, c1 = -x, c2 = -y, c3 = -z;
    const T a0 = c0 * T(0) - c1 * T(0) - c2 * T(0) - c3 * T(-1);
    const T a1 = c0 * T(0) + c1 * T(0) + c2 * T(-1) - c3 * T(0);
    const T a2 = c0 * T(0) - c1 * T(-1) + c2 * T(0) + c3 * T(0);
    const T a3 = c0 * T(-1) + c1 * T(0) - c2 * T(0) + c3 * T(0);
    const T d1 = -c1, d2 = -c2, d3 = -c3;
    const T r1 = a0 * d1 + a1 * c0 + a2 * d3 - a3 * d2;
    const T r2 = a0 * d2 - a1 * d3 + a2 * c0 + a3 * d1;
    const T r3 = a0 * d3 + a1 * d2 - a2 * d1 + a3 * c0;
    const T m = RealOps<T>::sqrt_(r1 * r1 + r2 * r2 + r3 * r3);
    g[0] = r1 / m; g[1] = r2 / m; g[2] = r3 / m;
    return true;
}

template <typename T>
__device__ __forceinline__ T rexp(T x) { return RealOps<T>::exp_(x); }

template <typename T>
__device__ __forceinline__ void rsincos(T x, T *s, T *c) { RealOps<T>::sincos_(x, s, c); }

// One frame row of the step tail, as pointers to that row's fields (global
// memory in loco_tail_kernel, shared memory in the fused Go1 env kernel).
template <typename T>
struct LocoRowIn {
    const T *q, *lin, *ang, *cmd, *fcmd, *pa, *fpa, *nom, *def, *jpos, *jvel, *jtau, *act;
    const T *air, *fh, *fhd, *fvel, *phase;
    const uint8_t *td, *con;
    bool done;
    const T *pert;  // [3] or null
};

template <bool GLOBAL, typename T>
__device__ __forceinline__ T ldv(const T *p) {
    if constexpr (GLOBAL) return __ldg(p);
    else return *p;
}

// rewards.total_reward (16 terms in TERM_REGISTRY order, rewards.py:97-211) and
// the clean observation row of envkit.build_locomotion_observation
// (envkit.py:147-193) in the privileged layout [S | contacts, torques, pert].
// Returns the unclipped total; t[16] receives the terms; ok = unit quaternion.
template <bool GLOBAL, typename T>
__device__ __forceinline__ T loco_row(const LocoRowIn<T> &f, const RewardCfg<T> &c, int nj, int nf,
                                      T *row, T *t, bool &ok) {
    const int S = 9 + 3 * nj + 3 + 2 * nf;
    // lin / ang velocity tracking (rewards.py:97-104): from the FRAME's command
    const T e0 = f.fcmd[0] - f.lin[0], e1 = f.fcmd[1] - f.lin[1];
    t[0] = rexp(-(e0 * e0 + e1 * e1) / c.sigma_lin);
    const T ea = f.fcmd[2] - f.ang[2];
    t[1] = rexp(-(ea * ea) / c.sigma_ang);
    // projected gravity -> orientation term + obs
    T g[3];
    ok = project_gravity(f.q, g);
    if (!ok) g[0] = g[1] = g[2] = T(NAN);  // InvalidInputError (mathcore.py:46-47)
    t[6] = g[0] * g[0] + g[1] * g[1];
    int o = 0;
    row[o++] = g[0]; row[o++] = g[1]; row[o++] = g[2];
    for (int k = 0; k < 3; ++k) row[o++] = f.lin[k];
    for (int k = 0; k < 3; ++k) row[o++] = f.ang[k];
    // joints: terms 7-11, 13 (gated) + obs joint_pos / joint_vel / prev_action / torque
    T tt = 0, jp = 0, ar = 0, en = 0, pose = 0, vv = 0;
    const int o_jp = 9, o_jv = 9 + nj, o_pa = 9 + 2 * nj, o_cmd = 9 + 3 * nj;
    const int o_ph = o_cmd + 3, o_con = S, o_tau = S + nf, o_pert = S + nf + nj;
    DK_UNROLL_J
    for (int j = 0; j < nj; ++j) {
        const T qj = ldv<GLOBAL>(f.jpos + j), vj = ldv<GLOBAL>(f.jvel + j);
        const T tj = ldv<GLOBAL>(f.jtau + j);
        tt = tt + tj * tj;
        const T d1 = qj - ldv<GLOBAL>(f.nom + j);
        jp = jp + d1 * d1;
        const T d2 = ldv<GLOBAL>(f.act + j) - ldv<GLOBAL>(f.fpa + j);
        ar = ar + d2 * d2;
        en = en + fabs(vj * tj);
        const T d3 = qj - ldv<GLOBAL>(f.def + j);
        pose = pose + d3 * d3;
        vv = vv + vj * vj;
        row[o_jp + j] = qj;
        row[o_jv + j] = vj;
        row[o_pa + j] = ldv<GLOBAL>(f.pa + j);
        row[o_tau + j] = tj;
    }
    t[7] = tt; t[8] = jp; t[9] = ar; t[10] = en;
    t[11] = rexp(-pose);
    for (int k = 0; k < 3; ++k) row[o_cmd + k] = f.cmd[k];
    // feet: terms 2-5 + obs phase cos/sin and contact flags
    T air_s = 0, clr = 0, ph = 0, slip = 0;
    const T span = c.airtime_max - c.airtime_min;
    DK_UNROLL_F
    for (int k = 0; k < nf; ++k) {
        T gain = (ldv<GLOBAL>(f.air + k) - c.airtime_min) * (f.td[k] ? T(1) : T(0));
        gain = gain < T(0) ? T(0) : (gain > span ? span : gain);  // np.clip
        air_s = air_s + gain;
        const T hk = ldv<GLOBAL>(f.fh + k), err_h = hk - ldv<GLOBAL>(f.fhd + k);
        const T vx = ldv<GLOBAL>(f.fvel + 2 * k), vy = ldv<GLOBAL>(f.fvel + 2 * k + 1);
        const T sp = RealOps<T>::sqrt_(vx * vx + vy * vy);
        clr = clr + err_h * err_h * RealOps<T>::sqrt_(sp);
        T sn, cs;
        rsincos(ldv<GLOBAL>(f.phase + k), &sn, &cs);
        const T tgt = c.swing_height * (sn > T(0) ? sn : T(0));  // swing_height_profile
        const T dz = hk - tgt;
        ph = ph + dz * dz;
        const T m = f.con[k] ? T(1) : T(0);
        const T cx = vx * m, cy = vy * m;
        slip = slip + (cx * cx + cy * cy);
        row[o_ph + 2 * k] = cs;
        row[o_ph + 2 * k + 1] = sn;
        row[o_con + k] = m;
    }
    t[2] = air_s; t[3] = clr; t[4] = rexp(-ph / c.sigma_phase); t[5] = slip;
    t[12] = f.done ? T(1) : T(0);
    const T cn = RealOps<T>::sqrt_(f.fcmd[0] * f.fcmd[0] + f.fcmd[1] * f.fcmd[1]);
    t[13] = !c.gated ? cn : (cn > T(0.1) ? T(0) : RealOps<T>::sqrt_(vv));
    t[14] = f.lin[2] * f.lin[2];
    t[15] = f.ang[0] * f.ang[0] + f.ang[1] * f.ang[1];
    T u = T(0);
#pragma unroll
    for (int k = 0; k < 16; ++k) u = u + c.w[k] * t[k];  // sum(weighted) in registry order
    for (int k = 0; k < 3; ++k) row[o_pert + k] = f.pert ? f.pert[k] : T(0);
    return u;
}

// uniform sensor noise per group, drawn in the reference's order from
// stream_rng(seed, env, episode, step) (envkit.py:41-49, 176-180)
template <typename T>
__device__ __forceinline__ void loco_row_noise(T *row, int nj, uint64_t seed, uint64_t env,
                                               uint32_t episode, uint64_t step,
                                               const double *noise) {
    Philox4x64 rng;
    rng.init(seed, env, episode, step);
    const int start[5] = {0, 3, 6, 9, 9 + nj}, len[5] = {3, 3, 3, nj, nj};
    for (int gi = 0; gi < 5; ++gi) {
        const double s = noise[gi];
        if (s > 0)
            for (int e = 0; e < len[gi]; ++e)
                row[start[gi] + e] = row[start[gi] + e] + (T)rng.uniform(-s, s);
    }
}

template <typename T>
__global__ void __launch_bounds__(128)
loco_tail_kernel(LocoFrames<T> f, const T *__restrict__ prev_action, const T *__restrict__ command,
                 const T *__restrict__ pert, RewardCfg<T> c, LocoArgs a, LocoOut<T> out,
                 unsigned long long *err) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int nj = a.nj, nf = a.nf;
    const int S = 9 + 3 * nj + 3 + 2 * nf;  // state slot
    const int P = S + nf + nj + 3;          // privileged slot
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    T *tile = reinterpret_cast<T *>(smem_raw) + (size_t)warp * 32 * P;
    T *row = tile + (size_t)lane * P;
    const int64_t rows = a.K * a.N;
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t r0 = r - lane;  // first row of this warp
    const bool live = r < rows;

    if (live) {
        LocoRowIn<T> in;
        in.q = f.q + 4 * r;
        in.lin = f.lin + 3 * r;
        in.ang = f.ang + 3 * r;
        in.cmd = (command ? command : f.cmd) + 3 * r;
        in.fcmd = f.cmd + 3 * r;
        in.pa = (prev_action ? prev_action : f.pact) + (int64_t)nj * r;
        in.fpa = f.pact + (int64_t)nj * r;
        in.nom = f.nom + f.nom_stride * r;
        in.def = f.def + f.def_stride * r;
        in.jpos = f.jpos + (int64_t)nj * r;
        in.jvel = f.jvel + (int64_t)nj * r;
        in.jtau = f.jtau + (int64_t)nj * r;
        in.act = f.act + (int64_t)nj * r;
        in.air = f.air + (int64_t)nf * r;
        in.fh = f.fh + (int64_t)nf * r;
        in.fhd = f.fhd + (int64_t)nf * r;
        in.fvel = f.fvel + (int64_t)2 * nf * r;
        in.phase = f.phase + (int64_t)nf * r;
        in.td = f.touchdown + (int64_t)nf * r;
        in.con = f.contact + (int64_t)nf * r;
        in.done = f.done[r] != 0;
        in.pert = pert ? pert + 3 * r : nullptr;
        T t[16];
        bool ok;
        const T u = loco_row<true>(in, c, nj, nf, row, t, ok);
        if (!ok) atomicMin(err, (unsigned long long)r);
        out.unclipped[r] = u;
        out.total[r] = T(0) > u ? T(0) : u;  // max(unclipped, 0.0)
        if (out.terms) {
#pragma unroll
            for (int k = 0; k < 16; ++k) out.terms[16 * r + k] = t[k];
        }
    }
    __syncwarp();
    const int64_t nrow = rows - r0 < 32 ? rows - r0 : 32;
    if (out.priv) {  // privileged slot: the clean signals + contacts, torques, perturbation
        for (int rr = 0; rr < nrow; ++rr) {
            T *dst = out.priv + (r0 + rr) * P;
            for (int col = lane; col < P; col += 32) dst[col] = tile[rr * P + col];
        }
    }
    if (live && a.has_noise) {
        const int64_t k = r / a.N, i = r - k * a.N;
        loco_row_noise(row, nj, a.seed, (uint64_t)(a.env0 + i), a.episode ? a.episode[i] : 0u,
                       a.step0 + (uint64_t)k, a.noise);
    }
    __syncwarp();
    if (out.state) {
        for (int rr = 0; rr < nrow; ++rr) {
            T *dst = out.state + (r0 + rr) * S;
            for (int col = lane; col < S; col += 32) dst[col] = tile[rr * P + col];
        }
    }
}

// ---------------------------------------------------------------------------
// Small batched kernels (one thread per element / row).

// action_to_target + pd_torque (envkit.py:111-131); a, prev, q, v [N, J]
template <typename T>
__global__ void pd_kernel(int64_t n, int nj, T kp, T kd, T scale, T limit, T lo, T hi, int relative,
                          const T *q_default, const T *a, const T *prev, const T *q, const T *v,
                          T *target, T *torque) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n * nj) return;
    const int j = (int)(e % nj);
    T t;
    if (!relative) {
        t = q_default[j] + scale * a[e];
    } else {
        t = prev[e] + scale * a[e];
        t = t < lo ? lo : t;  // np.clip(target, lo, hi)
        t = t > hi ? hi : t;
    }
    if (target) target[e] = t;
    T tau = kp * (t - q[e]) - kd * v[e];
    tau = tau < -limit ? -limit : tau;
    tau = tau > limit ? limit : tau;
    torque[e] = tau;
}

// wrap_angle(phi + 2*pi*f*dt) (mathcore.py:143-171): NumPy divmod semantics
template <typename T>
__device__ __forceinline__ T wrap_angle_dev(T phi) {
    const T two_pi = T(6.283185307179586), pi = T(3.141592653589793);
    const T x = phi + pi;
    T m = fmod(x, two_pi);
    if (m != T(0)) {
        if (m < T(0)) m = m + two_pi;
    } else {
        m = T(0);
    }
    return m - pi;
}

template <typename T>
__global__ void phase_kernel(int64_t n, int nf, const T *phi, const T *freq, const T *dt,
                             T *out_phi, T *out_cs) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n * nf) return;
    const int64_t i = e / nf;
    const T np_ = wrap_angle_dev(phi[e] + T(6.283185307179586) * freq[i] * dt[i]);
    if (out_phi) out_phi[e] = np_;
    if (out_cs) {  // phase_encode (mathcore.py:174-177)
        T s, c;
        RealOps<T>::sincos_(np_, &s, &c);
        out_cs[2 * e] = c;
        out_cs[2 * e + 1] = s;
    }
}

// progress_clip_reward (envkit.py:196-202)
template <typename T>
__global__ void progress_kernel(int64_t n, const T *raw, T *hist, T *reward) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const T h = hist[i], x = raw[i], d = x - h;
    reward[i] = T(0) > d ? T(0) : d;
    hist[i] = x > h ? x : h;
}

// apply_sensor_noise (randomization.py:88-108), in place on rows [N, dim]:
// kind 0 uniform U(-s, s), kind 1 gaussian Generator.normal(0, s) = 0 + s * z.
template <typename T>
__global__ void sensor_noise_kernel(int64_t n, int dim, T *obs, int nspec, const int *off,
                                    const int *len, const double *scale, const int *kind,
                                    uint64_t seed, int64_t env0, const uint32_t *episode,
                                    uint64_t step) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    Philox4x64 rng;
    rng.init(seed, (uint64_t)(env0 + i), episode ? episode[i] : 0u, step);
    for (int s = 0; s < nspec; ++s) {
        const double sc = scale[s];
        if (sc == 0.0) continue;
        const bool gauss = kind != nullptr && kind[s] == 1;
        for (int k = 0; k < len[s]; ++k) {
            T *x = obs + i * dim + off[s] + k;
            const double z = gauss ? __dadd_rn(0.0, __dmul_rn(sc, rng.standard_normal()))
                                   : rng.uniform(-sc, sc);
            *x = (T)__dadd_rn((double)*x, z);
        }
    }
}

// The same draws with one warp per world.  Philox is counter-based: word q of
// a world's stream is word q % 4 of the block whose counter is step + 1 + q / 4
// (NumPy bumps the 256-bit counter before each block), so the 32 lanes compute
// 32 consecutive words at once.  Uniform draws take one word each; Gaussian
// draws are speculated one word each (the ziggurat's first test accepts ~99%)
// and, from the first lane whose draw needs more, finished by lane 0 with the
// sequential generator positioned at that word (tail / wedge, exact).
__device__ __forceinline__ void philox_seek(Philox4x64 &r, uint64_t seed, uint64_t env,
                                            uint32_t episode, uint64_t step, uint64_t q) {
    r.init(seed, env, episode, step);
    const uint64_t b = q >> 2;
    const uint64_t c0 = step + 1 + b;
    r.ctr[0] = c0;
    r.ctr[1] = c0 < step ? 1 : 0;  // carry (counter words 2, 3 stay 0 for any sane q)
    r.block();
    r.pos = (int)(q & 3);
}
// The warp's block cache: lane l holds block base + l of the world's stream,
// i.e. words [4 base, 4 base + 128), so one Philox block per lane serves four
// 32-word rounds of draws instead of one.
struct WarpPhiloxCache {
    uint64_t w0, w1, w2, w3;
    uint64_t base;  // block index of lane 0's block (warp-uniform)
    bool valid;

    __device__ __forceinline__ void fill(uint64_t seed, uint64_t env, uint32_t episode,
                                         uint64_t step, uint64_t b0, int lane) {
        Philox4x64 r;
        philox_seek(r, seed, env, episode, step, (b0 + (uint64_t)lane) << 2);
        w0 = r.buf[0]; w1 = r.buf[1]; w2 = r.buf[2]; w3 = r.buf[3];
        base = b0;
        valid = true;
    }
    // word q (per lane) of the stream, q in [pos, pos + 32) for a warp-uniform pos;
    // every lane of the warp must call it.
    __device__ __forceinline__ uint64_t word(uint64_t seed, uint64_t env, uint32_t episode,
                                             uint64_t step, uint64_t pos, uint64_t q, int lane) {
        if (!valid || (pos >> 2) < base || ((pos + 31) >> 2) >= base + 32)
            fill(seed, env, episode, step, pos >> 2, lane);
        const int src = (int)((q >> 2) - base);
        const uint64_t a = __shfl_sync(0xffffffffu, w0, src), b = __shfl_sync(0xffffffffu, w1, src);
        const uint64_t c = __shfl_sync(0xffffffffu, w2, src), d = __shfl_sync(0xffffffffu, w3, src);
        const int j = (int)(q & 3);
        return j == 0 ? a : j == 1 ? b : j == 2 ? c : d;
    }
};

template <typename T>
__global__ void __launch_bounds__(128) sensor_noise_warp_kernel(
    int64_t n, int dim, T *obs, int nspec, const int *off, const int *len, const double *scale,
    const int *kind, uint64_t seed, int64_t env0, const uint32_t *episode, uint64_t step) {
    const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= n) return;
    const uint64_t env = (uint64_t)(env0 + i);
    const uint32_t ep = episode ? episode[i] : 0u;
    T *row = obs + i * dim;
    uint64_t pos = 0;  // next unread word of the world's stream
    WarpPhiloxCache cache;
    cache.valid = false;
    for (int s = 0; s < nspec; ++s) {
        const double sc = scale[s];
        if (sc == 0.0) continue;
        const int L = len[s];
        T *x = row + off[s];
        if (kind == nullptr || kind[s] != 1) {  // uniform(-sc, sc): one word per draw
            const double range = __dsub_rn(sc, -sc);
            for (int k0 = 0; k0 < L; k0 += 32) {
                const int k = k0 + lane;
                const uint64_t w = cache.word(seed, env, ep, step, pos + (uint64_t)k0,
                                              pos + (uint64_t)k, lane);
                if (k < L) {
                    const double u = __dmul_rn((double)(w >> 11), 1.0 / 9007199254740992.0);
                    x[k] = (T)__dadd_rn((double)x[k], __dadd_rn(-sc, __dmul_rn(range, u)));
                }
            }
            pos += (uint64_t)L;
            continue;
        }
        int done = 0;  // Gaussian: 0.0 + sc * standard_normal()
        while (done < L) {
            const int k = done + lane;
            const bool act = k < L;
            bool fast = false;
            double z = 0.0;
            uint64_t r = cache.word(seed, env, ep, step, pos, pos + (uint64_t)lane, lane);
            if (act) {
                const int idx = (int)(r & 0xff);
                r >>= 8;
                const uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
                z = __dmul_rn((double)rabs, __ldg(&dk_zig_wi[idx]));
                if (r & 1) z = -z;
                fast = rabs < __ldg(&dk_zig_ki[idx]);
            }
            const unsigned slow = __ballot_sync(0xffffffffu, act && !fast);
            const int nact = min(32, L - done);
            const int f = slow ? __ffs(slow) - 1 : nact;  // lanes < f are accepted
            if (lane < f) x[k] = (T)__dadd_rn((double)x[k], __dadd_rn(0.0, __dmul_rn(sc, z)));
            done += f;
            pos += (uint64_t)f;
            if (f < nact) {  // draw `done` needs the tail or wedge: finish it sequentially
                uint64_t npos = 0;
                if (lane == 0) {
                    Philox4x64 r;
                    philox_seek(r, seed, env, ep, step, pos);
                    const double zn = r.standard_normal();
                    x[done] = (T)__dadd_rn((double)x[done], __dadd_rn(0.0, __dmul_rn(sc, zn)));
                    npos = ((r.ctr[0] - step - 1) << 2) + (uint64_t)r.pos;
                }
                pos = __shfl_sync(0xffffffffu, npos, 0);
                done += 1;
            }
        }
    }
}

// randomize_params (randomization.py:156-181) for n worlds, f64: out [n, F]
// starts as nominal [F]; ranges r (spec order) perturb field[r] with
// distribution 0 additive base + U(lo, hi), 1 multiplicative base * U(lo, hi),
// 2 log-uniform base * exp(U(log lo, log hi)) (logs precomputed on the host),
// redrawn up to 100 times while a positive nominal goes non-positive.  A world
// that exhausts the tries reports world * nr + range through fail (atomicMin:
// the first such world, then its first such range -> ConfigError).
static __global__ void randomize_params_kernel(int64_t n, int nf, const double *nominal, int nr,
                                               const int *field, const int *dist,
                                               const double *lo, const double *hi,
                                               uint64_t seed, int64_t env0,
                                               const uint32_t *episode, uint64_t step,
                                               double *out, unsigned long long *fail) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double *o = out + i * nf;
    for (int f = 0; f < nf; ++f) o[f] = nominal[f];
    Philox4x64 rng;
    rng.init(seed, (uint64_t)(env0 + i), episode ? episode[i] : 0u, step);
    for (int r = 0; r < nr; ++r) {
        const double base = nominal[field[r]];
        const bool positive = base > 0.0;
        double value = 0.0;
        bool ok = false;
        for (int attempt = 0; attempt < 100 && !ok; ++attempt) {
            const double u = rng.uniform(lo[r], hi[r]);
            value = dist[r] == 0 ? __dadd_rn(base, u)
                  : dist[r] == 1 ? __dmul_rn(base, u)
                                 : __dmul_rn(base, exp(u));
            ok = !positive || value > 0.0;
        }
        if (!ok) atomicMin(fail, (unsigned long long)(i * nr + r));  // first world, then range
        o[field[r]] = value;
    }
}

// DelayLine (randomization.py:27-62), batched.  ring [n, cap, dim] with
// cap = max_delay + 1, head = next write slot, count = values held (<= cap).
static __global__ void delay_reset_kernel(int64_t n, int min_delay, int max_delay, uint64_t seed,
                                          int64_t env0, const uint32_t *episode, uint64_t step,
                                          int32_t *delay, int32_t *count, int32_t *head) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    PhiloxInts g;
    g.px.init(seed, (uint64_t)(env0 + i), episode ? episode[i] : 0u, step);
    delay[i] = (int32_t)g.integers(min_delay, (int64_t)max_delay + 1);  // randomization.py:46
    count[i] = 0;
    head[i] = 0;
}

template <typename T>
__global__ void delay_push_pop_kernel(int64_t n, int dim, int min_delay, int max_delay,
                                      int per_step, T *ring, int32_t *head, int32_t *count,
                                      const int32_t *delay, uint64_t seed, int64_t env0,
                                      const uint32_t *episode, uint64_t step, const T *value,
                                      T *out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int cap = max_delay + 1;
    T *rb = ring + i * (int64_t)cap * dim;
    int h = head[i], c = count[i];
    for (int k = 0; k < dim; ++k) rb[(int64_t)h * dim + k] = value[i * dim + k];  // append
    h = h + 1 == cap ? 0 : h + 1;
    c = c < cap ? c + 1 : cap;  // deque(maxlen=cap) drops the oldest
    int d = delay[i];
    if (per_step) {  // randomization.py:50-51
        PhiloxInts g;
        g.px.init(seed, (uint64_t)(env0 + i), episode ? episode[i] : 0u, step);
        d = (int)g.integers(min_delay, (int64_t)max_delay + 1);
    }
    int idx = c - 1 - d;
    if (idx < 0) idx = 0;  // warm-up: oldest available (randomization.py:60-61)
    int slot = h - c + idx;
    slot = slot < 0 ? slot + cap : slot;
    for (int k = 0; k < dim; ++k) out[i * dim + k] = rb[(int64_t)slot * dim + k];
    head[i] = h;
    count[i] = c;
}

// pose_injection (randomization.py:188-199), in place on rows [N, dim]; bounds [dim, 2]
template <typename T>
__global__ void pose_injection_kernel(int64_t n, int dim, T *pose, const double *bounds,
                                      double prob, uint64_t seed, int64_t env0,
                                      const uint32_t *episode, uint64_t step, uint8_t *injected) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    Philox4x64 rng;
    rng.init(seed, (uint64_t)(env0 + i), episode ? episode[i] : 0u, step);
    const bool inj = rng.uniform(0.0, 1.0) < prob;
    if (inj)
        for (int k = 0; k < dim; ++k) pose[i * dim + k] = (T)rng.uniform(bounds[2 * k], bounds[2 * k + 1]);
    if (injected) injected[i] = inj ? 1 : 0;
}

// curriculum_update (randomization.py:224-238); state [N,4] = (level,
// successes_at_level, episodes, total_successes)
static __global__ void curriculum_kernel(int64_t n, int64_t *state, const uint8_t *success,
                                  int64_t max_level, int64_t threshold) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int64_t *s = state + 4 * i;
    s[2] += 1;
    if (!success[i]) return;
    const int64_t succ = s[1] + 1;
    if (succ >= threshold && s[0] < max_level) {
        s[0] += 1;
        s[1] = 0;
    } else {
        s[1] = succ;
    }
    s[3] += 1;
}

}  // namespace dk

namespace dk {

template <typename T>
cudaError_t launch_loco_tail(const LocoFrames<T> &f, const T *prev_action, const T *command,
                             const T *pert, const RewardCfg<T> &c, const LocoArgs &a,
                             const LocoOut<T> &out, unsigned long long *err, cudaStream_t st) {
    const int64_t rows = a.K * a.N;
    if (rows == 0) return cudaSuccess;
    const int P = 9 + 3 * a.nj + 3 + 2 * a.nf + a.nf + a.nj + 3;
    const size_t per_warp = (size_t)32 * P * sizeof(T);
    int warps = 4;
    while (warps > 1 && warps * per_warp > 200 * 1024) warps /= 2;
    const size_t smem = warps * per_warp;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(loco_tail_kernel<T>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
    }
    const int bs = 32 * warps;
    loco_tail_kernel<T><<<(unsigned)((rows + bs - 1) / bs), bs, smem, st>>>(
        f, prev_action, command, pert, c, a, out, err);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_pd(int64_t n, int nj, T kp, T kd, T scale, T limit, T lo, T hi, int relative,
                      const T *q_default, const T *a, const T *prev, const T *q, const T *v,
                      T *target, T *torque, cudaStream_t st) {
    const int64_t m = n * nj;
    if (m == 0) return cudaSuccess;
    pd_kernel<T><<<(unsigned)((m + 255) / 256), 256, 0, st>>>(n, nj, kp, kd, scale, limit, lo, hi,
                                                             relative, q_default, a, prev, q, v,
                                                             target, torque);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_phase(int64_t n, int nf, const T *phi, const T *freq, const T *dt, T *out_phi,
                         T *out_cs, cudaStream_t st) {
    const int64_t m = n * nf;
    if (m == 0) return cudaSuccess;
    phase_kernel<T><<<(unsigned)((m + 255) / 256), 256, 0, st>>>(n, nf, phi, freq, dt, out_phi,
                                                                out_cs);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_progress(int64_t n, const T *raw, T *hist, T *reward, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    progress_kernel<T><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, raw, hist, reward);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_sensor_noise(int64_t n, int dim, T *obs, int nspec, const int *off,
                                const int *len, const double *scale, const int *kind,
                                uint64_t seed, int64_t env0, const uint32_t *episode,
                                uint64_t step, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    sensor_noise_warp_kernel<T><<<(unsigned)((n * 32 + 127) / 128), 128, 0, st>>>(
        n, dim, obs, nspec, off, len, scale, kind, seed, env0, episode, step);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_delay_push_pop(int64_t n, int dim, int min_delay, int max_delay, int per_step,
                                  T *ring, int32_t *head, int32_t *count, const int32_t *delay,
                                  uint64_t seed, int64_t env0, const uint32_t *episode,
                                  uint64_t step, const T *value, T *out, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    delay_push_pop_kernel<T><<<(unsigned)((n + 127) / 128), 128, 0, st>>>(
        n, dim, min_delay, max_delay, per_step, ring, head, count, delay, seed, env0, episode,
        step, value, out);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_pose_injection(int64_t n, int dim, T *pose, const double *bounds, double prob,
                                  uint64_t seed, int64_t env0, const uint32_t *episode,
                                  uint64_t step, uint8_t *injected, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    pose_injection_kernel<T><<<(unsigned)((n + 127) / 128), 128, 0, st>>>(
        n, dim, pose, bounds, prob, seed, env0, episode, step, injected);
    return cudaGetLastError();
}

#define DK_LOCO_LAUNCHERS(EXT, T)                                                                \
    EXT template cudaError_t launch_loco_tail<T>(const LocoFrames<T> &, const T *, const T *,    \
                                                 const T *, const RewardCfg<T> &,               \
                                                 const LocoArgs &, const LocoOut<T> &,          \
                                                 unsigned long long *, cudaStream_t);           \
    EXT template cudaError_t launch_pd<T>(int64_t, int, T, T, T, T, T, T, int, const T *,        \
                                          const T *, const T *, const T *, const T *, T *, T *, \
                                          cudaStream_t);                                        \
    EXT template cudaError_t launch_phase<T>(int64_t, int, const T *, const T *, const T *, T *, \
                                             T *, cudaStream_t);                                \
    EXT template cudaError_t launch_progress<T>(int64_t, const T *, T *, T *, cudaStream_t);     \
    EXT template cudaError_t launch_sensor_noise<T>(int64_t, int, T *, int, const int *,         \
                                                    const int *, const double *, const int *,    \
                                                    uint64_t, int64_t, const uint32_t *,        \
                                                    uint64_t, cudaStream_t);                    \
    EXT template cudaError_t launch_delay_push_pop<T>(int64_t, int, int, int, int, T *, int32_t *,  \
                                                      int32_t *, const int32_t *, uint64_t,      \
                                                      int64_t, const uint32_t *, uint64_t,       \
                                                      const T *, T *, cudaStream_t);             \
    EXT template cudaError_t launch_pose_injection<T>(int64_t, int, T *, const double *, double, \
                                                      uint64_t, int64_t, const uint32_t *,      \
                                                      uint64_t, uint8_t *, cudaStream_t);

}  // namespace dk
