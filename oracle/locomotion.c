/*
 * locomotion.c -- CPU restatement of the reference's locomotion step tail.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.c).  Restates, in float64:
 *   rewards.py:92-211      swing_height_profile, the 16 reward terms, total_reward
 *   envkit.py:111-131      action_to_target, pd_torque
 *   envkit.py:147-193      build_locomotion_observation (+ Philox-keyed uniform noise)
 *   envkit.py:196-202      progress_clip_reward
 *   mathcore.py:42-97      quat_check_unit, quat_mul/conj/rotate, project_gravity
 *   mathcore.py:143-177    wrap_angle, advance_phase, phase_encode
 *   randomization.py:27-62   DelayLine (reset / push_pop) with Generator.integers
 *   randomization.py:88-108  apply_sensor_noise, uniform and gaussian kinds
 *   randomization.py:156-181 randomize_params (additive / multiplicative / log-uniform,
 *                            positivity resampling, <= 100 tries)
 *   randomization.py:188-199, 224-238  pose injection, curriculum_update
 * NumPy dependencies restated (NumPy 2.3, numpy/random/src/distributions/):
 *   Generator.normal    = loc + scale * random_standard_normal (256-layer ziggurat,
 *                         tables in paper_2502_08844_b200/csrc/ziggurat_tables.h,
 *                         generated and checked by tools/gen_ziggurat_tables.py)
 *   Generator.integers  = random_bounded_uint64_fill: Lemire's nearly-divisionless
 *                         method on next_uint32 (Philox keeps the unused high half of
 *                         a 64-bit word for the next 32-bit draw) or next_uint64
 * Parity: pinned against tests/golden/loco_golden.npz (generated from the reference
 * by tests/golden/make_golden_loco.py).  Integer / selection logic is bit-exact;
 * sums of products are sequential here, where NumPy uses BLAS dot / pairwise sums
 * and SIMD sin/cos, so those agree to a few ulps (tolerance in the tests).
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

/* from oracle.c */
typedef struct {
    uint64_t ctr[4];
    uint64_t key[2];
    uint64_t buf[4];
    int pos;
} orc_philox_state;
void orc_philox_block(const uint64_t ctr_in[4], const uint64_t key_in[2], uint64_t out[4]);

static void px_init(orc_philox_state *p, uint64_t seed, uint64_t env, int64_t ep, uint64_t step) {
    p->key[0] = seed;
    p->key[1] = (env << 32) | ((uint64_t)ep & 0xFFFFFFFFULL);
    p->ctr[0] = step; p->ctr[1] = p->ctr[2] = p->ctr[3] = 0;
    p->pos = 4;
}
static uint64_t px_next(orc_philox_state *p) {
    if (p->pos < 4) return p->buf[p->pos++];
    if (++p->ctr[0] == 0)
        if (++p->ctr[1] == 0)
            if (++p->ctr[2] == 0) ++p->ctr[3];
    orc_philox_block(p->ctr, p->key, p->buf);
    p->pos = 1;
    return p->buf[0];
}
static double px_uniform(orc_philox_state *p, double lo, double hi) {
    double range = hi - lo;
    return lo + range * ((double)(px_next(p) >> 11) * (1.0 / 9007199254740992.0));
}
static double px_double(orc_philox_state *p) {
    return (double)(px_next(p) >> 11) * (1.0 / 9007199254740992.0);
}

#define DK_ZIG_QUAL static const
#include "../paper_2502_08844_b200/csrc/ziggurat_tables.h"

/* random_standard_normal (distributions.c) */
static double px_normal(orc_philox_state *p) {
    for (;;) {
        uint64_t r = px_next(p);
        const int idx = (int)(r & 0xff);
        r >>= 8;
        const int sign = (int)(r & 1);
        const uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
        double x = (double)rabs * dk_zig_wi[idx];
        if (sign) x = -x;
        if (rabs < dk_zig_ki[idx]) return x;
        if (idx == 0) {
            for (;;) {
                const double xx = -DK_ZIG_NOR_INV_R * log1p(-px_double(p));
                const double yy = -log1p(-px_double(p));
                if (yy + yy > xx * xx)
                    return ((rabs >> 8) & 1) ? -(DK_ZIG_NOR_R + xx) : DK_ZIG_NOR_R + xx;
            }
        } else {
            if (((dk_zig_fi[idx - 1] - dk_zig_fi[idx]) * px_double(p) + dk_zig_fi[idx]) <
                exp(-0.5 * x * x))
                return x;
        }
    }
}

/* Generator.integers(low, high) (high exclusive): random_bounded_uint64_fill */
typedef struct {
    orc_philox_state px;
    int has32;
    uint32_t u32;
} orc_px32;
static uint32_t px_next32(orc_px32 *p) {
    if (p->has32) {
        p->has32 = 0;
        return p->u32;
    }
    const uint64_t v = px_next(&p->px);
    p->has32 = 1;
    p->u32 = (uint32_t)(v >> 32);
    return (uint32_t)v;
}
static int64_t px_integers(orc_px32 *p, int64_t low, int64_t high) {
    const uint64_t rng = (uint64_t)(high - 1 - low);
    if (rng == 0) return low;
    if (rng <= 0xFFFFFFFFULL) {
        if (rng == 0xFFFFFFFFULL) return low + (int64_t)px_next32(p);
        const uint32_t excl = (uint32_t)rng + 1u;
        uint64_t m = (uint64_t)px_next32(p) * excl;
        uint32_t left = (uint32_t)m;
        if (left < excl) {
            const uint32_t thr = (uint32_t)(0xFFFFFFFFu - (uint32_t)rng) % excl;
            while (left < thr) {
                m = (uint64_t)px_next32(p) * excl;
                left = (uint32_t)m;
            }
        }
        return low + (int64_t)(m >> 32);
    }
    if (rng == 0xFFFFFFFFFFFFFFFFULL) return low + (int64_t)px_next(&p->px);
    const uint64_t excl = rng + 1;
    uint64_t x = px_next(&p->px);
    uint64_t left = x * excl;
    if (left < excl) {
        const uint64_t thr = (0xFFFFFFFFFFFFFFFFULL - rng) % excl;
        while (left < thr) {
            x = px_next(&p->px);
            left = x * excl;
        }
    }
    return low + (int64_t)(uint64_t)(((unsigned __int128)x * excl) >> 64);
}

/* RewardTermConfig, rewards.py:51-75, field order preserved */
typedef struct {
    double w_lin_vel, sigma_lin_vel, w_ang_vel, sigma_ang_vel, w_airtime, airtime_min,
        airtime_max, w_clearance, w_phase, sigma_phase, swing_height, w_slip, w_orientation,
        w_torque, w_joint_pos, w_action_rate, w_energy, w_pose, w_termination, w_standstill,
        w_lin_vel_z, w_ang_vel_xy;
    int32_t standstill_gated;
} orc_reward_cfg;

/* Batched frames: every field row-major [N, dim]; nominal / default may be
 * broadcast ([dim], stride 0). */
typedef struct {
    const double *base_orientation, *base_lin_vel, *base_ang_vel, *joint_pos, *joint_vel,
        *joint_torque, *foot_height, *foot_height_des, *foot_vel_xy;
    const uint8_t *foot_contact;
    const double *airtime;
    const uint8_t *touchdown;
    const double *phase, *command, *action, *prev_action, *joint_nominal, *joint_default;
    const uint8_t *done;
    int64_t nominal_stride, default_stride;
} orc_frames;

/* mathcore.py:42-48 + 51-61 + 64-66 + 76-79 + 93-97 */
static int project_gravity(const double *q, double *out) {
    double n = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    if (fabs(n - 1.0) > 1e-6) return 0; /* quaternion is not unit length */
    double c[4] = {q[0], -q[1], -q[2], -q[3]};        /* quat_conj(q) */
    double p[4] = {0.0, 0.0, 0.0, -1.0};              /* [0, GRAVITY_DIR] */
    double a[4], r[4];
    /* quat_mul(c, p) */
    a[0] = c[0] * p[0] - c[1] * p[1] - c[2] * p[2] - c[3] * p[3];
    a[1] = c[0] * p[1] + c[1] * p[0] + c[2] * p[3] - c[3] * p[2];
    a[2] = c[0] * p[2] - c[1] * p[3] + c[2] * p[0] + c[3] * p[1];
    a[3] = c[0] * p[3] + c[1] * p[2] - c[2] * p[1] + c[3] * p[0];
    double cc[4] = {c[0], -c[1], -c[2], -c[3]};       /* quat_conj(c) */
    r[0] = a[0] * cc[0] - a[1] * cc[1] - a[2] * cc[2] - a[3] * cc[3];
    r[1] = a[0] * cc[1] + a[1] * cc[0] + a[2] * cc[3] - a[3] * cc[2];
    r[2] = a[0] * cc[2] - a[1] * cc[3] + a[2] * cc[0] + a[3] * cc[1];
    r[3] = a[0] * cc[3] + a[1] * cc[2] - a[2] * cc[1] + a[3] * cc[0];
    double m = sqrt(r[1] * r[1] + r[2] * r[2] + r[3] * r[3]);
    out[0] = r[1] / m; out[1] = r[2] / m; out[2] = r[3] / m;
    return 1;
}

int orc_project_gravity(int64_t n, const double *q, double *out, uint8_t *ok) {
    int bad = 0;
    for (int64_t i = 0; i < n; ++i) {
        ok[i] = (uint8_t)project_gravity(q + 4 * i, out + 3 * i);
        bad += !ok[i];
    }
    return bad;
}

/* rewards.py:97-211.  terms [N,16] in TERM_REGISTRY order; returns the index of the
 * first frame with a non-unit quaternion, or -1. */
int64_t orc_total_reward(int64_t n, int nj, int nf, const orc_reward_cfg *c,
                         const orc_frames *f, double *terms, double *unclipped, double *total) {
    int64_t first_bad = n;
#pragma omp parallel for schedule(static) reduction(min : first_bad)
    for (int64_t i = 0; i < n; ++i) {
        const double *lin = f->base_lin_vel + 3 * i, *ang = f->base_ang_vel + 3 * i;
        const double *cmd = f->command + 3 * i;
        const double *jp = f->joint_pos + nj * i, *jv = f->joint_vel + nj * i;
        const double *jt = f->joint_torque + nj * i;
        const double *fh = f->foot_height + nf * i, *fhd = f->foot_height_des + nf * i;
        const double *fv = f->foot_vel_xy + 2 * nf * i, *air = f->airtime + nf * i;
        const double *ph = f->phase + nf * i;
        const uint8_t *con = f->foot_contact + nf * i, *td = f->touchdown + nf * i;
        const double *act = f->action + nj * i, *pact = f->prev_action + nj * i;
        const double *nom = f->joint_nominal + f->nominal_stride * i;
        const double *def = f->joint_default + f->default_stride * i;
        double t[16];
        double e0 = cmd[0] - lin[0], e1 = cmd[1] - lin[1];
        t[0] = exp(-(e0 * e0 + e1 * e1) / c->sigma_lin_vel);
        double ea = cmd[2] - ang[2];
        t[1] = exp(-(ea * ea) / c->sigma_ang_vel);
        double s = 0.0;
        for (int k = 0; k < nf; ++k) {
            double gain = (air[k] - c->airtime_min) * (td[k] ? 1.0 : 0.0);
            double hi = c->airtime_max - c->airtime_min;
            gain = gain < 0.0 ? 0.0 : (gain > hi ? hi : gain);
            s += gain;
        }
        t[2] = s;
        s = 0.0;
        for (int k = 0; k < nf; ++k) {
            double err = fh[k] - fhd[k];
            double sp = sqrt(fv[2 * k] * fv[2 * k] + fv[2 * k + 1] * fv[2 * k + 1]);
            s += err * err * sqrt(sp);
        }
        t[3] = s;
        s = 0.0;
        for (int k = 0; k < nf; ++k) {
            double sn = sin(ph[k]);
            double tgt = c->swing_height * (sn > 0.0 ? sn : 0.0);
            double d = fh[k] - tgt;
            s += d * d;
        }
        t[4] = exp(-s / c->sigma_phase);
        s = 0.0;
        for (int k = 0; k < nf; ++k) {
            double m = con[k] ? 1.0 : 0.0;
            double a = fv[2 * k] * m, b = fv[2 * k + 1] * m;
            s += a * a + b * b;
        }
        t[5] = s;
        double g[3];
        if (!project_gravity(f->base_orientation + 4 * i, g)) {
            if (i < first_bad) first_bad = i;
            g[0] = g[1] = g[2] = NAN;
        }
        t[6] = g[0] * g[0] + g[1] * g[1];
        double tt = 0.0, jpos = 0.0, ar = 0.0, en = 0.0, pose = 0.0, vv = 0.0;
        for (int j = 0; j < nj; ++j) {
            tt += jt[j] * jt[j];
            double d1 = jp[j] - nom[j];
            jpos += d1 * d1;
            double d2 = act[j] - pact[j];
            ar += d2 * d2;
            en += fabs(jv[j] * jt[j]);
            double d3 = jp[j] - def[j];
            pose += d3 * d3;
            vv += jv[j] * jv[j];
        }
        t[7] = tt; t[8] = jpos; t[9] = ar; t[10] = en;
        t[11] = exp(-pose);
        t[12] = f->done[i] ? 1.0 : 0.0;
        double cn = sqrt(cmd[0] * cmd[0] + cmd[1] * cmd[1]);
        t[13] = !c->standstill_gated ? cn : (cn > 0.1 ? 0.0 : sqrt(vv));
        t[14] = lin[2] * lin[2];
        t[15] = ang[0] * ang[0] + ang[1] * ang[1];
        const double w[16] = {c->w_lin_vel, c->w_ang_vel, c->w_airtime, c->w_clearance,
                              c->w_phase, c->w_slip, c->w_orientation, c->w_torque,
                              c->w_joint_pos, c->w_action_rate, c->w_energy, c->w_pose,
                              c->w_termination, c->w_standstill, c->w_lin_vel_z,
                              c->w_ang_vel_xy};
        double u = 0.0;
        for (int k = 0; k < 16; ++k) {
            terms[16 * i + k] = t[k];
            u += w[k] * t[k];
        }
        unclipped[i] = u;
        total[i] = 0.0 > u ? 0.0 : u;  /* max(unclipped, 0.0) */
    }
    return first_bad == n ? -1 : first_bad;
}

/* envkit.py:147-193.  state [N, 9 + 3*nj + 3 + 2*nf], priv [N, state + nf + nj + 3].
 * noise[5] = (gravity, lin_vel, ang_vel, joint_pos, joint_vel) scales; the stream of
 * world i is stream_rng(seed, env0 + i, episode, step).  pert [N,3] or NULL. */
int64_t orc_loco_obs(int64_t n, int nj, int nf, const orc_frames *f, const double *prev_action,
                     const double *command, const double *noise, uint64_t seed, int64_t env0,
                     int64_t episode, uint64_t step, const double *pert, double *state,
                     double *priv) {
    const int S = 9 + 3 * nj + 3 + 2 * nf, P = S + nf + nj + 3;
    int64_t first_bad = n;
#pragma omp parallel for schedule(static) reduction(min : first_bad)
    for (int64_t i = 0; i < n; ++i) {
        double clean[512];
        int o = 0;
        if (!project_gravity(f->base_orientation + 4 * i, clean)) {
            if (i < first_bad) first_bad = i;
            clean[0] = clean[1] = clean[2] = NAN;
        }
        o = 3;
        for (int k = 0; k < 3; ++k) clean[o++] = f->base_lin_vel[3 * i + k];
        for (int k = 0; k < 3; ++k) clean[o++] = f->base_ang_vel[3 * i + k];
        for (int k = 0; k < nj; ++k) clean[o++] = f->joint_pos[nj * i + k];
        for (int k = 0; k < nj; ++k) clean[o++] = f->joint_vel[nj * i + k];
        for (int k = 0; k < nj; ++k) clean[o++] = prev_action[nj * i + k];
        for (int k = 0; k < 3; ++k) clean[o++] = command[3 * i + k];
        for (int k = 0; k < nf; ++k) {
            clean[o++] = cos(f->phase[nf * i + k]);
            clean[o++] = sin(f->phase[nf * i + k]);
        }
        double *st = state + (int64_t)S * i;
        memcpy(st, clean, sizeof(double) * S);
        if (noise) {
            orc_philox_state px;
            px_init(&px, seed, (uint64_t)(env0 + i), episode, step);
            const int start[5] = {0, 3, 6, 9, 9 + nj}, len[5] = {3, 3, 3, nj, nj};
            for (int g = 0; g < 5; ++g) {
                double s = noise[g];
                if (s > 0)
                    for (int k = 0; k < len[g]; ++k)
                        st[start[g] + k] = st[start[g] + k] + px_uniform(&px, -s, s);
            }
        }
        double *pr = priv + (int64_t)P * i;
        memcpy(pr, clean, sizeof(double) * S);
        o = S;
        for (int k = 0; k < nf; ++k) pr[o++] = f->foot_contact[nf * i + k] ? 1.0 : 0.0;
        for (int k = 0; k < nj; ++k) pr[o++] = f->joint_torque[nj * i + k];
        for (int k = 0; k < 3; ++k) pr[o++] = pert ? pert[3 * i + k] : 0.0;
    }
    return first_bad == n ? -1 : first_bad;
}

/* envkit.py:111-131.  params = (kp, kd, action_scale, torque_limit, range_lo, range_hi,
 * relative); q_default [nj]. */
void orc_pd(int64_t n, int nj, const double *params, const double *q_default, const double *a,
            const double *prev_target, const double *q, const double *v, double *target,
            double *torque) {
    double kp = params[0], kd = params[1], sc = params[2], lim = params[3];
    double lo = params[4], hi = params[5];
    int rel = params[6] != 0.0;
    for (int64_t i = 0; i < n; ++i)
        for (int j = 0; j < nj; ++j) {
            int64_t e = i * nj + j;
            double t;
            if (!rel) {
                t = q_default[j] + sc * a[e];
            } else {
                t = prev_target[e] + sc * a[e];
                t = t < lo ? lo : t;  /* np.clip = minimum(maximum(x, lo), hi) */
                t = t > hi ? hi : t;
            }
            target[e] = t;
            double tau = kp * (t - q[e]) - kd * v[e];
            tau = tau < -lim ? -lim : tau;
            tau = tau > lim ? lim : tau;
            torque[e] = tau;
        }
}

/* envkit.py:196-202 */
void orc_progress_clip(int64_t n, const double *raw, const double *hist, double *reward,
                       double *new_hist) {
    for (int64_t i = 0; i < n; ++i) {
        double d = raw[i] - hist[i];
        reward[i] = 0.0 > d ? 0.0 : d;          /* max(raw - hist, 0.0) */
        new_hist[i] = raw[i] > hist[i] ? raw[i] : hist[i];  /* max(hist, raw) */
    }
}

/* mathcore.py:143-177 */
static double wrap(double phi) {
    const double two_pi = 2.0 * M_PI;
    double x = phi + M_PI;
    double m = fmod(x, two_pi);  /* npy_divmod: result takes the divisor's sign */
    if (m != 0.0) {
        if ((m < 0) != (two_pi < 0)) m += two_pi;
    } else {
        m = copysign(0.0, two_pi);
    }
    return m - M_PI;
}
void orc_wrap_angle(int64_t n, const double *in, double *out) {
    for (int64_t i = 0; i < n; ++i) out[i] = wrap(in[i]);
}
void orc_advance_phase(int64_t n, int nf, const double *phi, const double *freq,
                       const double *dt, double *out) {
    const double two_pi = 2.0 * M_PI;
    for (int64_t i = 0; i < n; ++i)
        for (int k = 0; k < nf; ++k) out[i * nf + k] = wrap(phi[i * nf + k] + two_pi * freq[i] * dt[i]);
}

/* randomization.py:88-108 (uniform kind): specs given as (offset, length, scale) triples
 * over one flat observation row; stream of row i = stream_rng(seed, env0 + i, ep, step). */
void orc_sensor_noise(int64_t n, int dim, const double *obs, int nspec, const int32_t *spec_off,
                      const int32_t *spec_len, const double *spec_scale,
                      const int32_t *spec_kind /* 0 uniform, 1 gaussian; NULL = uniform */,
                      uint64_t seed, int64_t env0, int64_t episode, uint64_t step, double *out) {
    for (int64_t i = 0; i < n; ++i) {
        memcpy(out + (int64_t)dim * i, obs + (int64_t)dim * i, sizeof(double) * dim);
        orc_philox_state px;
        px_init(&px, seed, (uint64_t)(env0 + i), episode, step);
        for (int s = 0; s < nspec; ++s) {
            double sc = spec_scale[s];
            if (sc == 0.0) continue;
            for (int k = 0; k < spec_len[s]; ++k) {
                double *x = out + (int64_t)dim * i + spec_off[s] + k;
                if (spec_kind && spec_kind[s] == 1)
                    *x = *x + (0.0 + sc * px_normal(&px));  /* Generator.normal(0, sc) */
                else
                    *x = *x + px_uniform(&px, -sc, sc);
            }
        }
    }
}

/* randomize_params (randomization.py:156-181) for n worlds: nominal [F];
 * ranges (field, distribution 0 additive / 1 multiplicative / 2 log-uniform,
 * low, high) in spec order; out [n, F].  Returns -1, or the first world whose
 * field could not be drawn positive in 100 tries (ConfigError). */
int64_t orc_randomize_params(int64_t n, int nf, const double *nominal, int nr, const int32_t *field,
                             const int32_t *dist, const double *low, const double *high,
                             uint64_t seed, int64_t env0, int64_t episode, uint64_t step,
                             double *out) {
    int64_t fail = -1;
    for (int64_t i = 0; i < n; ++i) {
        double *o = out + i * nf;
        memcpy(o, nominal, sizeof(double) * nf);
        orc_philox_state px;
        px_init(&px, seed, (uint64_t)(env0 + i), episode, step);
        for (int r = 0; r < nr; ++r) {
            const double base = nominal[field[r]];
            const int positive = base > 0;
            double value = 0.0;
            int ok = 0;
            for (int attempt = 0; attempt < 100; ++attempt) {
                if (dist[r] == 0)
                    value = base + px_uniform(&px, low[r], high[r]);
                else if (dist[r] == 1)
                    value = base * px_uniform(&px, low[r], high[r]);
                else
                    value = base * exp(px_uniform(&px, log(low[r]), log(high[r])));
                if (!positive || value > 0) {
                    ok = 1;
                    break;
                }
            }
            if (!ok && fail < 0) fail = i;
            o[field[r]] = value;
        }
    }
    return fail;
}

/* DelayLine (randomization.py:27-62), batched: ring [n, cap, dim] with
 * cap = max_delay + 1, head = next write slot, count = items held.
 * reset: count = head = 0 and, per world, delay = integers(min, max + 1) from
 * the world's stream (randomization.py:44-46). */
void orc_delay_reset(int64_t n, int min_delay, int max_delay, uint64_t seed, int64_t env0,
                     int64_t episode, uint64_t step, int32_t *delay, int32_t *count,
                     int32_t *head) {
    for (int64_t i = 0; i < n; ++i) {
        orc_px32 p;
        px_init(&p.px, seed, (uint64_t)(env0 + i), episode, step);
        p.has32 = 0;
        delay[i] = (int32_t)px_integers(&p, min_delay, (int64_t)max_delay + 1);
        count[i] = 0;
        head[i] = 0;
    }
}

/* push_pop (randomization.py:56-62): append value, draw the delay per step (or
 * use the episode's), return the element len-1-d (clamped to the oldest). */
void orc_delay_push_pop(int64_t n, int dim, int min_delay, int max_delay, int per_step,
                        double *ring, int32_t *head, int32_t *count, const int32_t *delay,
                        uint64_t seed, int64_t env0, int64_t episode, uint64_t step,
                        const double *value, double *out) {
    const int cap = max_delay + 1;
    for (int64_t i = 0; i < n; ++i) {
        double *rb = ring + i * (int64_t)cap * dim;
        memcpy(rb + (int64_t)head[i] * dim, value + i * dim, sizeof(double) * dim);
        head[i] = (head[i] + 1) % cap;
        if (count[i] < cap) count[i] += 1;
        int d = delay[i];
        if (per_step) {
            orc_px32 p;
            px_init(&p.px, seed, (uint64_t)(env0 + i), episode, step);
            p.has32 = 0;
            d = (int)px_integers(&p, min_delay, (int64_t)max_delay + 1);
        }
        int idx = count[i] - 1 - d;
        if (idx < 0) idx = 0;
        const int slot = ((head[i] - count[i] + idx) % cap + cap) % cap;
        memcpy(out + i * dim, rb + (int64_t)slot * dim, sizeof(double) * dim);
    }
}

/* Generator.standard_normal / integers on one stream (oracle self-checks) */
void orc_stream_normal(uint64_t seed, uint64_t env, int64_t episode, uint64_t step, int64_t count,
                       double *out) {
    orc_philox_state px;
    px_init(&px, seed, env, episode, step);
    for (int64_t k = 0; k < count; ++k) out[k] = px_normal(&px);
}
void orc_stream_integers(uint64_t seed, uint64_t env, int64_t episode, uint64_t step,
                         int64_t low, int64_t high, int64_t count, int64_t *out) {
    orc_px32 p;
    px_init(&p.px, seed, env, episode, step);
    p.has32 = 0;
    for (int64_t k = 0; k < count; ++k) out[k] = px_integers(&p, low, high);
}

/* randomization.py:188-199 */
void orc_pose_injection(int64_t n, int dim, const double *pose, const double *bounds /*[dim,2]*/,
                        double prob, uint64_t seed, int64_t env0, int64_t episode,
                        uint64_t step, double *out) {
    for (int64_t i = 0; i < n; ++i) {
        orc_philox_state px;
        px_init(&px, seed, (uint64_t)(env0 + i), episode, step);
        if (px_uniform(&px, 0.0, 1.0) < prob) {
            for (int k = 0; k < dim; ++k)
                out[i * dim + k] = px_uniform(&px, bounds[2 * k], bounds[2 * k + 1]);
        } else {
            memcpy(out + i * dim, pose + i * dim, sizeof(double) * dim);
        }
    }
}

/* randomization.py:206-238: state = (level, successes_at_level, episodes,
 * total_successes); cfg = (max_level, promotion_threshold). */
void orc_curriculum(int64_t n, int64_t *state, const uint8_t *success, int64_t max_level,
                    int64_t threshold) {
    for (int64_t i = 0; i < n; ++i) {
        int64_t *s = state + 4 * i;
        s[2] += 1;
        if (!success[i]) continue;
        int64_t succ = s[1] + 1, tot = s[3] + 1;
        if (succ >= threshold && s[0] < max_level) {
            s[0] += 1;
            s[1] = 0;
        } else {
            s[1] = succ;
        }
        s[3] = tot;
    }
}
