// tasks.cuh -- the four analytic tasks as device functors.
//
// Each task restates the reference's scalar task class (envkit.py:255-453)
// with the same operation order, so the f64 instantiation (built with
// --fmad=false) differs from the reference only through libm ulps.  A world
// carries its state plus the sin/cos of its angles: the reference evaluates
// the same trig of the post-step state up to three times (dynamics of the
// next step, reward, observation); here it is evaluated once per step.
//
// Interface per task:
//   A, O, I, NS              action / obs / info dims, state scalars
//   struct W                 registers of one world
//   load/store(W&, soa, i, N)  structure-of-arrays state in HBM
//   refresh(W&)              trig of the current state
//   control(a[A], P, u[A])   clipped action -> clipped force/torque (the
//                            min(max(a * limit, -limit), limit) of step_dynamics)
//   step_u(W&, u[A], P)      step_dynamics given u, + refresh
//   step(W&, a[A], P)        control + step_u
//   reward(W&, P, info[I])   reward + info terms of the current state
//   obs(W&, P, o[O])         state_obs of the current state
//   sample(W&, Philox&, P, wide)  sample_initial + refresh
#pragma once
#include <type_traits>
#include "envmath.cuh"

namespace dk {

#ifdef DK_F32_ORDER
constexpr bool kRefOrder = true;  // f32 in the reference's operation order (A/B build)
#else
constexpr bool kRefOrder = false;
#endif

// DynamicsParams (dynamics.py:40-60) in the kernel's real type.
template <typename T>
struct Params {
    T dt, gravity;
    T pend_mass, pend_length, pend_damping, pend_torque_limit;
    T cart_mass, pole_mass, pole_length, rail_limit, cart_force_limit;
    T link1_mass, link2_mass, link1_length, link2_length, link_damping;
    T elbow_torque_limit, reacher_torque_limit;
};

// ---------------------------------------------------------------------------
// PendulumSwingup (envkit.py:255-294)
template <typename T>
struct Pendulum {
    static constexpr int A = 1, O = 3, I = 1, NS = 2;
    struct W { T th, om, s, c; };
    static constexpr unsigned SLOT_FIELDS = 0xEu;  // om, s, c (reward / obs never read th)

    static __device__ __forceinline__ void load(W &w, const T *soa, int64_t i, int64_t n) {
        w.th = soa[i]; w.om = soa[n + i];
    }
    static __device__ __forceinline__ void store(const W &w, T *soa, int64_t i, int64_t n) {
        soa[i] = w.th; soa[n + i] = w.om;
    }
    static __device__ __forceinline__ void zero(W &w) { w.th = T(0); w.om = T(0); }
    static __device__ __forceinline__ void refresh(W &w) { RealOps<T>::sincos_(w.th, &w.s, &w.c); }
    static __device__ __forceinline__ void control(const T *a, const Params<T> &p, T *u) {
        u[0] = clip_sym(a[0] * p.pend_torque_limit, p.pend_torque_limit);
    }
    static __device__ __forceinline__ void step(W &w, const T *a, const Params<T> &p) {
        T u[A];
        control(a, p, u);
        step_u(w, u, p);
    }
    static __device__ __forceinline__ void step_u(W &w, const T *u, const Params<T> &p) {
        const T torque = u[0];
        const T m = p.pend_mass, l = p.pend_length;
        const T accel =
            RealOps<T>::div_(torque - p.pend_damping * w.om - m * p.gravity * l * w.s, m * l * l);
        w.om = w.om + p.dt * accel;
        w.th = w.th + p.dt * w.om;
        refresh(w);
    }
    static __device__ __forceinline__ T reward(const W &w, const Params<T> &, T *info) {
        const T r = tol<T>(-w.c, T(0.95), T(1.0), T(1.95));
        info[0] = r;
        return r;
    }
    static __device__ __forceinline__ void obs(const W &w, const Params<T> &, T *o) {
        o[0] = w.c; o[1] = w.s; o[2] = RealOps<T>::div_(w.om, T(10.0));
    }
    static __device__ __forceinline__ void sample(W &w, Philox4x64 &rng, const Params<T> &,
                                                  bool wide) {
        if (wide) {
            w.th = (T)rng.uniform(-3.141592653589793, 3.141592653589793);
            w.om = (T)rng.uniform(-6.0, 6.0);
        } else {
            w.th = (T)rng.uniform(-0.1, 0.1);
            w.om = (T)rng.uniform(-0.05, 0.05);
        }
        refresh(w);
    }
    static __device__ __forceinline__ void to_f64(const W &w, double *s4, double *t2) {
        s4[0] = w.th; s4[1] = w.om; s4[2] = 0.0; s4[3] = 0.0; t2[0] = 0.0; t2[1] = 0.0;
    }
    static __device__ __forceinline__ void from_f64(W &w, const double *s4, const double *) {
        w.th = (T)s4[0]; w.om = (T)s4[1];
    }
};

// ---------------------------------------------------------------------------
// CartpoleBalance (envkit.py:297-349)
template <typename T>
struct Cartpole {
    static constexpr int A = 1, O = 5, I = 3, NS = 4;
    struct W { T x, th, xd, thd, s, c; };
    static constexpr unsigned SLOT_FIELDS = 0x3Du;  // all but th (reward / obs use s, c)

    static __device__ __forceinline__ void load(W &w, const T *soa, int64_t i, int64_t n) {
        w.x = soa[i]; w.th = soa[n + i]; w.xd = soa[2 * n + i]; w.thd = soa[3 * n + i];
    }
    static __device__ __forceinline__ void store(const W &w, T *soa, int64_t i, int64_t n) {
        soa[i] = w.x; soa[n + i] = w.th; soa[2 * n + i] = w.xd; soa[3 * n + i] = w.thd;
    }
    static __device__ __forceinline__ void zero(W &w) { w.x = w.th = w.xd = w.thd = T(0); }
    static __device__ __forceinline__ void refresh(W &w) { RealOps<T>::sincos_(w.th, &w.s, &w.c); }
    static __device__ __forceinline__ void control(const T *a, const Params<T> &p, T *u) {
        u[0] = clip_sym(a[0] * p.cart_force_limit, p.cart_force_limit);
    }
    static __device__ __forceinline__ void step(W &w, const T *a, const Params<T> &p) {
        T u[A];
        control(a, p, u);
        step_u(w, u, p);
    }
    static __device__ __forceinline__ void step_u(W &w, const T *u, const Params<T> &p) {
        const T force = u[0];
        const T mc = p.cart_mass, mp = p.pole_mass, l = p.pole_length, g = p.gravity;
        const T m11 = mc + mp;
        const T m12 = mp * l * w.c;
        const T m22 = mp * l * l;
        const T r1 = force + mp * l * w.thd * w.thd * w.s;
        const T r2 = mp * g * l * w.s;
        const T det = m11 * m22 - m12 * m12;
        if constexpr (std::is_same<T, float>::value && !kRefOrder) {
            // f32 (tolerance-checked, not bit-exact): one reciprocal, and the
            // angle update folded as th + dt*thd + dt^2*thdd so that only one
            // FFMA follows the reciprocal on the th -> sincos -> th chain.
            const float rdet = RealOps<float>::div_(1.0f, det);
            const float nx = m22 * r1 - m12 * r2, nth = m11 * r2 - m12 * r1;
            const float dt = p.dt;
            const float thb = fmaf(dt, w.thd, w.th);
            w.xd = fmaf(dt * nx, rdet, w.xd);
            w.thd = fmaf(dt * nth, rdet, w.thd);
            w.th = fmaf(dt * dt * nth, rdet, thb);
            w.x = fmaf(dt, w.xd, w.x);
        } else {
            const T xddot = RealOps<T>::div_(m22 * r1 - m12 * r2, det);
            const T thetaddot = RealOps<T>::div_(m11 * r2 - m12 * r1, det);
            w.xd = w.xd + p.dt * xddot;
            w.thd = w.thd + p.dt * thetaddot;
            w.x = w.x + p.dt * w.xd;
            w.th = w.th + p.dt * w.thd;
        }
        // inelastic rail stop (envkit.py:330-333), branch-free; NaN passes
        // through unchanged as in the reference's if/elif
        const bool hit = fabs(w.x) > p.rail_limit;
        w.x = clamp_nan(w.x, -p.rail_limit, p.rail_limit);
        w.xd = hit ? T(0) : w.xd;
        refresh(w);
    }
    static __device__ __forceinline__ T reward(const W &w, const Params<T> &, T *info) {
        const T upright = tol<T>(w.c, T(0.95), T(1.0), T(1.95));
        const T centered = tol<T>(w.x, T(-0.25), T(0.25), T(1.55));
        const T still = T(0.5) * (T(1.0) + tol<T>(w.thd, T(-1.0), T(1.0), T(5.0)));
        info[0] = upright; info[1] = centered; info[2] = still;
        return upright * centered * still;
    }
    static __device__ __forceinline__ void obs(const W &w, const Params<T> &, T *o) {
        o[0] = w.x; o[1] = w.c; o[2] = w.s; o[3] = w.xd; o[4] = w.thd;
    }
    static __device__ __forceinline__ void sample(W &w, Philox4x64 &rng, const Params<T> &, bool) {
        w.x = (T)rng.uniform(-0.8, 0.8);
        w.th = (T)rng.uniform(-0.05, 0.05);
        w.xd = (T)rng.uniform(-0.01, 0.01);
        w.thd = (T)rng.uniform(-0.01, 0.01);
        refresh(w);
    }
    static __device__ __forceinline__ void to_f64(const W &w, double *s4, double *t2) {
        s4[0] = w.x; s4[1] = w.th; s4[2] = w.xd; s4[3] = w.thd; t2[0] = 0.0; t2[1] = 0.0;
    }
    static __device__ __forceinline__ void from_f64(W &w, const double *s4, const double *) {
        w.x = (T)s4[0]; w.th = (T)s4[1]; w.xd = (T)s4[2]; w.thd = (T)s4[3];
    }
};

// ---------------------------------------------------------------------------
// _TwoLink (envkit.py:352-380): point masses at the link ends, semi-implicit
// Euler.  Shared by AcrobotSwingup and ReacherEasy.
template <typename T>
struct TwoLinkW {
    T t1, t2, d1, d2;
    T s1, c1, s2, c2, s12, c12;  // trig of t1, t2, t1 + t2
    T tx, ty;                    // reacher target (unused by acrobot)
};

template <typename T>
__device__ __forceinline__ void twolink_refresh(TwoLinkW<T> &w) {
    RealOps<T>::sincos_(w.t1, &w.s1, &w.c1);
    RealOps<T>::sincos_(w.t2, &w.s2, &w.c2);
    if constexpr (std::is_same<T, float>::value && !kRefOrder) {
        // f32 (tolerance-checked): the sum angle by the addition formulas,
        // four FMA-pipe ops instead of a third sincos (error <= ~2 ulp)
        w.s12 = fmaf(w.s1, w.c2, w.c1 * w.s2);
        w.c12 = fmaf(w.c1, w.c2, -(w.s1 * w.s2));
    } else {
        // f64: the reference's math.sin / math.cos of t1 + t2 (envkit.py:365-366)
        RealOps<T>::sincos_(w.t1 + w.t2, &w.s12, &w.c12);
    }
}

template <typename T>
__device__ __forceinline__ void twolink_advance(TwoLinkW<T> &w, T tau1, T tau2, T gravity,
                                                const Params<T> &p) {
    const T m1 = p.link1_mass, m2 = p.link2_mass, l1 = p.link1_length, l2 = p.link2_length;
    const T d1 = w.d1, d2 = w.d2;
    const T m11 = (m1 + m2) * l1 * l1 + m2 * l2 * l2 + T(2) * m2 * l1 * l2 * w.c2;
    const T m12 = m2 * l2 * l2 + m2 * l1 * l2 * w.c2;
    const T m22 = m2 * l2 * l2;
    const T h = m2 * l1 * l2 * w.s2;
    const T cor1 = -h * (T(2) * d1 * d2 + d2 * d2);
    const T cor2 = h * d1 * d1;
    const T g1 = (m1 + m2) * gravity * l1 * w.s1 + m2 * gravity * l2 * w.s12;
    const T g2 = m2 * gravity * l2 * w.s12;
    const T rhs1 = tau1 - cor1 - g1 - p.link_damping * d1;
    const T rhs2 = tau2 - cor2 - g2 - p.link_damping * d2;
    const T det = m11 * m22 - m12 * m12;
    if constexpr (std::is_same<T, float>::value && !kRefOrder) {
        // f32 (tolerance-checked): one reciprocal; angles folded as
        // t + dt d + dt^2 a so one FFMA follows the reciprocal (as cartpole)
        const float rdet = RealOps<float>::div_(1.0f, det);
        const float n1 = m22 * rhs1 - m12 * rhs2, n2 = m11 * rhs2 - m12 * rhs1;
        const float dt = p.dt, dt2 = dt * dt;
        const float t1b = fmaf(dt, d1, w.t1), t2b = fmaf(dt, d2, w.t2);
        w.d1 = fmaf(dt * n1, rdet, d1);
        w.d2 = fmaf(dt * n2, rdet, d2);
        w.t1 = fmaf(dt2 * n1, rdet, t1b);
        w.t2 = fmaf(dt2 * n2, rdet, t2b);
    } else {
        const T a1 = RealOps<T>::div_(m22 * rhs1 - m12 * rhs2, det);
        const T a2 = RealOps<T>::div_(m11 * rhs2 - m12 * rhs1, det);
        w.d1 = d1 + p.dt * a1;
        w.d2 = d2 + p.dt * a2;
        w.t1 = w.t1 + p.dt * w.d1;
        w.t2 = w.t2 + p.dt * w.d2;
    }
    twolink_refresh(w);
}

// AcrobotSwingup (envkit.py:383-409)
template <typename T>
struct Acrobot {
    static constexpr int A = 1, O = 6, I = 1, NS = 4;
    static constexpr unsigned SLOT_FIELDS = ~0u;
    using W = TwoLinkW<T>;

    static __device__ __forceinline__ void load(W &w, const T *soa, int64_t i, int64_t n) {
        w.t1 = soa[i]; w.t2 = soa[n + i]; w.d1 = soa[2 * n + i]; w.d2 = soa[3 * n + i];
    }
    static __device__ __forceinline__ void store(const W &w, T *soa, int64_t i, int64_t n) {
        soa[i] = w.t1; soa[n + i] = w.t2; soa[2 * n + i] = w.d1; soa[3 * n + i] = w.d2;
    }
    static __device__ __forceinline__ void zero(W &w) { w.t1 = w.t2 = w.d1 = w.d2 = w.tx = w.ty = T(0); }
    static __device__ __forceinline__ void refresh(W &w) { twolink_refresh(w); }
    static __device__ __forceinline__ void control(const T *a, const Params<T> &p, T *u) {
        u[0] = clip_sym(a[0] * p.elbow_torque_limit, p.elbow_torque_limit);
    }
    static __device__ __forceinline__ void step_u(W &w, const T *u, const Params<T> &p) {
        twolink_advance(w, T(0), u[0], p.gravity, p);
    }
    static __device__ __forceinline__ void step(W &w, const T *a, const Params<T> &p) {
        T u[A];
        control(a, p, u);
        step_u(w, u, p);
    }
    static __device__ __forceinline__ T reward(const W &w, const Params<T> &p, T *info) {
        const T tip_y = -(p.link1_length * w.c1 + p.link2_length * w.c12);
        const T height = RealOps<T>::div_(tip_y, p.link1_length + p.link2_length);
        info[0] = height;
        return tol<T>(height, T(0.95), T(1.0), T(1.0));
    }
    static __device__ __forceinline__ void obs(const W &w, const Params<T> &, T *o) {
        o[0] = w.c1; o[1] = w.s1; o[2] = w.c2; o[3] = w.s2;
        o[4] = RealOps<T>::div_(w.d1, T(10.0)); o[5] = RealOps<T>::div_(w.d2, T(10.0));
    }
    static __device__ __forceinline__ void sample(W &w, Philox4x64 &rng, const Params<T> &, bool) {
        w.t1 = (T)rng.uniform(-0.1, 0.1);
        w.t2 = (T)rng.uniform(-0.1, 0.1);
        w.d1 = (T)rng.uniform(-0.05, 0.05);
        w.d2 = (T)rng.uniform(-0.05, 0.05);
        refresh(w);
    }
    static __device__ __forceinline__ void to_f64(const W &w, double *s4, double *t2) {
        s4[0] = w.t1; s4[1] = w.t2; s4[2] = w.d1; s4[3] = w.d2; t2[0] = 0.0; t2[1] = 0.0;
    }
    static __device__ __forceinline__ void from_f64(W &w, const double *s4, const double *) {
        w.t1 = (T)s4[0]; w.t2 = (T)s4[1]; w.d1 = (T)s4[2]; w.d2 = (T)s4[3];
    }
};

// ReacherEasy (envkit.py:412-453): gravity-free two-link, per-episode target.
template <typename T>
struct Reacher {
    static constexpr int A = 2, O = 10, I = 1, NS = 6;
    static constexpr unsigned SLOT_FIELDS = ~0u;
    using W = TwoLinkW<T>;

    static __device__ __forceinline__ void load(W &w, const T *soa, int64_t i, int64_t n) {
        w.t1 = soa[i]; w.t2 = soa[n + i]; w.d1 = soa[2 * n + i]; w.d2 = soa[3 * n + i];
        w.tx = soa[4 * n + i]; w.ty = soa[5 * n + i];
    }
    static __device__ __forceinline__ void store(const W &w, T *soa, int64_t i, int64_t n) {
        soa[i] = w.t1; soa[n + i] = w.t2; soa[2 * n + i] = w.d1; soa[3 * n + i] = w.d2;
        soa[4 * n + i] = w.tx; soa[5 * n + i] = w.ty;
    }
    static __device__ __forceinline__ void zero(W &w) { w.t1 = w.t2 = w.d1 = w.d2 = w.tx = w.ty = T(0); }
    static __device__ __forceinline__ void refresh(W &w) { twolink_refresh(w); }
    static __device__ __forceinline__ void control(const T *a, const Params<T> &p, T *u) {
        const T lim = p.reacher_torque_limit;
        u[0] = clip_sym(a[0] * lim, lim);
        u[1] = clip_sym(a[1] * lim, lim);
    }
    static __device__ __forceinline__ void step_u(W &w, const T *u, const Params<T> &p) {
        twolink_advance(w, u[0], u[1], T(0), p);
    }
    static __device__ __forceinline__ void step(W &w, const T *a, const Params<T> &p) {
        T u[A];
        control(a, p, u);
        step_u(w, u, p);
    }
    static __device__ __forceinline__ void tip(const W &w, const Params<T> &p, T &x, T &y) {
        x = p.link1_length * w.c1 + p.link2_length * w.c12;
        y = p.link1_length * w.s1 + p.link2_length * w.s12;
    }
    static __device__ __forceinline__ T reward(const W &w, const Params<T> &p, T *info) {
        T x, y;
        tip(w, p, x, y);
        const T dist = RealOps<T>::hypot_(x - w.tx, y - w.ty);
        info[0] = dist;
        return tol<T>(dist, T(0), T(0.1), T(0.6));
    }
    static __device__ __forceinline__ void obs(const W &w, const Params<T> &p, T *o) {
        T x, y;
        tip(w, p, x, y);
        o[0] = w.c1; o[1] = w.s1; o[2] = w.c2; o[3] = w.s2;
        o[4] = RealOps<T>::div_(w.d1, T(10.0)); o[5] = RealOps<T>::div_(w.d2, T(10.0));
        o[6] = w.tx; o[7] = w.ty; o[8] = w.tx - x; o[9] = w.ty - y;
    }
    static __device__ __forceinline__ void sample(W &w, Philox4x64 &rng, const Params<T> &, bool) {
        const double q0 = rng.uniform(-3.141592653589793, 3.141592653589793);
        const double q1 = rng.uniform(-3.141592653589793, 3.141592653589793);
        const double angle = rng.uniform(-3.141592653589793, 3.141592653589793);
        const double radius = rng.uniform(0.5, 1.9);
        double sa, ca;
        sincos(angle, &sa, &ca);
        w.t1 = (T)q0; w.t2 = (T)q1; w.d1 = T(0); w.d2 = T(0);
        w.tx = (T)__dmul_rn(radius, ca);
        w.ty = (T)__dmul_rn(radius, sa);
        refresh(w);
    }
    static __device__ __forceinline__ void to_f64(const W &w, double *s4, double *t2) {
        s4[0] = w.t1; s4[1] = w.t2; s4[2] = w.d1; s4[3] = w.d2; t2[0] = w.tx; t2[1] = w.ty;
    }
    static __device__ __forceinline__ void from_f64(W &w, const double *s4, const double *t2) {
        w.t1 = (T)s4[0]; w.t2 = (T)s4[1]; w.d1 = (T)s4[2]; w.d2 = (T)s4[3];
        w.tx = (T)t2[0]; w.ty = (T)t2[1];
    }
};

}  // namespace dk
