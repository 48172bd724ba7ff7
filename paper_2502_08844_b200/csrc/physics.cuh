// physics.cuh -- articulated contact physics step for Go1-shaped quadrupeds
// (north_star subsystems 2-5; C ABI in
// include/deskrl_b200.h "Articulated contact physics").
//
// The reference has no such code; parity is against the repo's
// own independent fp64 oracle (oracle/physics.c), labelled UNPINNED.
//
// Mapping: one QUAD of lanes per world, lane l = limb l.  The Go1 tree is a
// floating trunk with four identical 3-hinge chains, so every tree pass
// (forward kinematics, body velocities / accelerations, composite inertias,
// the recursive Newton-Euler backward pass) runs level by level down the
// lane's own chain, all four limbs of a world in parallel; trunk quantities
// are computed redundantly by the four lanes (no divergence, no hand-off)
// and every cross-limb sum is a 2-step xor-shuffle reduction
// ((l0 + l1) + (l2 + l3), identical in all four lanes).  A CTA holds 32
// worlds (128 threads); the model is staged in shared memory once per CTA.
//
// Linear algebra exploits the tree: the mass matrix (and the Newton Hessian
// M + J^T D J, since a contact on limb l touches only trunk and limb-l dofs)
// is ARROW-shaped -- four 3x3 limb blocks, 6x3 limb/trunk couplings, one 6x6
// trunk block -- so the Cholesky factorisation eliminates the limbs first
// (lane-local 3x3 factor + 6x3 solve), reduces the 6x6 Schur complement
// across the quad and factors it redundantly: no fill-in, no 18x18 dense
// factor.  Constraint rows live in shared memory, lane-major with an odd
// per-lane stride (conflict-free).  Per step: FK + RNE bias + CRB mass matrix, actuator PD,
// unconstrained acceleration, collision (floor vs trunk-box corners, thigh
// capsule ends, foot spheres), pyramidal contact rows + joint-limit rows with
// MuJoCo-style soft-constraint parameters, primal Newton with exact
// piecewise-linear line search, semi-implicit Euler.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/deskrl_b200.h"
#include "devguard.h"
#include "envmath.cuh"

namespace dk {
namespace phys {

#ifndef DK_PHYS_CTA_THREADS
#define DK_PHYS_CTA_THREADS 256
#endif
constexpr int QUAD = 4;
constexpr int THREADS = DK_PHYS_CTA_THREADS;  // largest CTA (launch bounds)
constexpr int WPC = THREADS / QUAD;           // worlds per (full) CTA
// shared memory per CTA: two CTAs per SM up to 128 threads, one above
constexpr size_t kSmemCap = THREADS >= 256 ? 220 * 1024 : 110 * 1024;
constexpr int RF = 13;             // row fields: J base 6, J limb 3, aref, D, x, y
constexpr int NS = DK_PHYS_NSENSOR;
#ifndef DK_PHYS_SYNC_LEVEL
#define DK_PHYS_SYNC_LEVEL 2  // CTA barriers per step: 1 at the start, 2 + Newton / Euler, 3 + CRB / rows
#endif

template <typename T>
struct LimbConst {
    T body_pos[3][3], axis[3][3], mass[3], ipos[3][3], inertia[3][3], range[3][2];
    T damping[3], armature[3], tlim[3], foot_pos[3];
};

template <typename T>
struct PhysConst {
    T h, g[3], mu, imp, kstiff, bdamp, rscale;  // rscale = (1 - imp) / imp
    T base_mass, base_ipos[3], base_inertia[3], base_box[3];
    T kp, kd, foot_radius, thigh_radius;
    int iterations, ls_iterations, collide_box, collide_thigh;
    int rows_per_lane;  // 4 (trunk contact) * collide_box + 4 * (2 * collide_thigh + 1) + 3
    LimbConst<T> limb[4];
};

template <typename T>
struct PhysArgs {
    int64_t n;
    int64_t num_steps;
    T *qpos;   // SoA [NQ][n]
    T *qvel;   // SoA [NV][n]
    const T *ctrl;  // [n][NU] row-major (caller layout)
    // diagnostics of the last step (nullable), caller layouts (row-major per world)
    T *qacc, *qfrc_bias, *qfrc_constraint, *act_force, *contact_dist, *contact_pos,
        *contact_force, *sensordata;
    int32_t *ncon, *contact_geom, *solver_iter;
    int32_t *bad;  // set to 1 if a factorisation broke down (non-SPD)
};

// ---------------------------------------------------------------- helpers

template <typename T> struct PMath;
template <> struct PMath<float> {
#ifndef DK_PHYS_LIBDEVICE_SINCOS
    // the branch-free sincos of the analytic tasks (envmath.cuh: 1.8e-7 abs error,
    // no Payne-Hanek slow path in the code stream): +2.5% on the Go1 env
    static __device__ __forceinline__ void sincos_(float x, float *s, float *c) { sincosf_fast(x, s, c); }
#else
    static __device__ __forceinline__ void sincos_(float x, float *s, float *c) { sincosf(x, s, c); }
#endif
    static __device__ __forceinline__ float sqrt_(float x) { return sqrtf(x); }
    static __device__ __forceinline__ float rsqrt_(float x) { return rsqrtf(x); }
};
template <> struct PMath<double> {
    static __device__ __forceinline__ void sincos_(double x, double *s, double *c) { sincos(x, s, c); }
    static __device__ __forceinline__ double sqrt_(double x) { return sqrt(x); }
    static __device__ __forceinline__ double rsqrt_(double x) { return rsqrt(x); }
};

__device__ __forceinline__ unsigned quad_mask() {
    return 0xFu << (threadIdx.x & 28u);
}

// (l0 + l1) + (l2 + l3): the same bits in all four lanes (IEEE + commutes)
template <typename T>
__device__ __forceinline__ T qsum(T v) {
    const unsigned m = quad_mask();
    v = v + __shfl_xor_sync(m, v, 1);
    return v + __shfl_xor_sync(m, v, 2);
}
__device__ __forceinline__ bool qall(bool b) {
    const unsigned m = quad_mask();
    int v = b ? 1 : 0;
    v &= __shfl_xor_sync(m, v, 1);
    v &= __shfl_xor_sync(m, v, 2);
    return v != 0;
}
__device__ __forceinline__ int qsumi(int v) {
    const unsigned m = quad_mask();
    v += __shfl_xor_sync(m, v, 1);
    return v + __shfl_xor_sync(m, v, 2);
}

template <typename T>
__device__ __forceinline__ void mat_vec3(const T *R, const T *v, T *o) {
#pragma unroll
    for (int r = 0; r < 3; ++r) o[r] = (R[3 * r] * v[0] + R[3 * r + 1] * v[1]) + R[3 * r + 2] * v[2];
}
template <typename T>
__device__ __forceinline__ void mat_tvec3(const T *R, const T *v, T *o) {
#pragma unroll
    for (int c = 0; c < 3; ++c) o[c] = (R[c] * v[0] + R[3 + c] * v[1]) + R[6 + c] * v[2];
}
template <typename T>
__device__ __forceinline__ void mat_mul3(const T *A, const T *B, T *C) {
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c)
            C[3 * r + c] = (A[3 * r] * B[c] + A[3 * r + 1] * B[3 + c]) + A[3 * r + 2] * B[6 + c];
}
template <typename T>
__device__ __forceinline__ void cross3(const T *a, const T *b, T *o) {
    o[0] = a[1] * b[2] - a[2] * b[1];
    o[1] = a[2] * b[0] - a[0] * b[2];
    o[2] = a[0] * b[1] - a[1] * b[0];
}
template <typename T>
__device__ __forceinline__ T dot3(const T *a, const T *b) {
    return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2];
}
template <typename T>
__device__ __forceinline__ T dot6(const T *a, const T *b) {
    return dot3(a, b) + dot3(a + 3, b + 3);
}
template <typename T>
__device__ __forceinline__ void quat2mat(const T *q, T *R) {
    const T q00 = q[0] * q[0], q01 = q[0] * q[1], q02 = q[0] * q[2], q03 = q[0] * q[3];
    const T q11 = q[1] * q[1], q12 = q[1] * q[2], q13 = q[1] * q[3];
    const T q22 = q[2] * q[2], q23 = q[2] * q[3], q33 = q[3] * q[3];
    R[0] = ((q00 + q11) - q22) - q33;
    R[4] = ((q00 - q11) + q22) - q33;
    R[8] = ((q00 - q11) - q22) + q33;
    R[1] = T(2) * (q12 - q03);
    R[2] = T(2) * (q13 + q02);
    R[3] = T(2) * (q12 + q03);
    R[5] = T(2) * (q23 - q01);
    R[6] = T(2) * (q13 - q02);
    R[7] = T(2) * (q23 + q01);
}
template <typename T>
__device__ __forceinline__ void axis_rot(const T *a, T q, T *R) {
    T s, c;
    PMath<T>::sincos_(q, &s, &c);
    const T t = T(1) - c;
    R[0] = t * a[0] * a[0] + c;
    R[1] = t * a[0] * a[1] - s * a[2];
    R[2] = t * a[0] * a[2] + s * a[1];
    R[3] = t * a[0] * a[1] + s * a[2];
    R[4] = t * a[1] * a[1] + c;
    R[5] = t * a[1] * a[2] - s * a[0];
    R[6] = t * a[0] * a[2] - s * a[1];
    R[7] = t * a[1] * a[2] + s * a[0];
    R[8] = t * a[2] * a[2] + c;
}

// 10-parameter spatial inertia about the trunk origin p0 (world frame):
// m, h = m (com - p0), I = I_com + m (|r|^2 1 - r r^T) as xx yy zz xy xz yz
template <typename T>
struct Inertia {
    T m, h[3], I[6];
    __device__ __forceinline__ void zero() {
        m = T(0);
#pragma unroll
        for (int i = 0; i < 3; ++i) h[i] = T(0);
#pragma unroll
        for (int i = 0; i < 6; ++i) I[i] = T(0);
    }
    __device__ __forceinline__ void add(const Inertia &o) {
        m = m + o.m;
#pragma unroll
        for (int i = 0; i < 3; ++i) h[i] = h[i] + o.h[i];
#pragma unroll
        for (int i = 0; i < 6; ++i) I[i] = I[i] + o.I[i];
    }
    __device__ __forceinline__ void qreduce() {
        m = qsum(m);
#pragma unroll
        for (int i = 0; i < 3; ++i) h[i] = qsum(h[i]);
#pragma unroll
        for (int i = 0; i < 6; ++i) I[i] = qsum(I[i]);
    }
    // rotational block times w
    __device__ __forceinline__ void Iw(const T *w, T *o) const {
        o[0] = (I[0] * w[0] + I[3] * w[1]) + I[4] * w[2];
        o[1] = (I[3] * w[0] + I[1] * w[1]) + I[5] * w[2];
        o[2] = (I[4] * w[0] + I[5] * w[1]) + I[2] * w[2];
    }
    // spatial force = this * motion [w; v]: [I w + h x v; m v - h x w]
    __device__ __forceinline__ void mul(const T *mv, T *f) const {
        T a[3], b[3], c[3];
        Iw(mv, a);
        cross3(h, mv + 3, b);
        cross3(h, mv, c);
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            f[i] = a[i] + b[i];
            f[3 + i] = m * mv[3 + i] - c[i];
        }
    }
};

// body inertia from mass, com (world) and principal inertia in a body frame R
template <typename T>
__device__ __forceinline__ void body_inertia(T mass, const T *com, const T *p0, const T *R,
                                             const T *pi, Inertia<T> &out) {
    T r[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) r[i] = com[i] - p0[i];
    // R diag(pi) R^T
    T Ic[6];
    const int ii[6] = {0, 1, 2, 0, 0, 1}, jj[6] = {0, 1, 2, 1, 2, 2};
#pragma unroll
    for (int e = 0; e < 6; ++e) {
        const int i = ii[e], j = jj[e];
        Ic[e] = (R[3 * i] * pi[0] * R[3 * j] + R[3 * i + 1] * pi[1] * R[3 * j + 1]) +
                R[3 * i + 2] * pi[2] * R[3 * j + 2];
    }
    const T rr = dot3(r, r);
    out.m = mass;
#pragma unroll
    for (int i = 0; i < 3; ++i) out.h[i] = mass * r[i];
    out.I[0] = Ic[0] + mass * (rr - r[0] * r[0]);
    out.I[1] = Ic[1] + mass * (rr - r[1] * r[1]);
    out.I[2] = Ic[2] + mass * (rr - r[2] * r[2]);
    out.I[3] = Ic[3] - mass * r[0] * r[1];
    out.I[4] = Ic[4] - mass * r[0] * r[2];
    out.I[5] = Ic[5] - mass * r[1] * r[2];
}

template <typename T>
__device__ __forceinline__ void cross_motion(const T *v, const T *u, T *o) {
    T a[3], b[3], c[3];
    cross3(v, u, a);
    cross3(v, u + 3, b);
    cross3(v + 3, u, c);
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        o[i] = a[i];
        o[3 + i] = b[i] + c[i];
    }
}
template <typename T>
__device__ __forceinline__ void cross_force(const T *v, const T *f, T *o) {
    T a[3], b[3], c[3];
    cross3(v, f, a);
    cross3(v + 3, f + 3, b);
    cross3(v, f + 3, c);
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        o[i] = a[i] + b[i];
        o[3 + i] = c[i];
    }
}

// ------------------------------------------------------- arrow factorisation
// Symmetric 18x18 matrix with limb blocks B_l (3x3), couplings C_l (6 trunk
// rows x 3 limb cols) and trunk block A (6x6).  Each lane holds its limb's
// B and C plus a redundant copy of A; factor() turns them into L_B, W and L_S
// (M = L L^T, L = [[L_B, 0], [W, L_S]]).
template <typename T>
struct Arrow {
    T B[6];      // limb block, lower: 00 10 11 20 21 22
    T C[6][3];   // coupling (trunk row, limb col)
    T A[21];     // trunk block, lower packed row-major: (i, j<=i) at i(i+1)/2 + j
    T iB[3], iA[6];  // after factor(): reciprocals of the diagonals of L_B / L_S

    static __device__ __forceinline__ int ai(int i, int j) { return i * (i + 1) / 2 + j; }

    // in place: B -> L_B, C -> W, A -> L_S; false if not positive definite.
    // One division per pivot (its reciprocal, kept in iB / iA), products
    // elsewhere: the factor and every solve multiply by the reciprocals instead of
    // dividing (IEEE division is a multi-instruction sequence on every SM pipe).
    // Apart (nullable): a lane-local addend of the trunk block, reduced across
    // the quad together with the Schur term -- A + sum_l (Apart_l - W_l W_l^T)
    // in one quad reduction per entry instead of two
    __device__ __forceinline__ bool factor(const T *Apart = nullptr) {
        bool ok = true;
        // 3x3 Cholesky of B
        // pivots: 1/l = rsqrt(s), l = s / l = s * (1/l)
        T l00 = B[0];
        ok &= l00 > T(0);
        const T i00 = PMath<T>::rsqrt_(l00);
        l00 = l00 * i00;
        const T l10 = B[1] * i00, l20 = B[3] * i00;
        T l11 = B[2] - l10 * l10;
        ok &= l11 > T(0);
        const T i11 = PMath<T>::rsqrt_(l11);
        l11 = l11 * i11;
        const T l21 = (B[4] - l20 * l10) * i11;
        T l22 = (B[5] - l20 * l20) - l21 * l21;
        ok &= l22 > T(0);
        const T i22 = PMath<T>::rsqrt_(l22);
        l22 = l22 * i22;
        B[0] = l00; B[1] = l10; B[2] = l11; B[3] = l20; B[4] = l21; B[5] = l22;
        iB[0] = i00; iB[1] = i11; iB[2] = i22;
        // W = C L_B^-T: row b solves L_B w = C_b
#pragma unroll
        for (int b = 0; b < 6; ++b) {
            const T w0 = C[b][0] * i00;
            const T w1 = (C[b][1] - l10 * w0) * i11;
            const T w2 = ((C[b][2] - l20 * w0) - l21 * w1) * i22;
            C[b][0] = w0; C[b][1] = w1; C[b][2] = w2;
        }
        // Schur complement S = A - sum_l W W^T, reduced across the quad
#pragma unroll
        for (int i = 0; i < 6; ++i)
#pragma unroll
            for (int j = 0; j <= i; ++j) {
                if (Apart) {
                    A[ai(i, j)] = A[ai(i, j)] + qsum(Apart[ai(i, j)] - dot3(C[i], C[j]));
                } else {
                    A[ai(i, j)] = A[ai(i, j)] - qsum(dot3(C[i], C[j]));
                }
            }
        // 6x6 Cholesky (redundant in all lanes).  Constant trip counts with
        // guards: LLVM unrolls inner loops first, and an inner loop whose bound
        // depends on j is left rolled ("nounroll") -- which demoted the whole
        // Arrow to local memory (608-byte stack frame, measured in the PTX)
#pragma unroll
        for (int j = 0; j < 6; ++j) {
            T s = A[ai(j, j)];
#pragma unroll
            for (int k = 0; k < 6; ++k)
                if (k < j) s = s - A[ai(j, k)] * A[ai(j, k)];
            ok &= s > T(0);
            const T id = PMath<T>::rsqrt_(s);
            const T d = s * id;
            A[ai(j, j)] = d;
            iA[j] = id;
#pragma unroll
            for (int i = 1; i < 6; ++i) {
                if (i > j) {
                    T t = A[ai(i, j)];
#pragma unroll
                    for (int k = 0; k < 6; ++k)
                        if (k < j) t = t - A[ai(i, k)] * A[ai(j, k)];
                    A[ai(i, j)] = t * id;
                }
            }
        }
        return qall(ok);
    }

    // forward half: y_l = L_B^-1 b_l (lane), y_s = L_S^-1 (b_s - sum_l W_l y_l)
    __device__ __forceinline__ void fwd(const T *bl, const T *bs, T *yl, T *ys) const {
        yl[0] = bl[0] * iB[0];
        yl[1] = (bl[1] - B[1] * yl[0]) * iB[1];
        yl[2] = ((bl[2] - B[3] * yl[0]) - B[4] * yl[1]) * iB[2];
        T r[6];
#pragma unroll
        for (int i = 0; i < 6; ++i) r[i] = bs[i] - qsum(dot3(C[i], yl));
        fwd_s(r, ys);
    }
    // lane-local variant for a row touching only limb l and the trunk:
    // the other limbs' b_l are zero, so no reduction
    __device__ __forceinline__ void fwd_local(const T *bl, const T *bs, T *yl, T *ys) const {
        yl[0] = bl[0] * iB[0];
        yl[1] = (bl[1] - B[1] * yl[0]) * iB[1];
        yl[2] = ((bl[2] - B[3] * yl[0]) - B[4] * yl[1]) * iB[2];
        T r[6];
#pragma unroll
        for (int i = 0; i < 6; ++i) r[i] = bs[i] - dot3(C[i], yl);
        fwd_s(r, ys);
    }
    __device__ __forceinline__ void fwd_s(const T *r, T *ys) const {
#pragma unroll
        for (int i = 0; i < 6; ++i) {
            T s = r[i];
#pragma unroll
            for (int k = 0; k < i; ++k) s = s - A[ai(i, k)] * ys[k];
            ys[i] = s * iA[i];
        }
    }
    // full solve M x = b (b_l per lane, b_s redundant; bs_part nullable: a
    // lane-local addend of b_s, reduced with the forward half's own reduction)
    __device__ __forceinline__ void solve(const T *bl, const T *bs, T *xl, T *xs,
                                          const T *bs_part = nullptr) const {
        T yl[3], ys[6];
        if (bs_part) {
            yl[0] = bl[0] * iB[0];
            yl[1] = (bl[1] - B[1] * yl[0]) * iB[1];
            yl[2] = ((bl[2] - B[3] * yl[0]) - B[4] * yl[1]) * iB[2];
            T r[6];
#pragma unroll
            for (int i = 0; i < 6; ++i) r[i] = bs[i] + qsum(bs_part[i] - dot3(C[i], yl));
            fwd_s(r, ys);
        } else {
            fwd(bl, bs, yl, ys);
        }
#pragma unroll
        for (int i = 5; i >= 0; --i) {
            T s = ys[i];
#pragma unroll
            for (int k = i + 1; k < 6; ++k) s = s - A[ai(k, i)] * xs[k];
            xs[i] = s * iA[i];
        }
        // x_l = L_B^-T (y_l - W^T x_s)
        T z[3];
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            T s = yl[j];
#pragma unroll
            for (int b = 0; b < 6; ++b) s = s - C[b][j] * xs[b];
            z[j] = s;
        }
        xl[2] = z[2] * iB[2];
        xl[1] = (z[1] - B[4] * xl[2]) * iB[1];
        xl[0] = ((z[0] - B[1] * xl[1]) - B[3] * xl[2]) * iB[0];
    }
};

// y = M x for an unfactored arrow matrix (x_l per lane, x_s redundant)
template <typename T>
__device__ __forceinline__ void arrow_mul(const Arrow<T> &M, const T *xl, const T *xs, T *yl,
                                          T *ys) {
    const T *B = M.B;
    yl[0] = ((B[0] * xl[0] + B[1] * xl[1]) + B[3] * xl[2]);
    yl[1] = ((B[1] * xl[0] + B[2] * xl[1]) + B[4] * xl[2]);
    yl[2] = ((B[3] * xl[0] + B[4] * xl[1]) + B[5] * xl[2]);
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        T s = T(0);
#pragma unroll
        for (int b = 0; b < 6; ++b) s = s + M.C[b][j] * xs[b];
        yl[j] = yl[j] + s;
    }
#pragma unroll
    for (int i = 0; i < 6; ++i) {
        T s = T(0);
#pragma unroll
        for (int j = 0; j < 6; ++j) s = s + M.A[i >= j ? Arrow<T>::ai(i, j) : Arrow<T>::ai(j, i)] * xs[j];
        ys[i] = s + qsum(dot3(M.C[i], xl));
    }
}

// ---------------------------------------------------------------- the step

template <typename T>
struct Lane {
    // state
    T pos[3], quat[4], q[3];    // trunk pos / quat, own limb joints
    T vlin[3], wb[3], qd[3];    // trunk lin vel (world), ang vel (trunk frame), own joint vels
    T ctrl[3];
    // per-world physical parameters (the model's, or a domain-randomised draw)
    T mu, base_mass, kp;
};

// rows in shared memory, lane-major: field f of row r of lane t at
// rows[t * S + r * RF + f], S = rows_per_lane * RF.  S is odd for every model
// (rows_per_lane = 4 box + 8 thigh + 7 is odd, RF = 13), so the 32 lanes of a
// warp hit 32 distinct banks; and per lane the fields of a row are immediate
// offsets from one row pointer (the [row][field][lane] layout this replaces
// spent 6% of the Go1 kernel's instructions on address arithmetic, ncu).
template <typename T>
struct Rows {
    T *p;  // this lane's rows
    __device__ __forceinline__ T &at(int r, int f) const { return p[r * RF + f]; }
};

enum { F_JB = 0, F_JL = 6, F_AREF = 9, F_D = 10, F_X = 11, F_Y = 12 };

// G1 inspection outputs (dk_phys_inspect): dense M [n][NV][NV] (armature, no
// implicit-damping term), qfrc_bias [n][NV], xpos / xipos [n][NBODY][3]
template <typename T>
struct PhysInspect {
    T *M, *bias, *xpos, *xipos;
    __host__ __device__ __forceinline__ bool on() const { return M || bias || xpos || xipos; }
};

// one physics step of the lane's world; returns false on a factorisation breakdown.
// With ins->on(), stops after the mass matrix and bias and writes them instead.
template <typename T>
__device__ bool phys_step(const PhysConst<T> &P, Lane<T> &L, Rows<T> rows, int lane_limb,
                          const PhysArgs<T> *dg, int64_t w, const PhysInspect<T> *ins = nullptr,
                          T *act_out = nullptr, bool cta_sync = false) {
    // CTA barriers at phase boundaries (cta_sync: CTA-uniform, every thread of
    // the CTA steps).  The step is ~240 KB of straight-line SASS and the SM
    // runs only ~2 warps per sub-partition at 8K worlds, so warps drifting
    // through different code each miss in the instruction cache ("no
    // instruction" was ~48% of stalls); aligned warps share the fetched lines
    // (measured: Go1 env 2.16e8 -> 3.12e8 physics steps/s with one barrier per
    // substep).
    auto phase_sync = [&](int level) {
        if (cta_sync && level <= DK_PHYS_SYNC_LEVEL) __syncthreads();
    };
    phase_sync(1);
    const LimbConst<T> &lm = P.limb[lane_limb];
    const T h = P.h;
    // ---------------- trunk FK and velocity (redundant in the quad)
    T R0[9];
    quat2mat(L.quat, R0);
    const T *p0 = L.pos;
    T ww[3];  // world angular velocity
    mat_vec3(R0, L.wb, ww);
    T vb[6] = {ww[0], ww[1], ww[2], L.vlin[0], L.vlin[1], L.vlin[2]};
    // trunk cdof rot axes = columns of R0 (a_i = R0 e_i)
    // cacc of the trunk: [0; -g] + sum_i cdof_dot_i w_i = [0; -g + v x w]
    T cacc_b[6];
    {
        T vxw[3];
        cross3(L.vlin, ww, vxw);
        cacc_b[0] = cacc_b[1] = cacc_b[2] = T(0);
#pragma unroll
        for (int i = 0; i < 3; ++i) cacc_b[3 + i] = vxw[i] - P.g[i];
    }
    // trunk body inertia (no reduction yet)
    Inertia<T> Ibase;
    {
        T off[3], com[3];
        mat_vec3(R0, &P.base_ipos[0], off);
#pragma unroll
        for (int i = 0; i < 3; ++i) com[i] = p0[i] + off[i];
        body_inertia(L.base_mass, com, p0, R0, P.base_inertia, Ibase);
        if (ins && lane_limb == 0)
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                if (ins->xpos) ins->xpos[w * DK_PHYS_NBODY * 3 + i] = p0[i];
                if (ins->xipos) ins->xipos[w * DK_PHYS_NBODY * 3 + i] = com[i];
            }
    }

    // ---------------- limb: FK, cdof, velocities, RNE forward, inertias
    T cdof[3][6];
    Inertia<T> Ib[3];
    T cfrc[3][6];
    T xpos1[3], xpos2[3], xpos3[3], foot[3];
    {
        T Rp[9], pp[3];
#pragma unroll
        for (int i = 0; i < 9; ++i) Rp[i] = R0[i];
#pragma unroll
        for (int i = 0; i < 3; ++i) pp[i] = p0[i];
        T vel[6], acc[6];
#pragma unroll
        for (int i = 0; i < 6; ++i) {
            vel[i] = vb[i];
            acc[i] = cacc_b[i];
        }
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            T off[3], pj[3], Rj[9], Rq[9], a[3];
            mat_vec3(Rp, lm.body_pos[j], off);
#pragma unroll
            for (int i = 0; i < 3; ++i) pj[i] = pp[i] + off[i];
            mat_vec3(Rp, lm.axis[j], a);
            axis_rot(lm.axis[j], L.q[j], Rq);
            mat_mul3(Rp, Rq, Rj);
            T rel[3], lin[3];
#pragma unroll
            for (int i = 0; i < 3; ++i) rel[i] = p0[i] - pj[i];
            cross3(a, rel, lin);
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                cdof[j][i] = a[i];
                cdof[j][3 + i] = lin[i];
            }
            // com, inertia
            T ioff[3], com[3];
            mat_vec3(Rj, lm.ipos[j], ioff);
#pragma unroll
            for (int i = 0; i < 3; ++i) com[i] = pj[i] + ioff[i];
            body_inertia(lm.mass[j], com, p0, Rj, lm.inertia[j], Ib[j]);
            if (ins) {
                const int64_t o = (w * DK_PHYS_NBODY + 1 + 3 * lane_limb + j) * 3;
#pragma unroll
                for (int i = 0; i < 3; ++i) {
                    if (ins->xpos) ins->xpos[o + i] = pj[i];
                    if (ins->xipos) ins->xipos[o + i] = com[i];
                }
            }
            // velocity, cdof_dot, acceleration, force
#pragma unroll
            for (int i = 0; i < 6; ++i) vel[i] = vel[i] + cdof[j][i] * L.qd[j];
            T cd[6];
            cross_motion(vel, cdof[j], cd);
#pragma unroll
            for (int i = 0; i < 6; ++i) acc[i] = acc[i] + cd[i] * L.qd[j];
            T Ia[6], Iv[6], vx[6];
            Ib[j].mul(acc, Ia);
            Ib[j].mul(vel, Iv);
            cross_force(vel, Iv, vx);
#pragma unroll
            for (int i = 0; i < 6; ++i) cfrc[j][i] = Ia[i] + vx[i];
            // positions kept for collision
            if (j == 1) {
#pragma unroll
                for (int i = 0; i < 3; ++i) xpos1[i] = pj[i];
            }
            if (j == 2) {
#pragma unroll
                for (int i = 0; i < 3; ++i) xpos2[i] = pj[i];
                T foff[3];
                mat_vec3(Rj, lm.foot_pos, foff);
#pragma unroll
                for (int i = 0; i < 3; ++i) foot[i] = pj[i] + foff[i];
            }
#pragma unroll
            for (int i = 0; i < 9; ++i) Rp[i] = Rj[i];
#pragma unroll
            for (int i = 0; i < 3; ++i) pp[i] = pj[i];
        }
        (void)xpos3;
    }
    // RNE backward along the limb; bias of the limb dofs
    T bias_l[3];
    T fl[6];
#pragma unroll
    for (int i = 0; i < 6; ++i) fl[i] = cfrc[2][i];
    bias_l[2] = dot6(cdof[2], fl);
#pragma unroll
    for (int i = 0; i < 6; ++i) fl[i] = cfrc[1][i] + fl[i];
    bias_l[1] = dot6(cdof[1], fl);
#pragma unroll
    for (int i = 0; i < 6; ++i) fl[i] = cfrc[0][i] + fl[i];
    bias_l[0] = dot6(cdof[0], fl);
    // trunk force: own body + sum over limbs
    T bias_s[6];
    {
        T Ia[6], Iv[6], vx[6], fb[6];
        Ibase.mul(cacc_b, Ia);
        Ibase.mul(vb, Iv);
        cross_force(vb, Iv, vx);
#pragma unroll
        for (int i = 0; i < 6; ++i) fb[i] = (Ia[i] + vx[i]) + qsum(fl[i]);
        // trans dof i: [0; e_i] -> fb.lin[i]; rot dof i: [R0 e_i; 0] -> a_i . fb.ang
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            bias_s[i] = fb[3 + i];
            bias_s[3 + i] = (R0[i] * fb[0] + R0[3 + i] * fb[1]) + R0[6 + i] * fb[2];
        }
    }

    phase_sync(3);
    // ---------------- CRB mass matrix (arrow) + armature + h * damping
    Arrow<T> M;
    {
        Inertia<T> Ic = Ib[2];
        T F[3][6];
        Ic.mul(cdof[2], F[2]);
        Ic.add(Ib[1]);
        Ic.mul(cdof[1], F[1]);
        Ic.add(Ib[0]);
        Ic.mul(cdof[0], F[0]);
        // limb block: M[j][k] = cdof_k . F_j (k <= j)
        M.B[0] = dot6(cdof[0], F[0]);
        M.B[1] = dot6(cdof[0], F[1]);
        M.B[2] = dot6(cdof[1], F[1]);
        M.B[3] = dot6(cdof[0], F[2]);
        M.B[4] = dot6(cdof[1], F[2]);
        M.B[5] = dot6(cdof[2], F[2]);
        const T hd = ins ? T(0) : h;  // inspection reports M without the implicit damping
        M.B[0] = M.B[0] + (lm.armature[0] + hd * lm.damping[0]);
        M.B[2] = M.B[2] + (lm.armature[1] + hd * lm.damping[1]);
        M.B[5] = M.B[5] + (lm.armature[2] + hd * lm.damping[2]);
        // coupling: trans b -> F.lin[b]; rot b -> a_b . F.ang
#pragma unroll
        for (int j = 0; j < 3; ++j) {
#pragma unroll
            for (int b = 0; b < 3; ++b) {
                M.C[b][j] = F[j][3 + b];
                M.C[3 + b][j] = (R0[b] * F[j][0] + R0[3 + b] * F[j][1]) + R0[6 + b] * F[j][2];
            }
        }
        // trunk composite inertia = trunk + sum over limbs of their composites
        Ic.qreduce();
        Ic.add(Ibase);
        // A: trans/trans m I; rot k/trans i: a_k . (h x e_i); rot/rot a_k . I a_i
        T a[3][3];  // a[i] = R0 e_i
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int r = 0; r < 3; ++r) a[i][r] = R0[3 * r + i];
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j <= i; ++j) M.A[Arrow<T>::ai(i, j)] = i == j ? Ic.m : T(0);
#pragma unroll
        for (int k = 0; k < 3; ++k) {
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                T e[3] = {T(0), T(0), T(0)};
                e[i] = T(1);
                T hx[3];
                cross3(Ic.h, e, hx);
                M.A[Arrow<T>::ai(3 + k, i)] = dot3(a[k], hx);
            }
            T Ia[3];
#pragma unroll
            for (int i = 0; i <= k; ++i) {
                Ic.Iw(a[i], Ia);
                M.A[Arrow<T>::ai(3 + k, 3 + i)] = dot3(a[k], Ia);
            }
        }
    }

    if (ins) {
        const int NV = DK_PHYS_NV;
        T *Mo = ins->M ? ins->M + w * NV * NV : nullptr;
        const int o = 6 + 3 * lane_limb;
        const int bi[3][3] = {{0, 1, 3}, {1, 2, 4}, {3, 4, 5}};
        if (Mo) {
            for (int j = 0; j < 3; ++j) {
                for (int k = 0; k < 3; ++k) Mo[(o + j) * NV + o + k] = M.B[bi[j][k]];
                for (int b = 0; b < 6; ++b) {
                    Mo[(o + j) * NV + b] = M.C[b][j];
                    Mo[b * NV + o + j] = M.C[b][j];
                }
                for (int l2 = 0; l2 < 4; ++l2)
                    if (l2 != lane_limb)
                        for (int k = 0; k < 3; ++k) Mo[(o + j) * NV + 6 + 3 * l2 + k] = T(0);
            }
            if (lane_limb == 0)
                for (int i = 0; i < 6; ++i)
                    for (int j = 0; j < 6; ++j)
                        Mo[i * NV + j] = M.A[i >= j ? Arrow<T>::ai(i, j) : Arrow<T>::ai(j, i)];
        }
        if (ins->bias) {
            for (int j = 0; j < 3; ++j) ins->bias[w * NV + o + j] = bias_l[j];
            if (lane_limb == 0)
                for (int i = 0; i < 6; ++i) ins->bias[w * NV + i] = bias_s[i];
        }
        return true;
    }

    // ---------------- forces
    T qf_l[3], qf_s[6], act[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        T tau = L.kp * (L.ctrl[j] - L.q[j]) - P.kd * L.qd[j];
        const T lim = lm.tlim[j];
        tau = tau < -lim ? -lim : (tau > lim ? lim : tau);
        act[j] = tau;
        if (act_out) act_out[j] = tau;
        qf_l[j] = (tau - lm.damping[j] * L.qd[j]) - bias_l[j];
    }
#pragma unroll
    for (int i = 0; i < 6; ++i) qf_s[i] = -bias_s[i];

    Arrow<T> LM = M;
    bool ok = LM.factor();
    T a_l[3], a_s[6];
    LM.solve(qf_l, qf_s, a_l, a_s);

    phase_sync(3);
    // ---------------- collision + constraint rows (lane-local)
    const T mu = L.mu;
    int nrow = 0;
    int ncon_lane = 0;
    // contact records of this lane: up to 1 trunk + 3 limb contacts
    T cdist[4], cpos[4][3];
    int cgeom[4];
    auto add_contact = [&](int geom, const T *centre, T radius, T dist, int ancestors) {
        // world point of the contact
        T p[3] = {centre[0], centre[1], centre[2] - (radius + T(0.5) * dist)};
        T r[3];
#pragma unroll
        for (int i = 0; i < 3; ++i) r[i] = p[i] - p0[i];
        // point Jacobian (trunk: trans e_i, rot a_i x r; limb dof k: lin_k + ang_k x r)
        T Jb[3][6], Jl[3][3];
#pragma unroll
        for (int i = 0; i < 3; ++i) {
#pragma unroll
            for (int c = 0; c < 3; ++c) Jb[c][i] = c == i ? T(1) : T(0);
            const T ai[3] = {R0[i], R0[3 + i], R0[6 + i]};
            T x[3];
            cross3(ai, r, x);
#pragma unroll
            for (int c = 0; c < 3; ++c) Jb[c][3 + i] = x[c];
        }
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            T x[3];
            cross3(cdof[k], r, x);
#pragma unroll
            for (int c = 0; c < 3; ++c) Jl[c][k] = k < ancestors ? cdof[k][3 + c] + x[c] : T(0);
        }
        // pyramid edges: n + mu t1, n - mu t1, n + mu t2, n - mu t2 (n = z, t1 = x, t2 = y)
        T Asum = T(0);
        T Aedge[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int tc = e < 2 ? 0 : 1;
            const T sg = (e & 1) ? -mu : mu;
            T jb[6], jl[3];
#pragma unroll
            for (int i = 0; i < 6; ++i) jb[i] = Jb[2][i] + sg * Jb[tc][i];
#pragma unroll
            for (int i = 0; i < 3; ++i) jl[i] = Jl[2][i] + sg * Jl[tc][i];
            const int rr = nrow + e;
#pragma unroll
            for (int i = 0; i < 6; ++i) rows.at(rr, F_JB + i) = jb[i];
#pragma unroll
            for (int i = 0; i < 3; ++i) rows.at(rr, F_JL + i) = jl[i];
            // J qvel: trunk dofs are (vlin, wb) in qvel order
            const T jv = ((dot3(jb, L.vlin) + dot3(jb + 3, L.wb)) + dot3(jl, L.qd));
            rows.at(rr, F_AREF) = -P.bdamp * jv - P.kstiff * P.imp * dist;
            T yl[3], ys[6];
            LM.fwd_local(jl, jb, yl, ys);
            Aedge[e] = dot3(yl, yl) + (dot3(ys, ys) + dot3(ys + 3, ys + 3));
        }
        Asum = ((Aedge[0] + Aedge[1]) + (Aedge[2] + Aedge[3])) * T(0.25);
        T R = P.rscale * Asum;
        R = R < T(1e-12) ? T(1e-12) : R;
        const T D = T(1) / R;
#pragma unroll
        for (int e = 0; e < 4; ++e) rows.at(nrow + e, F_D) = D;
        nrow += 4;
        cdist[ncon_lane] = dist;
#pragma unroll
        for (int i = 0; i < 3; ++i) cpos[ncon_lane][i] = p[i];
        cgeom[ncon_lane] = geom;
        ++ncon_lane;
    };
    // trunk box: this lane owns the lane_limb-th penetrating corner (corner order)
    int n_box = 0;
    if (P.collide_box) {
        int seen = 0;
        for (int s = 0; s < 8 && seen < 4; ++s) {
            const T loc[3] = {(s & 1) ? P.base_box[0] : -P.base_box[0],
                              (s & 2) ? P.base_box[1] : -P.base_box[1],
                              (s & 4) ? P.base_box[2] : -P.base_box[2]};
            T off[3], w[3];
            mat_vec3(R0, loc, off);
#pragma unroll
            for (int i = 0; i < 3; ++i) w[i] = p0[i] + off[i];
            if (w[2] < T(0)) {
                if (seen == lane_limb) add_contact(1, w, T(0), w[2], 0);
                ++seen;
            }
        }
        n_box = seen;
    }
    const int box_mine = ncon_lane;  // 0 or 1
    if (P.collide_thigh) {
        const T d0 = xpos1[2] - P.thigh_radius, d1 = xpos2[2] - P.thigh_radius;
        if (d0 < T(0)) add_contact(2 + 2 * lane_limb, xpos1, P.thigh_radius, d0, 2);
        if (d1 < T(0)) add_contact(2 + 2 * lane_limb, xpos2, P.thigh_radius, d1, 2);
    }
    {
        const T df = foot[2] - P.foot_radius;
        if (df < T(0)) add_contact(3 + 2 * lane_limb, foot, P.foot_radius, df, 3);
    }
    const int ncon_rows = nrow;
    // joint limits of the lane's limb
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        const T lo = L.q[j] - lm.range[j][0], hi = lm.range[j][1] - L.q[j];
#pragma unroll
        for (int side = 0; side < 2; ++side) {
            const T dist = side == 0 ? lo : hi;
            if (dist < T(0)) {
                const T s = side == 0 ? T(1) : T(-1);
#pragma unroll
                for (int i = 0; i < 6; ++i) rows.at(nrow, F_JB + i) = T(0);
#pragma unroll
                for (int i = 0; i < 3; ++i) rows.at(nrow, F_JL + i) = i == j ? s : T(0);
                const T jv = s * L.qd[j];
                rows.at(nrow, F_AREF) = -P.bdamp * jv - P.kstiff * P.imp * dist;
                T jl[3] = {T(0), T(0), T(0)}, jb[6] = {T(0), T(0), T(0), T(0), T(0), T(0)};
                jl[j] = s;
                T yl[3], ys[6];
                LM.fwd_local(jl, jb, yl, ys);
                const T A = dot3(yl, yl) + (dot3(ys, ys) + dot3(ys + 3, ys + 3));
                T R = P.rscale * A;
                R = R < T(1e-12) ? T(1e-12) : R;
                rows.at(nrow, F_D) = T(1) / R;
                ++nrow;
            }
        }
    }
    (void)ncon_rows;
    (void)box_mine;

    phase_sync(2);
    // ---------------- primal Newton with exact line search
    const int world_rows = qsumi(nrow);
    int it = 0;
    bool solving = world_rows > 0;
    // level 4: the iterations run CTA-uniformly (quads that converged sit out)
    // with a barrier per iteration
    const bool it_sync = cta_sync && DK_PHYS_SYNC_LEVEL >= 4;
    if (it_sync ? __syncthreads_or(solving) != 0 : solving) {
        // M a, carried across the iterations (a += alpha d  =>  M a += alpha M d):
        // one matrix product per iteration instead of three
        T Ma_l[3], Ma_s[6];
        arrow_mul(M, a_l, a_s, Ma_l, Ma_s);
        // one Newton iteration; true when a is the minimiser
        auto newton_iter = [&]() -> bool {
            // x = J a - aref, active set, gradient and Hessian pieces
            Arrow<T> H = M;
            T g_l[3], g_s[6], gsm_l[3], gsm_s[6];  // full / smooth (M a - qfrc) gradient
#pragma unroll
            for (int i = 0; i < 3; ++i) g_l[i] = gsm_l[i] = Ma_l[i] - qf_l[i];
#pragma unroll
            for (int i = 0; i < 6; ++i) g_s[i] = gsm_s[i] = Ma_s[i] - qf_s[i];
            T gs_part[6] = {T(0), T(0), T(0), T(0), T(0), T(0)};
            T Hs_part[21];
#pragma unroll
            for (int e = 0; e < 21; ++e) Hs_part[e] = T(0);
            unsigned act_bits = 0;
            for (int r = 0; r < nrow; ++r) {
                T jb[6], jl[3];
#pragma unroll
                for (int i = 0; i < 6; ++i) jb[i] = rows.at(r, F_JB + i);
#pragma unroll
                for (int i = 0; i < 3; ++i) jl[i] = rows.at(r, F_JL + i);
                const T x = ((dot3(jb, a_s) + dot3(jb + 3, a_s + 3)) + dot3(jl, a_l)) -
                            rows.at(r, F_AREF);
                rows.at(r, F_X) = x;
                if (x < T(0)) {
                    act_bits |= 1u << r;
                    const T D = rows.at(r, F_D);
                    const T Dx = D * x;
#pragma unroll
                    for (int i = 0; i < 3; ++i) g_l[i] = g_l[i] + Dx * jl[i];
#pragma unroll
                    for (int i = 0; i < 6; ++i) gs_part[i] = gs_part[i] + Dx * jb[i];
                    // H: limb block, coupling, trunk partial
                    H.B[0] = H.B[0] + D * jl[0] * jl[0];
                    H.B[1] = H.B[1] + D * jl[1] * jl[0];
                    H.B[2] = H.B[2] + D * jl[1] * jl[1];
                    H.B[3] = H.B[3] + D * jl[2] * jl[0];
                    H.B[4] = H.B[4] + D * jl[2] * jl[1];
                    H.B[5] = H.B[5] + D * jl[2] * jl[2];
#pragma unroll
                    for (int b = 0; b < 6; ++b)
#pragma unroll
                        for (int j = 0; j < 3; ++j) H.C[b][j] = H.C[b][j] + D * jb[b] * jl[j];
#pragma unroll
                    for (int i = 0; i < 6; ++i)
#pragma unroll
                        for (int j = 0; j <= i; ++j)
                            Hs_part[Arrow<T>::ai(i, j)] = Hs_part[Arrow<T>::ai(i, j)] + D * jb[i] * jb[j];
                }
            }
            // H's trunk block and the gradient's trunk part are reduced across
            // the quad inside the factor / the solve's forward half
            ok &= H.factor(Hs_part);
            T d_l[3], d_s[6];
            {
                T ng_l[3], ng_s[6], ngs_part[6];
#pragma unroll
                for (int i = 0; i < 3; ++i) ng_l[i] = -g_l[i];
#pragma unroll
                for (int i = 0; i < 6; ++i) {
                    ng_s[i] = -g_s[i];
                    ngs_part[i] = -gs_part[i];
                }
                H.solve(ng_l, ng_s, d_l, d_s, ngs_part);
            }
            // line search coefficients
            T c1, c2;
            T Md_l[3], Md_s[6];
            {
                arrow_mul(M, d_l, d_s, Md_l, Md_s);
                T p1 = T(0), p2 = T(0);
#pragma unroll
                for (int i = 0; i < 3; ++i) {
                    p1 = p1 + d_l[i] * gsm_l[i];
                    p2 = p2 + d_l[i] * Md_l[i];
                }
                T s1 = T(0), s2 = T(0);
#pragma unroll
                for (int i = 0; i < 6; ++i) {
                    s1 = s1 + d_s[i] * gsm_s[i];
                    s2 = s2 + d_s[i] * Md_s[i];
                }
                c1 = qsum(p1) + s1;
                c2 = qsum(p2) + s2;
            }
            for (int r = 0; r < nrow; ++r) {
                const T y = ((rows.at(r, F_JB + 0) * d_s[0] + rows.at(r, F_JB + 1) * d_s[1]) +
                             rows.at(r, F_JB + 2) * d_s[2]) +
                            ((rows.at(r, F_JB + 3) * d_s[3] + rows.at(r, F_JB + 4) * d_s[4]) +
                             rows.at(r, F_JB + 5) * d_s[5]) +
                            ((rows.at(r, F_JL + 0) * d_l[0] + rows.at(r, F_JL + 1) * d_l[1]) +
                             rows.at(r, F_JL + 2) * d_l[2]);
                rows.at(r, F_Y) = y;
            }
            if (!(c2 > T(0))) return true;  // zero step: already the minimiser
            T alpha = T(1), lo = T(0), hi = T(-1);  // hi < 0: unbounded
            bool exact = false;
            unsigned piece_bits = 0;
            for (int ls = 0; ls < P.ls_iterations; ++ls) {
                T p1 = T(0), p2 = T(0);
                piece_bits = 0;
                for (int r = 0; r < nrow; ++r) {
                    const T x = rows.at(r, F_X), y = rows.at(r, F_Y);
                    if (x + alpha * y < T(0)) {
                        piece_bits |= 1u << r;
                        const T D = rows.at(r, F_D);
                        p1 = p1 + D * x * y;
                        p2 = p2 + D * y * y;
                    }
                }
                p1 = c1 + qsum(p1);
                p2 = c2 + qsum(p2);
                const T dphi = p1 + alpha * p2;
                if (dphi < T(0)) lo = alpha;
                else hi = alpha;
                T an = -p1 / p2;
                bool same = true;
                for (int r = 0; r < nrow; ++r) {
                    const bool in = rows.at(r, F_X) + an * rows.at(r, F_Y) < T(0);
                    same &= in == (((piece_bits >> r) & 1u) != 0);
                }
                if (qall(same)) {
                    alpha = an;
                    exact = true;
                    break;
                }
                if (!(an > lo && (hi < T(0) || an < hi))) an = hi < T(0) ? T(2) * alpha : T(0.5) * (lo + hi);
                alpha = an;
            }
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                a_l[i] = a_l[i] + alpha * d_l[i];
                Ma_l[i] = Ma_l[i] + alpha * Md_l[i];
            }
#pragma unroll
            for (int i = 0; i < 6; ++i) {
                a_s[i] = a_s[i] + alpha * d_s[i];
                Ma_s[i] = Ma_s[i] + alpha * Md_s[i];
            }
            return qall(exact && piece_bits == act_bits);
        };
        for (int k = 0; k < P.iterations; ++k) {
            if (it_sync) {
                if (!__syncthreads_or(solving)) break;
            } else if (!solving) {
                break;
            }
            if (solving) {
                ++it;
                if (newton_iter()) solving = false;
            }
        }
    }

    // ---------------- diagnostics of this step (constraint forces at the final a)
    if (dg) {
        const int NV = DK_PHYS_NV, MC = DK_PHYS_MAXCON;
        T fc_l[3] = {T(0), T(0), T(0)}, fcs_part[6] = {T(0), T(0), T(0), T(0), T(0), T(0)};
        T fr[16];
        for (int r = 0; r < nrow; ++r) {
            T jb[6], jl[3];
#pragma unroll
            for (int i = 0; i < 6; ++i) jb[i] = rows.at(r, F_JB + i);
#pragma unroll
            for (int i = 0; i < 3; ++i) jl[i] = rows.at(r, F_JL + i);
            const T x = ((dot3(jb, a_s) + dot3(jb + 3, a_s + 3)) + dot3(jl, a_l)) -
                        rows.at(r, F_AREF);
            const T f = x < T(0) ? -rows.at(r, F_D) * x : T(0);
            if (r < 16) fr[r] = f;
#pragma unroll
            for (int i = 0; i < 3; ++i) fc_l[i] = fc_l[i] + jl[i] * f;
#pragma unroll
            for (int i = 0; i < 6; ++i) fcs_part[i] = fcs_part[i] + jb[i] * f;
        }
        T fc_s[6];
#pragma unroll
        for (int i = 0; i < 6; ++i) fc_s[i] = qsum(fcs_part[i]);
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            const int d = 6 + 3 * lane_limb + i;
            if (dg->qacc) dg->qacc[w * NV + d] = a_l[i];
            if (dg->qfrc_bias) dg->qfrc_bias[w * NV + d] = bias_l[i];
            if (dg->qfrc_constraint) dg->qfrc_constraint[w * NV + d] = fc_l[i];
            if (dg->act_force) dg->act_force[w * DK_PHYS_NU + 3 * lane_limb + i] = act[i];
        }
        // contacts in world order: trunk-box contacts (lane l owns the l-th
        // penetrating corner), then limbs 0..3 (capsule ends, foot)
        const int nbox_lane = (P.collide_box && lane_limb < n_box) ? 1 : 0;
        const int nlimb = ncon_lane - nbox_lane;
        const unsigned m = quad_mask();
        const int base_lane = threadIdx.x & 28;
        int pre = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int v = __shfl_sync(m, nlimb, base_lane + k);
            if (k < lane_limb) pre += v;
        }
        const int nb = n_box < 4 ? n_box : 4;
        const int ncon = qsumi(nlimb) + nb;
        for (int c = 0; c < ncon_lane; ++c) {
            const int slot = (c < nbox_lane) ? lane_limb : nb + pre + (c - nbox_lane);
            const int64_t o = w * MC + slot;
            if (dg->contact_dist) dg->contact_dist[o] = cdist[c];
            if (dg->contact_geom) {
                dg->contact_geom[2 * o] = 0;
                dg->contact_geom[2 * o + 1] = cgeom[c];
            }
            if (dg->contact_pos)
#pragma unroll
                for (int i = 0; i < 3; ++i) dg->contact_pos[3 * o + i] = cpos[c][i];
            if (dg->contact_force) {
                const T *fe = fr + 4 * c;
                dg->contact_force[3 * o + 0] = (fe[0] + fe[1]) + (fe[2] + fe[3]);
                dg->contact_force[3 * o + 1] = mu * (fe[0] - fe[1]);
                dg->contact_force[3 * o + 2] = mu * (fe[2] - fe[3]);
            }
        }
        // unused slots: the quad clears them round-robin
        for (int slot = ncon + lane_limb; slot < MC; slot += 4) {
            const int64_t o = w * MC + slot;
            if (dg->contact_dist) dg->contact_dist[o] = T(0);
            if (dg->contact_geom) dg->contact_geom[2 * o] = dg->contact_geom[2 * o + 1] = -1;
            if (dg->contact_pos)
#pragma unroll
                for (int i = 0; i < 3; ++i) dg->contact_pos[3 * o + i] = T(0);
            if (dg->contact_force)
#pragma unroll
                for (int i = 0; i < 3; ++i) dg->contact_force[3 * o + i] = T(0);
        }
        if (lane_limb == 0) {
#pragma unroll
            for (int i = 0; i < 6; ++i) {
                if (dg->qacc) dg->qacc[w * NV + i] = a_s[i];
                if (dg->qfrc_bias) dg->qfrc_bias[w * NV + i] = bias_s[i];
                if (dg->qfrc_constraint) dg->qfrc_constraint[w * NV + i] = fc_s[i];
            }
            if (dg->ncon) dg->ncon[w] = ncon;
            if (dg->solver_iter) dg->solver_iter[w] = it;
        }
    }

    phase_sync(2);
    // ---------------- semi-implicit Euler
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        L.vlin[i] = L.vlin[i] + h * a_s[i];
        L.wb[i] = L.wb[i] + h * a_s[3 + i];
        L.qd[i] = L.qd[i] + h * a_l[i];
    }
#pragma unroll
    for (int i = 0; i < 3; ++i) L.pos[i] = L.pos[i] + h * L.vlin[i];
    {
        const T wn = PMath<T>::sqrt_(dot3(L.wb, L.wb));
        T *q = L.quat;
        if (wn > T(0)) {
            const T ang = h * wn;
            T sh, ch;
            PMath<T>::sincos_(T(0.5) * ang, &sh, &ch);
            const T s = sh / wn;
            const T r[4] = {ch, s * L.wb[0], s * L.wb[1], s * L.wb[2]};
            const T n0 = ((q[0] * r[0] - q[1] * r[1]) - q[2] * r[2]) - q[3] * r[3];
            const T n1 = ((q[0] * r[1] + q[1] * r[0]) + q[2] * r[3]) - q[3] * r[2];
            const T n2 = ((q[0] * r[2] - q[1] * r[3]) + q[2] * r[0]) + q[3] * r[1];
            const T n3 = ((q[0] * r[3] + q[1] * r[2]) - q[2] * r[1]) + q[3] * r[0];
            q[0] = n0; q[1] = n1; q[2] = n2; q[3] = n3;
        }
        const T iqn = PMath<T>::rsqrt_(((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3]);
#pragma unroll
        for (int i = 0; i < 4; ++i) q[i] = q[i] * iqn;
    }
#pragma unroll
    for (int i = 0; i < 3; ++i) L.q[i] = L.q[i] + h * L.qd[i];
    return ok;
}

// sensordata of the lane's world (post-step state): each lane writes its
// limb's joint and foot entries, lane 0 the trunk entries
template <typename T>
__device__ void sensors(const PhysConst<T> &P, const Lane<T> &L, int lane_limb, T *s) {
    const LimbConst<T> &lm = P.limb[lane_limb];
    T R0[9];
    quat2mat(L.quat, R0);
    if (lane_limb == 0) {
#pragma unroll
        for (int i = 0; i < 4; ++i) s[i] = L.quat[i];
#pragma unroll
        for (int i = 0; i < 3; ++i) s[4 + i] = L.wb[i];
        T vl[3];
        mat_tvec3(R0, L.vlin, vl);
#pragma unroll
        for (int i = 0; i < 3; ++i) s[7 + i] = vl[i];
    }
    T Rp[9], pp[3];
#pragma unroll
    for (int i = 0; i < 9; ++i) Rp[i] = R0[i];
#pragma unroll
    for (int i = 0; i < 3; ++i) pp[i] = L.pos[i];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        T off[3], Rq[9], Rj[9];
        mat_vec3(Rp, lm.body_pos[j], off);
#pragma unroll
        for (int i = 0; i < 3; ++i) pp[i] = pp[i] + off[i];
        axis_rot(lm.axis[j], L.q[j], Rq);
        mat_mul3(Rp, Rq, Rj);
#pragma unroll
        for (int i = 0; i < 9; ++i) Rp[i] = Rj[i];
        s[10 + 3 * lane_limb + j] = L.q[j];
        s[22 + 3 * lane_limb + j] = L.qd[j];
    }
    T foff[3];
    mat_vec3(Rp, lm.foot_pos, foff);
#pragma unroll
    for (int i = 0; i < 3; ++i) s[34 + 3 * lane_limb + i] = pp[i] + foff[i];
}

// INSPECT: the dk_phys_inspect variant (its own instantiation, so the step
// kernel carries a single copy of phys_step)
template <typename T, bool INSPECT>
__global__ void __launch_bounds__(THREADS) phys_kernel(PhysConst<T> pc, PhysArgs<T> a,
                                                       PhysInspect<T> ins) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    PhysConst<T> &P = *reinterpret_cast<PhysConst<T> *>(smem_raw);
    T *rowbuf = reinterpret_cast<T *>(smem_raw + ((sizeof(PhysConst<T>) + 15) & ~size_t(15)));
    {   // stage the model in shared memory
        const uint32_t *src = reinterpret_cast<const uint32_t *>(&pc);
        uint32_t *dst = reinterpret_cast<uint32_t *>(smem_raw);
        for (int i = threadIdx.x; i < (int)(sizeof(PhysConst<T>) / 4); i += blockDim.x) dst[i] = src[i];
    }
    __syncthreads();
    const int tid = threadIdx.x;
    const int lane_limb = tid & 3;
    const int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 2) + (tid >> 2);
    if (w >= a.n) return;  // whole quads exit together
    const int64_t n = a.n;
    Lane<T> L;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        L.pos[i] = a.qpos[i * n + w];
        L.vlin[i] = a.qvel[i * n + w];
        L.wb[i] = a.qvel[(3 + i) * n + w];
        L.q[i] = a.qpos[(7 + 3 * lane_limb + i) * n + w];
        L.qd[i] = a.qvel[(6 + 3 * lane_limb + i) * n + w];
        L.ctrl[i] = a.ctrl[w * DK_PHYS_NU + 3 * lane_limb + i];
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) L.quat[i] = a.qpos[(3 + i) * n + w];
    L.mu = P.mu;
    L.base_mass = P.base_mass;
    L.kp = P.kp;
    Rows<T> rows{rowbuf + (size_t)tid * pc.rows_per_lane * RF};
    if constexpr (INSPECT) {
        phys_step(P, L, rows, lane_limb, static_cast<const PhysArgs<T> *>(nullptr), w, &ins);
        return;
    }
    bool ok = true;
    const bool want = a.qacc || a.qfrc_bias || a.qfrc_constraint || a.act_force || a.ncon ||
                      a.contact_geom || a.contact_dist || a.contact_pos || a.contact_force ||
                      a.solver_iter;
    // every thread of a full CTA steps: CTA barriers inside the step are safe
    const bool full = (int64_t)(blockIdx.x + 1) * (blockDim.x >> 2) <= n;
    for (int64_t s = 0; s < a.num_steps; ++s) {
        const bool last = want && s + 1 == a.num_steps;
        ok &= phys_step(P, L, rows, lane_limb, last ? &a : nullptr, w,
                        static_cast<const PhysInspect<T> *>(nullptr), static_cast<T *>(nullptr),
                        full);
    }
    // state back
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        if (lane_limb == 0) {
            a.qpos[i * n + w] = L.pos[i];
            a.qvel[i * n + w] = L.vlin[i];
            a.qvel[(3 + i) * n + w] = L.wb[i];
        }
        a.qpos[(7 + 3 * lane_limb + i) * n + w] = L.q[i];
        a.qvel[(6 + 3 * lane_limb + i) * n + w] = L.qd[i];
    }
    if (lane_limb == 0)
#pragma unroll
        for (int i = 0; i < 4; ++i) a.qpos[(3 + i) * n + w] = L.quat[i];
    if (!ok && a.bad) *a.bad = 1;
    if (a.sensordata) sensors(P, L, lane_limb, a.sensordata + w * NS);
}

}  // namespace phys
}  // namespace dk

namespace dk {
namespace phys {

template <typename T>
size_t phys_smem_bytes(const PhysConst<T> &pc, int threads) {
    return ((sizeof(PhysConst<T>) + 15) & ~size_t(15)) +
           (size_t)pc.rows_per_lane * RF * threads * sizeof(T);
}

// SM count of the current device (148 on B200), queried once per device
inline int phys_sm_count() {
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

// Threads per CTA for n worlds: one CTA per SM per wave (the registers of a
// 256-thread CTA fill the SM), as few waves as 64-world CTAs need, the worlds
// spread evenly over them -- 8192 worlds: 148 SMs x 56 worlds (224 threads)
// instead of 128 x 64 with 20 SMs idle.  One CTA per SM also keeps all of an
// SM's warps under the same phase barriers (measured: 256-thread CTAs 16%
// faster than two 128-thread CTAs per SM at 8192 worlds, 26% at 65536).
// Halved while the constraint rows do not fit the shared-memory cap.
template <class SmemFn>
inline int pick_threads(int64_t n, SmemFn smem_bytes) {
    const int64_t sms = phys_sm_count();
    const int64_t waves = (n + sms * WPC - 1) / (sms * WPC);
    const int64_t wpc = (n + sms * waves - 1) / (sms * waves);
    int threads = (int)((wpc * QUAD + 31) / 32 * 32);
    threads = threads < 32 ? 32 : (threads > THREADS ? THREADS : threads);
    while (threads > 32 && smem_bytes(threads) > kSmemCap) threads = (threads / 2 + 31) / 32 * 32;
    return threads;
}

template <typename T>
cudaError_t launch_phys(const PhysConst<T> &pc, const PhysArgs<T> &a, const PhysInspect<T> &ins,
                        cudaStream_t st) {
    const int threads = pick_threads(a.n, [&](int t) { return phys_smem_bytes(pc, t); });
    const size_t smem = phys_smem_bytes(pc, threads);
    static SmemOptIn optin[2];  // per device; [0] step, [1] inspect
    for (int k = 0; k < 2; ++k) {
        cudaError_t e = optin[k].ensure(
            k ? (const void *)phys_kernel<T, true> : (const void *)phys_kernel<T, false>, smem);
        if (e != cudaSuccess) return e;
    }
    const int wpc = threads / QUAD;
    const unsigned grid = (unsigned)((a.n + wpc - 1) / wpc);
    if (ins.on()) phys_kernel<T, true><<<grid, threads, smem, st>>>(pc, a, ins);
    else phys_kernel<T, false><<<grid, threads, smem, st>>>(pc, a, ins);
    return cudaGetLastError();
}

// SoA <-> row-major state transposes
template <typename T>
__global__ void soa_from_rows(const T *rows, T *soa, int64_t n, int width) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n * width) return;
    const int64_t w = i / width, c = i % width;
    soa[c * n + w] = rows[i];
}
template <typename T>
__global__ void rows_from_soa(const T *soa, T *rows, int64_t n, int width) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n * width) return;
    const int64_t w = i / width, c = i % width;
    rows[i] = soa[c * n + w];
}
template <typename T>
cudaError_t launch_transpose(const T *src, T *dst, int64_t n, int width, bool to_soa,
                             cudaStream_t st) {
    const int64_t total = n * width;
    const unsigned grid = (unsigned)((total + 255) / 256);
    if (to_soa) soa_from_rows<T><<<grid, 256, 0, st>>>(src, dst, n, width);
    else rows_from_soa<T><<<grid, 256, 0, st>>>(src, dst, n, width);
    return cudaGetLastError();
}

#define DK_PHYS_DECLARE(T)                                                                    \
    extern template cudaError_t launch_phys<T>(const PhysConst<T> &, const PhysArgs<T> &,    \
                                               const PhysInspect<T> &, cudaStream_t);         \
    extern template cudaError_t launch_transpose<T>(const T *, T *, int64_t, int, bool,       \
                                                    cudaStream_t);
#define DK_PHYS_INSTANTIATE(T)                                                                \
    template cudaError_t launch_phys<T>(const PhysConst<T> &, const PhysArgs<T> &,           \
                                        const PhysInspect<T> &, cudaStream_t);                \
    template cudaError_t launch_transpose<T>(const T *, T *, int64_t, int, bool, cudaStream_t);

}  // namespace phys
}  // namespace dk
