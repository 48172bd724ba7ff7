/*
 * physics.c -- CPU fp64 oracle of the articulated contact physics step
 * (include/deskrl_b200.h "Articulated contact
 * physics").
 *
 * TEST INFRASTRUCTURE ONLY: the checker for the B200 kernels in
 * paper_2502_08844_b200/csrc/physics.cuh, never linked into the product.
 *
 * PARITY UNPINNED.  The reference has no contact physics ("OUT OF
 * SCOPE -- the MJX/MuJoCo contact solver and all contact-rich environments";
 * PAPER.md:580 only fixes feet-only collision for the joystick tasks) and
 * MuJoCo/MJX are not in this container, so no golden vector exists.  This
 * file is an independent restatement of the algorithm the kernel implements,
 * deliberately written differently where it can be:
 *   - generic tree code over a parent array (the kernel is lane-per-limb);
 *   - the mass matrix as sum_b J_b^T I_b J_b over body Jacobians (the kernel
 *     uses composite rigid bodies);
 *   - dense 18x18 Cholesky (the kernel factors the arrow-structured matrix
 *     limb blocks first);
 * and is pinned instead by physical known-answer tests (tests/test_oracle_physics.py):
 * inverse dynamics consistency, free fall, kinetic energy from body
 * velocities, momentum conservation without gravity, static stance.
 * Only forward kinematics and collision distances use the kernel's exact
 * expression order, so contact counts and pairs can be compared bit for bit.
 * Compiled with -ffp-contract=off (two roundings per a*b+c, like the f64
 * kernel's --fmad=false).
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

#include "../include/deskrl_b200.h"

#define NB DK_PHYS_NBODY
#define NV DK_PHYS_NV
#define NQ DK_PHYS_NQ
#define MAXROW (DK_PHYS_MAXCON * 4 + 2 * 12)

/* ---------------------------------------------------------------- helpers */

static void mat_mul3(const double *A, const double *B, double *C) {
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c)
            C[3 * r + c] = (A[3 * r] * B[c] + A[3 * r + 1] * B[3 + c]) + A[3 * r + 2] * B[6 + c];
}
static void mat_vec3(const double *R, const double *v, double *o) {
    for (int r = 0; r < 3; ++r) o[r] = (R[3 * r] * v[0] + R[3 * r + 1] * v[1]) + R[3 * r + 2] * v[2];
}
static void mat_tvec3(const double *R, const double *v, double *o) {
    for (int c = 0; c < 3; ++c) o[c] = (R[c] * v[0] + R[3 + c] * v[1]) + R[6 + c] * v[2];
}
static void cross3(const double *a, const double *b, double *o) {
    o[0] = a[1] * b[2] - a[2] * b[1];
    o[1] = a[2] * b[0] - a[0] * b[2];
    o[2] = a[0] * b[1] - a[1] * b[0];
}
static double dot3(const double *a, const double *b) { return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2]; }

/* MuJoCo mju_quat2Mat's expression (the kernel uses the same) */
static void quat2mat(const double *q, double *R) {
    const double q00 = q[0] * q[0], q01 = q[0] * q[1], q02 = q[0] * q[2], q03 = q[0] * q[3];
    const double q11 = q[1] * q[1], q12 = q[1] * q[2], q13 = q[1] * q[3];
    const double q22 = q[2] * q[2], q23 = q[2] * q[3], q33 = q[3] * q[3];
    R[0] = ((q00 + q11) - q22) - q33;
    R[4] = ((q00 - q11) + q22) - q33;
    R[8] = ((q00 - q11) - q22) + q33;
    R[1] = 2.0 * (q12 - q03);
    R[2] = 2.0 * (q13 + q02);
    R[3] = 2.0 * (q12 + q03);
    R[5] = 2.0 * (q23 - q01);
    R[6] = 2.0 * (q13 - q02);
    R[7] = 2.0 * (q23 + q01);
}

/* rotation by angle q about unit axis a (Rodrigues, the kernel's expression) */
static void axis_rot(const double *a, double q, double *R) {
    const double c = cos(q), s = sin(q), t = 1.0 - c;
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

/* ------------------------------------------------------------------ tree */

typedef struct {
    int parent[NB];
    int dofadr[NB], dofnum[NB];
    double mass[NB], ipos[NB][3], inertia[NB][3], pos[NB][3], axis[NB][3];
    double armature[NV], damping[NV];
} tree_t;

static void build_tree(const dk_phys_model *m, tree_t *t) {
    memset(t, 0, sizeof(*t));
    t->parent[0] = -1;
    t->dofadr[0] = 0;
    t->dofnum[0] = 6;
    t->mass[0] = m->base_mass;
    for (int k = 0; k < 3; ++k) {
        t->ipos[0][k] = m->base_ipos[k];
        t->inertia[0][k] = m->base_inertia[k];
    }
    for (int l = 0; l < 4; ++l)
        for (int j = 0; j < 3; ++j) {
            const int b = 1 + 3 * l + j;
            t->parent[b] = j == 0 ? 0 : b - 1;
            t->dofadr[b] = 5 + b;
            t->dofnum[b] = 1;
            t->mass[b] = m->body_mass[l][j];
            for (int k = 0; k < 3; ++k) {
                t->ipos[b][k] = m->body_ipos[l][j][k];
                t->inertia[b][k] = m->body_inertia[l][j][k];
                t->pos[b][k] = m->body_pos[l][j][k];
                t->axis[b][k] = m->jnt_axis[l][j][k];
            }
            t->armature[5 + b] = m->dof_armature[l][j];
            t->damping[5 + b] = m->dof_damping[l][j];
        }
}

typedef struct {
    double xR[NB][9], xpos[NB][3], xipos[NB][3];
    double cdof[NV][6]; /* [angular; linear at the trunk origin p0], world frame */
    int dofbody[NV];
    double p0[3];
} kin_t;

/* forward kinematics (same expression order as the kernel) */
static void fk(const tree_t *t, const double *qpos, kin_t *k) {
    double q[4] = {qpos[3], qpos[4], qpos[5], qpos[6]};
    quat2mat(q, k->xR[0]);
    for (int i = 0; i < 3; ++i) k->xpos[0][i] = qpos[i];
    for (int b = 1; b < NB; ++b) {
        const int p = t->parent[b];
        double off[3], Rj[9];
        mat_vec3(k->xR[p], t->pos[b], off);
        for (int i = 0; i < 3; ++i) k->xpos[b][i] = k->xpos[p][i] + off[i];
        axis_rot(t->axis[b], qpos[1 + t->dofadr[b]], Rj);
        mat_mul3(k->xR[p], Rj, k->xR[b]);
    }
    for (int b = 0; b < NB; ++b) {
        double off[3];
        mat_vec3(k->xR[b], t->ipos[b], off);
        for (int i = 0; i < 3; ++i) k->xipos[b][i] = k->xpos[b][i] + off[i];
    }
    for (int i = 0; i < 3; ++i) k->p0[i] = k->xpos[0][i];
    /* motion subspaces */
    memset(k->cdof, 0, sizeof(k->cdof));
    for (int i = 0; i < 3; ++i) {
        k->cdof[i][3 + i] = 1.0;                  /* world-frame translation */
        for (int r = 0; r < 3; ++r) k->cdof[3 + i][r] = k->xR[0][3 * r + i]; /* trunk axis i */
        k->dofbody[i] = k->dofbody[3 + i] = 0;
    }
    for (int b = 1; b < NB; ++b) {
        const int d = t->dofadr[b];
        double a[3], rel[3], lin[3];
        mat_vec3(k->xR[t->parent[b]], t->axis[b], a);
        for (int i = 0; i < 3; ++i) rel[i] = k->p0[i] - k->xpos[b][i];
        cross3(a, rel, lin);
        for (int i = 0; i < 3; ++i) {
            k->cdof[d][i] = a[i];
            k->cdof[d][3 + i] = lin[i];
        }
        k->dofbody[d] = b;
    }
}

/* 6x6 spatial inertia of body b about p0 (world frame), [ang; lin] ordering:
 * [[I_p0, [h]x], [-[h]x, m 1]] with h = m (xipos - p0) */
static void body_inertia6(const tree_t *t, const kin_t *k, int b, double I6[6][6]) {
    const double *R = k->xR[b];
    double Ic[9], r[3];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double s = 0.0;
            for (int q = 0; q < 3; ++q) s += R[3 * i + q] * t->inertia[b][q] * R[3 * j + q];
            Ic[3 * i + j] = s;
        }
    for (int i = 0; i < 3; ++i) r[i] = k->xipos[b][i] - k->p0[i];
    const double m = t->mass[b], rr = dot3(r, r);
    double h[3] = {m * r[0], m * r[1], m * r[2]};
    memset(I6, 0, sizeof(double) * 36);
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) I6[i][j] = Ic[3 * i + j] + m * ((i == j ? rr : 0.0) - r[i] * r[j]);
    /* [h]x */
    const double hx[3][3] = {{0, -h[2], h[1]}, {h[2], 0, -h[0]}, {-h[1], h[0], 0}};
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            I6[i][3 + j] = hx[i][j];
            I6[3 + i][j] = -hx[i][j];
        }
    for (int i = 0; i < 3; ++i) I6[3 + i][3 + i] = m;
}

static int is_ancestor_dof(const tree_t *t, const kin_t *k, int d, int b) {
    for (int x = b; x >= 0; x = t->parent[x])
        if (k->dofbody[d] == x) return 1;
    return 0;
}

/* M = sum_b J_b^T I_b J_b (+ armature on the diagonal) */
static void mass_matrix(const tree_t *t, const kin_t *k, double M[NV][NV]) {
    memset(M, 0, sizeof(double) * NV * NV);
    for (int b = 0; b < NB; ++b) {
        double I6[6][6];
        body_inertia6(t, k, b, I6);
        double IJ[6][NV];
        memset(IJ, 0, sizeof(IJ));
        for (int d = 0; d < NV; ++d) {
            if (!is_ancestor_dof(t, k, d, b)) continue;
            for (int i = 0; i < 6; ++i) {
                double s = 0.0;
                for (int j = 0; j < 6; ++j) s += I6[i][j] * k->cdof[d][j];
                IJ[i][d] = s;
            }
        }
        for (int d1 = 0; d1 < NV; ++d1) {
            if (!is_ancestor_dof(t, k, d1, b)) continue;
            for (int d2 = 0; d2 < NV; ++d2) {
                double s = 0.0;
                for (int i = 0; i < 6; ++i) s += k->cdof[d1][i] * IJ[i][d2];
                M[d1][d2] += s;
            }
        }
    }
    for (int d = 0; d < NV; ++d) M[d][d] += t->armature[d];
}

static void cross_motion(const double *v, const double *u, double *o) { /* v x_m u */
    double a[3], b[3], c[3];
    cross3(v, u, a);
    cross3(v, u + 3, b);
    cross3(v + 3, u, c);
    for (int i = 0; i < 3; ++i) {
        o[i] = a[i];
        o[3 + i] = b[i] + c[i];
    }
}
static void cross_force(const double *v, const double *f, double *o) { /* v x_f f */
    double a[3], b[3], c[3];
    cross3(v, f, a);
    cross3(v + 3, f + 3, b);
    cross3(v, f + 3, c);
    for (int i = 0; i < 3; ++i) {
        o[i] = a[i] + b[i];
        o[3 + i] = c[i];
    }
}
static void mul6(double I6[6][6], const double *v, double *o) {
    for (int i = 0; i < 6; ++i) {
        double s = 0.0;
        for (int j = 0; j < 6; ++j) s += I6[i][j] * v[j];
        o[i] = s;
    }
}

/* recursive Newton-Euler: qfrc = M(q) qacc + C(q, qvel) qvel + g(q) */
static void rne(const dk_phys_model *m, const tree_t *t, const kin_t *k, const double *qvel,
                const double *qacc, double *qfrc) {
    double cvel[NB][6], cacc[NB][6], cfrc[NB][6];
    double cdof_dot[NV][6];
    for (int b = 0; b < NB; ++b) {
        const int p = t->parent[b];
        for (int i = 0; i < 6; ++i) cvel[b][i] = p < 0 ? 0.0 : cvel[p][i];
        for (int d = t->dofadr[b]; d < t->dofadr[b] + t->dofnum[b]; ++d)
            for (int i = 0; i < 6; ++i) cvel[b][i] += k->cdof[d][i] * qvel[d];
    }
    for (int d = 0; d < NV; ++d) {
        if (d < 3) {
            memset(cdof_dot[d], 0, sizeof(cdof_dot[d])); /* world-fixed translation axes */
        } else {
            cross_motion(cvel[k->dofbody[d]], k->cdof[d], cdof_dot[d]);
        }
    }
    for (int b = 0; b < NB; ++b) {
        const int p = t->parent[b];
        for (int i = 0; i < 6; ++i) {
            cacc[b][i] = p < 0 ? (i < 3 ? 0.0 : -m->gravity[i - 3]) : cacc[p][i];
        }
        for (int d = t->dofadr[b]; d < t->dofadr[b] + t->dofnum[b]; ++d)
            for (int i = 0; i < 6; ++i)
                cacc[b][i] += cdof_dot[d][i] * qvel[d] + (qacc ? k->cdof[d][i] * qacc[d] : 0.0);
        double I6[6][6], Ia[6], Iv[6], vx[6];
        body_inertia6(t, k, b, I6);
        mul6(I6, cacc[b], Ia);
        mul6(I6, cvel[b], Iv);
        cross_force(cvel[b], Iv, vx);
        for (int i = 0; i < 6; ++i) cfrc[b][i] = Ia[i] + vx[i];
    }
    for (int b = NB - 1; b > 0; --b)
        for (int i = 0; i < 6; ++i) cfrc[t->parent[b]][i] += cfrc[b][i];
    for (int d = 0; d < NV; ++d) {
        double s = 0.0;
        for (int i = 0; i < 6; ++i) s += k->cdof[d][i] * cfrc[k->dofbody[d]][i];
        qfrc[d] = s;
    }
    if (qacc)
        for (int d = 0; d < NV; ++d) qfrc[d] += t->armature[d] * qacc[d];
}

/* dense Cholesky A = L L^T in place (lower); returns 0 if not SPD */
static int chol(double A[NV][NV]) {
    for (int j = 0; j < NV; ++j) {
        double s = A[j][j];
        for (int k = 0; k < j; ++k) s -= A[j][k] * A[j][k];
        if (!(s > 0.0)) return 0;
        const double d = sqrt(s);
        A[j][j] = d;
        for (int i = j + 1; i < NV; ++i) {
            double t = A[i][j];
            for (int k = 0; k < j; ++k) t -= A[i][k] * A[j][k];
            A[i][j] = t / d;
        }
    }
    return 1;
}
static void chol_solve(double L[NV][NV], const double *b, double *x) {
    double y[NV];
    for (int i = 0; i < NV; ++i) {
        double s = b[i];
        for (int k = 0; k < i; ++k) s -= L[i][k] * y[k];
        y[i] = s / L[i][i];
    }
    for (int i = NV - 1; i >= 0; --i) {
        double s = y[i];
        for (int k = i + 1; k < NV; ++k) s -= L[k][i] * x[k];
        x[i] = s / L[i][i];
    }
}

/* ------------------------------------------------------------- collision */

typedef struct {
    int n;
    int geom[DK_PHYS_MAXCON];
    int body[DK_PHYS_MAXCON];
    double dist[DK_PHYS_MAXCON];
    double pos[DK_PHYS_MAXCON][3];
} contacts_t;

static void add_contact(contacts_t *c, int geom, int body, const double *centre, double radius,
                        double dist) {
    const int i = c->n++;
    c->geom[i] = geom;
    c->body[i] = body;
    c->dist[i] = dist;
    c->pos[i][0] = centre[0];
    c->pos[i][1] = centre[1];
    c->pos[i][2] = centre[2] - (radius + 0.5 * dist); /* midpoint between the surfaces */
}

/* plane z = 0 (normal +z) against trunk box corners, thigh capsule end
 * spheres and foot spheres, in geom order; a contact exists iff dist < 0 */
static void collide(const dk_phys_model *m, const kin_t *k, contacts_t *c) {
    c->n = 0;
    if (m->collide_box) {
        int nb = 0;
        for (int s = 0; s < 8 && nb < 4; ++s) {
            const double loc[3] = {(s & 1) ? m->base_box[0] : -m->base_box[0],
                                   (s & 2) ? m->base_box[1] : -m->base_box[1],
                                   (s & 4) ? m->base_box[2] : -m->base_box[2]};
            double off[3], w[3];
            mat_vec3(k->xR[0], loc, off);
            for (int i = 0; i < 3; ++i) w[i] = k->xpos[0][i] + off[i];
            const double dist = w[2];
            if (dist < 0.0) {
                add_contact(c, 1, 0, w, 0.0, dist);
                ++nb;
            }
        }
    }
    for (int l = 0; l < 4; ++l) {
        const int b1 = 2 + 3 * l, b2 = 3 + 3 * l;
        if (m->collide_thigh) {
            const double *e0 = k->xpos[b1], *e1 = k->xpos[b2];
            const double d0 = e0[2] - m->thigh_radius, d1 = e1[2] - m->thigh_radius;
            if (d0 < 0.0) add_contact(c, 2 + 2 * l, b1, e0, m->thigh_radius, d0);
            if (d1 < 0.0) add_contact(c, 2 + 2 * l, b1, e1, m->thigh_radius, d1);
        }
        double off[3], f[3];
        mat_vec3(k->xR[b2], m->foot_pos[l], off);
        for (int i = 0; i < 3; ++i) f[i] = k->xpos[b2][i] + off[i];
        const double df = f[2] - m->foot_radius;
        if (df < 0.0) add_contact(c, 3 + 2 * l, b2, f, m->foot_radius, df);
    }
}

/* translational Jacobian of a world point on body b: 3 x NV */
static void point_jac(const tree_t *t, const kin_t *k, int b, const double *p, double J[3][NV]) {
    memset(J, 0, sizeof(double) * 3 * NV);
    double r[3];
    for (int i = 0; i < 3; ++i) r[i] = p[i] - k->p0[i];
    for (int d = 0; d < NV; ++d) {
        if (!is_ancestor_dof(t, k, d, b)) continue;
        double wr[3];
        cross3(k->cdof[d], r, wr);
        for (int i = 0; i < 3; ++i) J[i][d] = k->cdof[d][3 + i] + wr[i];
    }
}

/* ------------------------------------------------------------------ step */

typedef struct {
    double qacc[NV], qfrc_bias[NV], qfrc_constraint[NV], act[12];
    int ncon, iters;
    int geom[DK_PHYS_MAXCON];
    double dist[DK_PHYS_MAXCON], pos[DK_PHYS_MAXCON][3], force[DK_PHYS_MAXCON][3];
} diag_t;

static int ls_piece_equal(const unsigned char *a, const unsigned char *b, int n) {
    for (int i = 0; i < n; ++i)
        if (a[i] != b[i]) return 0;
    return 1;
}

/* one physics step of one world, in place; returns 0 on a non-SPD matrix */
static int step_world(const dk_phys_model *m, const tree_t *t, double *qpos, double *qvel,
                      const double *ctrl, diag_t *dg) {
    const double h = m->timestep;
    kin_t k;
    fk(t, qpos, &k);
    double M[NV][NV], Mt[NV][NV], L[NV][NV];
    mass_matrix(t, &k, M);
    memcpy(Mt, M, sizeof(M));
    for (int d = 0; d < NV; ++d) Mt[d][d] += h * t->damping[d];
    double bias[NV];
    rne(m, t, &k, qvel, NULL, bias);
    double qfrc[NV];
    for (int d = 0; d < 6; ++d) qfrc[d] = -bias[d];
    for (int l = 0; l < 4; ++l)
        for (int j = 0; j < 3; ++j) {
            const int d = 6 + 3 * l + j;
            double tau = m->kp * (ctrl[3 * l + j] - qpos[7 + 3 * l + j]) - m->kd * qvel[d];
            const double lim = m->torque_limit[l][j];
            tau = tau < -lim ? -lim : (tau > lim ? lim : tau);
            dg->act[3 * l + j] = tau;
            qfrc[d] = (tau - t->damping[d] * qvel[d]) - bias[d];
        }
    memcpy(L, Mt, sizeof(Mt));
    if (!chol(L)) return 0;
    double a0[NV];
    chol_solve(L, qfrc, a0);

    /* constraint rows */
    contacts_t c;
    collide(m, &k, &c);
    static const double nrm[3] = {0, 0, 1}, t1[3] = {1, 0, 0}, t2[3] = {0, 1, 0};
    const double mu = m->friction;
    const double imp = m->solimp, tc = m->solref[0], dr = m->solref[1];
    const double kstiff = 1.0 / (imp * imp * tc * tc * dr * dr), bdamp = 2.0 / (imp * tc);
    double J[MAXROW][NV], aref[MAXROW], D[MAXROW];
    int nrow = 0;
    for (int ci = 0; ci < c.n; ++ci) {
        double Jp[3][NV];
        point_jac(t, &k, c.body[ci], c.pos[ci], Jp);
        for (int e = 0; e < 4; ++e) {
            const double *tt = e < 2 ? t1 : t2;
            const double sg = (e & 1) ? -mu : mu;
            for (int d = 0; d < NV; ++d)
                J[nrow][d] = dot3(nrm, (double[3]){Jp[0][d], Jp[1][d], Jp[2][d]}) +
                             sg * dot3(tt, (double[3]){Jp[0][d], Jp[1][d], Jp[2][d]});
            aref[nrow] = c.dist[ci]; /* position term, finished below */
            ++nrow;
        }
    }
    for (int l = 0; l < 4; ++l)
        for (int j = 0; j < 3; ++j) {
            const double q = qpos[7 + 3 * l + j];
            const double lo = q - m->jnt_range[l][j][0], hi = m->jnt_range[l][j][1] - q;
            if (lo < 0.0) {
                memset(J[nrow], 0, sizeof(J[nrow]));
                J[nrow][6 + 3 * l + j] = 1.0;
                aref[nrow++] = lo;
            }
            if (hi < 0.0) {
                memset(J[nrow], 0, sizeof(J[nrow]));
                J[nrow][6 + 3 * l + j] = -1.0;
                aref[nrow++] = hi;
            }
        }
    for (int i = 0; i < nrow; ++i) {
        double x[NV], jv = 0.0, A = 0.0;
        chol_solve(L, J[i], x);
        for (int d = 0; d < NV; ++d) {
            jv += J[i][d] * qvel[d];
            A += J[i][d] * x[d];
        }
        D[i] = A; /* A_ii for now; regularised below */
        aref[i] = -bdamp * jv - kstiff * imp * aref[i];
    }
    /* regulariser R = (1 - imp)/imp * A.  The four edges of a pyramid share one
     * A (their mean, A_n + mu^2 (A_t1 + A_t2)/2: the +-mu cross terms cancel),
     * so the penetration term alone produces no tangential force. */
    for (int ci = 0; ci < c.n; ++ci) {
        double *Ae = D + 4 * ci;
        const double Am = ((Ae[0] + Ae[1]) + (Ae[2] + Ae[3])) * 0.25;
        Ae[0] = Ae[1] = Ae[2] = Ae[3] = Am;
    }
    for (int i = 0; i < nrow; ++i) {
        double R = (1.0 - imp) / imp * D[i];
        if (R < 1e-12) R = 1e-12;
        D[i] = 1.0 / R;
    }

    /* primal Newton with exact line search */
    double a[NV];
    memcpy(a, a0, sizeof(a));
    unsigned char act[MAXROW], piece[MAXROW], trial[MAXROW];
    double x[MAXROW], y[MAXROW];
    int it = 0;
    for (; nrow > 0 && it < m->iterations; ++it) {
        for (int i = 0; i < nrow; ++i) {
            double s = 0.0;
            for (int d = 0; d < NV; ++d) s += J[i][d] * a[d];
            x[i] = s - aref[i];
            act[i] = x[i] < 0.0;
        }
        double g[NV], H[NV][NV], Ma[NV];
        for (int r = 0; r < NV; ++r) {
            double s = 0.0;
            for (int d = 0; d < NV; ++d) s += Mt[r][d] * a[d];
            Ma[r] = s;
            g[r] = s - qfrc[r];
        }
        memcpy(H, Mt, sizeof(H));
        for (int i = 0; i < nrow; ++i) {
            if (!act[i]) continue;
            for (int r = 0; r < NV; ++r) {
                g[r] += D[i] * x[i] * J[i][r];
                for (int q = 0; q < NV; ++q) H[r][q] += D[i] * J[i][r] * J[i][q];
            }
        }
        if (!chol(H)) return 0;
        double delta[NV], mg[NV];
        for (int r = 0; r < NV; ++r) mg[r] = -g[r];
        chol_solve(H, mg, delta);
        /* phi'(alpha) = c1 + alpha c2 + sum_{x+alpha y<0} D (x + alpha y) y */
        double c1 = 0.0, c2 = 0.0;
        for (int r = 0; r < NV; ++r) {
            double Md = 0.0;
            for (int d = 0; d < NV; ++d) Md += Mt[r][d] * delta[d];
            c1 += delta[r] * (Ma[r] - qfrc[r]);
            c2 += delta[r] * Md;
        }
        for (int i = 0; i < nrow; ++i) {
            double s = 0.0;
            for (int d = 0; d < NV; ++d) s += J[i][d] * delta[d];
            y[i] = s;
        }
        if (!(c2 > 0.0)) {  /* zero step: already the minimiser */
            ++it;
            break;
        }
        double alpha = 1.0, lo = 0.0, hi = INFINITY;
        int exact = 0;
        for (int ls = 0; ls < m->ls_iterations; ++ls) {
            double p1 = c1, p2 = c2;
            for (int i = 0; i < nrow; ++i) {
                const double z = x[i] + alpha * y[i];
                piece[i] = z < 0.0;
                if (piece[i]) {
                    p1 += D[i] * x[i] * y[i];
                    p2 += D[i] * y[i] * y[i];
                }
            }
            const double dphi = p1 + alpha * p2;
            if (dphi < 0.0) lo = alpha;
            else hi = alpha;
            double an = -p1 / p2;
            int same = 1;
            for (int i = 0; i < nrow; ++i) {
                trial[i] = x[i] + an * y[i] < 0.0;
                if (trial[i] != piece[i]) same = 0;
            }
            if (same) {
                alpha = an;
                exact = 1;
                break;
            }
            if (!(an > lo && an < hi)) an = isinf(hi) ? 2.0 * alpha : 0.5 * (lo + hi);
            alpha = an;
        }
        for (int d = 0; d < NV; ++d) a[d] += alpha * delta[d];
        if (exact && ls_piece_equal(piece, act, nrow)) {
            ++it;
            break; /* the Newton step was exact: a is the minimiser */
        }
    }
    /* constraint forces at the final acceleration */
    double f[MAXROW];
    for (int i = 0; i < nrow; ++i) {
        double s = 0.0;
        for (int d = 0; d < NV; ++d) s += J[i][d] * a[d];
        const double xi = s - aref[i];
        f[i] = xi < 0.0 ? -D[i] * xi : 0.0;
    }
    for (int d = 0; d < NV; ++d) {
        double s = 0.0;
        for (int i = 0; i < nrow; ++i) s += J[i][d] * f[i];
        dg->qfrc_constraint[d] = s;
        dg->qacc[d] = a[d];
        dg->qfrc_bias[d] = bias[d];
    }
    dg->ncon = c.n;
    dg->iters = it;
    for (int ci = 0; ci < c.n; ++ci) {
        const double *fe = f + 4 * ci;
        dg->geom[ci] = c.geom[ci];
        dg->dist[ci] = c.dist[ci];
        for (int i = 0; i < 3; ++i) dg->pos[ci][i] = c.pos[ci][i];
        dg->force[ci][0] = (fe[0] + fe[1]) + (fe[2] + fe[3]);
        dg->force[ci][1] = mu * (fe[0] - fe[1]);
        dg->force[ci][2] = mu * (fe[2] - fe[3]);
    }

    /* semi-implicit Euler: velocity first, then positions with the new velocity */
    for (int d = 0; d < NV; ++d) qvel[d] += h * a[d];
    for (int i = 0; i < 3; ++i) qpos[i] += h * qvel[i];
    {   /* quaternion: q <- q * exp(h w / 2), w in the trunk frame; renormalise */
        const double w[3] = {qvel[3], qvel[4], qvel[5]};
        const double wn = sqrt(dot3(w, w));
        double *q = qpos + 3;
        if (wn > 0.0) {
            const double ang = h * wn, s = sin(0.5 * ang) / wn, cc = cos(0.5 * ang);
            const double r[4] = {cc, s * w[0], s * w[1], s * w[2]};
            const double n0 = ((q[0] * r[0] - q[1] * r[1]) - q[2] * r[2]) - q[3] * r[3];
            const double n1 = ((q[0] * r[1] + q[1] * r[0]) + q[2] * r[3]) - q[3] * r[2];
            const double n2 = ((q[0] * r[2] - q[1] * r[3]) + q[2] * r[0]) + q[3] * r[1];
            const double n3 = ((q[0] * r[3] + q[1] * r[2]) - q[2] * r[1]) + q[3] * r[0];
            q[0] = n0; q[1] = n1; q[2] = n2; q[3] = n3;
        }
        const double qn = sqrt(((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3]);
        for (int i = 0; i < 4; ++i) q[i] = q[i] / qn;
    }
    for (int d = 6; d < NV; ++d) qpos[d + 1] += h * qvel[d];
    return 1;
}

static void sensors(const dk_phys_model *m, const tree_t *t, const double *qpos,
                    const double *qvel, double *s) {
    kin_t k;
    fk(t, qpos, &k);
    for (int i = 0; i < 4; ++i) s[i] = qpos[3 + i];
    for (int i = 0; i < 3; ++i) s[4 + i] = qvel[3 + i];
    mat_tvec3(k.xR[0], qvel, s + 7);
    for (int i = 0; i < 12; ++i) {
        s[10 + i] = qpos[7 + i];
        s[22 + i] = qvel[6 + i];
    }
    for (int l = 0; l < 4; ++l) {
        const int b2 = 3 + 3 * l;
        double off[3];
        mat_vec3(k.xR[b2], m->foot_pos[l], off);
        for (int i = 0; i < 3; ++i) s[34 + 3 * l + i] = k.xpos[b2][i] + off[i];
    }
}

/* ------------------------------------------------------------- exported */

/* Advance n worlds num_steps steps; the diag arrays (nullable) receive the
 * last step's outputs, laid out like dk_phys_diag.  Returns the number of
 * worlds that hit a non-SPD matrix (0 = ok). */
int orc_phys_step(const dk_phys_model *m, int64_t n, int64_t num_steps, double *qpos,
                  double *qvel, const double *ctrl, double *qacc, double *qfrc_bias,
                  double *qfrc_constraint, double *act_force, int32_t *ncon,
                  int32_t *contact_geom, double *contact_dist, double *contact_pos,
                  double *contact_force, int32_t *solver_iter, double *sensordata) {
    tree_t t;
    build_tree(m, &t);
    int bad = 0;
#pragma omp parallel for schedule(static) reduction(+ : bad)
    for (int64_t w = 0; w < n; ++w) {
        diag_t dg;
        memset(&dg, 0, sizeof(dg));
        double *qp = qpos + w * NQ, *qv = qvel + w * NV;
        for (int64_t s = 0; s < num_steps; ++s)
            if (!step_world(m, &t, qp, qv, ctrl + w * 12, &dg)) {
                ++bad;
                break;
            }
        for (int d = 0; d < NV; ++d) {
            if (qacc) qacc[w * NV + d] = dg.qacc[d];
            if (qfrc_bias) qfrc_bias[w * NV + d] = dg.qfrc_bias[d];
            if (qfrc_constraint) qfrc_constraint[w * NV + d] = dg.qfrc_constraint[d];
        }
        if (act_force)
            for (int i = 0; i < 12; ++i) act_force[w * 12 + i] = dg.act[i];
        if (ncon) ncon[w] = dg.ncon;
        if (solver_iter) solver_iter[w] = dg.iters;
        for (int ci = 0; ci < DK_PHYS_MAXCON; ++ci) {
            const int v = ci < dg.ncon;
            if (contact_geom) {
                contact_geom[(w * DK_PHYS_MAXCON + ci) * 2] = v ? 0 : -1;
                contact_geom[(w * DK_PHYS_MAXCON + ci) * 2 + 1] = v ? dg.geom[ci] : -1;
            }
            if (contact_dist) contact_dist[w * DK_PHYS_MAXCON + ci] = v ? dg.dist[ci] : 0.0;
            for (int i = 0; i < 3; ++i) {
                if (contact_pos) contact_pos[(w * DK_PHYS_MAXCON + ci) * 3 + i] = v ? dg.pos[ci][i] : 0.0;
                if (contact_force)
                    contact_force[(w * DK_PHYS_MAXCON + ci) * 3 + i] = v ? dg.force[ci][i] : 0.0;
            }
        }
        if (sensordata) sensors(m, &t, qp, qv, sensordata + w * DK_PHYS_NSENSOR);
    }
    return bad;
}

/* G1 inspection: M (with armature), bias, xpos, xipos of n worlds */
void orc_phys_inspect(const dk_phys_model *m, int64_t n, const double *qpos, const double *qvel,
                      double *Mout, double *bias, double *xpos, double *xipos) {
    tree_t t;
    build_tree(m, &t);
#pragma omp parallel for schedule(static)
    for (int64_t w = 0; w < n; ++w) {
        kin_t k;
        fk(&t, qpos + w * NQ, &k);
        if (Mout) {
            double M[NV][NV];
            mass_matrix(&t, &k, M);
            memcpy(Mout + w * NV * NV, M, sizeof(M));
        }
        if (bias) rne(m, &t, &k, qvel + w * NV, NULL, bias + w * NV);
        for (int b = 0; b < NB; ++b)
            for (int i = 0; i < 3; ++i) {
                if (xpos) xpos[(w * NB + b) * 3 + i] = k.xpos[b][i];
                if (xipos) xipos[(w * NB + b) * 3 + i] = k.xipos[b][i];
            }
    }
}

/* inverse dynamics (KAT support): qfrc = M qacc + bias via RNE with qacc */
void orc_phys_inverse(const dk_phys_model *m, int64_t n, const double *qpos, const double *qvel,
                      const double *qacc, double *qfrc) {
    tree_t t;
    build_tree(m, &t);
    for (int64_t w = 0; w < n; ++w) {
        kin_t k;
        fk(&t, qpos + w * NQ, &k);
        rne(m, &t, &k, qvel + w * NV, qacc + w * NV, qfrc + w * NV);
    }
}

/* kinetic energy from body velocities (independent of M) and potential energy */
void orc_phys_energy(const dk_phys_model *m, int64_t n, const double *qpos, const double *qvel,
                     double *kinetic, double *potential, double *momentum6) {
    tree_t t;
    build_tree(m, &t);
    for (int64_t w = 0; w < n; ++w) {
        kin_t k;
        fk(&t, qpos + w * NQ, &k);
        const double *qv = qvel + w * NV;
        double cvel[NB][6];
        double ke = 0.0, pe = 0.0, P[6] = {0};
        for (int b = 0; b < NB; ++b) {
            const int p = t.parent[b];
            for (int i = 0; i < 6; ++i) cvel[b][i] = p < 0 ? 0.0 : cvel[p][i];
            for (int d = t.dofadr[b]; d < t.dofadr[b] + t.dofnum[b]; ++d)
                for (int i = 0; i < 6; ++i) cvel[b][i] += k.cdof[d][i] * qv[d];
            /* com velocity and body-frame angular velocity */
            double r[3], wr[3], vc[3], wl[3];
            for (int i = 0; i < 3; ++i) r[i] = k.xipos[b][i] - k.p0[i];
            cross3(cvel[b], r, wr);
            for (int i = 0; i < 3; ++i) vc[i] = cvel[b][3 + i] + wr[i];
            mat_tvec3(k.xR[b], cvel[b], wl);
            const double mb = t.mass[b];
            ke += 0.5 * mb * dot3(vc, vc);
            for (int i = 0; i < 3; ++i) ke += 0.5 * t.inertia[b][i] * wl[i] * wl[i];
            pe -= mb * dot3(m->gravity, k.xipos[b]);
            /* momentum about the world origin: linear m vc, angular x m vc + I w */
            double Iw[3], Iwl[3], xm[3];
            for (int i = 0; i < 3; ++i) Iwl[i] = t.inertia[b][i] * wl[i];
            mat_vec3(k.xR[b], Iwl, Iw);
            double mv[3] = {mb * vc[0], mb * vc[1], mb * vc[2]};
            cross3(k.xipos[b], mv, xm);
            for (int i = 0; i < 3; ++i) {
                P[i] += mv[i];
                P[3 + i] += xm[i] + Iw[i];
            }
        }
        kinetic[w] = ke;
        potential[w] = pe;
        if (momentum6)
            for (int i = 0; i < 6; ++i) momentum6[w * 6 + i] = P[i];
    }
}

/* foot sphere centres [n][4][3] and their world velocities J(q) qvel [n][4][3] */
void orc_phys_foot_kin(const dk_phys_model *m, int64_t n, const double *qpos, const double *qvel,
                       double *pos, double *vel) {
    tree_t t;
    build_tree(m, &t);
    for (int64_t w = 0; w < n; ++w) {
        kin_t k;
        fk(&t, qpos + w * NQ, &k);
        for (int l = 0; l < 4; ++l) {
            const int b2 = 3 + 3 * l;
            double off[3], f[3], J[3][NV];
            mat_vec3(k.xR[b2], m->foot_pos[l], off);
            for (int i = 0; i < 3; ++i) f[i] = k.xpos[b2][i] + off[i];
            point_jac(&t, &k, b2, f, J);
            for (int i = 0; i < 3; ++i) {
                double s = 0.0;
                for (int d = 0; d < NV; ++d) s += J[i][d] * qvel[w * NV + d];
                pos[(w * 4 + l) * 3 + i] = f[i];
                vel[(w * 4 + l) * 3 + i] = s;
            }
        }
    }
}
