// capi_phys.cu -- extern "C" entry points of the articulated contact physics
// step (include/deskrl_b200.h "Articulated contact physics", SURVEY.md §8a
// G1-G4).  The handle owns the per-world state in HBM as structure of arrays
// (qpos [NQ][N], qvel [NV][N]); callers exchange row-major [N, NQ] / [N, NV]
// device buffers through dk_phys_set_state / dk_phys_get_state.
#include <cmath>
#include <cstdio>
#include <cstring>

#include "../../include/deskrl_b200.h"
#include "physics.cuh"

namespace dk {
namespace phys {
DK_PHYS_DECLARE(float)
DK_PHYS_DECLARE(double)
}  // namespace phys
}  // namespace dk

extern "C" int dk_internal_fail(int code, const char *msg);  // capi.cu

struct dk_phys {
    dk_phys_model model;
    int dtype = DK_F32;
    int device = 0;
    int64_t n = 0;
    void *qpos = nullptr;  // SoA [NQ][n]
    void *qvel = nullptr;  // SoA [NV][n]
    int32_t *bad = nullptr;
    int64_t launches = 0;
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

int validate(const dk_phys_model &m) {
    if (!(m.timestep > 0)) return dk_internal_fail(DK_ERR_CONFIG, "timestep must be > 0");
    if (!(m.solimp > 0 && m.solimp < 1))
        return dk_internal_fail(DK_ERR_CONFIG, "solimp must be in (0, 1)");
    if (!(m.solref[0] > 0 && m.solref[1] > 0))
        return dk_internal_fail(DK_ERR_CONFIG, "solref must be positive");
    if (m.iterations < 1 || m.ls_iterations < 1)
        return dk_internal_fail(DK_ERR_CONFIG, "iterations and ls_iterations must be >= 1");
    if (!(m.friction >= 0)) return dk_internal_fail(DK_ERR_CONFIG, "friction must be >= 0");
    if (!(m.base_mass > 0)) return dk_internal_fail(DK_ERR_CONFIG, "base_mass must be > 0");
    for (int l = 0; l < 4; ++l)
        for (int j = 0; j < 3; ++j) {
            const double *a = m.jnt_axis[l][j];
            const double nn = a[0] * a[0] + a[1] * a[1] + a[2] * a[2];
            if (std::fabs(nn - 1.0) > 1e-9)
                return dk_internal_fail(DK_ERR_CONFIG, "joint axes must be unit vectors");
            if (!(m.body_mass[l][j] > 0))
                return dk_internal_fail(DK_ERR_CONFIG, "body masses must be > 0");
            if (!(m.jnt_range[l][j][0] <= m.jnt_range[l][j][1]))
                return dk_internal_fail(DK_ERR_CONFIG, "joint range lower > upper");
        }
    return DK_OK;
}

template <typename T>
dk::phys::PhysConst<T> make_const(const dk_phys_model &m) {
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
    // the oracle's expressions, evaluated in double
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
int run(dk_phys *p, int64_t steps, const void *ctrl, const dk_phys_diag *d,
        const dk::phys::PhysInspect<T> &ins, cudaStream_t st) {
    dk::phys::PhysArgs<T> a;
    memset(&a, 0, sizeof(a));
    a.n = p->n;
    a.num_steps = steps;
    a.qpos = (T *)p->qpos;
    a.qvel = (T *)p->qvel;
    a.ctrl = (const T *)ctrl;
    a.bad = p->bad;
    if (d) {
        a.qacc = (T *)d->qacc;
        a.qfrc_bias = (T *)d->qfrc_bias;
        a.qfrc_constraint = (T *)d->qfrc_constraint;
        a.act_force = (T *)d->act_force;
        a.ncon = d->ncon;
        a.contact_geom = d->contact_geom;
        a.contact_dist = (T *)d->contact_dist;
        a.contact_pos = (T *)d->contact_pos;
        a.contact_force = (T *)d->contact_force;
        a.solver_iter = d->solver_iter;
        a.sensordata = (T *)d->sensordata;
    }
    const auto c = make_const<T>(p->model);
    p->launches += 1;
    return cuda_rc(dk::phys::launch_phys<T>(c, a, ins, st), "phys_kernel");
}

}  // namespace

extern "C" {

int dk_phys_default_model(dk_phys_model *m) {
    if (!m) return dk_internal_fail(DK_ERR_INVALID_INPUT, "null model");
    memset(m, 0, sizeof(*m));
    m->timestep = 0.004;
    m->gravity[2] = -9.81;
    m->friction = 0.6;
    m->solref[0] = 0.02;
    m->solref[1] = 1.0;
    m->solimp = 0.9;
    m->base_mass = 5.204;
    const double bipos[3] = {0.0223, 0.002, -0.0005};
    const double binert[3] = {0.0168128557, 0.063009565, 0.0716547275};
    const double bbox[3] = {0.1881, 0.04675, 0.057};
    for (int i = 0; i < 3; ++i) {
        m->base_ipos[i] = bipos[i];
        m->base_inertia[i] = binert[i];
        m->base_box[i] = bbox[i];
    }
    const double fxs[4] = {1, 1, -1, -1}, sys[4] = {-1, 1, -1, 1};  // FR FL RR RL
    for (int l = 0; l < 4; ++l) {
        const double fx = fxs[l], sy = sys[l];
        const double pos[3][3] = {{0.1881 * fx, 0.04675 * sy, 0.0}, {0.0, 0.08 * sy, 0.0},
                                  {0.0, 0.0, -0.213}};
        const double ax[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 1, 0}};
        const double mass[3] = {0.680, 1.009, 0.195862};
        const double ipos[3][3] = {{-0.005657 * fx, 0.008752 * sy, -0.000102},
                                   {-0.003342, -0.018054 * sy, -0.033451},
                                   {0.00429862, 0.000976676 * sy, -0.146197}};
        const double inert[3][3] = {{0.000334008, 0.000619101, 0.00040057},
                                    {0.00443176, 0.00448537, 0.000740309},
                                    {0.0011454, 0.0011588, 0.0000266}};
        const double range[3][2] = {{-0.863, 0.863}, {-0.686, 4.501}, {-2.818, -0.888}};
        const double tlim[3] = {23.7, 23.7, 35.55};
        for (int j = 0; j < 3; ++j) {
            for (int i = 0; i < 3; ++i) {
                m->body_pos[l][j][i] = pos[j][i];
                m->jnt_axis[l][j][i] = ax[j][i];
                m->body_ipos[l][j][i] = ipos[j][i];
                m->body_inertia[l][j][i] = inert[j][i];
            }
            m->body_mass[l][j] = mass[j];
            m->jnt_range[l][j][0] = range[j][0];
            m->jnt_range[l][j][1] = range[j][1];
            m->dof_damping[l][j] = 0.1;
            m->dof_armature[l][j] = 0.005;
            m->torque_limit[l][j] = tlim[j];
        }
        m->foot_pos[l][2] = -0.213;
    }
    m->kp = 35.0;
    m->kd = 0.5;
    m->foot_radius = 0.023;
    m->thigh_radius = 0.0245;
    m->iterations = 4;
    m->ls_iterations = 8;
    m->collide_box = 0;
    m->collide_thigh = 0;
    return DK_OK;
}

int dk_phys_create(const dk_phys_model *model, int dtype, int64_t n, int device, dk_phys **out) {
    if (!model || !out) return dk_internal_fail(DK_ERR_INVALID_INPUT, "null argument");
    *out = nullptr;
    if (dtype != DK_F32 && dtype != DK_F64)
        return dk_internal_fail(DK_ERR_CONFIG, "dtype must be DK_F32 or DK_F64");
    if (n < 1) return dk_internal_fail(DK_ERR_CONFIG, "num_worlds must be >= 1");
    int rc = validate(*model);
    if (rc) return rc;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev)
        return dk_internal_fail(DK_ERR_CUDA, "no such CUDA device");
    Guard g(device);
    dk_phys *p = new dk_phys;
    p->model = *model;
    p->dtype = dtype;
    p->device = device;
    p->n = n;
    const size_t esz = dtype == DK_F64 ? 8 : 4;
    cudaError_t e = cudaMalloc(&p->qpos, esz * DK_PHYS_NQ * n);
    if (e == cudaSuccess) e = cudaMalloc(&p->qvel, esz * DK_PHYS_NV * n);
    if (e == cudaSuccess) e = cudaMalloc((void **)&p->bad, sizeof(int32_t));
    if (e == cudaSuccess) e = cudaMemset(p->qvel, 0, esz * DK_PHYS_NV * n);
    if (e == cudaSuccess) e = cudaMemset(p->bad, 0, sizeof(int32_t));
    if (e == cudaSuccess) {  // every world at the home keyframe
        const double home[DK_PHYS_NQ] = {0, 0, 0.278, 1, 0, 0, 0, 0, 0.9, -1.8, 0, 0.9, -1.8,
                                         0, 0.9, -1.8, 0, 0.9, -1.8};
        for (int c = 0; c < DK_PHYS_NQ && e == cudaSuccess; ++c) {
            if (dtype == DK_F64) {
                double *tmp = new double[n];
                for (int64_t i = 0; i < n; ++i) tmp[i] = home[c];
                e = cudaMemcpy((double *)p->qpos + c * n, tmp, 8 * n, cudaMemcpyHostToDevice);
                delete[] tmp;
            } else {
                float *tmp = new float[n];
                for (int64_t i = 0; i < n; ++i) tmp[i] = (float)home[c];
                e = cudaMemcpy((float *)p->qpos + c * n, tmp, 4 * n, cudaMemcpyHostToDevice);
                delete[] tmp;
            }
        }
    }
    if (e != cudaSuccess) {
        cudaFree(p->qpos);
        cudaFree(p->qvel);
        cudaFree(p->bad);
        delete p;
        return cuda_rc(e, "dk_phys_create");
    }
    *out = p;
    return DK_OK;
}

int dk_phys_destroy(dk_phys *p) {
    if (!p) return DK_OK;
    Guard g(p->device);
    cudaFree(p->qpos);
    cudaFree(p->qvel);
    cudaFree(p->bad);
    delete p;
    return DK_OK;
}

int dk_phys_set_state(dk_phys *p, const void *qpos, const void *qvel, void *stream) {
    if (!p) return dk_internal_fail(DK_ERR_INVALID_INPUT, "null handle");
    Guard g(p->device);
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e = cudaSuccess;
    if (p->dtype == DK_F64) {
        if (qpos) e = dk::phys::launch_transpose<double>((const double *)qpos, (double *)p->qpos,
                                                         p->n, DK_PHYS_NQ, true, st);
        if (e == cudaSuccess && qvel)
            e = dk::phys::launch_transpose<double>((const double *)qvel, (double *)p->qvel, p->n,
                                                   DK_PHYS_NV, true, st);
    } else {
        if (qpos) e = dk::phys::launch_transpose<float>((const float *)qpos, (float *)p->qpos,
                                                        p->n, DK_PHYS_NQ, true, st);
        if (e == cudaSuccess && qvel)
            e = dk::phys::launch_transpose<float>((const float *)qvel, (float *)p->qvel, p->n,
                                                  DK_PHYS_NV, true, st);
    }
    return cuda_rc(e, "dk_phys_set_state");
}

int dk_phys_get_state(dk_phys *p, void *qpos, void *qvel, void *stream) {
    if (!p) return dk_internal_fail(DK_ERR_INVALID_INPUT, "null handle");
    Guard g(p->device);
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e = cudaSuccess;
    if (p->dtype == DK_F64) {
        if (qpos) e = dk::phys::launch_transpose<double>((const double *)p->qpos, (double *)qpos,
                                                         p->n, DK_PHYS_NQ, false, st);
        if (e == cudaSuccess && qvel)
            e = dk::phys::launch_transpose<double>((const double *)p->qvel, (double *)qvel, p->n,
                                                   DK_PHYS_NV, false, st);
    } else {
        if (qpos) e = dk::phys::launch_transpose<float>((const float *)p->qpos, (float *)qpos,
                                                        p->n, DK_PHYS_NQ, false, st);
        if (e == cudaSuccess && qvel)
            e = dk::phys::launch_transpose<float>((const float *)p->qvel, (float *)qvel, p->n,
                                                  DK_PHYS_NV, false, st);
    }
    return cuda_rc(e, "dk_phys_get_state");
}

int dk_phys_step(dk_phys *p, int64_t num_steps, const void *ctrl, const dk_phys_diag *diag,
                 void *stream) {
    if (!p) return dk_internal_fail(DK_ERR_INVALID_INPUT, "null handle");
    if (!ctrl) return dk_internal_fail(DK_ERR_INVALID_INPUT, "null ctrl");
    if (num_steps < 0) return dk_internal_fail(DK_ERR_INVALID_INPUT, "num_steps must be >= 0");
    if (num_steps == 0) return DK_OK;
    Guard g(p->device);
    cudaStream_t st = (cudaStream_t)stream;
    if (p->dtype == DK_F64) return run<double>(p, num_steps, ctrl, diag, {}, st);
    return run<float>(p, num_steps, ctrl, diag, {}, st);
}

int dk_phys_inspect(dk_phys *p, void *M, void *bias, void *xpos, void *xipos, void *stream) {
    if (!p) return dk_internal_fail(DK_ERR_INVALID_INPUT, "null handle");
    if (!M && !bias && !xpos && !xipos) return DK_OK;
    Guard g(p->device);
    cudaStream_t st = (cudaStream_t)stream;
    // ctrl is not read in inspection mode; pass the state buffer as a dummy
    if (p->dtype == DK_F64) {
        dk::phys::PhysInspect<double> ins{(double *)M, (double *)bias, (double *)xpos,
                                          (double *)xipos};
        return run<double>(p, 0, p->qpos, nullptr, ins, st);
    }
    dk::phys::PhysInspect<float> ins{(float *)M, (float *)bias, (float *)xpos, (float *)xipos};
    return run<float>(p, 0, p->qpos, nullptr, ins, st);
}

int dk_phys_check(dk_phys *p) {
    if (!p) return dk_internal_fail(DK_ERR_INVALID_INPUT, "null handle");
    Guard g(p->device);
    int32_t bad = 0;
    cudaError_t e = cudaMemcpy(&bad, p->bad, sizeof(int32_t), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_rc(e, "dk_phys_check");
    if (bad) {
        cudaMemset(p->bad, 0, sizeof(int32_t));
        return dk_internal_fail(DK_ERR_INVALID_INPUT,
                                "physics step: mass or Hessian matrix not positive definite "
                                "(non-finite state or control?)");
    }
    return DK_OK;
}

int64_t dk_phys_kernel_launches(const dk_phys *p) { return p ? p->launches : 0; }

}  // extern "C"
