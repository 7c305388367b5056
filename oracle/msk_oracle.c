/* TEST INFRASTRUCTURE ONLY — plain-C fp64 restatement of the reference hot
 * path (see msk_oracle.h for the file list).  Every function cites the
 * reference lines it restates.  Evaluation order follows the reference (and
 * the Eigen-shim semantics) so the two agree to ~1e-15; the build uses
 * -ffp-contract=off so no FMA contraction changes rounding.
 */
#include "msk_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define K_SIM_DT 0.002   /* skeleton.hpp:11 */
#define K_CTRL_DT 0.02   /* skeleton.hpp:12 */
#define K_SUBSTEPS 10    /* skeleton.hpp:13 */
#define K_MIN_FIBER 0.01 /* skeleton.hpp:14 */
#define MAX_NQ 512
#define MAX_NL 512

int32_t om_nq(const om_model *m) { return (m->floating ? 3 : 0) + m->n_joints; }
static int32_t nrd(const om_model *m) { return m->floating ? 3 : 0; }
int32_t om_obs_dim(const om_model *m) {           /* env.cpp:165-168 */
    return 3 * om_nq(m) + 6 * m->n_key + 4 * m->n_muscles;
}
int32_t om_delta_dim(const om_model *m) {         /* env.hpp:25-27 */
    return 3 + m->n_joints + 2 * m->n_key;
}

/* ---- muscle.cpp:9-56 ---------------------------------------------------- */
double om_force_length_active(double l_m) {
    const double d = (l_m - 1.0) / 0.45;
    return exp(-d * d);
}
double om_force_velocity(double v_m) {
    if (v_m <= -1.0) return 0.0;
    if (v_m < 0.0) return (v_m + 1.0) / (1.0 - v_m / 4.0);
    const double slope0 = 1.0 + 1.0 / 4.0;
    const double c = (1.4 - 1.0) / slope0;
    return (1.4 * v_m + c) / (v_m + c);
}
double om_force_passive(double l_m) {
    if (l_m <= 1.0) return 0.0;
    const double num = exp(4.0 * (l_m - 1.0)) - 1.0;
    const double den = exp(4.0 * 0.5) - 1.0;
    return num / den;
}
double om_mtu_force(double act, double l_m, double v_m, double f_max) {
    return f_max * (act * om_force_length_active(l_m) * om_force_velocity(v_m) + om_force_passive(l_m));
}
double om_activation_step(double act, double u, double dt, double tau_act, double tau_deact) {
    const double gain = 0.5 + 1.5 * act;                        /* muscle.cpp:43 */
    const double tau = u > act ? tau_act * gain : tau_deact / gain;
    double next = u + (act - u) * exp(-dt / tau);               /* muscle.cpp:52 */
    if (next < 0.0) next = 0.0;
    if (next > 1.0) next = 1.0;
    return next;
}
double om_wrap_angle(double a) {                                /* env.cpp:10-15 */
    const double pi = 3.14159265358979323846;
    a = fmod(a + pi, 2.0 * pi);
    if (a <= 0.0) a += 2.0 * pi;
    return a - pi;
}

/* ---- skeleton.cpp:82-127 ------------------------------------------------ */
typedef struct kin {
    double origin[2 * MAX_NL];
    double angle[MAX_NL];
    double anchor[2 * MAX_NL];
} kin_t;

static void fk(const om_model *m, const double *q, kin_t *k) {
    const int fc = m->floating ? 1 : 0;
    if (m->floating) {
        k->origin[0] = q[0];
        k->origin[1] = q[1];
        k->angle[0] = q[2];
    }
    for (int j = 0; j < m->n_joints; ++j) {
        const int child = fc + j, p = m->joint_parent[j];
        double po0 = 0.0, po1 = 0.0, pa = 0.0;
        if (p >= 0) {
            po0 = k->origin[2 * p];
            po1 = k->origin[2 * p + 1];
            pa = k->angle[p];
        }
        const double c = cos(pa), s = sin(pa);
        const double ax = m->joint_anchor[2 * j], az = m->joint_anchor[2 * j + 1];
        const double w0 = po0 + (c * ax + (-s) * az);
        const double w1 = po1 + (s * ax + c * az);
        k->anchor[2 * j] = w0;
        k->anchor[2 * j + 1] = w1;
        k->origin[2 * child] = w0;
        k->origin[2 * child + 1] = w1;
        k->angle[child] = pa + m->joint_mount[j] + q[nrd(m) + j];
    }
}

void om_forward_kinematics(const om_model *m, const double *q, double *origin, double *angle,
                           double *anchors) {
    static __thread kin_t k;
    fk(m, q, &k);
    memcpy(origin, k.origin, sizeof(double) * 2 * (size_t)m->n_links);
    memcpy(angle, k.angle, sizeof(double) * (size_t)m->n_links);
    memcpy(anchors, k.anchor, sizeof(double) * 2 * (size_t)m->n_joints);
}

static void world_point(const kin_t *k, int link, double lx, double lz, double *out) {
    if (link < 0) {
        out[0] = lx;
        out[1] = lz;
        return;
    }
    const double c = cos(k->angle[link]), s = sin(k->angle[link]);
    out[0] = k->origin[2 * link] + (c * lx + (-s) * lz);
    out[1] = k->origin[2 * link + 1] + (s * lx + c * lz);
}

/* joint_path (skeleton.cpp:23-34): joints root-first; returns count. */
static int joint_path(const om_model *m, int link, int *path) {
    int tmp[MAX_NL], n = 0;
    const int fc = m->floating ? 1 : 0;
    int cur = link;
    while (cur >= fc) {
        const int j = cur - fc;
        tmp[n++] = j;
        cur = m->joint_parent[j];
    }
    for (int i = 0; i < n; ++i) path[i] = tmp[n - 1 - i];
    return n;
}

/* point_jacobian (skeleton.cpp:115-127): J is 2 x nq, stored J[r*nq + c]. */
static void point_jacobian(const om_model *m, const kin_t *k, int link, const double *p, double *J) {
    const int nq = om_nq(m);
    memset(J, 0, sizeof(double) * 2 * (size_t)nq);
    if (link < 0) return;
    if (m->floating) {
        J[0 * nq + 0] = 1.0;
        J[1 * nq + 1] = 1.0;
        J[0 * nq + 2] = -(p[1] - k->origin[1]);
        J[1 * nq + 2] = p[0] - k->origin[0];
    }
    int path[MAX_NL];
    const int n = joint_path(m, link, path);
    for (int i = 0; i < n; ++i) {
        const int j = path[i], col = nrd(m) + j;
        J[0 * nq + col] = -(p[1] - k->anchor[2 * j + 1]);
        J[1 * nq + col] = p[0] - k->anchor[2 * j];
    }
}

/* mtu_length (skeleton.cpp:129-141) */
static double mtu_length_k(const om_model *m, const kin_t *k, int mu) {
    const int a = m->m_via_start[mu], b = m->m_via_start[mu + 1];
    double len = 0.0, prev[2], cur[2];
    world_point(k, m->via_link[a], m->via_offset[2 * a], m->via_offset[2 * a + 1], prev);
    for (int v = a + 1; v < b; ++v) {
        world_point(k, m->via_link[v], m->via_offset[2 * v], m->via_offset[2 * v + 1], cur);
        const double dx = cur[0] - prev[0], dz = cur[1] - prev[1];
        len += sqrt((0.0 + dx * dx) + dz * dz);
        prev[0] = cur[0];
        prev[1] = cur[1];
    }
    return len;
}

double om_mtu_length(const om_model *m, const double *q, int32_t muscle) {
    static __thread kin_t k;
    fk(m, q, &k);
    return mtu_length_k(m, &k, muscle);
}

/* moment_arms (skeleton.cpp:147-170) */
static void moment_arms_k(const om_model *m, const kin_t *k, double *Jm) {
    const int nq = om_nq(m);
    double Jp[2 * MAX_NQ], Jc[2 * MAX_NQ], dL[MAX_NQ];
    for (int mu = 0; mu < m->n_muscles; ++mu) {
        const int a = m->m_via_start[mu], b = m->m_via_start[mu + 1];
        double pp[2], pc[2];
        world_point(k, m->via_link[a], m->via_offset[2 * a], m->via_offset[2 * a + 1], pp);
        point_jacobian(m, k, m->via_link[a], pp, Jp);
        for (int c = 0; c < nq; ++c) dL[c] = 0.0;
        for (int v = a + 1; v < b; ++v) {
            world_point(k, m->via_link[v], m->via_offset[2 * v], m->via_offset[2 * v + 1], pc);
            point_jacobian(m, k, m->via_link[v], pc, Jc);
            const double s0 = pc[0] - pp[0], s1 = pc[1] - pp[1];
            const double len = sqrt((0.0 + s0 * s0) + s1 * s1);
            if (len > 1e-12) {
                const double u0 = s0 / len, u1 = s1 / len;
                for (int c = 0; c < nq; ++c)
                    dL[c] += (0.0 + u0 * (Jc[c] - Jp[c])) + u1 * (Jc[nq + c] - Jp[nq + c]);
            }
            pp[0] = pc[0];
            pp[1] = pc[1];
            memcpy(Jp, Jc, sizeof(double) * 2 * (size_t)nq);
        }
        for (int c = 0; c < nq; ++c) Jm[(size_t)mu * nq + c] = -dL[c];
    }
}

void om_moment_arms(const om_model *m, const double *q, double *Jm) {
    static __thread kin_t k;
    fk(m, q, &k);
    moment_arms_k(m, &k, Jm);
}

/* mass_matrix (skeleton.cpp:172-189) */
static void mass_matrix_k(const om_model *m, const kin_t *k, double *M) {
    const int nq = om_nq(m);
    double J[2 * MAX_NQ], Jw[MAX_NQ], com[2];
    int path[MAX_NL];
    memset(M, 0, sizeof(double) * (size_t)nq * nq);
    for (int l = 0; l < m->n_links; ++l) {
        world_point(k, l, m->link_com[l], 0.0, com);
        point_jacobian(m, k, l, com, J);
        for (int c = 0; c < nq; ++c) Jw[c] = 0.0;
        if (m->floating) Jw[2] = 1.0;
        const int n = joint_path(m, l, path);
        for (int i = 0; i < n; ++i) Jw[nrd(m) + path[i]] = 1.0;
        const double ms = m->link_mass[l], in = m->link_inertia[l];
        for (int j = 0; j < nq; ++j)
            for (int i = j; i < nq; ++i) {
                const double s = (0.0 + J[i] * J[j]) + J[nq + i] * J[nq + j];
                M[i * nq + j] += ms * s;
            }
        for (int j = 0; j < nq; ++j)
            for (int i = j; i < nq; ++i) M[i * nq + j] += in * (0.0 + Jw[i] * Jw[j]);
    }
    for (int i = 0; i < nq; ++i)
        for (int j = i + 1; j < nq; ++j) M[i * nq + j] = M[j * nq + i];
}

void om_mass_matrix(const om_model *m, const double *q, double *M) {
    static __thread kin_t k;
    fk(m, q, &k);
    mass_matrix_k(m, &k, M);
}

/* velocity_kinematics (skeleton.cpp:43-72) */
typedef struct velkin {
    double omega[MAX_NL];
    double v_origin[2 * MAX_NL];
    double anchor_vel[2 * MAX_NL];
} velkin_t;

static void velocity_kinematics(const om_model *m, const kin_t *k, const double *dq, velkin_t *vk) {
    const int fc = m->floating ? 1 : 0;
    if (m->floating) {
        vk->v_origin[0] = dq[0];
        vk->v_origin[1] = dq[1];
        vk->omega[0] = dq[2];
    }
    for (int j = 0; j < m->n_joints; ++j) {
        const int child = fc + j, p = m->joint_parent[j];
        double po = 0.0, av0 = 0.0, av1 = 0.0;
        if (p >= 0) {
            po = vk->omega[p];
            const double r0 = k->anchor[2 * j] - k->origin[2 * p];
            const double r1 = k->anchor[2 * j + 1] - k->origin[2 * p + 1];
            av0 = vk->v_origin[2 * p] + po * (-r1);
            av1 = vk->v_origin[2 * p + 1] + po * r0;
        }
        vk->anchor_vel[2 * j] = av0;
        vk->anchor_vel[2 * j + 1] = av1;
        vk->omega[child] = po + dq[nrd(m) + j];
        vk->v_origin[2 * child] = av0;
        vk->v_origin[2 * child + 1] = av1;
    }
}

/* material_point_velocity (skeleton.cpp:74-78) */
static void point_velocity(const velkin_t *vk, const kin_t *k, int link, const double *p, double *v) {
    if (link < 0) {
        v[0] = v[1] = 0.0;
        return;
    }
    const double r0 = p[0] - k->origin[2 * link], r1 = p[1] - k->origin[2 * link + 1];
    v[0] = vk->v_origin[2 * link] + vk->omega[link] * (-r1);
    v[1] = vk->v_origin[2 * link + 1] + vk->omega[link] * r0;
}

/* bias_forces (skeleton.cpp:191-233) */
static void bias_forces_k(const om_model *m, const kin_t *k, const double *q, const double *dq,
                          double *C) {
    const int nq = om_nq(m);
    velkin_t vk;
    velocity_kinematics(m, k, dq, &vk);
    double J[2 * MAX_NQ], com[2], vc[2];
    int path[MAX_NL];
    for (int i = 0; i < nq; ++i) C[i] = 0.0;
    for (int l = 0; l < m->n_links; ++l) {
        world_point(k, l, m->link_com[l], 0.0, com);
        point_jacobian(m, k, l, com, J);
        point_velocity(&vk, k, l, com, vc);
        double ab0 = 0.0, ab1 = 0.0;
        if (m->floating) {
            const double d0 = vc[0] - dq[0], d1 = vc[1] - dq[1];
            ab0 += dq[2] * (-d1);
            ab1 += dq[2] * d0;
        }
        const int n = joint_path(m, l, path);
        for (int i = 0; i < n; ++i) {
            const int j = path[i];
            const double d0 = vc[0] - vk.anchor_vel[2 * j], d1 = vc[1] - vk.anchor_vel[2 * j + 1];
            ab0 += dq[nrd(m) + j] * (-d1);
            ab1 += dq[nrd(m) + j] * d0;
        }
        const double ms = m->link_mass[l];
        for (int c = 0; c < nq; ++c) {
            const double jt_a = (0.0 + J[c] * ab0) + J[nq + c] * ab1;
            C[c] += ms * jt_a;
        }
        for (int c = 0; c < nq; ++c) {
            const double jt_g = (0.0 + J[c] * 0.0) + J[nq + c] * m->gravity;
            C[c] -= ms * jt_g;
        }
    }
    for (int j = 0; j < m->n_joints; ++j) {
        const int d = nrd(m) + j;
        C[d] += m->joint_damping[j] * dq[d];
        if (q[d] > m->joint_hi[j])
            C[d] += m->joint_limit_stiffness * (q[d] - m->joint_hi[j]);
        else if (q[d] < m->joint_lo[j])
            C[d] += m->joint_limit_stiffness * (q[d] - m->joint_lo[j]);
    }
}

void om_bias_forces(const om_model *m, const double *q, const double *dq, double *C) {
    static __thread kin_t k;
    fk(m, q, &k);
    bias_forces_k(m, &k, q, dq, C);
}

/* contact_forces (skeleton.cpp:235-262) */
static void contact_forces_k(const om_model *m, const kin_t *k, const double *dq, double *tau,
                             double *sf) {
    const int nq = om_nq(m);
    velkin_t vk;
    velocity_kinematics(m, k, dq, &vk);
    double J[2 * MAX_NQ], c[2], vcn[2], cp[2], vcp[2];
    for (int i = 0; i < nq; ++i) tau[i] = 0.0;
    for (int s = 0; s < m->n_spheres; ++s) {
        sf[2 * s] = sf[2 * s + 1] = 0.0;
        const int link = m->sphere_link[s];
        world_point(k, link, m->sphere_offset[2 * s], m->sphere_offset[2 * s + 1], c);
        const double pen = m->sphere_radius[s] - c[1];
        if (pen <= 0.0) continue;
        point_velocity(&vk, k, link, c, vcn);
        double fn = m->contact_k * pen - m->contact_c * vcn[1];
        if (fn < 0.0) fn = 0.0;
        if (fn <= 0.0) continue;
        cp[0] = c[0] - 0.0;
        cp[1] = c[1] - m->sphere_radius[s];
        point_velocity(&vk, k, link, cp, vcp);
        const double ft = -m->contact_mu * fn * tanh(vcp[0] / m->contact_vs);
        sf[2 * s] = ft;
        sf[2 * s + 1] = fn;
        point_jacobian(m, k, link, cp, J);
        for (int i = 0; i < nq; ++i) tau[i] += (0.0 + J[i] * ft) + J[nq + i] * fn;
    }
}

void om_contact_forces(const om_model *m, const double *q, const double *dq, double *tau, double *sf) {
    static __thread kin_t k;
    fk(m, q, &k);
    contact_forces_k(m, &k, dq, tau, sf);
}

/* Eigen::LDLT stand-in: diagonal pivoting LDL^T, in place on a copy. */
static void ldlt_solve(int n, const double *Min, const double *b, double *x) {
    static __thread double a[MAX_NQ * MAX_NQ];
    int perm[MAX_NQ];
    double y[MAX_NQ];
    memcpy(a, Min, sizeof(double) * (size_t)n * n);
    for (int i = 0; i < n; ++i) perm[i] = i;
#define A(i, j) a[(i) * n + (j)]
    for (int k = 0; k < n; ++k) {
        int piv = k;
        double best = fabs(A(k, k));
        for (int i = k + 1; i < n; ++i)
            if (fabs(A(i, i)) > best) {
                best = fabs(A(i, i));
                piv = i;
            }
        if (piv != k) {
            for (int c = 0; c < n; ++c) {
                const double t = A(k, c);
                A(k, c) = A(piv, c);
                A(piv, c) = t;
            }
            for (int r = 0; r < n; ++r) {
                const double t = A(r, k);
                A(r, k) = A(r, piv);
                A(r, piv) = t;
            }
            const int t = perm[k];
            perm[k] = perm[piv];
            perm[piv] = t;
        }
        const double d = A(k, k);
        for (int i = k + 1; i < n; ++i) {
            const double l = (d != 0.0) ? A(i, k) / d : 0.0;
            for (int j = k + 1; j <= i; ++j) A(i, j) -= l * A(j, k);
            for (int j = k + 1; j <= i; ++j) A(j, i) = A(i, j);
        }
        for (int i = k + 1; i < n; ++i) {
            A(i, k) = (d != 0.0) ? A(i, k) / d : 0.0;
            A(k, i) = A(i, k);
        }
    }
    for (int i = 0; i < n; ++i) y[i] = b[perm[i]];
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < i; ++j) y[i] -= A(i, j) * y[j];
    for (int i = 0; i < n; ++i) y[i] = (A(i, i) != 0.0) ? y[i] / A(i, i) : 0.0;
    for (int i = n - 1; i >= 0; --i)
        for (int j = i + 1; j < n; ++j) y[i] -= A(j, i) * y[j];
    for (int i = 0; i < n; ++i) x[perm[i]] = y[i];
#undef A
}

double om_mechanical_energy(const om_model *m, const double *q, const double *dq) {
    static __thread kin_t k;
    static __thread double M[MAX_NQ * MAX_NQ];
    const int nq = om_nq(m);
    fk(m, q, &k);
    mass_matrix_k(m, &k, M);
    double pe = 0.0, com[2];
    for (int l = 0; l < m->n_links; ++l) {
        world_point(&k, l, m->link_com[l], 0.0, com);
        pe += m->link_mass[l] * (-m->gravity) * com[1];
    }
    double ke = 0.0;
    for (int i = 0; i < nq; ++i) {
        double s = 0.0;
        for (int j = 0; j < nq; ++j) s += M[i * nq + j] * dq[j];
        ke += dq[i] * s;
    }
    return 0.5 * ke + pe;
}

void om_key_body_state(const om_model *m, const double *q, double *pos, double *ang) {
    static __thread kin_t k;
    fk(m, q, &k);
    for (int i = 0; i < m->n_key; ++i) {
        const int l = m->key_bodies[i];
        world_point(&k, l, m->link_com[l], 0.0, pos + 2 * i);
        ang[i] = k.angle[l];
    }
}

/* make_initial_state (skeleton.cpp:264-284) */
void om_make_initial_state(const om_model *m, const double *q, const double *dq, double init_act,
                           double *q_out, double *dq_out, double *act, double *l_m, double *v_m,
                           double *f_m) {
    static __thread kin_t k;
    const int nq = om_nq(m);
    for (int i = 0; i < nq; ++i) {
        q_out[i] = q[i];
        dq_out[i] = dq[i];
    }
    fk(m, q_out, &k);
    for (int mu = 0; mu < m->n_muscles; ++mu) {
        const double L = mtu_length_k(m, &k, mu);
        act[mu] = init_act;
        double lm = (L - m->m_slack[mu]) / m->m_lopt[mu];
        l_m[mu] = lm > K_MIN_FIBER ? lm : K_MIN_FIBER;
        v_m[mu] = 0.0;
        f_m[mu] = om_mtu_force(init_act, l_m[mu], 0.0, m->m_fmax[mu]);
    }
}

/* One substep of msk::step (skeleton.cpp:295-329). */
static int substep(const om_model *m, double *q, double *dq, double *act, double *l_m, double *v_m,
                   double *f_m, const double *u, double *muscle_power, double *grf, double *qdd_out,
                   double *forces, double *Jm, double *M) {
    static __thread kin_t k;
    const int nq = om_nq(m), nm = m->n_muscles;
    double tau_c[MAX_NQ], sf[2 * MAX_NL], C[MAX_NQ], tau[MAX_NQ], qdd[MAX_NQ];
    fk(m, q, &k);
    for (int mu = 0; mu < nm; ++mu) {
        double uu = u[mu];
        uu = uu < 0.0 ? 0.0 : (uu > 1.0 ? 1.0 : uu);
        act[mu] = om_activation_step(act[mu], uu, K_SIM_DT, m->m_tau_act[mu], m->m_tau_deact[mu]);
        const double prev_len = m->m_slack[mu] + l_m[mu] * m->m_lopt[mu];
        const double len = mtu_length_k(m, &k, mu);
        v_m[mu] = (len - prev_len) / K_SIM_DT / (m->m_lopt[mu] * m->m_vmax[mu]);
        const double lm = (len - m->m_slack[mu]) / m->m_lopt[mu];
        l_m[mu] = lm > K_MIN_FIBER ? lm : K_MIN_FIBER;
        f_m[mu] = om_mtu_force(act[mu], l_m[mu], v_m[mu], m->m_fmax[mu]);
        forces[mu] = f_m[mu];
        if (muscle_power)
            muscle_power[mu] += fabs(f_m[mu] * v_m[mu] * m->m_lopt[mu] * m->m_vmax[mu]) / K_SUBSTEPS;
    }
    moment_arms_k(m, &k, Jm);
    contact_forces_k(m, &k, dq, tau_c, sf);
    bias_forces_k(m, &k, q, dq, C);
    for (int c = 0; c < nq; ++c) {  /* tau = Jm^T F + tau_c - C  (skeleton.cpp:315) */
        double s = 0.0;
        for (int mu = 0; mu < nm; ++mu) s += Jm[(size_t)mu * nq + c] * forces[mu];
        tau[c] = (s + tau_c[c]) - C[c];
    }
    mass_matrix_k(m, &k, M);
    ldlt_solve(nq, M, tau, qdd);
    for (int i = 0; i < nq; ++i) dq[i] += qdd[i] * K_SIM_DT;
    for (int i = 0; i < nq; ++i) q[i] += dq[i] * K_SIM_DT;
    if (grf)
        for (int s = 0; s < m->n_spheres; ++s) {
            const int l = m->sphere_link[s];
            grf[2 * l] += sf[2 * s] / K_SUBSTEPS;
            grf[2 * l + 1] += sf[2 * s + 1] / K_SUBSTEPS;
        }
    if (qdd_out)
        for (int i = 0; i < nq; ++i) qdd_out[i] = qdd[i];
    for (int i = 0; i < nq; ++i)
        if (!isfinite(q[i]) || !isfinite(dq[i])) return 1;
    return 0;
}

typedef struct scratch {
    double *forces, *Jm, *M;
    int nm, nq;
} scratch_t;

static scratch_t *get_scratch(const om_model *m) {
    static __thread scratch_t s = {0, 0, 0, 0, 0};
    const int nq = om_nq(m), nm = m->n_muscles;
    if (s.nm < nm || s.nq < nq) {
        free(s.forces);
        free(s.Jm);
        free(s.M);
        s.forces = (double *)malloc(sizeof(double) * (size_t)nm);
        s.Jm = (double *)malloc(sizeof(double) * (size_t)nm * nq);
        s.M = (double *)malloc(sizeof(double) * (size_t)nq * nq);
        s.nm = nm;
        s.nq = nq;
    }
    return &s;
}

int32_t om_substep(const om_model *m, double *q, double *dq, double *act, double *l_m, double *v_m,
                   double *f_m, const double *u, double *qdd) {
    scratch_t *s = get_scratch(m);
    return substep(m, q, dq, act, l_m, v_m, f_m, u, NULL, NULL, qdd, s->forces, s->Jm, s->M);
}

int32_t om_step(const om_model *m, double *q, double *dq, double *act, double *l_m, double *v_m,
                double *f_m, double *t, const double *u, double *muscle_power, double *grf) {
    scratch_t *s = get_scratch(m);
    if (muscle_power)
        for (int i = 0; i < m->n_muscles; ++i) muscle_power[i] = 0.0;
    if (grf)
        for (int i = 0; i < 2 * m->n_links; ++i) grf[i] = 0.0;
    for (int sub = 0; sub < K_SUBSTEPS; ++sub) {
        const int bad = substep(m, q, dq, act, l_m, v_m, f_m, u, muscle_power, grf, NULL, s->forces,
                                s->Jm, s->M);
        *t += K_SIM_DT;  /* skeleton.cpp:321 advances t before the finite check */
        if (bad) return sub;
    }
    return -1;
}

/* ---- rng.hpp: std::mt19937_64 ------------------------------------------- */
void om_rng_seed(om_env *e, uint64_t seed) {
    e->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        e->mt[i] = 6364136223846793005ULL * (e->mt[i - 1] ^ (e->mt[i - 1] >> 62)) + (uint64_t)i;
    e->mti = 312;
}

uint64_t om_rng_raw(om_env *e) {
    static const uint64_t mag01[2] = {0ULL, 0xB5026F5AA96619E9ULL};
    const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
    if (e->mti >= 312) {
        int i;
        uint64_t x;
        for (i = 0; i < 312 - 156; ++i) {
            x = (e->mt[i] & UM) | (e->mt[i + 1] & LM);
            e->mt[i] = e->mt[i + 156] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
        }
        for (; i < 311; ++i) {
            x = (e->mt[i] & UM) | (e->mt[i + 1] & LM);
            e->mt[i] = e->mt[i + (156 - 312)] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
        }
        x = (e->mt[311] & UM) | (e->mt[0] & LM);
        e->mt[311] = e->mt[155] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
        e->mti = 0;
    }
    uint64_t x = e->mt[e->mti++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= (x >> 43);
    return x;
}

static double rng_uniform(om_env *e) { return (double)(om_rng_raw(e) >> 11) * 0x1.0p-53; }

/* ---- env.cpp ------------------------------------------------------------- */
void om_env_init(const om_model *m, const om_clip *c, const om_env_config *cfg, om_env *e,
                 uint64_t seed) {
    om_rng_seed(e, seed);
    const int bins = cfg->adaptive_bins > 1 ? cfg->adaptive_bins : 1;
    for (int b = 0; b < bins; ++b) e->failure_ema[b] = 0.0;
    om_make_initial_state(m, c->q, c->dq, cfg->init_activation, e->q, e->dq, e->act, e->l_m, e->v_m,
                          e->f_m);
    e->t = 0.0;
    e->t_index = e->start_index = e->steps = 0;
    e->done = 1;
    e->n_outcomes = 0;
}

static int sampler_bins(const om_env_config *cfg) {
    return cfg->adaptive_bins > 1 ? cfg->adaptive_bins : 1;
}

/* AdaptiveSampler::probabilities + sample (env.cpp:39-57) */
static int sampler_sample(const om_env_config *cfg, om_env *e) {
    const int bins = sampler_bins(cfg);
    double p[256];
    double total = 0.0;
    for (int b = 0; b < bins; ++b) total += e->failure_ema[b];
    for (int b = 0; b < bins; ++b) {
        p[b] = cfg->adaptive_mix / bins;
        if (total > 1e-12)
            p[b] += ((1.0 - cfg->adaptive_mix) * e->failure_ema[b]) / total;
        else
            p[b] += (1.0 - cfg->adaptive_mix) / bins;
    }
    double u = rng_uniform(e);
    for (int b = 0; b < bins; ++b) {
        u -= p[b];
        if (u <= 0.0) return b;
    }
    return bins - 1;
}

void om_sampler_record(const om_env_config *cfg, om_env *e, int32_t bin, int32_t failed) {
    const int bins = sampler_bins(cfg);
    if (bin < 0 || bin >= bins) return;
    e->failure_ema[bin] = cfg->adaptive_decay * e->failure_ema[bin] +
                          (1.0 - cfg->adaptive_decay) * (failed ? 1.0 : 0.0);
}

static int phase_bin(const om_clip *c, const om_env_config *cfg, int frame) {  /* env.cpp:89-93 */
    const int bins = sampler_bins(cfg);
    const int usable = c->frames - 1 > 1 ? c->frames - 1 : 1;
    int b = (int)((long)frame * bins / usable);
    return b < bins - 1 ? b : bins - 1;
}

static void finish_episode(const om_clip *c, const om_env_config *cfg, om_env *e, int failed) {
    e->done = 1;
    if (e->n_outcomes < e->outcome_cap) {
        e->outcome_bin[e->n_outcomes] = phase_bin(c, cfg, e->start_index);
        e->outcome_failed[e->n_outcomes] = (uint8_t)(failed ? 1 : 0);
    }
    e->n_outcomes++;
}

int32_t om_env_reset_to_frame(const om_model *m, const om_clip *c, const om_env_config *cfg,
                              om_env *e, int32_t frame, double *obs) {
    if (frame < 0 || frame >= c->frames - 1) return 1;  /* ContractError */
    const int nq = om_nq(m);
    e->t_index = frame;
    e->start_index = frame;
    e->steps = 0;
    e->done = 0;
    om_make_initial_state(m, c->q + (size_t)frame * nq, c->dq + (size_t)frame * nq,
                          cfg->init_activation, e->q, e->dq, e->act, e->l_m, e->v_m, e->f_m);
    e->t = frame * K_CTRL_DT;
    if (obs) om_env_observe(m, c, e, obs);
    return 0;
}

int32_t om_env_reset(const om_model *m, const om_clip *c, const om_env_config *cfg, om_env *e,
                     double *obs) {
    int frame = 0;
    if (cfg->rsi) {  /* env.cpp:110-119 */
        const int usable = c->frames - 1;
        const int bins = sampler_bins(cfg);
        const int bin = sampler_sample(cfg, e);
        const long lo = (long)bin * usable / bins;
        long hi = (long)(bin + 1) * usable / bins;
        if (hi <= lo) hi = lo + 1;
        frame = (int)(lo + (long)(om_rng_raw(e) % (uint64_t)(hi - lo)));
        if (frame > usable - 1) frame = usable - 1;
    }
    return om_env_reset_to_frame(m, c, cfg, e, frame, obs);
}

void om_env_observe(const om_model *m, const om_clip *c, const om_env *e, double *obs) {
    const int nq = om_nq(m), nm = m->n_muscles, nk = m->n_key;
    double pos[2 * MAX_NL], ang[MAX_NL];
    om_key_body_state(m, e->q, pos, ang);
    int o = 0;
    for (int i = 0; i < nq; ++i) obs[o++] = e->q[i];
    for (int i = 0; i < nq; ++i) obs[o++] = e->dq[i];
    for (int k = 0; k < nk; ++k) {
        obs[o++] = pos[2 * k];
        obs[o++] = pos[2 * k + 1];
    }
    for (int k = 0; k < nk; ++k) obs[o++] = ang[k];
    for (int i = 0; i < nm; ++i) obs[o++] = e->act[i];
    for (int i = 0; i < nm; ++i) obs[o++] = e->f_m[i];
    for (int i = 0; i < nm; ++i) obs[o++] = e->l_m[i];
    for (int i = 0; i < nm; ++i) obs[o++] = e->v_m[i];
    const size_t t = (size_t)e->t_index;
    for (int i = 0; i < nq; ++i) obs[o++] = c->q[t * nq + i];
    for (int i = 0; i < 2 * nk; ++i) obs[o++] = c->key_pos[t * 2 * nk + i];
    for (int i = 0; i < nk; ++i) obs[o++] = c->key_angle[t * nk + i];
}

void om_env_tracking_error(const om_model *m, const om_clip *c, const om_env *e, double *delta) {
    const int nq = om_nq(m), nj = m->n_joints, nk = m->n_key, r = nrd(m);
    const size_t t = (size_t)e->t_index;
    delta[0] = delta[1] = delta[2] = 0.0;
    if (m->floating) {  /* env.cpp:174-178 */
        delta[0] = e->q[0] - c->q[t * nq + 0];
        delta[1] = e->q[1] - c->q[t * nq + 1];
        delta[2] = om_wrap_angle(e->q[2] - c->q[t * nq + 2]);
    }
    for (int j = 0; j < nj; ++j) delta[3 + j] = e->q[r + j] - c->q[t * nq + r + j];
    double pos[2 * MAX_NL], ang[MAX_NL];
    om_key_body_state(m, e->q, pos, ang);
    for (int k = 0; k < nk; ++k) {
        delta[3 + nj + 2 * k] = pos[2 * k] - c->key_pos[t * 2 * nk + 2 * k];
        delta[3 + nj + 2 * k + 1] = pos[2 * k + 1] - c->key_pos[t * 2 * nk + 2 * k + 1];
    }
}

/* Env::step (env.cpp:206-263) */
int32_t om_env_step(const om_model *m, const om_clip *c, const om_env_config *cfg,
                    const om_reward_config *rc, om_env *e, const double *action, double *obs,
                    double *delta, double *reward_aux, double *muscle_power, double *grf) {
    const int nm = m->n_muscles, nk = m->n_key, nj = m->n_joints;
    if (e->done) return OM_NOT_STEPPED;
    for (int i = 0; i < nm; ++i)
        if (!isfinite(action[i])) return OM_BAD_ACTION;
    double *u = (double *)malloc(sizeof(double) * (size_t)nm);
    for (int i = 0; i < nm; ++i) {
        double a = action[i] > 0.0 ? action[i] : 0.0;  /* cwiseMax(0).cwiseMin(1) */
        u[i] = a < 1.0 ? a : 1.0;
    }
    double *pw = muscle_power;
    double *pw_tmp = NULL;
    if (!pw && rc && rc->mode == 2) pw = pw_tmp = (double *)malloc(sizeof(double) * (size_t)nm);
    const int bad = om_step(m, e->q, e->dq, e->act, e->l_m, e->v_m, e->f_m, &e->t, u, pw, grf);
    free(u);
    if (bad >= 0) {  /* env.cpp:218-229 */
        if (obs)
            for (int i = 0; i < om_obs_dim(m); ++i) obs[i] = 0.0;
        if (delta)
            for (int i = 0; i < om_delta_dim(m); ++i) delta[i] = 0.0;
        if (muscle_power)
            for (int i = 0; i < nm; ++i) muscle_power[i] = 0.0;
        if (grf)
            for (int i = 0; i < 2 * m->n_links; ++i) grf[i] = 0.0;
        if (reward_aux) *reward_aux = 0.0;
        finish_episode(c, cfg, e, 1);
        free(pw_tmp);
        return OM_DONE | OM_FAILED | OM_DIVERGED;
    }
    e->t_index++;
    e->steps++;
    double dbuf[4 * MAX_NL];
    double *d = delta ? delta : dbuf;
    om_env_tracking_error(m, c, e, d);
    if (obs) om_env_observe(m, c, e, obs);
    double aux = 0.0;
    if (rc && rc->mode == 1 && c->n_emg > 0) {  /* env.cpp:237-243 */
        const int n = rc->n_emg_channels;
        double s = 0.0;
        for (int ch = 0; ch < n; ++ch) {
            const double diff = c->emg[(size_t)e->t_index * c->n_emg + ch] - e->act[rc->emg_channel_map[ch]];
            s += diff * diff;
        }
        aux = n > 0 ? rc->w_emg * (-s / (double)n) : 0.0;
    } else if (rc && rc->mode == 2) {  /* env.cpp:244-246 */
        double s = 0.0;
        for (int i = 0; i < nm; ++i) s += pw[i];
        aux = rc->w_power * (-s / (nm > 1 ? nm : 1));
    }
    if (reward_aux) *reward_aux = aux;
    free(pw_tmp);
    int failed = 0;
    if (!e->eval_mode)
        for (int k = 0; k < nk; ++k) {
            const double dx = d[3 + nj + 2 * k], dz = d[3 + nj + 2 * k + 1];
            if (sqrt((0.0 + dx * dx) + dz * dz) > cfg->termination_body_err) failed = 1;
        }
    const int horizon = e->steps >= cfg->episode_horizon || e->t_index >= c->frames - 1;
    int flags = 0;
    if (failed || horizon) {
        flags |= OM_DONE;
        if (failed) flags |= OM_FAILED;
        finish_episode(c, cfg, e, failed);
    }
    return flags;
}

/* ---- Philox4x32-10 excitations ------------------------------------------ */
double om_excitation(uint64_t seed, uint32_t step, uint32_t global_env, int32_t muscle) {
    uint32_t c0 = step, c1 = global_env, c2 = (uint32_t)(muscle / 4), c3 = 0;
    uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
        const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
        c1 = (uint32_t)p1;
        c3 = (uint32_t)p0;
        c0 = n0;
        c2 = n2;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    const uint32_t out[4] = {c0, c1, c2, c3};
    return (double)(out[muscle % 4] >> 8) * (1.0 / 16777216.0);
}

/* ---- nn.cpp: Mlp as the tracking discriminator -------------------------- */
static void mlp_dims(int32_t layer, int32_t in, int32_t h, int32_t out, int32_t *r, int32_t *c) {
    /* Mlp::layer_dims (nn.cpp:9-14) */
    if (layer == 0) { *r = h; *c = in; }
    else if (layer < 3) { *r = h; *c = h; }
    else { *r = out; *c = h; }
}

int64_t om_mlp_param_count(int32_t in, int32_t hidden, int32_t out) {
    int64_t total = 0;
    for (int l = 0; l <= 3; ++l) {
        int32_t r, c;
        mlp_dims(l, in, hidden, out, &r, &c);
        total += (int64_t)r * c + r;
    }
    return total;
}

void om_mlp_init(double *theta, int32_t in, int32_t hidden, int32_t out, uint64_t seed, double final_init_scale) {
    /* nn.cpp:16-38 */
    const int64_t n = om_mlp_param_count(in, hidden, out);
    for (int64_t i = 0; i < n; ++i) theta[i] = 0.0;
    om_env rng;
    om_rng_seed(&rng, seed);
    int64_t off = 0;
    for (int l = 0; l <= 3; ++l) {
        int32_t r, c;
        mlp_dims(l, in, hidden, out, &r, &c);
        const double scale = (1.0 / sqrt((double)c)) * (l == 3 ? final_init_scale : 1.0);
        for (int32_t j = 0; j < c; ++j)
            for (int32_t i = 0; i < r; ++i) /* Rng::uniform(lo, hi), rng.hpp:30 */
                theta[off + (int64_t)j * r + i] = -scale + (scale - -scale) * rng_uniform(&rng);
        off += (int64_t)r * c + r; /* biases stay zero */
    }
}

void om_mlp_forward_sigmoid(const double *theta, int32_t in, int32_t hidden, const double *x, int32_t n, double *y) {
    /* nn.cpp:54-73: h1..h3 = tanh(W h + b), z = W4 h3 + b4, y = 1 / (1 + exp(-z)) */
    const int32_t h = hidden;
    double *a = (double *)malloc(sizeof(double) * (size_t)(h > in ? h : in));
    double *b = (double *)malloc(sizeof(double) * (size_t)h);
    for (int32_t row = 0; row < n; ++row) {
        for (int32_t k = 0; k < in; ++k) a[k] = x[(int64_t)row * in + k];
        int32_t cols = in;
        int64_t off = 0;
        for (int l = 0; l < 3; ++l) {
            const double *W = theta + off, *bias = theta + off + (int64_t)h * cols;
            for (int32_t i = 0; i < h; ++i) {
                double s = 0.0;
                for (int32_t k = 0; k < cols; ++k) s += a[k] * W[(int64_t)k * h + i];
                b[i] = tanh(s + bias[i]);
            }
            off += (int64_t)h * cols + h;
            cols = h;
            for (int32_t i = 0; i < h; ++i) a[i] = b[i];
        }
        const double *W4 = theta + off, *b4 = theta + off + h; /* out = 1: W4 is 1 x h */
        double z = 0.0;
        for (int32_t k = 0; k < h; ++k) z += a[k] * W4[k];
        z += b4[0];
        y[row] = 1.0 / (1.0 + exp(-z));
    }
    free(a);
    free(b);
}

double om_disc_reward(double d) {
    const double c = d < 1e-4 ? 1e-4 : (d > 1.0 - 1e-4 ? 1.0 - 1e-4 : d);
    return -log(1.0 - c);
}
