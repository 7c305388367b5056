/* TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference hot path.
 *
 * This header declares the parity oracle: a line-by-line fp64 restatement of
 *   /root/reference/proj/src/muscle.cpp     (Hill curves, activation ODE)
 *   /root/reference/proj/src/skeleton.cpp   (FK, Jacobians, moment arms, M, C,
 *                                            contact, 10-substep step)
 *   /root/reference/proj/src/env.cpp        (reset / RSI sampler / Δ / obs /
 *                                            reward_aux / termination)
 *   /root/reference/proj/include/msk/rng.hpp (mt19937_64 draws)
 * It is pinned against the reference itself (oracle/_ref, see oracle/Makefile)
 * and the SPEC.md known answers by tests/test_oracle.py.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu-baseline leg use it.
 */
#ifndef MSK_ORACLE_H
#define MSK_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Flat model description (model.hpp:11-73).  Arrays are owned by the caller. */
typedef struct om_model {
    int32_t floating;          /* RootType::FloatingPlanar */
    int32_t n_links, n_joints, n_muscles, n_key, n_spheres;
    double gravity, joint_limit_stiffness;
    const double *link_length, *link_mass, *link_inertia, *link_com;       /* n_links */
    const int32_t *joint_parent;                                           /* n_joints */
    const double *joint_anchor;                                            /* 2*n_joints */
    const double *joint_mount, *joint_lo, *joint_hi, *joint_damping;        /* n_joints */
    const double *m_fmax, *m_lopt, *m_vmax, *m_tau_act, *m_tau_deact, *m_slack; /* n_muscles */
    const int32_t *m_via_start;                                            /* n_muscles+1 */
    const int32_t *via_link;                                               /* V */
    const double *via_offset;                                              /* 2*V */
    const int32_t *sphere_link;                                            /* n_spheres */
    const double *sphere_offset, *sphere_radius;                           /* 2*ns, ns */
    double contact_k, contact_c, contact_mu, contact_vs;
    const int32_t *key_bodies;                                             /* n_key */
} om_model;

/* Clip (reference.hpp:13-28): row-major T x cols. */
typedef struct om_clip {
    int32_t frames;
    const double *q, *dq;          /* T x nq */
    const double *key_pos;         /* T x 2K */
    const double *key_angle;       /* T x K */
    int32_t n_emg;
    const double *emg;             /* T x n_emg (nullable) */
} om_clip;

typedef struct om_env_config {
    int32_t episode_horizon, rsi, adaptive_bins, pad0;
    double adaptive_mix, adaptive_decay, termination_body_err, init_activation;
} om_env_config;

typedef struct om_reward_config {
    int32_t mode, n_emg_channels; /* 0 imitation only, 1 emg, 2 power */
    double w_emg, w_power;
    const int32_t *emg_channel_map;
} om_reward_config;

/* One environment (env.hpp:128-141).  Caller allocates arrays of the model's
 * sizes; the oracle never allocates on the step path. */
typedef struct om_env {
    double *q, *dq;                         /* nq */
    double *act, *l_m, *v_m, *f_m;          /* nm */
    double t;
    int32_t t_index, start_index, steps, done, eval_mode;
    uint64_t mt[312];                       /* std::mt19937_64 */
    int32_t mti;
    double *failure_ema;                    /* adaptive_bins */
    int32_t n_outcomes, outcome_cap;
    int32_t *outcome_bin;
    uint8_t *outcome_failed;
} om_env;

enum { OM_DONE = 1, OM_FAILED = 2, OM_DIVERGED = 4, OM_NOT_STEPPED = 8, OM_BAD_ACTION = 16 };

int32_t om_nq(const om_model *m);
int32_t om_obs_dim(const om_model *m);
int32_t om_delta_dim(const om_model *m);

/* muscle.cpp */
double om_force_length_active(double l_m);
double om_force_velocity(double v_m);
double om_force_passive(double l_m);
double om_mtu_force(double act, double l_m, double v_m, double f_max);
double om_activation_step(double act, double u, double dt, double tau_act, double tau_deact);
double om_wrap_angle(double a);

/* skeleton.cpp */
void om_forward_kinematics(const om_model *m, const double *q, double *origin /*2nl*/,
                           double *angle /*nl*/, double *anchors /*2nj*/);
double om_mtu_length(const om_model *m, const double *q, int32_t muscle);
void om_moment_arms(const om_model *m, const double *q, double *Jm /* nm x nq row-major */);
void om_mass_matrix(const om_model *m, const double *q, double *M /* nq x nq */);
void om_bias_forces(const om_model *m, const double *q, const double *dq, double *C);
void om_contact_forces(const om_model *m, const double *q, const double *dq, double *tau,
                       double *sphere_force /* 2*ns */);
double om_mechanical_energy(const om_model *m, const double *q, const double *dq);
void om_key_body_state(const om_model *m, const double *q, double *pos /*2K*/, double *ang /*K*/);
void om_make_initial_state(const om_model *m, const double *q, const double *dq, double init_act,
                           double *q_out, double *dq_out, double *act, double *l_m, double *v_m,
                           double *f_m);
/* 10 substeps; returns -1 on success or the diverging substep index.
 * muscle_power (nm) and grf (2*nl, [link][xz]) are accumulated (nullable). */
int32_t om_step(const om_model *m, double *q, double *dq, double *act, double *l_m, double *v_m,
                double *f_m, double *t, const double *u, double *muscle_power, double *grf);
/* One substep only (debug / per-substep parity). qdd receives q̈ (nullable). */
int32_t om_substep(const om_model *m, double *q, double *dq, double *act, double *l_m, double *v_m,
                   double *f_m, const double *u, double *qdd);

/* rng.hpp */
void om_rng_seed(om_env *e, uint64_t seed);
uint64_t om_rng_raw(om_env *e);

/* env.cpp */
void om_env_init(const om_model *m, const om_clip *c, const om_env_config *cfg, om_env *e,
                 uint64_t seed);
int32_t om_env_reset(const om_model *m, const om_clip *c, const om_env_config *cfg, om_env *e,
                     double *obs);
int32_t om_env_reset_to_frame(const om_model *m, const om_clip *c, const om_env_config *cfg,
                              om_env *e, int32_t frame, double *obs);
void om_env_observe(const om_model *m, const om_clip *c, const om_env *e, double *obs);
void om_env_tracking_error(const om_model *m, const om_clip *c, const om_env *e, double *delta);
/* Returns flags (OM_*); outputs are written only when the env was stepped. */
int32_t om_env_step(const om_model *m, const om_clip *c, const om_env_config *cfg,
                    const om_reward_config *rc, om_env *e, const double *action, double *obs,
                    double *delta, double *reward_aux, double *muscle_power, double *grf);
void om_sampler_record(const om_env_config *cfg, om_env *e, int32_t bin, int32_t failed);

/* ---- nn.cpp: Mlp (3 tanh hidden layers) as the tracking discriminator ---- */
/* Parameter count of Mlp(in, hidden, out) (nn.cpp:16-27). */
int64_t om_mlp_param_count(int32_t in, int32_t hidden, int32_t out);
/* Mlp::Mlp(shape, seed) (nn.cpp:16-38): flat theta = W1 b1 W2 b2 W3 b3 W4 b4,
 * W column-major (Eigen default), W(i,j) ~ Rng(seed).uniform(-s, s) in column
 * order, s = 1/sqrt(cols) (x final_init_scale on the head), biases zero. */
void om_mlp_init(double *theta, int32_t in, int32_t hidden, int32_t out, uint64_t seed, double final_init_scale);
/* Mlp::forward with Head::Sigmoid (nn.cpp:54-73), out = 1: y[r] = D(x_r). */
void om_mlp_forward_sigmoid(const double *theta, int32_t in, int32_t hidden, const double *x, int32_t n, double *y);
/* reward_from_discriminator: -log(1 - clamp(d, 1e-4, 1 - 1e-4)). */
double om_disc_reward(double d);

/* Philox4x32-10 excitation in [0,1). */
double om_excitation(uint64_t seed, uint32_t step, uint32_t global_env, int32_t muscle);

#ifdef __cplusplus
}
#endif
#endif
