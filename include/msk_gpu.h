/* msk_gpu.h — C ABI of the B200-native batched musculoskeletal env-stepper.
 *
 * Drop-in for the data-parallel hot path of the reference's environment API
 * (/root/reference/proj/include/msk/env.hpp:86-145, class msk::Env): one
 * context holds E independent environments on one GPU and exposes the Env
 * verbs in batched form.  All buffers are caller-owned, row-major
 * [E x dim], and — unless the name ends in _host — DEVICE pointers; calls are
 * asynchronous on the given CUDA stream (passed as void*, a cudaStream_t;
 * NULL = legacy default stream).  No C++ exceptions cross this boundary:
 * every entry point returns an msk_status and msk_gpu_last_error() describes
 * the last failure.  There is no CPU fallback: a context can only be created
 * on a CUDA device with the sm_100a kernels of this library.
 *
 * Mapping to the reference (file:line of the interface each one replaces):
 *   msk_gpu_create          Env::Env (env.cpp:74-87) + load_model (model.cpp:198-204)
 *                           + load_reference (reference.cpp:88-93)
 *   msk_gpu_reset           Env::reset (env.cpp:108-121)
 *   msk_gpu_reset_to_frame  Env::reset_to_frame (env.cpp:95-106)
 *   msk_gpu_step            Env::step(action) (env.cpp:206-263) incl. msk::step
 *                           (skeleton.cpp:286-331); StepResult fields as buffers
 *   msk_gpu_observe         Env::observe (env.cpp:129-163)
 *   msk_gpu_tracking_error  Env::tracking_error (env.cpp:170-193) + TrackingError::flatten
 *   msk_gpu_force_state_to_reference  Env::force_state_to_reference (env.cpp:123-127)
 *   msk_gpu_set_eval_mode   Env::set_eval_mode (env.hpp:115)
 *   msk_gpu_get/set_state   Env::state / mutable_state (env.hpp:110-111) + EnvSerde (env.hpp:144)
 *   msk_gpu_get/set_sampler, msk_gpu_record_own_outcomes
 *                           Env::sampler (env.hpp:118-119), AdaptiveSampler::record (env.cpp:34-37)
 *   msk_gpu_drain_outcomes  Env::drain_episode_outcomes (env.cpp:200-204)
 *   msk_gpu_merge_outcomes  the order-fixed merge of SPEC.md:296 (global sampler convention)
 *   msk_gpu_rng_raw         Rng::raw (rng.hpp:24) of one env's mt19937_64 stream
 */
#ifndef MSK_GPU_H
#define MSK_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct msk_gpu_ctx msk_gpu_ctx;

typedef enum msk_status {
    MSK_OK = 0,
    MSK_ERR_CONTRACT = 1, /* bad argument / config / model (ContractError, ConfigError) */
    MSK_ERR_CUDA = 3      /* CUDA runtime error, or no sm_100 device */
} msk_status;

/* Per-env flag bits written by msk_gpu_step (StepResult::done/failed/diverged
 * plus the two ContractError cases of Env::step, which leave the env untouched). */
enum {
    MSK_FLAG_DONE = 1,
    MSK_FLAG_FAILED = 2,
    MSK_FLAG_DIVERGED = 4,
    MSK_FLAG_NOT_STEPPED = 8, /* env was already done (env.cpp:207) */
    MSK_FLAG_BAD_ACTION = 16  /* non-finite action (env.cpp:209) */
};

/* msk::EnvConfig (env.hpp:39-47); field order is ABI. */
typedef struct msk_env_config {
    int32_t episode_horizon; /* 250 */
    int32_t rsi;             /* 1 */
    int32_t adaptive_bins;   /* 10 */
    int32_t pad0;
    double adaptive_mix;         /* 0.2 */
    double adaptive_decay;       /* 0.99 */
    double termination_body_err; /* 0.5 m */
    double init_activation;      /* 0.01 */
} msk_env_config;

/* msk::RewardConfig (env.hpp:30-37). mode: 0 ImitationOnly, 1 ImitationEmg, 2 ImitationPower. */
typedef struct msk_reward_config {
    int32_t mode;
    int32_t n_emg_channels;
    double w_emg;   /* 100 */
    double w_power; /* 0.05 */
    const int32_t* emg_channel_map; /* host pointer, n_emg_channels muscle indices */
} msk_reward_config;

typedef struct msk_dims {
    int32_t n_envs, nq, n_muscles, obs_dim, delta_dim;
    int32_t n_links, n_joints, n_key, n_spheres, frames;
    int32_t floating, adaptive_bins;
} msk_dims;

/* Creates E envs (seed of env e = base_seed + global_env_offset + e, as
 * Env(seed) with one mt19937_64 each, env.cpp:76).  Envs start done
 * (env.hpp:140): call msk_gpu_reset before stepping.  cfg/rc may be NULL for
 * the reference defaults. */
int msk_gpu_create(const char* model_json_path, const char* clip_csv_path, const msk_env_config* cfg,
                   const msk_reward_config* rc, int32_t n_envs, uint64_t base_seed,
                   int64_t global_env_offset, int device, msk_gpu_ctx** out);
void msk_gpu_destroy(msk_gpu_ctx* ctx);
/* Last error of ctx (or of the calling thread when ctx is NULL). */
const char* msk_gpu_last_error(const msk_gpu_ctx* ctx);
int msk_gpu_dims(const msk_gpu_ctx* ctx, msk_dims* out);
int msk_gpu_set_eval_mode(msk_gpu_ctx* ctx, int32_t eval_mode);

/* Env::reset for every env whose mask byte has any of mask_bits set (mask NULL
 * = all envs).  Passing the step's flags with mask_bits = MSK_FLAG_DONE is the
 * batched auto-reset.  obs [E x obs_dim] (nullable) receives observe() of the
 * reset envs; start_frames [E] (nullable) their start frame. */
int msk_gpu_reset(msk_gpu_ctx* ctx, const uint8_t* mask, uint8_t mask_bits, float* obs, int32_t* start_frames,
                  void* stream);
/* Env::reset_to_frame.  bad [E] (nullable) is set to 1 for envs whose frame is
 * out of range (reference: ContractError); those envs are left untouched. */
int msk_gpu_reset_to_frame(msk_gpu_ctx* ctx, const int32_t* frames, const uint8_t* mask, float* obs, uint8_t* bad,
                           void* stream);

/* One control step (10 x 2 ms substeps) of every env.  actions [E x n_muscles]
 * (clipped to [0,1]); obs [E x obs_dim]; delta [E x delta_dim]; reward_aux [E];
 * flags [E] (MSK_FLAG_*); muscle_power [E x n_muscles] and contact_force
 * [E x n_links x 2] optional.  Every output except flags is nullable. */
int msk_gpu_step(msk_gpu_ctx* ctx, const float* actions, float* obs, float* delta, float* reward_aux,
                 uint8_t* flags, float* muscle_power, float* contact_force, void* stream);

/* Built-in tracking discriminator: the TrackingRewardFn of Env::step(action, fn)
 * (env.hpp:82, env.cpp:265-270) for the adversarial tracking reward
 * r = -log(1 - clamp(D(delta), 1e-4, 1 - 1e-4)), with
 * D = Mlp(in = delta_dim, hidden, out = 1, Head::Sigmoid) given by its flat f64
 * parameters in the reference layout (nn.cpp:16-38: W1 b1 W2 b2 W3 b3 W4 b4,
 * W column-major).  hidden: multiple of 16 in [16, 256].  Evaluated on the
 * tcgen05 tensor cores with fp32 accumulation; by default every operand is
 * split as hi + lo bf16 (3 MMAs per product, accurate tanh/exp/log): fp32-class,
 * ~1e-6 relative to the f64 Mlp (tests: <= 1e-5).  msk_gpu_set_discriminator_mode(ctx, 1)
 * selects the bf16-operand fast mode (~3e-3). */
int msk_gpu_set_discriminator(msk_gpu_ctx* ctx, const double* theta, int64_t n_params, int32_t hidden);
/* 0: fp32-class split-bf16 (default); 1: bf16 operands (fast). */
int msk_gpu_set_discriminator_mode(msk_gpu_ctx* ctx, int32_t mode);
/* Host helpers for the parameter blob: Mlp(in, hidden, out) parameter count and
 * the Mlp(shape, seed) initialisation (nn.cpp:16-38, msk::Rng = mt19937_64). */
int64_t msk_mlp_param_count(int32_t in, int32_t hidden, int32_t out);
int msk_mlp_init(double* theta, int32_t in, int32_t hidden, int32_t out, uint64_t seed, double final_init_scale);
int msk_gpu_clear_discriminator(msk_gpu_ctx* ctx);
/* reward[i] = r(D(delta_i)) for n rows of delta [n x delta_dim]. */
int msk_gpu_discriminator_reward(msk_gpu_ctx* ctx, const float* delta, int32_t n, float* reward, void* stream);
/* ---- discriminator training step (SPEC.md:412-421 train_discriminator) ------
 * One Adam step (nn.cpp:224-240: β1 0.9, β2 0.999, ε 1e-8; a non-finite
 * gradient skips the step) on
 *   loss = -log clamp(D(0)) - mean_i log(1 - clamp(D(Δ_i))) + λ mean_i ||∇_Δ D(Δ_i)||²
 * (clamp to [1e-4, 1 - 1e-4]; gradient penalty at the sampled Δ),
 * the gradient from Mlp::backward (nn.cpp:80-129) and
 * Mlp::gradient_penalty_backward (nn.cpp:131-222).  The learner's absent
 * train_discriminator (learn.cpp) is the interface replaced.  Master θ
 * (nn.cpp:16-38 layout) and Adam moments live on the device in f64; every GEMM
 * is the library's own tcgen05 kernel: math 0 = fp32-class (split-bf16 operands,
 * 3 MMAs per product), 1 = bf16 operands.  n_in, hidden <= 256.
 * delta: [rows x ld] f32 device rows (the
 * rollout's Δ), rows <= max_rows.  loss (device, nullable): {total, logistic,
 * mean penalty} at the pre-step parameters. */
typedef struct msk_disc_trainer msk_disc_trainer;
int msk_disc_trainer_create(int32_t n_in, int32_t hidden, const double* theta, int64_t n_params, double lr,
                            double grad_penalty, int32_t max_rows, int32_t math, int32_t device,
                            msk_disc_trainer** out);
void msk_disc_trainer_destroy(msk_disc_trainer* t);
const char* msk_disc_trainer_last_error(const msk_disc_trainer* t);
int msk_disc_train_step(msk_disc_trainer* t, const float* delta, int32_t rows, int32_t ld, double* loss,
                        void* stream);
/* Loss and dloss/dθ (f32, [n_params], device) without the Adam step. */
int msk_disc_trainer_gradient(msk_disc_trainer* t, const float* delta, int32_t rows, int32_t ld, float* grad,
                              double* loss, void* stream);
/* Synchronises; copies θ (f64, host) and the Adam step / skip counts. */
int msk_disc_trainer_get_params(msk_disc_trainer* t, double* theta, int64_t* adam_steps, int64_t* adam_skipped);
/* Refreshes ctx's reward discriminator (set earlier with the same shape) from
 * the trainer's θ on the device, stream-ordered (no host round trip). */
int msk_disc_trainer_publish(msk_disc_trainer* t, msk_gpu_ctx* ctx, void* stream);

/* Env::step(action, fn) with fn = the discriminator reward: msk_gpu_step plus
 * reward [E] = r(D(delta)) + reward_aux for stepped envs, 0 for diverged ones
 * (StepResult::reward stays 0, env.cpp:267-268), untouched for envs flagged
 * NOT_STEPPED / BAD_ACTION.  delta / reward_aux / flags may be null (internal
 * scratch). */
int msk_gpu_step_rewarded(msk_gpu_ctx* ctx, const float* actions, float* obs, float* delta, float* reward,
                          float* reward_aux, uint8_t* flags, float* muscle_power, float* contact_force,
                          void* stream);

/* Same verb with HOST buffers (pinned or pageable): copies actions in, steps,
 * and copies obs/delta/reward_aux/flags out, pipelined over env chunks so the
 * PCIe transfers overlap the step kernel.  Synchronous on return. */
int msk_gpu_step_host(msk_gpu_ctx* ctx, const float* actions_host, float* obs_host, float* delta_host,
                      float* reward_aux_host, uint8_t* flags_host);
/* Host-buffer Env::step(action, fn) with the discriminator reward (see
 * msk_gpu_step_rewarded); reward_host [E] required. */
int msk_gpu_step_host_rewarded(msk_gpu_ctx* ctx, const float* actions_host, float* obs_host, float* delta_host,
                               float* reward_host, float* reward_aux_host, uint8_t* flags_host);
/* Asynchronous host-buffer step (reward_host nullable = plain step): enqueues
 * the same pipeline and returns; the host buffers (pinned) must stay untouched
 * until msk_gpu_host_wait.  Lets a harness double-buffer env groups (one
 * context each) so one group's PCIe transfers overlap the other's step. */
int msk_gpu_step_host_async(msk_gpu_ctx* ctx, const float* actions_host, float* obs_host, float* delta_host,
                            float* reward_host, float* reward_aux_host, uint8_t* flags_host);
int msk_gpu_host_wait(msk_gpu_ctx* ctx);
/* Shape of the host-buffer pipeline: env chunks per call and streams (default
 * 4 x 4, best for one synchronous context; 1 chunk per context is best when a
 * harness double-buffers several contexts with msk_gpu_step_host_async). */
int msk_gpu_set_host_pipeline(msk_gpu_ctx* ctx, int32_t chunks, int32_t streams);

/* Diagnostics / parity: advance every active env's continuous state (q, q̇,
 * muscles, t) by n_substeps (1..9) 2 ms substeps of msk::step's loop body
 * (skeleton.cpp:295-329) with the given excitations, WITHOUT the env epilogue
 * (no t_index / observation / termination).  Lets a test compare forces and
 * accelerations from an identical state before they feed back into the state. */
int msk_gpu_substeps(msk_gpu_ctx* ctx, const float* actions, int32_t n_substeps, float* muscle_power,
                     float* contact_force, void* stream);

int msk_gpu_observe(msk_gpu_ctx* ctx, float* obs, void* stream);
int msk_gpu_tracking_error(msk_gpu_ctx* ctx, float* delta, void* stream);
int msk_gpu_force_state_to_reference(msk_gpu_ctx* ctx, void* stream);

/* State of every env (SimState, skeleton.hpp:27-32): q, dq [E x nq] (f64), act,
 * v_m, f_m [E x n_muscles] (f32), l_m [E x n_muscles] (f64: the fibre length
 * is the integrator state whose difference gives v_m, kept at the reference's
 * precision), t [E] (f64), ints [E x 4] = {t_index, start_index, steps, done}.
 * Muscle columns in reference order.  Any pointer may be NULL. */
int msk_gpu_get_state(msk_gpu_ctx* ctx, double* q, double* dq, float* act, double* l_m, float* v_m, float* f_m,
                      double* t, int32_t* ints, void* stream);
int msk_gpu_set_state(msk_gpu_ctx* ctx, const double* q, const double* dq, const float* act, const double* l_m,
                      const float* v_m, const float* f_m, const double* t, const int32_t* ints, void* stream);

/* mt19937_64 state of every env (Env::rng(), env.hpp:120; the engine state
 * Rng::serialize writes, rng.hpp:56-68): mt [E x 312] u64 words and mti [E] the
 * next-word index (312 = regenerate on the next draw), i.e. libstdc++'s _M_x /
 * _M_p.  Device pointers, either nullable; set clamps mti into [0, 312].  With
 * msk_gpu_get_state / set_state and the sampler this checkpoints a batch
 * completely: a restored batch replays the same reset frames. */
int msk_gpu_get_rng(msk_gpu_ctx* ctx, uint64_t* mt, int32_t* mti, void* stream);
int msk_gpu_set_rng(msk_gpu_ctx* ctx, const uint64_t* mt, const int32_t* mti, void* stream);

/* Adaptive sampler failure EMA [E x bins] (f64).  set: broadcast != 0 copies
 * one [bins] row to every env. */
int msk_gpu_get_sampler(msk_gpu_ctx* ctx, double* ema, void* stream);
int msk_gpu_set_sampler(msk_gpu_ctx* ctx, const double* ema, int32_t broadcast, void* stream);
/* Pending episode outcomes (Env::drain_episode_outcomes, env.cpp:200-204):
 * bins/failed [E x cap], counts [E] = the number of valid slots written; then
 * cleared.  The reference list is unbounded; here each env holds a ring of
 * msk_gpu_set_outcome_capacity slots (default 64, grown to `cap` by a drain or
 * exchange asking for more).  Outcomes that overflow the ring or the caller's
 * cap are never silent: they are counted (msk_gpu_outcomes_dropped). */
int msk_gpu_drain_outcomes(msk_gpu_ctx* ctx, int32_t* bins, uint8_t* failed, int32_t* counts, int32_t cap,
                           void* stream);
/* Per-env pending-outcome ring size (>= the steps between two drains; an env
 * ends at most one episode per step).  Pending outcomes are kept. */
int msk_gpu_set_outcome_capacity(msk_gpu_ctx* ctx, int32_t cap, void* stream);
/* Total outcomes lost to ring / drain-cap overflow since creation (synchronises
 * the device).  0 in any run whose drains keep up. */
int msk_gpu_outcomes_dropped(msk_gpu_ctx* ctx, int64_t* dropped);
/* Each env records its own pending outcomes into its own sampler, in order. */
int msk_gpu_record_own_outcomes(msk_gpu_ctx* ctx, void* stream);
/* Order-fixed merge: outcome blocks of n_envs_total envs in
 * global env order (e.g. the allgather of every rank's drain) are recorded in
 * env order then time order into ONE sampler, which is then copied to every
 * local env.  Identical on every rank, so replicas stay bit-identical. */
/* Iteration-boundary reductions for the per-rank stats block:
 * stats[7] += {env-steps, Σreward, Σreward², Σ episode length of envs done this
 * step, episodes, failures, divergences} over the envs stepped (flags from
 * msk_gpu_step; reward nullable); deterministic single-block reduction. */
int msk_gpu_rollout_stats(msk_gpu_ctx* ctx, const float* reward, const uint8_t* flags, double* stats, void* stream);
/* One rollout-iteration boundary of this rank (the C++ form of
 * paper_2603_29332_b200/dist.py iteration_exchange): drains the episode
 * outcomes (cap slots per env: the iteration's h steps), takes this rank's
 * rollout stats (stats_in [7] f64, see msk_gpu_rollout_stats) and the f64
 * column moments of obs [E x obs_dim], all-gathers the fixed-size block over
 * nccl_comm (an ncclComm_t; NULL = single rank; NCCL is loaded at run time
 * from libnccl.so.2), then applies the identical rank-ordered merge on the
 * device: outcomes into the replicated sampler (SPEC.md:296 order), stats
 * summed in rank order into stats_out [7] (nullable), and the observation
 * normaliser norm_state [1 + 2 obs_dim] = {count, mean, var} (f64, in/out)
 * folded rank by rank as RunningNorm::update (nn.cpp:246-270). */
int msk_gpu_iteration_exchange(msk_gpu_ctx* ctx, void* nccl_comm, int32_t cap, const float* obs,
                               const double* stats_in, double* norm_state, double* stats_out, void* stream);
/* Batch moments of obs [n x obs_dim] (RunningNorm::update's batch mean and
 * population variance, nn.cpp:246-256) in f64: out = [n, mean[D], var[D]]. */
int msk_gpu_obs_moments(msk_gpu_ctx* ctx, const float* obs, int32_t n, double* out, void* stream);
/* The same batch moments folded into a running acc [1 + 2 obs_dim] = {count,
 * mean, var} (f64, in/out) as RunningNorm::update (nn.cpp:257-270): count 0
 * takes the batch exactly, n = 0 leaves acc unchanged.  Accumulates an
 * iteration's h x E observations without a host round trip (three launches). */
int msk_gpu_obs_moments_fold(msk_gpu_ctx* ctx, const float* obs, int32_t n, double* acc, void* stream);
int msk_gpu_merge_outcomes(msk_gpu_ctx* ctx, const int32_t* bins, const uint8_t* failed, const int32_t* counts,
                           int64_t n_envs_total, int32_t cap, void* stream);

/* n raw mt19937_64 draws of env `env` (advances its stream). */
int msk_gpu_rng_raw(msk_gpu_ctx* ctx, int32_t env, int32_t n, uint64_t* out, void* stream);
/* Philox4x32-10 excitations u in [0,1) [E x n_muscles] for control step `step`
 * (key = seed, counter = {step, global env, muscle/4, 0}). */
int msk_gpu_fill_excitations(msk_gpu_ctx* ctx, uint64_t seed, uint32_t step, float* actions, void* stream);

/* Number of kernels launched by this context since creation (diagnostics). */
int64_t msk_gpu_launch_count(const msk_gpu_ctx* ctx);

/* Host-only: parse + validate a model and clip exactly as msk_gpu_create does
 * (ModelSpec::validate, model.cpp:18-86; ReferenceTrajectory::validate,
 * reference.cpp:11-33) without touching a GPU — the `msk model validate`
 * check.  dims (nullable) receives the sizes (n_envs = 0).
 * Returns MSK_OK or MSK_ERR_CONTRACT with msk_gpu_last_error(NULL) set. */
int msk_gpu_validate(const char* model_json_path, const char* clip_csv_path, msk_dims* dims);

/* Measured FFMA throughput of `device` in TFLOP/s (FP32 roofline denominator). */
int msk_gpu_fp32_peak_probe(int device, double* tflops);

/* ---- on-device policy sampling (SPEC.md:371-393 sample_action) -------------
 * a0 ~ N(mean(s), exp(log_std)) with mean = head_scale * Mlp_pi(norm(s)) +
 * head_offset (Head::Affine, nn.hpp:10-19), then n_ode explicit-Euler steps of
 * the flow field a += dt * Mlp_psi([phi(t), norm(s), a]) with
 * phi(t) = [t, sin 2 pi t, cos 2 pi t, sin 4 pi t, cos 4 pi t];
 * norm = RunningNorm::apply (nn.cpp:272-277).  Mlp_pi = Mlp(obs_dim, hidden,
 * n_actions), Mlp_psi = Mlp(5 + obs_dim + n_actions, hidden, n_actions), flat
 * f64 parameters in the nn.cpp:16-38 layout.  hidden: multiple of 64.  Every
 * layer runs as a tcgen05 GEMM with bf16 operands and fp32 accumulation.
 * Gaussian noise: Philox4x32-10 keyed by seed, counter (step, global env, ...). */
typedef struct msk_policy msk_policy;
int msk_policy_create(int32_t obs_dim, int32_t n_actions, int32_t hidden, const double* pi_theta,
                      int64_t pi_n_params, double head_scale, double head_offset, const double* log_std,
                      const double* psi_theta, int64_t psi_n_params, int32_t n_ode, double dt_ode, int32_t max_envs,
                      int32_t device, msk_policy** out);
void msk_policy_destroy(msk_policy* p);
const char* msk_policy_last_error(const msk_policy* p);
/* RunningNorm state (count 0 -> identity). */
int msk_policy_set_norm(msk_policy* p, const double* mean, const double* var, double count);
/* actions [n x n_actions] (device) = final a; a0 / logprob (nullable) = the
 * Gaussian sample and its log-density (explore = 0: a0 = mean, logprob = 0). */
int msk_policy_sample(msk_policy* p, const float* obs, int32_t n, int32_t explore, uint64_t seed, uint32_t step,
                      int64_t global_env_offset, float* actions, float* a0, float* logprob, void* stream);
/* Same, replayed from a CUDA graph (re-captured when any argument changes). */
int msk_policy_sample_graph(msk_policy* p, const float* obs, int32_t n, int32_t explore, uint64_t seed,
                            uint32_t step, int64_t global_env_offset, float* actions, float* a0, float* logprob,
                            void* stream);
int32_t msk_policy_time_features(double t, double* out5);
/* Test hook: Y = act(X W^T + b) through one tiled tensor-core GEMM (epi 0 tanh, 1 linear). */
int msk_gemm_test(const float* X, int32_t M, int32_t K, const double* W, const float* b, int32_t N, int32_t epi,
                  float* Y);
/* Diagnostic: average ms of `reps` back-to-back tanh GEMM layers (M x K by K x N,
 * zero operands) on the device, programmatic dependent launches. */
int msk_gemm_bench(int32_t M, int32_t K, int32_t N, int32_t reps, double* ms_per_gemm);

/* ---- on-device rollout buffer + GAE ----------------------
 * h control steps x E envs, step-major: obs, a0, actions, logprob, reward,
 * done (the step's flags; bit MSK_FLAG_DONE), value, delta.  msk_rollout_gae:
 * delta_t = r_t + gamma V_{t+1} (1 - done_t) - V_t, A_t = delta_t + gamma lam
 * (1 - done_t) A_{t+1} (V_h = bootstrap [E]), returns = A + V; normalize != 0
 * standardises the advantages over the batch.  Outputs [h x E] (nullable). */
typedef struct msk_rollout msk_rollout;
int msk_rollout_create(int32_t n_envs, int32_t horizon, int32_t obs_dim, int32_t act_dim, int32_t delta_dim,
                       int32_t device, msk_rollout** out);
void msk_rollout_destroy(msk_rollout* r);
const char* msk_rollout_last_error(const msk_rollout* r);
/* Store step t (device buffers [E x dim], each nullable). */
int msk_rollout_record(msk_rollout* r, int32_t t, const float* obs, const float* a0, const float* actions,
                       const float* logprob, const float* reward, const uint8_t* flags, const float* value,
                       const float* delta, void* stream);
int msk_rollout_gae(msk_rollout* r, const float* bootstrap_value, float gamma, float lam, int32_t normalize,
                    float* advantages, float* returns, void* stream);
/* Device pointer of a stored field: 0 obs, 1 a0, 2 actions, 3 logprob, 4 reward, 5 done, 6 value, 7 delta. */
void* msk_rollout_field(msk_rollout* r, int32_t field);
/* PPO minibatching ("epochs over shuffled minibatches"; the
 * learner's minibatch loop, learn.cpp, is absent): epoch `epoch`'s shuffle of
 * the h*E records is a keyed Feistel bijection of [0, h*E) (seed, epoch) —
 * deterministic, no sort; minibatch `index` holds records
 * perm(index*mb_size + j), j < mb_size (the last one may be short).  Gathers
 * the stored obs / a0 / actions / logprob / value and the last GAE's
 * advantages / returns into caller buffers [mb_size x dim] (each nullable);
 * record_ids (nullable) receives the record indices (t*E + env). */
int msk_rollout_minibatch(msk_rollout* r, uint64_t seed, int32_t epoch, int32_t index, int32_t mb_size,
                          float* obs, float* a0, float* actions, float* logprob, float* advantages, float* returns,
                          float* value, int32_t* record_ids, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MSK_GPU_H */
