// msk_gpu.hpp — C++ host API over the C ABI (include/msk_gpu.h).
//
// msk::gpu::EnvBatch mirrors the verbs of the reference's msk::Env
// (/root/reference/proj/include/msk/env.hpp:86-145) for E environments on one
// GPU: reset / reset_to_frame / step / observe / tracking_error /
// force_state_to_reference / set_eval_mode / sampler / drain_episode_outcomes.
// Buffers are device pointers, calls are asynchronous on the given stream, and
// C-ABI status codes are turned back into exceptions with the reference's
// categories (ContractError-like for status 1, runtime_error for CUDA).
// Header-only; link against libmsk_b200.so.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "msk_gpu.h"

namespace msk::gpu {

struct ContractError : std::logic_error {
    using std::logic_error::logic_error;
};
struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// msk::EnvConfig defaults (env.hpp:39-47).
struct EnvConfig {
    int episode_horizon = 250;
    bool rsi = true;
    int adaptive_bins = 10;
    double adaptive_mix = 0.2;
    double adaptive_decay = 0.99;
    double termination_body_err = 0.5;
    double init_activation = 0.01;
};

enum class RewardMode { ImitationOnly = 0, ImitationEmg = 1, ImitationPower = 2 };

// msk::RewardConfig defaults (env.hpp:32-37).
struct RewardConfig {
    RewardMode mode = RewardMode::ImitationOnly;
    double w_emg = 100.0;
    double w_power = 0.05;
    std::vector<int> emg_channel_map;
};

// Device output buffers of one step (StepResult fields, env.hpp:70-80); any may be null.
struct StepBuffers {
    float* observation = nullptr;    // [E x observation_dim]
    float* delta = nullptr;          // [E x delta_dim]
    float* reward_aux = nullptr;     // [E]
    uint8_t* flags = nullptr;        // [E] MSK_FLAG_*
    float* muscle_power = nullptr;   // [E x action_dim]
    float* contact_force = nullptr;  // [E x n_links x 2]
};

inline void check(int status, const msk_gpu_ctx* ctx) {
    if (status == MSK_OK) return;
    const std::string msg = msk_gpu_last_error(ctx);
    if (status == MSK_ERR_CONTRACT) throw ContractError(msg);
    throw CudaError(msg);
}

class EnvBatch {
public:
    EnvBatch(const std::string& model_json, const std::string& clip_csv, int n_envs, const EnvConfig& cfg = {},
             const RewardConfig& rw = {}, uint64_t base_seed = 0x5EED, int64_t global_env_offset = 0,
             int device = 0) {
        msk_env_config ec{cfg.episode_horizon, cfg.rsi ? 1 : 0, cfg.adaptive_bins, 0,
                          cfg.adaptive_mix, cfg.adaptive_decay, cfg.termination_body_err, cfg.init_activation};
        std::vector<int32_t> map(rw.emg_channel_map.begin(), rw.emg_channel_map.end());
        msk_reward_config rc{static_cast<int32_t>(rw.mode), static_cast<int32_t>(map.size()), rw.w_emg, rw.w_power,
                             map.empty() ? nullptr : map.data()};
        check(msk_gpu_create(model_json.c_str(), clip_csv.c_str(), &ec, &rc, n_envs, base_seed, global_env_offset,
                             device, &ctx_),
              nullptr);
        check(msk_gpu_dims(ctx_, &dims_), ctx_);
    }
    ~EnvBatch() { msk_gpu_destroy(ctx_); }
    EnvBatch(const EnvBatch&) = delete;
    EnvBatch& operator=(const EnvBatch&) = delete;

    // Env::reset for envs whose mask byte has any of mask_bits (mask null = all).
    void reset(const uint8_t* mask = nullptr, uint8_t mask_bits = 0xff, float* observation = nullptr,
               int32_t* start_frames = nullptr, void* stream = nullptr) {
        check(msk_gpu_reset(ctx_, mask, mask_bits, observation, start_frames, stream), ctx_);
    }
    void reset_to_frame(const int32_t* frames, const uint8_t* mask = nullptr, float* observation = nullptr,
                        uint8_t* bad = nullptr, void* stream = nullptr) {
        check(msk_gpu_reset_to_frame(ctx_, frames, mask, observation, bad, stream), ctx_);
    }
    void step(const float* actions, const StepBuffers& out, void* stream = nullptr) {
        check(msk_gpu_step(ctx_, actions, out.observation, out.delta, out.reward_aux, out.flags, out.muscle_power,
                           out.contact_force, stream),
              ctx_);
    }
    void step_host(const float* actions, float* observation, float* delta, float* reward_aux, uint8_t* flags) {
        check(msk_gpu_step_host(ctx_, actions, observation, delta, reward_aux, flags), ctx_);
    }
    // Env::step(action, fn) with the built-in discriminator as fn (env.cpp:265-270):
    // load D = Mlp(delta_dim, hidden, 1, Sigmoid) once, then step with a reward buffer.
    void set_discriminator(const std::vector<double>& theta, int hidden) {
        check(msk_gpu_set_discriminator(ctx_, theta.data(), static_cast<int64_t>(theta.size()), hidden), ctx_);
    }
    void step(const float* actions, const StepBuffers& out, float* reward, void* stream = nullptr) {
        check(msk_gpu_step_rewarded(ctx_, actions, out.observation, out.delta, reward, out.reward_aux, out.flags,
                                    out.muscle_power, out.contact_force, stream),
              ctx_);
    }
    void step_host(const float* actions, float* observation, float* delta, float* reward, float* reward_aux,
                   uint8_t* flags) {
        check(msk_gpu_step_host_rewarded(ctx_, actions, observation, delta, reward, reward_aux, flags), ctx_);
    }
    // Mlp(shape, seed) initial parameters (nn.cpp:16-38), e.g. for a frozen D.
    static std::vector<double> mlp_init(int in, int hidden, int out, uint64_t seed, double final_init_scale = 1.0) {
        std::vector<double> theta(static_cast<size_t>(msk_mlp_param_count(in, hidden, out)));
        if (msk_mlp_init(theta.data(), in, hidden, out, seed, final_init_scale) != MSK_OK)
            throw ContractError("mlp_init: bad shape");
        return theta;
    }
    void observe(float* observation, void* stream = nullptr) {
        check(msk_gpu_observe(ctx_, observation, stream), ctx_);
    }
    void tracking_error(float* delta, void* stream = nullptr) {
        check(msk_gpu_tracking_error(ctx_, delta, stream), ctx_);
    }
    void force_state_to_reference(void* stream = nullptr) {
        check(msk_gpu_force_state_to_reference(ctx_, stream), ctx_);
    }
    void set_eval_mode(bool eval) { check(msk_gpu_set_eval_mode(ctx_, eval ? 1 : 0), ctx_); }
    void drain_episode_outcomes(int32_t* bins, uint8_t* failed, int32_t* counts, int cap, void* stream = nullptr) {
        check(msk_gpu_drain_outcomes(ctx_, bins, failed, counts, cap, stream), ctx_);
    }
    void record_own_outcomes(void* stream = nullptr) { check(msk_gpu_record_own_outcomes(ctx_, stream), ctx_); }
    // Rollout-iteration boundary of this rank (drain, stats, obs moments, NCCL
    // all-gather over nccl_comm = an ncclComm_t or nullptr, rank-ordered merge).
    void iteration_exchange(int cap, const float* obs, const double* stats_in, double* norm_state,
                            double* stats_out = nullptr, void* nccl_comm = nullptr, void* stream = nullptr) {
        check(msk_gpu_iteration_exchange(ctx_, nccl_comm, cap, obs, stats_in, norm_state, stats_out, stream), ctx_);
    }
    void fill_excitations(uint64_t seed, uint32_t step, float* actions, void* stream = nullptr) {
        check(msk_gpu_fill_excitations(ctx_, seed, step, actions, stream), ctx_);
    }

    int n_envs() const { return dims_.n_envs; }
    int observation_dim() const { return dims_.obs_dim; }  // Env::observation_dim (env.cpp:165-168)
    int action_dim() const { return dims_.n_muscles; }     // Env::action_dim (env.hpp:105)
    int delta_dim() const { return dims_.delta_dim; }      // TrackingError::dim (env.hpp:25-27)
    int nq() const { return dims_.nq; }
    int frames() const { return dims_.frames; }
    msk_gpu_ctx* handle() { return ctx_; }

private:
    msk_gpu_ctx* ctx_ = nullptr;
    msk_dims dims_{};
};

// train_discriminator on the device: one Adam step per call
// on rows of Δ (e.g. the rollout buffer's), then publish() refreshes the
// EnvBatch's reward discriminator (same shape) without a host round trip.
class DiscTrainer {
public:
    DiscTrainer(int in, int hidden, const std::vector<double>& theta, double lr, double grad_penalty, int max_rows,
                bool tf32 = true, int device = 0)
        : n_(theta.size()) {
        const int st = msk_disc_trainer_create(in, hidden, theta.data(), static_cast<int64_t>(theta.size()), lr,
                                               grad_penalty, max_rows, tf32 ? 1 : 0, device, &t_);
        if (st != MSK_OK) {
            const std::string msg = msk_disc_trainer_last_error(nullptr);
            if (st == MSK_ERR_CONTRACT) throw ContractError(msg);
            throw CudaError(msg);
        }
    }
    ~DiscTrainer() { msk_disc_trainer_destroy(t_); }
    DiscTrainer(const DiscTrainer&) = delete;
    DiscTrainer& operator=(const DiscTrainer&) = delete;

    // loss (device, nullable): {total, logistic, mean penalty} before the step
    void step(const float* delta, int rows, int ld, double* loss = nullptr, void* stream = nullptr) {
        ck(msk_disc_train_step(t_, delta, rows, ld, loss, stream));
    }
    void publish(EnvBatch& env, void* stream = nullptr) {
        check(msk_disc_trainer_publish(t_, env.handle(), stream), env.handle());
    }
    std::vector<double> params(int64_t* adam_steps = nullptr, int64_t* skipped = nullptr) {
        std::vector<double> th(n_);
        ck(msk_disc_trainer_get_params(t_, th.data(), adam_steps, skipped));
        return th;
    }

private:
    void ck(int st) {
        if (st == MSK_OK) return;
        const std::string msg = msk_disc_trainer_last_error(t_);
        if (st == MSK_ERR_CONTRACT) throw ContractError(msg);
        throw CudaError(msg);
    }
    size_t n_ = 0;
    msk_disc_trainer* t_ = nullptr;
};

}  // namespace msk::gpu
