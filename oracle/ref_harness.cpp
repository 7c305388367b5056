// TEST INFRASTRUCTURE ONLY (parity checker + CPU baseline arm).
//
// Drives the reference's own msk::Env (compiled unchanged from
// /root/reference/proj/src against oracle/shim/Eigen) through a flat C ABI so
// Python tests can compare the CUDA path with the reference on identical
// inputs, and so bench.py can time the reference CPU path
// (ThreadPool::parallel_chunks fan-out, /root/reference/proj/src/thread_pool.cpp:45-64).
// Nothing here is linked into the product library.
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "msk/env.hpp"
#include "msk/errors.hpp"
#include "msk/model.hpp"
#include "msk/muscle.hpp"
#include "msk/nn.hpp"
#include "msk/reference.hpp"
#include "msk/skeleton.hpp"
#include "msk/thread_pool.hpp"

namespace msk {
// env.hpp:144 declares `friend struct EnvSerde`; the harness uses it to read
// and write the private episode bookkeeping (steps_, done_, ...).
struct EnvSerde {
    static int& steps(Env& e) { return e.steps_; }
    static int& t_index(Env& e) { return e.t_index_; }
    static int& start(Env& e) { return e.start_index_; }
    static bool& done(Env& e) { return e.done_; }
    static std::vector<std::pair<int, bool>>& outcomes(Env& e) { return e.episode_outcomes_; }
};
}  // namespace msk

namespace {

// Philox4x32-10 (Salmon et al. 2011); bit-identical to the device generator.
inline void philox4x32_10(uint32_t ctr[4], uint32_t key0, uint32_t key1) {
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = static_cast<uint64_t>(0xD2511F53u) * ctr[0];
        const uint64_t p1 = static_cast<uint64_t>(0xCD9E8D57u) * ctr[2];
        const uint32_t hi0 = static_cast<uint32_t>(p0 >> 32), lo0 = static_cast<uint32_t>(p0);
        const uint32_t hi1 = static_cast<uint32_t>(p1 >> 32), lo1 = static_cast<uint32_t>(p1);
        const uint32_t n0 = hi1 ^ ctr[1] ^ key0;
        const uint32_t n2 = hi0 ^ ctr[3] ^ key1;
        ctr[0] = n0;
        ctr[1] = lo1;
        ctr[2] = n2;
        ctr[3] = lo0;
        key0 += 0x9E3779B9u;
        key1 += 0xBB67AE85u;
    }
}

// Excitation u in [0,1) for (seed, step, global env, muscle); SURVEY §8(d).
inline double excitation(uint64_t seed, uint32_t step, uint32_t genv, int muscle) {
    uint32_t c[4] = {step, genv, static_cast<uint32_t>(muscle / 4), 0u};
    philox4x32_10(c, static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32));
    return static_cast<double>(c[muscle % 4] >> 8) * (1.0 / 16777216.0);
}

struct RefEnvConfig {
    int32_t episode_horizon;
    int32_t rsi;
    int32_t adaptive_bins;
    int32_t pad0;
    double adaptive_mix;
    double adaptive_decay;
    double termination_body_err;
    double init_activation;
};

struct RefRewardConfig {
    int32_t mode;  // 0 imitation-only, 1 emg, 2 power
    int32_t n_emg_channels;
    double w_emg;
    double w_power;
    const int32_t* emg_channel_map;
};

struct Batch {
    msk::ModelSpec spec;
    msk::ReferenceTrajectory ref;
    std::vector<std::unique_ptr<msk::Env>> envs;
    std::unique_ptr<msk::ThreadPool> pool;
    int obs_dim = 0, delta_dim = 0;
    std::unique_ptr<msk::Mlp> disc;  // tracking-reward discriminator for ref_bench (optional)
};

void set_err(char* err, int n, const std::string& msg) {
    if (err && n > 0) {
        std::snprintf(err, static_cast<size_t>(n), "%s", msg.c_str());
    }
}

enum : uint8_t {
    kDone = 1,
    kFailed = 2,
    kDiverged = 4,
    kNotStepped = 8,   // env was already done (reference: ContractError)
    kBadAction = 16,   // non-finite action (reference: ContractError)
};

void step_one(Batch& b, int e, const double* actions, double* obs, double* delta,
              double* reward_aux, uint8_t* flags, double* power, double* grf) {
    msk::Env& env = *b.envs[static_cast<size_t>(e)];
    const int nm = b.spec.n_muscles();
    Eigen::VectorXd a(nm);
    for (int m = 0; m < nm; ++m) a[m] = actions[static_cast<size_t>(e) * nm + m];
    uint8_t f = 0;
    if (env.done()) {
        flags[e] = kNotStepped;
        return;
    }
    if (!a.allFinite()) {
        flags[e] = kBadAction;
        return;
    }
    const msk::StepResult r = env.step(a);
    if (r.done) f |= kDone;
    if (r.failed) f |= kFailed;
    if (r.diverged) f |= kDiverged;
    flags[e] = f;
    if (obs)
        for (int i = 0; i < b.obs_dim; ++i) obs[static_cast<size_t>(e) * b.obs_dim + i] = r.observation[i];
    if (delta) {
        const Eigen::VectorXd d = r.delta.flatten();
        for (int i = 0; i < b.delta_dim; ++i) delta[static_cast<size_t>(e) * b.delta_dim + i] = d[i];
    }
    if (reward_aux) reward_aux[e] = r.reward_aux;
    if (power)
        for (int m = 0; m < nm; ++m) power[static_cast<size_t>(e) * nm + m] = r.muscle_power[m];
    if (grf) {
        const int nl = b.spec.n_links();
        for (int l = 0; l < nl; ++l) {
            grf[(static_cast<size_t>(e) * nl + l) * 2 + 0] = r.contact_force(0, l);
            grf[(static_cast<size_t>(e) * nl + l) * 2 + 1] = r.contact_force(1, l);
        }
    }
}

}  // namespace

extern "C" {

void* ref_create(const char* model_path, const char* clip_path, const RefEnvConfig* cfg,
                 const RefRewardConfig* rc, int32_t n_envs, uint64_t base_seed,
                 int64_t global_env_offset, char* err, int32_t errlen) {
    try {
        auto b = std::make_unique<Batch>();
        b->spec = msk::load_model(model_path);
        auto errs = b->spec.validate();
        if (!errs.empty()) throw msk::ConfigError("model: " + errs.front());
        if (clip_path && clip_path[0]) {
            b->ref = msk::load_reference(clip_path, b->spec);
        } else if (n_envs > 0) {
            throw msk::ContractError("ref_create: a clip is required when n_envs > 0");
        }
        msk::EnvConfig ec;
        if (cfg) {
            ec.episode_horizon = cfg->episode_horizon;
            ec.rsi = cfg->rsi != 0;
            ec.adaptive_bins = cfg->adaptive_bins;
            ec.adaptive_mix = cfg->adaptive_mix;
            ec.adaptive_decay = cfg->adaptive_decay;
            ec.termination_body_err = cfg->termination_body_err;
            ec.init_activation = cfg->init_activation;
        }
        msk::RewardConfig rw;
        if (rc) {
            rw.mode = rc->mode == 1   ? msk::RewardMode::ImitationEmg
                      : rc->mode == 2 ? msk::RewardMode::ImitationPower
                                      : msk::RewardMode::ImitationOnly;
            rw.w_emg = rc->w_emg;
            rw.w_power = rc->w_power;
            for (int i = 0; i < rc->n_emg_channels; ++i) rw.emg_channel_map.push_back(rc->emg_channel_map[i]);
        }
        for (int e = 0; e < n_envs; ++e)
            b->envs.push_back(std::make_unique<msk::Env>(
                b->spec, b->ref, ec, rw, base_seed + static_cast<uint64_t>(global_env_offset + e)));
        b->obs_dim = n_envs > 0 ? b->envs[0]->observation_dim() : 0;
        b->delta_dim = msk::TrackingError::dim(b->spec);
        return b.release();
    } catch (const std::exception& ex) {
        set_err(err, errlen, ex.what());
        return nullptr;
    }
}

void ref_destroy(void* h) { delete static_cast<Batch*>(h); }

void ref_dims(void* h, int32_t* out /* nq nm obs delta nlinks frames nk njoints floating nspheres */) {
    Batch& b = *static_cast<Batch*>(h);
    out[0] = b.spec.nq();
    out[1] = b.spec.n_muscles();
    out[2] = b.obs_dim;
    out[3] = b.delta_dim;
    out[4] = b.spec.n_links();
    out[5] = b.ref.frames();
    out[6] = b.spec.n_key_bodies();
    out[7] = b.spec.n_joints();
    out[8] = b.spec.root == msk::RootType::FloatingPlanar ? 1 : 0;
    out[9] = static_cast<int32_t>(b.spec.contact_spheres.size());
}

int ref_set_threads(void* h, int32_t threads) {
    Batch& b = *static_cast<Batch*>(h);
    b.pool = threads > 1 ? std::make_unique<msk::ThreadPool>(threads) : nullptr;
    return 0;
}

void ref_set_eval_mode(void* h, int32_t eval) {
    for (auto& e : static_cast<Batch*>(h)->envs) e->set_eval_mode(eval != 0);
}

// mask: nullptr = all envs.  frames_out (nullable) receives start frames.
int ref_reset(void* h, const uint8_t* mask, double* obs, int32_t* frames_out, char* err, int32_t errlen) {
    Batch& b = *static_cast<Batch*>(h);
    try {
        for (size_t e = 0; e < b.envs.size(); ++e) {
            if (mask && !mask[e]) continue;
            const Eigen::VectorXd o = b.envs[e]->reset();
            if (obs)
                for (int i = 0; i < b.obs_dim; ++i) obs[e * b.obs_dim + i] = o[i];
            if (frames_out) frames_out[e] = b.envs[e]->start_index();
        }
        return 0;
    } catch (const std::exception& ex) {
        set_err(err, errlen, ex.what());
        return 1;
    }
}

int ref_reset_to_frame(void* h, const int32_t* frames, const uint8_t* mask, double* obs, char* err,
                       int32_t errlen) {
    Batch& b = *static_cast<Batch*>(h);
    try {
        for (size_t e = 0; e < b.envs.size(); ++e) {
            if (mask && !mask[e]) continue;
            const Eigen::VectorXd o = b.envs[e]->reset_to_frame(frames[e]);
            if (obs)
                for (int i = 0; i < b.obs_dim; ++i) obs[e * b.obs_dim + i] = o[i];
        }
        return 0;
    } catch (const std::exception& ex) {
        set_err(err, errlen, ex.what());
        return 1;
    }
}

// Steps every env once (done envs are flagged kNotStepped and left untouched).
int ref_step(void* h, const double* actions, double* obs, double* delta, double* reward_aux,
             uint8_t* flags, double* power, double* grf) {
    Batch& b = *static_cast<Batch*>(h);
    const int n = static_cast<int>(b.envs.size());
    auto fn = [&](int begin, int end, int) {
        for (int e = begin; e < end; ++e) step_one(b, e, actions, obs, delta, reward_aux, flags, power, grf);
    };
    if (b.pool)
        b.pool->parallel_chunks(n, std::max(1, n / (4 * b.pool->workers())), fn);
    else
        fn(0, n, 0);
    return 0;
}

void ref_observe(void* h, double* obs) {
    Batch& b = *static_cast<Batch*>(h);
    for (size_t e = 0; e < b.envs.size(); ++e) {
        const Eigen::VectorXd o = b.envs[e]->observe();
        for (int i = 0; i < b.obs_dim; ++i) obs[e * b.obs_dim + i] = o[i];
    }
}

void ref_tracking_error(void* h, double* delta) {
    Batch& b = *static_cast<Batch*>(h);
    for (size_t e = 0; e < b.envs.size(); ++e) {
        const Eigen::VectorXd d = b.envs[e]->tracking_error().flatten();
        for (int i = 0; i < b.delta_dim; ++i) delta[e * b.delta_dim + i] = d[i];
    }
}

void ref_force_state_to_reference(void* h) {
    for (auto& e : static_cast<Batch*>(h)->envs) e->force_state_to_reference();
}

// State per env: q, dq (nq each), act, l_m, v_m, f_m (nm each), t, and the
// bookkeeping ints (t_index, start, steps, done).
void ref_get_state(void* h, double* q, double* dq, double* act, double* lm, double* vm, double* fm,
                   double* t, int32_t* ints /* E x 4 */) {
    Batch& b = *static_cast<Batch*>(h);
    const int nq = b.spec.nq(), nm = b.spec.n_muscles();
    for (size_t e = 0; e < b.envs.size(); ++e) {
        msk::Env& env = *b.envs[e];
        const msk::SimState& s = env.state();
        for (int i = 0; i < nq; ++i) {
            q[e * nq + i] = s.q[i];
            dq[e * nq + i] = s.dq[i];
        }
        for (int m = 0; m < nm; ++m) {
            act[e * nm + m] = s.muscles[static_cast<size_t>(m)].act;
            lm[e * nm + m] = s.muscles[static_cast<size_t>(m)].l_m;
            vm[e * nm + m] = s.muscles[static_cast<size_t>(m)].v_m;
            fm[e * nm + m] = s.muscles[static_cast<size_t>(m)].f_m;
        }
        t[e] = s.t;
        ints[e * 4 + 0] = msk::EnvSerde::t_index(env);
        ints[e * 4 + 1] = msk::EnvSerde::start(env);
        ints[e * 4 + 2] = msk::EnvSerde::steps(env);
        ints[e * 4 + 3] = msk::EnvSerde::done(env) ? 1 : 0;
    }
}

void ref_set_state(void* h, const double* q, const double* dq, const double* act, const double* lm,
                   const double* vm, const double* fm, const double* t, const int32_t* ints) {
    Batch& b = *static_cast<Batch*>(h);
    const int nq = b.spec.nq(), nm = b.spec.n_muscles();
    for (size_t e = 0; e < b.envs.size(); ++e) {
        msk::Env& env = *b.envs[e];
        msk::SimState& s = env.mutable_state();
        for (int i = 0; i < nq; ++i) {
            s.q[i] = q[e * nq + i];
            s.dq[i] = dq[e * nq + i];
        }
        for (int m = 0; m < nm; ++m) {
            s.muscles[static_cast<size_t>(m)].act = act[e * nm + m];
            s.muscles[static_cast<size_t>(m)].l_m = lm[e * nm + m];
            s.muscles[static_cast<size_t>(m)].v_m = vm[e * nm + m];
            s.muscles[static_cast<size_t>(m)].f_m = fm[e * nm + m];
        }
        s.t = t[e];
        msk::EnvSerde::t_index(env) = ints[e * 4 + 0];
        msk::EnvSerde::start(env) = ints[e * 4 + 1];
        msk::EnvSerde::steps(env) = ints[e * 4 + 2];
        msk::EnvSerde::done(env) = ints[e * 4 + 3] != 0;
    }
}

void ref_get_sampler(void* h, double* ema /* E x bins */) {
    Batch& b = *static_cast<Batch*>(h);
    for (size_t e = 0; e < b.envs.size(); ++e) {
        const auto& s = b.envs[e]->sampler();
        for (int i = 0; i < s.bins; ++i) ema[e * s.bins + i] = s.failure_ema[i];
    }
}

void ref_set_sampler(void* h, const double* ema /* E x bins */) {
    Batch& b = *static_cast<Batch*>(h);
    for (size_t e = 0; e < b.envs.size(); ++e) {
        auto& s = b.envs[e]->sampler();
        for (int i = 0; i < s.bins; ++i) s.failure_ema[i] = ema[e * s.bins + i];
    }
}

// Applies each env's pending outcomes to its own sampler, in order, then
// clears them (AdaptiveSampler::record, env.cpp:34-37).
void ref_record_own_outcomes(void* h) {
    Batch& b = *static_cast<Batch*>(h);
    for (auto& e : b.envs) {
        for (const auto& [bin, failed] : e->drain_episode_outcomes()) e->sampler().record(bin, failed);
    }
}

// Copies pending outcomes (E x cap), counts per env; clears them.
void ref_drain_outcomes(void* h, int32_t* bins, uint8_t* failed, int32_t* counts, int32_t cap) {
    Batch& b = *static_cast<Batch*>(h);
    for (size_t e = 0; e < b.envs.size(); ++e) {
        auto out = b.envs[e]->drain_episode_outcomes();
        const int n = static_cast<int>(std::min<size_t>(out.size(), static_cast<size_t>(cap)));
        counts[e] = static_cast<int32_t>(out.size());
        for (int i = 0; i < n; ++i) {
            bins[e * cap + i] = out[static_cast<size_t>(i)].first;
            failed[e * cap + i] = out[static_cast<size_t>(i)].second ? 1 : 0;
        }
    }
}

// Env e's Rng::serialize() text (rng.hpp:56-61) into buf; returns its length
// (or the needed length when len is too small).
int32_t ref_rng_serialize(void* h, int32_t e, char* buf, int32_t len) {
    Batch& b = *static_cast<Batch*>(h);
    const std::string s = b.envs[static_cast<size_t>(e)]->rng().serialize();
    if (static_cast<int32_t>(s.size()) < len) std::memcpy(buf, s.c_str(), s.size() + 1);
    return static_cast<int32_t>(s.size());
}

// Rng::deserialize (rng.hpp:63-68) of env e from text.
void ref_rng_deserialize(void* h, int32_t e, const char* text) {
    Batch& b = *static_cast<Batch*>(h);
    b.envs[static_cast<size_t>(e)]->rng().deserialize(text);
}

// Raw mt19937_64 draws of env e's stream (advances it).
void ref_rng_raw(void* h, int32_t e, int32_t n, uint64_t* out) {
    Batch& b = *static_cast<Batch*>(h);
    for (int i = 0; i < n; ++i) out[i] = b.envs[static_cast<size_t>(e)]->rng().raw();
}

// Rng(seed).uniform(lo, hi) draws (rng.hpp:26-30) of a fresh reference Rng:
// the stream Mlp::Mlp (nn.cpp:29-37) consumes for its weight init.
void ref_rng_uniform(uint64_t seed, double lo, double hi, int64_t n, double* out) {
    msk::Rng r(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = r.uniform(lo, hi);
}

// Philox excitations for a whole batch (E x nm), identical to the device's.
void ref_excitations(uint64_t seed, uint32_t step, int64_t global_env_offset, int32_t n_envs, int32_t nm,
                     double* out) {
    for (int e = 0; e < n_envs; ++e)
        for (int m = 0; m < nm; ++m)
            out[static_cast<size_t>(e) * nm + m] =
                excitation(seed, step, static_cast<uint32_t>(global_env_offset + e), m);
}

// Timed CPU loop: `steps` control steps of every env with Philox actions,
// done envs reset before their next step (the batched-harness convention).
// Returns wall seconds; *env_steps receives the number of env-steps taken.
// The reference's own Mlp(in = dΔ, hidden, 1, Head::Sigmoid) with parameters
// theta (nn.cpp:16-38 flat layout) as ref_bench's tracking reward; null clears it.
int32_t ref_set_discriminator(void* h, const double* theta, int64_t n, int32_t hidden) {
    Batch& b = *static_cast<Batch*>(h);
    if (!theta) {
        b.disc.reset();
        return 0;
    }
    msk::MlpShape sh;
    sh.in = b.delta_dim;
    sh.hidden = hidden;
    sh.out = 1;
    sh.head = msk::Head::Sigmoid;
    auto m = std::make_unique<msk::Mlp>(sh, 0);
    if (m->param_count() != n) return 1;
    for (int64_t i = 0; i < n; ++i) m->params()[i] = theta[i];
    b.disc = std::move(m);
    return 0;
}

double ref_bench(void* h, int32_t steps, uint64_t action_seed, int64_t* env_steps) {
    Batch& b = *static_cast<Batch*>(h);
    const int n = static_cast<int>(b.envs.size());
    const int nm = b.spec.n_muscles();
    std::vector<int64_t> counts(static_cast<size_t>(n), 0);
    uint32_t step_ctr = 0;
    auto fn = [&](int begin, int end, int) {
        Eigen::VectorXd a(nm);
        for (int e = begin; e < end; ++e) {
            msk::Env& env = *b.envs[static_cast<size_t>(e)];
            if (env.done()) env.reset();
            for (int m = 0; m < nm; ++m) a[m] = excitation(action_seed, step_ctr, static_cast<uint32_t>(e), m);
            if (b.disc)  // Env::step(action, fn), fn = reward_from_discriminator
                env.step(a, [&](const Eigen::VectorXd& d) {
                    const double y = b.disc->forward_one(d)[0];
                    return -std::log(1.0 - std::min(std::max(y, 1e-4), 1.0 - 1e-4));
                });
            else
                env.step(a);
            ++counts[static_cast<size_t>(e)];
        }
    };
    const auto t0 = std::chrono::steady_clock::now();
    for (int s = 0; s < steps; ++s, ++step_ctr) {
        if (b.pool)
            b.pool->parallel_chunks(n, std::max(1, n / (4 * b.pool->workers())), fn);
        else
            fn(0, n, 0);
    }
    const auto t1 = std::chrono::steady_clock::now();
    int64_t total = 0;
    for (int64_t c : counts) total += c;
    if (env_steps) *env_steps = total;
    return std::chrono::duration<double>(t1 - t0).count();
}

// ---- free functions of the reference, for known-answer tests ---------------

double ref_force_length_active(double l) { return msk::force_length_active(l); }
double ref_force_velocity(double v) { return msk::force_velocity(v); }
double ref_force_passive(double l) { return msk::force_passive(l); }
double ref_mtu_force(double act, double l, double v, double f_max) {
    msk::MuscleParams p;
    p.f_max = f_max;
    return msk::mtu_force(act, l, v, p);
}
double ref_activation_step(double act, double u, double dt, double tau_act, double tau_deact) {
    msk::MuscleParams p;
    p.tau_act = tau_act;
    p.tau_deact = tau_deact;
    return msk::activation_step(act, u, dt, p);
}
double ref_wrap_angle(double a) { return msk::wrap_angle(a); }

void ref_mass_matrix(void* h, const double* q, double* M) {
    Batch& b = *static_cast<Batch*>(h);
    const int nq = b.spec.nq();
    Eigen::VectorXd qv(nq);
    for (int i = 0; i < nq; ++i) qv[i] = q[i];
    const Eigen::MatrixXd m = msk::mass_matrix(b.spec, qv);
    for (int i = 0; i < nq; ++i)
        for (int j = 0; j < nq; ++j) M[i * nq + j] = m(i, j);
}

void ref_moment_arms(void* h, const double* q, double* Jm /* nm x nq */) {
    Batch& b = *static_cast<Batch*>(h);
    const int nq = b.spec.nq(), nm = b.spec.n_muscles();
    Eigen::VectorXd qv(nq);
    for (int i = 0; i < nq; ++i) qv[i] = q[i];
    const Eigen::MatrixXd m = msk::moment_arms(b.spec, qv);
    for (int i = 0; i < nm; ++i)
        for (int j = 0; j < nq; ++j) Jm[i * nq + j] = m(i, j);
}

void ref_bias_forces(void* h, const double* q, const double* dq, double* C) {
    Batch& b = *static_cast<Batch*>(h);
    const int nq = b.spec.nq();
    Eigen::VectorXd qv(nq), dqv(nq);
    for (int i = 0; i < nq; ++i) {
        qv[i] = q[i];
        dqv[i] = dq[i];
    }
    const Eigen::VectorXd c = msk::bias_forces(b.spec, qv, dqv);
    for (int i = 0; i < nq; ++i) C[i] = c[i];
}

double ref_mtu_length(void* h, const double* q, int32_t m) {
    Batch& b = *static_cast<Batch*>(h);
    Eigen::VectorXd qv(b.spec.nq());
    for (int i = 0; i < b.spec.nq(); ++i) qv[i] = q[i];
    return msk::mtu_length(b.spec, qv, m);
}

double ref_mechanical_energy(void* h, const double* q, const double* dq) {
    Batch& b = *static_cast<Batch*>(h);
    const int nq = b.spec.nq();
    Eigen::VectorXd qv(nq), dqv(nq);
    for (int i = 0; i < nq; ++i) {
        qv[i] = q[i];
        dqv[i] = dq[i];
    }
    return msk::mechanical_energy(b.spec, qv, dqv);
}

// Key-body COM positions (K x 2) and frame angles (K) at q.
void ref_key_bodies(void* h, const double* q, double* pos, double* ang) {
    Batch& b = *static_cast<Batch*>(h);
    Eigen::VectorXd qv(b.spec.nq());
    for (int i = 0; i < b.spec.nq(); ++i) qv[i] = q[i];
    const msk::Kinematics kin = msk::forward_kinematics(b.spec, qv);
    Eigen::Matrix2Xd p;
    Eigen::VectorXd a;
    msk::key_body_state(b.spec, kin, p, a);
    for (int k = 0; k < b.spec.n_key_bodies(); ++k) {
        pos[2 * k] = p(0, k);
        pos[2 * k + 1] = p(1, k);
        ang[k] = a[k];
    }
}

}  // extern "C"
