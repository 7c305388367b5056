// C++ host program driving the env-stepper through include/msk_gpu.hpp —
// the "C++ host code calling CUDA through a thin C-ABI" of north_star.
// Steps E whole-body envs with Philox excitations, auto-resets done envs,
// computes the tracking reward with the built-in tensor-core discriminator,
// and prints throughput, a checksum of the final observations and the mean reward.
//
//   build: make -C tools cpp_demo   (links paper_2603_29332_b200/libmsk_b200.so)
//   run:   tools/cpp_demo <model.json> <clip.csv> [envs] [steps] [policy_width]
// With policy_width > 0 the actions come from the on-device flow policy
// (msk_policy_*: Gaussian pi0 + 20-step flow ODE on the tensor cores) and every
// step is recorded into the on-device rollout buffer; every 8 steps GAE runs and
// the discriminator takes one training step on the iteration's Δ rows
// (msk_disc_trainer_*), published into the reward path.
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <memory>
#include <stdexcept>
#include <vector>

#include "msk_gpu.hpp"

int main(int argc, char** argv) {
    if (argc < 3) {
        std::fprintf(stderr, "usage: %s model.json clip.csv [envs] [steps]\n", argv[0]);
        return 2;
    }
    const int E = argc > 3 ? std::atoi(argv[3]) : 1024;
    const int steps = argc > 4 ? std::atoi(argv[4]) : 20;
    const int width = argc > 5 ? std::atoi(argv[5]) : 0;
    try {
        msk::gpu::EnvConfig cfg;
        cfg.episode_horizon = 1000;
        cfg.rsi = false;
        msk::gpu::EnvBatch env(argv[1], argv[2], E, cfg);
        env.set_eval_mode(true);
        float *actions, *obs, *delta, *raux;
        uint8_t* flags;
        cudaMalloc(&actions, sizeof(float) * E * env.action_dim());
        cudaMalloc(&obs, sizeof(float) * E * env.observation_dim());
        cudaMalloc(&delta, sizeof(float) * E * env.delta_dim());
        cudaMalloc(&raux, sizeof(float) * E);
        cudaMalloc(&flags, E);
        float* reward;
        cudaMalloc(&reward, sizeof(float) * E);
        // frozen tracking discriminator D = Mlp(delta_dim, 256, 1, Sigmoid), seed 7
        env.set_discriminator(msk::gpu::EnvBatch::mlp_init(env.delta_dim(), 256, 1, 7), 256);
        env.reset(nullptr, 0xff, obs);
        msk::gpu::StepBuffers out{obs, delta, raux, flags};
        // optional on-device policy + rollout buffer (C ABI)
        msk_policy* pol = nullptr;
        msk_rollout* ro = nullptr;
        std::unique_ptr<msk::gpu::DiscTrainer> dtrain;
        double* dloss = nullptr;
        // iteration boundary (msk_gpu_iteration_exchange; nccl_comm = nullptr: one rank)
        double *stats = nullptr, *stats_out = nullptr, *norm = nullptr;
        const int D = env.observation_dim();
        cudaMalloc(&stats, 7 * sizeof(double));
        cudaMalloc(&stats_out, 7 * sizeof(double));
        cudaMalloc(&norm, (1 + 2 * D) * sizeof(double));
        cudaMemset(stats, 0, 7 * sizeof(double));
        {
            std::vector<double> n0(1 + 2 * D, 0.0);
            for (int i = 0; i < D; ++i) n0[1 + D + i] = 1.0;  // RunningNorm(dim): count 0, mean 0, var 1
            cudaMemcpy(norm, n0.data(), n0.size() * sizeof(double), cudaMemcpyHostToDevice);
        }
        float *a0 = nullptr, *logp = nullptr, *value = nullptr, *adv = nullptr, *ret = nullptr;
        const int horizon = 8;
        if (width > 0) {
            const int D = env.observation_dim(), NM = env.action_dim();
            auto pi = msk::gpu::EnvBatch::mlp_init(D, width, NM, 1, 0.01);
            auto psi = msk::gpu::EnvBatch::mlp_init(5 + D + NM, width, NM, 2, 0.01);
            std::vector<double> log_std(NM, -1.0);
            if (msk_policy_create(D, NM, width, pi.data(), static_cast<int64_t>(pi.size()), 1.0, 0.5, log_std.data(),
                                  psi.data(), static_cast<int64_t>(psi.size()), 20, 0.05, E, 0, &pol) != MSK_OK)
                throw std::runtime_error(msk_policy_last_error(nullptr));
            if (msk_rollout_create(E, horizon, D, NM, env.delta_dim(), 0, &ro) != MSK_OK)
                throw std::runtime_error(msk_rollout_last_error(nullptr));
            cudaMalloc(&a0, sizeof(float) * E * NM);
            cudaMalloc(&logp, sizeof(float) * E);
            cudaMalloc(&value, sizeof(float) * E);
            cudaMemset(value, 0, sizeof(float) * E);
            cudaMalloc(&adv, sizeof(float) * E * horizon);
            cudaMalloc(&ret, sizeof(float) * E * horizon);
            dtrain = std::make_unique<msk::gpu::DiscTrainer>(
                env.delta_dim(), 256, msk::gpu::EnvBatch::mlp_init(env.delta_dim(), 256, 1, 7), 3e-5, 10.0,
                E * horizon);
            cudaMalloc(&dloss, 3 * sizeof(double));
        }
        auto one_step = [&](int s) {
            if (pol) {  // a = flow-refined Gaussian sample from the current observation
                msk_rollout_record(ro, s % horizon, obs, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                                   nullptr);
                if (msk_policy_sample_graph(pol, obs, E, 1, 0x5EED, static_cast<uint32_t>(s), 0, actions, a0, logp,
                                            nullptr) != MSK_OK)
                    throw std::runtime_error(msk_policy_last_error(pol));
            } else {
                env.fill_excitations(0x5EED, static_cast<uint32_t>(s), actions);
            }
            env.step(actions, out, reward);  // Env::step(action, fn): reward = r(D(Δ)) + reward_aux
            msk_gpu_rollout_stats(env.handle(), reward, flags, stats, nullptr);
            if ((s + 1) % horizon == 0) {  // drain, stats, obs moments, (all-gather), ordered merge
                env.iteration_exchange(horizon, obs, stats, norm, stats_out);
                cudaMemsetAsync(stats, 0, 7 * sizeof(double));
            }
            if (ro) {
                msk_rollout_record(ro, s % horizon, nullptr, a0, actions, logp, reward, flags, value, delta, nullptr);
                if ((s + 1) % horizon == 0) {
                    msk_rollout_gae(ro, value, 0.99f, 0.95f, 1, adv, ret, nullptr);
                    dtrain->step(static_cast<const float*>(msk_rollout_field(ro, 7)), E * horizon, env.delta_dim(),
                                 dloss);
                    dtrain->publish(env);
                }
            }
            env.reset(flags, MSK_FLAG_DONE, pol ? obs : nullptr);  // batched auto-reset
        };
        // one untimed iteration: graph capture, cuBLAS / module first-use costs
        for (int s = 0; s < horizon; ++s) one_step(s);
        cudaDeviceSynchronize();
        const auto t0 = std::chrono::steady_clock::now();
        for (int s = horizon; s < horizon + steps; ++s) one_step(s);
        cudaDeviceSynchronize();
        const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        std::vector<float> h(static_cast<size_t>(E) * env.observation_dim());
        cudaMemcpy(h.data(), obs, sizeof(float) * h.size(), cudaMemcpyDeviceToHost);
        double checksum = 0.0;
        for (float v : h) checksum += v;
        std::vector<float> hr(static_cast<size_t>(E));
        cudaMemcpy(hr.data(), reward, sizeof(float) * E, cudaMemcpyDeviceToHost);
        double rsum = 0.0;
        for (float v : hr) rsum += v;
        double lh[3] = {0, 0, 0}, so[7] = {0}, ncount = 0.0;
        if (dloss) cudaMemcpy(lh, dloss, sizeof(lh), cudaMemcpyDeviceToHost);
        cudaMemcpy(so, stats_out, sizeof(so), cudaMemcpyDeviceToHost);
        cudaMemcpy(&ncount, norm, sizeof(double), cudaMemcpyDeviceToHost);
        std::printf("envs=%d steps=%d policy_width=%d env-steps/s=%.0f obs_checksum=%.6e mean_reward=%.6f "
                    "disc_loss=%.6f last_iteration_steps=%.0f norm_count=%.0f\n",
                    E, steps, width, E * steps / secs, checksum, rsum / E, lh[0], so[0], ncount);
        cudaFree(stats);
        cudaFree(stats_out);
        cudaFree(norm);
        cudaFree(reward);
        if (dloss) cudaFree(dloss);
        if (pol) msk_policy_destroy(pol);
        if (ro) msk_rollout_destroy(ro);
        for (float* p : {a0, logp, value, adv, ret})
            if (p) cudaFree(p);
        cudaFree(actions);
        cudaFree(obs);
        cudaFree(delta);
        cudaFree(raux);
        cudaFree(flags);
    } catch (const std::exception& ex) {
        std::fprintf(stderr, "error: %s\n", ex.what());
        return 1;
    }
    return 0;
}
