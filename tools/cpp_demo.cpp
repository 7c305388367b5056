// C++ host program driving the env-stepper through include/msk_gpu.hpp —
// the "C++ host code calling CUDA through a thin C-ABI" of north_star.
// Steps E whole-body envs with Philox excitations, auto-resets done envs,
// computes the tracking reward with the built-in tensor-core discriminator,
// and prints throughput, a checksum of the final observations and the mean reward.
//
//   build: make -C tools cpp_demo   (links paper_2603_29332_b200/libmsk_b200.so)
//   run:   tools/cpp_demo <model.json> <clip.csv> [envs] [steps]
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "msk_gpu.hpp"

int main(int argc, char** argv) {
    if (argc < 3) {
        std::fprintf(stderr, "usage: %s model.json clip.csv [envs] [steps]\n", argv[0]);
        return 2;
    }
    const int E = argc > 3 ? std::atoi(argv[3]) : 1024;
    const int steps = argc > 4 ? std::atoi(argv[4]) : 20;
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
        cudaDeviceSynchronize();
        const auto t0 = std::chrono::steady_clock::now();
        for (int s = 0; s < steps; ++s) {
            env.fill_excitations(0x5EED, static_cast<uint32_t>(s), actions);
            env.step(actions, out, reward);  // Env::step(action, fn): reward = r(D(Δ)) + reward_aux
            env.reset(flags, MSK_FLAG_DONE);  // batched auto-reset
        }
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
        std::printf("envs=%d steps=%d env-steps/s=%.0f obs_checksum=%.6e mean_reward=%.6f\n", E, steps,
                    E * steps / secs, checksum, rsum / E);
        cudaFree(reward);
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
