// Device discriminator (tracking reward D(Δ)) — see disc.cu.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <vector>

namespace msk_b200 {

// Host-side images built from the Mlp flat parameters (nn.cpp:16-38).
struct DiscHost {
    int din = 0, hidden = 0, k1 = 0;  // k1 = din rounded up to the MMA K step (16)
    std::vector<uint16_t> w1, w2, w3;  // bf16 K-major core-matrix images (H x k1, H x H, H x H)
    std::vector<float> bias;           // b1 | b2 | b3 | w4 | b4 (4 H + 1 floats)
    // fp32-class (split-bf16) mode: W = hi + lo (both bf16), each layer's image in
    // K16-chunk-major order (chunk c = rows x 16 K, contiguous) for the streamed ring
    std::vector<uint16_t> c1_hi, c1_lo, c2_hi, c2_lo, c3_hi, c3_lo;
};

// Device view passed to the kernel by value.
struct DiscDev {
    int din = 0, hidden = 0, k1 = 0;
    uint32_t tmem_cols = 0;  // power of two >= max(32, hidden)
    const void* w1 = nullptr;
    const void* w2 = nullptr;
    const void* w3 = nullptr;
    const float* bias = nullptr;  // b1 | b2 | b3 | w4 | b4
    int precise = 1;  // 1: split-bf16 operands (hi + lo), accurate tanh: fp32-class; 0: bf16 fast mode
    const void* c_hi[3] = {nullptr, nullptr, nullptr};  // chunked split images (see DiscHost)
    const void* c_lo[3] = {nullptr, nullptr, nullptr};
};

DiscHost build_disc_images(const double* theta, long long n_params, int din, int hidden);
size_t disc_smem_bytes(const DiscDev& P);
cudaError_t prepare_disc(const DiscDev& P);
// reward[i] = r(D(delta_i)); with flags: reward = r + raux for stepped envs,
// 0 for diverged ones, untouched for NOT_STEPPED / BAD_ACTION rows.
cudaError_t launch_disc(const DiscDev& P, const float* delta, int ld, int n, const float* raux,
                        const uint8_t* flags, float* reward, cudaStream_t s, bool pdl);

// Rewrites P's images in place from f64 Mlp parameters on the device (same
// din / hidden), e.g. after a device training step (disc_train.cu).
cudaError_t launch_disc_repack(const double* theta, const DiscDev& P, cudaStream_t s);

}  // namespace msk_b200

struct msk_disc_trainer;
namespace msk_b200 {
const double* disc_trainer_theta(const msk_disc_trainer* t, int* din, int* hidden);
}
