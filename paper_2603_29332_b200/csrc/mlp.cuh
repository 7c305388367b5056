// Tiled bf16 GEMM on the tcgen05 tensor cores + MLP epilogues (see mlp.cu).
//
// Layouts ("tiled" = what the UMMA descriptors and 1-D TMA bulk copies read):
//   activations A [M x K]: blocks of 128 rows x 64 K (16 KB) at
//       ((mb * KB) + kb) * 16 KB, KB = K/64, rows/K padded with zeros;
//   weights     W [N x K]: blocks of 256 rows x 64 K (32 KB) at
//       ((nb * KB) + kb) * 32 KB;
// inside a block element (r, k) sits at ((r/8)*8 + k/8)*128 + (r%8)*16 + (k%8)*2
// (K-major core matrices, no swizzle: LBO = 128 B, SBO = 1024 B).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <vector>

namespace msk_b200 {

#ifndef MSK_GEMM_BN
#define MSK_GEMM_BN 256
#endif
constexpr int kGemmBM = 128, kGemmBN = MSK_GEMM_BN, kGemmBK = 64;

__host__ __device__ inline int pad_to(int x, int m) { return (x + m - 1) / m * m; }
inline size_t tiled_a_bytes(int M, int K) { return static_cast<size_t>(pad_to(M, kGemmBM)) * pad_to(K, kGemmBK) * 2; }
inline size_t tiled_w_bytes(int N, int K) { return static_cast<size_t>(pad_to(N, kGemmBN)) * pad_to(K, kGemmBK) * 2; }

// Host: pack a column-major (Eigen/Mlp layout) f64 matrix W[rows x cols] — or a
// column slice [c0, c0 + nc) of it — into the tiled bf16 weight image.
std::vector<uint16_t> pack_weights(const double* W, int rows, int cols, int c0, int nc);

enum GemmEpi : int {
    kEpiTanhTiled = 0,  // out_a (tiled bf16, K = N) = tanh(acc + bias[n] + addend[m, n])
    kEpiF32 = 1,        // out_f[m * ld + n] = acc + bias[n] (+ addend)           (n < n_valid)
    kEpiOde = 2,        // a[m * ld + n] += dt * (acc + bias[n]); out_a = bf16 tiled copy of the new a
    kEpiTanhPre = 3,    // z = scale * acc + bias[n] + addend[m, n]: out_f = z (f32), out_a = tanh(z) (tiled)
    kEpiTanhAcc = 4,    // y = tanh(acc + bias[n]): out_a = y (tiled), out_f[m, n] += y (f32 running sum)
};

struct GemmArgs {
    const void* A = nullptr;       // tiled activations
    const void* W = nullptr;       // tiled weights
    const float* bias = nullptr;   // [N] (nullable)
    const float* addend = nullptr; // fp32 row-major [M x ld_add] (nullable)
    int ld_add = 0;
    void* out_a = nullptr;         // tiled bf16 output (K = N padded) for the next layer
    float* out_f = nullptr;        // fp32 row-major output / ODE state
    int ld_f = 0;
    int M = 0, N = 0, K = 0;       // logical sizes (N, K padded internally)
    int n_valid = 0;               // columns of out_f that are written
    float dt = 0.0f;
    float scale = 1.0f, offset = 0.0f;  // kEpiF32: affine head y = scale * z + offset
    // > 0: out_f and addend are internal f32 buffers in the F4 layout [N/4][f4_rows][4]
    // (element (m, n) at ((n / 4) * f4_rows + m) * 4 + n % 4): a warp's 32 rows x one
    // float4 are 512 contiguous bytes in the row-per-thread epilogue.  0: row-major.
    int f4_rows = 0;
};

cudaError_t prepare_gemm();
// The ψ ODE's 3 n_ode − 1 hidden layers in one persistent launch (see mlp.cu
// ode_kernel): g2 / g3 / g1 carry W, bias, M, N = K = H and the f32 side buffers
// (g3: hsum, g1: z, scale = dt); x0 / y0 the two tiled activation images (x0
// holds tanh(z_0)); qd the per-step ψ1 biases.  H / 256 <= 8 (cluster size).
cudaError_t launch_ode(const GemmArgs& g2, const GemmArgs& g3, const GemmArgs& g1, void* x0, void* y0,
                       const float* qd, int n_ode, int H, cudaStream_t s);
size_t gemm_smem_bytes();
cudaError_t launch_gemm(const GemmArgs& g, int epi, cudaStream_t s);

// obs f32 [M x D] -> normalised (RunningNorm::apply) bf16 tiled A [M x D]
cudaError_t launch_obs_to_tiled(const float* obs, int M, int D, const float* mean, const float* inv_sd, void* out,
                                cudaStream_t s);
// f32 row-major [M x D] -> bf16 tiled (f4_rows > 0: x in the F4 layout of GemmArgs)
cudaError_t launch_f32_to_tiled(const float* x, int M, int D, int ld, void* out, cudaStream_t s, int f4_rows = 0);

}  // namespace msk_b200
