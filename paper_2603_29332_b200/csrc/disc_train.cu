// Discriminator training step on the device (second half;
// SPEC.md:412-421 train_discriminator):
//
//   loss = -log clamp(D(0)) - mean_i log(1 - clamp(D(Δ_i))) + λ mean_i ||∇_Δ D(Δ_i)||²
//
// followed by one Adam step (nn.cpp:224-240).  D = Mlp(in, W, 1, Head::Sigmoid)
// with master parameters θ in the reference's flat layout (nn.cpp:16-38, W
// column-major) and the Adam moments in f64 on the device.
//
// Structure (all activations column-major, R = B + 1 rows: the B Δ rows plus
// the zero input of the D(0) term as the last row):
//   * forward  H_l = tanh(H_{l-1} W_lᵀ + b_l), y = sigmoid(H_3 w_4 + b_4)
//     (nn.cpp:54-73);
//   * input gradient g = dy/dx (d-chain) and its forward tangent ζ_l, u_l
//     (nn.cpp:157-171);
//   * ONE reverse pass carrying [tangent; primal] adjoints stacked as 2R-row
//     matrices: the logistic loss's upstream (Mlp::backward, nn.cpp:80-129)
//     enters the primal adjoint of the head, so it rides the gradient-penalty
//     reverse pass (nn.cpp:173-221) — both are linear in the head adjoint;
//   * each weight gradient is one GEMM over the stacked 2R rows,
//     gW_l = [b_ζ; b_z]ᵀ [u; H] (the reference's two products in one);
//   * bias gradients: fixed-order column sums in f64; Adam in f64 with the
//     reference's non-finite-gradient skip evaluated on the device;
//   * each half of a stacked matrix is padded to Rp = R rounded up to 4 rows
//     (16-B aligned leading dimensions and half offsets, so cuBLAS picks its
//     sm100 tcgen05 kernels); the column kernels write zeros into the padding
//     and the GEMMs run over the padded extents.
// The GEMMs are plain library GEMMs (cuBLAS, f32 data) in the math mode the
// caller picks: FP32 (default) or TF32 tensor cores.  Only cuBLAS 12.0-level
// entry points are used: the process may already hold torch's bundled
// libcublas.so.12, which then serves these symbols (the BF16x9 FP32 emulation
// of cuBLAS 12.9 is therefore not used).  Elementwise / reduction work is
// fused into the kernels below.  This is the learner side of the loop,
// launched once per rollout iteration; the stepping path never calls it.
#include <cublas_v2.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/msk_gpu.h"
#include "disc.hpp"

namespace {

constexpr double kClampLo = 1e-4, kClampHi = 1.0 - 1e-4;
// Column-wise elementwise kernels: grid (row blocks, columns), 256 threads,
// 4 rows per thread (coalesced along the column-major rows, 4 loads in flight).
constexpr int kRowsPerThread = 4, kRowsPerBlock = 256 * kRowsPerThread;

// X2 bottom half: primal input rows (Δ, then one zero row) — a 32 x 32 tile
// transpose through shared memory (row-major Δ in, column-major X out).
__global__ void pack_input_kernel(const float* __restrict__ delta, int B, int ld, int din, int R, int Rp, float* X2) {
    __shared__ float tile[32][33];
    const int i0 = blockIdx.x * 32, j0 = blockIdx.y * 32;
    for (int r = threadIdx.y; r < 32; r += 8) {
        const int i = i0 + r, j = j0 + threadIdx.x;
        tile[r][threadIdx.x] = (i < B && j < din) ? delta[static_cast<size_t>(i) * ld + j] : 0.0f;
    }
    __syncthreads();
    for (int c = threadIdx.y; c < 32; c += 8) {
        const int j = j0 + c, i = i0 + threadIdx.x;
        if (j < din && i < Rp) X2[static_cast<size_t>(j) * 2 * Rp + Rp + i] = tile[threadIdx.x][c];
    }
}

// The column-wise kernels cover rows [0, Rp) of a half and write 0 to the
// padding rows [R, Rp), so every GEMM over a padded extent sees zeros there.

// x = tanh(x + b[col]) over a column-major block (leading dim ld).
__global__ void bias_tanh_kernel(float* x, int R, int Rp, int ld, const float* __restrict__ b) {
    const int j = blockIdx.y;
#pragma unroll
    for (int k = 0; k < kRowsPerThread; ++k) {
        const int i = blockIdx.x * kRowsPerBlock + k * 256 + threadIdx.x;
        if (i >= Rp) break;
        float* p = x + static_cast<size_t>(j) * ld + i;
        *p = i < R ? tanhf(*p + b[j]) : 0.0f;
    }
}

// Head (nn.cpp:66-68 sigmoid; SPEC.md:416 clamped logs): y, head' (d4), head'' (dd4),
// the logistic loss's head adjoint dz4 (Mlp::backward's dz4 = upstream * y (1 - y)),
// and the per-row logistic loss term.
__global__ void head_kernel(const float* __restrict__ z4, const float* __restrict__ b3, int B, int R, float* d4,
                            float* dd4, float* dz4, double* lrow) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= R) return;
    const double y = 1.0 / (1.0 + exp(-(static_cast<double>(z4[i]) + b3[0])));
    const double yc = fmin(fmax(y, kClampLo), kClampHi);
    const bool inside = y > kClampLo && y < kClampHi;
    const double d = y * (1.0 - y);
    d4[i] = static_cast<float>(d);
    dd4[i] = static_cast<float>(d * (1.0 - 2.0 * y));
    if (i < B) {  // -(1/B) log(1 - clamp(y)): upstream 1 / (B (1 - y))
        dz4[i] = inside ? static_cast<float>(y / B) : 0.0f;
        lrow[i] = -log(1.0 - yc) / B;
    } else {  // -log clamp(D(0)): upstream -1 / y
        dz4[i] = inside ? static_cast<float>(-(1.0 - y)) : 0.0f;
        lrow[i] = -log(yc);
    }
}

// d3 = (d4 ⊗ w4) ∘ (1 - H3²)   (nn.cpp:161)
__global__ void d3_kernel(const float* __restrict__ d4, const float* __restrict__ w4, const float* __restrict__ H3,
                          int ldh, int R, int Rp, float* d3, int ldd) {
    const int j = blockIdx.y;
#pragma unroll
    for (int k = 0; k < kRowsPerThread; ++k) {
        const int i = blockIdx.x * kRowsPerBlock + k * 256 + threadIdx.x;
        if (i >= Rp) break;
        const float h = H3[static_cast<size_t>(j) * ldh + i];
        d3[static_cast<size_t>(j) * ldd + i] = i < R ? d4[i] * w4[j] * (1.0f - h * h) : 0.0f;
    }
}

// out = x ∘ (1 - H²), x and out [R x H] (ld lx / lo), H read with leading dim ldh.
__global__ void gate_kernel(const float* x, int lx, const float* __restrict__ Hm, int ldh, int R, int Rp, float* out,
                            int lo) {
    const int j = blockIdx.y;
#pragma unroll
    for (int k = 0; k < kRowsPerThread; ++k) {
        const int i = blockIdx.x * kRowsPerBlock + k * 256 + threadIdx.x;
        if (i >= Rp) break;
        const float h = Hm[static_cast<size_t>(j) * ldh + i];
        out[static_cast<size_t>(j) * lo + i] = i < R ? x[static_cast<size_t>(j) * lx + i] * (1.0f - h * h) : 0.0f;
    }
}

// Penalty + head adjoints (nn.cpp:172, 187-188 with the logistic dz4 added to b_z4):
// V[i] = b_ζ4 = 2 w d4, V[Rp + i] = b_z4 = 2 w dd4 ζ4 + dz4, w = λ/B on Δ rows, 0 on the zero row.
__global__ void head2_kernel(const float* __restrict__ d4, const float* __restrict__ dd4,
                             const float* __restrict__ zeta4, const float* __restrict__ dz4, int B, int R, int Rp,
                             float lamB, float* V, double* prow) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= Rp) return;
    if (i >= R) {
        V[i] = V[Rp + i] = 0.0f;
        return;
    }
    const float w = i < B ? lamB : 0.0f;
    V[i] = 2.0f * w * d4[i];
    V[Rp + i] = 2.0f * w * dd4[i] * zeta4[i] + dz4[i];
    prow[i] = i < B ? static_cast<double>(d4[i]) * zeta4[i] / B : 0.0;
}

// Layer-3 adjoints from the head: [b_u3; b_h3] = V ⊗ w4, then the elementwise
// step below (nn.cpp:191-195).
// rev_elem: S = [b_u; b_h] (2R x H) -> [b_ζ; b_z] with
//   b_ζ = G ∘ b_u,  b_h += -2 H ∘ ζ ∘ b_u,  b_z = G ∘ b_h   (G = 1 - H²)
template <bool OUTER>
__global__ void rev_elem_kernel(float* S, const float* __restrict__ V, const float* __restrict__ w4,
                                const float* __restrict__ Hm, int ldh, const float* __restrict__ Z, int R, int Rp,
                                int H) {
    const size_t ld = 2 * static_cast<size_t>(Rp);
    const int j = blockIdx.y;
#pragma unroll
    for (int k = 0; k < kRowsPerThread; ++k) {
        const int i = blockIdx.x * kRowsPerBlock + k * 256 + threadIdx.x;
        if (i >= Rp) break;
        if (i >= R) {
            S[j * ld + i] = S[j * ld + Rp + i] = 0.0f;
            continue;
        }
        float bu, bh;
        if constexpr (OUTER) {
            bu = V[i] * w4[j];
            bh = V[Rp + i] * w4[j];
        } else {
            bu = S[j * ld + i];
            bh = S[j * ld + Rp + i];
        }
        const float h = Hm[static_cast<size_t>(j) * ldh + i];
        const float z = Z[static_cast<size_t>(j) * Rp + i];
        const float g = 1.0f - h * h;
        bh = fmaf(-2.0f * h * z, bu, bh);
        S[j * ld + i] = g * bu;
        S[j * ld + Rp + i] = g * bh;
    }
}

// out[j] = Σ_i x[j * ld + i], i < rows — fixed-order f64 sum, one block per column.
__global__ void __launch_bounds__(256) colsum_kernel(const float* __restrict__ x, int rows, size_t ld, float* out) {
    __shared__ double red[8];
    const int j = blockIdx.x;
    double s = 0.0;
    for (int i = threadIdx.x; i < rows; i += 256) s += x[j * ld + i];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < 8; ++w) t += red[w];
        out[j] = static_cast<float>(t);
    }
}

// loss[0] = total, loss[1] = logistic, loss[2] = mean penalty (f64, fixed order).
__global__ void __launch_bounds__(1024) loss_kernel(const double* __restrict__ lrow, const double* __restrict__ prow,
                                                    int R, double lam, double* loss) {
    __shared__ double red[2][32];
    double a = 0.0, b = 0.0;
    for (int i = threadIdx.x; i < R; i += 1024) {
        a += lrow[i];
        b += prow[i];
    }
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
    }
    if ((threadIdx.x & 31) == 0) {
        red[0][threadIdx.x >> 5] = a;
        red[1][threadIdx.x >> 5] = b;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0, p = 0.0;
        for (int w = 0; w < 32; ++w) {
            s += red[0][w];
            p += red[1][w];
        }
        loss[0] = s + lam * p;
        loss[1] = s;
        loss[2] = p;
    }
}

__global__ void finite_kernel(const float* __restrict__ g, long long n, int* bad) {
    bool b = false;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x)
        b |= !isfinite(g[i]);
    if (__any_sync(0xffffffffu, b) && (threadIdx.x & 31) == 0) atomicOr(bad, 1);
}

// Adam (nn.cpp:224-240), f64 moments and master parameters; skipped when the
// gradient has a non-finite entry (bad != 0).  counts = {step_count, skipped}.
__global__ void adam_kernel(const float* __restrict__ g, long long n, const int* bad, const long long* counts,
                            double lr, double b1, double b2, double eps, double* theta, double* m, double* v,
                            float* theta32) {
    if (*bad) return;
    const double t = static_cast<double>(counts[0] + 1);
    const double bc1 = 1.0 - pow(b1, t), bc2 = 1.0 - pow(b2, t);
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const double gi = g[i];
        const double mi = b1 * m[i] + (1.0 - b1) * gi;
        const double vi = b2 * v[i] + (1.0 - b2) * gi * gi;
        m[i] = mi;
        v[i] = vi;
        const double th = theta[i] - lr * (mi / bc1) / (sqrt(vi / bc2) + eps);
        theta[i] = th;
        theta32[i] = static_cast<float>(th);
    }
}

__global__ void adam_commit_kernel(int* bad, long long* counts) {
    if (*bad)
        ++counts[1];
    else
        ++counts[0];
    *bad = 0;
}

__global__ void to_f32_kernel(const double* x, long long n, float* y) {
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x)
        y[i] = static_cast<float>(x[i]);
}

int grid_for(size_t n) { return static_cast<int>(std::min<size_t>((n + 255) / 256, 148 * 16)); }

}  // namespace

struct msk_disc_trainer {
    int device = 0, din = 0, H = 0, max_rows = 0, math = 0;
    long long P = 0;
    long long o1 = 0, o2 = 0, o3 = 0;  // offsets of W1, W2, W3 (= w4) in θ
    double lr = 0.0, lam = 0.0;
    double *theta = nullptr, *m = nullptr, *v = nullptr;
    float *theta32 = nullptr, *grad = nullptr;
    long long* counts = nullptr;  // {Adam step_count, skipped}
    int* bad = nullptr;
    // activations / adjoints (column-major; R = max_rows + 1)
    float *X2 = nullptr, *A[4] = {}, *Z[4] = {}, *T1 = nullptr, *T2 = nullptr, *S1 = nullptr, *S2 = nullptr;
    float *z4 = nullptr, *d4 = nullptr, *dd4 = nullptr, *dz4 = nullptr, *zeta4 = nullptr, *V = nullptr;
    double *lrow = nullptr, *prow = nullptr, *loss = nullptr;
    cublasHandle_t blas = nullptr;
    std::vector<void*> allocs;
    std::string err;
};

namespace {
thread_local std::string g_dt_err;

int dtfail(msk_disc_trainer* t, const std::string& m, int code = MSK_ERR_CONTRACT) {
    g_dt_err = m;
    if (t) t->err = m;
    return code;
}

void ckc(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}
void ckb(cublasStatus_t s, const char* what) {
    if (s != CUBLAS_STATUS_SUCCESS) throw std::runtime_error(std::string(what) + ": cuBLAS status " + std::to_string(s));
}

template <class T>
T* talloc(msk_disc_trainer* t, size_t n) {
    void* p = nullptr;
    ckc(cudaMalloc(&p, std::max<size_t>(1, n) * sizeof(T)), "cudaMalloc");
    ckc(cudaMemset(p, 0, std::max<size_t>(1, n) * sizeof(T)), "cudaMemset");
    t->allocs.push_back(p);
    return static_cast<T*>(p);
}

cublasComputeType_t compute_type(int math) { return math == 1 ? CUBLAS_COMPUTE_32F_FAST_TF32 : CUBLAS_COMPUTE_32F; }

// C (m x n, ldc) = op(A) op(B), column-major f32.
void gemm(msk_disc_trainer* t, cublasOperation_t ta, cublasOperation_t tb, int m, int n, int k, const float* A,
          long long lda, const float* B, long long ldb, float* C, long long ldc) {
    const float one = 1.0f, zero = 0.0f;
    ckb(cublasGemmEx(t->blas, ta, tb, m, n, k, &one, A, CUDA_R_32F, static_cast<int>(lda), B, CUDA_R_32F,
                     static_cast<int>(ldb), &zero, C, CUDA_R_32F, static_cast<int>(ldc), compute_type(t->math),
                     CUBLAS_GEMM_DEFAULT),
        "cublasGemmEx");
}

// Loss and dloss/dθ (into t->grad) for B rows of Δ at the current parameters.
void loss_and_grad(msk_disc_trainer* t, const float* delta, int B, int ld, cudaStream_t s) {
    // R rows (B Δ rows + the zero row) stored with Rp = R rounded up to 4 rows per
    // half, so every leading dimension and half offset is 16-B aligned (the
    // aligned cuBLAS kernels); padding rows stay zero in every stacked buffer
    const int H = t->H, din = t->din, R = B + 1, Rp = (R + 3) & ~3;
    const long long R2 = 2LL * Rp;
    ckb(cublasSetStream(t->blas, s), "cublasSetStream");
    const float* th = t->theta32;
    const float *W0 = th, *b0 = th + static_cast<long long>(H) * din, *W1 = th + t->o1,
                *b1 = th + t->o1 + static_cast<long long>(H) * H, *W2 = th + t->o2,
                *b2 = th + t->o2 + static_cast<long long>(H) * H, *w4 = th + t->o3, *b3 = th + t->o3 + H;
    float* g = t->grad;
    float *gW0 = g, *gb0 = g + static_cast<long long>(H) * din, *gW1 = g + t->o1,
          *gb1 = g + t->o1 + static_cast<long long>(H) * H, *gW2 = g + t->o2,
          *gb2 = g + t->o2 + static_cast<long long>(H) * H, *gw4 = g + t->o3, *gb3 = g + t->o3 + H;
    const int gR = (Rp + 255) / 256;
    const dim3 eg((Rp + kRowsPerBlock - 1) / kRowsPerBlock, H);
    float *Xb = t->X2 + Rp, *Xt = t->X2;  // primal / tangent halves
    float* Ab[4];
    float* At[4];
    for (int l = 1; l <= 3; ++l) {
        At[l] = t->A[l];
        Ab[l] = t->A[l] + Rp;
    }

    // ---- forward (nn.cpp:54-73) ----
    pack_input_kernel<<<dim3((Rp + 31) / 32, (din + 31) / 32), dim3(32, 8), 0, s>>>(delta, B, ld, din, R, Rp, t->X2);
    gemm(t, CUBLAS_OP_N, CUBLAS_OP_T, Rp, H, din, Xb, R2, W0, H, Ab[1], R2);
    bias_tanh_kernel<<<eg, 256, 0, s>>>(Ab[1], R, Rp, R2, b0);
    gemm(t, CUBLAS_OP_N, CUBLAS_OP_T, Rp, H, H, Ab[1], R2, W1, H, Ab[2], R2);
    bias_tanh_kernel<<<eg, 256, 0, s>>>(Ab[2], R, Rp, R2, b1);
    gemm(t, CUBLAS_OP_N, CUBLAS_OP_T, Rp, H, H, Ab[2], R2, W2, H, Ab[3], R2);
    bias_tanh_kernel<<<eg, 256, 0, s>>>(Ab[3], R, Rp, R2, b2);
    gemm(t, CUBLAS_OP_N, CUBLAS_OP_T, Rp, 1, H, Ab[3], R2, w4, 1, t->z4, Rp);
    head_kernel<<<gR, 256, 0, s>>>(t->z4, b3, B, R, t->d4, t->dd4, t->dz4, t->lrow);

    // ---- input gradient g = dy/dx (nn.cpp:161-164) ----
    d3_kernel<<<eg, 256, 0, s>>>(t->d4, w4, Ab[3], R2, R, Rp, t->T1, Rp);
    gemm(t, CUBLAS_OP_N, CUBLAS_OP_N, Rp, H, H, t->T1, Rp, W2, H, t->T2, Rp);
    gate_kernel<<<eg, 256, 0, s>>>(t->T2, Rp, Ab[2], R2, R, Rp, t->T2, Rp);
    gemm(t, CUBLAS_OP_N, CUBLAS_OP_N, Rp, H, H, t->T2, Rp, W1, H, t->T1, Rp);
    gate_kernel<<<eg, 256, 0, s>>>(t->T1, Rp, Ab[1], R2, R, Rp, t->T1, Rp);
    gemm(t, CUBLAS_OP_N, CUBLAS_OP_N, Rp, din, H, t->T1, Rp, W0, H, Xt, R2);

    // ---- forward tangent along g (nn.cpp:167-171) ----
    gemm(t, CUBLAS_OP_N, CUBLAS_OP_T, Rp, H, din, Xt, R2, W0, H, t->Z[1], Rp);
    gate_kernel<<<eg, 256, 0, s>>>(t->Z[1], Rp, Ab[1], R2, R, Rp, At[1], R2);
    gemm(t, CUBLAS_OP_N, CUBLAS_OP_T, Rp, H, H, At[1], R2, W1, H, t->Z[2], Rp);
    gate_kernel<<<eg, 256, 0, s>>>(t->Z[2], Rp, Ab[2], R2, R, Rp, At[2], R2);
    gemm(t, CUBLAS_OP_N, CUBLAS_OP_T, Rp, H, H, At[2], R2, W2, H, t->Z[3], Rp);
    gate_kernel<<<eg, 256, 0, s>>>(t->Z[3], Rp, Ab[3], R2, R, Rp, At[3], R2);
    gemm(t, CUBLAS_OP_N, CUBLAS_OP_T, Rp, 1, H, At[3], R2, w4, 1, t->zeta4, Rp);
    head2_kernel<<<gR, 256, 0, s>>>(t->d4, t->dd4, t->zeta4, t->dz4, B, R, Rp, static_cast<float>(t->lam / B), t->V,
                                    t->prow);

    // ---- reverse pass over [tangent; primal] (nn.cpp:186-221 + nn.cpp:98-128) ----
    gemm(t, CUBLAS_OP_T, CUBLAS_OP_N, 1, H, static_cast<int>(R2), t->V, R2, t->A[3], R2, gw4, 1);
    colsum_kernel<<<1, 256, 0, s>>>(t->V + Rp, R, 0, gb3);
    rev_elem_kernel<true><<<eg, 256, 0, s>>>(t->S1, t->V, w4, Ab[3], R2, t->Z[3], R, Rp, H);
    // layer 2
    gemm(t, CUBLAS_OP_T, CUBLAS_OP_N, H, H, static_cast<int>(R2), t->S1, R2, t->A[2], R2, gW2, H);
    colsum_kernel<<<H, 256, 0, s>>>(t->S1 + Rp, R, R2, gb2);
    gemm(t, CUBLAS_OP_N, CUBLAS_OP_N, static_cast<int>(R2), H, H, t->S1, R2, W2, H, t->S2, R2);
    rev_elem_kernel<false><<<eg, 256, 0, s>>>(t->S2, nullptr, nullptr, Ab[2], R2, t->Z[2], R, Rp, H);
    // layer 1
    gemm(t, CUBLAS_OP_T, CUBLAS_OP_N, H, H, static_cast<int>(R2), t->S2, R2, t->A[1], R2, gW1, H);
    colsum_kernel<<<H, 256, 0, s>>>(t->S2 + Rp, R, R2, gb1);
    gemm(t, CUBLAS_OP_N, CUBLAS_OP_N, static_cast<int>(R2), H, H, t->S2, R2, W1, H, t->S1, R2);
    rev_elem_kernel<false><<<eg, 256, 0, s>>>(t->S1, nullptr, nullptr, Ab[1], R2, t->Z[1], R, Rp, H);
    // layer 0
    gemm(t, CUBLAS_OP_T, CUBLAS_OP_N, H, din, static_cast<int>(R2), t->S1, R2, t->X2, R2, gW0, H);
    colsum_kernel<<<H, 256, 0, s>>>(t->S1 + Rp, R, R2, gb0);

    loss_kernel<<<1, 1024, 0, s>>>(t->lrow, t->prow, R, t->lam, t->loss);
    ckc(cudaGetLastError(), "disc train kernels");
}

void check_rows(msk_disc_trainer* t, const float* delta, int rows, int ld) {
    if (!delta) throw std::invalid_argument("disc_train: delta is null");
    if (rows < 1 || rows > t->max_rows) throw std::invalid_argument("disc_train: rows must be in [1, max_rows]");
    if (ld < t->din) throw std::invalid_argument("disc_train: ld < input width");
}

}  // namespace

namespace msk_b200 {
const double* disc_trainer_theta(const msk_disc_trainer* t, int* din, int* hidden) {
    *din = t->din;
    *hidden = t->H;
    return t->theta;
}
}  // namespace msk_b200

extern "C" {

int msk_disc_trainer_create(int32_t n_in, int32_t hidden, const double* theta, int64_t n_params, double lr,
                            double grad_penalty, int32_t max_rows, int32_t math, int32_t device,
                            msk_disc_trainer** out) {
    if (!out) return dtfail(nullptr, "msk_disc_trainer_create: out is null");
    *out = nullptr;
    auto t = new msk_disc_trainer();
    try {
        if (n_in < 1 || hidden < 1 || max_rows < 1) throw std::invalid_argument("disc_trainer: bad dimensions");
        if (math < 0 || math > 1) throw std::invalid_argument("disc_trainer: math must be 0 (FP32) or 1 (TF32)");
        if (!theta) throw std::invalid_argument("disc_trainer: theta is null");
        if (!(lr > 0.0) || !(grad_penalty >= 0.0)) throw std::invalid_argument("disc_trainer: need lr > 0, λ >= 0");
        const long long H = hidden, din = n_in;
        const long long P = H * din + H + 2 * (H * H + H) + H + 1;
        if (n_params != P)
            throw std::invalid_argument("disc_trainer: parameter count " + std::to_string(n_params) + " != " +
                                        std::to_string(P) + " for Mlp(in, hidden, 1)");
        ckc(cudaSetDevice(device), "cudaSetDevice");
        int major = 0;
        ckc(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device), "cudaDeviceGetAttribute");
        if (major != 10) throw std::runtime_error("disc_trainer: needs an sm_100 device");
        t->device = device;
        t->din = n_in;
        t->H = hidden;
        t->max_rows = max_rows;
        t->math = math;
        t->P = P;
        t->o1 = H * din + H;
        t->o2 = t->o1 + H * H + H;
        t->o3 = t->o2 + H * H + H;
        t->lr = lr;
        t->lam = grad_penalty;
        t->theta = talloc<double>(t, P);
        t->m = talloc<double>(t, P);
        t->v = talloc<double>(t, P);
        t->theta32 = talloc<float>(t, P);
        t->grad = talloc<float>(t, P);
        t->counts = talloc<long long>(t, 2);
        t->bad = talloc<int>(t, 1);
        ckc(cudaMemcpy(t->theta, theta, P * sizeof(double), cudaMemcpyHostToDevice), "upload theta");
        to_f32_kernel<<<grid_for(P), 256>>>(t->theta, P, t->theta32);
        const size_t R = (static_cast<size_t>(max_rows) + 1 + 3) & ~static_cast<size_t>(3), RH = R * H;  // padded
        t->X2 = talloc<float>(t, 2 * R * din);
        for (int l = 1; l <= 3; ++l) {
            t->A[l] = talloc<float>(t, 2 * RH);
            t->Z[l] = talloc<float>(t, RH);
        }
        t->T1 = talloc<float>(t, RH);
        t->T2 = talloc<float>(t, RH);
        t->S1 = talloc<float>(t, 2 * RH);
        t->S2 = talloc<float>(t, 2 * RH);
        for (float** p : {&t->z4, &t->d4, &t->dd4, &t->dz4, &t->zeta4}) *p = talloc<float>(t, R);
        t->V = talloc<float>(t, 2 * R);
        t->lrow = talloc<double>(t, R);
        t->prow = talloc<double>(t, R);
        t->loss = talloc<double>(t, 3);
        ckb(cublasCreate(&t->blas), "cublasCreate");
        ckc(cudaDeviceSynchronize(), "disc_trainer init");
        *out = t;
        return MSK_OK;
    } catch (const std::invalid_argument& ex) {
        const int code = dtfail(nullptr, ex.what());
        msk_disc_trainer_destroy(t);
        return code;
    } catch (const std::exception& ex) {
        const int code = dtfail(nullptr, ex.what(), MSK_ERR_CUDA);
        msk_disc_trainer_destroy(t);
        return code;
    }
}

void msk_disc_trainer_destroy(msk_disc_trainer* t) {
    if (!t) return;
    cudaSetDevice(t->device);
    cudaDeviceSynchronize();
    if (t->blas) cublasDestroy(t->blas);
    for (void* p : t->allocs) cudaFree(p);
    delete t;
}

const char* msk_disc_trainer_last_error(const msk_disc_trainer* t) { return t ? t->err.c_str() : g_dt_err.c_str(); }

int msk_disc_trainer_gradient(msk_disc_trainer* t, const float* delta, int32_t rows, int32_t ld, float* grad,
                              double* loss, void* stream) {
    if (!t) return dtfail(nullptr, "null disc trainer");
    try {
        check_rows(t, delta, rows, ld);
        cudaSetDevice(t->device);
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        loss_and_grad(t, delta, rows, ld, s);
        if (grad) ckc(cudaMemcpyAsync(grad, t->grad, t->P * 4, cudaMemcpyDeviceToDevice, s), "copy grad");
        if (loss) ckc(cudaMemcpyAsync(loss, t->loss, 24, cudaMemcpyDeviceToDevice, s), "copy loss");
        return MSK_OK;
    } catch (const std::invalid_argument& ex) {
        return dtfail(t, ex.what());
    } catch (const std::exception& ex) {
        return dtfail(t, ex.what(), MSK_ERR_CUDA);
    }
}

int msk_disc_train_step(msk_disc_trainer* t, const float* delta, int32_t rows, int32_t ld, double* loss,
                        void* stream) {
    if (!t) return dtfail(nullptr, "null disc trainer");
    try {
        check_rows(t, delta, rows, ld);
        cudaSetDevice(t->device);
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        loss_and_grad(t, delta, rows, ld, s);
        finite_kernel<<<grid_for(t->P), 256, 0, s>>>(t->grad, t->P, t->bad);
        adam_kernel<<<grid_for(t->P), 256, 0, s>>>(t->grad, t->P, t->bad, t->counts, t->lr, 0.9, 0.999, 1e-8,
                                                   t->theta, t->m, t->v, t->theta32);
        adam_commit_kernel<<<1, 1, 0, s>>>(t->bad, t->counts);
        ckc(cudaGetLastError(), "adam");
        if (loss) ckc(cudaMemcpyAsync(loss, t->loss, 24, cudaMemcpyDeviceToDevice, s), "copy loss");
        return MSK_OK;
    } catch (const std::invalid_argument& ex) {
        return dtfail(t, ex.what());
    } catch (const std::exception& ex) {
        return dtfail(t, ex.what(), MSK_ERR_CUDA);
    }
}

int msk_disc_trainer_get_params(msk_disc_trainer* t, double* theta, int64_t* adam_steps, int64_t* adam_skipped) {
    if (!t) return dtfail(nullptr, "null disc trainer");
    try {
        cudaSetDevice(t->device);
        ckc(cudaDeviceSynchronize(), "disc trainer sync");
        if (theta) ckc(cudaMemcpy(theta, t->theta, t->P * 8, cudaMemcpyDeviceToHost), "download theta");
        long long c[2];
        ckc(cudaMemcpy(c, t->counts, 16, cudaMemcpyDeviceToHost), "download counts");
        if (adam_steps) *adam_steps = c[0];
        if (adam_skipped) *adam_skipped = c[1];
        return MSK_OK;
    } catch (const std::exception& ex) {
        return dtfail(t, ex.what(), MSK_ERR_CUDA);
    }
}

}  // extern "C"
