// On-device policy sampling (SPEC.md:371-393
// sample_action): a⁽⁰⁾ ~ N(mean(s), exp(log_std)) from the Gaussian initial
// sampler π⁽⁰⁾ (an Mlp with an affine head over normalised observations), then
// N_ODE explicit-Euler steps of the flow field ψ(t, s, a) (an Mlp over
// [φ(t), s, a]) write the final action into the step's action buffer:
//     a⁽ᵏ⁺¹⁾ = a⁽ᵏ⁾ + ψ(k·dt, s, a⁽ᵏ⁾)·dt,  k = 0 … N_ODE − 1.
// Every layer is one tcgen05 GEMM (mlp.cu).  ψ's first layer is split by
// input block: the observation part W1_s·s is computed once per control step
// (it does not change along the ODE) and the time part b1 + W1_t·φ(t_k) is a
// per-k bias precomputed on the host.  ψ depends on a only through its
// first-layer pre-activation z_k = W1_a a_k + W1_s s + b1 + W1_t φ(t_k), and
// a_{k+1} − a_k = dt (W4 h3_k + b4), so
//     z_{k+1} = z_k + dt (W1_a W4) h3_k + dt W1_a b4 + W1_t (φ(t_{k+1}) − φ(t_k))
//     a_N     = a_0 + dt W4 (Σ_k h3_k) + N dt b4
// with W1_a W4 (H x H) formed once in f64 on the host.  An ODE step is then
// three H x H layers (z update, layer 2, layer 3 — the z update keeps z in
// f32, layer 3 also accumulates Σ h3 in f32) and the action head runs once
// after the last step: 3 N + 1 GEMMs instead of 4 N.  The whole sample (π⁽⁰⁾,
// noise, the ODE) is captured once into a CUDA graph and replayed.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdlib>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/msk_gpu.h"
#include "mlp.cuh"

namespace msk_b200 {
namespace {

constexpr int kTimeFeatures = 5;  // φ(t) = [t, sin 2πt, cos 2πt, sin 4πt, cos 4πt]

void time_features(double t, double* f) {
    const double w = 2.0 * M_PI * t;
    f[0] = t;
    f[1] = std::sin(w);
    f[2] = std::cos(w);
    f[3] = std::sin(2.0 * w);
    f[4] = std::cos(2.0 * w);
}

// Philox4x32-10 (the excitation generator's round function) -> 4 uniforms in (0, 1]
__device__ __forceinline__ void philox4(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint64_t key,
                                        float (&u)[4]) {
    uint32_t k0 = static_cast<uint32_t>(key), k1 = static_cast<uint32_t>(key >> 32);
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
        const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0;
        c1 = lo1;
        c2 = n2;
        c3 = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    const uint32_t x[4] = {c0, c1, c2, c3};
#pragma unroll
    for (int i = 0; i < 4; ++i) u[i] = static_cast<float>((x[i] >> 8) + 1u) * (1.0f / 16777216.0f);
}

// One warp per row: a⁽⁰⁾ = mean + exp(log_std)·ε (explore) or mean
// (deterministic), Gaussian log-density of a⁽⁰⁾, bf16 tiled copy for ψ.
__global__ void set_step_kernel(uint32_t* d_step, uint32_t step) { *d_step = step; }

__global__ void sample_a0_kernel(int M, int nm, float* a, const float* log_std, int explore, uint64_t seed,
                                 const uint32_t* d_step, long long env_offset, float* a0_out, float* logprob,
                                 void* a_tiled) {
    const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    const uint32_t step = *d_step;  // set per call before a (possibly graph-replayed) sample
    if (row >= pad_to(M, kGemmBM)) return;
    const int kp = pad_to(nm, kGemmBK);
    float lp = 0.0f;
    for (int c = lane; c < kp / 8; c += 32) {  // 8 consecutive actions per lane
        float y[8], z[8];
        if (explore) {
            float u0[4], u1[4];
            const uint32_t env = static_cast<uint32_t>(env_offset + row);
            philox4(step, env, 2u * c, 0x706F6C69u, seed, u0);  // "poli"
            philox4(step, env, 2u * c + 1u, 0x706F6C69u, seed, u1);
            const float u[8] = {u0[0], u0[1], u0[2], u0[3], u1[0], u1[1], u1[2], u1[3]};
#pragma unroll
            for (int i = 0; i < 8; i += 2) {  // Box-Muller
                const float rr = sqrtf(-2.0f * __logf(u[i])), th = 6.283185307179586f * u[i + 1];
                z[i] = rr * __cosf(th);
                z[i + 1] = rr * __sinf(th);
            }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int n = 8 * c + i;
            y[i] = 0.0f;
            if (row < M && n < nm) {
                float* p = a + static_cast<size_t>(row) * nm + n;
                float v = *p;
                if (explore) {
                    const float ls = log_std[n];
                    v = fmaf(__expf(ls), z[i], v);
                    lp += -0.5f * z[i] * z[i] - ls - 0.91893853320467274f;  // log N(a0; mean, sd)
                }
                *p = v;
                if (a0_out) a0_out[static_cast<size_t>(row) * nm + n] = v;
                y[i] = v;
            }
        }
        char* base = static_cast<char*>(a_tiled) +
                     (static_cast<size_t>(row >> 7) * (kp / kGemmBK) + ((8 * c) >> 6)) * (kGemmBM * kGemmBK * 2);
        const int r = row & 127, k = (8 * c) & 63;
        const __nv_bfloat162 h0 = __floats2bfloat162_rn(y[0], y[1]), h1 = __floats2bfloat162_rn(y[2], y[3]);
        const __nv_bfloat162 h2 = __floats2bfloat162_rn(y[4], y[5]), h3 = __floats2bfloat162_rn(y[6], y[7]);
        uint4 pk;
        std::memcpy(&pk.x, &h0, 4);
        std::memcpy(&pk.y, &h1, 4);
        std::memcpy(&pk.z, &h2, 4);
        std::memcpy(&pk.w, &h3, 4);
        *reinterpret_cast<uint4*>(base + ((r >> 3) * 8 + (k >> 3)) * 128 + (r & 7) * 16) = pk;
    }
    for (int o = 16; o > 0; o >>= 1) lp += __shfl_xor_sync(0xffffffffu, lp, o);
    if (lane == 0 && logprob && row < M) logprob[row] = explore ? lp : 0.0f;
}

}  // namespace
}  // namespace msk_b200

using namespace msk_b200;

struct msk_policy {
    int device = 0, obs_dim = 0, nm = 0, hidden = 0, n_ode = 0, max_envs = 0;
    double dt = 0.0;
    float head_scale = 1.0f, head_offset = 0.0f;
    std::vector<void*> allocs;
    std::string err;
    // device weights (tiled bf16) and vectors (f32)
    void *pw1 = nullptr, *pw2 = nullptr, *pw3 = nullptr, *pw4 = nullptr;
    void *qw1s = nullptr, *qw1a = nullptr, *qw2 = nullptr, *qw3 = nullptr, *qw4 = nullptr;
    float *pb1 = nullptr, *pb2 = nullptr, *pb3 = nullptr, *pb4 = nullptr, *log_std = nullptr;
    float *qc = nullptr, *qb2 = nullptr, *qb3 = nullptr, *qb4 = nullptr;  // qc: [n_ode x H] time biases
    void* qm = nullptr;      // W1_a W4 (H x H), tiled bf16
    float* qd = nullptr;     // [n_ode - 1 x H]: dt W1_a b4 + W1_t (φ(t_{k+1}) − φ(t_k))
    float* qhb = nullptr;    // [NM]: N dt b4 / dt = N b4 (the head GEMM scales by dt)
    float *norm_mean = nullptr, *norm_inv_sd = nullptr;
    bool norm = false;
    // scratch
    void *s_t = nullptr, *a_t = nullptr, *h1 = nullptr, *h2 = nullptr;
    float* P = nullptr;
    float *z1 = nullptr, *hsum = nullptr;  // f32 [rows x H]: ψ layer-1 pre-activation, Σ_k h3_k
    uint32_t* d_step = nullptr;  // noise counter of the current call (outside the graph)
    // graph cache (keyed by the call's pointers / sizes)
    cudaGraphExec_t gexec = nullptr;
    cudaGraph_t graph = nullptr;
    struct Key {
        const float* obs;
        float* actions;
        float* a0;
        float* logprob;
        int n, explore;
        uint64_t seed;
        long long off;
    } key{};
    cudaStream_t cap_stream = nullptr;

    template <class T>
    T* dalloc(size_t n) {
        void* p = nullptr;
        if (cudaMalloc(&p, std::max<size_t>(1, n) * sizeof(T)) != cudaSuccess) throw std::runtime_error("cudaMalloc");
        cudaMemset(p, 0, std::max<size_t>(1, n) * sizeof(T));
        allocs.push_back(p);
        return static_cast<T*>(p);
    }
    template <class T>
    T* upload(const std::vector<T>& v) {
        T* p = dalloc<T>(v.size());
        cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
        return p;
    }
};

namespace {

thread_local std::string g_policy_err;

int pfail(msk_policy* p, const std::string& m, int code = MSK_ERR_CONTRACT) {
    g_policy_err = m;
    if (p) p->err = m;
    return code;
}

void ckp(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// Identity normaliser (mean 0, 1/sd 1), written into the same device buffers the
// sample kernels always read.
void set_identity_norm(msk_policy* p) {
    const std::vector<float> zero(p->obs_dim, 0.0f), one(p->obs_dim, 1.0f);
    ckp(cudaMemcpy(p->norm_mean, zero.data(), zero.size() * 4, cudaMemcpyHostToDevice), "norm");
    ckp(cudaMemcpy(p->norm_inv_sd, one.data(), one.size() * 4, cudaMemcpyHostToDevice), "norm");
    p->norm = false;
}


std::vector<float> to_f32(const double* x, size_t n) {
    std::vector<float> v(n);
    for (size_t i = 0; i < n; ++i) v[i] = static_cast<float>(x[i]);
    return v;
}

// Enqueue one sample (all kernels) on stream s.
void enqueue_sample(msk_policy* p, const float* obs, int n, int explore, uint64_t seed, long long env_offset,
                    float* actions, float* a0_out, float* logprob, cudaStream_t s) {
    const int H = p->hidden, D = p->obs_dim, NM = p->nm;
    // always normalise: the identity normaliser is mean 0, 1/sd 1 ((x - 0) * 1 == x bit for bit),
    // so a captured graph stays valid when msk_policy_set_norm changes the statistics
    ckp(launch_obs_to_tiled(obs, n, D, p->norm_mean, p->norm_inv_sd, p->s_t, s), "obs");
    GemmArgs g;
    g.M = n;
    // π⁽⁰⁾ mean: 3 tanh layers + affine head into the action buffer
    g.A = p->s_t; g.W = p->pw1; g.bias = p->pb1; g.N = H; g.K = D; g.out_a = p->h1;
    ckp(launch_gemm(g, kEpiTanhTiled, s), "pi1");
    g.A = p->h1; g.W = p->pw2; g.bias = p->pb2; g.K = H; g.out_a = p->h2;
    ckp(launch_gemm(g, kEpiTanhTiled, s), "pi2");
    g.A = p->h2; g.W = p->pw3; g.bias = p->pb3; g.out_a = p->h1;
    ckp(launch_gemm(g, kEpiTanhTiled, s), "pi3");
    GemmArgs hd = g;
    hd.A = p->h1; hd.W = p->pw4; hd.bias = p->pb4; hd.N = NM; hd.K = H; hd.out_a = nullptr;
    hd.out_f = actions; hd.ld_f = NM; hd.n_valid = NM; hd.scale = p->head_scale; hd.offset = p->head_offset;
    ckp(launch_gemm(hd, kEpiF32, s), "pi4");
    sample_a0_kernel<<<(pad_to(n, kGemmBM) + 7) / 8, 256, 0, s>>>(n, NM, actions, p->log_std, explore, seed,
                                                                  p->d_step, env_offset, a0_out, logprob, p->a_t);
    ckp(cudaGetLastError(), "a0");
    // ψ: P = W1_s · s once, then N_ODE Euler steps in the z-recurrence form
    // internal f32 buffers (P, z1, hsum) in the F4 layout (coalesced row-per-thread epilogues)
    const int f4 = (H % 4 == 0) ? pad_to(n, kGemmBM) : 0;
    GemmArgs pg;
    pg.M = n; pg.A = p->s_t; pg.W = p->qw1s; pg.N = H; pg.K = D; pg.out_f = p->P; pg.ld_f = H; pg.n_valid = H;
    pg.f4_rows = f4;
    ckp(launch_gemm(pg, kEpiF32, s), "psiP");
    if (p->n_ode == 0) return;
    GemmArgs z;  // z_0 = W1_a a_0 + P + b1 + W1_t φ(0)
    z.M = n; z.A = p->a_t; z.W = p->qw1a; z.bias = p->qc; z.addend = p->P; z.ld_add = H; z.N = H; z.K = NM;
    z.out_a = p->h1; z.out_f = p->z1; z.ld_f = H; z.f4_rows = f4;
    ckp(launch_gemm(z, kEpiTanhPre, s), "psi1");
    ckp(cudaMemsetAsync(p->hsum, 0, sizeof(float) * static_cast<size_t>(pad_to(n, kGemmBM)) * H, s), "hsum");
    void *x = p->h1, *y = p->h2;  // x: tanh(z_k)
    // MSK_POLICY_ODE=1: the 3 N_ODE - 1 hidden layers in one persistent launch (mlp.cu ode_kernel;
    // opt-in, slower at W = 1024); default: one pipelined GEMM launch per layer
    static const bool persistent = std::getenv("MSK_POLICY_ODE") != nullptr;
    if (persistent && pad_to(H, kGemmBN) / kGemmBN <= 8) {
        GemmArgs g2, g3, g1;
        g2.M = g3.M = g1.M = n;
        g2.N = g3.N = g1.N = H;
        g2.K = g3.K = g1.K = H;
        g2.W = p->qw2; g2.bias = p->qb2;
        g3.W = p->qw3; g3.bias = p->qb3; g3.out_f = p->hsum; g3.ld_f = H; g3.f4_rows = f4;
        g1.W = p->qm; g1.addend = p->z1; g1.ld_add = H; g1.out_f = p->z1; g1.ld_f = H; g1.f4_rows = f4;
        g1.scale = static_cast<float>(p->dt);
        ckp(launch_ode(g2, g3, g1, x, y, p->qd, p->n_ode, H, s), "ode");
        x = p->h1;
        y = p->h2;
    } else {
    for (int k = 0; k < p->n_ode; ++k) {
        GemmArgs q;
        q.M = n; q.N = H; q.K = H;
        q.A = x; q.W = p->qw2; q.bias = p->qb2; q.out_a = y;
        ckp(launch_gemm(q, kEpiTanhTiled, s), "psi2");
        q.A = y; q.W = p->qw3; q.bias = p->qb3; q.out_a = x; q.out_f = p->hsum; q.ld_f = H; q.f4_rows = f4;
        ckp(launch_gemm(q, kEpiTanhAcc, s), "psi3");
        if (k + 1 < p->n_ode) {  // z_{k+1} = z_k + dt (W1_a W4) h3_k + qd_k
            GemmArgs u;
            u.M = n; u.N = H; u.K = H; u.A = x; u.W = p->qm; u.bias = p->qd + static_cast<size_t>(k) * H;
            u.addend = p->z1; u.ld_add = H; u.out_f = p->z1; u.ld_f = H; u.out_a = y;
            u.scale = static_cast<float>(p->dt);
            u.f4_rows = f4;
            ckp(launch_gemm(u, kEpiTanhPre, s), "psi1");
            std::swap(x, y);
        }
    }
    }
    // a_N = a_0 + dt (W4 Σ_k h3_k + N b4), in place on the action buffer
    ckp(launch_f32_to_tiled(p->hsum, n, H, H, y, s, f4), "hsum tiles");
    GemmArgs fh;
    fh.M = n; fh.A = y; fh.W = p->qw4; fh.bias = p->qhb; fh.N = NM; fh.K = H; fh.out_f = actions; fh.ld_f = NM;
    fh.n_valid = NM; fh.scale = static_cast<float>(p->dt); fh.addend = actions; fh.ld_add = NM;
    ckp(launch_gemm(fh, kEpiF32, s), "psi4");
}

}  // namespace

extern "C" {

int msk_policy_create(int32_t obs_dim, int32_t n_actions, int32_t hidden, const double* pi_theta,
                      int64_t pi_n_params, double head_scale, double head_offset, const double* log_std,
                      const double* psi_theta, int64_t psi_n_params, int32_t n_ode, double dt_ode, int32_t max_envs,
                      int32_t device, msk_policy** out) {
    if (!out) return pfail(nullptr, "msk_policy_create: out is null");
    *out = nullptr;
    auto p = new msk_policy();
    try {
        if (obs_dim < 1 || n_actions < 1 || max_envs < 1 || n_ode < 0)
            throw std::invalid_argument("msk_policy_create: bad dimensions");
        if (hidden < 64 || hidden % 64 != 0) throw std::invalid_argument("policy hidden width must be a multiple of 64");
        if (!pi_theta || !psi_theta || !log_std) throw std::invalid_argument("msk_policy_create: null parameters");
        const int H = hidden, D = obs_dim, NM = n_actions, IN = kTimeFeatures + D + NM;
        auto count = [](int in, int h, int o) { return static_cast<int64_t>(h) * in + h + 2LL * (h * h + h) + static_cast<int64_t>(o) * h + o; };
        if (pi_n_params != count(D, H, NM))
            throw std::invalid_argument("policy pi parameter count " + std::to_string(pi_n_params) + " != Mlp(" +
                                        std::to_string(D) + ", " + std::to_string(H) + ", " + std::to_string(NM) + ")");
        if (psi_n_params != count(IN, H, NM))
            throw std::invalid_argument("policy psi parameter count " + std::to_string(psi_n_params) + " != Mlp(" +
                                        std::to_string(IN) + ", " + std::to_string(H) + ", " + std::to_string(NM) + ")");
        ckp(cudaSetDevice(device), "cudaSetDevice");
        p->device = device; p->obs_dim = D; p->nm = NM; p->hidden = H; p->n_ode = n_ode; p->dt = dt_ode;
        p->max_envs = max_envs;
        p->head_scale = static_cast<float>(head_scale);
        p->head_offset = static_cast<float>(head_offset);
        // π⁽⁰⁾: W1 b1 W2 b2 W3 b3 W4 b4 (nn.cpp:16-38 layout, W column-major)
        const double* t = pi_theta;
        p->pw1 = p->upload(pack_weights(t, H, D, 0, D)); t += static_cast<size_t>(H) * D;
        p->pb1 = p->upload(to_f32(t, H)); t += H;
        p->pw2 = p->upload(pack_weights(t, H, H, 0, H)); t += static_cast<size_t>(H) * H;
        p->pb2 = p->upload(to_f32(t, H)); t += H;
        p->pw3 = p->upload(pack_weights(t, H, H, 0, H)); t += static_cast<size_t>(H) * H;
        p->pb3 = p->upload(to_f32(t, H)); t += H;
        p->pw4 = p->upload(pack_weights(t, NM, H, 0, H)); t += static_cast<size_t>(NM) * H;
        p->pb4 = p->upload(to_f32(t, NM));
        p->log_std = p->upload(to_f32(log_std, NM));
        // ψ: input columns [φ(t) (5) | s (D) | a (NM)]
        t = psi_theta;
        const double* W1 = t;
        p->qw1s = p->upload(pack_weights(W1, H, IN, kTimeFeatures, D));
        p->qw1a = p->upload(pack_weights(W1, H, IN, kTimeFeatures + D, NM));
        t += static_cast<size_t>(H) * IN;
        const double* b1 = t;
        t += H;
        std::vector<float> qc(static_cast<size_t>(std::max(1, n_ode)) * H);
        for (int k = 0; k < n_ode; ++k) {  // b1 + W1_t φ(k dt) in f64
            double f[kTimeFeatures];
            time_features(k * dt_ode, f);
            for (int i = 0; i < H; ++i) {
                double z = b1[i];
                for (int j = 0; j < kTimeFeatures; ++j) z += W1[static_cast<size_t>(j) * H + i] * f[j];
                qc[static_cast<size_t>(k) * H + i] = static_cast<float>(z);
            }
        }
        p->qc = p->upload(qc);
        p->qw2 = p->upload(pack_weights(t, H, H, 0, H)); t += static_cast<size_t>(H) * H;
        p->qb2 = p->upload(to_f32(t, H)); t += H;
        p->qw3 = p->upload(pack_weights(t, H, H, 0, H)); t += static_cast<size_t>(H) * H;
        p->qb3 = p->upload(to_f32(t, H)); t += H;
        const double* W4 = t;  // NM x H, column-major
        p->qw4 = p->upload(pack_weights(t, NM, H, 0, H)); t += static_cast<size_t>(NM) * H;
        const double* b4 = t;
        p->qb4 = p->upload(to_f32(t, NM));
        {  // z-recurrence constants (see the header): W1_a W4, W1_a b4, time-bias differences
            const double* W1a = W1 + static_cast<size_t>(kTimeFeatures + D) * H;  // column a of W1_a at W1a + a H
            std::vector<double> Mq(static_cast<size_t>(H) * H, 0.0), v(H, 0.0);
            for (int kk = 0; kk < H; ++kk)
                for (int a = 0; a < NM; ++a) {
                    const double w4 = W4[static_cast<size_t>(kk) * NM + a];
                    const double* col = W1a + static_cast<size_t>(a) * H;
                    double* out = Mq.data() + static_cast<size_t>(kk) * H;
                    for (int i = 0; i < H; ++i) out[i] += col[i] * w4;
                }
            for (int a = 0; a < NM; ++a)
                for (int i = 0; i < H; ++i) v[i] += W1a[static_cast<size_t>(a) * H + i] * b4[a];
            p->qm = p->upload(pack_weights(Mq.data(), H, H, 0, H));
            std::vector<float> qd(static_cast<size_t>(std::max(1, n_ode - 1)) * H);
            for (int k = 0; k + 1 < n_ode; ++k)
                for (int i = 0; i < H; ++i) {
                    double dtime = 0.0;  // W1_t (φ(t_{k+1}) − φ(t_k))
                    double f0[kTimeFeatures], f1[kTimeFeatures];
                    time_features(k * dt_ode, f0);
                    time_features((k + 1) * dt_ode, f1);
                    for (int j = 0; j < kTimeFeatures; ++j) dtime += W1[static_cast<size_t>(j) * H + i] * (f1[j] - f0[j]);
                    qd[static_cast<size_t>(k) * H + i] = static_cast<float>(dt_ode * v[i] + dtime);
                }
            p->qd = p->upload(qd);
            std::vector<float> hb(NM);
            for (int a = 0; a < NM; ++a) hb[a] = static_cast<float>(n_ode * b4[a]);
            p->qhb = p->upload(hb);
        }
        // scratch
        p->s_t = p->dalloc<char>(tiled_a_bytes(max_envs, D));
        p->a_t = p->dalloc<char>(tiled_a_bytes(max_envs, NM));
        p->h1 = p->dalloc<char>(tiled_a_bytes(max_envs, H));
        p->h2 = p->dalloc<char>(tiled_a_bytes(max_envs, H));
        p->P = p->dalloc<float>(static_cast<size_t>(pad_to(max_envs, kGemmBM)) * H);
        p->z1 = p->dalloc<float>(static_cast<size_t>(pad_to(max_envs, kGemmBM)) * H);
        p->hsum = p->dalloc<float>(static_cast<size_t>(pad_to(max_envs, kGemmBM)) * H);
        p->norm_mean = p->dalloc<float>(D);
        p->norm_inv_sd = p->dalloc<float>(D);
        p->d_step = p->dalloc<uint32_t>(1);
        set_identity_norm(p);
        ckp(prepare_gemm(), "cudaFuncSetAttribute(gemm)");
        ckp(cudaStreamCreateWithFlags(&p->cap_stream, cudaStreamNonBlocking), "stream");
        *out = p;
        return MSK_OK;
    } catch (const std::exception& ex) {
        const int code = pfail(nullptr, ex.what());
        msk_policy_destroy(p);
        return code;
    }
}

void msk_policy_destroy(msk_policy* p) {
    if (!p) return;
    cudaSetDevice(p->device);
    cudaDeviceSynchronize();
    if (p->gexec) cudaGraphExecDestroy(p->gexec);
    if (p->graph) cudaGraphDestroy(p->graph);
    if (p->cap_stream) cudaStreamDestroy(p->cap_stream);
    for (void* a : p->allocs) cudaFree(a);
    delete p;
}

const char* msk_policy_last_error(const msk_policy* p) { return p ? p->err.c_str() : g_policy_err.c_str(); }

int msk_policy_set_norm(msk_policy* p, const double* mean, const double* var, double count) {
    if (!p) return pfail(nullptr, "null policy");
    try {
        ckp(cudaSetDevice(p->device), "cudaSetDevice");
        if (count == 0.0 || !mean || !var) {  // RunningNorm::apply with count 0 is the identity (nn.cpp:273)
            set_identity_norm(p);
            return MSK_OK;
        }
        std::vector<float> m(p->obs_dim), is(p->obs_dim);
        for (int i = 0; i < p->obs_dim; ++i) {
            m[i] = static_cast<float>(mean[i]);
            is[i] = static_cast<float>(1.0 / std::max(std::sqrt(var[i] + 1e-8), 1e-6));  // nn.cpp:274
        }
        ckp(cudaMemcpy(p->norm_mean, m.data(), m.size() * 4, cudaMemcpyHostToDevice), "norm");
        ckp(cudaMemcpy(p->norm_inv_sd, is.data(), is.size() * 4, cudaMemcpyHostToDevice), "norm");
        p->norm = true;
        return MSK_OK;
    } catch (const std::exception& ex) {
        return pfail(p, ex.what(), MSK_ERR_CUDA);
    }
}

int msk_policy_sample(msk_policy* p, const float* obs, int32_t n, int32_t explore, uint64_t seed, uint32_t step,
                      int64_t global_env_offset, float* actions, float* a0, float* logprob, void* stream) {
    if (!p) return pfail(nullptr, "null policy");
    try {
        if (!obs || !actions || n < 1 || n > p->max_envs) throw std::invalid_argument("policy_sample: bad arguments");
        ckp(cudaSetDevice(p->device), "cudaSetDevice");
        set_step_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(p->d_step, step);
        enqueue_sample(p, obs, n, explore, seed, global_env_offset, actions, a0, logprob,
                       static_cast<cudaStream_t>(stream));
        return MSK_OK;
    } catch (const std::invalid_argument& ex) {
        return pfail(p, ex.what());
    } catch (const std::exception& ex) {
        return pfail(p, ex.what(), MSK_ERR_CUDA);
    }
}

// Same sample replayed from a CUDA graph (captured on first use and whenever
// the pointers / sizes / seed change; the per-call noise counter lives in
// device memory, so a new step just relaunches the graph — one launch instead
// of ~4 N_ODE + 6).
int msk_policy_sample_graph(msk_policy* p, const float* obs, int32_t n, int32_t explore, uint64_t seed,
                            uint32_t step, int64_t global_env_offset, float* actions, float* a0, float* logprob,
                            void* stream) {
    if (!p) return pfail(nullptr, "null policy");
    try {
        if (!obs || !actions || n < 1 || n > p->max_envs) throw std::invalid_argument("policy_sample: bad arguments");
        ckp(cudaSetDevice(p->device), "cudaSetDevice");
        const msk_policy::Key k{obs, actions, a0, logprob, n, explore, seed, global_env_offset};
        if (!p->gexec || std::memcmp(&k, &p->key, sizeof k) != 0) {
            cudaGraph_t g = nullptr;
            ckp(cudaStreamBeginCapture(p->cap_stream, cudaStreamCaptureModeThreadLocal), "capture");
            enqueue_sample(p, obs, n, explore, seed, global_env_offset, actions, a0, logprob, p->cap_stream);
            ckp(cudaStreamEndCapture(p->cap_stream, &g), "end capture");
            if (p->gexec) {
                cudaGraphExecUpdateResultInfo info;
                if (cudaGraphExecUpdate(p->gexec, g, &info) != cudaSuccess) {
                    cudaGetLastError();
                    cudaGraphExecDestroy(p->gexec);
                    p->gexec = nullptr;
                }
            }
            if (!p->gexec) ckp(cudaGraphInstantiate(&p->gexec, g, 0), "instantiate");
            if (p->graph) cudaGraphDestroy(p->graph);
            p->graph = g;
            p->key = k;
        }
        set_step_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(p->d_step, step);
        ckp(cudaGraphLaunch(p->gexec, static_cast<cudaStream_t>(stream)), "graph launch");
        return MSK_OK;
    } catch (const std::invalid_argument& ex) {
        return pfail(p, ex.what());
    } catch (const std::exception& ex) {
        return pfail(p, ex.what(), MSK_ERR_CUDA);
    }
}

int32_t msk_policy_time_features(double t, double* out5) {
    if (!out5) return 0;
    time_features(t, out5);
    return kTimeFeatures;
}

// Test hook: one tiled GEMM Y = act(X W^T + b) from f32 row-major X [M x K] and
// a column-major f64 W [N x K] (Mlp layout); epi 0 = tanh (bf16 tiled, read
// back to f32 Y), 1 = linear f32.
int msk_gemm_test(const float* X, int32_t M, int32_t K, const double* W_host, const float* b_host, int32_t N,
                  int32_t epi, float* Y) {
    try {
        ckp(prepare_gemm(), "prepare");
        std::vector<uint16_t> wi = pack_weights(W_host, N, K, 0, K);
        void *dW, *dX, *dO;
        float *db = nullptr, *dY;
        ckp(cudaMalloc(&dW, wi.size() * 2), "m");
        ckp(cudaMemcpy(dW, wi.data(), wi.size() * 2, cudaMemcpyHostToDevice), "c");
        ckp(cudaMalloc(&dX, tiled_a_bytes(M, K)), "m");
        ckp(cudaMemset(dX, 0, tiled_a_bytes(M, K)), "z");
        ckp(cudaMalloc(&dO, tiled_a_bytes(M, N)), "m");
        ckp(cudaMemset(dO, 0, tiled_a_bytes(M, N)), "z");
        ckp(cudaMalloc(&dY, static_cast<size_t>(M) * N * 4), "m");
        if (b_host) {
            ckp(cudaMalloc(&db, static_cast<size_t>(N) * 4), "m");
            ckp(cudaMemcpy(db, b_host, static_cast<size_t>(N) * 4, cudaMemcpyHostToDevice), "c");
        }
        float* dXf;
        ckp(cudaMalloc(&dXf, static_cast<size_t>(M) * K * 4), "m");
        ckp(cudaMemcpy(dXf, X, static_cast<size_t>(M) * K * 4, cudaMemcpyHostToDevice), "c");
        ckp(launch_f32_to_tiled(dXf, M, K, K, dX, nullptr), "tile");
        GemmArgs g;
        g.A = dX; g.W = dW; g.bias = db; g.M = M; g.N = N; g.K = K;
        if (epi == 0) {
            g.out_a = dO;
            ckp(launch_gemm(g, kEpiTanhTiled, nullptr), "gemm");
            // unpack the tiled bf16 output to f32 row-major on the host
            std::vector<uint16_t> o(tiled_a_bytes(M, N) / 2);
            ckp(cudaMemcpy(o.data(), dO, o.size() * 2, cudaMemcpyDeviceToHost), "c");
            const int KB = pad_to(N, kGemmBK) / kGemmBK;
            for (int m = 0; m < M; ++m)
                for (int n = 0; n < N; ++n) {
                    const size_t blk = static_cast<size_t>(m / kGemmBM) * KB + n / kGemmBK;
                    const uint32_t u = static_cast<uint32_t>(o[(blk * kGemmBM * kGemmBK * 2 +
                                                               (((m % 128) >> 3) * 8 + ((n % 64) >> 3)) * 128 +
                                                               (m & 7) * 16 + (n & 7) * 2) / 2])
                                       << 16;
                    float f;
                    std::memcpy(&f, &u, 4);
                    Y[static_cast<size_t>(m) * N + n] = f;
                }
        } else {
            g.out_f = dY; g.ld_f = N; g.n_valid = N;
            ckp(launch_gemm(g, kEpiF32, nullptr), "gemm");
            ckp(cudaMemcpy(Y, dY, static_cast<size_t>(M) * N * 4, cudaMemcpyDeviceToHost), "c");
        }
        ckp(cudaDeviceSynchronize(), "sync");
        cudaFree(dW); cudaFree(dX); cudaFree(dO); cudaFree(dY); cudaFree(dXf);
        if (db) cudaFree(db);
        return MSK_OK;
    } catch (const std::exception& ex) {
        return pfail(nullptr, ex.what(), MSK_ERR_CUDA);
    }
}

// Diagnostic: average time of `reps` back-to-back tanh GEMM layers [M x K] x [K x N]^T
// on device buffers (programmatic dependent launches, as in the policy sample).
int msk_gemm_bench(int32_t M, int32_t K, int32_t N, int32_t reps, double* ms_per_gemm) {
    try {
        ckp(prepare_gemm(), "prepare");
        void *dW, *dX, *dO;
        ckp(cudaMalloc(&dW, tiled_w_bytes(N, K)), "m");
        ckp(cudaMemset(dW, 0, tiled_w_bytes(N, K)), "z");
        ckp(cudaMalloc(&dX, tiled_a_bytes(M, K)), "m");
        ckp(cudaMemset(dX, 0, tiled_a_bytes(M, K)), "z");
        ckp(cudaMalloc(&dO, tiled_a_bytes(M, N)), "m");
        GemmArgs g;
        g.A = dX; g.W = dW; g.M = M; g.N = N; g.K = K; g.out_a = dO;
        cudaStream_t s;
        ckp(cudaStreamCreate(&s), "stream");
        for (int i = 0; i < 3; ++i) ckp(launch_gemm(g, kEpiTanhTiled, s), "gemm");
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0, s);
        for (int i = 0; i < reps; ++i) ckp(launch_gemm(g, kEpiTanhTiled, s), "gemm");
        cudaEventRecord(e1, s);
        ckp(cudaEventSynchronize(e1), "sync");
        float ms = 0.0f;
        cudaEventElapsedTime(&ms, e0, e1);
        *ms_per_gemm = ms / reps;
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        cudaStreamDestroy(s);
        cudaFree(dW); cudaFree(dX); cudaFree(dO);
        return MSK_OK;
    } catch (const std::exception& ex) {
        return pfail(nullptr, ex.what(), MSK_ERR_CUDA);
    }
}

}  // extern "C"
