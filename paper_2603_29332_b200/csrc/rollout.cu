// On-device rollout buffer + GAE.
//
// The buffer holds h control steps of E envs in step-major rows ([t][env][...])
// so every per-step record and the GAE recursion read/write coalesced rows:
// observation, base action a⁽⁰⁾, final action a, log-prob of a⁽⁰⁾, reward, done,
// value estimate, tracking error Δ (the RolloutBuffer fields of SPEC.md:379).
// compute_gae: δ_t = r_t + γ V_{t+1} (1 − done_t) − V_t,
// A_t = δ_t + γ λ (1 − done_t) A_{t+1} (V_h = bootstrap), returns = A + V, then
// advantages normalised to zero mean / unit variance over the whole batch
// (deterministic single-block f64 reduction).
#include <cuda_runtime.h>

#include <algorithm>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/msk_gpu.h"

namespace {

__global__ void gae_kernel(int E, int h, const float* reward, const uint8_t* done, const float* value,
                           const float* bootstrap, float gamma, float lam, float* adv, float* ret) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= E) return;
    float next_v = bootstrap[e], next_a = 0.0f;
    for (int t = h - 1; t >= 0; --t) {
        const size_t i = static_cast<size_t>(t) * E + e;
        const float nd = (done[i] & 1) ? 0.0f : 1.0f;  // MSK_FLAG_DONE bit
        const float v = value[i];
        const float delta = reward[i] + gamma * next_v * nd - v;
        next_a = delta + gamma * lam * nd * next_a;
        adv[i] = next_a;
        ret[i] = next_a + v;
        next_v = v;
    }
}

// One block: mean and std of n advantages (f64, fixed order), then normalise.
__global__ void __launch_bounds__(1024) normalize_kernel(long long n, float* adv) {
    __shared__ double red[2][32];
    double s = 0.0, q = 0.0;
    for (long long i = threadIdx.x; i < n; i += blockDim.x) {
        const double v = adv[i];
        s += v;
        q += v * v;
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int o = 16; o > 0; o >>= 1) {
        s += __shfl_xor_sync(0xffffffffu, s, o);
        q += __shfl_xor_sync(0xffffffffu, q, o);
    }
    if (lane == 0) {
        red[0][warp] = s;
        red[1][warp] = q;
    }
    __syncthreads();
    if (warp == 0) {
        s = lane < (blockDim.x >> 5) ? red[0][lane] : 0.0;
        q = lane < (blockDim.x >> 5) ? red[1][lane] : 0.0;
        for (int o = 16; o > 0; o >>= 1) {
            s += __shfl_xor_sync(0xffffffffu, s, o);
            q += __shfl_xor_sync(0xffffffffu, q, o);
        }
        if (lane == 0) {
            const double mean = s / static_cast<double>(n);
            const double var = fmax(q / static_cast<double>(n) - mean * mean, 0.0);
            red[0][0] = mean;
            red[1][0] = 1.0 / (sqrt(var) + 1e-8);
        }
    }
    __syncthreads();
    const double mean = red[0][0], inv = red[1][0];
    for (long long i = threadIdx.x; i < n; i += blockDim.x) adv[i] = static_cast<float>((adv[i] - mean) * inv);
}

// ---- PPO minibatching (epochs over shuffled minibatches) ----
// The epoch's shuffle is a keyed bijection of [0, n): a 4-round Feistel
// network on the smallest even-bit-width domain >= n, cycle-walked into
// [0, n) (format-preserving, no sort, O(1) per record, deterministic in
// (seed, epoch)).
__device__ __forceinline__ uint32_t mix32(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352du;
    x ^= x >> 15;
    x *= 0x846ca68bu;
    x ^= x >> 16;
    return x;
}

__host__ __device__ inline int feistel_half_bits(long long n) {
    int bits = 2;
    while ((1ll << bits) < n) bits += 2;
    return bits / 2;
}

__device__ __forceinline__ uint32_t feistel_perm(uint32_t x, long long n, int hb, uint64_t key) {
    const uint32_t mask = (1u << hb) - 1u;
    do {
        uint32_t l = x >> hb, r = x & mask;
#pragma unroll
        for (int round = 0; round < 4; ++round) {
            const uint32_t k = static_cast<uint32_t>(key >> (16 * round)) ^ (0x9E3779B9u * (round + 1));
            const uint32_t t = l ^ (mix32(r ^ k) & mask);
            l = r;
            r = t;
        }
        x = (l << hb) | r;
    } while (x >= static_cast<uint32_t>(n));
    return x;
}

struct MbOut {
    float *obs, *a0, *act, *logp, *adv, *ret, *value;
    int* ids;
};

// One warp per minibatch row: record id, then the row copies (16-B vectors
// when the row width allows).
__global__ void minibatch_kernel(long long n, int hb, uint64_t key, long long first, int rows, int obs_dim,
                                 int act_dim, const float* obs, const float* a0, const float* act,
                                 const float* logp, const float* adv, const float* ret, const float* value,
                                 MbOut o) {
    const int j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (j >= rows) return;
    const uint32_t i = feistel_perm(static_cast<uint32_t>(first + j), n, hb, key);
    auto copy_row = [&](float* dst, const float* src, int dim) {
        if (!dst || dim == 0) return;
        const float* sp = src + static_cast<size_t>(i) * dim;
        float* dp = dst + static_cast<size_t>(j) * dim;
        // 16-B vectors only when both rows are 16-B aligned (a C-ABI caller may pass
        // an offset / sub-buffer pointer)
        if ((dim & 3) == 0 && ((reinterpret_cast<uintptr_t>(sp) | reinterpret_cast<uintptr_t>(dp)) & 15) == 0) {
            for (int c = lane; c < dim / 4; c += 32)
                reinterpret_cast<float4*>(dp)[c] = reinterpret_cast<const float4*>(sp)[c];
        } else {
            for (int c = lane; c < dim; c += 32) dp[c] = sp[c];
        }
    };
    copy_row(o.obs, obs, obs_dim);
    copy_row(o.a0, a0, act_dim);
    copy_row(o.act, act, act_dim);
    if (lane == 0) {
        if (o.logp) o.logp[j] = logp[i];
        if (o.adv) o.adv[j] = adv[i];
        if (o.ret) o.ret[j] = ret[i];
        if (o.value) o.value[j] = value[i];
        if (o.ids) o.ids[j] = static_cast<int>(i);
    }
}

}  // namespace

struct msk_rollout {
    int device = 0, E = 0, h = 0, obs_dim = 0, act_dim = 0, delta_dim = 0;
    float *obs = nullptr, *a0 = nullptr, *act = nullptr, *logp = nullptr, *reward = nullptr, *value = nullptr,
          *delta = nullptr, *adv = nullptr, *ret = nullptr;
    uint8_t* done = nullptr;
    std::vector<void*> allocs;
    std::string err;
};

namespace {
thread_local std::string g_rollout_err;

int rfail(msk_rollout* r, const std::string& m, int code = MSK_ERR_CONTRACT) {
    g_rollout_err = m;
    if (r) r->err = m;
    return code;
}

template <class T>
T* ralloc(msk_rollout* r, size_t n) {
    void* p = nullptr;
    if (cudaMalloc(&p, std::max<size_t>(1, n) * sizeof(T)) != cudaSuccess) throw std::runtime_error("cudaMalloc");
    cudaMemset(p, 0, std::max<size_t>(1, n) * sizeof(T));
    r->allocs.push_back(p);
    return static_cast<T*>(p);
}

void copy_rows(void* dst, const void* src, size_t bytes, cudaStream_t s) {
    if (src && dst) {
        const cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, s);
        if (e != cudaSuccess) throw std::runtime_error(cudaGetErrorString(e));
    }
}
}  // namespace

extern "C" {

int msk_rollout_create(int32_t n_envs, int32_t horizon, int32_t obs_dim, int32_t act_dim, int32_t delta_dim,
                       int32_t device, msk_rollout** out) {
    if (!out) return rfail(nullptr, "msk_rollout_create: out is null");
    *out = nullptr;
    auto r = new msk_rollout();
    try {
        if (n_envs < 1 || horizon < 1 || obs_dim < 0 || act_dim < 0 || delta_dim < 0)
            throw std::invalid_argument("msk_rollout_create: bad dimensions");
        if (cudaSetDevice(device) != cudaSuccess) throw std::runtime_error("cudaSetDevice");
        r->device = device;
        r->E = n_envs;
        r->h = horizon;
        r->obs_dim = obs_dim;
        r->act_dim = act_dim;
        r->delta_dim = delta_dim;
        const size_t n = static_cast<size_t>(n_envs) * horizon;
        r->obs = ralloc<float>(r, n * obs_dim);
        r->a0 = ralloc<float>(r, n * act_dim);
        r->act = ralloc<float>(r, n * act_dim);
        r->logp = ralloc<float>(r, n);
        r->reward = ralloc<float>(r, n);
        r->value = ralloc<float>(r, n);
        r->delta = ralloc<float>(r, n * delta_dim);
        r->adv = ralloc<float>(r, n);
        r->ret = ralloc<float>(r, n);
        r->done = ralloc<uint8_t>(r, n);
        *out = r;
        return MSK_OK;
    } catch (const std::exception& ex) {
        const int code = rfail(nullptr, ex.what(), MSK_ERR_CUDA);
        msk_rollout_destroy(r);
        return code;
    }
}

void msk_rollout_destroy(msk_rollout* r) {
    if (!r) return;
    cudaSetDevice(r->device);
    cudaDeviceSynchronize();
    for (void* p : r->allocs) cudaFree(p);
    delete r;
}

const char* msk_rollout_last_error(const msk_rollout* r) { return r ? r->err.c_str() : g_rollout_err.c_str(); }

int msk_rollout_record(msk_rollout* r, int32_t t, const float* obs, const float* a0, const float* actions,
                       const float* logprob, const float* reward, const uint8_t* flags, const float* value,
                       const float* delta, void* stream) {
    if (!r) return rfail(nullptr, "null rollout");
    try {
        if (t < 0 || t >= r->h) throw std::invalid_argument("rollout_record: step out of range");
        cudaSetDevice(r->device);
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        const size_t E = r->E, row = static_cast<size_t>(t) * E;
        copy_rows(r->obs + row * r->obs_dim, obs, E * r->obs_dim * 4, s);
        copy_rows(r->a0 + row * r->act_dim, a0, E * r->act_dim * 4, s);
        copy_rows(r->act + row * r->act_dim, actions, E * r->act_dim * 4, s);
        copy_rows(r->logp + row, logprob, E * 4, s);
        copy_rows(r->reward + row, reward, E * 4, s);
        copy_rows(r->done + row, flags, E, s);  // any nonzero MSK_FLAG_DONE bit reads as done
        copy_rows(r->value + row, value, E * 4, s);
        copy_rows(r->delta + row * r->delta_dim, delta, E * r->delta_dim * 4, s);
        return MSK_OK;
    } catch (const std::invalid_argument& ex) {
        return rfail(r, ex.what());
    } catch (const std::exception& ex) {
        return rfail(r, ex.what(), MSK_ERR_CUDA);
    }
}

int msk_rollout_gae(msk_rollout* r, const float* bootstrap_value, float gamma, float lam, int32_t normalize,
                    float* advantages, float* returns, void* stream) {
    if (!r) return rfail(nullptr, "null rollout");
    try {
        if (!bootstrap_value) throw std::invalid_argument("rollout_gae: bootstrap values required");
        cudaSetDevice(r->device);
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        gae_kernel<<<(r->E + 255) / 256, 256, 0, s>>>(r->E, r->h, r->reward, r->done, r->value, bootstrap_value,
                                                      gamma, lam, r->adv, r->ret);
        if (normalize) normalize_kernel<<<1, 1024, 0, s>>>(static_cast<long long>(r->E) * r->h, r->adv);
        const size_t n = static_cast<size_t>(r->E) * r->h;
        copy_rows(advantages, r->adv, n * 4, s);
        copy_rows(returns, r->ret, n * 4, s);
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) throw std::runtime_error(cudaGetErrorString(e));
        return MSK_OK;
    } catch (const std::invalid_argument& ex) {
        return rfail(r, ex.what());
    } catch (const std::exception& ex) {
        return rfail(r, ex.what(), MSK_ERR_CUDA);
    }
}

int msk_rollout_minibatch(msk_rollout* r, uint64_t seed, int32_t epoch, int32_t index, int32_t mb_size,
                          float* obs, float* a0, float* actions, float* logprob, float* advantages, float* returns,
                          float* value, int32_t* record_ids, void* stream) {
    if (!r) return rfail(nullptr, "null rollout");
    try {
        const long long n = static_cast<long long>(r->E) * r->h;
        if (n >= (1ll << 31)) throw std::invalid_argument("rollout_minibatch: more than 2^31 records");
        if (mb_size < 1 || index < 0 || static_cast<long long>(index) * mb_size >= n)
            throw std::invalid_argument("rollout_minibatch: minibatch out of range");
        cudaSetDevice(r->device);
        const long long first = static_cast<long long>(index) * mb_size;
        const int rows = static_cast<int>(std::min<long long>(mb_size, n - first));
        // key: (seed, epoch) mixed on the host (splitmix64)
        uint64_t z = seed + 0x9E3779B97F4A7C15ull * (static_cast<uint64_t>(epoch) + 1);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
        const MbOut o{obs, a0, actions, logprob, advantages, returns, value, record_ids};
        minibatch_kernel<<<(rows + 7) / 8, 256, 0, static_cast<cudaStream_t>(stream)>>>(
            n, feistel_half_bits(n), z, first, rows, r->obs_dim, r->act_dim, r->obs, r->a0, r->act, r->logp,
            r->adv, r->ret, r->value, o);
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) throw std::runtime_error(cudaGetErrorString(e));
        return MSK_OK;
    } catch (const std::invalid_argument& ex) {
        return rfail(r, ex.what());
    } catch (const std::exception& ex) {
        return rfail(r, ex.what(), MSK_ERR_CUDA);
    }
}

// Device pointers of the stored fields (step-major [h x E x dim]); field:
// 0 obs, 1 a0, 2 actions, 3 logprob, 4 reward, 5 done (u8), 6 value, 7 delta.
void* msk_rollout_field(msk_rollout* r, int32_t field) {
    if (!r) return nullptr;
    switch (field) {
        case 0: return r->obs;
        case 1: return r->a0;
        case 2: return r->act;
        case 3: return r->logp;
        case 4: return r->reward;
        case 5: return r->done;
        case 6: return r->value;
        case 7: return r->delta;
        default: return nullptr;
    }
}

}  // extern "C"
