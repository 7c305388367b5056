// C ABI (include/msk_gpu.h): context ownership, device tables, launches.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <exception>
#include <random>
#include <string>
#include <vector>

#include "../../include/msk_gpu.h"
#include "device.cuh"
#include "disc.hpp"
#include "model.hpp"

namespace msk_b200 {

// NVTX range over a C-ABI call (header-only NVTX v3: a no-op unless a profiler is attached)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};
cudaError_t prepare_kernels(int smem_bytes_per_block);
int envs_per_block();
int lanes_per_env();
int step_envs_per_warp();
void launch_step(const DevModel&, const DevState&, int env0, int n, const float* actions, float* obs, float* delta,
                 float* raux, uint8_t* flags, float* power, float* grf, cudaStream_t, int n_substeps = kSubsteps);
void launch_reset(const DevModel&, const DevState&, int n, int mode, const uint8_t* mask, uint8_t bits,
                  const int* frames_in, float* obs, int* frames_out, uint8_t* bad, cudaStream_t);
void launch_observe(const DevModel&, const DevState&, int n, float* obs, float* delta, cudaStream_t);
void launch_seed(const DevState&, int n, uint64_t base_seed, cudaStream_t);
void launch_rng_raw(const DevState&, int e, int n, uint64_t* out, cudaStream_t);
void launch_record_own(const DevModel&, const DevState&, int n, cudaStream_t);
void launch_merge(const DevModel&, const DevState&, int n_local, const int* bins, const uint8_t* failed,
                  const int* counts, long long n_total, int cap, double* global_ema, cudaStream_t);
void launch_broadcast_ema(const DevState&, int n, int bins, const double* row, cudaStream_t);
void launch_drain(const DevState&, int n, int cap, int* bins, uint8_t* failed, int* counts, cudaStream_t);
void launch_set_mti(const DevState&, int n, const int* mti, cudaStream_t);
void launch_get_ints(const DevState&, int n, int* ints, cudaStream_t);
void launch_set_ints(const DevState&, int n, const int* ints, cudaStream_t);
void launch_permute_muscles(const DevModel&, int n, const float* src, float* dst, int to_internal, cudaStream_t);
void launch_permute_muscles(const DevModel&, int n, const double* src, double* dst, int to_internal, cudaStream_t);
void launch_rollout_stats(const DevState&, int n, const float* reward, const uint8_t* flags, double* stats,
                          cudaStream_t);
int obs_moments_chunks(int n);
void launch_obs_moments(const float* x, int n, int D, double* part, double* out, cudaStream_t, bool fold = false);
void launch_excitations(int n, int nm, long long env_offset, uint64_t seed, uint32_t step, float* out,
                        cudaStream_t);
void launch_merge_block(const DevModel& M, const int* bins, const uint8_t* failed, const int* counts, long long n,
                        int cap, double* global_ema, cudaStream_t s);
void launch_exchange_fold(const unsigned char* gathered, size_t block_bytes, int world, size_t off_stats,
                          size_t off_mom, int D, double* norm, double* stats_out, cudaStream_t s);
double measure_fp32_peak_tflops();
}  // namespace msk_b200

using namespace msk_b200;

namespace {

thread_local std::string g_last_error;

struct CudaFail : std::exception {
    std::string msg;
    explicit CudaFail(std::string m) : msg(std::move(m)) {}
    const char* what() const noexcept override { return msg.c_str(); }
};

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CudaFail(std::string(what) + ": " + cudaGetErrorString(e));
}

constexpr int kMaxHostStreams = 8;
// host-buffer pipeline shape (chunks, streams); MSK_HOST_CHUNKS / MSK_HOST_STREAMS override
int host_knob(const char* name, int dflt, int lo, int hi) {
    const char* v = std::getenv(name);
    if (!v) return dflt;
    return std::max(lo, std::min(hi, std::atoi(v)));
}

}  // namespace

struct msk_gpu_ctx {
    int device = 0;
    int n_envs = 0;
    long long env_offset = 0;
    CompiledModel cm;
    DevModel M{};
    DevState St{};
    std::vector<void*> allocs;
    std::string err;
    long long launches = 0;
    int obs_dim = 0, delta_dim = 0;
    // host-buffer path
    cudaStream_t hs[kMaxHostStreams] = {};
    int host_chunks = 4, host_streams = 4;
    int pipe_chunks = 0, pipe_streams = 0;  // msk_gpu_set_host_pipeline before the first host step
    float* h_actions = nullptr;  // device staging
    float* h_obs = nullptr;
    float* h_delta = nullptr;
    float* h_raux = nullptr;
    uint8_t* h_flags = nullptr;
    float* h_reward = nullptr;
    double* mom_part = nullptr;  // obs-moment partials (msk_gpu_obs_moments)
    size_t mom_cap = 0;
    double* global_ema = nullptr;
    // device discriminator (msk_gpu_set_discriminator)
    DiscDev disc{};
    std::vector<void*> disc_allocs;
    bool disc_fast = false;  // msk_gpu_set_discriminator_mode: bf16 fast mode instead of split-bf16
    // iteration exchange (msk_gpu_iteration_exchange): this rank's block and the gathered blocks
    unsigned char* x_block = nullptr;
    unsigned char* x_gathered = nullptr;
    size_t x_block_bytes = 0, x_gathered_bytes = 0;
    void* x_hdr = nullptr;  // layout header all-gather (multi-rank)
    int x_checked_cap = -1;
    float* r_delta = nullptr;  // scratch when the caller passes no Δ / reward_aux / flags
    float* r_raux = nullptr;
    uint8_t* r_flags = nullptr;

    template <class T>
    T* dalloc(size_t n) {
        void* p = nullptr;
        ck(cudaMalloc(&p, std::max<size_t>(1, n) * sizeof(T)), "cudaMalloc");
        ck(cudaMemset(p, 0, std::max<size_t>(1, n) * sizeof(T)), "cudaMemset");
        allocs.push_back(p);
        return static_cast<T*>(p);
    }
    template <class T>
    const T* upload(const std::vector<T>& v) {
        T* p = dalloc<T>(v.size());
        if (!v.empty()) ck(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice), "upload");
        return p;
    }
    void count(int n = 1) { launches += n; }
    void check_launch() { ck(cudaGetLastError(), "kernel launch"); }
};

namespace {

int fail(msk_gpu_ctx* ctx, int code, const std::string& msg) {
    g_last_error = msg;
    if (ctx) ctx->err = msg;
    return code;
}

template <class F>
int guarded(msk_gpu_ctx* ctx, F&& f) {
    if (!ctx) return fail(nullptr, MSK_ERR_CONTRACT, "null context");
    try {
        ck(cudaSetDevice(ctx->device), "cudaSetDevice");
        f();
        return MSK_OK;
    } catch (const CudaFail& ex) {
        return fail(ctx, MSK_ERR_CUDA, ex.what());
    } catch (const std::exception& ex) {
        return fail(ctx, MSK_ERR_CONTRACT, ex.what());
    }
}

cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

constexpr int kDefaultOutCap = 64;

// Zeroed device buffer owned outside ctx->allocs (resizable tables).
void* raw_alloc(size_t bytes) {
    void* p = nullptr;
    ck(cudaMalloc(&p, std::max<size_t>(1, bytes)), "cudaMalloc");
    ck(cudaMemset(p, 0, std::max<size_t>(1, bytes)), "cudaMemset");
    return p;
}

// Grow the per-env pending-outcome ring to `cap` slots (never shrinks): the
// pending entries move with a pitched copy on `s`, after which the old ring is
// released (the host waits for s once; resizing is rare).
void grow_outcome_ring(msk_gpu_ctx* ctx, int cap, cudaStream_t s) {
    DevState& S = ctx->St;
    if (cap <= S.out_cap) return;
    const size_t E = ctx->n_envs;
    int* nb = static_cast<int*>(raw_alloc(E * cap * sizeof(int)));
    uint8_t* nf = static_cast<uint8_t*>(raw_alloc(E * cap));
    ck(cudaMemcpy2DAsync(nb, cap * sizeof(int), S.out_bin, S.out_cap * sizeof(int), S.out_cap * sizeof(int), E,
                         cudaMemcpyDeviceToDevice, s),
       "grow outcome ring");
    ck(cudaMemcpy2DAsync(nf, cap, S.out_failed, S.out_cap, S.out_cap, E, cudaMemcpyDeviceToDevice, s),
       "grow outcome ring");
    ck(cudaStreamSynchronize(s), "grow outcome ring");
    cudaFree(S.out_bin);
    cudaFree(S.out_failed);
    S.out_bin = nb;
    S.out_failed = nf;
    S.out_cap = cap;
}

int align16(int x) { return (x + 15) & ~15; }

// Balanced joint-torque sums.  The moment slots of joint j (fixed (muscle,
// segment) order, CompiledModel::joint_slot_start) are cut into pieces of at most
// ceil(n_pairs / G) consecutive slots; pieces go to the G lanes longest first
// (each to the least-loaded lane), and a lane's pieces are laid out as one list:
// element i of lane l lives in slot i G + l, so every lane sums its list with
// conflict-free shared loads and stores a piece's partial sum at the piece's last
// element (flag = piece id).  A joint's torque is then the sum of its pieces in
// piece order — a fixed summation order, like the joint-major loop it replaces,
// with max-over-lanes work ~n_pairs / G instead of the largest joints' slot counts.
struct TorquePlan {
    std::vector<int> slot_new;      // old slot (0..n_pairs, n_pairs = dummy) -> new slot
    std::vector<uint8_t> flag;      // len * G: piece id ending at that element, else 0xff
    std::vector<uint8_t> piece0;    // nj + 1: pieces of joint j = [piece0[j], piece0[j+1])
    int len = 0, n_pieces = 0;
};

TorquePlan plan_torques(const CompiledModel& c, int G) {
    TorquePlan P;
    const int np = c.n_pairs;
    // piece size: ~n_pairs / G, grown until the partial sums fit the frame scratch
    // (one f64 per 8 B: 2 per link; one piece per joint fits since n_joints <= n_links)
    int cap = std::max(1, (np + G - 1) / G);
    auto count = [&](int cp) {
        int n = 0;
        for (int j = 0; j < c.nj; ++j) n += (c.joint_slot_start[j + 1] - c.joint_slot_start[j] + cp - 1) / cp;
        return n;
    };
    const int lim = std::min(2 * c.nl, 255);
    while (count(cap) > lim && cap < np) ++cap;
    if (count(cap) > lim) throw ConfigError("model too large: more than 255 joints with muscle moments");
    struct Piece { int joint, s0, n; };
    std::vector<Piece> pieces;
    P.piece0.assign(c.nj + 1, 0);
    for (int j = 0; j < c.nj; ++j) {
        P.piece0[j] = static_cast<uint8_t>(pieces.size());
        const int a = c.joint_slot_start[j], b = c.joint_slot_start[j + 1], n = b - a;
        const int k = (n + cap - 1) / cap;
        for (int q = 0; q < k; ++q) {
            const int lo = a + static_cast<int>(static_cast<long>(n) * q / k);
            const int hi = a + static_cast<int>(static_cast<long>(n) * (q + 1) / k);
            pieces.push_back({j, lo, hi - lo});
        }
    }
    P.piece0[c.nj] = static_cast<uint8_t>(pieces.size());
    P.n_pieces = static_cast<int>(pieces.size());
    std::vector<int> order(pieces.size());
    for (size_t i = 0; i < order.size(); ++i) order[i] = static_cast<int>(i);
    std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return pieces[x].n > pieces[y].n; });
    std::vector<std::vector<int>> lane(G);
    std::vector<int> load(G, 0);
    for (int id : order) {
        const int l = static_cast<int>(std::min_element(load.begin(), load.end()) - load.begin());
        lane[l].push_back(id);
        load[l] += pieces[id].n;
    }
    P.len = std::max(1, *std::max_element(load.begin(), load.end()));
    P.slot_new.assign(np + 1, 0);
    P.flag.assign(static_cast<size_t>(P.len) * G, 0xff);
    for (int l = 0; l < G; ++l) {
        int i = 0;
        for (int id : lane[l]) {
            const Piece& pc = pieces[id];
            for (int t = 0; t < pc.n; ++t, ++i) P.slot_new[pc.s0 + t] = i * G + l;
            if (pc.n > 0) P.flag[static_cast<size_t>(i - 1) * G + l] = static_cast<uint8_t>(id);
        }
    }
    P.slot_new[np] = P.len * G;  // dummy slot after the lists
    return P;
}

}  // namespace

extern "C" {

int msk_gpu_create(const char* model_json_path, const char* clip_csv_path, const msk_env_config* cfg,
                   const msk_reward_config* rc, int32_t n_envs, uint64_t base_seed, int64_t global_env_offset,
                   int device, msk_gpu_ctx** out) {
    if (!out) return fail(nullptr, MSK_ERR_CONTRACT, "msk_gpu_create: out is null");
    *out = nullptr;
    auto ctx = new msk_gpu_ctx();
    try {
        if (n_envs < 1) throw ConfigError("msk_gpu_create: n_envs must be >= 1");
        if (!model_json_path || !clip_csv_path) throw ConfigError("msk_gpu_create: model and clip paths required");
        // load_model does not call ModelSpec::validate (model.cpp:198-204) and neither does
        // Env::Env (env.cpp:74-87): only the structure the device tables need is enforced
        const ModelSpec spec = load_model(model_json_path);
        const auto errs = spec.device_envelope();
        if (!errs.empty()) throw ConfigError("model '" + std::string(model_json_path) + "': " + errs.front());
        const Clip clip = load_clip(clip_csv_path, spec);
        msk_env_config ec{250, 1, 10, 0, 0.2, 0.99, 0.5, 0.01};
        if (cfg) ec = *cfg;
        msk_reward_config rw{0, 0, 100.0, 0.05, nullptr};
        if (rc) rw = *rc;
        std::vector<int32_t> emg_map(rw.emg_channel_map, rw.emg_channel_map + std::max(0, rw.n_emg_channels));
        for (int ch : emg_map)
            if (ch < 0 || ch >= static_cast<int>(spec.muscles.size()))
                throw ConfigError("env: emg channel map references missing muscle");
        if (rw.mode == 1 && static_cast<int>(emg_map.size()) != clip.n_emg)
            throw ConfigError("env: emg channel map size must match reference emg columns");
        ctx->cm = compile_model(spec);
        const CompiledModel& c = ctx->cm;
        if (c.nq > 32 * kMaxQSlots) throw ConfigError("model too large: n_q > 128");

        int ndev = 0;
        ck(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
        if (device < 0 || device >= ndev) throw CudaFail("no CUDA device " + std::to_string(device));
        cudaDeviceProp prop{};
        ck(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
        if (prop.major != 10) throw CudaFail("msk_gpu requires an sm_100 (Blackwell B200) device, found sm_" +
                                             std::to_string(prop.major) + std::to_string(prop.minor));
        ctx->device = device;
        ck(cudaSetDevice(device), "cudaSetDevice");
        ctx->n_envs = n_envs;
        ctx->env_offset = global_env_offset;

        DevModel& M = ctx->M;
        M.nl = c.nl;
        M.nj = c.nj;
        M.nq = c.nq;
        M.nrd = c.nrd;
        M.nm = c.nm;
        M.nk = c.nk;
        M.ns = c.ns;
        M.floating = c.floating;
        M.n_levels = c.n_levels;
        M.n_pairs = c.n_pairs;
        M.frames = clip.frames;
        M.n_emg = clip.n_emg;
        if (ec.adaptive_bins > 1024) throw ConfigError("env: adaptive_bins > 1024 not supported on the device");
        M.bins = std::max(1, ec.adaptive_bins);
        M.gravity = c.gravity;
        M.k_lim = c.k_lim;
        M.k_lim_d = c.k_lim_d;
        M.c_k = c.c_k;
        M.c_c = c.c_c;
        M.c_mu = c.c_mu;
        M.inv_c_vs = c.inv_c_vs;
        const TorquePlan tq = plan_torques(c, lanes_per_env());
        M.tq_len = tq.len;
        M.n_pairs = tq.len * lanes_per_env();  // slots incl. the lists' padding; dummy slot = n_pairs
        std::vector<float4> p0h, kfh;  // host copies for the chunk-major fast-path table
        std::vector<double2> p1ah, p1bh;
        {
            std::vector<float4> la(c.nl), sp(c.ns);
            for (int l = 0; l < c.nl; ++l) la[l] = make_float4(c.link_ax[l], c.link_az[l], c.link_com[l], c.link_mass[l]);
            for (int s = 0; s < c.ns; ++s) sp[s] = make_float4(c.sphere_x[s], c.sphere_z[s], c.sphere_r[s], 0.f);
            M.link_a = ctx->upload(la);
            M.sphere = ctx->upload(sp);
            const size_t nsg = static_cast<size_t>(c.max_seg) * c.nm;
            std::vector<float4> p0(c.nm), kf(nsg);
            std::vector<double2> p1a(c.nm), p1b(c.nm);
            for (int m = 0; m < c.nm; ++m) {
                p0[m] = make_float4(c.pk_p0[4 * m], c.pk_p0[4 * m + 1], c.pk_p0[4 * m + 2], c.pk_p0[4 * m + 3]);
                p1a[m] = make_double2(c.pk_p1[4 * m], c.pk_p1[4 * m + 1]);
                p1b[m] = make_double2(c.pk_p1[4 * m + 2], c.pk_p1[4 * m + 3]);
            }
            // |A + R c|^2 = |A|^2 + |c|^2 + 2 (cos A.c + sin (A_z c_x - A_x c_z)).  The
            // K constants are rounded to f32 once (a fixed ~1e-8 relative perturbation of
            // the geometry); reset and step both evaluate lengths from these same values,
            // so the fibre-velocity difference L - prev_len sees no mismatch.
            for (size_t i = 0; i < nsg; ++i) {
                const double ax = c.pk_geo[4 * i], az = c.pk_geo[4 * i + 1];
                const double cx = c.pk_geo[4 * i + 2], cz = c.pk_geo[4 * i + 3];
                const int info = c.pk_info[i], kind = info & 3;
                float k1 = 0.f, k2 = 0.f, k3 = 0.f;
                if (kind == 0) {
                    k1 = static_cast<float>(ax * ax);  // same-link: constant length in ax
                } else if (kind == 1) {
                    k1 = static_cast<float>(ax * ax + az * az + cx * cx + cz * cz);
                    k2 = static_cast<float>(ax * cx + az * cz);
                    k3 = static_cast<float>(az * cx - ax * cz);
                }
                // kinds 0/1 carry a moment slot (remapped to the torque lists), kind 2 a via index
                const int info_new = kind == 2 ? info : (info & 0x7ff) | (tq.slot_new[info >> 11] << 11);
                float w;
                std::memcpy(&w, &info_new, sizeof w);
                kf[i] = make_float4(k1, k2, k3, w);
            }
            M.m_p0 = ctx->upload(p0);
            M.m_p1a = ctx->upload(p1a);
            M.m_p1b = ctx->upload(p1b);
            M.seg_kf = ctx->upload(kf);
            p0h = std::move(p0);
            p1ah = std::move(p1a);
            p1bh = std::move(p1b);
            kfh = std::move(kf);
        }
        M.max_seg = c.max_seg;
        M.has_general = c.has_general;
        {  // fast path over the muscles without a general segment ([0, n_fast), sorted by
           // segment count) in chunk runs by padded segment count: a lane group's chunk of
           // G consecutive muscles pads to the count of its last muscle; the generic loop
           // takes the rest ([gen0, nm))
            const bool fast = c.n_fast > 0 && c.max_seg_fast <= 4;
            const int nf = fast ? c.n_fast : 0;
            M.fast_nseg = fast ? std::max(1, c.max_seg_fast) : 0;
            M.gen0 = nf;
            const int G = lanes_per_env();
            std::vector<int> chunk_ns;
            for (int m0 = 0; m0 < nf; m0 += G) chunk_ns.push_back(c.pk_meta[std::min(m0 + G, nf) - 1] & 0xff);
            for (int k = 0; k <= 5; ++k) {
                int m = nf;
                for (size_t ch = 0; ch < chunk_ns.size(); ++ch)
                    if (chunk_ns[ch] >= k) {
                        m = static_cast<int>(ch) * G;
                        break;
                    }
                M.seg_run[k] = k == 5 ? nf : m;
            }
            M.seg_run[0] = 0;
            // chunk-major record table of the fast range (device.cuh mtab)
            std::vector<unsigned char> tab;
            const size_t fb = static_cast<size_t>(G) * 16;
            for (int k = 0; k <= 4; ++k) {
                M.mrun_off[k] = static_cast<int>(tab.size());
                for (int m0 = M.seg_run[k]; m0 < M.seg_run[k + 1]; m0 += G) {
                    const size_t r0 = tab.size();
                    tab.resize(r0 + (3 + k) * fb, 0);
                    for (int i = 0; i < G && m0 + i < nf; ++i) {
                        const int m = m0 + i;
                        unsigned char* e = tab.data() + r0 + 16 * i;
                        std::memcpy(e, &p0h[m], 16);
                        std::memcpy(e + fb, &p1ah[m], 16);
                        std::memcpy(e + 2 * fb, &p1bh[m], 16);
                        for (int g = 0; g < k; ++g) std::memcpy(e + (3 + g) * fb, &kfh[static_cast<size_t>(g) * c.nm + m], 16);
                    }
                }
            }
            if (tab.empty()) tab.resize(16, 0);
            M.mtab = ctx->upload(tab);
        }
        M.link_parent = ctx->upload(c.link_parent);
        M.link_dof = ctx->upload(c.link_dof);
        M.link_inertia = ctx->upload(c.link_inertia);
        M.link_mount = ctx->upload(c.link_mount);
        M.level_start = ctx->upload(c.level_start);
        M.level_links = ctx->upload(c.level_links);
        M.child_start = ctx->upload(c.child_start);
        M.child_list = ctx->upload(c.child_list);
        M.sphere_start = ctx->upload(c.sphere_start);
        M.sphere_link = ctx->upload(c.sphere_link);
        M.joint_damping = ctx->upload(c.joint_damping);
        M.joint_lo = ctx->upload(c.joint_lo);
        M.joint_hi = ctx->upload(c.joint_hi);
        M.joint_slot_start = ctx->upload(c.joint_slot_start);
        M.m_meta = ctx->upload(c.pk_meta);
        M.m_int = ctx->upload(c.m_int);
        M.seg_info = ctx->upload(c.pk_info);
        M.m_pair_start = ctx->upload(c.m_pair_start);
        M.via_link = ctx->upload(c.via_link);
        M.via_x = ctx->upload(c.via_x);
        M.via_z = ctx->upload(c.via_z);
        M.pair_joint = ctx->upload(c.pair_joint);
        M.pair_via = ctx->upload(c.pair_via);
        {
            std::vector<int32_t> ps(c.pair_slot.size());
            for (size_t i = 0; i < ps.size(); ++i) ps[i] = tq.slot_new[c.pair_slot[i]];
            M.pair_slot = ctx->upload(ps);
        }
        M.pair_sign = ctx->upload(c.pair_sign);
        M.key_bodies = ctx->upload(c.key_bodies);
        M.clip_q = ctx->upload(clip.q);
        M.clip_dq = ctx->upload(clip.dq);
        M.clip_kp = ctx->upload(clip.key_pos);
        M.clip_ka = ctx->upload(clip.key_angle);
        M.clip_emg = ctx->upload(clip.emg);
        M.horizon = ec.episode_horizon;
        M.rsi = ec.rsi;
        M.eval_mode = 0;
        M.reward_mode = rw.mode;
        M.n_emg_ch = static_cast<int>(emg_map.size());
        M.mix = ec.adaptive_mix;
        M.decay = ec.adaptive_decay;
        M.term_err = ec.termination_body_err;
        M.init_act = ec.init_activation;
        M.w_emg = static_cast<float>(rw.w_emg);
        M.w_power = static_cast<float>(rw.w_power);
        std::vector<int32_t> emg_int(emg_map.size());  // channel -> internal muscle index
        for (size_t ch = 0; ch < emg_map.size(); ++ch) emg_int[ch] = c.m_int[emg_map[ch]];
        M.emg_map = ctx->upload(emg_int);
        // per-env shared-memory layout (~8 KB for the whole-body model)
        int off = 16 * c.nl;  // kin
        M.off_relcs = off;
        off = align16(off + 16 * c.nq);
        M.off_dqf = off;
        off = align16(off + 4 * c.nq);
        M.off_tau = off;
        off = align16(off + 4 * c.nq);
        M.off_root = off;
        off = align16(off + 16);
        M.off_union = off;
        off = align16(off + 4 * std::max({M.n_pairs + 1, kLinkStride * c.nl, 2 * c.nq}));  // +1: dummy slot
        M.off_kind = off;  // f64 link frames, only for models with general muscle segments
        if (c.has_general) off = align16(off + 32 * c.nl);
        M.off_pen = off;  // contact-sphere penetrations
        off = align16(off + 4 * c.ns);
        M.smem_env_bytes = off;
        {  // block-shared tree table: link {anchor, com, mass}, inertia, packed meta,
           // child lists and the depth-level schedule (u8 indices, n_links <= 255)
            if (c.nl > 255 || c.n_levels > 255) throw ConfigError("model too large: n_links > 255");
            int t = 0;
            M.tab_off_a = t;
            t += 16 * c.nl;
            M.tab_off_in = t;
            t += 4 * c.nl;
            M.tab_off_meta = t;
            t += 4 * c.nl;
            M.tab_off_child = t;
            t += c.nl;
            M.tab_off_lvl = t;
            t += c.nl;
            M.tab_off_lvs = t;
            t += c.n_levels + 1;
            t = align16(t);
            M.tab_off_work = t;  // per (level, slot < 32) work words of the tree passes
            t += 4 * 32 * c.n_levels;
            M.tab_off_tq = t;  // joint-torque lists: piece flags, then pieces per joint
            t += static_cast<int>(tq.flag.size());
            M.tab_off_tqp = t;
            t += c.nj + 1;
            M.tab_off_chain = t;  // per level: chain flag | super-level end (see the work-word slots below)
            t += c.n_levels;
            M.tab_off_slstart = t;  // per level: first level of its super-level
            t += c.n_levels;
            M.tab_bytes = align16(t);
            std::vector<unsigned char> blob(M.tab_bytes, 0);
            auto put = [&](int at, const void* src, size_t n) { std::memcpy(blob.data() + at, src, n); };
            for (int l = 0; l < c.nl; ++l) {
                const float a[4] = {c.link_ax[l], c.link_az[l], c.link_com[l], c.link_mass[l]};
                put(M.tab_off_a + 16 * l, a, 16);
                // rotational inertia about the link origin, I + m com^2 (the frame-independent
                // (0,0) entry of the spatial inertia; the sweep no longer forms it per substep)
                const float i0 = static_cast<float>(static_cast<double>(c.link_inertia[l]) +
                                                    static_cast<double>(c.link_mass[l]) * c.link_com[l] * c.link_com[l]);
                put(M.tab_off_in + 4 * l, &i0, 4);
                const int nchild = c.child_start[l + 1] - c.child_start[l];
                const int has_sph = c.sphere_start[l + 1] > c.sphere_start[l] ? 1 : 0;
                const int meta = (c.link_parent[l] + 1) | (nchild << 8) | (c.child_start[l] << 16) | (has_sph << 24);
                put(M.tab_off_meta + 4 * l, &meta, 4);
                blob[M.tab_off_child + l] = static_cast<unsigned char>(l < static_cast<int>(c.child_list.size())
                                                                          ? c.child_list[l] : 0);
                blob[M.tab_off_lvl + l] = static_cast<unsigned char>(c.level_links[l]);
            }
            for (int d = 0; d <= c.n_levels; ++d) blob[M.tab_off_lvs + d] = static_cast<unsigned char>(c.level_start[d]);
            // work word of slot i of level d: link | (parent + 1) << 8 | child_off << 16 |
            // nchild << 24 | has_sphere << 28 | simple level << 29 | valid << 31 (one shared load per level).
            // Chain levels: every link of level d is its parent's only child (and no link of
            // level d - 1 has more than one child).  Their links take their parent's slot, so
            // the step kernel's passes run each lane down (or up) a chain of such levels in
            // registers, with no warp barrier in between (tree_sweep_chain & co.); slots of a
            // chain level can have gaps (a leaf parent), every pass skips invalid slots.
            std::vector<int> slot_of(c.nl, -1);
            for (int d = 0; d < c.n_levels; ++d) {
                const int b = c.level_start[d], n = c.level_start[d + 1] - b;
                if (n > 32) throw ConfigError("model too wide: a tree level has more than 32 links");
                bool chain = d > 0;
                for (int i = 0; i < n && chain; ++i) {
                    const int l = c.level_links[b + i], pl = c.link_parent[l];
                    chain = pl >= 0 && c.child_start[pl + 1] - c.child_start[pl] == 1 && l >= c.floating;
                }
                blob[M.tab_off_chain + d] = chain ? 0x80 : 0;
                for (int i = 0; i < n; ++i) {
                    const int l = c.level_links[b + i];
                    slot_of[l] = chain ? slot_of[c.link_parent[l]] : i;
                }
            }
            for (int d0 = 0; d0 < c.n_levels;) {  // super-levels [d0, d1): first -> end, last -> first
                int d1 = d0 + 1;
                while (d1 < c.n_levels && (blob[M.tab_off_chain + d1] & 0x80)) ++d1;
                if (d1 > 127) throw ConfigError("model too deep: more than 127 tree levels");
                blob[M.tab_off_chain + d0] |= static_cast<unsigned char>(d1);
                for (int d = d0; d < d1; ++d) blob[M.tab_off_slstart + d] = static_cast<unsigned char>(d0);
                d0 = d1;
            }
            for (int d = 0; d < c.n_levels; ++d) {
                const int b = c.level_start[d], n = c.level_start[d + 1] - b;
                // bit 29: the level is "simple" — every link has a parent link and a joint DOF
                // (no root, no child of the fixed base), so the passes skip those branches
                bool simple = true;
                for (int i = 0; i < n; ++i) {
                    const int l = c.level_links[b + i];
                    simple = simple && c.link_parent[l] >= 0 && l >= c.floating;
                }
                for (int i = 0; i < n; ++i) {
                    const int l = c.level_links[b + i];
                    const int nchild = c.child_start[l + 1] - c.child_start[l];
                    if (nchild > 15) throw ConfigError("model too wide: a link has more than 15 children");
                    const int has_sph = c.sphere_start[l + 1] > c.sphere_start[l] ? 1 : 0;
                    const uint32_t w = static_cast<uint32_t>(l) | (static_cast<uint32_t>(c.link_parent[l] + 1) << 8) |
                                       (static_cast<uint32_t>(c.child_start[l]) << 16) |
                                       (static_cast<uint32_t>(nchild) << 24) | (static_cast<uint32_t>(has_sph) << 28) |
                                       (static_cast<uint32_t>(simple) << 29) | (1u << 31);
                    put(M.tab_off_work + 4 * (32 * d + slot_of[l]), &w, 4);
                }
            }
            put(M.tab_off_tq, tq.flag.data(), tq.flag.size());
            put(M.tab_off_tqp, tq.piece0.data(), tq.piece0.size());
            M.tab_blob = reinterpret_cast<const int4*>(ctx->upload(blob));
        }
        // as many env slots per block as shared memory allows (28 for the whole-body models)
        // (minus the reset kernel's static env list, kResetRange ints)
        const int avail = static_cast<int>(prop.sharedMemPerBlockOptin) - M.tab_bytes - 1088;
        M.epb = std::min(envs_per_block(), avail / std::max(1, M.smem_env_bytes));
        M.epb -= M.epb % step_envs_per_warp();  // the env-vectorised step kernel fills whole warps
        if (M.epb < 1)
            throw ConfigError("model needs " + std::to_string(M.tab_bytes + M.smem_env_bytes) +
                              " B of shared memory per env");
        const int per_block = M.tab_bytes + M.epb * M.smem_env_bytes;
        ck(prepare_kernels(per_block), "cudaFuncSetAttribute");

        DevState& S = ctx->St;
        const size_t E = static_cast<size_t>(n_envs);
        S.q = ctx->dalloc<double>(E * c.nq);
        S.dq = ctx->dalloc<double>(E * c.nq);
        S.act = ctx->dalloc<float>(E * c.nm);
        S.lm = ctx->dalloc<double>(E * c.nm);
        S.vm = ctx->dalloc<float>(E * c.nm);
        S.fm = ctx->dalloc<float>(E * c.nm);
        S.t = ctx->dalloc<double>(E);
        S.t_index = ctx->dalloc<int>(E);
        S.start = ctx->dalloc<int>(E);
        S.steps = ctx->dalloc<int>(E);
        S.done = ctx->dalloc<uint8_t>(E);
        S.mt = ctx->dalloc<uint64_t>(E * 312);
        S.mti = ctx->dalloc<int>(E);
        S.ema = ctx->dalloc<double>(E * M.bins);
        // pending-outcome ring: kDefaultOutCap slots per env (an env ends at most one
        // episode per step); grown on demand by drain / exchange with a larger cap or
        // by msk_gpu_set_outcome_capacity; outcomes past it are counted in out_dropped
        S.out_cap = kDefaultOutCap;
        S.out_bin = static_cast<int*>(raw_alloc(E * S.out_cap * sizeof(int)));
        S.out_failed = static_cast<uint8_t*>(raw_alloc(E * S.out_cap));
        S.out_count = ctx->dalloc<int>(E);
        S.out_dropped = ctx->dalloc<unsigned long long>(1);
        S.power_scratch = rw.mode == 2 ? ctx->dalloc<float>(E * c.nm) : nullptr;
        S.u = ctx->dalloc<float>(E * c.nm);
        S.u_bad = ctx->dalloc<uint8_t>(E);
        ctx->global_ema = ctx->dalloc<double>(M.bins);
        ctx->obs_dim = 3 * c.nq + 6 * c.nk + 4 * c.nm;
        // obs-moment partials for a whole batch, allocated up front (no allocation,
        // hence no implicit sync, at the first iteration boundary)
        ctx->mom_cap = static_cast<size_t>(obs_moments_chunks(n_envs)) * ctx->obs_dim * 2 + 1;
        ctx->mom_part = ctx->dalloc<double>(ctx->mom_cap);
        ctx->delta_dim = 3 + c.nj + 2 * c.nk;

        launch_seed(S, n_envs, base_seed + static_cast<uint64_t>(global_env_offset), nullptr);
        launch_reset(M, S, n_envs, 3 /* kResetInit */, nullptr, 0, nullptr, nullptr, nullptr, nullptr, nullptr);
        ctx->count(2);
        ctx->check_launch();
        ck(cudaDeviceSynchronize(), "create");
        *out = ctx;
        return MSK_OK;
    } catch (const CudaFail& ex) {
        const int code = fail(nullptr, MSK_ERR_CUDA, ex.what());
        msk_gpu_destroy(ctx);
        return code;
    } catch (const std::exception& ex) {
        const int code = fail(nullptr, MSK_ERR_CONTRACT, ex.what());
        msk_gpu_destroy(ctx);
        return code;
    }
}

void msk_gpu_destroy(msk_gpu_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaDeviceSynchronize();
    if (ctx->x_block) cudaFree(ctx->x_block);
    if (ctx->St.out_bin) cudaFree(ctx->St.out_bin);
    if (ctx->St.out_failed) cudaFree(ctx->St.out_failed);
    if (ctx->x_gathered) cudaFree(ctx->x_gathered);
    if (ctx->x_hdr) cudaFree(ctx->x_hdr);
    for (void* p : ctx->allocs) cudaFree(p);
    for (void* p : ctx->disc_allocs) cudaFree(p);
    for (auto& s : ctx->hs)
        if (s) cudaStreamDestroy(s);
    delete ctx;
}

const char* msk_gpu_last_error(const msk_gpu_ctx* ctx) {
    return ctx ? ctx->err.c_str() : g_last_error.c_str();
}

int msk_gpu_dims(const msk_gpu_ctx* ctx, msk_dims* out) {
    if (!ctx || !out) return fail(nullptr, MSK_ERR_CONTRACT, "msk_gpu_dims: null argument");
    const auto& c = ctx->cm;
    out->n_envs = ctx->n_envs;
    out->nq = c.nq;
    out->n_muscles = c.nm;
    out->obs_dim = ctx->obs_dim;
    out->delta_dim = ctx->delta_dim;
    out->n_links = c.nl;
    out->n_joints = c.nj;
    out->n_key = c.nk;
    out->n_spheres = c.ns;
    out->frames = ctx->M.frames;
    out->floating = c.floating;
    out->adaptive_bins = ctx->M.bins;
    return MSK_OK;
}

int msk_gpu_set_eval_mode(msk_gpu_ctx* ctx, int32_t eval_mode) {
    return guarded(ctx, [&] { ctx->M.eval_mode = eval_mode != 0; });
}

int msk_gpu_reset(msk_gpu_ctx* ctx, const uint8_t* mask, uint8_t mask_bits, float* obs, int32_t* start_frames,
                  void* stream) {
    const msk_b200::NvtxRange nvtx_("msk_gpu_reset");
    return guarded(ctx, [&] {
        launch_reset(ctx->M, ctx->St, ctx->n_envs, 0, mask, mask ? mask_bits : 0, nullptr, obs, start_frames, nullptr,
                     as_stream(stream));
        ctx->count();
        ctx->check_launch();
    });
}

int msk_gpu_reset_to_frame(msk_gpu_ctx* ctx, const int32_t* frames, const uint8_t* mask, float* obs, uint8_t* bad,
                           void* stream) {
    return guarded(ctx, [&] {
        if (!frames) throw ConfigError("reset_to_frame: frames is null");
        launch_reset(ctx->M, ctx->St, ctx->n_envs, 1, mask, 0xff, frames, obs, nullptr, bad, as_stream(stream));
        ctx->count();
        ctx->check_launch();
    });
}

int msk_gpu_step(msk_gpu_ctx* ctx, const float* actions, float* obs, float* delta, float* reward_aux, uint8_t* flags,
                 float* muscle_power, float* contact_force, void* stream) {
    const msk_b200::NvtxRange nvtx_("msk_gpu_step");
    return guarded(ctx, [&] {
        if (!actions) throw ConfigError("step: actions is null");
        launch_step(ctx->M, ctx->St, 0, ctx->n_envs, actions, obs, delta, reward_aux, flags, muscle_power,
                    contact_force, as_stream(stream));
        ctx->count(2);  // prep_actions + step
        ctx->check_launch();
    });
}

int msk_gpu_substeps(msk_gpu_ctx* ctx, const float* actions, int32_t n_substeps, float* muscle_power,
                     float* contact_force, void* stream) {
    return guarded(ctx, [&] {
        if (!actions || n_substeps < 1 || n_substeps >= kSubsteps)
            throw ConfigError("substeps: actions required and 1 <= n_substeps < 10");
        launch_step(ctx->M, ctx->St, 0, ctx->n_envs, actions, nullptr, nullptr, nullptr, nullptr, muscle_power,
                    contact_force, as_stream(stream), n_substeps);
        ctx->count(2);
        ctx->check_launch();
    });
}

int msk_gpu_set_discriminator_mode(msk_gpu_ctx* ctx, int32_t mode) {
    return guarded(ctx, [&] {
        if (mode != 0 && mode != 1) throw ConfigError("set_discriminator_mode: mode must be 0 (fp32-class) or 1 (bf16)");
        ctx->disc_fast = mode == 1;
        ctx->disc.precise = ctx->disc_fast ? 0 : 1;
    });
}

int msk_gpu_set_discriminator(msk_gpu_ctx* ctx, const double* theta, int64_t n_params, int32_t hidden) {
    return guarded(ctx, [&] {
        if (!theta) throw ConfigError("set_discriminator: theta is null");
        const DiscHost h = build_disc_images(theta, n_params, ctx->delta_dim, hidden);
        for (void* p : ctx->disc_allocs) cudaFree(p);
        ctx->disc_allocs.clear();
        auto up = [&](const void* src, size_t bytes) {
            void* p = nullptr;
            ck(cudaMalloc(&p, bytes), "cudaMalloc");
            ctx->disc_allocs.push_back(p);
            ck(cudaMemcpy(p, src, bytes, cudaMemcpyHostToDevice), "upload discriminator");
            return p;
        };
        DiscDev d;
        d.din = h.din;
        d.hidden = h.hidden;
        d.k1 = h.k1;
        d.tmem_cols = 32;
        while (d.tmem_cols < static_cast<uint32_t>(h.hidden)) d.tmem_cols <<= 1;
        d.w1 = up(h.w1.data(), h.w1.size() * 2);
        d.w2 = up(h.w2.data(), h.w2.size() * 2);
        d.w3 = up(h.w3.data(), h.w3.size() * 2);
        d.bias = static_cast<const float*>(up(h.bias.data(), h.bias.size() * 4));
        d.c_hi[0] = up(h.c1_hi.data(), h.c1_hi.size() * 2);
        d.c_lo[0] = up(h.c1_lo.data(), h.c1_lo.size() * 2);
        d.c_hi[1] = up(h.c2_hi.data(), h.c2_hi.size() * 2);
        d.c_lo[1] = up(h.c2_lo.data(), h.c2_lo.size() * 2);
        d.c_hi[2] = up(h.c3_hi.data(), h.c3_hi.size() * 2);
        d.c_lo[2] = up(h.c3_lo.data(), h.c3_lo.size() * 2);
        d.precise = ctx->disc_fast ? 0 : 1;
        ck(prepare_disc(d), "cudaFuncSetAttribute(disc)");
        ctx->disc = d;
        if (!ctx->r_delta) {
            ctx->r_delta = ctx->dalloc<float>(static_cast<size_t>(ctx->n_envs) * ctx->delta_dim);
            ctx->r_raux = ctx->dalloc<float>(ctx->n_envs);
            ctx->r_flags = ctx->dalloc<uint8_t>(ctx->n_envs);
        }
    });
}

int64_t msk_mlp_param_count(int32_t in, int32_t hidden, int32_t out) {
    if (in < 1 || hidden < 1 || out < 1) return -1;
    return static_cast<int64_t>(hidden) * in + hidden + 2 * (static_cast<int64_t>(hidden) * hidden + hidden) +
           static_cast<int64_t>(out) * hidden + out;
}

int msk_mlp_init(double* theta, int32_t in, int32_t hidden, int32_t out, uint64_t seed, double final_init_scale) {
    // Mlp::Mlp(shape, seed) (nn.cpp:16-38) with msk::Rng (rng.hpp:13-30): W(i, j)
    // ~ uniform(-s, s) in column-major order, s = 1/sqrt(cols) (x final_init_scale
    // on the head), biases zero.
    const int64_t n = msk_mlp_param_count(in, hidden, out);
    if (!theta || n < 0) return fail(nullptr, MSK_ERR_CONTRACT, "msk_mlp_init: bad shape");
    std::mt19937_64 eng(seed);
    const int dims[4][2] = {{hidden, in}, {hidden, hidden}, {hidden, hidden}, {out, hidden}};
    int64_t off = 0;
    for (int l = 0; l < 4; ++l) {
        const int r = dims[l][0], c = dims[l][1];
        const double s = (1.0 / std::sqrt(static_cast<double>(c))) * (l == 3 ? final_init_scale : 1.0);
        for (int j = 0; j < c; ++j)
            for (int i = 0; i < r; ++i)
                theta[off + static_cast<int64_t>(j) * r + i] = -s + (s - -s) * (static_cast<double>(eng() >> 11) * 0x1.0p-53);
        off += static_cast<int64_t>(r) * c;
        for (int i = 0; i < r; ++i) theta[off + i] = 0.0;
        off += r;
    }
    return MSK_OK;
}

int msk_gpu_clear_discriminator(msk_gpu_ctx* ctx) {
    return guarded(ctx, [&] {
        ck(cudaDeviceSynchronize(), "clear_discriminator");
        for (void* p : ctx->disc_allocs) cudaFree(p);
        ctx->disc_allocs.clear();
        ctx->disc = DiscDev{};
    });
}

int msk_disc_trainer_publish(msk_disc_trainer* trainer, msk_gpu_ctx* ctx, void* stream) {
    return guarded(ctx, [&] {
        if (!trainer) throw ConfigError("disc_trainer_publish: trainer is null");
        int din = 0, hidden = 0;
        const double* theta = disc_trainer_theta(trainer, &din, &hidden);
        if (!ctx->disc.w1) throw ConfigError("disc_trainer_publish: set a discriminator of the same shape first");
        if (din != ctx->disc.din || hidden != ctx->disc.hidden)
            throw ConfigError("disc_trainer_publish: trainer shape differs from the context's discriminator");
        ck(launch_disc_repack(theta, ctx->disc, as_stream(stream)), "disc repack");
        ctx->count();
    });
}

int msk_gpu_discriminator_reward(msk_gpu_ctx* ctx, const float* delta, int32_t n, float* reward, void* stream) {
    const msk_b200::NvtxRange nvtx_("msk_gpu_discriminator_reward");
    return guarded(ctx, [&] {
        if (!ctx->disc.w1) throw ConfigError("discriminator_reward: no discriminator set");
        if (!delta || !reward || n < 0) throw ConfigError("discriminator_reward: bad arguments");
        ck(launch_disc(ctx->disc, delta, ctx->delta_dim, n, nullptr, nullptr, reward, as_stream(stream), false),
           "launch discriminator");
        ctx->count();
    });
}

int msk_gpu_step_rewarded(msk_gpu_ctx* ctx, const float* actions, float* obs, float* delta, float* reward,
                          float* reward_aux, uint8_t* flags, float* muscle_power, float* contact_force,
                          void* stream) {
    const msk_b200::NvtxRange nvtx_("msk_gpu_step_rewarded");
    return guarded(ctx, [&] {
        if (!actions || !reward) throw ConfigError("step_rewarded: actions and reward are required");
        if (!ctx->disc.w1) throw ConfigError("step_rewarded: no discriminator set");
        float* d = delta ? delta : ctx->r_delta;
        float* ra = reward_aux ? reward_aux : ctx->r_raux;
        uint8_t* f = flags ? flags : ctx->r_flags;
        cudaStream_t s = as_stream(stream);
        launch_step(ctx->M, ctx->St, 0, ctx->n_envs, actions, obs, d, ra, f, muscle_power, contact_force, s);
        ctx->count(2);  // prep_actions + step
        ctx->check_launch();
        // D(Δ) on the tensor cores, launched as a programmatic dependent of the step
        ck(launch_disc(ctx->disc, d, ctx->delta_dim, ctx->n_envs, ra, f, reward, s, true), "launch discriminator");
        ctx->count();
    });
}

namespace {

// Host-buffer step, optionally with the discriminator reward.  Chunked
// pipeline: H2D(actions c) -> step(c) [-> D(c)] -> D2H(outputs c), chunks on
// separate streams so chunk c's transfers overlap the other chunks' kernels.
void step_host_impl(msk_gpu_ctx* ctx, const float* actions_host, float* obs_host, float* delta_host,
                    float* reward_host, float* reward_aux_host, uint8_t* flags_host, bool wait) {
    if (!actions_host) throw ConfigError("step_host: actions is null");
    if (reward_host && !ctx->disc.w1) throw ConfigError("step_host: reward requested but no discriminator set");
    const size_t E = static_cast<size_t>(ctx->n_envs);
    const int nm = ctx->cm.nm;
    if (!ctx->hs[0]) {
        ctx->host_chunks = ctx->pipe_chunks ? ctx->pipe_chunks : host_knob("MSK_HOST_CHUNKS", 4, 1, 64);
        ctx->host_streams =
            ctx->pipe_streams ? ctx->pipe_streams : host_knob("MSK_HOST_STREAMS", 4, 1, kMaxHostStreams);
        for (int i = 0; i < ctx->host_streams; ++i)
            ck(cudaStreamCreateWithFlags(&ctx->hs[i], cudaStreamNonBlocking), "stream");
        ctx->h_actions = ctx->dalloc<float>(E * nm);
        ctx->h_obs = ctx->dalloc<float>(E * ctx->obs_dim);
        ctx->h_delta = ctx->dalloc<float>(E * ctx->delta_dim);
        ctx->h_raux = ctx->dalloc<float>(E);
        ctx->h_flags = ctx->dalloc<uint8_t>(E);
        ctx->h_reward = ctx->dalloc<float>(E);
    }
    const int chunks = static_cast<int>(std::min<size_t>(ctx->host_chunks, E));
    const size_t per = (E + chunks - 1) / chunks;
    for (int c = 0; c < chunks; ++c) {
        const size_t e0 = c * per;
        if (e0 >= E) break;  // ragged E: ceil-sized chunks can run out before `chunks`
        const size_t n = std::min(per, E - e0);
        cudaStream_t s = ctx->hs[c % ctx->host_streams];
        ck(cudaMemcpyAsync(ctx->h_actions + e0 * nm, actions_host + e0 * nm, n * nm * sizeof(float),
                           cudaMemcpyHostToDevice, s),
           "H2D actions");
        launch_step(ctx->M, ctx->St, static_cast<int>(e0), static_cast<int>(n), ctx->h_actions + e0 * nm,
                    ctx->h_obs + e0 * ctx->obs_dim, ctx->h_delta + e0 * ctx->delta_dim, ctx->h_raux + e0,
                    ctx->h_flags + e0, nullptr, nullptr, s);
        ctx->count(2);  // prep_actions + step
        ctx->check_launch();
        if (reward_host) {
            ck(launch_disc(ctx->disc, ctx->h_delta + e0 * ctx->delta_dim, ctx->delta_dim, static_cast<int>(n),
                           ctx->h_raux + e0, ctx->h_flags + e0, ctx->h_reward + e0, s, true),
               "launch discriminator");
            ctx->count();
            ck(cudaMemcpyAsync(reward_host + e0, ctx->h_reward + e0, n * sizeof(float), cudaMemcpyDeviceToHost, s),
               "D2H reward");
        }
        if (obs_host)
            ck(cudaMemcpyAsync(obs_host + e0 * ctx->obs_dim, ctx->h_obs + e0 * ctx->obs_dim,
                               n * ctx->obs_dim * sizeof(float), cudaMemcpyDeviceToHost, s),
               "D2H obs");
        if (delta_host)
            ck(cudaMemcpyAsync(delta_host + e0 * ctx->delta_dim, ctx->h_delta + e0 * ctx->delta_dim,
                               n * ctx->delta_dim * sizeof(float), cudaMemcpyDeviceToHost, s),
               "D2H delta");
        if (reward_aux_host)
            ck(cudaMemcpyAsync(reward_aux_host + e0, ctx->h_raux + e0, n * sizeof(float), cudaMemcpyDeviceToHost, s),
               "D2H reward_aux");
        if (flags_host)
            ck(cudaMemcpyAsync(flags_host + e0, ctx->h_flags + e0, n, cudaMemcpyDeviceToHost, s), "D2H flags");
    }
    if (wait)
        for (int i = 0; i < ctx->host_streams; ++i) ck(cudaStreamSynchronize(ctx->hs[i]), "step_host sync");
}

}  // namespace

int msk_gpu_step_host(msk_gpu_ctx* ctx, const float* actions_host, float* obs_host, float* delta_host,
                      float* reward_aux_host, uint8_t* flags_host) {
    const msk_b200::NvtxRange nvtx_("msk_gpu_step_host");
    return guarded(ctx, [&] {
        step_host_impl(ctx, actions_host, obs_host, delta_host, nullptr, reward_aux_host, flags_host, true);
    });
}

int msk_gpu_step_host_rewarded(msk_gpu_ctx* ctx, const float* actions_host, float* obs_host, float* delta_host,
                               float* reward_host, float* reward_aux_host, uint8_t* flags_host) {
    const msk_b200::NvtxRange nvtx_("msk_gpu_step_host_rewarded");
    return guarded(ctx, [&] {
        if (!reward_host) throw ConfigError("step_host_rewarded: reward is null");
        step_host_impl(ctx, actions_host, obs_host, delta_host, reward_host, reward_aux_host, flags_host, true);
    });
}

int msk_gpu_step_host_async(msk_gpu_ctx* ctx, const float* actions_host, float* obs_host, float* delta_host,
                            float* reward_host, float* reward_aux_host, uint8_t* flags_host) {
    const msk_b200::NvtxRange nvtx_("msk_gpu_step_host_async");
    return guarded(ctx, [&] {
        step_host_impl(ctx, actions_host, obs_host, delta_host, reward_host, reward_aux_host, flags_host, false);
    });
}

int msk_gpu_set_host_pipeline(msk_gpu_ctx* ctx, int32_t chunks, int32_t streams) {
    return guarded(ctx, [&] {
        if (chunks < 1 || chunks > 64 || streams < 1 || streams > kMaxHostStreams)
            throw ConfigError("set_host_pipeline: chunks in [1, 64], streams in [1, 8]");
        for (int i = 0; i < ctx->host_streams; ++i)
            if (ctx->hs[i]) ck(cudaStreamSynchronize(ctx->hs[i]), "set_host_pipeline");
        if (!ctx->hs[0]) {  // not yet initialised: the first host step creates the streams
            ctx->pipe_chunks = chunks;
            ctx->pipe_streams = streams;
            return;
        }
        for (int i = ctx->host_streams; i < streams; ++i)
            ck(cudaStreamCreateWithFlags(&ctx->hs[i], cudaStreamNonBlocking), "stream");
        ctx->host_chunks = chunks;
        ctx->host_streams = std::max(ctx->host_streams, streams);
    });
}

int msk_gpu_host_wait(msk_gpu_ctx* ctx) {
    return guarded(ctx, [&] {
        for (int i = 0; i < ctx->host_streams; ++i)
            if (ctx->hs[i]) ck(cudaStreamSynchronize(ctx->hs[i]), "host_wait");
    });
}

int msk_gpu_observe(msk_gpu_ctx* ctx, float* obs, void* stream) {
    const msk_b200::NvtxRange nvtx_("msk_gpu_observe");
    return guarded(ctx, [&] {
        launch_observe(ctx->M, ctx->St, ctx->n_envs, obs, nullptr, as_stream(stream));
        ctx->count();
        ctx->check_launch();
    });
}

int msk_gpu_tracking_error(msk_gpu_ctx* ctx, float* delta, void* stream) {
    return guarded(ctx, [&] {
        launch_observe(ctx->M, ctx->St, ctx->n_envs, nullptr, delta, as_stream(stream));
        ctx->count();
        ctx->check_launch();
    });
}

int msk_gpu_force_state_to_reference(msk_gpu_ctx* ctx, void* stream) {
    return guarded(ctx, [&] {
        launch_reset(ctx->M, ctx->St, ctx->n_envs, 2, nullptr, 0, nullptr, nullptr, nullptr, nullptr,
                     as_stream(stream));
        ctx->count();
        ctx->check_launch();
    });
}

int msk_gpu_get_state(msk_gpu_ctx* ctx, double* q, double* dq, float* act, double* l_m, float* v_m, float* f_m,
                      double* t, int32_t* ints, void* stream) {
    return guarded(ctx, [&] {
        const size_t E = ctx->n_envs, nq = ctx->cm.nq;
        cudaStream_t s = as_stream(stream);
        auto cp = [&](void* dst, const void* src, size_t bytes) {
            if (dst) ck(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, s), "get_state");
        };
        cp(q, ctx->St.q, E * nq * 8);
        cp(dq, ctx->St.dq, E * nq * 8);
        // muscle rows: internal (segment-count) order -> reference order
        for (auto [dst, src] : {std::pair<float*, const float*>{act, ctx->St.act}, {v_m, ctx->St.vm}, {f_m, ctx->St.fm}})
            if (dst) {
                launch_permute_muscles(ctx->M, ctx->n_envs, src, dst, 0, s);
                ctx->count();
                ctx->check_launch();
            }
        if (l_m) {
            launch_permute_muscles(ctx->M, ctx->n_envs, ctx->St.lm, l_m, 0, s);
            ctx->count();
            ctx->check_launch();
        }
        cp(t, ctx->St.t, E * 8);
        if (ints) {
            launch_get_ints(ctx->St, ctx->n_envs, ints, s);
            ctx->count();
            ctx->check_launch();
        }
    });
}

int msk_gpu_set_state(msk_gpu_ctx* ctx, const double* q, const double* dq, const float* act, const double* l_m,
                      const float* v_m, const float* f_m, const double* t, const int32_t* ints, void* stream) {
    return guarded(ctx, [&] {
        const size_t E = ctx->n_envs, nq = ctx->cm.nq;
        cudaStream_t s = as_stream(stream);
        auto cp = [&](void* dst, const void* src, size_t bytes) {
            if (src) ck(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, s), "set_state");
        };
        cp(ctx->St.q, q, E * nq * 8);
        cp(ctx->St.dq, dq, E * nq * 8);
        for (auto [dst, src] : {std::pair<float*, const float*>{ctx->St.act, act}, {ctx->St.vm, v_m}, {ctx->St.fm, f_m}})
            if (src) {
                launch_permute_muscles(ctx->M, ctx->n_envs, src, dst, 1, s);
                ctx->count();
                ctx->check_launch();
            }
        if (l_m) {
            launch_permute_muscles(ctx->M, ctx->n_envs, l_m, ctx->St.lm, 1, s);
            ctx->count();
            ctx->check_launch();
        }
        cp(ctx->St.t, t, E * 8);
        if (ints) {
            launch_set_ints(ctx->St, ctx->n_envs, ints, s);
            ctx->count();
            ctx->check_launch();
        }
    });
}

int msk_gpu_get_sampler(msk_gpu_ctx* ctx, double* ema, void* stream) {
    return guarded(ctx, [&] {
        ck(cudaMemcpyAsync(ema, ctx->St.ema, sizeof(double) * ctx->n_envs * ctx->M.bins, cudaMemcpyDeviceToDevice,
                           as_stream(stream)),
           "get_sampler");
    });
}

int msk_gpu_set_sampler(msk_gpu_ctx* ctx, const double* ema, int32_t broadcast, void* stream) {
    return guarded(ctx, [&] {
        if (broadcast) {
            launch_broadcast_ema(ctx->St, ctx->n_envs, ctx->M.bins, ema, as_stream(stream));
            ctx->count();
            ctx->check_launch();
        } else {
            ck(cudaMemcpyAsync(ctx->St.ema, ema, sizeof(double) * ctx->n_envs * ctx->M.bins,
                               cudaMemcpyDeviceToDevice, as_stream(stream)),
               "set_sampler");
        }
    });
}

int msk_gpu_drain_outcomes(msk_gpu_ctx* ctx, int32_t* bins, uint8_t* failed, int32_t* counts, int32_t cap,
                           void* stream) {
    const msk_b200::NvtxRange nvtx_("msk_gpu_drain_outcomes");
    return guarded(ctx, [&] {
        if (!bins || !failed || !counts || cap < 0) throw ConfigError("drain_outcomes: bad arguments");
        grow_outcome_ring(ctx, cap, as_stream(stream));  // sized for the caller's next drain
        launch_drain(ctx->St, ctx->n_envs, cap, bins, failed, counts, as_stream(stream));
        ctx->count();
        ctx->check_launch();
    });
}

int msk_gpu_rollout_stats(msk_gpu_ctx* ctx, const float* reward, const uint8_t* flags, double* stats,
                          void* stream) {
    const msk_b200::NvtxRange nvtx_("msk_gpu_rollout_stats");
    return guarded(ctx, [&] {
        if (!flags || !stats) throw ConfigError("rollout_stats: flags and stats are required");
        launch_rollout_stats(ctx->St, ctx->n_envs, reward, flags, stats, as_stream(stream));
        ctx->count();
        ctx->check_launch();
    });
}

namespace {
void obs_moments_impl(msk_gpu_ctx* ctx, const float* obs, int32_t n, double* out, void* stream, bool fold) {
    if ((!obs && n > 0) || !out || n < 0) throw ConfigError("obs_moments: bad arguments");
    const size_t need = static_cast<size_t>(obs_moments_chunks(n)) * ctx->obs_dim * 2 + 1;
    if (need > ctx->mom_cap) {
        ctx->mom_part = ctx->dalloc<double>(need);
        ctx->mom_cap = need;
    }
    launch_obs_moments(obs, n, ctx->obs_dim, ctx->mom_part, out, as_stream(stream), fold);
    ctx->count(n > 0 ? 2 : (fold ? 0 : 1));
    ctx->check_launch();
}
}  // namespace

int msk_gpu_obs_moments(msk_gpu_ctx* ctx, const float* obs, int32_t n, double* out, void* stream) {
    const msk_b200::NvtxRange nvtx_("msk_gpu_obs_moments");
    return guarded(ctx, [&] { obs_moments_impl(ctx, obs, n, out, stream, false); });
}

int msk_gpu_obs_moments_fold(msk_gpu_ctx* ctx, const float* obs, int32_t n, double* acc, void* stream) {
    const msk_b200::NvtxRange nvtx_("msk_gpu_obs_moments_fold");
    return guarded(ctx, [&] { obs_moments_impl(ctx, obs, n, acc, stream, true); });
}

int msk_gpu_record_own_outcomes(msk_gpu_ctx* ctx, void* stream) {
    return guarded(ctx, [&] {
        launch_record_own(ctx->M, ctx->St, ctx->n_envs, as_stream(stream));
        ctx->count();
        ctx->check_launch();
    });
}

int msk_gpu_merge_outcomes(msk_gpu_ctx* ctx, const int32_t* bins, const uint8_t* failed, const int32_t* counts,
                           int64_t n_envs_total, int32_t cap, void* stream) {
    return guarded(ctx, [&] {
        if (!bins || !failed || !counts || cap < 0 || n_envs_total < 0)
            throw ConfigError("merge_outcomes: bad arguments");
        // the global sampler starts from env 0's current EMA (all envs hold the
        // same replicated EMA under this convention)
        ck(cudaMemcpyAsync(ctx->global_ema, ctx->St.ema, sizeof(double) * ctx->M.bins, cudaMemcpyDeviceToDevice,
                           as_stream(stream)),
           "merge_outcomes");
        launch_merge(ctx->M, ctx->St, ctx->n_envs, bins, failed, counts, n_envs_total, cap, ctx->global_ema,
                     as_stream(stream));
        ctx->count(2);
        ctx->check_launch();
    });
}

}  // extern "C"

namespace {
// NCCL is resolved at run time (dlopen of libnccl.so.2, e.g. the copy the
// process already holds), so the library has no link-time NCCL dependency.
struct NcclApi {
    decltype(&ncclAllGather) all_gather = nullptr;
    decltype(&ncclCommCount) count = nullptr;
    bool ok = false;
};
const NcclApi& nccl_api() {
    static const NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return a;
        a.all_gather = reinterpret_cast<decltype(&ncclAllGather)>(dlsym(h, "ncclAllGather"));
        a.count = reinterpret_cast<decltype(&ncclCommCount)>(dlsym(h, "ncclCommCount"));
        a.ok = a.all_gather && a.count;
        return a;
    }();
    return api;
}
size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }
}  // namespace

extern "C" {

int msk_gpu_iteration_exchange(msk_gpu_ctx* ctx, void* nccl_comm, int32_t cap, const float* obs,
                               const double* stats_in, double* norm_state, double* stats_out, void* stream) {
    const msk_b200::NvtxRange nvtx_("msk_gpu_iteration_exchange");
    return guarded(ctx, [&] {
        if (cap < 1 || !obs || !stats_in || !norm_state) throw ConfigError("iteration_exchange: bad arguments");
        cudaStream_t s = as_stream(stream);
        const size_t E = ctx->n_envs, D = ctx->obs_dim;
        // block: bins i32 [E cap] | failed u8 [E cap] | counts i32 [E] | stats f64 [7] | moments f64 [1 + 2D]
        const size_t off_failed = align_up(4 * E * cap, 16), off_counts = align_up(off_failed + E * cap, 16);
        const size_t off_stats = align_up(off_counts + 4 * E, 16), off_mom = align_up(off_stats + 8 * 7, 16);
        const size_t bytes = align_up(off_mom + 8 * (1 + 2 * D), 16);
        int world = 1;
        if (nccl_comm) {
            if (!nccl_api().ok) throw CudaFail("iteration_exchange: libnccl.so.2 not loadable");
            if (nccl_api().count(static_cast<ncclComm_t>(nccl_comm), &world) != ncclSuccess)
                throw CudaFail("iteration_exchange: ncclCommCount failed");
        }
        if (world > 1 && cap != ctx->x_checked_cap) {
            // every rank must build the same block layout, or ncclAllGather would hang or
            // mix ranks' data: all-gather a fixed 32-B header {E, cap, D, bytes} first
            // (once per cap; E and D are fixed per context) and fail on any mismatch
            const int64_t hdr[4] = {static_cast<int64_t>(E), cap, static_cast<int64_t>(D),
                                    static_cast<int64_t>(bytes)};
            if (ctx->x_hdr) cudaFree(ctx->x_hdr);
            ctx->x_hdr = nullptr;
            ck(cudaMalloc(&ctx->x_hdr, 32 * (1 + static_cast<size_t>(world))), "cudaMalloc");
            ck(cudaMemcpyAsync(ctx->x_hdr, hdr, 32, cudaMemcpyHostToDevice, s), "exchange header");
            if (nccl_api().all_gather(ctx->x_hdr, static_cast<unsigned char*>(ctx->x_hdr) + 32, 32, ncclUint8,
                                      static_cast<ncclComm_t>(nccl_comm), s) != ncclSuccess)
                throw CudaFail("iteration_exchange: ncclAllGather (header) failed");
            std::vector<int64_t> all(4 * static_cast<size_t>(world));
            ck(cudaMemcpyAsync(all.data(), static_cast<unsigned char*>(ctx->x_hdr) + 32, 32 * world,
                               cudaMemcpyDeviceToHost, s),
               "exchange header");
            ck(cudaStreamSynchronize(s), "exchange header");
            for (int r = 0; r < world; ++r)
                if (!std::equal(hdr, hdr + 4, all.data() + 4 * r))
                    throw ConfigError("iteration_exchange: rank " + std::to_string(r) + " has {envs " +
                                      std::to_string(all[4 * r]) + ", cap " + std::to_string(all[4 * r + 1]) +
                                      ", obs_dim " + std::to_string(all[4 * r + 2]) + "}, this rank {" +
                                      std::to_string(E) + ", " + std::to_string(cap) + ", " + std::to_string(D) +
                                      "}: every rank must exchange the same block layout");
            ctx->x_checked_cap = cap;
        }
        grow_outcome_ring(ctx, cap, s);
        if (bytes != ctx->x_block_bytes) {
            if (ctx->x_block) cudaFree(ctx->x_block);
            ck(cudaMalloc(&ctx->x_block, bytes), "cudaMalloc");
            ctx->x_block_bytes = bytes;
        }
        if (world > 1 && bytes * world != ctx->x_gathered_bytes) {
            if (ctx->x_gathered) cudaFree(ctx->x_gathered);
            ck(cudaMalloc(&ctx->x_gathered, bytes * world), "cudaMalloc");
            ctx->x_gathered_bytes = bytes * world;
        }
        unsigned char* b = ctx->x_block;
        launch_drain(ctx->St, ctx->n_envs, cap, reinterpret_cast<int*>(b), b + off_failed,
                     reinterpret_cast<int*>(b + off_counts), s);
        ck(cudaMemcpyAsync(b + off_stats, stats_in, 8 * 7, cudaMemcpyDeviceToDevice, s), "stats");
        const size_t need = static_cast<size_t>(obs_moments_chunks(ctx->n_envs)) * D * 2 + 1;
        if (need > ctx->mom_cap) {
            ctx->mom_part = ctx->dalloc<double>(need);
            ctx->mom_cap = need;
        }
        launch_obs_moments(obs, ctx->n_envs, static_cast<int>(D), ctx->mom_part, reinterpret_cast<double*>(b + off_mom),
                           s);
        unsigned char* g = b;
        if (world > 1) {
            if (nccl_api().all_gather(b, ctx->x_gathered, bytes, ncclUint8, static_cast<ncclComm_t>(nccl_comm), s) !=
                ncclSuccess)
                throw CudaFail("iteration_exchange: ncclAllGather failed");
            g = ctx->x_gathered;
        }
        // identical rank-ordered merge on every rank: outcomes (global env order =
        // rank order, then env, then time) into the replicated sampler, stats and
        // observation moments folded in rank order
        ck(cudaMemcpyAsync(ctx->global_ema, ctx->St.ema, sizeof(double) * ctx->M.bins, cudaMemcpyDeviceToDevice, s),
           "ema");
        for (int r = 0; r < world; ++r) {
            const unsigned char* br = g + r * bytes;
            launch_merge_block(ctx->M, reinterpret_cast<const int*>(br), br + off_failed,
                               reinterpret_cast<const int*>(br + off_counts), static_cast<long long>(E), cap,
                               ctx->global_ema, s);
        }
        launch_broadcast_ema(ctx->St, ctx->n_envs, ctx->M.bins, ctx->global_ema, s);
        launch_exchange_fold(g, bytes, world, off_stats, off_mom, static_cast<int>(D), norm_state, stats_out, s);
        ctx->count(5 + world);
        ctx->check_launch();
    });
}

int msk_gpu_get_rng(msk_gpu_ctx* ctx, uint64_t* mt, int32_t* mti, void* stream) {
    return guarded(ctx, [&] {
        const size_t E = ctx->n_envs;
        cudaStream_t s = as_stream(stream);
        if (mt) ck(cudaMemcpyAsync(mt, ctx->St.mt, E * 312 * 8, cudaMemcpyDeviceToDevice, s), "get_rng");
        if (mti) ck(cudaMemcpyAsync(mti, ctx->St.mti, E * 4, cudaMemcpyDeviceToDevice, s), "get_rng");
    });
}

int msk_gpu_set_rng(msk_gpu_ctx* ctx, const uint64_t* mt, const int32_t* mti, void* stream) {
    return guarded(ctx, [&] {
        const size_t E = ctx->n_envs;
        cudaStream_t s = as_stream(stream);
        if (mt) ck(cudaMemcpyAsync(ctx->St.mt, mt, E * 312 * 8, cudaMemcpyDeviceToDevice, s), "set_rng");
        if (mti) {
            launch_set_mti(ctx->St, ctx->n_envs, mti, s);  // clamps the index into [0, 312]
            ctx->count();
            ctx->check_launch();
        }
    });
}

int msk_gpu_set_outcome_capacity(msk_gpu_ctx* ctx, int32_t cap, void* stream) {
    return guarded(ctx, [&] {
        if (cap < 1 || cap > (1 << 20)) throw ConfigError("set_outcome_capacity: cap must be in [1, 2^20]");
        grow_outcome_ring(ctx, cap, as_stream(stream));
    });
}

int msk_gpu_outcomes_dropped(msk_gpu_ctx* ctx, int64_t* dropped) {
    return guarded(ctx, [&] {
        if (!dropped) throw ConfigError("outcomes_dropped: null argument");
        unsigned long long v = 0;
        ck(cudaDeviceSynchronize(), "outcomes_dropped");
        ck(cudaMemcpy(&v, ctx->St.out_dropped, sizeof v, cudaMemcpyDeviceToHost), "outcomes_dropped");
        *dropped = static_cast<int64_t>(v);
    });
}

int msk_gpu_rng_raw(msk_gpu_ctx* ctx, int32_t env, int32_t n, uint64_t* out, void* stream) {
    return guarded(ctx, [&] {
        if (env < 0 || env >= ctx->n_envs || n < 0 || !out) throw ConfigError("rng_raw: bad arguments");
        launch_rng_raw(ctx->St, env, n, out, as_stream(stream));
        ctx->count();
        ctx->check_launch();
    });
}

int msk_gpu_fill_excitations(msk_gpu_ctx* ctx, uint64_t seed, uint32_t step, float* actions, void* stream) {
    return guarded(ctx, [&] {
        if (!actions) throw ConfigError("fill_excitations: actions is null");
        launch_excitations(ctx->n_envs, ctx->cm.nm, ctx->env_offset, seed, step, actions, as_stream(stream));
        ctx->count();
        ctx->check_launch();
    });
}

int64_t msk_gpu_launch_count(const msk_gpu_ctx* ctx) { return ctx ? ctx->launches : 0; }

int msk_gpu_validate(const char* model_json_path, const char* clip_csv_path, msk_dims* dims) {
    try {
        if (!model_json_path) throw ConfigError("validate: model path is null");
        const ModelSpec spec = load_model(model_json_path);
        const auto errs = spec.validate();
        if (!errs.empty()) throw ConfigError("model '" + std::string(model_json_path) + "': " + errs.front());
        Clip clip;
        if (clip_csv_path && clip_csv_path[0]) clip = load_clip(clip_csv_path, spec);
        const CompiledModel c = compile_model(spec);
        if (dims) {
            dims->n_envs = 0;
            dims->nq = c.nq;
            dims->n_muscles = c.nm;
            dims->obs_dim = 3 * c.nq + 6 * c.nk + 4 * c.nm;
            dims->delta_dim = 3 + c.nj + 2 * c.nk;
            dims->n_links = c.nl;
            dims->n_joints = c.nj;
            dims->n_key = c.nk;
            dims->n_spheres = c.ns;
            dims->frames = clip.frames;
            dims->floating = c.floating;
            dims->adaptive_bins = 0;
        }
        return MSK_OK;
    } catch (const std::exception& ex) {
        return fail(nullptr, MSK_ERR_CONTRACT, ex.what());
    }
}

int msk_gpu_fp32_peak_probe(int device, double* tflops) {
    try {
        if (!tflops) throw ConfigError("fp32_peak_probe: null output");
        ck(cudaSetDevice(device), "cudaSetDevice");
        *tflops = measure_fp32_peak_tflops();
        return MSK_OK;
    } catch (const CudaFail& ex) {
        return fail(nullptr, MSK_ERR_CUDA, ex.what());
    } catch (const std::exception& ex) {
        return fail(nullptr, MSK_ERR_CONTRACT, ex.what());
    }
}

}  // extern "C"
