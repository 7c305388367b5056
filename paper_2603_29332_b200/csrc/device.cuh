// Device-side data structures shared by the kernels and the host context.
#pragma once

#include <cstdint>

namespace msk_b200 {

constexpr int kSubsteps = 10;        // skeleton.hpp:13
constexpr double kSimDt = 0.002;     // skeleton.hpp:11
constexpr double kCtrlDt = 0.02;     // skeleton.hpp:12
constexpr float kMinFiber = 0.01f;   // skeleton.hpp:14
constexpr int kMaxQSlots = 4;        // nq <= 128 (DOF d lives in lane d%32, slot d/32)
constexpr int kMaxLinkSlots = 4;     // n_links <= 128 for per-lane GRF accumulators

enum : uint8_t {
    kFlagDone = 1,
    kFlagFailed = 2,
    kFlagDiverged = 4,
    kFlagNotStepped = 8,
    kFlagBadAction = 16,
};

// Read-only model + clip + config tables (device pointers), passed by value.
struct DevModel {
    int nl, nj, nq, nrd, nm, nk, ns, floating, n_levels, n_pairs;
    int frames, n_emg, bins;
    float gravity, k_lim, c_k, c_c, c_mu, inv_c_vs;
    double k_lim_d;
    // links
    const int* link_parent;
    const int* link_dof;
    const float* link_ax;
    const float* link_az;
    const float* link_com;
    const float* link_mass;
    const float* link_inertia;
    const double* link_mount;
    const int* level_start;
    const int* level_links;
    const int* child_start;
    const int* child_list;
    const int* sphere_start;
    const float* sphere_x;
    const float* sphere_z;
    const float* sphere_r;
    // joints
    const float* joint_damping;
    const double* joint_lo;
    const double* joint_hi;
    const int* joint_slot_start;
    // muscles
    const float* m_fmax;
    const float* m_lopt;
    const float* m_inv_lopt;
    const float* m_slack;
    const float* m_kv;
    const float* m_ndt_act;
    const float* m_ndt_deact;
    const float* m_pw;
    const int* m_via_start;
    const int* m_pair_start;
    const int* m_seg_start;
    const int* seg_info;
    const int* seg_slot;
    const float* seg_ax;
    const float* seg_az;
    const float* seg_cx;
    const float* seg_cz;
    const int* via_link;
    const float* via_x;
    const float* via_z;
    const int* pair_joint;
    const int* pair_via;
    const int* pair_slot;
    const float* pair_sign;
    const int* key_bodies;
    // clip (row-major T x cols, f64)
    const double* clip_q;
    const double* clip_dq;
    const double* clip_kp;
    const double* clip_ka;
    const double* clip_emg;
    // EnvConfig / RewardConfig
    int horizon, rsi, eval_mode, reward_mode, n_emg_ch;
    double mix, decay, term_err, init_act;
    float w_emg, w_power;
    const int* emg_map;
    // per-env smem layout (bytes from the warp's base)
    int smem_env_bytes, off_theta, off_qang, off_dqf, off_tau, off_union, off_root, off_relcs;
};

// Per-env mutable state (device pointers, env-major rows).
struct DevState {
    double* q;        // E x nq
    double* dq;       // E x nq
    float* act;       // E x nm
    float* lm;        // E x nm
    float* vm;        // E x nm
    float* fm;        // E x nm
    double* t;        // E
    int* t_index;     // E
    int* start;       // E
    int* steps;       // E
    uint8_t* done;    // E
    uint64_t* mt;     // E x 312
    int* mti;         // E
    double* ema;      // E x bins
    int* out_bin;     // E x out_cap
    uint8_t* out_failed;
    int* out_count;   // E
    int out_cap;
    float* power_scratch;  // E x nm (reward mode 2 without a caller buffer)
};

}  // namespace msk_b200
