// Device-side data structures shared by the kernels and the host context.
#pragma once

#include <cstdint>

#include <vector_types.h>

namespace msk_b200 {

constexpr int kSubsteps = 10;        // skeleton.hpp:13
constexpr double kSimDt = 0.002;     // skeleton.hpp:11
constexpr double kCtrlDt = 0.02;     // skeleton.hpp:12
constexpr float kMinFiber = 0.01f;   // skeleton.hpp:14
constexpr int kMaxQSlots = 4;        // nq <= 128 (DOF d lives in lane d%32, slot d/32)
constexpr int kLinkStride = 14;      // floats per link in the ABA scratch

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
    int frames, n_emg, bins, max_seg, has_general;
    float gravity, k_lim, c_k, c_c, c_mu, inv_c_vs;
    double k_lim_d;
    // links
    const int* link_parent;
    const int* link_dof;
    const float4* link_a;  // {anchor x, anchor z (parent frame), com offset, mass}
    const float* link_inertia;
    const double* link_mount;
    const int* level_start;
    const int* level_links;
    const int* child_start;
    const int* child_list;
    const int* sphere_start;
    const float4* sphere;  // {x, z, radius, 0}
    const int* sphere_link;
    // joints
    const float* joint_damping;
    const double* joint_lo;
    const double* joint_hi;
    const int* joint_slot_start;
    // muscles (packed; see CompiledModel)
    const float4* m_p0;    // {f_max, -dt/tau_act log2(e), -dt/tau_deact log2(e), l_opt v_max / 10}
    const double2* m_p1a;  // {slack, l_opt}
    const double2* m_p1b;  // {1/l_opt, 1/(dt l_opt v_max)}
    const int* m_meta;     // nseg | general << 8 | reference index << 9 (general muscles last, then by nseg)
    const int* m_int;      // reference index -> internal index
    int seg_run[6];        // [k, k+1): muscles (whole lane-group chunks) padded to k segments, k = 0..4
    int fast_nseg;         // NSEG of the fast path (0: the generic loop over all muscles)
    int gen0;              // first muscle (device order) of the generic loop: general muscles (or 0, or nm)
    // Fast-path muscle constants, chunk-major: one record per lane-group chunk of the
    // fast range with (3 + k) fields of G x 16 B each — p0 | p1a | p1b | K of segment
    // 0..k-1 — for a chunk of run k; lane i's entry of field f at f G 16 + 16 i, so
    // one chunk pointer serves every load of a muscle (immediate offsets).
    const unsigned char* mtab;
    int mrun_off[5];       // byte offset of run k's first chunk record
    // Same-link / adjacent segment k of muscle m at [k * nm + m] (coalesced over m):
    // {K1, K2h, K3h, info bits} with |s|^2 = K1 + 2 (cos K2h + sin K3h) and
    // r x A = cos K3h - sin K2h (cos/sin of the child joint's own angle, f64).
    const float4* seg_kf;
    const int* seg_info;   // [k * nm + m] kind | dof << 2 | slot << 11
    // general (non-adjacent) segments, world frame
    const int* m_pair_start;
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
    int smem_env_bytes, off_relcs, off_dqf, off_tau, off_root, off_union, off_kind, off_pen;
    int epb;  // envs per block actually used (<= the compiled warps x envs-per-warp; fewer for big models)
    // block-shared tree table at the head of dynamic smem (bytes)
    const int4* tab_blob;
    int tab_bytes, tab_off_a, tab_off_in, tab_off_meta, tab_off_child, tab_off_lvl, tab_off_lvs, tab_off_work;
    int tab_off_tq, tab_off_tqp, tab_off_chain, tab_off_slstart;  // joint-torque lists (capi.cu plan_torques): u8 flags [tq_len][G], u8 pieces [nj+1]
    int tq_len;                   // elements per lane of the joint-torque lists
};

// Per-env mutable state (device pointers, env-major rows).
struct DevState {
    double* q;        // E x nq
    double* dq;       // E x nq
    float* act;       // E x nm
    double* lm;       // E x nm (f64: prev_len = slack + l_m l_opt feeds the v_m difference)
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
    int* out_count;   // E (pending outcomes, may exceed out_cap: the excess is dropped and counted)
    int out_cap;
    unsigned long long* out_dropped;  // [1] outcomes lost to ring / drain-cap overflow (never silent)
    float* power_scratch;  // E x nm (reward mode 2 without a caller buffer)
    float* u;              // E x nm: the step's clamped excitations, device muscle order
    uint8_t* u_bad;        // E: the step's action row had a non-finite entry
};

}  // namespace msk_b200
