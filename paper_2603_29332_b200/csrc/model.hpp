// Host-side model and clip ingest + the "model compiler" that lays a
// ModelSpec out as flat device tables (structure of arrays).
//
// Parsing mirrors the reference's rules so the same files are accepted and
// rejected: unknown JSON keys are hard errors (json_util.hpp:14-23,
// model.cpp:94-196), ModelSpec::validate (model.cpp:18-86), and the clip CSV
// column contract + validation of load_reference (reference.cpp:11-93).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace msk_b200 {

struct ConfigError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

struct LinkSpec {
    std::string name;
    double length = 1.0, mass = 1.0, inertia = 0.1, com = 0.5;
};
struct JointSpec {
    std::string name;
    int child = 0, parent = -1;
    double ax = 0.0, az = 0.0, mount = 0.0, lo = -3.0, hi = 3.0, damping = 0.0;
};
struct Via {
    int link = -1;
    double x = 0.0, z = 0.0;
};
struct MuscleSpec {
    std::string name;
    double f_max = 1000.0, l_opt = 0.1, v_max = 10.0, tau_act = 0.010, tau_deact = 0.040, slack = 0.0;
    std::vector<Via> vias;
};
struct SphereSpec {
    int link = 0;
    double x = 0.0, z = 0.0, radius = 0.02;
};

struct ModelSpec {
    std::string name;
    bool floating = false;
    double gravity = -9.81, k_lim = 200.0;
    double c_k = 2.0e4, c_c = 500.0, c_mu = 0.9, c_vs = 0.05;
    std::vector<LinkSpec> links;
    std::vector<JointSpec> joints;
    std::vector<MuscleSpec> muscles;
    std::vector<SphereSpec> spheres;
    std::vector<int> key_bodies;

    int nrd() const { return floating ? 3 : 0; }
    int nq() const { return nrd() + static_cast<int>(joints.size()); }
    std::vector<std::string> validate() const;
    // Structural subset msk_gpu_create enforces (the reference's load_model runs no validation).
    std::vector<std::string> device_envelope() const;
};

struct Clip {
    double rate = 50.0;
    int frames = 0, nq = 0, nk = 0, n_emg = 0;
    std::vector<double> q, dq, key_pos, key_angle, emg;  // row-major T x cols
};

ModelSpec load_model(const std::string& path);
Clip load_clip(const std::string& path, const ModelSpec& spec);

// Flat tables consumed by the kernels.  Link l keeps the reference's index
// (parents precede children, model.cpp:37-46).
struct CompiledModel {
    int nl = 0, nj = 0, nq = 0, nrd = 0, nm = 0, nk = 0, ns = 0, floating = 0;
    int n_levels = 0, n_pairs = 0, n_via = 0, max_via = 0;
    float gravity = 0, k_lim = 0, c_k = 0, c_c = 0, c_mu = 0, inv_c_vs = 0;
    double k_lim_d = 0;
    // links
    std::vector<int32_t> link_parent, link_dof;  // dof = -1 for the floating root
    std::vector<float> link_ax, link_az, link_com, link_mass, link_inertia;
    std::vector<double> link_mount;
    std::vector<int32_t> level_start, level_links;  // links grouped by tree depth
    std::vector<int32_t> child_start, child_list;   // children in index order
    std::vector<int32_t> sphere_start;               // per-link CSR into spheres
    std::vector<float> sphere_x, sphere_z, sphere_r;
    std::vector<int32_t> sphere_link;                // per CSR slot
    // joints (dof = nrd + j)
    std::vector<float> joint_damping;
    std::vector<double> joint_lo, joint_hi;
    std::vector<int32_t> joint_slot_start;           // nj+1: pair slots grouped by joint
    // muscles
    std::vector<float> m_fmax, m_ndt_act, m_ndt_deact, m_pw;
    // fibre-length chain kept in f64: v_m = (L - prev_len)/(dt l_opt v_max)
    // amplifies length error by ~1/(dt l_opt v_max) (SURVEY.md §7 hard part 1)
    std::vector<double> m_lopt, m_inv_lopt, m_slack, m_kv;
    std::vector<int32_t> m_via_start, m_pair_start, m_seg_start;
    std::vector<int32_t> via_link;
    std::vector<float> via_x, via_z;
    // Path segments (via k-1 -> k).  Most segments join a link and its parent
    // ("adjacent"): their length, direction and moment arm about the child's
    // joint are evaluated in the parent's frame from constants and the joint's
    // own rotation only, so no world coordinates (and no large-magnitude fp32
    // cancellation) enter the fibre length.  seg_info = kind | dof << 8 with
    // kind 0 = same link (constant length in seg_ax), 1 = adjacent
    // (seg_ax/az = anchor - parent-side offset, seg_cx/cz = child-side offset,
    // seg_slot = torque slot of the child joint), 2 = general (world frame,
    // pairs in pair_*; seg_slot = global via index of the segment end).
    std::vector<int32_t> seg_info, seg_slot;
    std::vector<float> seg_ax, seg_az, seg_cx, seg_cz;
    // pairs of general segments: joint, end via, slot, sign
    std::vector<int32_t> pair_joint, pair_via, pair_slot;  // pair_via: global via index of segment END
    std::vector<float> pair_sign;                          // +1: endpoint = seg start, -1: seg end
    std::vector<int32_t> key_bodies;

    // ---- packed device layout (what the step kernel reads) ----
    // per muscle: p0 = {f_max, -dt/tau_act, -dt/tau_deact, l_opt v_max / 10} (f32x4),
    // p1 = {slack, l_opt, 1/l_opt, 1/(dt l_opt v_max)} (f64x4), meta = nseg | general << 8 | m_ext << 9.
    // Segment k of muscle m lives at [k * nm + m] so a warp's 32 muscles read
    // 32 consecutive records (coalesced): geo = {ax, az, cx, cz},
    // info = kind | dof << 2 | slot << 11 (kind 2: slot = global via index of the end).
    int max_seg = 0, has_general = 0;
    int n_fast = 0, max_seg_fast = 0;  // muscles without a general segment (device order [0, n_fast)), their max nseg
    // internal muscle order (general muscles last, then by segment count): m_ext[i] = reference
    // index of internal muscle i, m_int = its inverse; pk_meta carries m_ext << 9
    std::vector<int32_t> m_ext, m_int;
    std::vector<float> pk_p0, pk_geo;
    std::vector<double> pk_p1;
    std::vector<int32_t> pk_meta, pk_info;
};

CompiledModel compile_model(const ModelSpec& spec);

}  // namespace msk_b200
