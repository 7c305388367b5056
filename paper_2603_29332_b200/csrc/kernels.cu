// sm_100a kernels of the batched env-stepper.
//
// One warp owns one environment for a whole control step: the 10 substeps
// of msk::step (skeleton.cpp:286-331) run on-chip, with per-env scratch in
// shared memory and nothing but the step's inputs/outputs touching HBM.
//
// Per substep (lane-parallel phases separated by __syncwarp):
//   1. FK, root-relative, level by level over the tree      (skeleton.cpp:82-107)
//   2. muscles: activation ODE, via-point path length, fibre
//      kinematics, Hill force, and the J_m^T F contributions of
//      every segment/joint pair into a per-env slot table   (muscle.cpp:9-56, skeleton.cpp:129-170, 298-315)
//   3. joint torques: fixed-order sum of each joint's slots,
//      minus damping and joint-limit penalty                (skeleton.cpp:222-231)
//   4. velocity kinematics                                   (skeleton.cpp:43-72)
//   5. articulated-body recursion for q̈ = M^{-1}(τ + J^T f_ext − C):
//      per-link spatial inertia + bias + gravity + contact, a
//      leaf-to-root pass and a root-to-leaf pass (the tree-sparse
//      L^T D L factor/solve of M; no n_q x n_q matrix is formed)
//                                                             (skeleton.cpp:172-262, 316-317)
//   6. semi-implicit Euler in f64 + divergence check         (skeleton.cpp:319-328)
// then the env epilogue: Δ, observation, reward_aux, termination, episode
// outcome (env.cpp:129-263).  Reductions use fixed orders (no float atomics),
// so a step is bit-reproducible.
#include <cuda_runtime.h>

#include <cstdint>

#include "device.cuh"

namespace msk_b200 {

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr float kTwoPiHi = 6.28318548202514648f;       // float(2*pi)
constexpr float kTwoPiLo = -1.74845553e-7f;            // 2*pi - float(2*pi)
constexpr float kInvTwoPi = 0.159154943091895336f;
constexpr double kPi = 3.14159265358979323846;

struct EnvSmem {
    float4* kin;    // nl: cos, sin, origin x, origin z (root-relative)
    float* theta;   // nl: link angle reduced to ~(-pi, pi]
    float* qang;    // nq: float(mount + q) per joint dof; reduced root pitch at [2]
    float* dqf;     // nq
    float* tau;     // nq: joint torque, then q̈
    float* un;      // union: pair slots | 16 floats per link (ABA)
    float* root;    // [0] root x, [1] root z (absolute, floating base only)
    float2* relcs;  // nq: cos, sin of each joint's own rotation (mount + q), from f64
};

__device__ __forceinline__ EnvSmem carve(unsigned char* base, const DevModel& M) {
    EnvSmem s;
    s.kin = reinterpret_cast<float4*>(base);
    s.theta = reinterpret_cast<float*>(base + M.off_theta);
    s.qang = reinterpret_cast<float*>(base + M.off_qang);
    s.dqf = reinterpret_cast<float*>(base + M.off_dqf);
    s.tau = reinterpret_cast<float*>(base + M.off_tau);
    s.un = reinterpret_cast<float*>(base + M.off_union);
    s.root = reinterpret_cast<float*>(base + M.off_root);
    s.relcs = reinterpret_cast<float2*>(base + M.off_relcs);
    return s;
}

__device__ __forceinline__ float reduce_angle(float a) {
    const float k = rintf(a * kInvTwoPi);
    return fmaf(-k, kTwoPiLo, fmaf(-k, kTwoPiHi, a));
}

__device__ __forceinline__ float reduce_angle_d(double a) {
    return static_cast<float>(a - 2.0 * kPi * rint(a * (0.5 / kPi)));
}

// ---- Hill-type muscle (muscle.cpp:9-40) -----------------------------------
__device__ __forceinline__ float hill_fl(float l) {
    const float d = (l - 1.0f) * (1.0f / 0.45f);
    return expf(-d * d);
}
__device__ __forceinline__ float hill_fv(float v) {
    if (v <= -1.0f) return 0.0f;
    if (v < 0.0f) return (v + 1.0f) / (1.0f - v * 0.25f);
    constexpr float c = 0.32f;  // (1.4 - 1) / (1 + 1/4)
    return (1.4f * v + c) / (v + c);
}
__device__ __forceinline__ float hill_fp(float l) {
    if (l <= 1.0f) return 0.0f;
    return (expf(4.0f * (l - 1.0f)) - 1.0f) * (1.0f / 6.38905609893065f);
}
__device__ __forceinline__ float mtu_force(float act, float l, float v, float fmax) {
    return fmax * (act * hill_fl(l) * hill_fv(v) + hill_fp(l));
}

// World (root-relative) position of a via point.
__device__ __forceinline__ float2 via_point(const DevModel& M, const float4* kin, int v) {
    const int l = __ldg(M.via_link + v);
    const float x = __ldg(M.via_x + v), z = __ldg(M.via_z + v);
    if (l < 0) return make_float2(x, z);
    const float4 k = kin[l];
    return make_float2(fmaf(k.x, x, fmaf(-k.y, z, k.z)), fmaf(k.y, x, fmaf(k.x, z, k.w)));
}

// Per-DOF float views (joint angle incl. mount, velocity) for the tree passes.
__device__ __forceinline__ void publish_dofs(const DevModel& M, const EnvSmem& S, const double* qd,
                                             const double* dqd, int lane) {
#pragma unroll
    for (int k = 0; k < kMaxQSlots; ++k) {
        const int d = lane + 32 * k;
        if (d < M.nq) {
            float a;
            if (d >= M.nrd) {
                const int l = M.floating + (d - M.nrd);
                const double rel = __ldg(M.link_mount + l) + qd[k];
                a = static_cast<float>(rel);
                double sn, cs;
                sincos(rel, &sn, &cs);
                S.relcs[d] = make_float2(static_cast<float>(cs), static_cast<float>(sn));
            } else if (d == 2) {
                a = reduce_angle_d(qd[k]);
            } else {
                a = 0.0f;
                S.root[d] = static_cast<float>(qd[k]);
            }
            S.qang[d] = a;
            S.dqf[d] = static_cast<float>(dqd[k]);
        }
    }
}

// Forward kinematics level by level (skeleton.cpp:82-107), root-relative.
__device__ __forceinline__ void fk_pass(const DevModel& M, const EnvSmem& S, int lane) {
    for (int lev = 0; lev < M.n_levels; ++lev) {
        const int b = __ldg(M.level_start + lev), n = __ldg(M.level_start + lev + 1) - b;
        for (int i = lane; i < n; i += 32) {
            const int l = __ldg(M.level_links + b + i);
            const int dof = __ldg(M.link_dof + l);
            float th, ox, oz;
            if (dof < 0) {  // floating root: origin at (0,0) relative, pitch q2
                th = S.qang[2];
                ox = 0.0f;
                oz = 0.0f;
            } else {
                const int p = __ldg(M.link_parent + l);
                const float ax = __ldg(M.link_ax + l), az = __ldg(M.link_az + l);
                if (p >= 0) {
                    const float4 kp = S.kin[p];
                    ox = fmaf(kp.x, ax, fmaf(-kp.y, az, kp.z));
                    oz = fmaf(kp.y, ax, fmaf(kp.x, az, kp.w));
                    th = reduce_angle(S.theta[p] + S.qang[dof]);
                } else {
                    ox = ax;
                    oz = az;
                    th = reduce_angle(S.qang[dof]);
                }
            }
            float sn, cs;
            sincosf(th, &sn, &cs);
            S.theta[l] = th;
            S.kin[l] = make_float4(cs, sn, ox, oz);
        }
        __syncwarp();
    }
}

// Velocity kinematics (skeleton.cpp:43-72): per link (omega, v_origin) into un[16 l + 0..2].
__device__ __forceinline__ void vel_pass(const DevModel& M, const EnvSmem& S, int lane) {
    for (int lev = 0; lev < M.n_levels; ++lev) {
        const int b = __ldg(M.level_start + lev), n = __ldg(M.level_start + lev + 1) - b;
        for (int i = lane; i < n; i += 32) {
            const int l = __ldg(M.level_links + b + i);
            const int dof = __ldg(M.link_dof + l);
            float w, vx, vz;
            if (dof < 0) {
                w = S.dqf[2];
                vx = S.dqf[0];
                vz = S.dqf[1];
            } else {
                const int p = __ldg(M.link_parent + l);
                if (p >= 0) {
                    const float* up = S.un + 16 * p;
                    const float wp = up[0];
                    const float4 kl = S.kin[l], kp = S.kin[p];
                    const float rx = kl.z - kp.z, rz = kl.w - kp.w;
                    vx = fmaf(-wp, rz, up[1]);
                    vz = fmaf(wp, rx, up[2]);
                    w = wp + S.dqf[dof];
                } else {
                    vx = 0.0f;
                    vz = 0.0f;
                    w = S.dqf[dof];
                }
            }
            float* u = S.un + 16 * l;
            u[0] = w;
            u[1] = vx;
            u[2] = vz;
        }
        __syncwarp();
    }
}

// Path length of muscle m (skeleton.cpp:129-141), segment by segment.  Adjacent
// segments are evaluated in the parent's frame from the joint's own rotation.
__device__ __forceinline__ float muscle_length(const DevModel& M, const EnvSmem& S, int m) {
    const int s0 = __ldg(M.m_seg_start + m), s1 = __ldg(M.m_seg_start + m + 1);
    float L = 0.0f;
    for (int s = s0; s < s1; ++s) {
        const int info = __ldg(M.seg_info + s), kind = info & 3;
        if (kind == 0) {
            L += __ldg(M.seg_ax + s);
        } else if (kind == 1) {
            const float2 cs = S.relcs[info >> 8];
            const float cx = __ldg(M.seg_cx + s), cz = __ldg(M.seg_cz + s);
            const float sx = fmaf(cs.x, cx, fmaf(-cs.y, cz, __ldg(M.seg_ax + s)));
            const float sz = fmaf(cs.y, cx, fmaf(cs.x, cz, __ldg(M.seg_az + s)));
            L += sqrtf(fmaf(sx, sx, sz * sz));
        } else {
            const int v = __ldg(M.seg_slot + s);
            const float2 pe = via_point(M, S.kin, v), ps = via_point(M, S.kin, v - 1);
            const float dx = pe.x - ps.x, dz = pe.y - ps.y;
            L += sqrtf(fmaf(dx, dx, dz * dz));
        }
    }
    return L;
}

// J_m^T F contributions of muscle m (force F) into the per-env slot table:
// -F * dL_i/dq_j for every joint j between a segment's two links
// (skeleton.cpp:147-170 with the GEMV of :315 folded in).
__device__ __forceinline__ void muscle_torques(const DevModel& M, const EnvSmem& S, int m, float F) {
    const int s0 = __ldg(M.m_seg_start + m), s1 = __ldg(M.m_seg_start + m + 1);
    for (int s = s0; s < s1; ++s) {
        const int info = __ldg(M.seg_info + s);
        if ((info & 3) != 1) continue;
        const float2 cs = S.relcs[info >> 8];
        const float cx = __ldg(M.seg_cx + s), cz = __ldg(M.seg_cz + s);
        const float ax = __ldg(M.seg_ax + s), az = __ldg(M.seg_az + s);
        const float rx = fmaf(cs.x, cx, -cs.y * cz), rz = fmaf(cs.y, cx, cs.x * cz);
        const float sx = ax + rx, sz = az + rz;
        const float len = sqrtf(fmaf(sx, sx, sz * sz));
        // moment about the child's joint: -F (r x A) / |A + r|, r = child-side
        // offset rotated into the parent frame, A = anchor - parent-side offset
        const float val = len > 1e-12f ? -F * fmaf(rx, az, -rz * ax) / len : 0.0f;
        S.un[__ldg(M.seg_slot + s)] = val;
    }
    const int p0 = __ldg(M.m_pair_start + m), p1 = __ldg(M.m_pair_start + m + 1);
    for (int p = p0; p < p1; ++p) {  // general (non-adjacent) segments, world frame
        const int ve = __ldg(M.pair_via + p), j = __ldg(M.pair_joint + p);
        const float sg = __ldg(M.pair_sign + p);
        const float2 pe = via_point(M, S.kin, ve);
        const float2 ps = via_point(M, S.kin, ve - 1);
        const float sx = pe.x - ps.x, sz = pe.y - ps.y;
        const float len = sqrtf(fmaf(sx, sx, sz * sz));
        float val = 0.0f;
        if (len > 1e-12f) {
            const float inv = 1.0f / len;
            const float ux = sx * inv, uz = sz * inv;
            const float4 ka = S.kin[M.floating + j];
            const float2 pt = sg < 0.0f ? pe : ps;
            const float rx = pt.x - ka.z, rz = pt.y - ka.w;
            val = sg * F * fmaf(rx, uz, -rz * ux);
        }
        S.un[__ldg(M.pair_slot + p)] = val;
    }
}

// Key-body COM (absolute) and unreduced frame angle (skeleton.cpp:346-357).
__device__ __forceinline__ void key_body(const DevModel& M, const EnvSmem& S, const double* qsm, int k,
                                         double& x, double& z, double& ang) {
    const int l = __ldg(M.key_bodies + k);
    const float4 kl = S.kin[l];
    const float c = __ldg(M.link_com + l);
    x = static_cast<double>(fmaf(kl.x, c, kl.z));
    z = static_cast<double>(fmaf(kl.y, c, kl.w));
    double a = 0.0;
    int cur = l;
    while (cur >= 0) {
        const int dof = __ldg(M.link_dof + cur);
        if (dof < 0) {
            a += qsm[2];
            break;
        }
        a += __ldg(M.link_mount + cur) + qsm[dof];
        cur = __ldg(M.link_parent + cur);
    }
    ang = a;
    if (M.floating) {
        x += qsm[0];
        z += qsm[1];
    }
}

__device__ double wrap_angle(double a) {  // env.cpp:10-15
    a = fmod(a + kPi, 2.0 * kPi);
    if (a <= 0.0) a += 2.0 * kPi;
    return a - kPi;
}

__device__ __forceinline__ int phase_bin(const DevModel& M, int frame) {  // env.cpp:89-93
    const int usable = max(1, M.frames - 1);
    const int b = static_cast<int>(static_cast<long long>(frame) * M.bins / usable);
    return min(b, M.bins - 1);
}

// Env::observe (env.cpp:129-163) for one env; qsm = f64 q in smem, dq from global.
__device__ void write_obs(const DevModel& M, const DevState& St, const EnvSmem& S, const double* qsm, int e,
                          int t_index, float* obs_row, int lane) {
    const int nq = M.nq, nm = M.nm, nk = M.nk;
    int o = 0;
    for (int i = lane; i < nq; i += 32) obs_row[o + i] = static_cast<float>(qsm[i]);
    o += nq;
    for (int i = lane; i < nq; i += 32) obs_row[o + i] = static_cast<float>(St.dq[static_cast<size_t>(e) * nq + i]);
    o += nq;
    for (int k = lane; k < nk; k += 32) {
        double x, z, a;
        key_body(M, S, qsm, k, x, z, a);
        obs_row[o + 2 * k] = static_cast<float>(x);
        obs_row[o + 2 * k + 1] = static_cast<float>(z);
        obs_row[o + 2 * nk + k] = static_cast<float>(a);
    }
    o += 3 * nk;
    const size_t mb = static_cast<size_t>(e) * nm;
    for (int i = lane; i < nm; i += 32) {
        obs_row[o + i] = St.act[mb + i];
        obs_row[o + nm + i] = St.fm[mb + i];
        obs_row[o + 2 * nm + i] = St.lm[mb + i];
        obs_row[o + 3 * nm + i] = St.vm[mb + i];
    }
    o += 4 * nm;
    const size_t t = static_cast<size_t>(t_index);
    for (int i = lane; i < nq; i += 32) obs_row[o + i] = static_cast<float>(M.clip_q[t * nq + i]);
    o += nq;
    for (int i = lane; i < 2 * nk; i += 32) obs_row[o + i] = static_cast<float>(M.clip_kp[t * 2 * nk + i]);
    o += 2 * nk;
    for (int i = lane; i < nk; i += 32) obs_row[o + i] = static_cast<float>(M.clip_ka[t * nk + i]);
}

// Env::tracking_error (env.cpp:170-193) -> Δ row (f64 values rounded once).
// Returns (via shuffle-OR) whether any key body exceeds the termination radius.
__device__ bool write_delta(const DevModel& M, const EnvSmem& S, const double* qsm, int t_index, float* drow,
                            int lane) {
    const int nq = M.nq, nj = M.nj, nk = M.nk, nrd = M.nrd;
    const size_t t = static_cast<size_t>(t_index);
    if (lane < 3) {
        double v = 0.0;
        if (M.floating) {
            const double d = qsm[lane] - M.clip_q[t * nq + lane];
            v = lane == 2 ? wrap_angle(d) : d;
        }
        if (drow) drow[lane] = static_cast<float>(v);
    }
    if (drow)
        for (int j = lane; j < nj; j += 32)
            drow[3 + j] = static_cast<float>(qsm[nrd + j] - M.clip_q[t * nq + nrd + j]);
    bool far = false;
    for (int k = lane; k < nk; k += 32) {
        double x, z, a;
        key_body(M, S, qsm, k, x, z, a);
        const double dx = x - M.clip_kp[t * 2 * nk + 2 * k];
        const double dz = z - M.clip_kp[t * 2 * nk + 2 * k + 1];
        if (drow) {
            drow[3 + nj + 2 * k] = static_cast<float>(dx);
            drow[3 + nj + 2 * k + 1] = static_cast<float>(dz);
        }
        if (sqrt(dx * dx + dz * dz) > M.term_err) far = true;
    }
    return __any_sync(kFull, far);
}

// make_initial_state (skeleton.cpp:264-284) for the env's muscles, given FK in smem.
__device__ void init_muscles(const DevModel& M, const DevState& St, const EnvSmem& S, int e, int lane) {
    const size_t mb = static_cast<size_t>(e) * M.nm;
    const float a0 = static_cast<float>(M.init_act);
    for (int m = lane; m < M.nm; m += 32) {
        const float L = muscle_length(M, S, m);
        const float lm = fmaxf((L - __ldg(M.m_slack + m)) * __ldg(M.m_inv_lopt + m), kMinFiber);
        St.act[mb + m] = a0;
        St.lm[mb + m] = lm;
        St.vm[mb + m] = 0.0f;
        St.fm[mb + m] = mtu_force(a0, lm, 0.0f, __ldg(M.m_fmax + m));
    }
}

// mt19937_64 (rng.hpp:71) — state in global memory, one thread.
__device__ uint64_t mt_next(uint64_t* mt, int* mti) {
    constexpr uint64_t kUM = 0xFFFFFFFF80000000ULL, kLM = 0x7FFFFFFFULL, kA = 0xB5026F5AA96619E9ULL;
    if (*mti >= 312) {
        for (int i = 0; i < 312; ++i) {
            const uint64_t x = (mt[i] & kUM) | (mt[(i + 1) % 312] & kLM);
            uint64_t y = x >> 1;
            if (x & 1ULL) y ^= kA;
            mt[i] = mt[(i + 156) % 312] ^ y;
        }
        *mti = 0;
    }
    uint64_t x = mt[(*mti)++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= (x >> 43);
    return x;
}

// Env::reset frame choice with RSI (env.cpp:108-121 + AdaptiveSampler, env.cpp:39-57).
// Strict IEEE f64 (no contraction) so the sampled bin is bit-exact.
__device__ int rsi_frame(const DevModel& M, const DevState& St, int e) {
    const int bins = M.bins;
    const double* ema = St.ema + static_cast<size_t>(e) * bins;
    uint64_t* mt = St.mt + static_cast<size_t>(e) * 312;
    int* mti = St.mti + e;
    double total = 0.0;
    for (int b = 0; b < bins; ++b) total = __dadd_rn(total, ema[b]);
    const double base = __ddiv_rn(M.mix, static_cast<double>(bins));
    double u = __dmul_rn(static_cast<double>(mt_next(mt, mti) >> 11), 0x1.0p-53);
    int bin = bins - 1;
    for (int b = 0; b < bins; ++b) {
        double p;
        if (total > 1e-12)
            p = __dadd_rn(base, __ddiv_rn(__dmul_rn(__dsub_rn(1.0, M.mix), ema[b]), total));
        else
            p = __dadd_rn(base, __ddiv_rn(__dsub_rn(1.0, M.mix), static_cast<double>(bins)));
        u = __dsub_rn(u, p);
        if (u <= 0.0) {
            bin = b;
            break;
        }
    }
    const int usable = M.frames - 1;
    const long long lo = static_cast<long long>(bin) * usable / bins;
    long long hi = static_cast<long long>(bin + 1) * usable / bins;
    if (hi <= lo) hi = lo + 1;
    const uint64_t r = mt_next(mt, mti) % static_cast<uint64_t>(hi - lo);
    int frame = static_cast<int>(lo + static_cast<long long>(r));
    return min(frame, usable - 1);
}

}  // namespace

// ============================================================================
// step kernel: warp per env, WPB envs per block
// ============================================================================
template <int WPB>
__global__ void __launch_bounds__(WPB * 32) step_kernel(DevModel M, DevState St, int env0, int n_envs,
                                                        const float* __restrict__ actions, float* obs,
                                                        float* delta, float* reward_aux, uint8_t* flags,
                                                        float* power, float* grf) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int le = blockIdx.x * WPB + warp;  // env index local to this launch
    if (le >= n_envs) return;
    const int e = env0 + le;
    const EnvSmem S = carve(smem + warp * M.smem_env_bytes, M);
    const int nq = M.nq, nm = M.nm, nl = M.nl, nrd = M.nrd;
    const size_t mb = static_cast<size_t>(e) * nm;
    const float* act_row = actions + static_cast<size_t>(le) * nm;

    // Contract checks of Env::step (env.cpp:207-210): env untouched on failure.
    if (St.done[e]) {
        if (lane == 0 && flags) flags[le] = kFlagNotStepped;
        return;
    }
    {
        bool bad = false;
        for (int m = lane; m < nm; m += 32) bad |= !isfinite(act_row[m]);
        if (__any_sync(kFull, bad)) {
            if (lane == 0 && flags) flags[le] = kFlagBadAction;
            return;
        }
    }

    double qd[kMaxQSlots], dqd[kMaxQSlots];
#pragma unroll
    for (int k = 0; k < kMaxQSlots; ++k) {
        const int d = lane + 32 * k;
        qd[k] = d < nq ? St.q[static_cast<size_t>(e) * nq + d] : 0.0;
        dqd[k] = d < nq ? St.dq[static_cast<size_t>(e) * nq + d] : 0.0;
    }
    publish_dofs(M, S, qd, dqd, lane);
    float grf_acc[kMaxLinkSlots][2];
#pragma unroll
    for (int k = 0; k < kMaxLinkSlots; ++k) grf_acc[k][0] = grf_acc[k][1] = 0.0f;
    float* pw = power ? power + static_cast<size_t>(le) * nm
                      : (M.reward_mode == 2 ? St.power_scratch + mb : nullptr);
    if (pw)
        for (int m = lane; m < nm; m += 32) pw[m] = 0.0f;
    __syncwarp();

    const float dt = static_cast<float>(kSimDt);
    int diverged_at = -1;
    for (int sub = 0; sub < kSubsteps; ++sub) {
        // ---- 1. forward kinematics ----
        fk_pass(M, S, lane);

        // ---- 2. muscles + J_m^T F pair contributions ----
        for (int m = lane; m < nm; m += 32) {
            const float u = fminf(fmaxf(act_row[m], 0.0f), 1.0f);
            const float a0 = St.act[mb + m];
            const float lm0 = St.lm[mb + m];
            // activation_step (muscle.cpp:42-56), tau frozen at the step start
            const float gain = fmaf(1.5f, a0, 0.5f);
            const float ex = u > a0 ? expf(__ldg(M.m_ndt_act + m) / gain) : expf(__ldg(M.m_ndt_deact + m) * gain);
            const float a1 = fminf(fmaxf(fmaf(a0 - u, ex, u), 0.0f), 1.0f);
            const float slack = __ldg(M.m_slack + m), lopt = __ldg(M.m_lopt + m);
            const float prev_len = fmaf(lm0, lopt, slack);
            const float L = muscle_length(M, S, m);
            const float vm = (L - prev_len) * __ldg(M.m_kv + m);
            const float lm1 = fmaxf((L - slack) * __ldg(M.m_inv_lopt + m), kMinFiber);
            const float F = mtu_force(a1, lm1, vm, __ldg(M.m_fmax + m));
            St.act[mb + m] = a1;
            St.lm[mb + m] = lm1;
            St.vm[mb + m] = vm;
            St.fm[mb + m] = F;
            if (pw) pw[m] += fabsf(F * vm * __ldg(M.m_pw + m));
            muscle_torques(M, S, m, F);
        }
        __syncwarp();

        // ---- 3. joint torques: fixed-order slot sums, damping, limits ----
#pragma unroll
        for (int k = 0; k < kMaxQSlots; ++k) {
            const int d = lane + 32 * k;
            if (d >= nrd && d < nq) {
                const int j = d - nrd;
                const int s0 = __ldg(M.joint_slot_start + j), s1 = __ldg(M.joint_slot_start + j + 1);
                float t = 0.0f;
                for (int s = s0; s < s1; ++s) t += S.un[s];
                t -= __ldg(M.joint_damping + j) * static_cast<float>(dqd[k]);
                const double hi = __ldg(M.joint_hi + j), lo = __ldg(M.joint_lo + j);
                if (qd[k] > hi)
                    t -= static_cast<float>(M.k_lim_d * (qd[k] - hi));
                else if (qd[k] < lo)
                    t -= static_cast<float>(M.k_lim_d * (qd[k] - lo));
                S.tau[d] = t;
            }
        }
        __syncwarp();

        // ---- 4. velocities ----
        vel_pass(M, S, lane);

        // ---- 5a. per-link spatial inertia, bias force, gravity, contact ----
#pragma unroll
        for (int k = 0; k < kMaxLinkSlots; ++k) {
            const int l = lane + 32 * k;
            if (l < nl) {
                float* u = S.un + 16 * l;
                const float w = u[0], vx = u[1], vz = u[2];
                const float4 kl = S.kin[l];
                const float m = __ldg(M.link_mass + l), I = __ldg(M.link_inertia + l);
                const float cc = __ldg(M.link_com + l);
                const float cx = cc * kl.x, cz = cc * kl.y;
                const float i00 = fmaf(m, fmaf(cx, cx, cz * cz), I), i01 = -m * cz, i02 = m * cx;
                // h = I V ; p = V x* h
                const float h1 = fmaf(i01, w, m * vx), h2 = fmaf(i02, w, m * vz);
                float p0 = fmaf(vx, h2, -vz * h1), p1 = -w * h2, p2 = w * h1;
                // gravity at the COM: f = (c x F, 0, m g)
                const float mg = m * M.gravity;
                p0 -= cx * mg;
                p2 -= mg;
                // contact spheres on this link (skeleton.cpp:235-262)
                const int s0 = __ldg(M.sphere_start + l), s1 = __ldg(M.sphere_start + l + 1);
                for (int s = s0; s < s1; ++s) {
                    const float ox = __ldg(M.sphere_x + s), oz = __ldg(M.sphere_z + s), r = __ldg(M.sphere_r + s);
                    const float rx = fmaf(kl.x, ox, -kl.y * oz), rz = fmaf(kl.y, ox, kl.x * oz);
                    const float cz_abs = kl.w + rz + (M.floating ? S.root[1] : 0.0f);
                    const float pen = r - cz_abs;
                    float fx = 0.0f, fz = 0.0f;
                    if (pen > 0.0f) {
                        const float vcz = fmaf(w, rx, vz);
                        const float fn = fmaxf(0.0f, fmaf(M.c_k, pen, -M.c_c * vcz));
                        if (fn > 0.0f) {
                            const float qz = rz - r;  // contact point relative to the link origin
                            const float vcx = fmaf(-w, qz, vx);
                            const float ft = -M.c_mu * fn * tanhf(vcx * M.inv_c_vs);
                            fx = ft;
                            fz = fn;
                            p0 -= fmaf(rx, fn, -qz * ft);
                            p1 -= ft;
                            p2 -= fn;
                        }
                    }
                    grf_acc[k][0] += fx * 0.1f;
                    grf_acc[k][1] += fz * 0.1f;
                }
                const int dof = __ldg(M.link_dof + l);
                float c1 = 0.0f, c2 = 0.0f;
                if (dof >= 0) {
                    const float qdot = S.dqf[dof];
                    c1 = qdot * vz;
                    c2 = -qdot * vx;
                }
                u[0] = i00;
                u[1] = i01;
                u[2] = i02;
                u[3] = m;
                u[4] = 0.0f;
                u[5] = m;
                u[6] = p0;
                u[7] = p1;
                u[8] = p2;
                u[14] = c1;
                u[15] = c2;
            }
        }
        __syncwarp();

        // ---- 5b. articulated-body pass, leaves -> root ----
        for (int lev = M.n_levels - 1; lev >= 0; --lev) {
            const int b = __ldg(M.level_start + lev), n = __ldg(M.level_start + lev + 1) - b;
            for (int i = lane; i < n; i += 32) {
                const int l = __ldg(M.level_links + b + i);
                float* u = S.un + 16 * l;
                float I00 = u[0], I01 = u[1], I02 = u[2], I11 = u[3], I12 = u[4], I22 = u[5];
                float P0 = u[6], P1 = u[7], P2 = u[8];
                const int c0 = __ldg(M.child_start + l), c1 = __ldg(M.child_start + l + 1);
                for (int c = c0; c < c1; ++c) {
                    const float* uc = S.un + 16 * __ldg(M.child_list + c);
                    I00 += uc[0];
                    I01 += uc[1];
                    I02 += uc[2];
                    I11 += uc[3];
                    I12 += uc[4];
                    I22 += uc[5];
                    P0 += uc[6];
                    P1 += uc[7];
                    P2 += uc[8];
                }
                const int dof = __ldg(M.link_dof + l);
                if (dof < 0) {  // floating root keeps its full articulated inertia
                    u[0] = I00; u[1] = I01; u[2] = I02; u[3] = I11; u[4] = I12; u[5] = I22;
                    u[6] = P0; u[7] = P1; u[8] = P2;
                    continue;
                }
                const float invD = 1.0f / I00;
                const float uu = S.tau[dof] - P0;
                // Ia = IA - U U^T / D (first row/column vanish)
                const float a = I11 - I01 * I01 * invD;
                const float bb = I12 - I01 * I02 * invD;
                const float cq = I22 - I02 * I02 * invD;
                const float c1v = u[14], c2v = u[15];
                const float k = uu * invD;
                const float q0 = S.tau[dof];                       // P0 + U0 * u / D
                const float q1 = fmaf(I01, k, fmaf(a, c1v, fmaf(bb, c2v, P1)));
                const float q2 = fmaf(I02, k, fmaf(bb, c1v, fmaf(cq, c2v, P2)));
                u[9] = I00;
                u[10] = I01;
                u[11] = I02;
                u[12] = invD;
                u[13] = uu;
                const int p = __ldg(M.link_parent + l);
                if (p >= 0) {  // shift to the parent's origin: X^T Ia X, X^T pa
                    const float4 kl = S.kin[l], kp = S.kin[p];
                    const float dx = kl.z - kp.z, dz = kl.w - kp.w;
                    const float al = fmaf(-a, dz, bb * dx), be = fmaf(-bb, dz, cq * dx);
                    u[0] = fmaf(-dz, al, be * dx);
                    u[1] = al;
                    u[2] = be;
                    u[3] = a;
                    u[4] = bb;
                    u[5] = cq;
                    u[6] = fmaf(-dz, q1, fmaf(dx, q2, q0));
                    u[7] = q1;
                    u[8] = q2;
                }
            }
            __syncwarp();
        }

        // ---- 5c. root solve + articulated-body pass, root -> leaves ----
        if (M.floating && lane == 0) {
            float* u = S.un;  // link 0
            // solve IA A = -pA (3x3 SPD, Cholesky)
            const float l00 = sqrtf(u[0]);
            const float l10 = u[1] / l00, l20 = u[2] / l00;
            const float l11 = sqrtf(u[3] - l10 * l10);
            const float l21 = (u[4] - l20 * l10) / l11;
            const float l22 = sqrtf(u[5] - l20 * l20 - l21 * l21);
            const float y0 = -u[6] / l00;
            const float y1 = (-u[7] - l10 * y0) / l11;
            const float y2 = (-u[8] - l20 * y0 - l21 * y1) / l22;
            const float x2 = y2 / l22;
            const float x1 = (y1 - l21 * x2) / l11;
            const float x0 = (y0 - l10 * x1 - l20 * x2) / l00;
            u[0] = x0;
            u[1] = x1;
            u[2] = x2;
            const float wd = S.dqf[2];
            S.tau[0] = x1 - wd * S.dqf[1];
            S.tau[1] = x2 + wd * S.dqf[0];
            S.tau[2] = x0;
        }
        __syncwarp();
        for (int lev = 0; lev < M.n_levels; ++lev) {
            const int b = __ldg(M.level_start + lev), n = __ldg(M.level_start + lev + 1) - b;
            for (int i = lane; i < n; i += 32) {
                const int l = __ldg(M.level_links + b + i);
                const int dof = __ldg(M.link_dof + l);
                if (dof < 0) continue;
                float* u = S.un + 16 * l;
                const int p = __ldg(M.link_parent + l);
                float A0 = 0.0f, A1 = u[14], A2 = u[15];
                if (p >= 0) {
                    const float* up = S.un + 16 * p;
                    const float4 kl = S.kin[l], kp = S.kin[p];
                    const float dx = kl.z - kp.z, dz = kl.w - kp.w;
                    A0 = up[0];
                    A1 += fmaf(-up[0], dz, up[1]);
                    A2 += fmaf(up[0], dx, up[2]);
                }
                const float qdd = (u[13] - fmaf(u[9], A0, fmaf(u[10], A1, u[11] * A2))) * u[12];
                u[0] = A0 + qdd;
                u[1] = A1;
                u[2] = A2;
                S.tau[dof] = qdd;
            }
            __syncwarp();
        }

        // ---- 6. semi-implicit Euler (f64) + divergence check ----
        bool bad = false;
#pragma unroll
        for (int k = 0; k < kMaxQSlots; ++k) {
            const int d = lane + 32 * k;
            if (d < nq) {
                dqd[k] += static_cast<double>(S.tau[d]) * kSimDt;
                qd[k] += dqd[k] * kSimDt;
                bad |= !isfinite(qd[k]) || !isfinite(dqd[k]);
            }
        }
        __syncwarp();
        publish_dofs(M, S, qd, dqd, lane);
        __syncwarp();
        if (__any_sync(kFull, bad)) {
            diverged_at = sub;
            break;
        }
    }
    (void)dt;

    // ---- write back the simulation state ----
#pragma unroll
    for (int k = 0; k < kMaxQSlots; ++k) {
        const int d = lane + 32 * k;
        if (d < nq) {
            St.q[static_cast<size_t>(e) * nq + d] = qd[k];
            St.dq[static_cast<size_t>(e) * nq + d] = dqd[k];
        }
    }
    const int n_sub = diverged_at >= 0 ? diverged_at + 1 : kSubsteps;
    if (lane == 0) {
        double t = St.t[e];
        for (int s = 0; s < n_sub; ++s) t += kSimDt;
        St.t[e] = t;
    }
    const int obs_dim = 3 * nq + 6 * M.nk + 4 * nm;
    const int ddim = 3 + M.nj + 2 * M.nk;
    float* obs_row = obs ? obs + static_cast<size_t>(le) * obs_dim : nullptr;
    float* drow = delta ? delta + static_cast<size_t>(le) * ddim : nullptr;

    if (diverged_at >= 0) {  // env.cpp:214-229
        if (obs_row)
            for (int i = lane; i < obs_dim; i += 32) obs_row[i] = 0.0f;
        if (drow)
            for (int i = lane; i < ddim; i += 32) drow[i] = 0.0f;
        if (power)
            for (int m = lane; m < nm; m += 32) power[static_cast<size_t>(le) * nm + m] = 0.0f;
        if (grf)
            for (int i = lane; i < 2 * nl; i += 32) grf[static_cast<size_t>(le) * 2 * nl + i] = 0.0f;
        if (lane == 0) {
            if (reward_aux) reward_aux[le] = 0.0f;
            if (flags) flags[le] = kFlagDone | kFlagFailed | kFlagDiverged;
            St.done[e] = 1;
            const int c = St.out_count[e];
            if (c < St.out_cap) {
                St.out_bin[static_cast<size_t>(e) * St.out_cap + c] = phase_bin(M, St.start[e]);
                St.out_failed[static_cast<size_t>(e) * St.out_cap + c] = 1;
            }
            St.out_count[e] = c + 1;
        }
        return;
    }

    if (grf) {
#pragma unroll
        for (int k = 0; k < kMaxLinkSlots; ++k) {
            const int l = lane + 32 * k;
            if (l < nl) {
                grf[(static_cast<size_t>(le) * nl + l) * 2 + 0] = grf_acc[k][0];
                grf[(static_cast<size_t>(le) * nl + l) * 2 + 1] = grf_acc[k][1];
            }
        }
    }

    // ---- env epilogue (env.cpp:231-262) ----
    const int t_index = St.t_index[e] + 1;
    const int steps = St.steps[e] + 1;
    fk_pass(M, S, lane);
    double* qsm = reinterpret_cast<double*>(S.un);  // f64 q for Δ / obs
#pragma unroll
    for (int k = 0; k < kMaxQSlots; ++k) {
        const int d = lane + 32 * k;
        if (d < nq) qsm[d] = qd[k];
    }
    __syncwarp();
    const bool far = write_delta(M, S, qsm, t_index, drow, lane);
    if (obs_row) write_obs(M, St, S, qsm, e, t_index, obs_row, lane);

    float aux = 0.0f;
    if (M.reward_mode == 1 && M.n_emg > 0) {
        float s = 0.0f;
        for (int ch = lane; ch < M.n_emg_ch; ch += 32) {
            const float d = static_cast<float>(M.clip_emg[static_cast<size_t>(t_index) * M.n_emg + ch]) -
                            St.act[mb + __ldg(M.emg_map + ch)];
            s = fmaf(d, d, s);
        }
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
        aux = M.n_emg_ch > 0 ? M.w_emg * (-s / static_cast<float>(M.n_emg_ch)) : 0.0f;
    } else if (M.reward_mode == 2) {
        float s = 0.0f;
        for (int m = lane; m < nm; m += 32) s += pw[m];
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
        aux = M.w_power * (-s / static_cast<float>(max(1, nm)));
    }
    if (lane == 0) {
        const bool failed = !M.eval_mode && far;
        const bool horizon = steps >= M.horizon || t_index >= M.frames - 1;
        uint8_t f = 0;
        if (failed || horizon) {
            f = kFlagDone | (failed ? kFlagFailed : 0);
            St.done[e] = 1;
            const int c = St.out_count[e];
            if (c < St.out_cap) {
                St.out_bin[static_cast<size_t>(e) * St.out_cap + c] = phase_bin(M, St.start[e]);
                St.out_failed[static_cast<size_t>(e) * St.out_cap + c] = failed ? 1 : 0;
            }
            St.out_count[e] = c + 1;
        }
        St.t_index[e] = t_index;
        St.steps[e] = steps;
        if (flags) flags[le] = f;
        if (reward_aux) reward_aux[le] = aux;
    }
}

// ============================================================================
// reset / observe / tracking-error / force-to-reference: warp per env
// ============================================================================
enum ResetMode : int { kResetSample = 0, kResetFrame = 1, kResetForce = 2, kResetInit = 3 };

template <int WPB>
__global__ void __launch_bounds__(WPB * 32) reset_kernel(DevModel M, DevState St, int n_envs, int mode,
                                                         const uint8_t* mask, uint8_t mask_bits,
                                                         const int* frames_in, float* obs, int* frames_out,
                                                         uint8_t* bad) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int e = blockIdx.x * WPB + warp;
    if (e >= n_envs) return;
    if (mask && !(mask[e] & mask_bits)) return;
    const EnvSmem S = carve(smem + warp * M.smem_env_bytes, M);
    const int nq = M.nq;
    int frame = 0;
    if (mode == kResetSample) {
        if (lane == 0) frame = M.rsi ? rsi_frame(M, St, e) : 0;
        frame = __shfl_sync(kFull, frame, 0);
    } else if (mode == kResetFrame) {
        frame = frames_in[e];
        if (frame < 0 || frame >= M.frames - 1) {  // ContractError in env.cpp:96-97
            if (lane == 0 && bad) bad[e] = 1;
            return;
        }
        if (lane == 0 && bad) bad[e] = 0;
    } else if (mode == kResetForce) {
        frame = St.t_index[e];
    }  // kResetInit: frame 0 (Env::Env, env.cpp:86)
    const double* cq = M.clip_q + static_cast<size_t>(frame) * nq;
    const double* cdq = M.clip_dq + static_cast<size_t>(frame) * nq;
    double qd[kMaxQSlots], dqd[kMaxQSlots];
#pragma unroll
    for (int k = 0; k < kMaxQSlots; ++k) {
        const int d = lane + 32 * k;
        qd[k] = d < nq ? cq[d] : 0.0;
        dqd[k] = d < nq ? cdq[d] : 0.0;
        if (d < nq) {
            St.q[static_cast<size_t>(e) * nq + d] = qd[k];
            St.dq[static_cast<size_t>(e) * nq + d] = dqd[k];
        }
    }
    publish_dofs(M, S, qd, dqd, lane);
    __syncwarp();
    fk_pass(M, S, lane);
    init_muscles(M, St, S, e, lane);
    if (lane == 0) {
        St.t[e] = frame * kCtrlDt;
        if (mode == kResetInit) {  // constructed envs are done until reset (env.hpp:140)
            St.t_index[e] = 0;
            St.start[e] = 0;
            St.steps[e] = 0;
            St.done[e] = 1;
        } else if (mode != kResetForce) {
            St.t_index[e] = frame;
            St.start[e] = frame;
            St.steps[e] = 0;
            St.done[e] = 0;
        }
        if (frames_out) frames_out[e] = frame;
    }
    if (obs) {
        double* qsm = reinterpret_cast<double*>(S.un);
#pragma unroll
        for (int k = 0; k < kMaxQSlots; ++k) {
            const int d = lane + 32 * k;
            if (d < nq) qsm[d] = qd[k];
        }
        __syncwarp();
        const int obs_dim = 3 * nq + 6 * M.nk + 4 * M.nm;
        write_obs(M, St, S, qsm, e, frame, obs + static_cast<size_t>(e) * obs_dim, lane);
    }
}

template <int WPB>
__global__ void __launch_bounds__(WPB * 32) observe_kernel(DevModel M, DevState St, int n_envs, float* obs,
                                                           float* delta) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int e = blockIdx.x * WPB + warp;
    if (e >= n_envs) return;
    const EnvSmem S = carve(smem + warp * M.smem_env_bytes, M);
    const int nq = M.nq;
    double qd[kMaxQSlots], dqd[kMaxQSlots];
#pragma unroll
    for (int k = 0; k < kMaxQSlots; ++k) {
        const int d = lane + 32 * k;
        qd[k] = d < nq ? St.q[static_cast<size_t>(e) * nq + d] : 0.0;
        dqd[k] = d < nq ? St.dq[static_cast<size_t>(e) * nq + d] : 0.0;
    }
    publish_dofs(M, S, qd, dqd, lane);
    __syncwarp();
    fk_pass(M, S, lane);
    double* qsm = reinterpret_cast<double*>(S.un);
#pragma unroll
    for (int k = 0; k < kMaxQSlots; ++k) {
        const int d = lane + 32 * k;
        if (d < nq) qsm[d] = qd[k];
    }
    __syncwarp();
    const int t_index = St.t_index[e];
    if (delta) write_delta(M, S, qsm, t_index, delta + static_cast<size_t>(e) * (3 + M.nj + 2 * M.nk), lane);
    if (obs) write_obs(M, St, S, qsm, e, t_index, obs + static_cast<size_t>(e) * (3 * nq + 6 * M.nk + 4 * M.nm), lane);
}

// ============================================================================
// small per-env kernels
// ============================================================================
__global__ void seed_kernel(DevState St, int n_envs, uint64_t base_seed) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n_envs) return;
    uint64_t* mt = St.mt + static_cast<size_t>(e) * 312;
    uint64_t x = base_seed + static_cast<uint64_t>(e);
    mt[0] = x;
    for (int i = 1; i < 312; ++i) {
        x = 6364136223846793005ULL * (x ^ (x >> 62)) + static_cast<uint64_t>(i);
        mt[i] = x;
    }
    St.mti[e] = 312;
}

__global__ void rng_raw_kernel(DevState St, int e, int n, uint64_t* out) {
    if (blockIdx.x == 0 && threadIdx.x == 0)
        for (int i = 0; i < n; ++i) out[i] = mt_next(St.mt + static_cast<size_t>(e) * 312, St.mti + e);
}

// AdaptiveSampler::record (env.cpp:34-37), strict IEEE f64.
__device__ __forceinline__ void sampler_record(double* ema, int bins, double decay, int bin, int failed) {
    if (bin < 0 || bin >= bins) return;
    ema[bin] = __dadd_rn(__dmul_rn(decay, ema[bin]), __dmul_rn(__dsub_rn(1.0, decay), failed ? 1.0 : 0.0));
}

__global__ void record_own_kernel(DevModel M, DevState St, int n_envs) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n_envs) return;
    const int n = min(St.out_count[e], St.out_cap);
    for (int i = 0; i < n; ++i)
        sampler_record(St.ema + static_cast<size_t>(e) * M.bins, M.bins, M.decay,
                       St.out_bin[static_cast<size_t>(e) * St.out_cap + i],
                       St.out_failed[static_cast<size_t>(e) * St.out_cap + i]);
    St.out_count[e] = 0;
}

// Ordered merge into one sampler (env order, then time order), then broadcast.
__global__ void merge_kernel(DevModel M, DevState St, int n_local, const int* bins, const uint8_t* failed,
                             const int* counts, long long n_total, int cap, double* global_ema) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        for (long long g = 0; g < n_total; ++g) {
            const int n = min(counts[g], cap);
            for (int i = 0; i < n; ++i)
                sampler_record(global_ema, M.bins, M.decay, bins[g * cap + i], failed[g * cap + i]);
        }
    }
}

__global__ void broadcast_ema_kernel(DevState St, int n_envs, int bins, const double* row) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n_envs * bins) St.ema[i] = row[i % bins];
}

__global__ void drain_kernel(DevState St, int n_envs, int cap, int* bins, uint8_t* failed, int* counts) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n_envs) return;
    const int c = St.out_count[e];
    counts[e] = c;
    const int n = min(min(c, St.out_cap), cap);
    for (int i = 0; i < n; ++i) {
        bins[static_cast<size_t>(e) * cap + i] = St.out_bin[static_cast<size_t>(e) * St.out_cap + i];
        failed[static_cast<size_t>(e) * cap + i] = St.out_failed[static_cast<size_t>(e) * St.out_cap + i];
    }
    St.out_count[e] = 0;
}

__global__ void get_ints_kernel(DevState St, int n_envs, int* ints) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n_envs) return;
    ints[4 * e + 0] = St.t_index[e];
    ints[4 * e + 1] = St.start[e];
    ints[4 * e + 2] = St.steps[e];
    ints[4 * e + 3] = St.done[e];
}

__global__ void set_ints_kernel(DevState St, int n_envs, const int* ints) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n_envs) return;
    St.t_index[e] = ints[4 * e + 0];
    St.start[e] = ints[4 * e + 1];
    St.steps[e] = ints[4 * e + 2];
    St.done[e] = static_cast<uint8_t>(ints[4 * e + 3] != 0);
}

// Philox4x32-10 excitations, one thread per (env, group of 4 muscles).
__global__ void excitation_kernel(int n_envs, int nm, long long env_offset, uint64_t seed, uint32_t step,
                                  float* out) {
    const int groups = (nm + 3) / 4;
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= static_cast<long long>(n_envs) * groups) return;
    const int e = static_cast<int>(i / groups), g = static_cast<int>(i % groups);
    uint32_t c0 = step, c1 = static_cast<uint32_t>(env_offset + e), c2 = static_cast<uint32_t>(g), c3 = 0;
    uint32_t k0 = static_cast<uint32_t>(seed), k1 = static_cast<uint32_t>(seed >> 32);
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
    const uint32_t r4[4] = {c0, c1, c2, c3};
    float* row = out + static_cast<size_t>(e) * nm;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int m = 4 * g + k;
        if (m < nm) row[m] = static_cast<float>(r4[k] >> 8) * (1.0f / 16777216.0f);
    }
}

// FFMA throughput probe (roofline denominator for the FP32-bound step kernel):
// 8 independent FMA chains per thread, 2 flops per FMA.
__global__ void fma_probe_kernel(float* out, int iters) {
    float a0 = threadIdx.x * 1e-3f, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6,
          a7 = a0 + 7;
    const float b = 0.999999f, c = 1e-7f;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            a0 = fmaf(a0, b, c);
            a1 = fmaf(a1, b, c);
            a2 = fmaf(a2, b, c);
            a3 = fmaf(a3, b, c);
            a4 = fmaf(a4, b, c);
            a5 = fmaf(a5, b, c);
            a6 = fmaf(a6, b, c);
            a7 = fmaf(a7, b, c);
        }
    }
    if (a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7 == 1234.5f) out[0] = a0;
}

double measure_fp32_peak_tflops() {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    float* out = nullptr;
    cudaMalloc(&out, sizeof(float));
    const int blocks = sms * 8, threads = 256, iters = 2048;
    fma_probe_kernel<<<blocks, threads>>>(out, 64);  // warm-up
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
        cudaEventRecord(e0);
        fma_probe_kernel<<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    const double flops = 2.0 * 8 * 16 * static_cast<double>(iters) * blocks * threads;
    return flops / (best * 1e-3) / 1e12;
}

// ============================================================================
// host-side launch wrappers
// ============================================================================
constexpr int kWPB = 4;

cudaError_t prepare_kernels(int smem_bytes_per_block) {
    cudaError_t err;
    if ((err = cudaFuncSetAttribute(step_kernel<kWPB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    smem_bytes_per_block)) != cudaSuccess)
        return err;
    if ((err = cudaFuncSetAttribute(reset_kernel<kWPB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    smem_bytes_per_block)) != cudaSuccess)
        return err;
    return cudaFuncSetAttribute(observe_kernel<kWPB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                smem_bytes_per_block);
}

int envs_per_block() { return kWPB; }

void launch_step(const DevModel& M, const DevState& St, int env0, int n, const float* actions, float* obs,
                 float* delta, float* raux, uint8_t* flags, float* power, float* grf, cudaStream_t s) {
    const int blocks = (n + kWPB - 1) / kWPB;
    step_kernel<kWPB><<<blocks, kWPB * 32, kWPB * M.smem_env_bytes, s>>>(M, St, env0, n, actions, obs, delta,
                                                                         raux, flags, power, grf);
}

void launch_reset(const DevModel& M, const DevState& St, int n, int mode, const uint8_t* mask, uint8_t bits,
                  const int* frames_in, float* obs, int* frames_out, uint8_t* bad, cudaStream_t s) {
    const int blocks = (n + kWPB - 1) / kWPB;
    reset_kernel<kWPB><<<blocks, kWPB * 32, kWPB * M.smem_env_bytes, s>>>(M, St, n, mode, mask, bits, frames_in,
                                                                          obs, frames_out, bad);
}

void launch_observe(const DevModel& M, const DevState& St, int n, float* obs, float* delta, cudaStream_t s) {
    const int blocks = (n + kWPB - 1) / kWPB;
    observe_kernel<kWPB><<<blocks, kWPB * 32, kWPB * M.smem_env_bytes, s>>>(M, St, n, obs, delta);
}

void launch_seed(const DevState& St, int n, uint64_t base_seed, cudaStream_t s) {
    seed_kernel<<<(n + 127) / 128, 128, 0, s>>>(St, n, base_seed);
}

void launch_rng_raw(const DevState& St, int e, int n, uint64_t* out, cudaStream_t s) {
    rng_raw_kernel<<<1, 32, 0, s>>>(St, e, n, out);
}

void launch_record_own(const DevModel& M, const DevState& St, int n, cudaStream_t s) {
    record_own_kernel<<<(n + 127) / 128, 128, 0, s>>>(M, St, n);
}

void launch_merge(const DevModel& M, const DevState& St, int n_local, const int* bins, const uint8_t* failed,
                  const int* counts, long long n_total, int cap, double* global_ema, cudaStream_t s) {
    merge_kernel<<<1, 32, 0, s>>>(M, St, n_local, bins, failed, counts, n_total, cap, global_ema);
    const int tot = n_local * M.bins;
    broadcast_ema_kernel<<<(tot + 255) / 256, 256, 0, s>>>(St, n_local, M.bins, global_ema);
}

void launch_broadcast_ema(const DevState& St, int n, int bins, const double* row, cudaStream_t s) {
    broadcast_ema_kernel<<<(n * bins + 255) / 256, 256, 0, s>>>(St, n, bins, row);
}

void launch_drain(const DevState& St, int n, int cap, int* bins, uint8_t* failed, int* counts, cudaStream_t s) {
    drain_kernel<<<(n + 127) / 128, 128, 0, s>>>(St, n, cap, bins, failed, counts);
}

void launch_get_ints(const DevState& St, int n, int* ints, cudaStream_t s) {
    get_ints_kernel<<<(n + 127) / 128, 128, 0, s>>>(St, n, ints);
}

void launch_set_ints(const DevState& St, int n, const int* ints, cudaStream_t s) {
    set_ints_kernel<<<(n + 127) / 128, 128, 0, s>>>(St, n, ints);
}

void launch_excitations(int n, int nm, long long env_offset, uint64_t seed, uint32_t step, float* out,
                        cudaStream_t s) {
    const long long tot = static_cast<long long>(n) * ((nm + 3) / 4);
    excitation_kernel<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, s>>>(n, nm, env_offset, seed, step, out);
}

}  // namespace msk_b200
