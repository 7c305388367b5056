// sm_100a kernels of the batched env-stepper.
//
// One warp owns one environment for a whole control step: the 10 substeps
// of msk::step (skeleton.cpp:286-331) run on-chip, with per-env scratch in
// shared memory and nothing but the step's inputs/outputs touching HBM.
//
// Per substep (lane-parallel phases separated by __syncwarp):
//   1. muscles: activation ODE, path length in f64 (each segment in its
//      parent link's frame), fibre kinematics, Hill force, and the J_m^T F
//      contribution of each segment into a per-env slot table
//                                    (muscle.cpp:9-56, skeleton.cpp:129-170, 298-315)
//   2. joint torques: fixed-order sum of each joint's slots, minus damping
//      and the joint-limit penalty   (skeleton.cpp:222-231)
//   3. one root-to-leaf sweep: FK (rotation composition), velocity
//      kinematics, and each link's spatial inertia / bias / gravity /
//      contact wrench               (skeleton.cpp:43-107, 191-262)
//   4. articulated-body recursion, leaf-to-root then root-to-leaf: the
//      tree-sparse L D L^T factor/solve of M(q) q̈ = τ + J^T f − C without
//      forming the n_q x n_q matrix  (skeleton.cpp:172-189, 316-317)
//   5. semi-implicit Euler in f64 + divergence check (skeleton.cpp:319-328)
// then the env epilogue: Δ, observation, reward_aux, termination, episode
// outcome (env.cpp:129-263).  Reductions use fixed orders (no float atomics),
// so a step is bit-reproducible.
#include <cuda_runtime.h>

#include <cstdlib>
#include <stdexcept>

#include <cstdint>

#include "device.cuh"

namespace msk_b200 {

namespace {

constexpr double kPi = 3.14159265358979323846;

// Optional per-phase cycle counters (build with -DMSK_PHASE_TIMERS; read with
// msk_gpu_phase_cycles): lane 0 of every warp adds clock64() deltas.
#ifdef MSK_PHASE_TIMERS
__device__ unsigned long long g_phase_cycles[8];
#define PHASE_T0() long long phase_t_ = clock64()
#define PHASE_MARK(i)                                                                          \
    do {                                                                                       \
        const long long n_ = clock64();                                                        \
        if ((threadIdx.x & 31) == 0) atomicAdd(&g_phase_cycles[i], (unsigned long long)(n_ - phase_t_)); \
        phase_t_ = n_;                                                                         \
    } while (0)
#else
#define PHASE_T0() \
    do {           \
    } while (0)
#define PHASE_MARK(i) \
    do {              \
    } while (0)
#endif

struct EnvSmem {
    float4* kin;     // nl: cos, sin, origin x, origin z (root-relative)
    double2* relcs;  // nq: cos, sin of each joint's own rotation (mount + q), f64
    float* dqf;      // nq
    float* tau;      // nq: joint torque, then q̈
    float* root;     // [0] root x, [1] root z (absolute), [2] cos q2, [3] sin q2
    float* un;       // union: pair slots | kLinkStride floats per link (ABA) | f64 q
    double2* kind;   // 2 nl (general-segment models only): f64 {cos, sin}, {origin x, z} (root-relative)
    float* pen;      // ns: contact-sphere penetration (f64 geometry) of the substep
    // block-shared tree table (copied once per block; see CompiledModel tab_*)
    const float4* ta;      // nl: {anchor x, anchor z, com, mass}
    const float* tin;      // nl: inertia
    const int* tmeta;      // nl: (parent + 1) | nchild << 8 | child_off << 16 | has_sphere << 24
    const uint8_t* tchild; // child lists
    const uint8_t* tlvl;   // links grouped by depth
    const uint8_t* tlvs;   // level starts
    const uint32_t* twork; // [level][32] work words (see capi.cu): link, parent, children, sphere flag
    const uint8_t* tqf;    // [tq_len][G] joint-torque list flags: piece id ending at the element, else 0xff
    const uint8_t* tqp;    // nj + 1: pieces of joint j = [tqp[j], tqp[j+1])
    const uint8_t* tchain; // n_levels: 0x80 = chain level (its links sit in their parent's slot) | super-level end
    const uint8_t* tslstart;  // n_levels: first level of the level's super-level
    int G;                 // lanes per env (32 or 16)
    unsigned hm;           // mask of this env's lanes
};

// Block prologue: stage the tree table (model constants of the tree passes)
// into the head of shared memory with one TMA bulk copy (cp.async.bulk,
// completion on an mbarrier).  Must be reached by every thread of the block.
__device__ __forceinline__ void load_tree_table(unsigned char* smem, const DevModel& M) {
    __shared__ __align__(8) uint64_t bar;
    const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(&bar));
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(M.tab_bytes) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
                     "l"(M.tab_blob), "r"(M.tab_bytes), "r"(b)
                     : "memory");
    }
    __syncthreads();  // barrier initialised before anyone waits on it
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "TAB_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t"
        "@!p bra TAB_WAIT_%=;\n\t}" ::"r"(b)
        : "memory");
}

__device__ __forceinline__ EnvSmem carve(unsigned char* smem0, int slot, const DevModel& M, int G, unsigned hm) {
    // The CTA's shared-window address of the dynamic smem, pinned in a register
    // (opaque to the optimiser): otherwise, at the 72-register cap, every pass
    // rematerialises it from SR_CgaCtaId (4 instructions per tree level), +1 %.
    uint32_t sb = static_cast<uint32_t>(__cvta_generic_to_shared(smem0));
    asm volatile("" : "+r"(sb));
    unsigned char* smem = static_cast<unsigned char*>(__cvta_shared_to_generic(sb));
    EnvSmem s;
    s.G = G;
    s.hm = hm;
    unsigned char* base = smem + M.tab_bytes + slot * M.smem_env_bytes;
    s.kin = reinterpret_cast<float4*>(base);
    s.relcs = reinterpret_cast<double2*>(base + M.off_relcs);
    s.dqf = reinterpret_cast<float*>(base + M.off_dqf);
    s.tau = reinterpret_cast<float*>(base + M.off_tau);
    s.root = reinterpret_cast<float*>(base + M.off_root);
    s.un = reinterpret_cast<float*>(base + M.off_union);
    s.kind = reinterpret_cast<double2*>(base + M.off_kind);
    s.pen = reinterpret_cast<float*>(base + M.off_pen);
    s.ta = reinterpret_cast<const float4*>(smem + M.tab_off_a);
    s.tin = reinterpret_cast<const float*>(smem + M.tab_off_in);
    s.tmeta = reinterpret_cast<const int*>(smem + M.tab_off_meta);
    s.tchild = smem + M.tab_off_child;
    s.tlvl = smem + M.tab_off_lvl;
    s.tlvs = smem + M.tab_off_lvs;
    s.twork = reinterpret_cast<const uint32_t*>(smem + M.tab_off_work);
    s.tqf = smem + M.tab_off_tq;
    s.tqp = smem + M.tab_off_tqp;
    s.tchain = smem + M.tab_off_chain;
    s.tslstart = smem + M.tab_off_slstart;
    return s;
}

// Work word fields (capi.cu tree table): valid slots are packed at the front of a level.
__device__ __forceinline__ int ww_link(uint32_t w) { return static_cast<int>(w & 0xff); }
__device__ __forceinline__ int ww_parent(uint32_t w) { return static_cast<int>((w >> 8) & 0xff) - 1; }
__device__ __forceinline__ int ww_child0(uint32_t w) { return static_cast<int>((w >> 16) & 0xff); }
__device__ __forceinline__ int ww_nchild(uint32_t w) { return static_cast<int>((w >> 24) & 0xf); }

// Origin (x, z) half of a link's frame record {cos, sin, x, z}: an 8-B load.
// During the substeps (tree_sweep<true>) the record holds the origin RELATIVE
// to the parent's origin instead (R_p anchor): the passes only use differences.
__device__ __forceinline__ float2 frame_rel(const EnvSmem& S, int l) {
    return reinterpret_cast<const float2*>(S.kin + l)[1];
}
__device__ __forceinline__ float2 frame_origin(const EnvSmem& S, int l) {
    return reinterpret_cast<const float2*>(S.kin + l)[1];
}

__device__ __forceinline__ int link_dof(const DevModel& M, int l) {
    return l >= M.floating ? M.nrd + l - M.floating : -1;
}

// ---- SFU helpers (flush-to-zero approximations; operands here are O(1)) ----
__device__ __forceinline__ float ex2_ftz(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float rcp_ftz(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float rsqrt_ftz(float x) {
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
constexpr float kLog2e = 1.4426950408889634f;

// l_m = std::max((L - slack) / l_opt, kMinFiberLength) (skeleton.cpp:279, 305):
// std::max's compare-select, NaN in the first argument propagates as there.
__device__ __forceinline__ double fiber_clamp(double x) {
    return x < static_cast<double>(kMinFiber) ? static_cast<double>(kMinFiber) : x;
}

// Read-only model-constant loads (non-coherent path; the tables never change
// during a launch).
__device__ __forceinline__ float4 ldc4(const float4* p) { return __ldg(p); }
__device__ __forceinline__ double2 ldc2d(const double2* p) { return __ldg(p); }

// ---- Hill-type muscle (muscle.cpp:9-40) -----------------------------------
__device__ __forceinline__ float hill_fl(float l) {  // exp(-((l-1)/0.45)^2)
    const float d = l - 1.0f;
    return ex2_ftz(d * d * (-kLog2e / (0.45f * 0.45f)));
}
__device__ __forceinline__ float hill_fv(float v) {  // branch-free: one reciprocal, selects
    constexpr float c = 0.32f;  // (1.4 - 1) / (1 + 1/4)
    const bool neg = v < 0.0f;
    const float num = neg ? v + 1.0f : fmaf(1.4f, v, c);
    const float den = neg ? fmaf(-0.25f, v, 1.0f) : v + c;
    const float fv = num * rcp_ftz(den);
    return v <= -1.0f ? 0.0f : fv;
}
__device__ __forceinline__ float hill_fp(float l) {  // (exp(4(l-1)) - 1) / (e^2 - 1)
    if (l <= 1.0f) return 0.0f;
    return (ex2_ftz((l - 1.0f) * (4.0f * kLog2e)) - 1.0f) * (1.0f / 6.38905609893065f);
}
__device__ __forceinline__ float mtu_force(float act, float l, float v, float fmax) {
    return fmax * (act * hill_fl(l) * hill_fv(v) + hill_fp(l));
}

#ifdef MSK_F64_HILL  // diagnostics build: the Hill force in f64 (muscle.cpp:9-40 arithmetic)
__device__ __forceinline__ float mtu_force_d(float act, double l, double v, float fmax) {
    const double d = (l - 1.0) / 0.45;
    const double fl = exp(-d * d);
    double fv;
    if (v <= -1.0) fv = 0.0;
    else if (v < 0.0) fv = (v + 1.0) / (1.0 - v / 4.0);
    else fv = (1.4 * v + 0.32) / (v + 0.32);
    const double fp = l > 1.0 ? (exp(4.0 * (l - 1.0)) - 1.0) / (exp(2.0) - 1.0) : 0.0;
    return static_cast<float>(static_cast<double>(fmax) * (static_cast<double>(act) * fl * fv + fp));
}
#endif

// sqrt of a non-negative f64 from the f32 rsqrt seed plus one f64 Newton
// correction (~46 bits); also returns the f32 reciprocal length.  x is clamped
// at ~1e-30 through its high word (one integer max; negative rounding noise has
// the sign bit set and clamps too) so degenerate/padding segments stay finite.
__device__ __forceinline__ double sqrt_d(double x, float& inv) {
    x = __hiloint2double(max(__double2hiint(x), 0x39B4484B), __double2loint(x));
    const float r = rsqrt_ftz(static_cast<float>(x));
    inv = r;
    const double rd = static_cast<double>(r);
    const double s = x * rd;
    return fma(fma(-s, s, x), 0.5 * rd, s);
}

// World (root-relative) position of a via point from the f64 frames (fk_d):
// the general segments' lengths feed v_m = (L - prev_len) / (dt l_opt v_max), so they need the
// reference's f64 precision like the adjacent (K-form) segments.
__device__ __forceinline__ double2 via_point_d(const DevModel& M, const double2* kind, int v) {
    const int l = __ldg(M.via_link + v);
    const double x = __ldg(M.via_x + v), z = __ldg(M.via_z + v);
    if (l < 0) return make_double2(x, z);
    const double2 cs = kind[2 * l], o = kind[2 * l + 1];
    return make_double2(fma(cs.x, x, fma(-cs.y, z, o.x)), fma(cs.y, x, fma(cs.x, z, o.y)));
}

__device__ __forceinline__ double general_seg_len(const DevModel& M, const EnvSmem& S, int v_end) {
    const double2 pe = via_point_d(M, S.kind, v_end), ps = via_point_d(M, S.kind, v_end - 1);
    const double dx = pe.x - ps.x, dz = pe.y - ps.y;
    float inv;
    return sqrt_d(fma(dx, dx, dz * dz), inv);  // f32 rsqrt seed + one f64 Newton step (~46 bits)
}

// Same-link (kind 0) or adjacent (kind 1) segment from its K constants
// (device.cuh seg_kf), evaluated in the parent's frame with the child joint's
// own f64 rotation: |s|^2 = K1 + 2 (c K2h + s K3h).  Returns |s| (f64) and the
// moment-arm factor (r x A) / |s| about the child joint.  Same-link segments
// have K = (len^2, 0, 0) and padding K = 0, so neither needs a branch.
__device__ __forceinline__ double kseg(const EnvSmem& S, float4 k, int info, float& arm) {
    const double2 cs = S.relcs[(info >> 2) & 511];
    const double k2 = k.y, k3 = k.z;
    float inv;
    const double len = sqrt_d(fma(2.0, fma(cs.x, k2, cs.y * k3), static_cast<double>(k.x)), inv);
    arm = static_cast<float>(fma(cs.x, k3, -cs.y * k2)) * inv;
    return len;
}

// Path length of muscle m (skeleton.cpp:129-141) — used by make_initial_state.
__device__ __forceinline__ double muscle_length(const DevModel& M, const EnvSmem& S, int m) {
    const int nseg = __ldg(M.m_meta + m) & 0xff;
    double L = 0.0;
    for (int k = 0; k < nseg; ++k) {
        const float4 kf = __ldg(M.seg_kf + k * M.nm + m);
        const int info = __float_as_int(kf.w);
        float arm;
        L += (info & 3) == 2 ? general_seg_len(M, S, info >> 11) : kseg(S, kf, info, arm);
    }
    return L;
}

// J_m^T F of the general (non-adjacent) segments of muscle m (reference index),
// world frame (skeleton.cpp:147-170): the segment direction and the lever arm
// about the joint from the f64 frames (fk_d), the moment rounded to f32 once.
// A segment's pairs (one per joint on its tree path) are consecutive, so its via
// points, direction and reciprocal length are computed once per segment.
__device__ void general_pairs(const DevModel& M, const EnvSmem& S, int m, float F) {
    const int p0 = __ldg(M.m_pair_start + m), p1 = __ldg(M.m_pair_start + m + 1);
    int ve_cur = -1;
    double2 pe = make_double2(0.0, 0.0), ps = make_double2(0.0, 0.0);
    double sx = 0.0, sz = 0.0, inv_len = 0.0;
    bool ok = false;
    for (int p = p0; p < p1; ++p) {
        const int ve = __ldg(M.pair_via + p), j = __ldg(M.pair_joint + p);
        const float sg = __ldg(M.pair_sign + p);
        if (ve != ve_cur) {
            ve_cur = ve;
            pe = via_point_d(M, S.kind, ve);
            ps = via_point_d(M, S.kind, ve - 1);
            sx = pe.x - ps.x;
            sz = pe.y - ps.y;
            const double l2 = fma(sx, sx, sz * sz);
            ok = l2 > 1e-24;  // |s| > 1e-12 (skeleton.cpp:160)
            float inv32;
            const double len = sqrt_d(l2, inv32);
            inv_len = 1.0 / len;
        }
        float val = 0.0f;
        if (ok) {
            const double2 ka = S.kind[2 * (M.floating + j) + 1];  // joint j's child-link origin
            const double2 pt = sg < 0.0f ? pe : ps;
            const double rx = pt.x - ka.x, rz = pt.y - ka.y;
            val = static_cast<float>(static_cast<double>(sg * F) * (fma(rx, sz, -rz * sx) * inv_len));
        }
        S.un[__ldg(M.pair_slot + p)] = val;
    }
}

// Per-DOF views for the tree passes: each joint's own rotation (f64 sincos of
// mount + q), root pitch rotation, root position, and f32 velocities.
template <int QS>
__device__ __forceinline__ void publish_dofs(const DevModel& M, const EnvSmem& S, const double* qd,
                                             const double* dqd, int lane) {
#pragma unroll
    for (int k = 0; k < QS; ++k) {
        const int d = lane + S.G * k;
        if (d < M.nq) {
            if (d >= M.nrd) {
                const int l = M.floating + (d - M.nrd);
                double sn, cs;
                sincos(__ldg(M.link_mount + l) + qd[k], &sn, &cs);
                S.relcs[d] = make_double2(cs, sn);
            } else if (d == 2) {
                double sn, cs;
                sincos(qd[k], &sn, &cs);
                S.root[2] = static_cast<float>(cs);
                S.root[3] = static_cast<float>(sn);
                S.relcs[2] = make_double2(cs, sn);  // (unused root slot) f64 pitch for fk_d
            } else {
                S.root[d] = static_cast<float>(qd[k]);
                reinterpret_cast<double*>(S.relcs)[d] = qd[k];  // relcs[0] = f64 root (x, z)
            }
            S.dqf[d] = static_cast<float>(dqd[k]);
        }
    }
}

// f64 world height of a point given in link l's frame (skeleton.cpp:82-113):
// walks the joint chain up to the root, p <- anchor + R(mount + q) p, each
// joint's rotation in f64 (relcs); the floating root adds R(q2) and (q0, q1)
// (relcs[2], relcs[0]).
__device__ __forceinline__ double sphere_height_d(const DevModel& M, const EnvSmem& S, int l, float px, float pz) {
    double x = px, z = pz;
    int cur = l;
    while (cur >= M.floating) {
        const double2 r = S.relcs[M.nrd + cur - M.floating];
        const float4 a = S.ta[cur];
        const double nx = fma(r.x, x, fma(-r.y, z, static_cast<double>(a.x)));
        z = fma(r.y, x, fma(r.x, z, static_cast<double>(a.y)));
        x = nx;
        cur = (S.tmeta[cur] & 0xff) - 1;
    }
    if (M.floating) {
        const double2 r = S.relcs[2], o = S.relcs[0];
        z = fma(r.y, x, fma(r.x, z, o.y));
    }
    return z;
}

// Penetration depth of every contact sphere from its f64 world height: the
// contact force is discontinuous at pen = 0 when the sphere moves down
// (f_n = -c z' there, skeleton.cpp:243-248), so the branch must be taken where
// the reference's f64 takes it (an f32 height flips it for |pen| < ~1e-7 m).
__device__ __forceinline__ void sphere_pen_d(const DevModel& M, const EnvSmem& S, int lane) {
    for (int sp = lane; sp < M.ns; sp += S.G) {
        const float4 sd = __ldg(M.sphere + sp);
        S.pen[sp] = static_cast<float>(static_cast<double>(sd.z) - sphere_height_d(M, S, __ldg(M.sphere_link + sp),
                                                                                      sd.x, sd.y));
    }
    __syncwarp(S.hm);
}

// One link of the root-to-leaf sweep (tree_sweep).  kSimple: the level has no
// root and no child of the fixed base (work-word bit 29), so the link has a
// parent and a joint DOF = l + nrd - floating.
// Parent state forwarded in registers along a chain of levels (tree_sweep_chain).
struct SweepPar {
    float c, s, w, vx, vz;
};

template <bool kFull, bool kSimple, bool kFwd = false>
__device__ __forceinline__ SweepPar sweep_link(const DevModel& M, const EnvSmem& S, uint32_t ww, int dofoff,
                                               float* grf, const SweepPar& par = SweepPar{}) {
    static_assert(!kFwd || (kFull && kSimple), "forwarding: substep sweep of a chain level");
    const int l = ww_link(ww);
    const int dof = kSimple ? l + dofoff : link_dof(M, l);
    const float4 la = S.ta[l];
    float c, s, ox, oz, w = 0.0f, vx = 0.0f, vz = 0.0f;
    if (!kSimple && dof < 0) {  // floating root: origin (0,0) relative, pitch q2
        c = S.root[2];
        s = S.root[3];
        ox = 0.0f;
        oz = 0.0f;
        if (kFull) {
            w = S.dqf[2];
            vx = S.dqf[0];
            vz = S.dqf[1];
        }
    } else {
        const int p = ww_parent(ww);
        const double2 rd = S.relcs[dof];
        const float cr = static_cast<float>(rd.x), sr = static_cast<float>(rd.y);
        if (kSimple || p >= 0) {
            float4 kp;
            float2 wv;   // parent (omega, v_x)
            float pvz;   // parent v_z
            if constexpr (kFwd) {
                kp = make_float4(par.c, par.s, 0.0f, 0.0f);
                wv = make_float2(par.w, par.vx);
                pvz = par.vz;
            } else {
                kp = S.kin[p];
                if (kFull) {
                    const float* up = S.un + kLinkStride * p;
                    wv = reinterpret_cast<const float2*>(up)[5];
                    pvz = up[9];
                }
            }
            // kFull: origin relative to the parent's (frame_rel); else absolute (root-relative)
            ox = fmaf(kp.x, la.x, kFull ? -kp.y * la.y : fmaf(-kp.y, la.y, kp.z));
            oz = fmaf(kp.y, la.x, kFull ? kp.x * la.y : fmaf(kp.x, la.y, kp.w));
            c = fmaf(kp.x, cr, -kp.y * sr);
            s = fmaf(kp.y, cr, kp.x * sr);
            if (kFull) {
                w = wv.x + S.dqf[dof];
                vx = fmaf(-wv.x, oz, wv.y);
                vz = fmaf(wv.x, ox, pvz);
            }
        } else {
            ox = la.x;
            oz = la.y;
            c = cr;
            s = sr;
            if (kFull) w = S.dqf[dof];
        }
    }
    S.kin[l] = make_float4(c, s, ox, oz);
    if (!kFull) return SweepPar{};
    float* u = S.un + kLinkStride * l;
    // link record (14 floats): [0..5] articulated inertia, [6..8] bias force,
    // [9] u/D, [10..11] U1/D, U2/D, [12..13] c; velocity (omega, v_x | v_z)
    // lives in [10..11 | 9] during this sweep only
    reinterpret_cast<float2*>(u)[5] = make_float2(w, vx);
    u[9] = vz;
    const float m = la.w;
    const float cx = la.z * c, cz = la.z * s;
    const float i00 = S.tin[l], i01 = -m * cz, i02 = m * cx;  // tin: I + m com^2 (about the origin)
    const float h1 = fmaf(i01, w, m * vx), h2 = fmaf(i02, w, m * vz);
    const float mg = m * M.gravity;
    float p0 = fmaf(vx, h2, -vz * h1) - cx * mg, p1 = -w * h2, p2 = fmaf(w, h1, -mg);
    if ((ww >> 28) & 1) {  // link carries contact spheres
        const int s0 = __ldg(M.sphere_start + l), s1 = __ldg(M.sphere_start + l + 1);
        float gx = 0.0f, gz = 0.0f;
        for (int sp = s0; sp < s1; ++sp) {
            const float4 sd = __ldg(M.sphere + sp);
            const float rx = fmaf(c, sd.x, -s * sd.y), rz = fmaf(s, sd.x, c * sd.y);
            // penetration from the f64 world height (sphere_pen_d)
            const float pen = S.pen[sp];
            if (pen > 0.0f) {
                const float fn = fmaxf(0.0f, fmaf(M.c_k, pen, -M.c_c * fmaf(w, rx, vz)));
                if (fn > 0.0f) {
                    const float qz = rz - sd.z;  // contact point relative to the origin
                    const float ft = -M.c_mu * fn * tanhf(fmaf(-w, qz, vx) * M.inv_c_vs);
                    p0 -= fmaf(rx, fn, -qz * ft);
                    p1 -= ft;
                    p2 -= fn;
                    gx += ft * 0.1f;
                    gz += fn * 0.1f;
                }
            }
        }
        if (grf) {
            grf[2 * l] += gx;
            grf[2 * l + 1] += gz;
        }
    }
    float c1 = 0.0f, c2 = 0.0f;
    if (kSimple || dof >= 0) {  // c = V x S qdot at the joint: (0, qdot v_z, -qdot v_x)
        const float qdot = S.dqf[dof];
        c1 = qdot * vz;
        c2 = -qdot * vx;
    }
    float2* u2 = reinterpret_cast<float2*>(u);  // 8-B aligned (stride 14 floats)
    u2[0] = make_float2(i00, i01);
    u2[1] = make_float2(i02, m);
    u2[2] = make_float2(0.0f, m);
    u2[3] = make_float2(p0, p1);
    u[8] = p2;
    u2[6] = make_float2(c1, c2);
    return SweepPar{c, s, w, vx, vz};
}

// Root-to-leaf sweep.  FK by rotation composition R_l = R_p R_joint
// (skeleton.cpp:82-107, root-relative); with kFull also velocity kinematics
// (skeleton.cpp:43-72) and each link's own articulated-body terms: spatial
// inertia about its origin, bias force V x* I V, gravity at the COM and the
// penalty contact wrench of its spheres (skeleton.cpp:191-262).  GRF of the
// substep (sphere_force / 10, skeleton.cpp:323-325) accumulates into grf.
template <bool kFull>
__device__ __forceinline__ void tree_sweep(const DevModel& M, const EnvSmem& S, int lane, float* grf) {
    const int dofoff = M.nrd - M.floating;
    for (int lev = 0; lev < M.n_levels; ++lev) {
        for (int i = lane; i < 32; i += S.G) {
            const uint32_t ww = S.twork[32 * lev + i];
            if (!(ww >> 31)) continue;
            if ((ww >> 29) & 1)
                sweep_link<kFull, true>(M, S, ww, dofoff, grf);
            else
                sweep_link<kFull, false>(M, S, ww, dofoff, grf);
        }
        __syncwarp(S.hm);
    }
}

// Super-levels: a non-chain level followed by its chain levels (capi.cu): one
// lane runs its slot's links down the chain with the parent state in registers
// and no warp barrier between the levels (wb700: 15 levels -> 6 super-levels).
// tchain[lev] (capi.cu): bit 7 = chain level; bits 0-6 = one past the
// super-level's last level (for lev = its first level).
__device__ __forceinline__ int superlevel_end(const DevModel& M, const EnvSmem& S, int lev) {
    return S.tchain[lev] & 0x7f;
}

// tree_sweep<true> over super-levels (one slot per lane: G = 32).
__device__ __forceinline__ void tree_sweep_chain(const DevModel& M, const EnvSmem& S, int lane, float* grf) {
    const int dofoff = M.nrd - M.floating;
    for (int lev = 0; lev < M.n_levels;) {
        const int end = superlevel_end(M, S, lev);
        uint32_t ww = S.twork[32 * lev + lane];
        if (ww >> 31) {
            SweepPar par = ((ww >> 29) & 1) ? sweep_link<true, true>(M, S, ww, dofoff, grf)
                                            : sweep_link<true, false>(M, S, ww, dofoff, grf);
            for (int d = lev + 1; d < end; ++d) {
                ww = S.twork[32 * d + lane];
                if (!(ww >> 31)) break;
                par = sweep_link<true, true, true>(M, S, ww, dofoff, grf, par);
            }
        }
        __syncwarp(S.hm);
        lev = end;
    }
}

// f64 forward kinematics (skeleton.cpp:82-107, root-relative) into S.kind, for
// models with general (non-adjacent) muscle segments: rotation composition
// R_l = R_p R_joint with each joint's f64 rotation (relcs), origins
// o_l = o_p + R_p anchor.
__device__ __forceinline__ void fk_d(const DevModel& M, const EnvSmem& S, int lane) {
    for (int lev = 0; lev < M.n_levels; ++lev) {
        for (int i = lane; i < 32; i += S.G) {
            const uint32_t ww = S.twork[32 * lev + i];
            if (!(ww >> 31)) continue;
            const int l = ww_link(ww);
            const int dof = link_dof(M, l);
            double2 cs, o;
            if (dof < 0) {  // floating root: origin 0 (root-relative), pitch q2
                cs = S.relcs[2];
                o = make_double2(0.0, 0.0);
            } else {
                const double2 r = S.relcs[dof];
                const int p = ww_parent(ww);
                const float4 la = S.ta[l];
                if (p >= 0) {
                    const double2 cp = S.kind[2 * p], op = S.kind[2 * p + 1];
                    const double ax = la.x, az = la.y;
                    o = make_double2(fma(cp.x, ax, fma(-cp.y, az, op.x)), fma(cp.y, ax, fma(cp.x, az, op.y)));
                    cs = make_double2(fma(cp.x, r.x, -cp.y * r.y), fma(cp.y, r.x, cp.x * r.y));
                } else {
                    o = make_double2(la.x, la.y);
                    cs = r;
                }
            }
            S.kind[2 * l] = cs;
            S.kind[2 * l + 1] = o;
        }
        __syncwarp(S.hm);
    }
}

// Key-body COM (absolute) and unreduced frame angle (skeleton.cpp:346-357).
template <bool kAngle = true>
__device__ __forceinline__ void key_body(const DevModel& M, const EnvSmem& S, const double* qsm, int k,
                                         double& x, double& z, double& ang) {
    const int l = __ldg(M.key_bodies + k);
    const float4 kl = S.kin[l];
    const float c = S.ta[l].z;
    x = static_cast<double>(fmaf(kl.x, c, kl.z));
    z = static_cast<double>(fmaf(kl.y, c, kl.w));
    double a = 0.0;
    int cur = kAngle ? l : -1;  // the angle walks the path to the root: only when asked for
    while (cur >= 0) {
        const int dof = link_dof(M, cur);
        if (dof < 0) {
            a += qsm[2];
            break;
        }
        a += __ldg(M.link_mount + cur) + qsm[dof];
        cur = (S.tmeta[cur] & 0xff) - 1;
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
    for (int i = lane; i < nq; i += S.G) obs_row[o + i] = static_cast<float>(qsm[i]);
    o += nq;
    for (int i = lane; i < nq; i += S.G) obs_row[o + i] = static_cast<float>(St.dq[static_cast<size_t>(e) * nq + i]);
    o += nq;
    for (int k = lane; k < nk; k += S.G) {
        double x, z, a;
        key_body(M, S, qsm, k, x, z, a);
        obs_row[o + 2 * k] = static_cast<float>(x);
        obs_row[o + 2 * k + 1] = static_cast<float>(z);
        obs_row[o + 2 * nk + k] = static_cast<float>(a);
    }
    o += 3 * nk;
    const size_t mb = static_cast<size_t>(e) * nm;
    // reference slot x <- internal muscle m_int[x]; 4 slots per lane in flight
    // (all loads issued before the stores, which may alias them)
    for (int x0 = 0; x0 < nm; x0 += 4 * S.G) {
        float v[4][4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int x = x0 + j * S.G + lane;
            if (x < nm) {
                const size_t i = mb + __ldg(M.m_int + x);
                v[j][0] = St.act[i];
                v[j][1] = St.fm[i];
                v[j][2] = static_cast<float>(St.lm[i]);
                v[j][3] = St.vm[i];
            }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int x = x0 + j * S.G + lane;
            if (x < nm) {
                obs_row[o + x] = v[j][0];
                obs_row[o + nm + x] = v[j][1];
                obs_row[o + 2 * nm + x] = v[j][2];
                obs_row[o + 3 * nm + x] = v[j][3];
            }
        }
    }
    o += 4 * nm;
    const size_t t = static_cast<size_t>(t_index);
    for (int i = lane; i < nq; i += S.G) obs_row[o + i] = static_cast<float>(M.clip_q[t * nq + i]);
    o += nq;
    for (int i = lane; i < 2 * nk; i += S.G) obs_row[o + i] = static_cast<float>(M.clip_kp[t * 2 * nk + i]);
    o += 2 * nk;
    for (int i = lane; i < nk; i += S.G) obs_row[o + i] = static_cast<float>(M.clip_ka[t * nk + i]);
}

// Env::tracking_error (env.cpp:170-193) -> Δ row (f64 values rounded once).
// Returns (warp-uniform) whether any key body exceeds the termination radius.
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
        for (int j = lane; j < nj; j += S.G)
            drow[3 + j] = static_cast<float>(qsm[nrd + j] - M.clip_q[t * nq + nrd + j]);
    bool far = false;
    for (int k = lane; k < nk; k += S.G) {
        double x, z, a;
        key_body<false>(M, S, qsm, k, x, z, a);
        const double dx = x - M.clip_kp[t * 2 * nk + 2 * k];
        const double dz = z - M.clip_kp[t * 2 * nk + 2 * k + 1];
        if (drow) {
            drow[3 + nj + 2 * k] = static_cast<float>(dx);
            drow[3 + nj + 2 * k + 1] = static_cast<float>(dz);
        }
        if (sqrt(dx * dx + dz * dz) > M.term_err) far = true;
    }
    return __any_sync(S.hm, far);
}

// make_initial_state (skeleton.cpp:264-284) for the env's muscles (relcs/FK in smem).
// make_initial_state's muscle part for the fast-path run of NS segments
// [m0, m1): the chunk records (M.mtab) give every load of a muscle up front
// (no per-muscle segment-count lookup ahead of the segment loads).
template <int NS>
__device__ __forceinline__ void init_run(const DevModel& M, const DevState& St, const EnvSmem& S, size_t mb, int lane,
                                         int m0, int m1, float a0) {
    const int G = S.G, field = 16 * G, rec_bytes = (3 + NS) * field;
    for (int m = m0 + lane; m < m1; m += G) {
        const unsigned char* rec = M.mtab + M.mrun_off[NS] + ((m - m0) / G) * rec_bytes + 16 * ((m - m0) % G);
        float4 kc[NS];
#pragma unroll
        for (int k = 0; k < NS; ++k) kc[k] = ldc4(reinterpret_cast<const float4*>(rec + (3 + k) * field));
        const float fmax_ = ldc4(reinterpret_cast<const float4*>(rec)).x;
        const double2 pa = ldc2d(reinterpret_cast<const double2*>(rec + field));
        const double2 pb = ldc2d(reinterpret_cast<const double2*>(rec + 2 * field));
        float arm;
        double L = kseg(S, kc[0], __float_as_int(kc[0].w), arm);
#pragma unroll
        for (int k = 1; k < NS; ++k) L += kseg(S, kc[k], __float_as_int(kc[k].w), arm);
        const double lm = fiber_clamp((L - pa.x) * pb.x);
        St.act[mb + m] = a0;
        St.lm[mb + m] = lm;
        St.vm[mb + m] = 0.0f;
        St.fm[mb + m] = mtu_force(a0, static_cast<float>(lm), 0.0f, fmax_);
    }
}

__device__ void init_muscles(const DevModel& M, const DevState& St, const EnvSmem& S, int e, int lane) {
    const size_t mb = static_cast<size_t>(e) * M.nm;
    const float a0 = static_cast<float>(M.init_act);
    int m_begin = 0;
    if (M.fast_nseg > 0) {  // same-link / adjacent segments only: chunk runs by segment count
        const int* r = M.seg_run;
        if (r[0] < r[1]) {  // zero segments: L = 0
            for (int m = r[0] + lane; m < r[1]; m += S.G) {
                const double2 pa = __ldg(M.m_p1a + m), pb = __ldg(M.m_p1b + m);
                const double lm = fiber_clamp((0.0 - pa.x) * pb.x);
                St.act[mb + m] = a0;
                St.lm[mb + m] = lm;
                St.vm[mb + m] = 0.0f;
                St.fm[mb + m] = mtu_force(a0, static_cast<float>(lm), 0.0f, __ldg(M.m_p0 + m).x);
            }
        }
        init_run<1>(M, St, S, mb, lane, r[1], r[2], a0);
        init_run<2>(M, St, S, mb, lane, r[2], r[3], a0);
        init_run<3>(M, St, S, mb, lane, r[3], r[4], a0);
        init_run<4>(M, St, S, mb, lane, r[4], r[5], a0);
        m_begin = M.gen0;
    }
    for (int m = m_begin + lane; m < M.nm; m += S.G) {
        const double2 pa = __ldg(M.m_p1a + m), pb = __ldg(M.m_p1b + m);
        const double L = muscle_length(M, S, m);
        const double lm = fiber_clamp((L - pa.x) * pb.x);
        St.act[mb + m] = a0;
        St.lm[mb + m] = lm;
        St.vm[mb + m] = 0.0f;
        St.fm[mb + m] = mtu_force(a0, static_cast<float>(lm), 0.0f, __ldg(M.m_p0 + m).x);
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

// One substep of every muscle of the env (lanes over muscles):
// activation_step (muscle.cpp:42-56, tau frozen at the step start), path length
// in f64, fibre kinematics (skeleton.cpp:302-305, prev_len from the stored,
// clamped l_m exactly as the reference), Hill force (muscle.cpp:36-40),
// substep power (skeleton.cpp:308-309), and for every adjacent segment the
// moment about its child joint -F (r x A) / |A + r| into the slot table.
// NSEG > 0: fast path for models whose segments are all adjacent/same-link
// (segments padded to NSEG, branch-free); NSEG == 0: generic path.
// Activation, fibre kinematics and Hill force of muscle m given its path
// length L; stores the muscle state, accumulates power, returns F.
// l_m is f64 state: prev_len = slack + l_m l_opt must reproduce the previous
// substep's path length to ~1e-16 (v_m divides the difference by dt l_opt v_max,
// ~1e-3), as in the reference's f64 SimState.  v_m / f_m are stored only at the
// last substep (nothing reads them in between).
// This env's muscle rows (device order), formed once per run of the muscle phase.
struct MuscleRows {
    const float* u;  // the step's clamped excitations
    float* act;
    double* lm;
    float* vm;
    float* fm;
};

__device__ __forceinline__ MuscleRows muscle_rows(const DevState& St, const float* act_row, size_t mb) {
    return MuscleRows{act_row, St.act + mb, St.lm + mb, St.vm + mb, St.fm + mb};
}

// activation_step (muscle.cpp:42-56), fibre kinematics and the Hill force: the
// new activation a1, fibre length lm1 and velocity vm; returns F.
__device__ __forceinline__ float muscle_force(float4 p0, double2 pa, double2 pb, float u, float a0, double lm0,
                                              double L, float& a1, double& lm1, float& vm) {
    const float gain = fmaf(1.5f, a0, 0.5f);
    const float ex = ex2_ftz(u > a0 ? p0.y * rcp_ftz(gain) : p0.z * gain);  // p0.y/z carry log2(e)
    a1 = fminf(fmaxf(fmaf(a0 - u, ex, u), 0.0f), 1.0f);
    const double prev_len = fma(lm0, pa.y, pa.x);
    vm = static_cast<float>((L - prev_len) * pb.y);
    lm1 = fiber_clamp((L - pa.x) * pb.x);
#ifdef MSK_F64_HILL
    return mtu_force_d(a1, lm1, (L - prev_len) * pb.y, p0.x);
#else
    return mtu_force(a1, static_cast<float>(lm1), vm, p0.x);
#endif
}

__device__ __forceinline__ float muscle_update(const MuscleRows& R, int m, int ext, float4 p0, double2 pa,
                                               double2 pb, float u, float a0, double lm0, double L, float* pw,
                                               bool last) {
    float a1, vm;
    double lm1;
    const float F = muscle_force(p0, pa, pb, u, a0, lm0, L, a1, lm1, vm);
    R.act[m] = a1;
    R.lm[m] = lm1;
    if (last) {
        R.vm[m] = vm;
        R.fm[m] = F;
    }
    if (pw) pw[ext] += fabsf(F * vm * p0.w);
    return F;
}

// Fast path: the muscles [m0, m1) of run NS (whole chunks of the lane group,
// muscles sorted by segment count), NS segments each — a compile-time count, so
// the segment loop unrolls without predicates (padding segments have K = 0 and
// write the dummy slot).  Every constant of a muscle comes from its chunk record
// (M.mtab: one pointer, immediate field offsets) and the env's muscle rows
// advance by pointer increments; the power accumulation is compiled in only when
// requested (kPow), not predicated per muscle.
template <int NS, bool kPow, int G>
__device__ __forceinline__ void muscle_run(const DevModel& M, const DevState& St, const EnvSmem& S,
                                           const float* act_row, size_t mb, float* pw, int lane, bool last, int m0,
                                           int m1) {
    int m = m0 + lane;
    if (m >= m1) return;
    constexpr int kField = G * 16, kRec = (3 + NS) * kField;
    const unsigned char* rec = M.mtab + M.mrun_off[NS] + 16 * lane;
    const float* up = act_row + m;
    float* ap = St.act + mb + m;
    double* lp = St.lm + mb + m;
    for (; m < m1; m += G, rec += kRec, up += G, ap += G, lp += G) {
        float4 kc[NS > 0 ? NS : 1];
#pragma unroll
        for (int k = 0; k < NS; ++k) kc[k] = ldc4(reinterpret_cast<const float4*>(rec + (3 + k) * kField));
        // {f_max, -dt/tau_act log2e, -dt/tau_deact log2e, l_opt v_max/10}, {slack, l_opt}, {1/l_opt, 1/(dt l_opt v_max)}
        const float4 p0 = ldc4(reinterpret_cast<const float4*>(rec));
        const double2 pa = ldc2d(reinterpret_cast<const double2*>(rec + kField));
        const double2 pb = ldc2d(reinterpret_cast<const double2*>(rec + 2 * kField));
        const float u = *up;  // clamped, device order (prep_actions_kernel)
        const float a0 = *ap;
        const double lm0 = *lp;
        float tq[NS > 0 ? NS : 1];
        double L = 0.0;
        if constexpr (NS > 0) {  // (not 0.0 + len: the add cannot be folded under IEEE signed zeros)
            L = kseg(S, kc[0], __float_as_int(kc[0].w), tq[0]);
#pragma unroll
            for (int k = 1; k < NS; ++k) L += kseg(S, kc[k], __float_as_int(kc[k].w), tq[k]);
        }
        float a1, vm;
        double lm1;
        const float F = muscle_force(p0, pa, pb, u, a0, lm0, L, a1, lm1, vm);
        *ap = a1;
        *lp = lm1;
        if (last) {
            St.vm[mb + m] = vm;
            St.fm[mb + m] = F;
        }
        if constexpr (kPow) pw[__ldg(M.m_meta + m) >> 9] += fabsf(F * vm * p0.w);
#pragma unroll
        for (int k = 0; k < NS; ++k) S.un[__float_as_int(kc[k].w) >> 11] = -F * tq[k];
    }
}

// Muscles [m_begin, nm) through the generic per-segment loop (general segments
// from the f64 frames of fk_d, adjacent ones in K-form).
__device__ __forceinline__ void muscle_generic(const DevModel& M, const DevState& St, const EnvSmem& S,
                                               const float* act_row, size_t mb, float* pw, int lane, bool last,
                                               int m_begin) {
    const int nm = M.nm;
    for (int m = m_begin + lane; m < nm; m += S.G) {
        const int meta = __ldg(M.m_meta + m);
        const int nseg = meta & 0xff, ext = meta >> 9;
        const float4 p0 = __ldg(M.m_p0 + m);
        const double2 pa = __ldg(M.m_p1a + m), pb = __ldg(M.m_p1b + m);
        const MuscleRows R = muscle_rows(St, act_row, mb);
        const float u = R.u[m];
        const float a0 = R.act[m];
        const double lm0 = R.lm[m];
        double L = 0.0;
        for (int k = 0; k < nseg; ++k) {
            const float4 kf = __ldg(M.seg_kf + k * nm + m);
            const int info = __float_as_int(kf.w);
            float arm;
            L += (info & 3) == 2 ? general_seg_len(M, S, info >> 11) : kseg(S, kf, info, arm);
        }
        const float F = muscle_update(R, m, ext, p0, pa, pb, u, a0, lm0, L, pw, last);
        for (int k = 0; k < nseg; ++k) {
            const float4 kf = __ldg(M.seg_kf + k * nm + m);
            const int info = __float_as_int(kf.w);
            if ((info & 3) != 1) continue;
            float arm;
            kseg(S, kf, info, arm);
            S.un[info >> 11] = -F * arm;
        }
        if ((meta >> 8) & 1) general_pairs(M, S, ext, F);
    }
}

template <int NSEG, bool kPow, int G>
__device__ __forceinline__ void muscle_runs(const DevModel& M, const DevState& St, const EnvSmem& S,
                                            const float* act_row, size_t mb, float* pw, int lane, bool last) {
    // runs of chunks by padded segment count (M.seg_run, muscle units): 0, 1, ..., NSEG,
    // over the muscles without a general segment
    muscle_run<0, kPow, G>(M, St, S, act_row, mb, pw, lane, last, M.seg_run[0], M.seg_run[1]);
    if constexpr (NSEG >= 1) muscle_run<1, kPow, G>(M, St, S, act_row, mb, pw, lane, last, M.seg_run[1], M.seg_run[2]);
    if constexpr (NSEG >= 2) muscle_run<2, kPow, G>(M, St, S, act_row, mb, pw, lane, last, M.seg_run[2], M.seg_run[3]);
    if constexpr (NSEG >= 3) muscle_run<3, kPow, G>(M, St, S, act_row, mb, pw, lane, last, M.seg_run[3], M.seg_run[4]);
    if constexpr (NSEG >= 4) muscle_run<4, kPow, G>(M, St, S, act_row, mb, pw, lane, last, M.seg_run[4], M.seg_run[5]);
}

template <int NSEG, int G = 32>
__device__ __forceinline__ void muscle_phase(const DevModel& M, const DevState& St, const EnvSmem& S,
                                             const float* act_row, size_t mb, float* pw, int lane, bool last) {
    if constexpr (NSEG > 0) {
        if (pw)
            muscle_runs<NSEG, true, G>(M, St, S, act_row, mb, pw, lane, last);
        else
            muscle_runs<NSEG, false, G>(M, St, S, act_row, mb, pw, lane, last);
        // general muscles follow from M.gen0
        if (M.gen0 < M.nm) muscle_generic(M, St, S, act_row, mb, pw, lane, last, M.gen0);
    } else {
        muscle_generic(M, St, S, act_row, mb, pw, lane, last, 0);
    }
}

// Joint torques J_m^T F from the moment slots in a fixed summation order, in two
// parts (capi.cu plan_torques).  piece_sums: each lane runs down its list of
// slots (element i at slot i G + lane: conflict-free) and stores every piece's
// partial sum into the link-frame scratch (frames are dead between the
// integration and the next tree sweep); joint_torque: a joint's pieces in piece
// order, then damping and the joint-limit spring (skeleton.cpp:271-290).
// The sums run in f64 (exact for up to ~2^29 f32 terms of similar magnitude):
// agonist / antagonist moments cancel, so an f32 chain of ~n_pairs / G terms
// would round visibly; the joint torque is rounded to f32 once.
__device__ __forceinline__ void piece_sums(const DevModel& M, const EnvSmem& S, int lane) {
    double* part = reinterpret_cast<double*>(S.kin);
    const uint8_t* fl = S.tqf + lane;
    const float* un = S.un + lane;
    const int G = S.G, n = M.tq_len;
    double acc = 0.0;
#pragma unroll 4
    for (int i = 0; i < n; ++i) {
        acc += static_cast<double>(un[i * G]);
        const int f = fl[i * G];
        if (f != 0xff) {
            part[f] = acc;
            acc = 0.0;
        }
    }
}

__device__ __forceinline__ float joint_torque(const DevModel& M, const EnvSmem& S, int j, double q, double dq) {
    const double* part = reinterpret_cast<const double*>(S.kin);
    const int p1 = S.tqp[j + 1];
    double ts = 0.0;
    for (int p = S.tqp[j]; p < p1; ++p) ts += part[p];
    float t = static_cast<float>(ts);
    t -= __ldg(M.joint_damping + j) * static_cast<float>(dq);
    const double hi = __ldg(M.joint_hi + j), lo = __ldg(M.joint_lo + j);
    if (q > hi)
        t -= static_cast<float>(M.k_lim_d * (q - hi));
    else if (q < lo)
        t -= static_cast<float>(M.k_lim_d * (q - lo));
    return t;
}

// Articulated-body pass, leaves -> root (per link U = IA e0, D, Schur
// complement, shift to the parent origin; children summed in fixed order).
// A link's articulated inertia and bias shifted to its parent's origin (the
// parent's children sum): forwarded in registers along a chain (aba_up_chain).
struct UpRec {
    float2 r0, r1, r2, r3;
    float p2;
};

// kFwdIn: the link's only child's shifted record comes in registers (chain);
// kStoreOut: the shifted record goes to shared memory for a parent in another
// lane / super-level (else it is only returned).
template <bool kSimple, bool kFwdIn = false, bool kStoreOut = true>
__device__ __forceinline__ UpRec aba_up_link(const DevModel& M, const EnvSmem& S, uint32_t ww, int dofoff,
                                             const UpRec& child = UpRec{}) {
    const int l = ww_link(ww);
    float* u = S.un + kLinkStride * l;
    float2* u2 = reinterpret_cast<float2*>(u);
    float2 r0 = u2[0], r1 = u2[1], r2 = u2[2], r3 = u2[3];
    float P2 = u[8];
    if constexpr (kFwdIn) {
        r0.x += child.r0.x;
        r0.y += child.r0.y;
        r1.x += child.r1.x;
        r1.y += child.r1.y;
        r2.x += child.r2.x;
        r2.y += child.r2.y;
        r3.x += child.r3.x;
        r3.y += child.r3.y;
        P2 += child.p2;
    } else {
        const int c0 = ww_child0(ww), c1 = c0 + ww_nchild(ww);
#pragma unroll 1  // mostly one child: an unrolled 4/2/1 cascade costs more branches than it saves (A/B +1.8 %)
        for (int c = c0; c < c1; ++c) {
            const float* uc = S.un + kLinkStride * S.tchild[c];
            const float2* uc2 = reinterpret_cast<const float2*>(uc);
            const float2 a0 = uc2[0], a1 = uc2[1], a2 = uc2[2], a3 = uc2[3];
            r0.x += a0.x;
            r0.y += a0.y;
            r1.x += a1.x;
            r1.y += a1.y;
            r2.x += a2.x;
            r2.y += a2.y;
            r3.x += a3.x;
            r3.y += a3.y;
            P2 += uc[8];
        }
    }
    const float I00 = r0.x, I01 = r0.y, I02 = r1.x, I11 = r1.y, I12 = r2.x, I22 = r2.y;
    const float P0 = r3.x, P1 = r3.y;
    const int dof = kSimple ? l + dofoff : link_dof(M, l);
    if (!kSimple && dof < 0) {  // floating root keeps its full articulated inertia
        u2[0] = r0;
        u2[1] = r1;
        u2[2] = r2;
        u2[3] = r3;
        u[8] = P2;
        return UpRec{};
    }
    // hinge with S = (1,0,0) at the link origin: U = IA[:,0], D = U0
    const float invD = rcp_ftz(I00);  // (IEEE 1/x costs a range check + slow-path call)
    const float t = S.tau[dof];
    const float uu = (t - P0) * invD;               // u / D
    const float U1 = I01 * invD, U2 = I02 * invD;   // U / D
    const float a = fmaf(-I01, U1, I11);            // Ia = IA - U U^T / D
    const float bb = fmaf(-I01, U2, I12);
    const float cq = fmaf(-I02, U2, I22);
    const float2 cv = u2[6];
    // pa = pA + Ia c + U u / D   (pa[0] = tau)
    const float q1 = fmaf(I01, uu, fmaf(a, cv.x, fmaf(bb, cv.y, P1)));
    const float q2 = fmaf(I02, uu, fmaf(bb, cv.x, fmaf(cq, cv.y, P2)));
    u[9] = uu;
    u2[5] = make_float2(U1, U2);
    const int p = ww_parent(ww);
    UpRec out{};
    if (kSimple || p >= 0) {  // shift to the parent's origin: X^T Ia X, X^T pa
        const float2 d = frame_rel(S, l);  // origin relative to the parent's
        const float dx = d.x, dz = d.y;
        const float al = fmaf(-a, dz, bb * dx), be = fmaf(-bb, dz, cq * dx);
        out.r0 = make_float2(fmaf(-dz, al, be * dx), al);
        out.r1 = make_float2(be, a);
        out.r2 = make_float2(bb, cq);
        out.r3 = make_float2(fmaf(-dz, q1, fmaf(dx, q2, t)), q1);
        out.p2 = q2;
        if (kStoreOut) {
            u2[0] = out.r0;
            u2[1] = out.r1;
            u2[2] = out.r2;
            u2[3] = out.r3;
            u[8] = out.p2;
        }
    }
    return out;
}

// aba_up over super-levels, bottom up (one slot per lane: G = 32): each lane
// takes its slot's chain from the deepest link (children, in the next
// super-level, summed from shared memory) up to the super-level's first link,
// each link's only child's shifted record forwarded in registers; only the
// first link's record (its parent sits in another super-level) is stored.
__device__ __forceinline__ void aba_up_chain(const DevModel& M, const EnvSmem& S, int lane) {
    const int dofoff = M.nrd - M.floating;
    for (int end = M.n_levels; end > 0;) {
        const int lev = S.tslstart[end - 1];  // the super-level's first level
        const uint32_t wl = S.twork[32 * (end - 1) + lane];
        if (lev == end - 1) {  // a single level: children from shared memory, record stored
            if (wl >> 31) {
                if ((wl >> 29) & 1)
                    aba_up_link<true>(M, S, wl, dofoff);
                else
                    aba_up_link<false>(M, S, wl, dofoff);
            }
        } else {
            // deepest level (children in the next super-level); a chain that ends higher up
            // ends in a leaf, whose forwarded child record is zero
            UpRec rc{};
            if (wl >> 31) rc = aba_up_link<true, false, false>(M, S, wl, dofoff);  // chain levels are simple
            for (int d = end - 2; d > lev; --d) {
                const uint32_t ww = S.twork[32 * d + lane];
                if (ww >> 31) rc = aba_up_link<true, true, false>(M, S, ww, dofoff, rc);
            }
            const uint32_t wt = S.twork[32 * lev + lane];
            if (wt >> 31) {
                if ((wt >> 29) & 1)
                    aba_up_link<true, true, true>(M, S, wt, dofoff, rc);
                else
                    aba_up_link<false, true, true>(M, S, wt, dofoff, rc);
            }
        }
        __syncwarp(S.hm);
        end = lev;
    }
}

__device__ __forceinline__ void aba_up(const DevModel& M, const EnvSmem& S, int lane) {
    const int dofoff = M.nrd - M.floating;
    for (int lev = M.n_levels - 1; lev >= 0; --lev) {
        for (int i = lane; i < 32; i += S.G) {
            const uint32_t ww = S.twork[32 * lev + i];
            if (!(ww >> 31)) continue;
            if ((ww >> 29) & 1)
                aba_up_link<true>(M, S, ww, dofoff);
            else
                aba_up_link<false>(M, S, ww, dofoff);
        }
        __syncwarp(S.hm);
    }
}

// A link's spatial acceleration terms {A0 + q̈, A1, A2} as its children read them.
struct DownPar {
    float a0, a1, a2;
};

// One link of the root-to-leaf articulated-body pass: q̈ into S.tau.  kFwd:
// the parent's terms come in registers (chain); store: its children read them
// from shared memory (another lane / super-level).
template <bool kSimple, bool kFwd = false>
__device__ __forceinline__ DownPar aba_down_link(const DevModel& M, const EnvSmem& S, uint32_t ww, int dofoff,
                                                 const DownPar& par = DownPar{}, bool store = true) {
    const int l = ww_link(ww);
    const int dof = kSimple ? l + dofoff : link_dof(M, l);
    float* u = S.un + kLinkStride * l;
    if (!kSimple && dof < 0) return DownPar{u[0], u[1], u[2]};  // floating root: the root solve's terms
    const int p = ww_parent(ww);
    float2* u2 = reinterpret_cast<float2*>(u);
    const float2 cv = u2[6];
    float A0 = 0.0f, A1 = cv.x, A2 = cv.y;
    if (kSimple || p >= 0) {
        float2 a01;
        float a2;
        if constexpr (kFwd) {
            a01 = make_float2(par.a0, par.a1);
            a2 = par.a2;
        } else {
            const float* up = S.un + kLinkStride * p;
            a01 = reinterpret_cast<const float2*>(up)[0];
            a2 = up[2];
        }
        const float2 d = frame_rel(S, l);  // origin relative to the parent's
        const float dx = d.x, dz = d.y;
        A0 = a01.x;
        A1 += fmaf(-a01.x, dz, a01.y);
        A2 += fmaf(a01.x, dx, a2);
    }
    // q̈ = (u - U^T A) / D with U0 = D
    const float2 U = u2[5];
    const float qdd = u[9] - A0 - fmaf(U.x, A1, U.y * A2);
    if (store) {
        u2[0] = make_float2(A0 + qdd, A1);
        u[2] = A2;
    }
    S.tau[dof] = qdd;
    return DownPar{A0 + qdd, A1, A2};
}

// Floating root (link 0): solve IA A = -pA (3x3 SPD, Cholesky with reciprocal
// pivots) and the root's coordinate accelerations.
__device__ __forceinline__ void root_solve(const EnvSmem& S) {
    {
        float* u = S.un;
        const float i00 = rsqrt_ftz(u[0]);
        const float l10 = u[1] * i00, l20 = u[2] * i00;
        const float i11 = rsqrt_ftz(u[3] - l10 * l10);
        const float l21 = (u[4] - l20 * l10) * i11;
        const float i22 = rsqrt_ftz(u[5] - l20 * l20 - l21 * l21);
        const float y0 = -u[6] * i00;
        const float y1 = (-u[7] - l10 * y0) * i11;
        const float y2 = (-u[8] - l20 * y0 - l21 * y1) * i22;
        const float x2 = y2 * i22;
        const float x1 = (y1 - l21 * x2) * i11;
        const float x0 = (y0 - l10 * x1 - l20 * x2) * i00;
        u[0] = x0;
        u[1] = x1;
        u[2] = x2;
        // spatial -> coordinate acceleration of the root (x, z, pitch)
        const float wd = S.dqf[2];
        S.tau[0] = fmaf(-wd, S.dqf[1], x1);
        S.tau[1] = fmaf(wd, S.dqf[0], x2);
        S.tau[2] = x0;
    }
}

// Floating-root solve (3x3 Cholesky) + articulated-body pass, root -> leaves:
// q̈ into S.tau.
__device__ __forceinline__ void aba_down(const DevModel& M, const EnvSmem& S, int lane) {
    const int dofoff = M.nrd - M.floating;
    if (M.floating && lane == 0) root_solve(S);
    __syncwarp(S.hm);
    for (int lev = 0; lev < M.n_levels; ++lev) {
        for (int i = lane; i < 32; i += S.G) {
            const uint32_t ww = S.twork[32 * lev + i];
            if (!(ww >> 31)) continue;
            if ((ww >> 29) & 1)
                aba_down_link<true>(M, S, ww, dofoff);
            else
                aba_down_link<false>(M, S, ww, dofoff);
        }
        __syncwarp(S.hm);
    }
}

// aba_down over super-levels (one slot per lane: G = 32); the root solve first.
__device__ __forceinline__ void aba_down_chain(const DevModel& M, const EnvSmem& S, int lane) {
    const int dofoff = M.nrd - M.floating;
    if (M.floating && lane == 0) root_solve(S);
    __syncwarp(S.hm);
    for (int lev = 0; lev < M.n_levels;) {
        const int end = superlevel_end(M, S, lev);
        uint32_t ww = S.twork[32 * lev + lane];
        if (ww >> 31) {
            DownPar par = ((ww >> 29) & 1) ? aba_down_link<true>(M, S, ww, dofoff, DownPar{}, lev == end - 1)
                                           : aba_down_link<false>(M, S, ww, dofoff, DownPar{}, lev == end - 1);
            for (int d = lev + 1; d < end; ++d) {
                ww = S.twork[32 * d + lane];
                if (!(ww >> 31)) break;
                par = aba_down_link<true, true>(M, S, ww, dofoff, par, d == end - 1);
            }
        }
        __syncwarp(S.hm);
        lev = end;
    }
}

// Loads an env's q, dq (f64) into the DOF-owning lanes.
template <int QS>
__device__ __forceinline__ void load_dofs(const DevModel& M, const EnvSmem& S, const double* q, const double* dq,
                                          double* qd, double* dqd, int lane) {
#pragma unroll
    for (int k = 0; k < QS; ++k) {
        const int d = lane + S.G * k;
        qd[k] = d < M.nq ? q[d] : 0.0;
        dqd[k] = d < M.nq ? dq[d] : 0.0;
    }
}

// f64 q into the union scratch for the Δ / observation epilogue.
template <int QS>
__device__ __forceinline__ double* stage_q(const DevModel& M, const EnvSmem& S, const double* qd, int lane) {
    double* qsm = reinterpret_cast<double*>(S.un);
#pragma unroll
    for (int k = 0; k < QS; ++k) {
        const int d = lane + S.G * k;
        if (d < M.nq) qsm[d] = qd[k];
    }
    __syncwarp(S.hm);
    return qsm;
}

// Env epilogue of a control step (env.cpp:214-262): state write-back, then for a
// diverged env zeroed outputs and the failure flag, else Δ, observation,
// reward_aux, termination and the episode outcome.  Shared by the step kernels.
template <int QS>
__device__ __forceinline__ void step_epilogue(const DevModel& M, const DevState& St, const EnvSmem& S, int e, int le,
                                              const double (&qd)[QS], const double (&dqd)[QS], int diverged_at,
                                              int n_substeps, float* obs, float* delta, float* reward_aux,
                                              uint8_t* flags, float* power, float* grf_row, float* pw, int lane) {
    const int nq = M.nq, nm = M.nm, nl = M.nl;
    const size_t mb = static_cast<size_t>(e) * nm;
    // ---- write back the simulation state ----
#pragma unroll
    for (int k = 0; k < QS; ++k) {
        const int d = lane + S.G * k;
        if (d < nq) {
            St.q[static_cast<size_t>(e) * nq + d] = qd[k];
            St.dq[static_cast<size_t>(e) * nq + d] = dqd[k];
        }
    }
    const int n_sub = diverged_at >= 0 ? diverged_at + 1 : n_substeps;
    if (lane == 0) {
        double t = St.t[e];
        for (int s = 0; s < n_sub; ++s) t += kSimDt;
        St.t[e] = t;
    }
    if (n_substeps != kSubsteps) return;  // msk_gpu_substeps: continuous state only
    const int obs_dim = 3 * nq + 6 * M.nk + 4 * nm;
    const int ddim = 3 + M.nj + 2 * M.nk;
    float* obs_row = obs ? obs + static_cast<size_t>(le) * obs_dim : nullptr;
    float* drow = delta ? delta + static_cast<size_t>(le) * ddim : nullptr;

    if (diverged_at >= 0) {  // env.cpp:214-229
        if (obs_row)
            for (int i = lane; i < obs_dim; i += S.G) obs_row[i] = 0.0f;
        if (drow)
            for (int i = lane; i < ddim; i += S.G) drow[i] = 0.0f;
        if (power)
            for (int m = lane; m < nm; m += S.G) power[static_cast<size_t>(le) * nm + m] = 0.0f;
        if (grf_row)
            for (int i = lane; i < 2 * nl; i += S.G) grf_row[i] = 0.0f;
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

    // ---- env epilogue (env.cpp:231-262) ----
    const int t_index = St.t_index[e] + 1;
    const int steps = St.steps[e] + 1;
    tree_sweep<false>(M, S, lane, nullptr);
    const double* qsm = stage_q<QS>(M, S, qd, lane);
    const bool far = write_delta(M, S, qsm, t_index, drow, lane);
    if (obs_row) write_obs(M, St, S, qsm, e, t_index, obs_row, lane);

    float aux = 0.0f;
    if (M.reward_mode == 1 && M.n_emg > 0) {
        float s = 0.0f;
        for (int ch = lane; ch < M.n_emg_ch; ch += S.G) {
            const float d = static_cast<float>(M.clip_emg[static_cast<size_t>(t_index) * M.n_emg + ch]) -
                            St.act[mb + __ldg(M.emg_map + ch)];
            s = fmaf(d, d, s);
        }
        for (int o = S.G >> 1; o > 0; o >>= 1) s += __shfl_xor_sync(S.hm, s, o);
        aux = M.n_emg_ch > 0 ? M.w_emg * (-s / static_cast<float>(M.n_emg_ch)) : 0.0f;
    } else if (M.reward_mode == 2) {
        float s = 0.0f;
        for (int m = lane; m < nm; m += S.G) s += pw[m];
        for (int o = S.G >> 1; o > 0; o >>= 1) s += __shfl_xor_sync(S.hm, s, o);
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

}  // namespace

// ============================================================================
// Env::step's action handling (env.cpp:208-213) once per control step: the
// non-finite check (per-env flag) and the clamp to [0, 1], written in the
// device's muscle order so the 10 substeps read each warp's 32 excitations as
// one coalesced 128-B line instead of gathering them from the reference-order
// row every substep.  One warp per env: coalesced reads, row-local scatter.
// ============================================================================
__global__ void prep_actions_kernel(DevModel M, DevState St, int env0, int n_envs, const float* __restrict__ actions) {
    const int le = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (le >= n_envs) return;
    const int nm = M.nm, e = env0 + le;
    const float* row = actions + static_cast<size_t>(le) * nm;
    float* u = St.u + static_cast<size_t>(e) * nm;
    bool bad = false;
    for (int x = lane; x < nm; x += 32) {
        const float a = row[x];
        bad |= !isfinite(a);
        u[__ldg(M.m_int + x)] = fminf(fmaxf(a, 0.0f), 1.0f);
    }
    bad = __any_sync(0xffffffffu, bad);
    if (lane == 0) St.u_bad[e] = bad ? 1 : 0;
}

// ============================================================================
// step kernel: warp per env, WPB envs per block
// ============================================================================
// QSL: DOF register slots per lane (n_q <= 32 QSL); fewer slots, fewer live registers.
template <int WPB, int MINB, int NSEG, int EPW, int QSL>
__global__ void __launch_bounds__(WPB * 32, MINB) step_kernel(DevModel M, DevState St, int env0, int n_envs,
                                                              const float* __restrict__ actions, float* obs,
                                                              float* delta, float* reward_aux, uint8_t* flags,
                                                              float* power, float* grf, int n_substeps) {
    // n_substeps: kSubsteps for Env::step; fewer only for the msk_gpu_substeps
    // diagnostic (state advanced by that many substeps, no env epilogue)
    extern __shared__ __align__(16) unsigned char smem[];
    static_assert(QSL >= 1 && QSL <= kMaxQSlots, "DOF slots");
    constexpr int G = 32 / EPW, QS = QSL * EPW;
    const int warp = threadIdx.x >> 5, grp = (threadIdx.x & 31) / G, lane = threadIdx.x & (G - 1);
    const unsigned hm = EPW == 1 ? 0xffffffffu : (0xffffu << (16 * grp));
    const int slot = warp * EPW + grp;            // env slot of this block (< M.epb active)
    const int le = blockIdx.x * M.epb + slot;     // env index local to this launch
    load_tree_table(smem, M);
    if (slot >= M.epb || le >= n_envs) return;
    const int e = env0 + le;
    const EnvSmem S = carve(smem, warp * EPW + grp, M, G, hm);
    const int nq = M.nq, nm = M.nm, nl = M.nl, nrd = M.nrd;
    const size_t mb = static_cast<size_t>(e) * nm;
    const float* act_row = St.u + mb;  // this step's clamped excitations in device muscle order

    // Contract checks of Env::step (env.cpp:207-210): env untouched on failure.
    bool active = true;
    if (St.done[e]) {
        if (lane == 0 && flags) flags[le] = kFlagNotStepped;
        active = false;
    }
    if (active) {
        if (St.u_bad[e]) {
            if (lane == 0 && flags) flags[le] = kFlagBadAction;
            active = false;
        }
    }
    if (!active) return;

    double qd[QS], dqd[QS];
    load_dofs<QS>(M, S, St.q + static_cast<size_t>(e) * nq, St.dq + static_cast<size_t>(e) * nq, qd, dqd, lane);
    publish_dofs<QS>(M, S, qd, dqd, lane);
    float* pw = power ? power + static_cast<size_t>(le) * nm
                      : (M.reward_mode == 2 ? St.power_scratch + mb : nullptr);
    if (pw)
        for (int m = lane; m < nm; m += S.G) pw[m] = 0.0f;
    float* grf_row = grf ? grf + static_cast<size_t>(le) * 2 * nl : nullptr;
    if (grf_row)
        for (int i = lane; i < 2 * nl; i += S.G) grf_row[i] = 0.0f;
    __syncwarp(S.hm);

    PHASE_T0();
    int diverged_at = -1;
    for (int sub = 0; sub < n_substeps; ++sub) {
        if (M.has_general) fk_d(M, S, lane);  // f64 world frames of the general segments

        // ---- 1. muscles + J_m^T F contributions ----
        muscle_phase<NSEG, G>(M, St, S, act_row, mb, pw, lane, sub == n_substeps - 1);
        __syncwarp(S.hm);

        PHASE_MARK(0);
        // ---- 2. joint torques: fixed-order slot sums, damping, limits ----
        piece_sums(M, S, lane);
        __syncwarp(S.hm);
#pragma unroll
        for (int k = 0; k < QS; ++k) {
            const int d = lane + S.G * k;
            if (d >= nrd && d < nq) S.tau[d] = joint_torque(M, S, d - nrd, qd[k], dqd[k]);
        }
        __syncwarp(S.hm);

        PHASE_MARK(1);
        {
            // ---- 3. FK + velocities + per-link articulated-body terms ----
            if (M.ns) sphere_pen_d(M, S, lane);
            if constexpr (G == 32)  // one slot per lane: chains of levels in registers
                tree_sweep_chain(M, S, lane, grf_row);
            else
                tree_sweep<true>(M, S, lane, grf_row);

            PHASE_MARK(2);
            // ---- 4a. articulated-body pass, leaves -> root ----
            if constexpr (G == 32)
                aba_up_chain(M, S, lane);
            else
                aba_up(M, S, lane);

            PHASE_MARK(3);
            // ---- 4b. root solve + articulated-body pass, root -> leaves ----
            if constexpr (G == 32)
                aba_down_chain(M, S, lane);
            else
                aba_down(M, S, lane);
        }

        PHASE_MARK(4);
        // ---- 5. semi-implicit Euler (f64) + divergence check ----
        bool bad = false;
#pragma unroll
        for (int k = 0; k < QS; ++k) {
            const int d = lane + S.G * k;
            if (d < nq) {
                dqd[k] += static_cast<double>(S.tau[d]) * kSimDt;
                qd[k] += dqd[k] * kSimDt;
                bad |= !isfinite(qd[k]) || !isfinite(dqd[k]);
            }
        }
        __syncwarp(S.hm);
        publish_dofs<QS>(M, S, qd, dqd, lane);
        __syncwarp(S.hm);
        if (__any_sync(S.hm, bad)) {
            diverged_at = sub;
            break;
        }
    }

    PHASE_MARK(5);
    step_epilogue<QS>(M, St, S, e, le, qd, dqd, diverged_at, n_substeps, obs, delta, reward_aux, flags, power, grf_row,
                      pw, lane);
}

// ============================================================================
// step kernel with quad tree passes: one warp per env for the muscle phase,
// torques and integration (as step_kernel), but the three tree passes of Q env
// warps run on ONE warp of the group — 32/Q lanes per env (tree levels hold 1-11
// links), so their instructions serve Q envs while the other Q-1 warps free
// their issue slots.  Named barriers (one per group) order the phases; every
// warp runs every substep (inactive / diverged envs do no work but still meet
// the barriers).  Same per-env arithmetic as step_kernel.
// ============================================================================
template <int WPB, int Q, int NSEG, int QSL>
__global__ void __launch_bounds__(WPB * 32, 1) stepq_kernel(DevModel M, DevState St, int env0, int n_envs,
                                                             const float* __restrict__ actions, float* obs,
                                                             float* delta, float* reward_aux, uint8_t* flags,
                                                             float* power, float* grf, int n_substeps) {
    extern __shared__ __align__(16) unsigned char smem[];
    static_assert(QSL >= 1 && QSL <= kMaxQSlots, "DOF slots");
    static_assert(WPB % Q == 0 && (Q == 2 || Q == 4), "tree groups");
    constexpr int QS = QSL, GQ = 32 / Q;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int group = warp / Q;
    load_tree_table(smem, M);
    const int nq = M.nq, nm = M.nm, nl = M.nl, nrd = M.nrd;
    const auto group_bar = [&]() { asm volatile("bar.sync %0, %1;" ::"r"(1 + group), "n"(Q * 32) : "memory"); };

    // this warp's env (muscle phase / integration / epilogue)
    const int slot = warp;
    const bool has_slot = slot < M.epb;
    const int le = blockIdx.x * M.epb + slot;
    const bool exists = has_slot && le < n_envs;
    const int e = env0 + (exists ? le : 0);
    bool live = exists;
    if (live && St.done[e]) {  // contract checks of Env::step (env.cpp:207-210)
        if (lane == 0 && flags) flags[le] = kFlagNotStepped;
        live = false;
    }
    if (live && St.u_bad[e]) {
        if (lane == 0 && flags) flags[le] = kFlagBadAction;
        live = false;
    }
    const bool stepped = live;
    const EnvSmem S = carve(smem, has_slot ? slot : 0, M, 32, 0xffffffffu);
    const size_t mb = static_cast<size_t>(e) * nm;
    const float* act_row = St.u + mb;
    float* pw = nullptr;
    float* grf_row = nullptr;
    double qd[QS], dqd[QS];
    if (stepped) {
        pw = power ? power + static_cast<size_t>(le) * nm : (M.reward_mode == 2 ? St.power_scratch + mb : nullptr);
        grf_row = grf ? grf + static_cast<size_t>(le) * 2 * nl : nullptr;
        load_dofs<QS>(M, S, St.q + static_cast<size_t>(e) * nq, St.dq + static_cast<size_t>(e) * nq, qd, dqd, lane);
        publish_dofs<QS>(M, S, qd, dqd, lane);
        if (pw)
            for (int m = lane; m < nm; m += 32) pw[m] = 0.0f;
        if (grf_row)
            for (int i = lane; i < 2 * nl; i += 32) grf_row[i] = 0.0f;
    }
    __syncwarp();

    // the group's tree view (used by the group's first warp): env of lane group g
    const bool leader = (warp % Q) == 0;
    const int g = lane / GQ, glane = lane % GQ;
    const int tslot = group * Q + g;
    const int tle = blockIdx.x * M.epb + tslot;
    bool t_act = tslot < M.epb && tle < n_envs;  // the tree pass of an existing env slot
    float* tgrf = nullptr;
    if (leader && t_act) {
        const int te = env0 + tle;
        const bool t_step = !St.done[te] && !St.u_bad[te];
        tgrf = (grf && t_step) ? grf + static_cast<size_t>(tle) * 2 * nl : nullptr;
    }
    const EnvSmem ST = carve(smem, t_act ? tslot : 0, M, GQ, (GQ == 32 ? 0xffffffffu : ((1u << GQ) - 1u) << (GQ * g)));

    int diverged_at = -1;
    for (int sub = 0; sub < n_substeps; ++sub) {
        if (live) {
            if (M.has_general) fk_d(M, S, lane);
            muscle_phase<NSEG>(M, St, S, act_row, mb, pw, lane, sub == n_substeps - 1);
            __syncwarp();
            piece_sums(M, S, lane);  // joint torques: fixed-order slot sums, damping, limits
            __syncwarp();
#pragma unroll
            for (int k = 0; k < QS; ++k) {
                const int d = lane + 32 * k;
                if (d >= nrd && d < nq) S.tau[d] = joint_torque(M, S, d - nrd, qd[k], dqd[k]);
            }
        }
        group_bar();  // the group's torques and joint states are in shared memory
        if (leader && t_act) {
            if (M.ns) sphere_pen_d(M, ST, glane);
            tree_sweep<true>(M, ST, glane, tgrf);
            aba_up(M, ST, glane);
            aba_down(M, ST, glane);
        }
        group_bar();  // q̈ of every env of the group is in shared memory
        if (live) {
            bool bad = false;
#pragma unroll
            for (int k = 0; k < QS; ++k) {
                const int d = lane + 32 * k;
                if (d < nq) {
                    dqd[k] += static_cast<double>(S.tau[d]) * kSimDt;
                    qd[k] += dqd[k] * kSimDt;
                    bad |= !isfinite(qd[k]) || !isfinite(dqd[k]);
                }
            }
            __syncwarp();
            publish_dofs<QS>(M, S, qd, dqd, lane);
            __syncwarp();
            if (__any_sync(0xffffffffu, bad)) {
                diverged_at = sub;
                live = false;  // frozen at the diverging substep (msk::step throws there)
            }
        }
    }
    if (stepped)
        step_epilogue<QS>(M, St, S, e, le, qd, dqd, diverged_at, n_substeps, obs, delta, reward_aux, flags, power,
                          grf_row, pw, lane);
}

// ============================================================================
// step kernel, NE envs per thread ("env-vectorised"): every lane of a warp
// advances NE environments at once — muscle constants, tree tables, work words,
// loop control and address arithmetic are shared by the NE envs, and each
// thread carries NE independent dependency chains (ILP instead of warps).
// Same arithmetic per env as step_kernel (bit-identical results); a block is
// WPB warps x NE env slots (slot = warp * NE + k).
// ============================================================================
namespace {

template <int NE>
struct EnvRowsN {
    MuscleRows R[NE];
    float* pw[NE];
    bool live[NE];
};

// One muscle (device index m, NS segments) for the NE envs.
template <int NS, int NE>
__device__ __forceinline__ void muscle_one_n(const DevModel& M, const EnvRowsN<NE>& V, const EnvSmem (&S)[NE], int m,
                                             bool last) {
    const int nm = M.nm;
    float4 kc[NS > 0 ? NS : 1];
#pragma unroll
    for (int k = 0; k < NS; ++k) kc[k] = ldc4(M.seg_kf + k * nm + m);
    const float4 p0 = ldc4(M.m_p0 + m);
    const double2 pa = ldc2d(M.m_p1a + m), pb = ldc2d(M.m_p1b + m);
    bool anypw = false;
#pragma unroll
    for (int e = 0; e < NE; ++e) anypw |= V.pw[e] != nullptr;
    const int ext = anypw ? (__ldg(M.m_meta + m) >> 9) : 0;
    float u[NE], a0[NE];
    double lm0[NE];
#pragma unroll
    for (int e = 0; e < NE; ++e) {
        u[e] = V.R[e].u[m];
        a0[e] = V.R[e].act[m];
        lm0[e] = V.R[e].lm[m];
    }
#pragma unroll
    for (int e = 0; e < NE; ++e) {
        double L = 0.0;
        float tq[NS > 0 ? NS : 1];
#pragma unroll
        for (int k = 0; k < NS; ++k) L += kseg(S[e], kc[k], __float_as_int(kc[k].w), tq[k]);
        // activation + fibre kinematics + Hill force (muscle_update), state stores gated by live
        const float gain = fmaf(1.5f, a0[e], 0.5f);
        const float ex = ex2_ftz(u[e] > a0[e] ? p0.y * rcp_ftz(gain) : p0.z * gain);
        const float a1 = fminf(fmaxf(fmaf(a0[e] - u[e], ex, u[e]), 0.0f), 1.0f);
        const double prev_len = fma(lm0[e], pa.y, pa.x);
        const float vm = static_cast<float>((L - prev_len) * pb.y);
        const double lm1 = fiber_clamp((L - pa.x) * pb.x);
        const float F = mtu_force(a1, static_cast<float>(lm1), vm, p0.x);
        if (V.live[e]) {
            V.R[e].act[m] = a1;
            V.R[e].lm[m] = lm1;
            if (last) {
                V.R[e].vm[m] = vm;
                V.R[e].fm[m] = F;
            }
            if (V.pw[e]) V.pw[e][ext] += fabsf(F * vm * p0.w);
        }
#pragma unroll
        for (int k = 0; k < NS; ++k) S[e].un[__float_as_int(kc[k].w) >> 11] = -F * tq[k];
    }
}

template <int NS, int NE>
__device__ __forceinline__ void muscle_run_n(const DevModel& M, const EnvRowsN<NE>& V, const EnvSmem (&S)[NE], int lane,
                                             bool last, int m0, int m1) {
    if (m0 + lane >= m1) return;
    for (int m = m0 + lane; m < m1; m += 32) muscle_one_n<NS, NE>(M, V, S, m, last);
}

template <int NSEG, int NE>
__device__ __forceinline__ void muscle_phase_n(const DevModel& M, const DevState& St, const EnvSmem (&S)[NE],
                                               const EnvRowsN<NE>& V, const size_t (&mb)[NE], int lane, bool last) {
    if constexpr (NSEG > 0) {
        muscle_run_n<0, NE>(M, V, S, lane, last, M.seg_run[0], M.seg_run[1]);
        if constexpr (NSEG >= 1) muscle_run_n<1, NE>(M, V, S, lane, last, M.seg_run[1], M.seg_run[2]);
        if constexpr (NSEG >= 2) muscle_run_n<2, NE>(M, V, S, lane, last, M.seg_run[2], M.seg_run[3]);
        if constexpr (NSEG >= 3) muscle_run_n<3, NE>(M, V, S, lane, last, M.seg_run[3], M.seg_run[4]);
        if constexpr (NSEG >= 4) muscle_run_n<4, NE>(M, V, S, lane, last, M.seg_run[4], M.seg_run[5]);
        if (M.gen0 < M.nm)  // general muscles: the single-env generic loop per live env
#pragma unroll
            for (int e = 0; e < NE; ++e)
                if (V.live[e]) muscle_generic(M, St, S[e], V.R[e].u, mb[e], V.pw[e], lane, last, M.gen0);
    } else {  // generic segments: the single-env path per live env
#pragma unroll
        for (int e = 0; e < NE; ++e)
            if (V.live[e]) muscle_phase<0>(M, St, S[e], V.R[e].u, mb[e], V.pw[e], lane, last);
    }
}

// Root-to-leaf sweep (tree_sweep<true>) for NE envs: the link's table entries,
// work word and parent index are read once.
template <int NE>
__device__ __forceinline__ void tree_sweep_n(const DevModel& M, const EnvSmem (&S)[NE], int lane, float* const (&grf)[NE]) {
    const EnvSmem& S0 = S[0];
    for (int lev = 0; lev < M.n_levels; ++lev) {
        const uint32_t ww = S0.twork[32 * lev + lane];
        if (ww >> 31) {
            const int l = ww_link(ww);
            const int dof = link_dof(M, l);
            const int p = ww_parent(ww);
            const float4 la = S0.ta[l];
            const float m = la.w, I = S0.tin[l], mg = m * M.gravity;
#pragma unroll
            for (int e = 0; e < NE; ++e) {
                float c, s, ox, oz, w, vx = 0.0f, vz = 0.0f;
                if (dof < 0) {  // floating root: origin (0,0) relative, pitch q2
                    c = S[e].root[2];
                    s = S[e].root[3];
                    ox = 0.0f;
                    oz = 0.0f;
                    w = S[e].dqf[2];
                    vx = S[e].dqf[0];
                    vz = S[e].dqf[1];
                } else {
                    const double2 rd = S[e].relcs[dof];
                    const float cr = static_cast<float>(rd.x), sr = static_cast<float>(rd.y);
                    w = S[e].dqf[dof];
                    if (p >= 0) {
                        const float4 kp = S[e].kin[p];
                        ox = fmaf(kp.x, la.x, fmaf(-kp.y, la.y, kp.z));
                        oz = fmaf(kp.y, la.x, fmaf(kp.x, la.y, kp.w));
                        c = fmaf(kp.x, cr, -kp.y * sr);
                        s = fmaf(kp.y, cr, kp.x * sr);
                        const float* up = S[e].un + kLinkStride * p;
                        const float2 wv = reinterpret_cast<const float2*>(up)[5];  // parent (omega, v_x)
                        w += wv.x;
                        vx = fmaf(-wv.x, oz - kp.w, wv.y);
                        vz = fmaf(wv.x, ox - kp.z, up[9]);
                    } else {
                        ox = la.x;
                        oz = la.y;
                        c = cr;
                        s = sr;
                    }
                }
                S[e].kin[l] = make_float4(c, s, ox, oz);
                float* u = S[e].un + kLinkStride * l;
                reinterpret_cast<float2*>(u)[5] = make_float2(w, vx);
                u[9] = vz;
                const float cx = la.z * c, cz = la.z * s;
                const float i00 = I, i01 = -m * cz, i02 = m * cx;
                const float h1 = fmaf(i01, w, m * vx), h2 = fmaf(i02, w, m * vz);
                float p0 = fmaf(vx, h2, -vz * h1) - cx * mg, p1 = -w * h2, p2 = fmaf(w, h1, -mg);
                if ((ww >> 28) & 1) {  // link carries contact spheres
                    const int s0 = __ldg(M.sphere_start + l), s1 = __ldg(M.sphere_start + l + 1);
                    float gx = 0.0f, gz = 0.0f;
                    for (int sp = s0; sp < s1; ++sp) {
                        const float4 sd = __ldg(M.sphere + sp);
                        const float rx = fmaf(c, sd.x, -s * sd.y), rz = fmaf(s, sd.x, c * sd.y);
                        const float pen = S[e].pen[sp];
                        if (pen > 0.0f) {
                            const float fn = fmaxf(0.0f, fmaf(M.c_k, pen, -M.c_c * fmaf(w, rx, vz)));
                            if (fn > 0.0f) {
                                const float qz = rz - sd.z;
                                const float ft = -M.c_mu * fn * tanhf(fmaf(-w, qz, vx) * M.inv_c_vs);
                                p0 -= fmaf(rx, fn, -qz * ft);
                                p1 -= ft;
                                p2 -= fn;
                                gx += ft * 0.1f;
                                gz += fn * 0.1f;
                            }
                        }
                    }
                    if (grf[e]) {
                        grf[e][2 * l] += gx;
                        grf[e][2 * l + 1] += gz;
                    }
                }
                float c1 = 0.0f, c2 = 0.0f;
                if (dof >= 0) {
                    const float qdot = S[e].dqf[dof];
                    c1 = qdot * vz;
                    c2 = -qdot * vx;
                }
                float2* u2 = reinterpret_cast<float2*>(u);
                u2[0] = make_float2(i00, i01);
                u2[1] = make_float2(i02, m);
                u2[2] = make_float2(0.0f, m);
                u2[3] = make_float2(p0, p1);
                u[8] = p2;
                u2[6] = make_float2(c1, c2);
            }
        }
        __syncwarp();
    }
}

// Articulated-body pass, leaves -> root (aba_up) for NE envs.
template <int NE>
__device__ __forceinline__ void aba_up_n(const DevModel& M, const EnvSmem (&S)[NE], int lane) {
    const EnvSmem& S0 = S[0];
    for (int lev = M.n_levels - 1; lev >= 0; --lev) {
        const uint32_t ww = S0.twork[32 * lev + lane];
        if (ww >> 31) {
            const int l = ww_link(ww);
            const int c0 = ww_child0(ww), c1 = c0 + ww_nchild(ww);
            const int dof = link_dof(M, l);
            const int p = ww_parent(ww);
            float dx = 0.0f, dz = 0.0f;
#pragma unroll
            for (int e = 0; e < NE; ++e) {
                float* u = S[e].un + kLinkStride * l;
                float2* u2 = reinterpret_cast<float2*>(u);
                float2 r0 = u2[0], r1 = u2[1], r2 = u2[2], r3 = u2[3];
                float P2 = u[8];
#pragma unroll 1
                for (int c = c0; c < c1; ++c) {
                    const float* uc = S[e].un + kLinkStride * S0.tchild[c];
                    const float2* uc2 = reinterpret_cast<const float2*>(uc);
                    const float2 a0 = uc2[0], a1 = uc2[1], a2 = uc2[2], a3 = uc2[3];
                    r0.x += a0.x;
                    r0.y += a0.y;
                    r1.x += a1.x;
                    r1.y += a1.y;
                    r2.x += a2.x;
                    r2.y += a2.y;
                    r3.x += a3.x;
                    r3.y += a3.y;
                    P2 += uc[8];
                }
                if (dof < 0) {  // floating root keeps its full articulated inertia
                    u2[0] = r0;
                    u2[1] = r1;
                    u2[2] = r2;
                    u2[3] = r3;
                    u[8] = P2;
                    continue;
                }
                const float I00 = r0.x, I01 = r0.y, I02 = r1.x, I11 = r1.y, I12 = r2.x, I22 = r2.y;
                const float P0 = r3.x, P1 = r3.y;
                const float invD = rcp_ftz(I00);
                const float t = S[e].tau[dof];
                const float uu = (t - P0) * invD;
                const float U1 = I01 * invD, U2 = I02 * invD;
                const float a = fmaf(-I01, U1, I11);
                const float bb = fmaf(-I01, U2, I12);
                const float cq = fmaf(-I02, U2, I22);
                const float2 cv = u2[6];
                const float q1 = fmaf(I01, uu, fmaf(a, cv.x, fmaf(bb, cv.y, P1)));
                const float q2 = fmaf(I02, uu, fmaf(bb, cv.x, fmaf(cq, cv.y, P2)));
                u[9] = uu;
                u2[5] = make_float2(U1, U2);
                if (p >= 0) {  // shift to the parent's origin: X^T Ia X, X^T pa
                    const float2 ol = frame_origin(S[e], l), op = frame_origin(S[e], p);
                    dx = ol.x - op.x;
                    dz = ol.y - op.y;
                    const float al = fmaf(-a, dz, bb * dx), be = fmaf(-bb, dz, cq * dx);
                    u2[0] = make_float2(fmaf(-dz, al, be * dx), al);
                    u2[1] = make_float2(be, a);
                    u2[2] = make_float2(bb, cq);
                    u2[3] = make_float2(fmaf(-dz, q1, fmaf(dx, q2, t)), q1);
                    u[8] = q2;
                }
            }
        }
        __syncwarp();
    }
}

// Floating-root solve + articulated-body pass, root -> leaves (aba_down) for NE envs.
template <int NE>
__device__ __forceinline__ void aba_down_n(const DevModel& M, const EnvSmem (&S)[NE], int lane) {
    if (M.floating && lane < NE) {  // one lane per env: the 3x3 root solve
#pragma unroll
        for (int e = 0; e < NE; ++e) {
            if (e != lane) continue;
            float* u = S[e].un;
            const float i00 = rsqrt_ftz(u[0]);
            const float l10 = u[1] * i00, l20 = u[2] * i00;
            const float i11 = rsqrt_ftz(u[3] - l10 * l10);
            const float l21 = (u[4] - l20 * l10) * i11;
            const float i22 = rsqrt_ftz(u[5] - l20 * l20 - l21 * l21);
            const float y0 = -u[6] * i00;
            const float y1 = (-u[7] - l10 * y0) * i11;
            const float y2 = (-u[8] - l20 * y0 - l21 * y1) * i22;
            const float x2 = y2 * i22;
            const float x1 = (y1 - l21 * x2) * i11;
            const float x0 = (y0 - l10 * x1 - l20 * x2) * i00;
            u[0] = x0;
            u[1] = x1;
            u[2] = x2;
            const float wd = S[e].dqf[2];
            S[e].tau[0] = fmaf(-wd, S[e].dqf[1], x1);
            S[e].tau[1] = fmaf(wd, S[e].dqf[0], x2);
            S[e].tau[2] = x0;
        }
    }
    __syncwarp();
    const EnvSmem& S0 = S[0];
    for (int lev = 0; lev < M.n_levels; ++lev) {
        const uint32_t ww = S0.twork[32 * lev + lane];
        if (ww >> 31) {
            const int l = ww_link(ww);
            const int dof = link_dof(M, l);
            const int p = ww_parent(ww);
            if (dof >= 0) {
#pragma unroll
                for (int e = 0; e < NE; ++e) {
                    float* u = S[e].un + kLinkStride * l;
                    float2* u2 = reinterpret_cast<float2*>(u);
                    const float2 cv = u2[6];
                    float A0 = 0.0f, A1 = cv.x, A2 = cv.y;
                    if (p >= 0) {
                        const float* up = S[e].un + kLinkStride * p;
                        const float2 a01 = reinterpret_cast<const float2*>(up)[0];
                        const float a2 = up[2];
                        const float2 ol = frame_origin(S[e], l), op = frame_origin(S[e], p);
                        const float dx = ol.x - op.x, dz = ol.y - op.y;
                        A0 = a01.x;
                        A1 += fmaf(-a01.x, dz, a01.y);
                        A2 += fmaf(a01.x, dx, a2);
                    }
                    const float2 U = u2[5];
                    const float qdd = u[9] - A0 - fmaf(U.x, A1, U.y * A2);
                    u2[0] = make_float2(A0 + qdd, A1);
                    u[2] = A2;
                    S[e].tau[dof] = qdd;
                }
            }
        }
        __syncwarp();
    }
}

}  // namespace

template <int WPB, int NE, int NSEG, int QSL>
__global__ void __launch_bounds__(WPB * 32, 1) stepn_kernel(DevModel M, DevState St, int env0, int n_envs,
                                                             const float* __restrict__ actions, float* obs,
                                                             float* delta, float* reward_aux, uint8_t* flags,
                                                             float* power, float* grf, int n_substeps) {
    extern __shared__ __align__(16) unsigned char smem[];
    static_assert(QSL >= 1 && QSL <= kMaxQSlots, "DOF slots");
    constexpr int QS = QSL;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    load_tree_table(smem, M);
    const int slot0 = warp * NE;
    if (slot0 >= M.epb) return;
    const int nq = M.nq, nm = M.nm, nl = M.nl, nrd = M.nrd;
    EnvSmem S[NE];
    EnvRowsN<NE> V;
    int le[NE], ev[NE];
    size_t mb[NE];
    bool exists[NE];
    float* grf_row[NE];
    int n_live = 0;
#pragma unroll
    for (int k = 0; k < NE; ++k) {
        const int slot = min(slot0 + k, M.epb - 1);
        S[k] = carve(smem, slot, M, 32, 0xffffffffu);
        le[k] = blockIdx.x * M.epb + slot0 + k;
        exists[k] = slot0 + k < M.epb && le[k] < n_envs;
        ev[k] = env0 + (exists[k] ? le[k] : min(le[0], n_envs - 1));  // loads of a missing env use a real row
        mb[k] = static_cast<size_t>(ev[k]) * nm;
        bool act = exists[k];
        if (act && St.done[ev[k]]) {  // contract checks of Env::step (env.cpp:207-210)
            if (lane == 0 && flags) flags[le[k]] = kFlagNotStepped;
            act = false;
        }
        if (act && St.u_bad[ev[k]]) {
            if (lane == 0 && flags) flags[le[k]] = kFlagBadAction;
            act = false;
        }
        V.live[k] = act;
        n_live += act;
        V.R[k] = muscle_rows(St, St.u + mb[k], mb[k]);
        V.pw[k] = power ? power + static_cast<size_t>(exists[k] ? le[k] : 0) * nm
                        : (M.reward_mode == 2 ? St.power_scratch + mb[k] : nullptr);
        grf_row[k] = (grf && exists[k]) ? grf + static_cast<size_t>(le[k]) * 2 * nl : nullptr;
    }
    if (n_live == 0) return;
    bool stepped[NE];
    double qd[NE][QS], dqd[NE][QS];
#pragma unroll
    for (int k = 0; k < NE; ++k) {
        stepped[k] = V.live[k];
        if (!V.live[k]) {  // not stepped: its caller rows stay untouched
            V.pw[k] = nullptr;
            grf_row[k] = nullptr;
        }
        load_dofs<QS>(M, S[k], St.q + static_cast<size_t>(ev[k]) * nq, St.dq + static_cast<size_t>(ev[k]) * nq, qd[k],
                      dqd[k], lane);
        publish_dofs<QS>(M, S[k], qd[k], dqd[k], lane);
        if (V.live[k] && V.pw[k])
            for (int m = lane; m < nm; m += 32) V.pw[k][m] = 0.0f;
        if (grf_row[k])
            for (int i = lane; i < 2 * nl; i += 32) grf_row[k][i] = 0.0f;
    }
    __syncwarp();

    int diverged_at[NE];
#pragma unroll
    for (int k = 0; k < NE; ++k) diverged_at[k] = -1;
    for (int sub = 0; sub < n_substeps; ++sub) {
        if (M.has_general)
#pragma unroll
            for (int k = 0; k < NE; ++k) fk_d(M, S[k], lane);

        // ---- 1. muscles + J_m^T F contributions ----
        muscle_phase_n<NSEG, NE>(M, St, S, V, mb, lane, sub == n_substeps - 1);
        __syncwarp();

        // ---- 2. joint torques: fixed-order slot sums, damping, limits ----
#pragma unroll
        for (int k = 0; k < NE; ++k) piece_sums(M, S[k], lane);
        __syncwarp();
#pragma unroll
        for (int kq = 0; kq < QS; ++kq) {
            const int d = lane + 32 * kq;
            if (d >= nrd && d < nq) {
#pragma unroll
                for (int k = 0; k < NE; ++k) S[k].tau[d] = joint_torque(M, S[k], d - nrd, qd[k][kq], dqd[k][kq]);
            }
        }
        __syncwarp();

        // ---- 3. FK + velocities + per-link articulated-body terms ----
        if (M.ns)
#pragma unroll
            for (int k = 0; k < NE; ++k) sphere_pen_d(M, S[k], lane);
        tree_sweep_n<NE>(M, S, lane, grf_row);
        // ---- 4. articulated-body passes ----
        aba_up_n<NE>(M, S, lane);
        aba_down_n<NE>(M, S, lane);

        // ---- 5. semi-implicit Euler (f64) + divergence check ----
        bool bad[NE];
#pragma unroll
        for (int k = 0; k < NE; ++k) {
            bad[k] = false;
            if (!V.live[k]) continue;
#pragma unroll
            for (int kq = 0; kq < QS; ++kq) {
                const int d = lane + 32 * kq;
                if (d < nq) {
                    dqd[k][kq] += static_cast<double>(S[k].tau[d]) * kSimDt;
                    qd[k][kq] += dqd[k][kq] * kSimDt;
                    bad[k] |= !isfinite(qd[k][kq]) || !isfinite(dqd[k][kq]);
                }
            }
        }
        __syncwarp();
        int alive = 0;
#pragma unroll
        for (int k = 0; k < NE; ++k) {
            if (V.live[k]) publish_dofs<QS>(M, S[k], qd[k], dqd[k], lane);
            if (V.live[k] && __any_sync(0xffffffffu, bad[k])) {
                diverged_at[k] = sub;
                V.live[k] = false;  // frozen at the diverging substep (msk::step throws there)
            }
            alive += V.live[k];
        }
        __syncwarp();
        if (alive == 0) break;
    }

#pragma unroll
    for (int k = 0; k < NE; ++k)
        if (stepped[k])
            step_epilogue<QS>(M, St, S[k], ev[k], le[k], qd[k], dqd[k], diverged_at[k], n_substeps, obs, delta,
                              reward_aux, flags, power, grf_row[k], V.pw[k], lane);
}

// ============================================================================
// reset / observe / tracking-error / force-to-reference: warp per env
// ============================================================================
enum ResetMode : int { kResetSample = 0, kResetFrame = 1, kResetForce = 2, kResetInit = 3 };

// Env::reset / reset_to_frame / force_state_to_reference / construction of env e
// by one warp (env slot S): frame choice, make_initial_state, observe.
template <int EPW>
__device__ __forceinline__ void reset_env(const DevModel& M, const DevState& St, const EnvSmem& S, int e, int mode,
                                          const int* frames_in, float* obs, int* frames_out, uint8_t* bad,
                                          int lane) {
    constexpr int QS = kMaxQSlots * EPW;
    const int nq = M.nq;
    int frame = 0;
    if (mode == kResetSample) {
        if (lane == 0) frame = M.rsi ? rsi_frame(M, St, e) : 0;
        frame = __shfl_sync(S.hm, frame, 0, S.G);
    } else if (mode == kResetFrame) {
        frame = frames_in[e];
        if (frame < 0 || frame >= M.frames - 1) {  // ContractError in env.cpp:96-97
            if (lane == 0 && bad) bad[e] = 1;
            return;  // (this env only)
        }
        if (lane == 0 && bad) bad[e] = 0;
    } else if (mode == kResetForce) {
        frame = St.t_index[e];
    }  // kResetInit: frame 0 (Env::Env, env.cpp:86)
    double qd[QS], dqd[QS];
    load_dofs<QS>(M, S, M.clip_q + static_cast<size_t>(frame) * nq, M.clip_dq + static_cast<size_t>(frame) * nq, qd, dqd,
              lane);
#pragma unroll
    for (int k = 0; k < QS; ++k) {
        const int d = lane + S.G * k;
        if (d < nq) {
            St.q[static_cast<size_t>(e) * nq + d] = qd[k];
            St.dq[static_cast<size_t>(e) * nq + d] = dqd[k];
        }
    }
    publish_dofs<QS>(M, S, qd, dqd, lane);
    __syncwarp(S.hm);
    tree_sweep<false>(M, S, lane, nullptr);  // (f32 frames for the observation)
    if (M.has_general) fk_d(M, S, lane);
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
        const double* qsm = stage_q<QS>(M, S, qd, lane);
        const int obs_dim = 3 * nq + 6 * M.nk + 4 * M.nm;
        write_obs(M, St, S, qsm, e, frame, obs + static_cast<size_t>(e) * obs_dim, lane);
    }
}

// Each block owns a contiguous range of at most kResetRange envs: it compacts
// the range's selected envs (mask & mask_bits; all when mask is null) in shared
// memory and its env slots work through them.  A masked auto-reset that selects
// a few envs per range thus runs in one wave over <= 148 blocks, instead of
// scheduling every block of the env grid (one per SM, 28 env slots of smem).
constexpr int kResetRange = 256;

template <int WPB, int MINB, int EPW>
__global__ void __launch_bounds__(WPB * 32, MINB) reset_kernel(DevModel M, DevState St, int n_envs, int range,
                                                               int mode, const uint8_t* mask, uint8_t mask_bits,
                                                               const int* frames_in, float* obs, int* frames_out,
                                                               uint8_t* bad) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ int s_list[kResetRange];
    __shared__ int s_cnt;
    constexpr int G = 32 / EPW;
    const int warp = threadIdx.x >> 5, grp = (threadIdx.x & 31) / G, lane = threadIdx.x & (G - 1);
    const unsigned hm = EPW == 1 ? 0xffffffffu : (0xffffu << (16 * grp));
    const int e0 = blockIdx.x * range, n_range = min(range, n_envs - e0);
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    // every env of the range is visited whatever the block size (blockDim.x strides);
    // the list order is not significant (each env's reset is independent)
    for (int t0 = 0; t0 < n_range; t0 += blockDim.x) {
        const int t = t0 + threadIdx.x, wl = threadIdx.x & 31;
        const bool sel = t < n_range && (!mask || (mask[e0 + t] & mask_bits));
        const unsigned b = __ballot_sync(0xffffffffu, sel);
        int base = 0;
        if (wl == 0 && b) base = atomicAdd(&s_cnt, __popc(b));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (sel) s_list[base + __popc(b & ((1u << wl) - 1))] = e0 + t;
    }
    __syncthreads();
    const int cnt = s_cnt;
    if (cnt == 0) return;
    load_tree_table(smem, M);
    const int slot = warp * EPW + grp;
    if (slot >= M.epb) return;
    const EnvSmem S = carve(smem, slot, M, G, hm);
    for (int k = slot; k < cnt; k += M.epb) {
        reset_env<EPW>(M, St, S, s_list[k], mode, frames_in, obs, frames_out, bad, lane);
        __syncwarp(hm);
    }
}

template <int WPB, int MINB, int EPW>
__global__ void __launch_bounds__(WPB * 32, MINB) observe_kernel(DevModel M, DevState St, int n_envs, float* obs,
                                                                 float* delta) {
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr int G = 32 / EPW, QS = kMaxQSlots * EPW;
    const int warp = threadIdx.x >> 5, grp = (threadIdx.x & 31) / G, lane = threadIdx.x & (G - 1);
    const unsigned hm = EPW == 1 ? 0xffffffffu : (0xffffu << (16 * grp));
    const int slot = warp * EPW + grp, e = blockIdx.x * M.epb + slot;
    load_tree_table(smem, M);
    if (slot >= M.epb || e >= n_envs) return;
    const EnvSmem S = carve(smem, warp * EPW + grp, M, G, hm);
    const int nq = M.nq;
    double qd[QS], dqd[QS];
    load_dofs<QS>(M, S, St.q + static_cast<size_t>(e) * nq, St.dq + static_cast<size_t>(e) * nq, qd, dqd, lane);
    publish_dofs<QS>(M, S, qd, dqd, lane);
    __syncwarp(S.hm);
    tree_sweep<false>(M, S, lane, nullptr);
    const double* qsm = stage_q<QS>(M, S, qd, lane);
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

__global__ void set_mti_kernel(DevState St, int n_envs, const int* mti) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e < n_envs) St.mti[e] = min(max(mti[e], 0), 312);
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
    const int c = St.out_count[e];
    const int n = min(c, St.out_cap);
    for (int i = 0; i < n; ++i)
        sampler_record(St.ema + static_cast<size_t>(e) * M.bins, M.bins, M.decay,
                       St.out_bin[static_cast<size_t>(e) * St.out_cap + i],
                       St.out_failed[static_cast<size_t>(e) * St.out_cap + i]);
    if (c > n) atomicAdd(St.out_dropped, static_cast<unsigned long long>(c - n));  // ring overflow: counted
    St.out_count[e] = 0;
}

// Ordered merge into one sampler (env order, then time order), then broadcast.
// Ordered merge of all ranks' outcomes into the global sampler EMA (global env
// order, then time order — the sequential AdaptiveSampler::record of
// env.cpp:34-37).  Bins are independent, so thread b < bins applies, in order,
// exactly the outcomes of bin b (bit-identical to the sequential loop); the
// block compacts each 1024-env chunk's outcomes into shared memory with a
// block-wide scan so the per-bin passes read contiguous smem.
constexpr int kMergeThreads = 1024, kMergeList = 4096;

__global__ void __launch_bounds__(kMergeThreads) merge_kernel(DevModel M, const int* bins, const uint8_t* failed,
                                                              const int* counts, long long n_total, int cap,
                                                              double* global_ema) {
    __shared__ int s_bin[kMergeList];
    __shared__ uint8_t s_fail[kMergeList];
    __shared__ int s_scan[kMergeThreads];
    __shared__ double s_ema[kMergeThreads];  // bins <= 1024
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid < M.bins) s_ema[tid] = global_ema[tid];
    const double keep = M.decay, gain = __dsub_rn(1.0, M.decay);
    for (long long base = 0; base < n_total; base += kMergeThreads) {
        const long long g = base + tid;
        const int c = g < n_total ? max(0, min(counts[g], cap)) : 0;
        s_scan[tid] = c;  // inclusive Hillis-Steele scan of the chunk's counts
        __syncthreads();
        for (int o = 1; o < kMergeThreads; o <<= 1) {
            const int v = tid >= o ? s_scan[tid - o] : 0;
            __syncthreads();
            s_scan[tid] += v;
            __syncthreads();
        }
        const int off = s_scan[tid] - c, tot = s_scan[kMergeThreads - 1];
        for (int p0 = 0; p0 < tot; p0 += kMergeList) {
            for (int i = 0; i < c; ++i) {
                const int idx = off + i - p0;
                if (idx >= 0 && idx < kMergeList) {
                    s_bin[idx] = bins[g * cap + i];
                    s_fail[idx] = failed[g * cap + i];
                }
            }
            __syncthreads();
            // warp w owns bins w, w + 32, ...: it finds its bin's outcomes 32 list
            // entries at a time (ballot) and applies them in list order, so each
            // bin's EMA sees exactly the sequential order of AdaptiveSampler::record
            const int n = min(kMergeList, tot - p0);
            for (int b = warp; b < M.bins; b += kMergeThreads / 32) {
                double ema = s_ema[b];
                for (int j0 = 0; j0 < n; j0 += 32) {
                    const int j = j0 + lane;
                    const bool hit = j < n && s_bin[j] == b;
                    unsigned mk = __ballot_sync(0xffffffffu, hit);
                    const unsigned fm = __ballot_sync(0xffffffffu, hit && s_fail[j]);
                    while (mk) {
                        const int i = __ffs(mk) - 1;
                        mk &= mk - 1;
                        ema = __dadd_rn(__dmul_rn(keep, ema), __dmul_rn(gain, (fm >> i) & 1 ? 1.0 : 0.0));
                    }
                }
                if (lane == 0) s_ema[b] = ema;
            }
            __syncthreads();
        }
        __syncthreads();
    }
    if (tid < M.bins) global_ema[tid] = s_ema[tid];
}

__global__ void broadcast_ema_kernel(DevState St, int n_envs, int bins, const double* row) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n_envs * bins) St.ema[i] = row[i % bins];
}

__global__ void drain_kernel(DevState St, int n_envs, int cap, int* bins, uint8_t* failed, int* counts) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n_envs) return;
    const int c = St.out_count[e];
    const int n = min(min(c, St.out_cap), cap);
    counts[e] = n;  // only valid slots are ever reported (the merge reads counts[e] entries)
    for (int i = 0; i < n; ++i) {
        bins[static_cast<size_t>(e) * cap + i] = St.out_bin[static_cast<size_t>(e) * St.out_cap + i];
        failed[static_cast<size_t>(e) * cap + i] = St.out_failed[static_cast<size_t>(e) * St.out_cap + i];
    }
    // outcomes beyond the ring or the caller's cap are not silently lost: counted
    if (c > n) atomicAdd(St.out_dropped, static_cast<unsigned long long>(c - n));
    St.out_count[e] = 0;
}

// Muscle rows between the internal (segment-count sorted) order and the
// reference order: to_internal ? dst[i] = src[ext(i)] : dst[ext(i)] = src[i].
template <class T>
__global__ void permute_muscles_kernel(DevModel M, int n_envs, const T* src, T* dst, int to_internal) {
    const long long tot = static_cast<long long>(n_envs) * M.nm;
    for (long long g = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; g < tot;
         g += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long row = g / M.nm;
        const int i = static_cast<int>(g - row * M.nm);
        const long long x = row * M.nm + (__ldg(M.m_meta + i) >> 9);
        if (to_internal)
            dst[g] = src[x];
        else
            dst[x] = src[g];
    }
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
    const int groups = (nm + 3) / 4;  // (n_envs * groups < 2^31: checked by the launcher)
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_envs * groups) return;
    const int e = i / groups, g = i - e * groups;
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
    constexpr float kScale = 1.0f / 16777216.0f;
    if ((nm & 3) == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0) {  // 16-B aligned rows: one vector store
        reinterpret_cast<float4*>(row)[g] = make_float4(static_cast<float>(r4[0] >> 8) * kScale,
                                                        static_cast<float>(r4[1] >> 8) * kScale,
                                                        static_cast<float>(r4[2] >> 8) * kScale,
                                                        static_cast<float>(r4[3] >> 8) * kScale);
        return;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int m = 4 * g + k;
        if (m < nm) row[m] = static_cast<float>(r4[k] >> 8) * kScale;
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
#ifndef MSK_EPW
#define MSK_EPW 1   // envs per warp: 1 (32 lanes per env) or 2 (16 lanes per env)
#endif
#ifndef MSK_WPB
#define MSK_WPB (28 / MSK_EPW)  // warps per block: one 896-thread block = 28 envs per SM
#endif
#ifndef MSK_MINB
#define MSK_MINB 1  // 28 envs resident per SM -> 4096 envs in one wave; one tree table per SM
#endif
constexpr int kEPW = MSK_EPW;
constexpr int kWPB = MSK_WPB;
constexpr int kMinB = MSK_MINB;
constexpr int kEnvsPerBlock = kWPB * kEPW;

// Fast-path segment count for a model (0 = generic path).
int step_variant(const DevModel& M) { return M.fast_nseg; }
// DOF register slots per lane: 3 covers n_q <= 96 (the whole-body models), else 4.
int step_qslots(const DevModel& M) { return M.nq <= 96 ? 3 : kMaxQSlots; }

// Envs per thread of the step kernel (MSK_NE: 1 = step_kernel, the default; 2 or 4 =
// stepn_kernel, opt-in: 15 % fewer instructions at NE = 2 but half the warps per SM,
// and the 128-register cap of 4 warps per SM partition leaves no room for the ILP
// that would hide the per-env dependency chains — measured 0.628 / 0.870 ms vs 0.551 ms).
// Envs per tree warp of the step kernel (MSK_TREEQ: 1 = step_kernel, 2 or 4 = stepq_kernel).
int step_treeq() {
    static const int q = [] {
        const char* v = std::getenv("MSK_TREEQ");
        const int x = v ? std::atoi(v) : 1;
        return (x == 1 || x == 2 || x == 4) ? x : 1;
    }();
    return kEPW == 1 && kWPB % 4 == 0 ? q : 1;
}

int step_ne() {
    static const int ne = [] {
        const char* v = std::getenv("MSK_NE");
        const int x = v ? std::atoi(v) : 1;
        return (x == 1 || x == 2 || x == 4) ? x : 1;
    }();
    return kEPW == 1 ? ne : 1;
}

template <int NSEG, int QSL>
cudaError_t set_step_smem(int bytes) {
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(stepn_kernel<14, 2, NSEG, QSL>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes)))
        return e;
    if ((e = cudaFuncSetAttribute(stepn_kernel<7, 4, NSEG, QSL>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes)))
        return e;
    if ((e = cudaFuncSetAttribute(stepq_kernel<kWPB, 2, NSEG, QSL>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes)))
        return e;
    if ((e = cudaFuncSetAttribute(stepq_kernel<kWPB, 4, NSEG, QSL>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes)))
        return e;
    return cudaFuncSetAttribute(step_kernel<kWPB, kMinB, NSEG, kEPW, QSL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                bytes);
}

size_t block_smem(const DevModel& M) {
    return static_cast<size_t>(M.tab_bytes) + static_cast<size_t>(M.epb) * M.smem_env_bytes;
}

cudaError_t prepare_kernels(int smem_bytes_per_block) {
    cudaError_t err;
    if ((err = set_step_smem<0, 4>(smem_bytes_per_block)) != cudaSuccess) return err;
    if ((err = set_step_smem<1, 4>(smem_bytes_per_block)) != cudaSuccess) return err;
    if ((err = set_step_smem<2, 4>(smem_bytes_per_block)) != cudaSuccess) return err;
    if ((err = set_step_smem<3, 4>(smem_bytes_per_block)) != cudaSuccess) return err;
    if ((err = set_step_smem<4, 4>(smem_bytes_per_block)) != cudaSuccess) return err;
    if ((err = set_step_smem<0, 3>(smem_bytes_per_block)) != cudaSuccess) return err;
    if ((err = set_step_smem<2, 3>(smem_bytes_per_block)) != cudaSuccess) return err;
    if ((err = set_step_smem<3, 3>(smem_bytes_per_block)) != cudaSuccess) return err;
    if ((err = cudaFuncSetAttribute(reset_kernel<kWPB, kMinB, kEPW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    smem_bytes_per_block)) != cudaSuccess)
        return err;
    return cudaFuncSetAttribute(observe_kernel<kWPB, kMinB, kEPW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                smem_bytes_per_block);
}

int envs_per_block() { return kEnvsPerBlock; }
int step_envs_per_warp() { return step_ne(); }
int lanes_per_env() { return 32 / kEPW; }

void launch_step(const DevModel& M, const DevState& St, int env0, int n, const float* actions, float* obs,
                 float* delta, float* raux, uint8_t* flags, float* power, float* grf, cudaStream_t s,
                 int n_substeps) {
    const int blocks = (n + M.epb - 1) / M.epb;
    const size_t smem = block_smem(M);
    const int ne = step_ne(), tq = step_treeq();
#define MSK_STEP(NS, QSL)                                                                                          \
    do {                                                                                                           \
        if (tq == 2 && ne == 1)                                                                                    \
            stepq_kernel<kWPB, 2, NS, QSL><<<blocks, kWPB * 32, smem, s>>>(M, St, env0, n, actions, obs, delta,   \
                                                                             raux, flags, power, grf, n_substeps); \
        else if (tq == 4 && ne == 1)                                                                               \
            stepq_kernel<kWPB, 4, NS, QSL><<<blocks, kWPB * 32, smem, s>>>(M, St, env0, n, actions, obs, delta,   \
                                                                             raux, flags, power, grf, n_substeps); \
        else if (ne == 2)                                                                                          \
            stepn_kernel<14, 2, NS, QSL><<<blocks, 14 * 32, smem, s>>>(M, St, env0, n, actions, obs, delta, raux,  \
                                                                         flags, power, grf, n_substeps);           \
        else if (ne == 4)                                                                                          \
            stepn_kernel<7, 4, NS, QSL><<<blocks, 7 * 32, smem, s>>>(M, St, env0, n, actions, obs, delta, raux,    \
                                                                       flags, power, grf, n_substeps);             \
        else                                                                                                       \
            step_kernel<kWPB, kMinB, NS, kEPW, QSL><<<blocks, kWPB * 32, smem, s>>>(                               \
                M, St, env0, n, actions, obs, delta, raux, flags, power, grf, n_substeps);                         \
    } while (0)
    prep_actions_kernel<<<(n + 7) / 8, 256, 0, s>>>(M, St, env0, n, actions);
    const int v = step_variant(M);
    if (step_qslots(M) == 3 && (v == 0 || v == 2 || v == 3)) {  // whole-body sized models
        switch (v) {
            case 2: MSK_STEP(2, 3); break;
            case 3: MSK_STEP(3, 3); break;
            default: MSK_STEP(0, 3); break;
        }
    } else {
        switch (v) {
            case 1: MSK_STEP(1, 4); break;
            case 2: MSK_STEP(2, 4); break;
            case 3: MSK_STEP(3, 4); break;
            case 4: MSK_STEP(4, 4); break;
            default: MSK_STEP(0, 4); break;
        }
    }
#undef MSK_STEP
}

void launch_reset(const DevModel& M, const DevState& St, int n, int mode, const uint8_t* mask, uint8_t bits,
                  const int* frames_in, float* obs, int* frames_out, uint8_t* bad, cudaStream_t s) {
    static const int sms = [] {
        int dev = 0, v = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        return v;
    }();
    // one wave of blocks when the ranges allow it, ranges of <= kResetRange envs
    const int blocks = std::max(std::min((n + M.epb - 1) / M.epb, sms), (n + kResetRange - 1) / kResetRange);
    const int range = (n + blocks - 1) / blocks;
    reset_kernel<kWPB, kMinB, kEPW><<<blocks, kWPB * 32, block_smem(M), s>>>(M, St, n, range, mode, mask, bits,
                                                                                frames_in, obs, frames_out, bad);
}

void launch_observe(const DevModel& M, const DevState& St, int n, float* obs, float* delta, cudaStream_t s) {
    const int blocks = (n + M.epb - 1) / M.epb;
    observe_kernel<kWPB, kMinB, kEPW><<<blocks, kWPB * 32, block_smem(M), s>>>(M, St, n, obs, delta);
}

void launch_seed(const DevState& St, int n, uint64_t base_seed, cudaStream_t s) {
    seed_kernel<<<(n + 127) / 128, 128, 0, s>>>(St, n, base_seed);
}

void launch_rng_raw(const DevState& St, int e, int n, uint64_t* out, cudaStream_t s) {
    rng_raw_kernel<<<1, 32, 0, s>>>(St, e, n, out);
}

void launch_set_mti(const DevState& St, int n, const int* mti, cudaStream_t s) {
    set_mti_kernel<<<(n + 127) / 128, 128, 0, s>>>(St, n, mti);
}

void launch_record_own(const DevModel& M, const DevState& St, int n, cudaStream_t s) {
    record_own_kernel<<<(n + 127) / 128, 128, 0, s>>>(M, St, n);
}

void launch_merge(const DevModel& M, const DevState& St, int n_local, const int* bins, const uint8_t* failed,
                  const int* counts, long long n_total, int cap, double* global_ema, cudaStream_t s) {
    merge_kernel<<<1, kMergeThreads, 0, s>>>(M, bins, failed, counts, n_total, cap, global_ema);
    const int tot = n_local * M.bins;
    broadcast_ema_kernel<<<(tot + 255) / 256, 256, 0, s>>>(St, n_local, M.bins, global_ema);
}

// One rank's outcome block into the running global EMA (no broadcast): the
// per-rank form of launch_merge for blocks gathered rank by rank.
void launch_merge_block(const DevModel& M, const int* bins, const uint8_t* failed, const int* counts, long long n,
                        int cap, double* global_ema, cudaStream_t s) {
    merge_kernel<<<1, kMergeThreads, 0, s>>>(M, bins, failed, counts, n, cap, global_ema);
}

// Rank-ordered iteration merge of the gathered blocks' statistics and
// observation moments (dist.py merged_iteration, RunningNorm::update
// nn.cpp:246-270), with the same IEEE operation order as the torch path (no
// contraction): stats_out[k] = sum over ranks in order; norm = (count, mean[D],
// var[D]) folded rank by rank.  One block; threads over D.
__global__ void exchange_fold_kernel(const unsigned char* gathered, size_t block_bytes, int world, size_t off_stats,
                                     size_t off_mom, int D, double* norm, double* stats_out) {
    if (stats_out && threadIdx.x < 7) {
        double acc = 0.0;
        for (int r = 0; r < world; ++r)
            acc = __dadd_rn(acc, reinterpret_cast<const double*>(gathered + r * block_bytes + off_stats)[threadIdx.x]);
        stats_out[threadIdx.x] = acc;
    }
    __shared__ double c0;
    if (threadIdx.x == 0) c0 = norm[0];
    __syncthreads();  // everyone has the pre-fold count before norm[0] is rewritten
    const double count0 = c0;
    if (threadIdx.x == 0) {  // the folded count (the same for every column)
        double count = count0;
        for (int r = 0; r < world; ++r) {
            const double n = reinterpret_cast<const double*>(gathered + r * block_bytes + off_mom)[0];
            if (n != 0.0) count = __dadd_rn(count, n);
        }
        norm[0] = count;
    }
    for (int d = threadIdx.x; d < D; d += blockDim.x) {
        double count = count0, mean = norm[1 + d], var = norm[1 + D + d];
        for (int r = 0; r < world; ++r) {
            const double* m = reinterpret_cast<const double*>(gathered + r * block_bytes + off_mom);
            const double n = m[0], bmean = m[1 + d], bvar = m[1 + D + d];
            if (n == 0.0) continue;
            const double tot = __dadd_rn(count, n);
            if (count == 0.0) {
                mean = bmean;
                var = bvar;
            } else {
                const double delta = __dsub_rn(bmean, mean);
                const double a = __dadd_rn(__dmul_rn(var, count), __dmul_rn(bvar, n));
                const double b = __dmul_rn(__dmul_rn(delta, delta), __ddiv_rn(__dmul_rn(count, n), tot));
                var = __ddiv_rn(__dadd_rn(a, b), tot);
                mean = __dadd_rn(mean, __dmul_rn(delta, __ddiv_rn(n, tot)));
            }
            count = tot;
        }
        norm[1 + d] = mean;
        norm[1 + D + d] = var;
    }
}

void launch_exchange_fold(const unsigned char* gathered, size_t block_bytes, int world, size_t off_stats,
                          size_t off_mom, int D, double* norm, double* stats_out, cudaStream_t s) {
    exchange_fold_kernel<<<1, 1024, 0, s>>>(gathered, block_bytes, world, off_stats, off_mom, D, norm, stats_out);
}

void launch_broadcast_ema(const DevState& St, int n, int bins, const double* row, cudaStream_t s) {
    broadcast_ema_kernel<<<(n * bins + 255) / 256, 256, 0, s>>>(St, n, bins, row);
}

// ---- iteration-boundary reductions (SURVEY §8(e) block contents) ----------
// Rollout statistics of one control step, added into stats[7] = {env-steps,
// Σr, Σr², Σ episode length (done envs), episodes, failures, divergences}.
// One block, fixed-order tree reduction: deterministic.
__global__ void __launch_bounds__(1024) rollout_stats_kernel(DevState St, int n, const float* reward,
                                                             const uint8_t* flags, double* stats) {
    __shared__ double red[7][32];
    double a[7] = {0, 0, 0, 0, 0, 0, 0};
    for (int e = threadIdx.x; e < n; e += blockDim.x) {
        const uint8_t f = flags[e];
        if (f & (kFlagNotStepped | kFlagBadAction)) continue;
        const double r = reward ? static_cast<double>(reward[e]) : 0.0;
        a[0] += 1.0;
        a[1] += r;
        a[2] += r * r;
        if (f & kFlagDone) {
            a[3] += static_cast<double>(St.steps[e]);
            a[4] += 1.0;
        }
        if (f & kFlagFailed) a[5] += 1.0;
        if (f & kFlagDiverged) a[6] += 1.0;
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < 7; ++k) {
        double v = a[k];
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) red[k][warp] = v;
    }
    __syncthreads();
    if (warp == 0) {
        const int nw = blockDim.x >> 5;
#pragma unroll
        for (int k = 0; k < 7; ++k) {
            double v = lane < nw ? red[k][lane] : 0.0;
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (lane == 0) stats[k] += v;
        }
    }
}

// Column moments of an [n x D] f32 batch in f64 (RunningNorm::update's batch
// terms, nn.cpp:246-256): pass 1 gives per row-chunk (mean, M2) per column in
// ONE read of the chunk (sums shifted by the chunk's first row: exact enough in
// f64 for f32 data, ~1e-15 relative), pass 2 merges the chunks (the Chan et al.
// merge in closed form), writing out = [n, mean[D], var[D]] (population variance) — or, with
// `fold`, folding those batch moments into the running {count, mean, var} at
// out exactly as dist.running_norm_fold_t / RunningNorm::update (nn.cpp:257-270).
constexpr int kMomRows = 64;

__global__ void obs_moments_part_kernel(const float* x, int n, int D, double* part, const double* acc,
                                        double* acc_count) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x, k = blockIdx.y;
    if (acc && c == 0 && k == 0) *acc_count = acc[0];  // the fold's running count, read before it advances
    if (c >= D) return;
    const int r0 = k * kMomRows, r1 = min(n, r0 + kMomRows);
    const float* col = x + static_cast<size_t>(r0) * D + c;
    const double sh = static_cast<double>(col[0]);
    double s1 = 0.0, s2 = 0.0;
#pragma unroll 8
    for (int r = 0; r < r1 - r0; ++r) {
        const double d = static_cast<double>(col[static_cast<size_t>(r) * D]) - sh;
        s1 += d;
        s2 = fma(d, d, s2);
    }
    const double nk = static_cast<double>(r1 - r0);
    part[(static_cast<size_t>(k) * D + c) * 2] = sh + s1 / nk;
    part[(static_cast<size_t>(k) * D + c) * 2 + 1] = fmax(s2 - s1 * (s1 / nk), 0.0);
}

// Two columns per thread (8-B loads; even D, 8-B aligned rows), same arithmetic.
__global__ void obs_moments_part2_kernel(const float* x, int n, int D, double* part, const double* acc,
                                         double* acc_count) {
    const int c = 2 * (blockIdx.x * blockDim.x + threadIdx.x), k = blockIdx.y;
    if (acc && c == 0 && k == 0) *acc_count = acc[0];
    if (c >= D) return;
    const int r0 = k * kMomRows, r1 = min(n, r0 + kMomRows);
    const float2* col = reinterpret_cast<const float2*>(x + static_cast<size_t>(r0) * D + c);
    const int D2 = D / 2;
    const float2 v0 = col[0];
    const double sa = v0.x, sb = v0.y;
    double a1 = 0.0, a2 = 0.0, b1 = 0.0, b2 = 0.0;
#pragma unroll 8
    for (int r = 0; r < r1 - r0; ++r) {
        const float2 v = col[static_cast<size_t>(r) * D2];
        const double da = static_cast<double>(v.x) - sa, db = static_cast<double>(v.y) - sb;
        a1 += da;
        a2 = fma(da, da, a2);
        b1 += db;
        b2 = fma(db, db, b2);
    }
    const double nk = static_cast<double>(r1 - r0);
    double* o = part + (static_cast<size_t>(k) * D + c) * 2;
    o[0] = sa + a1 / nk;
    o[1] = fmax(a2 - a1 * (a1 / nk), 0.0);
    o[2] = sb + b1 / nk;
    o[3] = fmax(b2 - b1 * (b1 / nk), 0.0);
}

// Chunk merge: 32 columns x kMomGroups chunk groups per block; the groups' sums
// are added in group order (fixed), in closed form: mean = sum n_k m_k / n,
// M2 = sum (M2_k + n_k (m_k - mean)^2) — the Chan merge's result.
constexpr int kMomGroups = 8;

__global__ void __launch_bounds__(32 * kMomGroups) obs_moments_merge_kernel(const double* part, int n, int D,
                                                                            int chunks, double* out,
                                                                            const double* acc_count) {
    __shared__ double red[kMomGroups][32];
    const int tx = threadIdx.x, ty = threadIdx.y, c = blockIdx.x * 32 + tx;
    const int per = (chunks + kMomGroups - 1) / kMomGroups, k0 = ty * per, k1 = min(chunks, k0 + per);
    double s = 0.0;
    if (c < D)
        for (int k = k0; k < k1; ++k)
            s = fma(static_cast<double>(min(n - k * kMomRows, kMomRows)), part[(static_cast<size_t>(k) * D + c) * 2], s);
    red[ty][tx] = s;
    __syncthreads();
    double tot = 0.0;
    for (int g = 0; g < kMomGroups; ++g) tot += red[g][tx];
    const double mean = n > 0 ? tot / static_cast<double>(n) : 0.0;
    __syncthreads();
    double q = 0.0;
    if (c < D)
        for (int k = k0; k < k1; ++k) {
            const double nk = static_cast<double>(min(n - k * kMomRows, kMomRows));
            const double d = part[(static_cast<size_t>(k) * D + c) * 2] - mean;
            q += fma(nk * d, d, part[(static_cast<size_t>(k) * D + c) * 2 + 1]);
        }
    red[ty][tx] = q;
    __syncthreads();
    if (ty != 0) return;
    double m2 = 0.0;
    for (int g = 0; g < kMomGroups; ++g) m2 += red[g][tx];
    const double bn = static_cast<double>(n), bvar = n > 0 ? m2 / bn : 0.0;
    if (!acc_count) {
        if (c == 0) out[0] = bn;
        if (c < D) {
            out[1 + c] = mean;
            out[1 + D + c] = bvar;
        }
        return;
    }
    // running_norm_fold_t: tot = count + n; delta = bmean - mean;
    // var = (var count + bvar n + delta^2 (count n / tot)) / tot; mean += delta (n / tot)
    const double count = *acc_count;
    if (n == 0) return;
    if (c == 0) out[0] = __dadd_rn(count, bn);
    if (c >= D) return;
    if (count == 0.0) {
        out[1 + c] = mean;
        out[1 + D + c] = bvar;
    } else {
        const double tn = __dadd_rn(count, bn);
        const double rm = out[1 + c], rv = out[1 + D + c];
        const double delta = __dadd_rn(mean, -rm);
        const double w = __ddiv_rn(__dmul_rn(count, bn), tn);
        const double num = __dadd_rn(__dadd_rn(__dmul_rn(rv, count), __dmul_rn(bvar, bn)),
                                     __dmul_rn(__dmul_rn(delta, delta), w));
        out[1 + D + c] = __ddiv_rn(num, tn);
        out[1 + c] = __dadd_rn(rm, __dmul_rn(delta, __ddiv_rn(bn, tn)));
    }
}

void launch_rollout_stats(const DevState& St, int n, const float* reward, const uint8_t* flags, double* stats,
                          cudaStream_t s) {
    rollout_stats_kernel<<<1, 1024, 0, s>>>(St, n, reward, flags, stats);
}

int obs_moments_chunks(int n) { return (n + kMomRows - 1) / kMomRows; }

// part: chunks x D x 2 partials + 1 (the fold's running count, snapshot by the part kernel)
void launch_obs_moments(const float* x, int n, int D, double* part, double* out, cudaStream_t s, bool fold) {
    const int chunks = obs_moments_chunks(n);
    double* cnt = part + static_cast<size_t>(chunks) * D * 2;
    if (chunks > 0 && D % 2 == 0 && (reinterpret_cast<uintptr_t>(x) & 7) == 0)
        obs_moments_part2_kernel<<<dim3((D / 2 + 127) / 128, chunks), 128, 0, s>>>(x, n, D, part,
                                                                                  fold ? out : nullptr, cnt);
    else if (chunks > 0)
        obs_moments_part_kernel<<<dim3((D + 127) / 128, chunks), 128, 0, s>>>(x, n, D, part, fold ? out : nullptr, cnt);
    else if (fold)
        return;  // an empty batch leaves the running moments unchanged
    obs_moments_merge_kernel<<<(D + 31) / 32, dim3(32, kMomGroups), 0, s>>>(part, n, D, chunks, out,
                                                                          fold ? cnt : nullptr);
}

void launch_drain(const DevState& St, int n, int cap, int* bins, uint8_t* failed, int* counts, cudaStream_t s) {
    drain_kernel<<<(n + 127) / 128, 128, 0, s>>>(St, n, cap, bins, failed, counts);
}

void launch_permute_muscles(const DevModel& M, int n, const float* src, float* dst, int to_internal, cudaStream_t s) {
    const long long tot = static_cast<long long>(n) * M.nm;
    const int blocks = static_cast<int>(std::min<long long>((tot + 255) / 256, 148 * 16));
    permute_muscles_kernel<float><<<blocks, 256, 0, s>>>(M, n, src, dst, to_internal);
}

void launch_permute_muscles(const DevModel& M, int n, const double* src, double* dst, int to_internal,
                            cudaStream_t s) {
    const long long tot = static_cast<long long>(n) * M.nm;
    const int blocks = static_cast<int>(std::min<long long>((tot + 255) / 256, 148 * 16));
    permute_muscles_kernel<double><<<blocks, 256, 0, s>>>(M, n, src, dst, to_internal);
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
    if (tot >= (1ll << 31)) throw std::runtime_error("fill_excitations: batch too large");
    excitation_kernel<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, s>>>(n, nm, env_offset, seed, step, out);
}

}  // namespace msk_b200

#ifdef MSK_PHASE_TIMERS
// Diagnostics build only: per-phase cycle totals (summed over warps and substeps).
extern "C" int msk_gpu_phase_cycles(unsigned long long* out, int reset) {
    if (cudaMemcpyFromSymbol(out, msk_b200::g_phase_cycles, sizeof(unsigned long long) * 8) != cudaSuccess) return 3;
    if (reset) {
        const unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        cudaMemcpyToSymbol(msk_b200::g_phase_cycles, z, sizeof(z));
    }
    return 0;
}
#endif
