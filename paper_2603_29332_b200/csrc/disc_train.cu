// Discriminator training step on the device (second half;
// SPEC.md:412-421 train_discriminator):
//
//   loss = -log clamp(D(0)) - mean_i log(1 - clamp(D(Δ_i))) + λ mean_i ||∇_Δ D(Δ_i)||²
//
// followed by one Adam step (nn.cpp:224-240).  D = Mlp(in, W, 1, Head::Sigmoid)
// with master parameters θ in the reference's flat layout (nn.cpp:16-38, W
// column-major) and the Adam moments in f64 on the device.
//
// The reference composes Mlp::backward (nn.cpp:80-129) for the logistic terms
// with Mlp::gradient_penalty_backward (nn.cpp:131-222: input gradient g, its
// forward tangent, then a reverse pass through primal + tangent).  Here, over
// R = B + 1 rows (the B Δ rows plus the zero input of the D(0) term):
//   * forward   H_l = tanh(H_{l-1} W_lᵀ + b_l), y = sigmoid(H_3 w_4 + b_4)
//   * input gradient g = dy/dx (d-chain) and its forward tangent ζ_l, u_l
//   * ONE reverse pass carrying [tangent; primal] adjoints: the logistic
//     loss's head adjoint enters the primal adjoint of the penalty's reverse
//     pass (both are linear in the head adjoint);
//   * weight gradients gW_l = b_ζᵀ u + b_zᵀ H (one split-K GEMM over 2R rows),
//     bias gradients as column sums of the primal adjoints.
//
// Every product is a hand-written tcgen05 GEMM (no cuBLAS):
//   * operands live in HBM as "split images": x = hi + lo, both bf16, in
//     128 x 128 blocks of 8 x 8 core matrices ordered column-group-major, so the
//     SAME image is a K-major operand (row GEMMs, K = columns) and an MN-major
//     operand (weight-gradient GEMMs, K = rows);
//   * fp32-class mode (math 0): three MMAs per product (lo·hi + hi·lo + hi·hi,
//     fp32 TMEM accumulation), ~2^-17 relative operands; fast mode (math 1):
//     hi·hi only (bf16 operands);
//   * row GEMMs (M = 128 rows per CTA, N = the layer width ≤ 256 in two
//     128-column MMAs, K in 32-column stages through a 4-stage bulk-copy ring)
//     fuse every elementwise step into the epilogue: bias + tanh, the sigmoid
//     head (row dot product, clamped logs, d4 / dd4 / logistic adjoint), the
//     gates ∘(1 - H²), the penalty head, and the reverse elementwise step; the
//     reverse GEMMs compute tangent and primal rows of the same tile in one CTA
//     (two TMEM accumulators sharing each weight stage) so that step pairs them;
//   * column sums (bias gradients, w4 gradient) are per-warp butterfly
//     reductions in the epilogues, reduced later in a fixed order;
//   * weight-gradient GEMMs split K = 2R over ~148 CTAs (MN-major operands from
//     1 KB bulk-copy pieces), fp32 partials reduced in a fixed order in f64.
// Everything is deterministic (no atomics).  This is the learner side of the
// loop, launched once per rollout iteration; the stepping path never calls it.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/msk_gpu.h"
#include "disc.hpp"

namespace {

using bf16 = __nv_bfloat16;
constexpr double kClampLo = 1e-4, kClampHi = 1.0 - 1e-4;

// ---- split images -----------------------------------------------------------
// [rows_p x cols_p] (both multiples of 128) as 128 x 128 blocks of 16384
// elements, block (rb, cb) at rb * (cols_p / 128) + cb; inside a block the 8 x 8
// core matrices (8 rows x 8 consecutive columns = 128 B) are column-group-major:
// core (rg, cg) at (cg * 16 + rg) * 128 B.
__host__ __device__ __forceinline__ size_t iofs(int r, int c, int cols_p) {
    return (static_cast<size_t>(r >> 7) * (cols_p >> 7) + (c >> 7)) * 16384 +
           static_cast<size_t>((((c & 127) >> 3) << 4) + ((r & 127) >> 3)) * 64 + (r & 7) * 8 + (c & 7);
}

struct Img {
    bf16* hi = nullptr;
    bf16* lo = nullptr;
    int cols_p = 0;
};

__device__ __forceinline__ uint32_t pack2(bf16 a, bf16 b) {
    return static_cast<uint32_t>(__bfloat16_as_ushort(a)) | (static_cast<uint32_t>(__bfloat16_as_ushort(b)) << 16);
}

// 8 consecutive columns of one row: x = hi + lo.
__device__ __forceinline__ void store8(const Img& im, int r, int c, const float* v) {
    uint32_t h[4], l[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const bf16 a = __float2bfloat16_rn(v[2 * i]), b = __float2bfloat16_rn(v[2 * i + 1]);
        h[i] = pack2(a, b);
        l[i] = pack2(__float2bfloat16_rn(v[2 * i] - __bfloat162float(a)),
                     __float2bfloat16_rn(v[2 * i + 1] - __bfloat162float(b)));
    }
    const size_t o = iofs(r, c, im.cols_p);
    *reinterpret_cast<uint4*>(im.hi + o) = make_uint4(h[0], h[1], h[2], h[3]);
    *reinterpret_cast<uint4*>(im.lo + o) = make_uint4(l[0], l[1], l[2], l[3]);
}
__device__ __forceinline__ void load8(const Img& im, int r, int c, float* v) {
    const size_t o = iofs(r, c, im.cols_p);
    const uint4 h = *reinterpret_cast<const uint4*>(im.hi + o), l = *reinterpret_cast<const uint4*>(im.lo + o);
    const uint32_t hw[4] = {h.x, h.y, h.z, h.w}, lw[4] = {l.x, l.y, l.z, l.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        v[2 * i] = __uint_as_float(hw[i] << 16) + __uint_as_float(lw[i] << 16);
        v[2 * i + 1] = __uint_as_float(hw[i] & 0xffff0000u) + __uint_as_float(lw[i] & 0xffff0000u);
    }
}
__device__ __forceinline__ void store32(const Img& im, int r, int c, const float (&v)[32]) {
#pragma unroll
    for (int j = 0; j < 4; ++j) store8(im, r, c + 8 * j, v + 8 * j);
}
__device__ __forceinline__ void load32(const Img& im, int r, int c, float (&v)[32]) {
#pragma unroll
    for (int j = 0; j < 4; ++j) load8(im, r, c + 8 * j, v + 8 * j);
}

// ---- tcgen05 / bulk-copy helpers ------------------------------------------------
__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "DTW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra DTW_%=;\n\t}" ::"r"(su32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     su32(dst)),
                 "l"(src), "r"(bytes), "r"(su32(b))
                 : "memory");
}
// shared-memory matrix descriptor, no swizzle: LBO = K-group stride, SBO = MN-group stride
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return static_cast<uint64_t>((addr >> 4) & 0x3FFF) | (static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16) |
           (static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}
// kind::f16: D f32, A/B bf16, M = 128, N = 128; mn = 1 -> both operands MN-major
__host__ __device__ constexpr uint32_t idesc128(int mn) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(mn) << 15) | (static_cast<uint32_t>(mn) << 16) |
           (static_cast<uint32_t>(128 >> 3) << 17) | (static_cast<uint32_t>(128 >> 4) << 24);
}
__device__ __forceinline__ void mma(uint32_t tmem, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
        "l"(da), "l"(db), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void commit(uint64_t* b) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(b))
                 : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// Column sums over the 32 rows (lanes) of a warp for 32 columns: butterfly
// reduce-scatter (31 shuffles), lane l ends with column l; written to dst[lane].
__device__ __forceinline__ void colsum32(float (&x)[32], float* dst, int lane) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        const bool up = (lane & o) != 0;
#pragma unroll
        for (int i = 0; i < o; ++i) {
            const float send = up ? x[i] : x[i + o];
            const float keep = up ? x[i + o] : x[i];
            x[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
    }
    dst[lane] = x[0];
}

// ---- row GEMMs: C[128-row tile x N] = A[tile x K] · Wᵀ, N ≤ 256 ------------------
// Persistent: each CTA loops over units (a 128-row tile, or for the dual reverse
// GEMMs a (tile, 128-column half) pair); two TMEM accumulator buffers, so the
// epilogue of one unit overlaps the mainloop of the next.
constexpr int kRowEpiWarps = 16;                      // 4 per TMEM lane quarter, one column slice each
constexpr int kRowThreads = 64 + 32 * kRowEpiWarps;   // + warp 0 bulk-copy producer, warp 1 MMA issuer
constexpr int kKC = 32;                               // K columns per pipeline stage
constexpr int kChunk = 128 * kKC * 2;                 // 8 KB: one image's 128-row x 32-column slice (contiguous)
constexpr int kRowStages = 4;
constexpr int kRowStageBytes = 6 * kChunk;            // A (hi, lo) x 1-2 halves + B (hi, lo) x 1-2 blocks
constexpr size_t kRowSmem = static_cast<size_t>(kRowStages) * kRowStageBytes + 256 + (2 * 4 * 128 + 2 * 256) * 4;

enum Epi : int {
    kEpiTanh = 0,  // out0 = tanh(acc + bias)
    kEpiHead,      // out0 = H3 = tanh(acc + bias); head row scalars; out1 = d3 = d4 w4 ∘ (1 - H3²)
    kEpiGate,      // out0 = acc ∘ (1 - h²)
    kEpiPlain,     // out0 = acc
    kEpiTHead,     // penalty head: zeta4, V; out0 = S_t, out1 = S_p (layer-3 reverse step); w4 / b column sums
    kEpiRev        // dual: bu = acc_t, bh = acc_p; h, u = G∘ζ -> out0 = S_t, out1 = S_p (reverse step); b column sums
};

struct RowArgs {
    const bf16* a_hi[2] = {nullptr, nullptr};  // A images (kEpiRev: [0] tangent rows, [1] primal rows)
    const bf16* a_lo[2] = {nullptr, nullptr};
    int a_cols = 0;                      // K (multiple of 128)
    const bf16* w_hi = nullptr;          // weight image: rows = N, cols = K
    const bf16* w_lo = nullptr;
    int nb = 1;                          // N / 128
    int n_valid = 0;                     // valid output columns (bias / w4 length)
    int rows = 0;                        // valid rows R
    int tiles = 0;                       // 128-row tiles
    int passes = 3;
    const float* bias = nullptr;         // [N]
    const float* w4 = nullptr;           // head weights [N]
    const float* b4 = nullptr;           // head bias
    Img h, z;                            // gate activations H_l, gated tangent u_l (kEpiRev)
    Img out[2];
    float *d4 = nullptr, *dd4 = nullptr, *dz4 = nullptr, *vh = nullptr;
    double *lrow = nullptr, *prow = nullptr;
    float* colpart[2] = {nullptr, nullptr};  // [CTAs * 4 x ldc] per-(CTA, warp) column sums
    int ldc = 0;
    int B = 0;
    float lamB = 0.0f;
};

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void store16(const Img& im, int r, int c, const float (&v)[16]) {
    store8(im, r, c, v);
    store8(im, r, c + 8, v + 8);
}
__device__ __forceinline__ void load16(const Img& im, int r, int c, float (&v)[16]) {
    load8(im, r, c, v);
    load8(im, r, c + 8, v + 8);
}
// Column sums over the 32 rows (lanes) of a warp for 16 columns: butterfly
// reduce-scatter over lane bits 3..0, then the two lane halves combined; lanes
// 0-15 add their column's sum into acc (f64, accumulated over the warp's tiles in
// a fixed order: deterministic).
__device__ __forceinline__ void colsum16(float (&x)[16], double& acc, int lane) {
#pragma unroll
    for (int o = 8; o >= 1; o >>= 1) {
        const bool up = (lane & o) != 0;
#pragma unroll
        for (int i = 0; i < o; ++i) {
            const float send = up ? x[i] : x[i + o];
            const float keep = up ? x[i + o] : x[i];
            x[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
    }
    x[0] += __shfl_xor_sync(0xffffffffu, x[0], 16);
    acc += static_cast<double>(x[0]);
}
__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, %0;" ::"n"(32 * kRowEpiWarps) : "memory"); }

// One unit's epilogue by one epilogue warp: TMEM lane quarter q (rows), column
// slice j (a quarter of the unit's columns), 16 columns per TMEM load.
template <int EPI>
__device__ __forceinline__ void row_unit_epilogue(const RowArgs& g, uint32_t tacc, float* sdot, const float* sb,
                                                  const float* sw, int mb, int nh, int q, int j, int lane,
                                                  double (&cacc)[2][4]) {
    constexpr bool kDual = EPI == kEpiRev;
    const int rt = q * 32 + lane, r = mb * 128 + rt;
    const bool valid = r < g.rows;
    const int ncols = kDual ? 128 : g.nb * 128, sl = ncols >> 2, c_lo = j * sl, c_hi = c_lo + sl;
    const int obase = kDual ? nh * 128 : 0;  // output column of accumulator column 0
    const uint32_t tl = tacc + (static_cast<uint32_t>(q * 32) << 16);
    float v[16], x[16];

    if constexpr (EPI == kEpiTanh || EPI == kEpiGate || EPI == kEpiPlain) {
        for (int c = c_lo; c < c_hi; c += 16) {
            tmem_ld16(tl + c, v);
            if (EPI == kEpiTanh) {
#pragma unroll
                for (int i = 0; i < 16; ++i) v[i] = valid ? tanhf(v[i] + sb[c + i]) : 0.0f;
                store16(g.out[0], r, c, v);
            } else if (EPI == kEpiPlain) {
#pragma unroll
                for (int i = 0; i < 16; ++i) v[i] = valid ? v[i] : 0.0f;
                store16(g.out[0], r, c, v);
            } else {
                load16(g.h, r, c, x);
#pragma unroll
                for (int i = 0; i < 16; ++i) v[i] = valid ? v[i] * (1.0f - x[i] * x[i]) : 0.0f;
                store16(g.out[0], r, c, v);
            }
        }
    } else if constexpr (EPI == kEpiHead) {
        // pass 1: H3 and the row dot product z4 = H3 · w4
        float dot = 0.0f;
        for (int c = c_lo; c < c_hi; c += 16) {
            tmem_ld16(tl + c, v);
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                v[i] = valid ? tanhf(v[i] + sb[c + i]) : 0.0f;
                dot = fmaf(v[i], sw[c + i], dot);
            }
            store16(g.out[0], r, c, v);
        }
        sdot[j * 128 + rt] = dot;
        epi_bar();
        const float z4 = (sdot[rt] + sdot[128 + rt]) + (sdot[256 + rt] + sdot[384 + rt]);
        // sigmoid head + clamped logs (nn.cpp:66-68) in f64
        const double y = 1.0 / (1.0 + exp(-(static_cast<double>(z4) + g.b4[0])));
        const double yc = fmin(fmax(y, kClampLo), kClampHi);
        const bool inside = y > kClampLo && y < kClampHi;
        const double d = y * (1.0 - y);
        const float d4 = valid ? static_cast<float>(d) : 0.0f;
        if (valid && j == 0) {
            g.d4[r] = d4;
            g.dd4[r] = static_cast<float>(d * (1.0 - 2.0 * y));
            if (r < g.B) {  // -(1/B) log(1 - clamp(y)): upstream 1 / (B (1 - y)) -> dz4 = y / B
                g.dz4[r] = inside ? static_cast<float>(y / g.B) : 0.0f;
                g.lrow[r] = -log(1.0 - yc) / g.B;
            } else {  // -log clamp(D(0)): upstream -1 / y -> dz4 = -(1 - y)
                g.dz4[r] = inside ? static_cast<float>(-(1.0 - y)) : 0.0f;
                g.lrow[r] = -log(yc);
            }
        }
        // pass 2: d3 = d4 w4 ∘ (1 - H3²)  (nn.cpp:161), H3 read back (L2) from pass 1's image
        for (int c = c_lo; c < c_hi; c += 16) {
            load16(g.out[0], r, c, x);
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] = valid ? d4 * sw[c + i] * (1.0f - x[i] * x[i]) : 0.0f;
            store16(g.out[1], r, c, v);
        }
    } else if constexpr (EPI == kEpiTHead) {
        // pass 1: u3 = ζ3 ∘ (1 - H3²), zeta4 = u3 · w4  (nn.cpp:167-171)
        float dot = 0.0f;
        for (int c = c_lo; c < c_hi; c += 16) {
            tmem_ld16(tl + c, v);
            load16(g.h, r, c, x);
#pragma unroll
            for (int i = 0; i < 16; ++i) dot = fmaf(v[i] * (1.0f - x[i] * x[i]), sw[c + i], dot);
        }
        sdot[j * 128 + rt] = dot;
        epi_bar();
        const float zeta4 = (sdot[rt] + sdot[128 + rt]) + (sdot[256 + rt] + sdot[384 + rt]);
        // penalty + head adjoints (nn.cpp:172, 187-188; the logistic dz4 rides b_z4)
        float vu = 0.0f, vhv = 0.0f;
        if (valid) {
            const float w = r < g.B ? g.lamB : 0.0f, d4 = g.d4[r];
            vu = 2.0f * w * d4;
            vhv = 2.0f * w * g.dd4[r] * zeta4 + g.dz4[r];
            if (j == 0) {
                g.vh[r] = vhv;
                g.prow[r] = r < g.B ? static_cast<double>(d4) * zeta4 / g.B : 0.0;
            }
        }
        // pass 2: layer-3 reverse step and the w4 / b2 column sums
        for (int c = c_lo; c < c_hi; c += 16) {
            tmem_ld16(tl + c, v);
            load16(g.h, r, c, x);
            float st[16], sp[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const float h = x[i], gt = 1.0f - h * h, w4 = sw[c + i];
                const float bu = vu * w4, bh = fmaf(-2.0f * h * v[i], bu, vhv * w4);
                st[i] = gt * bu;
                sp[i] = gt * bh;
                x[i] = fmaf(vu, v[i] * gt, vhv * h);  // gw4 term: b_ζ4 u3 + b_z4 H3
            }
            store16(g.out[0], r, c, st);
            store16(g.out[1], r, c, sp);
            colsum16(x, cacc[0][(c - c_lo) >> 4], lane);
            colsum16(sp, cacc[1][(c - c_lo) >> 4], lane);
        }
    } else {  // kEpiRev: accumulator columns [0, 128) tangent rows (b_u), [128, 256) primal rows (b_h)
        // b_ζ = G∘b_u, b_z = G∘(b_h − 2H∘ζ∘b_u) = G∘b_h − 2H∘u∘b_u with u = G∘ζ, the gated
        // tangent stored as the next layer's operand (g.z): no pre-gate tangent image
        for (int c = c_lo; c < c_hi; c += 16) {
            float bh[16], ut[16];
            const int oc = obase + c;
            tmem_ld16(tl + c, v);
            tmem_ld16(tl + 128 + c, bh);
            load16(g.h, r, oc, x);
            load16(g.z, r, oc, ut);
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const float h = x[i], gt = 1.0f - h * h;
                const float sp = fmaf(-2.0f * h * ut[i], v[i], gt * bh[i]);
                v[i] = valid ? gt * v[i] : 0.0f;
                bh[i] = valid ? sp : 0.0f;
            }
            store16(g.out[0], r, oc, v);
            store16(g.out[1], r, oc, bh);
            colsum16(bh, cacc[0][(c - c_lo) >> 4], lane);
        }
    }
}

template <int EPI>
__global__ void __launch_bounds__(kRowThreads, 1) row_gemm_kernel(const RowArgs g) {
    constexpr bool kDual = EPI == kEpiRev;
    constexpr int kA = kDual ? 2 : 1;
    extern __shared__ __align__(1024) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kRowStages * kRowStageBytes);
    uint64_t* empty = full + kRowStages;
    uint64_t* acc_full = empty + kRowStages;  // [2]
    uint64_t* acc_empty = acc_full + 2;       // [2]
    uint32_t* tslot = reinterpret_cast<uint32_t*>(acc_empty + 2);
    float* sdot = reinterpret_cast<float*>(smem + kRowStages * kRowStageBytes + 256);  // [2][4][128] row partial dots
    float* sb = sdot + 2 * 4 * 128;                                                     // [256] bias
    float* sw = sb + 256;                                                               // [256] head weights
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int KC = g.a_cols / kKC, kblk = g.a_cols >> 7;
    const int nbu = kDual ? 1 : g.nb;                        // B blocks per unit
    const int units = kDual ? g.tiles * g.nb : g.tiles;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kRowStages; ++s) {
            bar_init(&full[s], 1);
            bar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            bar_init(&acc_full[b], 1);
            bar_init(&acc_empty[b], kRowEpiWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(tslot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tslot;

    // stage slots: A (hi, lo) per half, then B (hi, lo) per 128-column block
    if (warp == 0 && lane == 0) {
        const bool lo = g.passes == 3;
        const uint32_t bytes = static_cast<uint32_t>((kA + nbu) * (lo ? 2 : 1) * kChunk);
        int gk = 0;
        for (int u = blockIdx.x; u < units; u += gridDim.x) {
            const int mb = kDual ? u / g.nb : u, n0 = kDual ? u % g.nb : 0;
            for (int kc = 0; kc < KC; ++kc, ++gk) {
                const int s = gk % kRowStages;
                if (gk >= kRowStages) bar_wait(&empty[s], ((gk / kRowStages) - 1) & 1);
                unsigned char* st = smem + s * kRowStageBytes;
                bar_expect(&full[s], bytes);
                const size_t aoff = (static_cast<size_t>(mb) * kblk + (kc >> 2)) * 16384 + (kc & 3) * 4096;
#pragma unroll
                for (int a = 0; a < kA; ++a) {
                    bulk(st + (2 * a) * kChunk, g.a_hi[a] + aoff, kChunk, &full[s]);
                    if (lo) bulk(st + (2 * a + 1) * kChunk, g.a_lo[a] + aoff, kChunk, &full[s]);
                }
                for (int n = 0; n < nbu; ++n) {
                    const size_t woff = (static_cast<size_t>(n0 + n) * kblk + (kc >> 2)) * 16384 + (kc & 3) * 4096;
                    bulk(st + (2 * kA + 2 * n) * kChunk, g.w_hi + woff, kChunk, &full[s]);
                    if (lo) bulk(st + (2 * kA + 2 * n + 1) * kChunk, g.w_lo + woff, kChunk, &full[s]);
                }
            }
        }
    } else if (warp == 1 && lane == 0) {
        constexpr uint32_t id = idesc128(0);
        int gk = 0, it = 0;
        for (int u = blockIdx.x; u < units; u += gridDim.x, ++it) {
            const int buf = it & 1;
            if (it >= 2) bar_wait(&acc_empty[buf], ((it >> 1) - 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t tb = tmem + buf * 256;
            for (int kc = 0; kc < KC; ++kc, ++gk) {
                const int s = gk % kRowStages;
                bar_wait(&full[s], (gk / kRowStages) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t st = su32(smem + s * kRowStageBytes);
#pragma unroll
                for (int ks = 0; ks < kKC / 16; ++ks) {
#pragma unroll
                    for (int a = 0; a < kA; ++a) {
                        const uint64_t ah = sdesc(st + (2 * a) * kChunk + ks * 4096, 2048, 128);
                        const uint64_t al = sdesc(st + (2 * a + 1) * kChunk + ks * 4096, 2048, 128);
                        for (int n = 0; n < nbu; ++n) {
                            const uint64_t bh = sdesc(st + (2 * kA + 2 * n) * kChunk + ks * 4096, 2048, 128);
                            const uint64_t bl = sdesc(st + (2 * kA + 2 * n + 1) * kChunk + ks * 4096, 2048, 128);
                            const uint32_t tm = tb + (a + n) * 128;
                            const uint32_t acc = (kc > 0 || ks > 0) ? 1u : 0u;
                            if (g.passes == 3) {  // small terms first
                                mma(tm, al, bh, id, acc);
                                mma(tm, ah, bl, id, 1u);
                                mma(tm, ah, bh, id, 1u);
                            } else {
                                mma(tm, ah, bh, id, acc);
                            }
                        }
                    }
                }
                commit(&empty[s]);
            }
            commit(&acc_full[buf]);
        }
    } else if (warp >= 2) {
        // bias / head weights, zero past the valid columns (padding stays 0)
        for (int c = threadIdx.x - 64; c < 256; c += 32 * kRowEpiWarps) {
            sb[c] = (g.bias && c < g.n_valid) ? g.bias[c] : 0.0f;
            sw[c] = (g.w4 && c < g.n_valid) ? g.w4[c] : 0.0f;
        }
        epi_bar();
        const int q = warp & 3, j = (warp - 2) >> 2;
        double cacc[2][4] = {{0.0, 0.0, 0.0, 0.0}, {0.0, 0.0, 0.0, 0.0}};  // column sums of this warp's slice
        int it = 0;
        for (int u = blockIdx.x; u < units; u += gridDim.x, ++it) {
            const int buf = it & 1;
            bar_wait(&acc_full[buf], (it >> 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            row_unit_epilogue<EPI>(g, tmem + buf * 256, sdot + buf * 512, sb, sw, kDual ? u / g.nb : u,
                                   kDual ? u % g.nb : 0, q, j, lane, cacc);
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&acc_empty[buf])) : "memory");
        }
        if (EPI == kEpiTHead || EPI == kEpiRev) {  // one partial row per (CTA, lane quarter); the slice's columns
            // (a dual CTA always serves the same column half: gridDim.x is even or covers every unit once)
            const int ncols = kDual ? 128 : g.nb * 128, sl = ncols >> 2, c_lo = j * sl;
            const int obase = kDual ? (blockIdx.x % g.nb) * 128 : 0;
            if (lane < 16)
                for (int ci = 0; ci < (sl >> 4); ++ci)
#pragma unroll
                    for (int v = 0; v < 2; ++v)
                        if (g.colpart[v])
                            g.colpart[v][static_cast<size_t>(blockIdx.x * 4 + q) * g.ldc + obase + c_lo + 16 * ci +
                                         lane] = static_cast<float>(cacc[v][ci]);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

// ---- weight-gradient GEMMs: gW[o, i] = Σ_r S_t[r,o] A_t[r,i] + S_p[r,o] A_p[r,i] ---
// CTA (o-tile, split) accumulates its share of the 32-row chunks of both halves
// in TMEM (M = 128 o, N = 128 i per MMA, both operands MN-major) and writes an
// fp32 partial [split][i][o] (o contiguous = the θ layout of W).  A chunk of an
// image (32 rows x 128 columns, 16 column groups of 512 B, 2 KB apart in the
// block) is ONE 5-D TMA tensor copy (see img_tmap), landing with column groups
// 512 B apart: MN-group stride (SBO) 512 B, K-group (row-group) stride 128 B.
constexpr int kWgThreads = 192;  // warp 0 TMA producer, warp 1 MMA issuer, warps 2-5 epilogue
constexpr int kWgRows = 32;
constexpr int kWgBlk = 16 * 512;           // 8 KB: 128 columns x 32 rows
constexpr int kWgStages = 4;
constexpr int kWgStageBytes = 6 * kWgBlk;  // S hi/lo + A hi/lo for <= 2 column blocks
constexpr size_t kWgSmem = static_cast<size_t>(kWgStages) * kWgStageBytes + 256;

struct alignas(64) WgMaps {
    CUtensorMap s[2][2];  // [half][hi, lo]
    CUtensorMap a[2][2];
};

struct WgArgs {
    int s_cols = 0;  // M extent (o), multiple of 128
    int a_cols = 0;  // N extent (i), 128 or 256
    int chunks = 0;  // 32-row chunks per half
    int splits = 1;
    int passes = 3;
    float* part = nullptr;
};

__device__ __forceinline__ void tma5(void* dst, const CUtensorMap* map, int c1, int c3, int c4, uint64_t* b) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, "
        "%6}], [%7];" ::"r"(su32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(0), "r"(c1), "r"(0), "r"(c3), "r"(c4), "r"(su32(b))
        : "memory");
}

__global__ void __launch_bounds__(kWgThreads, 1) wgrad_kernel(const __grid_constant__ WgMaps maps, const WgArgs g) {
    extern __shared__ __align__(1024) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kWgStages * kWgStageBytes);
    uint64_t* empty = full + kWgStages;
    uint64_t* acc_full = empty + kWgStages;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(acc_full + 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ot = blockIdx.x, sp = blockIdx.y, nb = g.a_cols >> 7;
    const int total = 2 * g.chunks;
    const int t0 = static_cast<int>(static_cast<long long>(sp) * total / g.splits);
    const int t1 = static_cast<int>(static_cast<long long>(sp + 1) * total / g.splits);

    if (threadIdx.x == 0) {
        for (int s = 0; s < kWgStages; ++s) {
            bar_init(&full[s], 1);
            bar_init(&empty[s], 1);
        }
        bar_init(acc_full, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(tslot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tslot;

    if (warp == 0 && lane == 0) {
        const bool lo = g.passes == 3;
        const uint32_t bytes = static_cast<uint32_t>((1 + nb) * (lo ? 2 : 1) * kWgBlk);
        for (int t = t0; t < t1; ++t) {
            const int k = t - t0, s = k % kWgStages;
            if (k >= kWgStages) bar_wait(&empty[s], ((k / kWgStages) - 1) & 1);
            bar_expect(&full[s], bytes);
            const int half = t >= g.chunks ? 1 : 0, row0 = (t - half * g.chunks) * kWgRows;
            const int rb = row0 >> 7, qt = (row0 >> 5) & 3;
            unsigned char* st = smem + s * kWgStageBytes;
            // slots: 0 S_hi, 1 S_lo, 2 + 2n A_hi(n), 3 + 2n A_lo(n)
            tma5(st, &maps.s[half][0], qt, ot, rb, &full[s]);
            if (lo) tma5(st + kWgBlk, &maps.s[half][1], qt, ot, rb, &full[s]);
            for (int n = 0; n < nb; ++n) {
                tma5(st + (2 + 2 * n) * kWgBlk, &maps.a[half][0], qt, n, rb, &full[s]);
                if (lo) tma5(st + (3 + 2 * n) * kWgBlk, &maps.a[half][1], qt, n, rb, &full[s]);
            }
        }
    } else if (warp == 1 && lane == 0) {
        constexpr uint32_t id = idesc128(1);
        for (int t = t0; t < t1; ++t) {
            const int k = t - t0, s = k % kWgStages;
            bar_wait(&full[s], (k / kWgStages) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t st = su32(smem + s * kWgStageBytes);
#pragma unroll
            for (int ks = 0; ks < kWgRows / 16; ++ks) {
                const uint64_t sh = sdesc(st + ks * 256, 128, 512), sl = sdesc(st + kWgBlk + ks * 256, 128, 512);
                for (int n = 0; n < nb; ++n) {
                    const uint64_t ah = sdesc(st + (2 + 2 * n) * kWgBlk + ks * 256, 128, 512);
                    const uint64_t al = sdesc(st + (3 + 2 * n) * kWgBlk + ks * 256, 128, 512);
                    const uint32_t tm = tmem + n * 128, acc = (k > 0 || ks > 0) ? 1u : 0u;
                    if (g.passes == 3) {
                        mma(tm, sl, ah, id, acc);
                        mma(tm, sh, al, id, 1u);
                        mma(tm, sh, ah, id, 1u);
                    } else {
                        mma(tm, sh, ah, id, acc);
                    }
                }
            }
            commit(&empty[s]);
        }
        commit(acc_full);
    } else if (warp >= 2) {
        const int q = warp & 3, o = ot * 128 + q * 32 + lane;
        bar_wait(acc_full, 0);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t tl = tmem + (static_cast<uint32_t>(q * 32) << 16);
        float* dst = g.part + static_cast<size_t>(sp) * g.a_cols * g.s_cols + o;
        const bool empty_range = t1 <= t0;
        for (int c = 0; c < g.a_cols; c += 32) {
            float v[32];
            tmem_ld32(tl + c, v);
#pragma unroll
            for (int i = 0; i < 32; ++i) dst[static_cast<size_t>(c + i) * g.s_cols] = empty_range ? 0.0f : v[i];
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
}

// ---- small kernels ---------------------------------------------------------------
// X image rows [0, rows_p): Δ rows, then the zero row (D(0) term), zeros after;
// one thread per (row, 8-column group).
__global__ void pack_input_kernel(const float* __restrict__ delta, int B, int ld, int din, int rows_p, Img X) {
    // consecutive threads = consecutive rows of one 8-column group: a warp's 16-B
    // stores fill 512 contiguous bytes of the column-group-major image
    const int groups = X.cols_p >> 3;
    const long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (t >= static_cast<long long>(rows_p) * groups) return;
    const int r = static_cast<int>(t % rows_p), c0 = static_cast<int>(t / rows_p) * 8;
    float v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int c = c0 + i;
        v[i] = (r < B && c < din) ? delta[static_cast<size_t>(r) * ld + c] : 0.0f;
    }
    store8(X, r, c0, v);
}

// Weight images from the f64 master parameters: fwd (rows = out, cols = in) and
// bwd (rows = in, cols = out) of each hidden layer W (out x in, column-major in θ).
struct WPack {
    const double* W[3];
    int out[3], in[3];
    Img fwd[3], bwd[3];
};
__global__ void pack_weights_kernel(WPack P) {
    const int l = blockIdx.y >> 1, tr = blockIdx.y & 1;
    const Img& im = tr ? P.bwd[l] : P.fwd[l];
    const int rows_p = tr ? ((P.in[l] + 127) & ~127) : ((P.out[l] + 127) & ~127);
    const int groups = im.cols_p >> 3;
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= rows_p * groups) return;
    const int n = t / groups, k0 = (t % groups) * 8;
    uint32_t h[4], lw[4];
#pragma unroll
    for (int i = 0; i < 8; i += 2) {
        double w[2];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const int k = k0 + i + j;
            const int o = tr ? k : n, c = tr ? n : k;  // W[o, c]
            w[j] = (o < P.out[l] && c < P.in[l]) ? P.W[l][static_cast<size_t>(c) * P.out[l] + o] : 0.0;
        }
        const bf16 a = __double2bfloat16(w[0]), b = __double2bfloat16(w[1]);
        h[i / 2] = pack2(a, b);
        lw[i / 2] = pack2(__double2bfloat16(w[0] - static_cast<double>(__bfloat162float(a))),
                          __double2bfloat16(w[1] - static_cast<double>(__bfloat162float(b))));
    }
    const size_t o = iofs(n, k0, im.cols_p);
    *reinterpret_cast<uint4*>(im.hi + o) = make_uint4(h[0], h[1], h[2], h[3]);
    *reinterpret_cast<uint4*>(im.lo + o) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
}

// All fixed-order gradient reductions in one launch (blockIdx.y = job):
//   jobs 0-2: grad_W[i * out + o] = Σ_s part[s][i][o] (f64; four interleaved
//             partial sums combined in a fixed order), one thread per element;
//   (the column sums of the bias / w4 gradients: colsum_reduce_kernel).
struct RedJobs {
    const float* part[3];
    int splits[3], a_cols[3], n_in[3];
    float* gW[3];
    const float* cp[4];
    float* cout[4];
    int s_cols, n_out, cp_rows, ldc;
};
__global__ void __launch_bounds__(256) grad_reduce_kernel(const RedJobs J) {
    const int job = blockIdx.y;
    if (job < 3) {
        const int t = blockIdx.x * 256 + threadIdx.x;
        if (t >= J.n_in[job] * J.n_out) return;
        const int i = t / J.n_out, o = t % J.n_out;
        const float* p = J.part[job] + static_cast<size_t>(i) * J.s_cols + o;
        const size_t st = static_cast<size_t>(J.a_cols[job]) * J.s_cols;
        double s[4] = {0.0, 0.0, 0.0, 0.0};
        int k = 0;
        for (; k + 3 < J.splits[job]; k += 4)
#pragma unroll
            for (int u = 0; u < 4; ++u) s[u] += p[(k + u) * st];
        for (; k < J.splits[job]; ++k) s[0] += p[k * st];
        J.gW[job][t] = static_cast<float>((s[0] + s[1]) + (s[2] + s[3]));
    }
}

// Column sums out[j] = Σ_rows colpart[row][j] (blockIdx.y = vector): 32 columns per
// 1024-thread block, lanes = columns (coalesced rows), 32 warps = row strides, four
// interleaved f64 accumulators per thread; fixed-order combination.
__global__ void __launch_bounds__(1024) colsum_reduce_kernel(const RedJobs J) {
    __shared__ double red[32][33];
    const int v = blockIdx.y;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, j = blockIdx.x * 32 + lane;
    double s[4] = {0.0, 0.0, 0.0, 0.0};
    if (j < J.n_out) {
        const float* c = J.cp[v] + j;
        int r = w;
        for (; r + 96 < J.cp_rows; r += 128)
#pragma unroll
            for (int u = 0; u < 4; ++u) s[u] += c[static_cast<size_t>(r + 32 * u) * J.ldc];
        for (; r < J.cp_rows; r += 32) s[0] += c[static_cast<size_t>(r) * J.ldc];
    }
    red[w][lane] = (s[0] + s[1]) + (s[2] + s[3]);
    __syncthreads();
    if (w == 0 && j < J.n_out) {
        double t = 0.0;
        for (int k = 0; k < 32; ++k) t += red[k][lane];
        J.cout[v][j] = static_cast<float>(t);
    }
}


// Row reductions of the loss terms and the head-bias gradient, fixed order:
// block b sums rows [b R / nb, (b + 1) R / nb) into part[b] = {Σ lrow, Σ prow, Σ b_z4};
// loss_final then sums the blocks in order: loss = {total, logistic, mean penalty},
// gb4 = Σ b_z4.
constexpr int kLossBlocks = 148;
__global__ void __launch_bounds__(256) loss_part_kernel(const double* __restrict__ lrow,
                                                        const double* __restrict__ prow, const float* __restrict__ vh,
                                                        int R, double* part) {
    __shared__ double red[3][8];
    const int i0 = static_cast<int>(static_cast<long long>(blockIdx.x) * R / gridDim.x);
    const int i1 = static_cast<int>(static_cast<long long>(blockIdx.x + 1) * R / gridDim.x);
    double a = 0.0, b = 0.0, c = 0.0;
    for (int i = i0 + threadIdx.x; i < i1; i += 256) {
        a += lrow[i];
        b += prow[i];
        c += vh[i];
    }
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
        c += __shfl_xor_sync(0xffffffffu, c, o);
    }
    if ((threadIdx.x & 31) == 0) {
        red[0][threadIdx.x >> 5] = a;
        red[1][threadIdx.x >> 5] = b;
        red[2][threadIdx.x >> 5] = c;
    }
    __syncthreads();
    if (threadIdx.x < 3) {
        double t = 0.0;
        for (int w = 0; w < 8; ++w) t += red[threadIdx.x][w];
        part[blockIdx.x * 3 + threadIdx.x] = t;
    }
}
__global__ void loss_final_kernel(const double* __restrict__ part, int nb, double lam, double* loss, float* gb4) {
    const int lane = threadIdx.x;  // one warp: lane-strided sums, fixed butterfly
    double s = 0.0, p = 0.0, g = 0.0;
    for (int k = lane; k < nb; k += 32) {
        s += part[3 * k];
        p += part[3 * k + 1];
        g += part[3 * k + 2];
    }
    for (int o = 16; o > 0; o >>= 1) {
        s += __shfl_xor_sync(0xffffffffu, s, o);
        p += __shfl_xor_sync(0xffffffffu, p, o);
        g += __shfl_xor_sync(0xffffffffu, g, o);
    }
    if (lane == 0) {
        loss[0] = s + lam * p;
        loss[1] = s;
        loss[2] = p;
        *gb4 = static_cast<float>(g);
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
    int Hp = 0, Dp = 0, rows_p = 0;  // padded widths, padded row capacity (multiple of 128)
    long long P = 0;
    long long o1 = 0, o2 = 0, o3 = 0;  // offsets of W1, W2, W3 (= w4) in θ
    double lr = 0.0, lam = 0.0;
    double *theta = nullptr, *m = nullptr, *v = nullptr;
    float *theta32 = nullptr, *grad = nullptr;
    long long* counts = nullptr;  // {Adam step_count, skipped}
    int* bad = nullptr;
    // split images (see iofs)
    Img X, Xt, H1, H2, H3, D3, T2, T1, At1, At2, St, Sp, Ut, Up;
    Img Wf[3], Wb[3];
    float *d4 = nullptr, *dd4 = nullptr, *dz4 = nullptr, *vh = nullptr;
    double *lrow = nullptr, *prow = nullptr, *loss = nullptr, *lpart = nullptr;
    float* colpart[4] = {};  // gw4, gb2, gb1, gb0 per-warp column sums
    float* part[3] = {};     // weight-gradient partials
    int splits[3] = {1, 1, 1};
    std::vector<void*> allocs;
    std::vector<std::pair<const void*, CUtensorMap>> maps;  // weight-gradient operand views of the image planes
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

template <class T>
T* talloc(msk_disc_trainer* t, size_t n) {
    void* p = nullptr;
    ckc(cudaMalloc(&p, std::max<size_t>(1, n) * sizeof(T)), "cudaMalloc");
    ckc(cudaMemset(p, 0, std::max<size_t>(1, n) * sizeof(T)), "cudaMemset");
    t->allocs.push_back(p);
    return static_cast<T*>(p);
}

// 5-D tensor map of one plane of a split image for the weight-gradient GEMMs, in
// 4-byte units: {128 (4 row groups = 512 B), 4 row quarters, 16 column groups,
// column blocks, row blocks}; box {128, 1, 16, 1, 1} = a 32-row x 128-column chunk.
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
CUtensorMap img_tmap(const bf16* plane, int rows_p, int cols_p) {
    if (!g_encode) {
        cudaDriverEntryPointQueryResult q;
        void* fn = nullptr;
        ckc(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q), "cuTensorMapEncodeTiled");
        if (!fn || q != cudaDriverEntryPointSuccess) throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
        g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    CUtensorMap m;
    const cuuint64_t dims[5] = {128, 4, 16, static_cast<cuuint64_t>(cols_p >> 7), static_cast<cuuint64_t>(rows_p >> 7)};
    const cuuint64_t strides[4] = {512, 2048, 32768, 32768ull * (cols_p >> 7)};  // bytes, dims 1..4
    const cuuint32_t box[5] = {128, 1, 16, 1, 1}, estr[5] = {1, 1, 1, 1, 1};
    const CUresult r = g_encode(&m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 5, const_cast<bf16*>(plane), dims, strides, box,
                                estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled failed: " + std::to_string(r));
    return m;
}

Img img_alloc(msk_disc_trainer* t, int rows_p, int cols_p) {
    Img im;
    im.cols_p = cols_p;
    im.hi = talloc<bf16>(t, static_cast<size_t>(rows_p) * cols_p);
    im.lo = talloc<bf16>(t, static_cast<size_t>(rows_p) * cols_p);
    t->maps.emplace_back(im.hi, img_tmap(im.hi, rows_p, cols_p));
    t->maps.emplace_back(im.lo, img_tmap(im.lo, rows_p, cols_p));
    return im;
}

bool g_prepared = false;
template <int EPI>
void prep_row() {
    ckc(cudaFuncSetAttribute(row_gemm_kernel<EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(kRowSmem)),
        "cudaFuncSetAttribute");
}
int g_sms = 148;
void prepare_kernels() {
    if (g_prepared) return;
    prep_row<kEpiTanh>();
    prep_row<kEpiHead>();
    prep_row<kEpiGate>();
    prep_row<kEpiPlain>();
    prep_row<kEpiTHead>();
    prep_row<kEpiRev>();
    int dev = 0;
    ckc(cudaGetDevice(&dev), "cudaGetDevice");
    ckc(cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev), "cudaDeviceGetAttribute");
    ckc(cudaFuncSetAttribute(wgrad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kWgSmem)),
        "cudaFuncSetAttribute");
    g_prepared = true;
}

template <int EPI>
void row(RowArgs a, int tiles, cudaStream_t s) {
    a.tiles = tiles;
    const int units = EPI == kEpiRev ? tiles * a.nb : tiles;
    row_gemm_kernel<EPI><<<std::min(units, g_sms), kRowThreads, kRowSmem, s>>>(a);
}

RowArgs rargs(const msk_disc_trainer* t, const Img& A, const Img& W, int n_out, int rows) {
    RowArgs a;
    a.a_hi[0] = A.hi;
    a.a_lo[0] = A.lo;
    a.a_cols = A.cols_p;
    a.w_hi = W.hi;
    a.w_lo = W.lo;
    a.nb = n_out >> 7;
    a.n_valid = t->H;  // bias / w4 length (only the hidden-width epilogues read them)
    a.rows = rows;
    a.passes = t->math == 0 ? 3 : 1;
    return a;
}

const CUtensorMap& tmap_of(const msk_disc_trainer* t, const void* plane) {
    for (const auto& m : t->maps)
        if (m.first == plane) return m.second;
    throw std::runtime_error("disc_train: no tensor map for an image plane");
}

void wgrad(const msk_disc_trainer* t, const Img& S0, const Img& S1, const Img& A0, const Img& A1, int chunks,
           int splits, float* part, cudaStream_t s) {
    WgMaps m;
    const Img* ims[4] = {&S0, &S1, &A0, &A1};
    for (int k = 0; k < 4; ++k) {
        CUtensorMap* dst = k < 2 ? m.s[k] : m.a[k - 2];
        dst[0] = tmap_of(t, ims[k]->hi);
        dst[1] = tmap_of(t, ims[k]->lo);
    }
    WgArgs w;
    w.s_cols = S0.cols_p;
    w.a_cols = A0.cols_p;
    w.chunks = chunks;
    w.splits = splits;
    w.passes = t->math == 0 ? 3 : 1;
    w.part = part;
    wgrad_kernel<<<dim3(S0.cols_p >> 7, splits), kWgThreads, kWgSmem, s>>>(m, w);
}

// splits of a weight-gradient GEMM: ~one wave of CTAs over the o-tiles
int wg_splits(int o_tiles, int total_chunks) { return std::max(1, std::min((148 + o_tiles - 1) / o_tiles, total_chunks)); }

void pack_weights(msk_disc_trainer* t, cudaStream_t s) {
    WPack P;
    const long long off[3] = {0, t->o1, t->o2};
    for (int l = 0; l < 3; ++l) {
        P.W[l] = t->theta + off[l];
        P.out[l] = t->H;
        P.in[l] = l == 0 ? t->din : t->H;
        P.fwd[l] = t->Wf[l];
        P.bwd[l] = t->Wb[l];
    }
    const int maxn = std::max(t->Hp, t->Dp) * (std::max(t->Hp, t->Dp) >> 3);
    pack_weights_kernel<<<dim3((maxn + 255) / 256, 6), 256, 0, s>>>(P);
}

// Loss and dloss/dθ (into t->grad) for B rows of Δ at the current parameters.
void loss_and_grad(msk_disc_trainer* t, const float* delta, int B, int ld, cudaStream_t s) {
    const int H = t->H, din = t->din, R = B + 1, tiles = (R + 127) / 128, rows_p = tiles * 128;
    const int chunks = (R + kWgRows - 1) / kWgRows;
    const float* th = t->theta32;
    const float *b0 = th + static_cast<long long>(H) * din, *b1 = th + t->o1 + static_cast<long long>(H) * H,
                *b2 = th + t->o2 + static_cast<long long>(H) * H, *w4 = th + t->o3, *b4 = th + t->o3 + H;
    float* g = t->grad;
    float *gW0 = g, *gb0 = g + static_cast<long long>(H) * din, *gW1 = g + t->o1,
          *gb1 = g + t->o1 + static_cast<long long>(H) * H, *gW2 = g + t->o2,
          *gb2 = g + t->o2 + static_cast<long long>(H) * H, *gw4 = g + t->o3, *gb4 = g + t->o3 + H;
    const int Hp = t->Hp, Dp = t->Dp;

    // per-(CTA, lane quarter) column-sum partials: rows a kernel's grid does not reach stay 0
    const int cp_rows = std::min(tiles * 2, g_sms) * 4;
    for (int k = 0; k < 4; ++k)
        ckc(cudaMemsetAsync(t->colpart[k], 0, static_cast<size_t>(cp_rows) * Hp * sizeof(float), s), "colpart");
    {
        const long long n = static_cast<long long>(rows_p) * (Dp >> 3);
        pack_input_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(delta, B, ld, din, rows_p, t->X);
    }
    // ---- forward (nn.cpp:54-73) + head (nn.cpp:66-68) ----
    RowArgs a = rargs(t, t->X, t->Wf[0], Hp, R);
    a.bias = b0;
    a.out[0] = t->H1;
    row<kEpiTanh>(a, tiles, s);
    a = rargs(t, t->H1, t->Wf[1], Hp, R);
    a.bias = b1;
    a.out[0] = t->H2;
    row<kEpiTanh>(a, tiles, s);
    a = rargs(t, t->H2, t->Wf[2], Hp, R);
    a.bias = b2;
    a.w4 = w4;
    a.b4 = b4;
    a.out[0] = t->H3;
    a.out[1] = t->D3;
    a.d4 = t->d4;
    a.dd4 = t->dd4;
    a.dz4 = t->dz4;
    a.lrow = t->lrow;
    a.B = B;
    row<kEpiHead>(a, tiles, s);
    // ---- input gradient g = dy/dx (nn.cpp:161-164) ----
    a = rargs(t, t->D3, t->Wb[2], Hp, R);
    a.h = t->H2;
    a.out[0] = t->T2;
    row<kEpiGate>(a, tiles, s);
    a = rargs(t, t->T2, t->Wb[1], Hp, R);
    a.h = t->H1;
    a.out[0] = t->T1;
    row<kEpiGate>(a, tiles, s);
    a = rargs(t, t->T1, t->Wb[0], Dp, R);
    a.out[0] = t->Xt;
    row<kEpiPlain>(a, tiles, s);
    // ---- forward tangent along g (nn.cpp:167-171) ----
    a = rargs(t, t->Xt, t->Wf[0], Hp, R);
    a.h = t->H1;
    a.out[0] = t->At1;
    row<kEpiGate>(a, tiles, s);
    a = rargs(t, t->At1, t->Wf[1], Hp, R);
    a.h = t->H2;
    a.out[0] = t->At2;
    row<kEpiGate>(a, tiles, s);
    a = rargs(t, t->At2, t->Wf[2], Hp, R);
    a.h = t->H3;
    a.w4 = w4;
    a.d4 = t->d4;
    a.dd4 = t->dd4;
    a.dz4 = t->dz4;
    a.vh = t->vh;
    a.prow = t->prow;
    a.B = B;
    a.lamB = static_cast<float>(t->lam / B);
    a.out[0] = t->St;
    a.out[1] = t->Sp;
    a.colpart[0] = t->colpart[0];
    a.colpart[1] = t->colpart[1];
    a.ldc = Hp;
    row<kEpiTHead>(a, tiles, s);
    // ---- reverse pass over [tangent; primal] (nn.cpp:186-221 + nn.cpp:98-128) ----
    wgrad(t, t->St, t->Sp, t->At2, t->H2, chunks, t->splits[2], t->part[2], s);
    a = rargs(t, t->St, t->Wb[2], Hp, R);
    a.a_hi[1] = t->Sp.hi;
    a.a_lo[1] = t->Sp.lo;
    a.h = t->H2;
    a.z = t->At2;
    a.out[0] = t->Ut;
    a.out[1] = t->Up;
    a.colpart[0] = t->colpart[2];
    a.ldc = Hp;
    row<kEpiRev>(a, tiles, s);
    wgrad(t, t->Ut, t->Up, t->At1, t->H1, chunks, t->splits[1], t->part[1], s);
    a = rargs(t, t->Ut, t->Wb[1], Hp, R);
    a.a_hi[1] = t->Up.hi;
    a.a_lo[1] = t->Up.lo;
    a.h = t->H1;
    a.z = t->At1;
    a.out[0] = t->St;
    a.out[1] = t->Sp;
    a.colpart[0] = t->colpart[3];
    a.ldc = Hp;
    row<kEpiRev>(a, tiles, s);
    wgrad(t, t->St, t->Sp, t->Xt, t->X, chunks, t->splits[0], t->part[0], s);
    // ---- fixed-order reductions into the θ-layout gradient ----
    {
        RedJobs J;
        float* gws[3] = {gW0, gW1, gW2};
        for (int l = 0; l < 3; ++l) {
            J.part[l] = t->part[l];
            J.splits[l] = t->splits[l];
            J.a_cols[l] = l == 0 ? Dp : Hp;
            J.n_in[l] = l == 0 ? din : H;
            J.gW[l] = gws[l];
        }
        float* couts[4] = {gw4, gb2, gb1, gb0};
        for (int k = 0; k < 4; ++k) {
            J.cp[k] = t->colpart[k];
            J.cout[k] = couts[k];
        }
        J.s_cols = Hp;
        J.n_out = H;
        J.cp_rows = cp_rows;  // CTAs of the widest (dual) row GEMM x 4 lane quarters
        J.ldc = Hp;
        grad_reduce_kernel<<<dim3((std::max(din, H) * H + 255) / 256, 3), 256, 0, s>>>(J);
        colsum_reduce_kernel<<<dim3((H + 31) / 32, 4), 1024, 0, s>>>(J);
    }
    const int lb = std::min(kLossBlocks, R);
    loss_part_kernel<<<lb, 256, 0, s>>>(t->lrow, t->prow, t->vh, R, t->lpart);
    loss_final_kernel<<<1, 32, 0, s>>>(t->lpart, lb, t->lam, t->loss, gb4);
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
        if (n_in > 256 || hidden > 256)
            throw std::invalid_argument("disc_trainer: input width and hidden width must be <= 256");
        if (math < 0 || math > 1)
            throw std::invalid_argument("disc_trainer: math must be 0 (fp32-class split-bf16) or 1 (bf16)");
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
        prepare_kernels();
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
        t->Hp = static_cast<int>((H + 127) & ~127LL);
        t->Dp = static_cast<int>((din + 127) & ~127LL);
        t->theta = talloc<double>(t, P);
        t->m = talloc<double>(t, P);
        t->v = talloc<double>(t, P);
        t->theta32 = talloc<float>(t, P);
        t->grad = talloc<float>(t, P);
        t->counts = talloc<long long>(t, 2);
        t->bad = talloc<int>(t, 1);
        ckc(cudaMemcpy(t->theta, theta, P * sizeof(double), cudaMemcpyHostToDevice), "upload theta");
        to_f32_kernel<<<grid_for(P), 256>>>(t->theta, P, t->theta32);
        const int tiles = (max_rows + 1 + 127) / 128, rows_p = tiles * 128;
        t->rows_p = rows_p;
        const int Hp = t->Hp, Dp = t->Dp;
        t->X = img_alloc(t, rows_p, Dp);
        t->Xt = img_alloc(t, rows_p, Dp);
        for (Img* im : {&t->H1, &t->H2, &t->H3, &t->D3, &t->T2, &t->T1, &t->At1, &t->At2, &t->St, &t->Sp, &t->Ut,
                        &t->Up})
            *im = img_alloc(t, rows_p, Hp);
        for (int l = 0; l < 3; ++l) {
            const int inp = l == 0 ? Dp : Hp;
            t->Wf[l] = img_alloc(t, Hp, inp);
            t->Wb[l] = img_alloc(t, inp, Hp);
        }
        for (float** p : {&t->d4, &t->dd4, &t->dz4, &t->vh}) *p = talloc<float>(t, rows_p);
        t->lrow = talloc<double>(t, rows_p);
        t->prow = talloc<double>(t, rows_p);
        t->loss = talloc<double>(t, 3);
        t->lpart = talloc<double>(t, 3 * kLossBlocks);
        for (int k = 0; k < 4; ++k) t->colpart[k] = talloc<float>(t, static_cast<size_t>(std::max(tiles, 148) * 2) * 4 * Hp);
        const int total = 2 * ((max_rows + 1 + kWgRows - 1) / kWgRows);
        for (int l = 0; l < 3; ++l) {
            t->splits[l] = wg_splits(Hp >> 7, total);
            t->part[l] = talloc<float>(t, static_cast<size_t>(t->splits[l]) * (l == 0 ? Dp : Hp) * Hp);
        }
        pack_weights(t, nullptr);
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
    nvtxRangePushA("msk_disc_train_step");
    struct Pop {
        ~Pop() { nvtxRangePop(); }
    } pop_;
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
        pack_weights(t, s);  // the GEMM images of the new θ
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
