// Pipelined bf16 GEMM on the 5th-generation tensor cores with MLP epilogues:
// the building block of the on-device policy (π⁽⁰⁾ mean MLP and the flow field
// ψ) — one CTA per 128 x 256 output tile:
//   warp 0   TMA producer: 1-D bulk copies of pre-tiled A (16 KB) and W (32 KB)
//            K-blocks into a 4-stage shared-memory ring (mbarrier complete_tx);
//   warp 1   allocates 256 TMEM columns; one thread issues 4 tcgen05.mma
//            (M = 128, N = 256, K = 16) per K-block and commits each stage back
//            to the producer, then the accumulator to the epilogue;
//   warps 2-5 epilogue: tcgen05.ld of their TMEM lane quarter, bias (+ addend),
//            tanh -> bf16 tiled (next layer's A), fp32 affine head, or the flow
//            ODE update a += dt * ψ.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "mlp.cuh"

namespace msk_b200 {

namespace {

#ifndef MSK_GEMM_STAGES
#define MSK_GEMM_STAGES 4
#endif
#ifndef MSK_GEMM_MINB
#define MSK_GEMM_MINB 1
#endif
constexpr int kStages = MSK_GEMM_STAGES;
constexpr int kABytes = kGemmBM * kGemmBK * 2;  // 16 KB
constexpr int kWBytes = kGemmBN * kGemmBK * 2;  // 32 KB
// warp 0: TMA producer, warp 1: MMA issuer, warps 2-9: epilogue (two warps per
// TMEM lane quarter, each converting one 128-column half of the tile)
#ifndef MSK_GEMM_EPIW
#define MSK_GEMM_EPIW 8  // epilogue warps: 4 x (column slices per TMEM lane quarter)
#endif
constexpr int kEpiWarps = MSK_GEMM_EPIW;
constexpr int kGemmThreads = 64 + 32 * kEpiWarps;
constexpr int kEpiSlices = kEpiWarps / 4;

__host__ __device__ constexpr uint32_t blk_off(int r, int k) {  // inside a (rows x 64) block
    return static_cast<uint32_t>(((r >> 3) * 8 + (k >> 3)) * 128 + (r & 7) * 16 + (k & 7) * 2);
}

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
        "GW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra GW_%=;\n\t}" ::"r"(su32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     su32(dst)),
                 "l"(src), "r"(bytes), "r"(su32(b))
                 : "memory");
}
// 1-D bulk copy of `bytes` into the same CTA-relative offset of every CTA in
// ctaMask (TMA multicast), completing on each destination's mbarrier.
__device__ __forceinline__ void bulk_mc(void* dst, const void* src, uint32_t bytes, uint64_t* b, uint16_t mask) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], "
        "%4;" ::"r"(su32(dst)),
        "l"(src), "r"(bytes), "r"(su32(b)), "h"(mask)
        : "memory");
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

__device__ __forceinline__ uint64_t sdesc(uint32_t addr) {  // LBO 128 B, SBO 1024 B, version 1, no swizzle
    return static_cast<uint64_t>((addr >> 4) & 0x3FFF) | (static_cast<uint64_t>(128 >> 4) << 16) |
           (static_cast<uint64_t>(1024 >> 4) << 32) | (1ull << 46);
}
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(kGemmBN >> 3) << 17) |
                            (static_cast<uint32_t>(kGemmBM >> 4) << 24);

__device__ __forceinline__ void ld16(uint32_t taddr, float (&v)[16]) {
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

__device__ __forceinline__ void ld32(uint32_t taddr, float (&v)[2][16]) {
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
    for (int i = 0; i < 32; ++i) v[i >> 4][i & 15] = __uint_as_float(r[i]);
}

__device__ __forceinline__ float tanh_a(float x) {
    float y;
    asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ uint32_t bf2(float a, float b) {
    const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<const uint32_t*>(&h);
}

// 16 consecutive columns [n0, n0 + 16) of row m into a tiled bf16 image with
// KB = K/64 column blocks (two 16-B stores).
__device__ __forceinline__ void store_tiled16(void* img, int KB, int m, int n0, const float (&y)[16]) {
    char* base = static_cast<char*>(img) + (static_cast<size_t>(m >> 7) * KB + (n0 >> 6)) * kABytes;
    const int r = m & 127, k = n0 & 63;
    uint4 lo = make_uint4(bf2(y[0], y[1]), bf2(y[2], y[3]), bf2(y[4], y[5]), bf2(y[6], y[7]));
    uint4 hi = make_uint4(bf2(y[8], y[9]), bf2(y[10], y[11]), bf2(y[12], y[13]), bf2(y[14], y[15]));
    *reinterpret_cast<uint4*>(base + blk_off(r, k)) = lo;
    *reinterpret_cast<uint4*>(base + blk_off(r, k + 8)) = hi;
}

// Epilogues read at most one f32 source per output element: the addend (tanh
// layers with an addend, the affine head) or the running value they update
// (kEpiTanhAcc's sum, kEpiOde's action).  It is loaded 32 columns ahead into
// registers, so its (L2) latency overlaps the MMA tail and the TMEM loads.
// Row-major sources are addressed by row pointer; F4 sources (g.f4_rows > 0) by
// (base, m).
template <int EPI>
__device__ __forceinline__ const float* epi_src(const GemmArgs& g, int m, int& ld) {
    if (m >= g.M) return nullptr;
    if (EPI == kEpiTanhAcc || EPI == kEpiOde) {
        ld = g.ld_f;
        return g.out_f;
    }
    ld = g.ld_add;
    return g.addend;
}
template <int EPI>
__device__ __forceinline__ int epi_limit(const GemmArgs& g) {
    return (EPI == kEpiF32 || EPI == kEpiOde) ? g.n_valid : g.N;
}

// 32 source values of row m at columns [n0, n0 + 32) (0 outside the valid range).
// f4 > 0: base is an F4 buffer (see GemmArgs::f4_rows), row is unused.
__device__ __forceinline__ void load_src32(const float* row, const float* base, int f4, int m, int n0, int limit,
                                           bool vec, float (&x)[32]) {
    if (f4 > 0 && base) {
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
            float4 t = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
            if (n0 + i < limit)
                t = *reinterpret_cast<const float4*>(base + (static_cast<size_t>((n0 + i) >> 2) * f4 + m) * 4);
            x[i] = t.x;
            x[i + 1] = t.y;
            x[i + 2] = t.z;
            x[i + 3] = t.w;
        }
        return;
    }
    if (!row) {
#pragma unroll
        for (int i = 0; i < 32; ++i) x[i] = 0.0f;
        return;
    }
    if (vec && n0 + 32 <= limit) {
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
            const float4 t = *reinterpret_cast<const float4*>(row + n0 + i);
            x[i] = t.x;
            x[i + 1] = t.y;
            x[i + 2] = t.z;
            x[i + 3] = t.w;
        }
    } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) x[i] = n0 + i < limit ? row[n0 + i] : 0.0f;
    }
}

// 16 columns [n0, n0 + 16) of row m into an f32 output: row-major (op = row
// pointer) or F4 (base, m).
__device__ __forceinline__ void store_f16cols(float* op, float* base, int f4, int m, int n0, int limit, bool vec,
                                              const float* v) {
    if (f4 > 0) {
#pragma unroll
        for (int i = 0; i < 16; i += 4)
            if (n0 + i < limit)
                *reinterpret_cast<float4*>(base + (static_cast<size_t>((n0 + i) >> 2) * f4 + m) * 4) =
                    make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
        return;
    }
    if (vec && n0 + 16 <= limit) {
#pragma unroll
        for (int i = 0; i < 16; i += 4)
            *reinterpret_cast<float4*>(op + n0 + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
    } else {
#pragma unroll
        for (int i = 0; i < 16; ++i)
            if (n0 + i < limit) op[n0 + i] = v[i];
    }
}

// Bias / activation / store of 16 consecutive accumulator columns [n0, n0 + 16)
// of output row m (sb = the tile's staged biases of those columns, src = the
// preloaded f32 source values of those columns).
template <int EPI>
__device__ __forceinline__ void epi16(const GemmArgs& g, void* out_a, int m, int n0, int n_out_pad, const float* sb,
                                      const float* src, float (&v)[16]) {
    constexpr bool kTanh = EPI == kEpiTanhTiled || EPI == kEpiTanhPre || EPI == kEpiTanhAcc;
    const int f4 = g.f4_rows;
    float* orow = (m < g.M && g.out_f) ? (f4 > 0 ? g.out_f : g.out_f + static_cast<size_t>(m) * g.ld_f) : nullptr;
    const bool vec = (g.ld_f & 3) == 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = EPI == kEpiTanhPre ? fmaf(g.scale, v[i], sb[i]) : v[i] + sb[i];
    if (kTanh) {
        if (EPI != kEpiTanhAcc) {  // addend (0 when absent)
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] += src[i];
        }
        if (EPI == kEpiTanhPre && orow) store_f16cols(orow, g.out_f, f4, m, n0, g.N, vec, v);  // f32 pre-activation
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = n0 + i < g.N ? tanh_a(v[i]) : 0.0f;
        if (EPI == kEpiTanhAcc && orow) {  // running f32 sum of the activations
            float y[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) y[i] = src[i] + v[i];
            store_f16cols(orow, g.out_f, f4, m, n0, g.N, vec, y);
        }
        store_tiled16(out_a, n_out_pad / kGemmBK, m, n0, v);
    } else if (EPI == kEpiF32) {
        if (orow) {
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] = fmaf(g.scale, v[i], g.offset) + src[i];
            store_f16cols(orow, g.out_f, f4, m, n0, g.n_valid, vec, v);
        }
    } else {  // kEpiOde: a += dt * psi
        float y[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) y[i] = (orow && n0 + i < g.n_valid) ? fmaf(g.dt, v[i], src[i]) : 0.0f;
        if (orow) store_f16cols(orow, g.out_f, f4, m, n0, g.n_valid, vec, y);
        if (out_a) store_tiled16(out_a, n_out_pad / kGemmBK, m, n0, y);
    }
}

// Epilogue of one 128 x 256 output tile (row tile mb, column tile nb) by the
// eight epilogue warps (2-9): warp w reads TMEM lanes 32 (w % 4) .. + 31 (the
// hardware's lane-quarter rule) and columns [128 h, 128 h + 128), h = (w - 2) / 4,
// 32 columns per TMEM load (one wait per load).
template <int EPI>
__device__ __forceinline__ void gemm_epilogue(const GemmArgs& g, uint32_t tmem, float* sbias, uint64_t* acc_full,
                                              int mb, int nb, int warp, int lane, uint32_t parity = 0,
                                              void* out_a = nullptr, const float* bias = nullptr) {
    // out_a / bias: per-call overrides of g's (the persistent ODE kernel's layers)
    const float* bs = bias ? bias : g.bias;
    for (int i = threadIdx.x - 64; i < kGemmBN; i += kGemmThreads - 64) {  // stage the tile's biases
        const int n = nb * kGemmBN + i;
        sbias[i] = (bs && n < g.N) ? bs[n] : 0.0f;
    }
    void* oa = out_a ? out_a : g.out_a;
    const int q = warp & 3, r = q * 32 + lane, m = mb * kGemmBM + r;
    const int c_lo = ((warp - 2) / 4) * (kGemmBN / kEpiSlices), c_hi = c_lo + kGemmBN / kEpiSlices;
    int lds = 0;
    const float* sp = epi_src<EPI>(g, m, lds);
    const int f4 = g.f4_rows;
    const float* srow = (sp && f4 <= 0) ? sp + static_cast<size_t>(m) * lds : nullptr;
    const int limit = epi_limit<EPI>(g);
    const bool svec = (lds & 3) == 0;
    float cur[32], nxt[32];
    load_src32(srow, sp, f4, m, nb * kGemmBN + c_lo, limit, svec, cur);  // overlaps the MMA tail
    asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");  // epilogue warps only
    bar_wait(acc_full, parity);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t trow = tmem + (static_cast<uint32_t>(q * 32) << 16);
    const int n_out_pad = pad_to(EPI == kEpiOde ? g.n_valid : g.N, kGemmBK);  // tiled output width
    const int n_end = EPI == kEpiF32 ? g.n_valid : n_out_pad;
    for (int c = c_lo; c < c_hi; c += 32) {
        const int n0 = nb * kGemmBN + c;
        if (n0 >= n_end) break;  // columns past the valid / padded output width
        if (c + 32 < c_hi) load_src32(srow, sp, f4, m, n0 + 32, limit, svec, nxt);
        float v[2][16];
        ld32(trow + c, v);
        epi16<EPI>(g, oa, m, n0, n_out_pad, sbias + c, cur, v[0]);
        if (n0 + 16 < n_end) epi16<EPI>(g, oa, m, n0 + 16, n_out_pad, sbias + c + 16, cur + 16, v[1]);
#pragma unroll
        for (int i = 0; i < 32; ++i) cur[i] = nxt[i];
    }
}

// CL > 1: a cluster of CL CTAs along M shares each weight K-block: CTA r loads
// slice r of it and multicasts it to the whole cluster, so the per-SM weight
// traffic drops by CL; every MMA commit frees the stage in all CTAs of the
// cluster (multicast commit), which is what each producer waits for.
template <int EPI, int CL>
__global__ void __launch_bounds__(kGemmThreads, MSK_GEMM_MINB) gemm_kernel(GemmArgs g) {
extern __shared__ __align__(1024) unsigned char smem[];
unsigned char* sA = smem;                                    // kStages x 16 KB
unsigned char* sW = smem + kStages * kABytes;                // kStages x 32 KB
uint64_t* full = reinterpret_cast<uint64_t*>(sW + kStages * kWBytes);
uint64_t* empty = full + kStages;
uint64_t* acc_full = empty + kStages;
uint32_t* tslot = reinterpret_cast<uint32_t*>(acc_full + 1);
float* sbias = reinterpret_cast<float*>(smem + kStages * (kABytes + kWBytes) + 128);  // this tile's 256 biases
const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
const int mb = blockIdx.x, nb = blockIdx.y;
const int KB = pad_to(g.K, kGemmBK) / kGemmBK;

if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
        bar_init(&full[s], 1);
        bar_init(&empty[s], CL);  // one release per cluster CTA's MMAs
    }
    bar_init(acc_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
if constexpr (CL > 1) cluster_sync();  // peers' barriers exist before any multicast
if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tslot)),
                 "n"(kGemmBN)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
__syncthreads();
asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
const uint32_t tmem = *tslot;
// inputs may be the previous kernel's outputs (programmatic dependent launch)
asm volatile("griddepcontrol.wait;" ::: "memory");

if (warp == 0 && lane == 0) {  // TMA producer
    const char* A = static_cast<const char*>(g.A) + static_cast<size_t>(mb) * KB * kABytes;
    const char* W = static_cast<const char*>(g.W) + static_cast<size_t>(nb) * KB * kWBytes;
    const uint32_t rank = CL > 1 ? cluster_rank() : 0;
    constexpr uint32_t kSlice = kWBytes / CL;
    for (int kb = 0; kb < KB; ++kb) {
        const int s = kb % kStages;
        if (kb >= kStages) bar_wait(&empty[s], ((kb / kStages) - 1) & 1);
        bar_expect(&full[s], kABytes + kWBytes);
        bulk(sA + s * kABytes, A + static_cast<size_t>(kb) * kABytes, kABytes, &full[s]);
        if constexpr (CL == 1) {
            bulk(sW + s * kWBytes, W + static_cast<size_t>(kb) * kWBytes, kWBytes, &full[s]);
        } else {
            bulk_mc(sW + s * kWBytes + rank * kSlice, W + static_cast<size_t>(kb) * kWBytes + rank * kSlice, kSlice,
                    &full[s], static_cast<uint16_t>((1u << CL) - 1));
        }
    }
} else if (warp == 1 && lane == 0) {  // MMA issuer
    for (int kb = 0; kb < KB; ++kb) {
        const int s = kb % kStages;
        bar_wait(&full[s], (kb / kStages) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t a0 = su32(sA + s * kABytes), w0 = su32(sW + s * kWBytes);
#pragma unroll
        for (int k = 0; k < kGemmBK / 16; ++k) {
            const uint32_t acc = (kb > 0 || k > 0) ? 1u : 0u;
            asm volatile(
                "{\n\t.reg .pred p;\n\t"
                "setp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                "l"(sdesc(a0 + 256 * k)), "l"(sdesc(w0 + 256 * k)), "r"(kIdesc), "r"(acc)
                : "memory");
        }
        if constexpr (CL == 1) {
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                             su32(&empty[s]))
                         : "memory");
        } else {  // stage s of this CTA is free: tell every producer in the cluster
            asm volatile(
                "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], "
                "%1;" ::"r"(su32(&empty[s])),
                "h"(static_cast<uint16_t>((1u << CL) - 1))
                : "memory");
        }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     su32(acc_full))
                 : "memory");
} else if (warp >= 2) {
    gemm_epilogue<EPI>(g, tmem, sbias, acc_full, mb, nb, warp, lane);
}
asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
__syncthreads();
if constexpr (CL > 1) cluster_sync();  // no CTA leaves while peers may still signal it
if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kGemmBN) : "memory");
}

// CTA-pair variant (tcgen05 cta_group::2): a cluster of two CTAs computes a
// 256 x 256 tile with one M = 256 UMMA per K-step issued by the leader (rank 0).
// Each CTA stages its own 128 rows of A and its own 128-row half of the weight
// block (16 + 16 KB per K-block instead of 16 + 32 KB), so the bytes each SM
// ingests per flop drop by 1.5x.  Both CTAs' copies are 2-D TMA tensor loads
// with .cta_group::2 whose completion is counted on the LEADER's stage barrier
// (the barrier address with the peer bit cleared); the leader's producer
// expects the pair's bytes.  The leader's MMA commits are multicast to both
// CTAs (stage release, accumulator ready); each CTA's TMEM holds its own 128
// accumulator rows, so the epilogue is unchanged.
constexpr uint32_t kIdesc2 = (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(kGemmBN >> 3) << 17) |
                             (static_cast<uint32_t>((2 * kGemmBM) >> 4) << 24);
constexpr uint32_t kPeerBitMask = 0xFEFFFFFFu;

__device__ __forceinline__ void bar_wait_cluster(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "GWC_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra GWC_%=;\n\t}" ::"r"(su32(b)),
        "r"(parity)
        : "memory");
}
// 16 KB chunk (row coordinate y of a [rows x 2 KB] view of a tiled image) into
// this CTA's smem, completing on the pair leader's barrier.
__device__ __forceinline__ void tma_pair(void* dst, const CUtensorMap* map, int y, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
        "%3}], [%4];" ::"r"(su32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(0), "r"(y), "r"(su32(bar) & kPeerBitMask)
        : "memory");
}

template <int EPI>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm2_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapW, GemmArgs g) {
    extern __shared__ __align__(1024) unsigned char smem[];
    constexpr int kWHalf = kWBytes / 2;                           // 128 weight rows x 64 K
    unsigned char* sA = smem;                                     // kStages x 16 KB
    unsigned char* sW = smem + kStages * kABytes;                 // kStages x 16 KB (this CTA's half)
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * (kABytes + kWBytes));
    uint64_t* empty = full + kStages;
    uint64_t* acc_full = empty + kStages;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(acc_full + 1);
    float* sbias = reinterpret_cast<float*>(smem + kStages * (kABytes + kWBytes) + 128);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int mb = blockIdx.x, nb = blockIdx.y;
    const int KB = pad_to(g.K, kGemmBK) / kGemmBK;
    const uint32_t rank = cluster_rank();

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            bar_init(&full[s], 1);   // leader: its producer's expect_tx arrival (+ both CTAs' bytes)
            bar_init(&empty[s], 1);  // the leader's (multicast) MMA commit
        }
        bar_init(acc_full, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    cluster_sync();
    if (warp == 1) {  // both CTAs: the pair's TMEM (same column base in each)
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(tslot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tslot;
    asm volatile("griddepcontrol.wait;" ::: "memory");

    if (warp == 0 && lane == 0) {  // TMA producer (both CTAs)
        const int ya = mb * KB * (kABytes / 2048);
        const int yw = nb * KB * (kWBytes / 2048) + static_cast<int>(rank) * (kWHalf / 2048);
        for (int kb = 0; kb < KB; ++kb) {
            const int s = kb % kStages;
            if (kb >= kStages) bar_wait(&empty[s], ((kb / kStages) - 1) & 1);
            if (rank == 0) bar_expect(&full[s], 2 * (kABytes + kWHalf));
            tma_pair(sA + s * kABytes, &mapA, ya + kb * (kABytes / 2048), &full[s]);
            tma_pair(sW + s * kWHalf, &mapW, yw + kb * (kWBytes / 2048), &full[s]);
        }
    } else if (warp == 1 && lane == 0 && rank == 0) {  // MMA issuer for the pair
        for (int kb = 0; kb < KB; ++kb) {
            const int s = kb % kStages;
            bar_wait_cluster(&full[s], (kb / kStages) & 1);  // both CTAs' bytes landed
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t a0 = su32(sA + s * kABytes), w0 = su32(sW + s * kWHalf);
#pragma unroll
            for (int k = 0; k < kGemmBK / 16; ++k) {
                const uint32_t acc = (kb > 0 || k > 0) ? 1u : 0u;
                asm volatile(
                    "{\n\t.reg .pred p;\n\t"
                    "setp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                    "l"(sdesc(a0 + 256 * k)), "l"(sdesc(w0 + 256 * k)), "r"(kIdesc2), "r"(acc)
                    : "memory");
            }
            asm volatile(
                "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], "
                "%1;" ::"r"(su32(&empty[s])),
                "h"(static_cast<uint16_t>(3))
                : "memory");
        }
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                su32(acc_full)),
            "h"(static_cast<uint16_t>(3))
            : "memory");
    } else if (warp >= 2) {
        gemm_epilogue<EPI>(g, tmem, sbias, acc_full, mb, nb, warp, lane);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    cluster_sync();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
}

// 2-D tensor map over a tiled image viewed as [bytes / 2 KB] rows of 256 u64:
// one 16 KB box = 8 rows (a 128-row A block or a 128-row weight half-block).
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
bool tile_map(const void* base, size_t bytes, CUtensorMap* m) {
    if (!g_encode) {
        cudaDriverEntryPointQueryResult q;
        void* fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn ||
            q != cudaDriverEntryPointSuccess)
            return false;
        g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    const cuuint64_t dims[2] = {256, static_cast<cuuint64_t>(bytes / 2048)};
    const cuuint64_t strides[1] = {2048};
    const cuuint32_t box[2] = {256, 8}, estr[2] = {1, 1};
    return g_encode(m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, const_cast<void*>(base), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// ---- persistent flow-ODE kernel ------------------------------------------------
// The 3 N_ODE − 1 hidden layers of the ψ ODE (policy.cu enqueue_sample: per step
// k, ψ2: y = tanh(x W2ᵀ + b2); ψ3: x = tanh(y W3ᵀ + b3), Σh += x; ψ1 (k < N−1):
// z += dt x Wmᵀ + qd_k, y = tanh(z), then x ↔ y) in ONE launch: a cluster of
// H/256 CTAs owns a 128-row block, CTA (mb, nb) its 128 × 256 output tile in
// every layer.  A layer's A operand is the whole row block written by the
// cluster in the previous layer's epilogue: each CTA's epilogue, once its tile is
// stored, arrives (DSMEM, release.cluster) on every cluster CTA's layer_ready
// mbarrier; the producer waits on its own before loading the next layer's A
// (weights of the next layer are issued before that wait, into ring stages the
// previous mainloop has freed).  Removes the per-layer launch, CTA setup,
// TMEM allocation and weight-fill cost of separate GEMM launches.  Opt-in
// (MSK_POLICY_ODE=1): measured 1.05 vs 0.875 ms per sample — the cluster-wide
// per-layer dependency and the three epilogue kinds in one register allocation
// (spills) cost more than the per-launch overhead it removes.
struct OdeArgs {
    GemmArgs g2, g3, g1;  // per-layer templates (ψ2, ψ3, ψ1); A / out_a / bias set per layer
    void* buf[2];         // tiled activation images x_k = buf[k % 2], y_k = buf[(k + 1) % 2]
    const float* qd;      // [n_ode - 1 x H] per-step ψ1 bias
    int n_ode, H;
};

__global__ void __launch_bounds__(kGemmThreads, 1) ode_kernel(const OdeArgs o) {
    extern __shared__ __align__(1024) unsigned char smem[];
    unsigned char* sA = smem;
    unsigned char* sW = smem + kStages * kABytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(sW + kStages * kWBytes);
    uint64_t* empty = full + kStages;
    uint64_t* acc_full = empty + kStages;
    uint64_t* ready = acc_full + 1;  // layer_ready: one arrival per cluster CTA per layer
    uint32_t* tslot = reinterpret_cast<uint32_t*>(ready + 1);
    float* sbias = reinterpret_cast<float*>(smem + kStages * (kABytes + kWBytes) + 128);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int mb = blockIdx.x, nb = blockIdx.y, nt = gridDim.y;
    const int KB = pad_to(o.H, kGemmBK) / kGemmBK;
    const int NL = 3 * o.n_ode - 1;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            bar_init(&full[s], 1);
            bar_init(&empty[s], 1);
        }
        bar_init(acc_full, 1);
        bar_init(ready, nt);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    cluster_sync();  // peers' ready barriers exist before any remote arrive
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tslot)),
                     "n"(kGemmBN)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tslot;
    asm volatile("griddepcontrol.wait;" ::: "memory");  // z_0 = tanh(...) of the preceding launch

    if (warp == 0 && lane == 0) {  // producer: the ring runs on across layers
        int gk = 0;
        for (int l = 0; l < NL; ++l) {
            const int k = l / 3, t = l % 3;
            const void* Al = t == 1 ? o.buf[(k + 1) & 1] : o.buf[k & 1];
            const void* Wl = t == 0 ? o.g2.W : (t == 1 ? o.g3.W : o.g1.W);
            const char* A = static_cast<const char*>(Al) + static_cast<size_t>(mb) * KB * kABytes;
            const char* W = static_cast<const char*>(Wl) + static_cast<size_t>(nb) * KB * kWBytes;
            for (int kb = 0; kb < KB; ++kb, ++gk) {
                const int s = gk % kStages;
                if (gk >= kStages) bar_wait(&empty[s], ((gk / kStages) - 1) & 1);
                bar_expect(&full[s], kABytes + kWBytes);
                bulk(sW + s * kWBytes, W + static_cast<size_t>(kb) * kWBytes, kWBytes, &full[s]);
                if (kb == 0 && l > 0) {  // this layer's A: the cluster's previous-layer tiles
                    bar_wait_cluster(ready, (l - 1) & 1);
                    asm volatile("fence.proxy.async.global;" ::: "memory");
                }
                bulk(sA + s * kABytes, A + static_cast<size_t>(kb) * kABytes, kABytes, &full[s]);
            }
        }
    } else if (warp == 1 && lane == 0) {  // MMA issuer
        int gk = 0;
        for (int l = 0; l < NL; ++l) {
            for (int kb = 0; kb < KB; ++kb, ++gk) {
                const int s = gk % kStages;
                bar_wait(&full[s], (gk / kStages) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t a0 = su32(sA + s * kABytes), w0 = su32(sW + s * kWBytes);
#pragma unroll
                for (int k = 0; k < kGemmBK / 16; ++k) {
                    const uint32_t acc = (kb > 0 || k > 0) ? 1u : 0u;
                    asm volatile(
                        "{\n\t.reg .pred p;\n\t"
                        "setp.ne.b32 p, %4, 0;\n\t"
                        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                        "l"(sdesc(a0 + 256 * k)), "l"(sdesc(w0 + 256 * k)), "r"(kIdesc), "r"(acc)
                        : "memory");
                }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                 su32(&empty[s]))
                             : "memory");
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                             su32(acc_full))
                         : "memory");
            // the accumulator is reused: wait until every cluster CTA finished this layer's epilogue
            // (this CTA's included) before the next layer's MMAs overwrite it
            if (l + 1 < NL) bar_wait_cluster(ready, l & 1);
        }
    } else if (warp >= 2) {
        for (int l = 0; l < NL; ++l) {
            const int k = l / 3, t = l % 3;
            const uint32_t par = l & 1;
            // the layer's epilogue on the kernel-parameter templates (no local copies)
            if (t == 0)
                gemm_epilogue<kEpiTanhTiled>(o.g2, tmem, sbias, acc_full, mb, nb, warp, lane, par,
                                            o.buf[(k + 1) & 1], nullptr);
            else if (t == 1)
                gemm_epilogue<kEpiTanhAcc>(o.g3, tmem, sbias, acc_full, mb, nb, warp, lane, par, o.buf[k & 1],
                                          nullptr);
            else
                gemm_epilogue<kEpiTanhPre>(o.g1, tmem, sbias, acc_full, mb, nb, warp, lane, par,
                                          o.buf[(k + 1) & 1], o.qd + static_cast<size_t>(k) * o.H);
            // tile stored: make it visible to the peers' bulk copies, then signal every cluster CTA
            asm volatile("fence.proxy.async.global;" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");
            if (threadIdx.x == 64) {
                asm volatile("fence.acq_rel.cluster;" ::: "memory");
                for (int c = 0; c < nt; ++c) {
                    uint32_t remote;
                    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(su32(ready)), "r"(c));
                    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote)
                                 : "memory");
                }
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    cluster_sync();  // no CTA leaves while peers may still signal it
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kGemmBN) : "memory");
}

__global__ void obs_to_tiled_kernel(const float* obs, int M, int D, int ld, const float* mean, const float* inv_sd,
                                    void* out, int f4) {
    // one thread per (row, 8-column chunk) of the padded [Mpad x Kpad] image
    const int Kp = pad_to(D, kGemmBK), chunks = Kp / 8;
    const long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    const int Mp = pad_to(M, kGemmBM);
    if (t >= static_cast<long long>(Mp) * chunks) return;
    const int m = static_cast<int>(t / chunks), k0 = static_cast<int>(t % chunks) * 8;
    float y[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int k = k0 + i;
        float x = 0.0f;
        if (m < M && k < D) {
            x = f4 > 0 ? obs[(static_cast<size_t>(k >> 2) * f4 + m) * 4 + (k & 3)] : obs[static_cast<size_t>(m) * ld + k];
            if (mean) x = (x - mean[k]) * inv_sd[k];
        }
        y[i] = x;
    }
    char* base = static_cast<char*>(out) + (static_cast<size_t>(m >> 7) * (Kp / kGemmBK) + (k0 >> 6)) * kABytes;
    *reinterpret_cast<uint4*>(base + blk_off(m & 127, k0 & 63)) =
        make_uint4(bf2(y[0], y[1]), bf2(y[2], y[3]), bf2(y[4], y[5]), bf2(y[6], y[7]));
}

}  // namespace

std::vector<uint16_t> pack_weights(const double* W, int rows, int cols, int c0, int nc) {
    const int Np = pad_to(rows, kGemmBN), Kp = pad_to(nc, kGemmBK), KB = Kp / kGemmBK;
    std::vector<uint16_t> img(static_cast<size_t>(Np) * Kp, 0);
    for (int n = 0; n < rows; ++n)
        for (int k = 0; k < nc; ++k) {
            const __nv_bfloat16 b = __float2bfloat16_rn(static_cast<float>(W[static_cast<size_t>(c0 + k) * rows + n]));
            uint16_t u;
            std::memcpy(&u, &b, 2);
            const size_t blk = static_cast<size_t>(n / kGemmBN) * KB + k / kGemmBK;
            img[(blk * kWBytes + blk_off(n % kGemmBN, k % kGemmBK)) / 2] = u;
        }
    return img;
}

size_t gemm_smem_bytes() { return static_cast<size_t>(kStages) * (kABytes + kWBytes) + 128 + kGemmBN * 4; }

namespace {
template <int EPI>
cudaError_t prepare_epi(int bytes) {
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(gemm2_kernel<EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes))) return e;
    if ((e = cudaFuncSetAttribute(gemm_kernel<EPI, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes))) return e;
    if ((e = cudaFuncSetAttribute(gemm_kernel<EPI, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes))) return e;
    return cudaFuncSetAttribute(gemm_kernel<EPI, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}
template <int EPI>
cudaError_t launch_epi(cudaLaunchConfig_t& cfg, int cl, const GemmArgs& g, const CUtensorMap* maps) {
    if (cl == -2) return cudaLaunchKernelEx(&cfg, gemm2_kernel<EPI>, maps[0], maps[1], g);
    switch (cl) {
        case 4: return cudaLaunchKernelEx(&cfg, gemm_kernel<EPI, 4>, g);
        case 2: return cudaLaunchKernelEx(&cfg, gemm_kernel<EPI, 2>, g);
        default: return cudaLaunchKernelEx(&cfg, gemm_kernel<EPI, 1>, g);
    }
}
}  // namespace

cudaError_t prepare_gemm() {
    cudaError_t e;
    const int bytes = static_cast<int>(gemm_smem_bytes());
    if ((e = prepare_epi<kEpiTanhTiled>(bytes))) return e;
    if ((e = prepare_epi<kEpiF32>(bytes))) return e;
    if ((e = prepare_epi<kEpiTanhPre>(bytes))) return e;
    if ((e = prepare_epi<kEpiTanhAcc>(bytes))) return e;
    return prepare_epi<kEpiOde>(bytes);
}

// Weight-multicast cluster size for a grid with `mt` row tiles (MSK_GEMM_CLUSTER overrides).
static int gemm_cluster(int mt) {
    static const int forced = [] {
        const char* v = std::getenv("MSK_GEMM_CLUSTER");
        return v ? std::atoi(v) : 0;
    }();
    if (forced == 2 || forced == 4) return mt % forced == 0 ? forced : 1;
    return 1;  // measured: weight multicast saves L2 traffic but no time at these sizes
}

cudaError_t launch_gemm(const GemmArgs& g, int epi, cudaStream_t s) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(pad_to(g.M, kGemmBM) / kGemmBM, pad_to(g.N, kGemmBN) / kGemmBN);
    cfg.blockDim = dim3(kGemmThreads);
    cfg.dynamicSmemBytes = gemm_smem_bytes();
    cfg.stream = s;
    // MSK_GEMM_2CTA: CTA pairs (cta_group::2, needs an even number of row tiles).  Opt-in:
    // measured 14.2 vs 13.4 us per K = 1024 layer at 4096 rows — halving the bytes each SM
    // ingests does not pay, the layer is bound by fill / epilogue, not operand ingest.
    static const bool pair = std::getenv("MSK_GEMM_2CTA") != nullptr;
    CUtensorMap maps[2];
    bool use2 = pair && cfg.gridDim.x % 2 == 0;
    if (use2)
        use2 = tile_map(g.A, tiled_a_bytes(g.M, g.K), &maps[0]) && tile_map(g.W, tiled_w_bytes(g.N, g.K), &maps[1]);
    const int cl = use2 ? 2 : gemm_cluster(static_cast<int>(cfg.gridDim.x));
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = cl;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    const int sel = use2 ? -2 : cl;
    switch (epi) {
        case kEpiTanhTiled: return launch_epi<kEpiTanhTiled>(cfg, sel, g, maps);
        case kEpiF32: return launch_epi<kEpiF32>(cfg, sel, g, maps);
        case kEpiTanhPre: return launch_epi<kEpiTanhPre>(cfg, sel, g, maps);
        case kEpiTanhAcc: return launch_epi<kEpiTanhAcc>(cfg, sel, g, maps);
        default: return launch_epi<kEpiOde>(cfg, sel, g, maps);
    }
}

cudaError_t launch_ode(const GemmArgs& g2, const GemmArgs& g3, const GemmArgs& g1, void* x0, void* y0,
                       const float* qd, int n_ode, int H, cudaStream_t s) {
    static bool prepared = false;
    if (!prepared) {
        cudaError_t e = cudaFuncSetAttribute(ode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(gemm_smem_bytes()));
        if (e) return e;
        prepared = true;
    }
    OdeArgs o;
    o.g2 = g2;
    o.g3 = g3;
    o.g1 = g1;
    o.buf[0] = x0;
    o.buf[1] = y0;
    o.qd = qd;
    o.n_ode = n_ode;
    o.H = H;
    cudaLaunchConfig_t cfg{};
    const int nt = pad_to(H, kGemmBN) / kGemmBN;
    cfg.gridDim = dim3(pad_to(g2.M, kGemmBM) / kGemmBM, nt);
    cfg.blockDim = dim3(kGemmThreads);
    cfg.dynamicSmemBytes = gemm_smem_bytes();
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = 1;
    attr[1].val.clusterDim.y = nt;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    return cudaLaunchKernelEx(&cfg, ode_kernel, o);
}

cudaError_t launch_obs_to_tiled(const float* obs, int M, int D, const float* mean, const float* inv_sd, void* out,
                                cudaStream_t s) {
    const long long n = static_cast<long long>(pad_to(M, kGemmBM)) * (pad_to(D, kGemmBK) / 8);
    obs_to_tiled_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(obs, M, D, D, mean, inv_sd, out, 0);
    return cudaGetLastError();
}

cudaError_t launch_f32_to_tiled(const float* x, int M, int D, int ld, void* out, cudaStream_t s, int f4_rows) {
    const long long n = static_cast<long long>(pad_to(M, kGemmBM)) * (pad_to(D, kGemmBK) / 8);
    obs_to_tiled_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(x, M, D, ld, nullptr, nullptr, out,
                                                                               f4_rows);
    return cudaGetLastError();
}

}  // namespace msk_b200
