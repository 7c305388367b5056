// Discriminator tracking reward on the 5th-generation tensor cores (sm_100a).
//
// r = -log(1 - clamp(D(Δ), 1e-4, 1 - 1e-4)),  D = sigmoid(MLP: Δ -> 3 x tanh(H) -> 1)
// (reward_from_discriminator; Mlp::forward with Head::Sigmoid,
// nn.cpp:54-73; parameters in the Mlp flat layout of nn.cpp:16-38).  In
// Env::step(action, fn) the reward is fn(Δ) + reward_aux for a non-diverged
// step (env.cpp:265-270); that is what the fused mode writes.
//
// One CTA per 128-row tile of Δ, 128 threads (4 warps), one tile resident per SM:
//   * weights are pre-laid-out on the host as bf16 K-major "core matrix" images
//     (8 rows x 16 B atoms, SWIZZLE_NONE) and staged global -> smem with 1-D TMA
//     bulk copies (cp.async.bulk + mbarrier complete_tx);
//   * each hidden layer is ONE chain of tcgen05.mma.kind::f16 (M = 128, N = H,
//     K = 16 per instruction) issued by a single thread, accumulating in TMEM
//     (H fp32 columns x 128 lanes);
//   * the epilogue (warp w owns TMEM lanes 32w..32w+31 = rows) loads the
//     accumulator with tcgen05.ld, adds the bias, applies tanh in fp32 and
//     writes bf16 back to smem as the next layer's A operand; the head (N = 1)
//     is an fp32 dot product in registers, then sigmoid / clamp / log.
// Launched right after the step kernel with programmatic dependent launch, so
// the TMEM allocation and the first weight copy overlap the step's tail.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <vector>

#include "disc.hpp"

namespace msk_b200 {

namespace {

constexpr int kTileM = 128;
constexpr int kThreads = 128;
constexpr uint8_t kFlagDiverged = 4, kFlagSkip = 8 | 16;  // NOT_STEPPED | BAD_ACTION: untouched

// byte offset of element (r, k) in a K-major SWIZZLE_NONE core-matrix image
// with K columns: 8-row groups at SBO = (K/8)*128 B, 8-element K chunks at 128 B
__host__ __device__ constexpr uint32_t img_off(int r, int k, int K) {
    return static_cast<uint32_t>(((r >> 3) * (K >> 3) + (k >> 3)) * 128 + (r & 7) * 16 + (k & 7) * 2);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// tcgen05 shared-memory matrix descriptor (K-major, no swizzle): start address,
// leading byte offset (K-chunk stride), stride byte offset (8-row-group stride),
// version 1 (bits 46-47), layout type 0 (bits 61-63).
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return static_cast<uint64_t>((addr >> 4) & 0x3FFF) | (static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16) |
           (static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

// kind::f16 instruction descriptor: D f32, A/B bf16, both K-major, M = 128, N = n.
__device__ __forceinline__ uint32_t instr_desc(int n) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(n >> 3) << 17) |
           (static_cast<uint32_t>(kTileM >> 4) << 24);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// 1-D TMA bulk copy global -> shared, completion counted on the mbarrier.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// Stage `bytes` (multiple of 16) of a weight image; one thread.
__device__ __forceinline__ void stage_weights(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    mbar_expect_tx(bar, bytes);
    constexpr uint32_t kPiece = 32768;
    for (uint32_t o = 0; o < bytes; o += kPiece)
        bulk_g2s(static_cast<char*>(dst) + o, static_cast<const char*>(src) + o, (bytes - o < kPiece ? bytes - o : kPiece), bar);
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void proxy_fence() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// One layer: D[tmem] = A[128 x K] * W[N x K]^T, K/16 MMAs from one thread, then
// a commit that arrives on `bar` when they (and their smem reads) are done.
__device__ __forceinline__ void mma_layer(uint32_t tmem, const void* sa, const void* sw, int K, int N, uint64_t* bar) {
    const uint32_t a0 = smem_u32(sa), w0 = smem_u32(sw), sbo = static_cast<uint32_t>(K >> 3) * 128;
    const uint32_t idesc = instr_desc(N);
    for (int s = 0; s < K / 16; ++s) {
        const uint64_t da = smem_desc(a0 + 256 * s, 128, sbo), dw = smem_desc(w0 + 256 * s, 128, sbo);
        const uint32_t acc = s > 0;
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "setp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
            "l"(da), "l"(dw), "r"(idesc), "r"(acc)
            : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

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

__device__ __forceinline__ float tanh_fast(float x) {
    float y;
    asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
    const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<const uint32_t*>(&h);
}

// Hidden-layer epilogue: row r's H accumulators -> tanh(acc + b) -> bf16 into the
// next layer's A image (K = H).
__device__ __forceinline__ void epilogue_hidden(uint32_t tmem_row, const float* bias, char* sa, int r, int H) {
    for (int c = 0; c < H; c += 16) {
        float v[16];
        tmem_ld16(tmem_row + c, v);
        uint32_t p[8];
#pragma unroll
        for (int i = 0; i < 8; ++i)
            p[i] = pack_bf16(tanh_fast(v[2 * i] + bias[c + 2 * i]), tanh_fast(v[2 * i + 1] + bias[c + 2 * i + 1]));
        *reinterpret_cast<uint4*>(sa + img_off(r, c, H)) = make_uint4(p[0], p[1], p[2], p[3]);
        *reinterpret_cast<uint4*>(sa + img_off(r, c + 8, H)) = make_uint4(p[4], p[5], p[6], p[7]);
    }
}

__global__ void __launch_bounds__(kThreads, 1)
    disc_reward_kernel(DiscDev P, const float* __restrict__ delta, int ld, int n, const float* __restrict__ raux,
                       const uint8_t* __restrict__ flags, float* __restrict__ reward) {
    extern __shared__ __align__(1024) unsigned char smem[];
    const int H = P.hidden, K1 = P.k1, Kmax = K1 > H ? K1 : H;
    char* sa = reinterpret_cast<char*>(smem);                                      // 128 x Kmax bf16
    char* sw = sa + kTileM * Kmax * 2;                                             // H x Kmax bf16
    float* sb = reinterpret_cast<float*>(sw + static_cast<size_t>(H) * Kmax * 2);  // b1 b2 b3 w4
    uint64_t* bars = reinterpret_cast<uint64_t*>(sb + 4 * H);                      // [0] weights, [1] mma
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int row0 = blockIdx.x * kTileM;

    if (tid == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {  // TMEM: H fp32 columns (power of two >= 32)
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(P.tmem_cols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    for (int i = tid; i < 4 * H; i += kThreads) sb[i] = P.bias[i];
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    if (tid == 0) stage_weights(sw, P.w1, static_cast<uint32_t>(H) * K1 * 2, &bars[0]);

    // Δ is the previous kernel's output: wait for it (programmatic dependent launch)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    for (int i = tid; i < kTileM * K1; i += kThreads) {
        const int r = i / K1, k = i - r * K1, row = row0 + r;
        const float x = (row < n && k < P.din) ? delta[static_cast<size_t>(row) * ld + k] : 0.0f;
        *reinterpret_cast<__nv_bfloat16*>(sa + img_off(r, k, K1)) = __float2bfloat16_rn(x);
    }
    proxy_fence();
    __syncthreads();

    const int r = warp * 32 + lane;                          // this thread's row of the tile
    const uint32_t trow = tmem + (static_cast<uint32_t>(warp * 32) << 16);  // TMEM lane base of this warp
    uint32_t wphase = 0, mphase = 0;
    for (int layer = 0; layer < 3; ++layer) {
        const int K = layer == 0 ? K1 : H;
        if (tid == 0) {
            mbar_wait(&bars[0], wphase);
            tc_fence_after();
            mma_layer(tmem, sa, sw, K, H, &bars[1]);
        }
        wphase ^= 1;
        mbar_wait(&bars[1], mphase);
        mphase ^= 1;
        tc_fence_after();
        if (layer < 2) {
            if (tid == 0) stage_weights(sw, layer == 0 ? P.w2 : P.w3, static_cast<uint32_t>(H) * H * 2, &bars[0]);
            epilogue_hidden(trow, sb + layer * H, sa, r, H);
            proxy_fence();
            tc_fence_before();
            __syncthreads();
            tc_fence_after();
        }
    }
    // head: z = w4 . tanh(acc3 + b3) + b4 (fp32), D = sigmoid(z)
    float z = 0.0f;
    for (int c = 0; c < H; c += 16) {
        float v[16];
        tmem_ld16(trow + c, v);
#pragma unroll
        for (int i = 0; i < 16; ++i) z = fmaf(tanh_fast(v[i] + sb[2 * H + c + i]), sb[3 * H + c + i], z);
    }
    z += __ldg(P.bias + 4 * H);  // b4
    const int row = row0 + r;
    if (row < n) {
        float d = 1.0f / (1.0f + __expf(-z));
        d = fminf(fmaxf(d, 1e-4f), 1.0f - 1e-4f);
        const float rw = -log1pf(-d);
        if (!flags) {
            reward[row] = rw;
        } else {
            const uint8_t f = flags[row];
            if (!(f & kFlagSkip)) reward[row] = (f & kFlagDiverged) ? 0.0f : rw + (raux ? raux[row] : 0.0f);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(P.tmem_cols)
                     : "memory");
}

// ---------------------------------------------------------------------------
// fp32-class mode (split bf16): every operand x = hi + lo with hi = bf16(x),
// lo = bf16(x - hi) (16 significant bits), and each product A W^T is formed
// as A_hi W_hi + A_hi W_lo + A_lo W_hi on the tensor cores with fp32
// accumulation in TMEM (the dropped A_lo W_lo term and the residual of the
// split are ~2^-16 relative); tanh / exp / log are the accurate fp32 ones.
// The activations (A hi / lo, 128 x K) stay in shared memory; the weights are
// streamed in K16 chunks (hi + lo, N x 16 each) through a 4-stage TMA ring, one
// thread issuing the bulk copies and the MMAs (3 per chunk, commit per chunk
// frees its stage).
// ---------------------------------------------------------------------------
constexpr int kRing = 4;

// element (r, kk) of a K16 chunk image (N rows x 16 K): two 8-K core-matrix columns
__host__ __device__ constexpr uint32_t chunk_off(int r, int kk) {
    return static_cast<uint32_t>(((r >> 3) * 2 + (kk >> 3)) * 128 + (r & 7) * 16 + (kk & 7) * 2);
}

__device__ __forceinline__ void mma_f16(uint32_t tmem, uint64_t da, uint64_t dw, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
        "l"(da), "l"(dw), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void split_bf16(float x, __nv_bfloat16& hi, __nv_bfloat16& lo) {
    hi = __float2bfloat16_rn(x);
    lo = __float2bfloat16_rn(x - __bfloat162float(hi));
}

constexpr int kThreadsP = 256;  // precise kernel: two warps per TMEM lane quarter (column halves)

__global__ void __launch_bounds__(kThreadsP, 1)
    disc_reward_precise_kernel(DiscDev P, const float* __restrict__ delta, int ld, int n, const float* __restrict__ raux,
                               const uint8_t* __restrict__ flags, float* __restrict__ reward) {
    extern __shared__ __align__(1024) unsigned char smem[];
    const int H = P.hidden, K1 = P.k1, Kmax = K1 > H ? K1 : H;
    const uint32_t chunk_bytes = static_cast<uint32_t>(H) * 32;   // N x 16 bf16
    char* sa_hi = reinterpret_cast<char*>(smem);                     // 128 x Kmax bf16
    char* sa_lo = sa_hi + kTileM * Kmax * 2;
    char* ring = sa_lo + kTileM * Kmax * 2;                          // kRing x (hi | lo) chunks
    float* sb = reinterpret_cast<float*>(ring + kRing * 2 * chunk_bytes);  // b1 b2 b3 w4
    uint64_t* full = reinterpret_cast<uint64_t*>(sb + 4 * H);      // [kRing]
    uint64_t* empty = full + kRing;                                  // [kRing]
    uint64_t* done = empty + kRing;                                  // [1] layer's MMAs complete
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int row0 = blockIdx.x * kTileM;

    if (tid == 0) {
        for (int i = 0; i < kRing; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        mbar_init(done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(P.tmem_cols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    for (int i = tid; i < 4 * H; i += kThreadsP) sb[i] = P.bias[i];
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    // ring bookkeeping (thread 0 only): chunks consumed from each stage so far.  A
    // stage's n-th load completes full[] phase n and its n-th commit empty[] phase
    // n; a stage is refilled only after its last commit, so no phase is skipped.
    uint32_t uses[kRing] = {0, 0, 0, 0};
    auto load_chunk = [&](int layer, int c, int st) {
        mbar_expect_tx(&full[st], 2 * chunk_bytes);
        bulk_g2s(ring + (2 * st) * chunk_bytes, static_cast<const char*>(P.c_hi[layer]) + c * chunk_bytes, chunk_bytes,
                 &full[st]);
        bulk_g2s(ring + (2 * st + 1) * chunk_bytes, static_cast<const char*>(P.c_lo[layer]) + c * chunk_bytes,
                 chunk_bytes, &full[st]);
    };
    if (tid == 0)  // the first layer's leading chunks do not depend on Δ
        for (int c = 0; c < kRing && c < K1 / 16; ++c) load_chunk(0, c, c);

    asm volatile("griddepcontrol.wait;" ::: "memory");  // Δ = the previous kernel's output
    for (int i = tid; i < kTileM * K1; i += kThreadsP) {
        const int r = i / K1, k = i - r * K1, row = row0 + r;
        const float x = (row < n && k < P.din) ? delta[static_cast<size_t>(row) * ld + k] : 0.0f;
        __nv_bfloat16 hi, lo;
        split_bf16(x, hi, lo);
        *reinterpret_cast<__nv_bfloat16*>(sa_hi + img_off(r, k, K1)) = hi;
        *reinterpret_cast<__nv_bfloat16*>(sa_lo + img_off(r, k, K1)) = lo;
    }
    proxy_fence();
    __syncthreads();

    // epilogue: warp w reads TMEM lane quarter w % 4 (rows), column half w / 4
    const int q = warp & 3, half = warp >> 2, r = q * 32 + lane;
    const bool split = H % 32 == 0;  // halves of whole 16-column TMEM loads; else warps 0-3 take all columns
    const int c_lo = split ? half * (H / 2) : (half ? H : 0), c_hi = split ? c_lo + H / 2 : H;
    const uint32_t trow = tmem + (static_cast<uint32_t>(q * 32) << 16);
    float* sdot = reinterpret_cast<float*>(tmem_slot + 4);  // [2][128] head partial dot products
    const uint32_t idesc = instr_desc(H);
    uint32_t done_phase = 0;
    for (int layer = 0; layer < 3; ++layer) {
        const int K = layer == 0 ? K1 : H, nch = K / 16;
        if (tid == 0) {
            if (layer > 0)  // stages are free (the previous layer's MMAs completed)
                for (int c = 0; c < kRing && c < nch; ++c) load_chunk(layer, c, c);
            const uint32_t a_hi = smem_u32(sa_hi), a_lo = smem_u32(sa_lo), sbo = static_cast<uint32_t>(K >> 3) * 128;
            for (int c = 0; c < nch; ++c) {
                const int st = c % kRing;
                mbar_wait(&full[st], uses[st] & 1);
                ++uses[st];
                tc_fence_after();
                const uint32_t w_hi = smem_u32(ring + (2 * st) * chunk_bytes), w_lo = w_hi + chunk_bytes;
                const uint64_t dah = smem_desc(a_hi + 256 * c, 128, sbo), dal = smem_desc(a_lo + 256 * c, 128, sbo);
                const uint64_t dwh = smem_desc(w_hi, 128, 256), dwl = smem_desc(w_lo, 128, 256);
                mma_f16(tmem, dal, dwh, idesc, c > 0);  // small terms first
                mma_f16(tmem, dah, dwl, idesc, 1);
                mma_f16(tmem, dah, dwh, idesc, 1);
                mma_commit(&empty[st]);
                // refill the previous chunk's stage once its MMAs are done (this
                // chunk's MMAs are already queued behind them)
                if (c > 0 && c - 1 + kRing < nch) {
                    const int sp = (c - 1) % kRing;
                    mbar_wait(&empty[sp], (uses[sp] - 1) & 1);
                    load_chunk(layer, c - 1 + kRing, sp);
                }
            }
            mma_commit(done);
        }
        mbar_wait(done, done_phase);
        done_phase ^= 1;
        tc_fence_after();
        if (layer < 2) {
            for (int c = c_lo; c < c_hi; c += 16) {  // tanh(acc + b) -> split bf16 A for the next layer (K = H)
                float v[16];
                tmem_ld16(trow + c, v);
#pragma unroll
                for (int j = 0; j < 16; j += 8) {  // 8 columns = one 16-B core-matrix row per plane
                    uint32_t hw[4], lw[4];
#pragma unroll
                    for (int i = 0; i < 8; i += 2) {
                        __nv_bfloat16 h0, l0, h1, l1;
                        split_bf16(tanhf(v[j + i] + sb[layer * H + c + j + i]), h0, l0);
                        split_bf16(tanhf(v[j + i + 1] + sb[layer * H + c + j + i + 1]), h1, l1);
                        hw[i / 2] = static_cast<uint32_t>(__bfloat16_as_ushort(h0)) |
                                    (static_cast<uint32_t>(__bfloat16_as_ushort(h1)) << 16);
                        lw[i / 2] = static_cast<uint32_t>(__bfloat16_as_ushort(l0)) |
                                    (static_cast<uint32_t>(__bfloat16_as_ushort(l1)) << 16);
                    }
                    *reinterpret_cast<uint4*>(sa_hi + img_off(r, c + j, H)) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
                    *reinterpret_cast<uint4*>(sa_lo + img_off(r, c + j, H)) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
                }
            }
            proxy_fence();
            tc_fence_before();
            __syncthreads();
            tc_fence_after();
        }
    }
    float z = 0.0f;
    for (int c = c_lo; c < c_hi; c += 16) {
        float v[16];
        tmem_ld16(trow + c, v);
#pragma unroll
        for (int i = 0; i < 16; ++i) z = fmaf(tanhf(v[i] + sb[2 * H + c + i]), sb[3 * H + c + i], z);
    }
    sdot[half * kTileM + r] = z;
    __syncthreads();
    if (half == 0) z = (sdot[r] + sdot[kTileM + r]) + __ldg(P.bias + 4 * H);
    const int row = row0 + r;
    if (half == 0 && row < n) {
        float d = 1.0f / (1.0f + expf(-z));
        d = fminf(fmaxf(d, 1e-4f), 1.0f - 1e-4f);
        const float rw = -log1pf(-d);
        if (!flags) {
            reward[row] = rw;
        } else {
            const uint8_t f = flags[row];
            if (!(f & kFlagSkip)) reward[row] = (f & kFlagDiverged) ? 0.0f : rw + (raux ? raux[row] : 0.0f);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(P.tmem_cols)
                     : "memory");
}

}  // namespace

size_t disc_smem_bytes(const DiscDev& P) {
    const int Kmax = std::max(P.k1, P.hidden);
    if (P.precise)  // A hi + lo, the weight ring, biases, barriers
        return 2 * static_cast<size_t>(kTileM) * Kmax * 2 + static_cast<size_t>(kRing) * 2 * P.hidden * 32 +
               16 * P.hidden + 128 + 2 * kTileM * 4;
    return static_cast<size_t>(kTileM) * Kmax * 2 + static_cast<size_t>(P.hidden) * Kmax * 2 + 16 * P.hidden + 64;
}

// Host: Mlp flat parameters (f64, nn.cpp layout) -> device images.
DiscHost build_disc_images(const double* theta, long long n_params, int din, int hidden) {
    if (hidden < 16 || hidden > 256 || hidden % 16 != 0)
        throw std::invalid_argument("discriminator hidden width must be a multiple of 16 in [16, 256]");
    if (din < 1 || din > 256) throw std::invalid_argument("discriminator input width out of range");
    const int H = hidden, K1 = (din + 15) / 16 * 16;
    const long long expect = static_cast<long long>(H) * din + H + 2LL * (H * H + H) + H + 1;
    if (n_params != expect)
        throw std::invalid_argument("discriminator parameter count " + std::to_string(n_params) + " != " +
                                    std::to_string(expect) + " for Mlp(in=" + std::to_string(din) +
                                    ", hidden=" + std::to_string(H) + ", out=1)");
    DiscHost h;
    h.din = din;
    h.hidden = H;
    h.k1 = K1;
    auto image = [&](const double* W, int rows, int cols, int K) {  // W column-major rows x cols
        std::vector<uint16_t> img(static_cast<size_t>(rows) * K, 0);
        for (int r = 0; r < rows; ++r)
            for (int k = 0; k < cols; ++k) {
                const __nv_bfloat16 b = __float2bfloat16_rn(static_cast<float>(W[static_cast<size_t>(k) * rows + r]));
                uint16_t u;
                std::memcpy(&u, &b, 2);
                img[img_off(r, k, K) / 2] = u;
            }
        return img;
    };
    // split-bf16 chunked images: chunk c of a K-column image = rows x 16 K (chunk_off)
    auto chunked = [&](const double* W, int rows, int cols, int K, std::vector<uint16_t>& hi,
                       std::vector<uint16_t>& lo) {
        hi.assign(static_cast<size_t>(rows) * K, 0);
        lo.assign(static_cast<size_t>(rows) * K, 0);
        for (int r = 0; r < rows; ++r)
            for (int k = 0; k < cols; ++k) {
                const float x = static_cast<float>(W[static_cast<size_t>(k) * rows + r]);
                const __nv_bfloat16 bh = __float2bfloat16_rn(x);
                const __nv_bfloat16 bl = __float2bfloat16_rn(x - __bfloat162float(bh));
                const size_t at = (static_cast<size_t>(k >> 4) * rows * 16 * 2 + chunk_off(r, k & 15)) / 2;
                std::memcpy(&hi[at], &bh, 2);
                std::memcpy(&lo[at], &bl, 2);
            }
    };
    long long o = 0;
    chunked(theta + o, H, din, K1, h.c1_hi, h.c1_lo);
    h.w1 = image(theta + o, H, din, K1);
    o += static_cast<long long>(H) * din;
    const double* b1 = theta + o;
    o += H;
    chunked(theta + o, H, H, H, h.c2_hi, h.c2_lo);
    h.w2 = image(theta + o, H, H, H);
    o += static_cast<long long>(H) * H;
    const double* b2 = theta + o;
    o += H;
    chunked(theta + o, H, H, H, h.c3_hi, h.c3_lo);
    h.w3 = image(theta + o, H, H, H);
    o += static_cast<long long>(H) * H;
    const double* b3 = theta + o;
    o += H;
    const double* w4 = theta + o;  // 1 x H
    o += H;
    h.bias.resize(4 * static_cast<size_t>(H) + 1);
    h.bias[4 * static_cast<size_t>(H)] = static_cast<float>(theta[o]);  // b4
    for (int i = 0; i < H; ++i) {
        h.bias[i] = static_cast<float>(b1[i]);
        h.bias[H + i] = static_cast<float>(b2[i]);
        h.bias[2 * H + i] = static_cast<float>(b3[i]);
        h.bias[3 * H + i] = static_cast<float>(w4[i]);
    }
    return h;
}

cudaError_t prepare_disc(const DiscDev& P) {
    DiscDev q = P;
    q.precise = 0;
    cudaError_t e = cudaFuncSetAttribute(disc_reward_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(disc_smem_bytes(q)));
    if (e != cudaSuccess) return e;
    q.precise = 1;
    return cudaFuncSetAttribute(disc_reward_precise_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(disc_smem_bytes(q)));
}

cudaError_t launch_disc(const DiscDev& P, const float* delta, int ld, int n, const float* raux,
                        const uint8_t* flags, float* reward, cudaStream_t s, bool pdl) {
    if (n <= 0) return cudaSuccess;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((n + kTileM - 1) / kTileM);
    cfg.blockDim = dim3(P.precise ? kThreadsP : kThreads);
    cfg.dynamicSmemBytes = disc_smem_bytes(P);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    if (P.precise) return cudaLaunchKernelEx(&cfg, disc_reward_precise_kernel, P, delta, ld, n, raux, flags, reward);
    return cudaLaunchKernelEx(&cfg, disc_reward_kernel, P, delta, ld, n, raux, flags, reward);
}

// Device-side refresh of the images from f64 parameters (same layout as
// build_disc_images): used when the discriminator is trained on the device.
// One weight element into both image sets: the bf16 core-matrix image (fast
// mode) and the split hi / lo K16-chunk images (fp32-class mode).
__device__ __forceinline__ void put_weight(const DiscDev& P, int layer, int r, int k, int K, int rows, double v) {
    const float x = static_cast<float>(v);
    char* fast = reinterpret_cast<char*>(const_cast<void*>(layer == 0 ? P.w1 : layer == 1 ? P.w2 : P.w3));
    *reinterpret_cast<__nv_bfloat16*>(fast + img_off(r, k, K)) = __float2bfloat16_rn(x);
    const __nv_bfloat16 hi = __float2bfloat16_rn(x), lo = __float2bfloat16_rn(x - __bfloat162float(hi));
    const size_t at = static_cast<size_t>(k >> 4) * rows * 32 + chunk_off(r, k & 15);
    *reinterpret_cast<__nv_bfloat16*>(static_cast<char*>(const_cast<void*>(P.c_hi[layer])) + at) = hi;
    *reinterpret_cast<__nv_bfloat16*>(static_cast<char*>(const_cast<void*>(P.c_lo[layer])) + at) = lo;
}

__global__ void disc_repack_kernel(const double* __restrict__ theta, DiscDev P) {
    const int din = P.din, H = P.hidden, K1 = P.k1;
    float* bias = const_cast<float*>(P.bias);
    const long long o1 = static_cast<long long>(H) * din + H, o2 = o1 + static_cast<long long>(H) * H + H,
                    o3 = o2 + static_cast<long long>(H) * H + H;
    const long long n1 = static_cast<long long>(H) * K1, n2 = static_cast<long long>(H) * H;
    for (long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; t < n1 + 2 * n2 + 4 * H + 1;
         t += static_cast<long long>(gridDim.x) * blockDim.x) {
        if (t < n1) {  // W1 (H x din, zero-padded to K1)
            const int r = static_cast<int>(t % H), k = static_cast<int>(t / H);
            const double v = k < din ? theta[static_cast<long long>(k) * H + r] : 0.0;
            put_weight(P, 0, r, k, K1, H, v);
        } else if (t < n1 + 2 * n2) {  // W2, W3 (H x H)
            const long long u = t - n1;
            const int which = static_cast<int>(u / n2);
            const long long e = u % n2;
            const int r = static_cast<int>(e % H), k = static_cast<int>(e / H);
            const double v = theta[(which ? o2 : o1) + static_cast<long long>(k) * H + r];
            put_weight(P, 1 + which, r, k, H, H, v);
        } else {  // b1 | b2 | b3 | w4 | b4
            const int i = static_cast<int>(t - n1 - 2 * n2), part = i / H, c = i % H;
            const long long src = part == 0 ? static_cast<long long>(H) * din + c
                                  : part == 1 ? o1 + static_cast<long long>(H) * H + c
                                  : part == 2 ? o2 + static_cast<long long>(H) * H + c
                                  : part == 3 ? o3 + c
                                              : o3 + H;
            bias[i] = static_cast<float>(theta[src]);
        }
    }
}

cudaError_t launch_disc_repack(const double* theta, const DiscDev& P, cudaStream_t s) {
    disc_repack_kernel<<<296, 256, 0, s>>>(theta, P);
    return cudaGetLastError();
}

}  // namespace msk_b200
