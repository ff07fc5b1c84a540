// Fused Gate-SDF MLP on 5th-generation tensor cores (sm_100a): tcgen05.mma with the activation
// operand A and the accumulator D both in tensor memory (TMEM), weights B in shared memory staged by
// bulk-async copies (cp.async.bulk, the TMA engine), bias + activation + bf16 pack in the epilogue,
// the output layer and the finite-difference guidance combine fused into the last epilogue.
//
// Method (PAPER.md:168 "query the decoder for every predicted position", :40 latent concatenated with
// every sampled state, folded here into the per-frame bias b1' = W1[:,3:] z + b1; Eq. 10
// with the BASELINE configs[1] terms 50 exp(-s/0.1) - 0.5 grad(s).v, reading R12):
//   a1 = bf16(act(W1[:, :3] p_c + b1'))                     layer 1 on CUDA cores (fp32), K = 3
//   a_l = bf16(act(W_l a_{l-1} + b_l)), l = 2..n_hidden     tensor cores, bf16 x bf16 -> fp32 (TMEM)
//   s = w_out . a_L + b_out                                 fused into the last epilogue (fp32)
//   term = w_sdf exp(min(-s/scale, emax)) - w_guide |v| (s(p_c + h d) - s(p_c)) / h
//
// Tile = 128 query rows (64 states x {p_c, p_c + h d} with guidance). One persistent CTA per SM walks
// tiles; per tile and GEMM layer the work is split into four MMA units (N-half h, K-half c), so the
// epilogue of N-half 0 overlaps the MMAs of N-half 1 and the next layer's K-half-0 MMAs overlap the
// epilogue of N-half 1 (DESIGN.md §K2 for the schedule and why it keeps the tensor pipe busy).
// TMEM columns: D [0, H) fp32 accumulator; A0 [H, 3H/2), A1 [3H/2, 2H) bf16 activations (2 per column).
// Warp roles: warp 0 = MMA issuer (one thread) + TMEM allocator; warp 1 = weight producer;
// warps 4..11 = epilogue (warp w owns TMEM lanes 32 (w%4).. and one column quarter of each N-half).
#include <cuda_bf16.h>
#include <stdint.h>

#include <cstring>

#include "../../include/mppi.h"
#include "mppi_internal.cuh"

namespace mppi {
namespace tc {

constexpr int kThreads = 384;
constexpr int kEpiWarp0 = 4;
constexpr int kEpiWarps = 8;
constexpr int kTileRows = 128;
constexpr int kRingSlots = 4;

// ------------------------------------------------------------------ PTX wrappers
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t a, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.b32 %0, 1, 0, P1;\n\t}"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
    return ok != 0;
}
// Bounded wait: a schedule bug traps (launch error) instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t a = smem_u32(bar);
    uint32_t n = 0;
    while (!mbar_try_wait(a, parity)) {
        if (++n > (1u << 26)) __trap();
    }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
// D[tmem] (+)= A[tmem] x B[smem]^T  (M=128, N from idesc, K=16; bf16 in, fp32 accumulate)
__device__ __forceinline__ void tc_mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                          uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
        "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void named_bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// UMMA shared-memory descriptor: K-major, 128-byte swizzle, 8-row atoms 1024 B apart (SBO).
__device__ __forceinline__ uint64_t smem_desc_sw128(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// Instruction descriptor kind::f16: D fp32, A/B bf16, both K-major, M = 128.
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ float tanh_approx(float x) {
    float y;
    asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
template <int ACT>
__device__ __forceinline__ float act_fn(float x) {
    if constexpr (ACT == MPPI_ACT_RELU) {
        return fmaxf(x, 0.f);
    } else if constexpr (ACT == MPPI_ACT_SILU) {
        const float h = 0.5f * x;             // silu(x) = x sigmoid(x) = h + h tanh(h), h = x/2
        return fmaf(h, tanh_approx(h), h);
    } else {
        return fmaxf(x, 0.f) + log1pf(__expf(-fabsf(x)));
    }
}

// ------------------------------------------------------------------ kernel
template <int H, int G>
struct Cfg {
    static constexpr int HALF = H / 2;                       // N (and K) extent of one MMA unit
    static constexpr int UNIT_BYTES = HALF * HALF * 2;       // bf16 B block of one unit
    static constexpr bool RESIDENT = (size_t)G * 4 * UNIT_BYTES <= 160 * 1024;
    static constexpr int W_BYTES = RESIDENT ? G * 4 * UNIT_BYTES : kRingSlots * UNIT_BYTES;
    static constexpr int TMEM_COLS = 2 * H;                  // D (H) + two A regions (H/2 each)
    static constexpr int A0 = H;                             // TMEM column of A region 0
    static constexpr int QW = HALF / 2;                      // epilogue columns per warp per unit
    static constexpr int SMEM = 1024 /*align*/ + W_BYTES + 4 * (G * H) + 4 * H + 16 * H + 4 * 2 * 2 * kTileRows +
                                64 * 8 /*barriers*/ + 16;
};

template <int H, int G, int ACT>
__global__ void __launch_bounds__(kThreads, 1)
    k_mlp_tc(Params p, const float4* __restrict__ rows, long long n_rows, int ctrl_fixed, int states_mode,
             const uint8_t* __restrict__ wimg, const float* __restrict__ hid_b, const float* __restrict__ w_out,
             const float* __restrict__ b_out, const float4* __restrict__ w1p, const float* __restrict__ b1f,
             float* __restrict__ sdf_out, float* __restrict__ terms) {
    using C = Cfg<H, G>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t* s_w = smem;                                             // weights (resident) or ring
    float* s_hb = (float*)(s_w + C::W_BYTES);                        // [G][H]
    float* s_wo = s_hb + G * H;                                      // [H]
    float4* s_w1 = (float4*)(s_wo + H);                              // [H]
    float* s_part = (float*)(s_w1 + H);                              // [2 parity][2 ch][128]
    uint64_t* bars = (uint64_t*)(s_part + 2 * 2 * kTileRows);
    uint64_t* bar_aready = bars + 0;    // [region 2][chunk 2]
    uint64_t* bar_dfree = bars + 4;     // [2]
    uint64_t* bar_mma = bars + 6;       // [2]
    uint64_t* bar_full = bars + 8;      // [kRingSlots] (resident: [0] = weights loaded)
    uint64_t* bar_empty = bars + 16;    // [kRingSlots]
    uint32_t* s_tmem = (uint32_t*)(bars + 32);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long n_tiles = (n_rows + kTileRows - 1) / kTileRows;

    // ---- setup
    for (int i = threadIdx.x; i < G * H; i += kThreads) s_hb[i] = hid_b[i];
    for (int i = threadIdx.x; i < H; i += kThreads) { s_wo[i] = w_out[i]; s_w1[i] = w1p[i]; }
    if (threadIdx.x == 0) {
        for (int i = 0; i < 4; ++i) mbar_init(bar_aready + i, kEpiWarps);
        for (int i = 0; i < 2; ++i) { mbar_init(bar_dfree + i, kEpiWarps); mbar_init(bar_mma + i, 1); }
        for (int i = 0; i < kRingSlots; ++i) { mbar_init(bar_full + i, 1); mbar_init(bar_empty + i, 1); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(s_tmem)),
                     "r"(C::TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *s_tmem;

    if (warp == 1) {
        // ================= weight producer
        if (lane == 0) {
            if constexpr (C::RESIDENT) {
                if (blockIdx.x < n_tiles) {
                    mbar_expect_tx(bar_full, (uint32_t)C::W_BYTES);
                    for (int u = 0; u < G * 4; ++u)
                        bulk_g2s(s_w + (size_t)u * C::UNIT_BYTES, wimg + (size_t)u * C::UNIT_BYTES, C::UNIT_BYTES,
                                 bar_full);
                }
            } else {
                uint32_t it = 0;
                for (long long tile = blockIdx.x; tile < n_tiles; tile += gridDim.x)
                    for (int u = 0; u < G * 4; ++u, ++it) {
                        const uint32_t slot = it % kRingSlots;
                        if (it >= kRingSlots) mbar_wait(bar_empty + slot, ((it / kRingSlots) - 1) & 1);
                        mbar_expect_tx(bar_full + slot, (uint32_t)C::UNIT_BYTES);
                        bulk_g2s(s_w + (size_t)slot * C::UNIT_BYTES, wimg + (size_t)u * C::UNIT_BYTES, C::UNIT_BYTES,
                                 bar_full + slot);
                    }
            }
        }
    } else if (warp == 0) {
        // ================= MMA issuer (single thread)
        if (lane == 0) {
            constexpr uint32_t idesc = idesc_bf16(128, C::HALF);
            const uint32_t w_base = smem_u32(s_w);
            uint32_t stage = 0;            // A stage counter (region = stage & 1)
            uint32_t d_use[2] = {0, 0};    // uses of D half h so far
            uint32_t it = 0;               // weight ring iterator
            bool weights_ready = false;
            for (long long tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
                for (int l = 0; l < G; ++l, ++stage) {
                    const uint32_t region = stage & 1;
                    const uint32_t a_col = (uint32_t)C::A0 + region * (H / 2);
                    for (int h = 0; h < 2; ++h)
                        for (int c = 0; c < 2; ++c) {
                            if (h == 0) {
                                mbar_wait(bar_aready + region * 2 + c, (stage >> 1) & 1);
                            }
                            if (c == 0) {
                                if (d_use[h] > 0) mbar_wait(bar_dfree + h, (d_use[h] - 1) & 1);
                                ++d_use[h];
                            }
                            uint32_t b_addr;
                            if constexpr (C::RESIDENT) {
                                if (!weights_ready) { mbar_wait(bar_full, 0); weights_ready = true; }
                                b_addr = w_base + (uint32_t)(((l * 2 + h) * 2 + c) * C::UNIT_BYTES);
                            } else {
                                const uint32_t slot = it % kRingSlots;
                                mbar_wait(bar_full + slot, (it / kRingSlots) & 1);
                                b_addr = w_base + slot * (uint32_t)C::UNIT_BYTES;
                            }
                            tc_fence_after();
#pragma unroll
                            for (int j = 0; j < C::HALF / 16; ++j) {
                                const int kk = j * 16;
                                const uint32_t boff = (uint32_t)((kk / 64) * (C::HALF * 128) + (kk % 64) * 2);
                                const uint64_t bdesc = smem_desc_sw128(b_addr + boff);
                                const uint32_t a_t = tmem + a_col + (uint32_t)((c * C::HALF + kk) / 2);
                                const uint32_t d_t = tmem + (uint32_t)(h * C::HALF);
                                tc_mma_ts(d_t, a_t, bdesc, idesc, (c > 0 || j > 0) ? 1u : 0u);
                            }
                            if constexpr (!C::RESIDENT) {
                                tc_commit(bar_empty + (it % kRingSlots));
                                ++it;
                            }
                            if (c == 1) tc_commit(bar_mma + h);
                        }
                }
            }
        }
    } else if (warp >= kEpiWarp0) {
        // ================= epilogue (8 warps)
        const int e = warp - kEpiWarp0;
        const int g = warp & 3;            // TMEM lane quarter
        const int ch = e >> 2;             // column quarter within an N-half
        const int row_in_tile = g * 32 + lane;
        const uint32_t lane_addr = (uint32_t)(g * 32) << 16;
        uint32_t stage = 0;                // A stage produced next
        uint32_t mma_cnt[2] = {0, 0};
        long long tile = blockIdx.x;
        // layer 1 (CUDA cores): a1 = act(W1p p + b1') -> bf16 -> TMEM A region of `stage`
        auto layer1 = [&](long long t1) {
            const long long row = t1 * kTileRows + row_in_tile;
            float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
            int bb = ctrl_fixed;
            if (row < n_rows) {
                q = rows[row];
                if (states_mode) bb = (int)((row / p.rps) / ((long long)p.T * p.K));
            }
            const float* bf = b1f + (size_t)bb * H;
            const uint32_t region = stage & 1;
            const uint32_t a_col = (uint32_t)C::A0 + region * (H / 2);
            for (int c = 0; c < 2; ++c) {
#pragma unroll
                for (int q32 = 0; q32 < C::QW / 32; ++q32) {
                    const int j0 = c * C::HALF + ch * C::QW + q32 * 32;
                    uint32_t packed[16];
#pragma unroll
                    for (int i = 0; i < 32; i += 2) {
                        const float4 w0 = s_w1[j0 + i], w1 = s_w1[j0 + i + 1];
                        const float x0 = fmaf(w0.x, q.x, fmaf(w0.y, q.y, fmaf(w0.z, q.z, __ldg(bf + j0 + i))));
                        const float x1 = fmaf(w1.x, q.x, fmaf(w1.y, q.y, fmaf(w1.z, q.z, __ldg(bf + j0 + i + 1))));
                        packed[i / 2] = pack_bf16x2(act_fn<ACT>(x0), act_fn<ACT>(x1));
                    }
                    tmem_st16(tmem + lane_addr + a_col + (uint32_t)(j0 / 2), packed);
                }
                tmem_wait_st();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(bar_aready + region * 2 + c);
            }
            ++stage;
            return q.w;   // |v| of this row (meaningful on even rows in states mode)
        };

        float nv = 0.f;
        if (tile < n_tiles) nv = layer1(tile);
        for (; tile < n_tiles; tile += gridDim.x) {
            const long long next = tile + gridDim.x;
            float sdot = 0.f;
            for (int l = 0; l < G; ++l) {
                const bool last = (l == G - 1);
                float nv_next = 0.f;
                if (last && next < n_tiles) nv_next = layer1(next);   // overlaps the last layer's MMAs
                const uint32_t region = stage & 1;                   // region this layer's output goes to
                const uint32_t a_col = (uint32_t)C::A0 + region * (H / 2);
                for (int h = 0; h < 2; ++h) {
                    mbar_wait(bar_mma + h, mma_cnt[h] & 1);
                    ++mma_cnt[h];
                    tc_fence_after();
#pragma unroll
                    for (int q32 = 0; q32 < C::QW / 32; ++q32) {
                        const int j0 = h * C::HALF + ch * C::QW + q32 * 32;
                        uint32_t acc[32];
                        tmem_ld32(tmem + lane_addr + (uint32_t)j0, acc);
                        tmem_wait_ld();
                        const float* bias = s_hb + l * H + j0;
                        if (!last) {
                            uint32_t packed[16];
#pragma unroll
                            for (int i = 0; i < 32; i += 2) {
                                const float x0 = __uint_as_float(acc[i]) + bias[i];
                                const float x1 = __uint_as_float(acc[i + 1]) + bias[i + 1];
                                packed[i / 2] = pack_bf16x2(act_fn<ACT>(x0), act_fn<ACT>(x1));
                            }
                            tmem_st16(tmem + lane_addr + a_col + (uint32_t)(j0 / 2), packed);
                        } else {
#pragma unroll
                            for (int i = 0; i < 32; i += 2) {
                                const float x0 = __uint_as_float(acc[i]) + bias[i];
                                const float x1 = __uint_as_float(acc[i + 1]) + bias[i + 1];
                                const uint32_t pk = pack_bf16x2(act_fn<ACT>(x0), act_fn<ACT>(x1));
                                sdot = fmaf(__uint_as_float(pk << 16), s_wo[j0 + i], sdot);
                                sdot = fmaf(__uint_as_float(pk & 0xFFFF0000u), s_wo[j0 + i + 1], sdot);
                            }
                        }
                    }
                    if (!last) tmem_wait_st();
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) {
                        mbar_arrive(bar_dfree + h);
                        if (!last) mbar_arrive(bar_aready + region * 2 + h);
                    }
                }
                if (!last) ++stage;
                if (last) {
                    // ---- output: combine the two column quarters, FD pair, write
                    const int par = (int)(((tile - blockIdx.x) / gridDim.x) & 1);
                    float* part = s_part + par * 2 * kTileRows;
                    part[ch * kTileRows + row_in_tile] = sdot;
                    named_bar_sync(1, kEpiWarps * 32);
                    if (ch == 0) {
                        const float s = part[row_in_tile] + part[kTileRows + row_in_tile] + __ldg(b_out);
                        const long long row = tile * kTileRows + row_in_tile;
                        if (row < n_rows && sdf_out) sdf_out[row] = s;
                        if (states_mode) {
                            float term;
                            if (p.rps == 2) {
                                const float s1 = __shfl_xor_sync(0xFFFFFFFFu, s, 1);
                                term = p.w_sdf * __expf(fminf(-s * p.inv_sdf_scale, p.sdf_exp_max)) -
                                       p.w_guide * nv * (s1 - s) * p.inv_fd_h;
                                if ((lane & 1) == 0 && row < n_rows) terms[row >> 1] = term;
                            } else {
                                term = p.w_sdf * __expf(fminf(-s * p.inv_sdf_scale, p.sdf_exp_max));
                                if (row < n_rows) terms[row] = term;
                            }
                        }
                    }
                    nv = nv_next;
                }
            }
        }
    }
    // ---- teardown
    __syncwarp();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::TMEM_COLS));
}

template <int H, int G, int ACT>
cudaError_t launch_t(const Params& p, const Buffers& b, const float4* rows, long long n_rows, int ctrl_fixed,
                     float* sdf_out, bool states_mode, cudaStream_t s) {
    using C = Cfg<H, G>;
    static bool attr_set = false;
    static int n_sm = 0;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(k_mlp_tc<H, G, ACT>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
        if (e != cudaSuccess) return e;
        int dev;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
        attr_set = true;
    }
    const long long tiles = (n_rows + kTileRows - 1) / kTileRows;
    if (tiles == 0) return cudaSuccess;
    const int grid = (int)(tiles < n_sm ? tiles : n_sm);
    k_mlp_tc<H, G, ACT><<<grid, kThreads, C::SMEM, s>>>(p, rows, n_rows, ctrl_fixed, states_mode ? 1 : 0, b.hid_wbf,
                                                         b.hid_b, b.w_out, b.b_out, b.w1p, b.b1f, sdf_out, b.terms);
    return cudaGetLastError();
}

}  // namespace tc

bool mlp_tc_supported(int H, int G, int act) {
    return (H == 128 || H == 256) && G >= 1 && G <= 3 && act >= 0 && act <= 2;
}

size_t mlp_tc_weight_bytes(int H, int G) { return (size_t)G * H * H * 2; }

// Global image = the shared-memory image: [layer][N-half h][K-half c] blocks of HALF x HALF bf16;
// inside a block, [64-wide K chunk][row n][128 B] with the 16-byte groups of row n XOR-swizzled by
// (n % 8) (UMMA SWIZZLE_128B, K-major, 8-row atoms of 1024 B).
void mlp_tc_pack_weights(int H, int G, const float* W, uint8_t* out) {
    const int HALF = H / 2;
    const size_t unit = (size_t)HALF * HALF * 2;
    for (int l = 0; l < G; ++l)
        for (int h = 0; h < 2; ++h)
            for (int c = 0; c < 2; ++c) {
                uint8_t* blk = out + (size_t)((l * 2 + h) * 2 + c) * unit;
                for (int nn = 0; nn < HALF; ++nn)
                    for (int kk = 0; kk < HALF; ++kk) {
                        const float v = W[(size_t)l * H * H + (size_t)(h * HALF + nn) * H + (c * HALF + kk)];
                        uint32_t u;
                        std::memcpy(&u, &v, 4);   // already a bf16 value: the top 16 bits are exact
                        const uint16_t bits = (uint16_t)(u >> 16);
                        const int kc = kk / 64, w = kk % 64;
                        const size_t off = (size_t)kc * HALF * 128 + (size_t)nn * 128 + (size_t)(((w / 8) ^ (nn % 8)) * 16) +
                                           (size_t)(w % 8) * 2;
                        std::memcpy(blk + off, &bits, 2);
                    }
            }
}

cudaError_t launch_mlp_tc(const Params& p, const Buffers& b, const float4* rows, long long n_rows, int ctrl_fixed,
                          float* sdf_out, bool states_mode, cudaStream_t s) {
#define MPPI_TC_CASE(HH, GG, AA) \
    if (p.H == HH && p.n_gemm == GG && p.act == AA) return tc::launch_t<HH, GG, AA>(p, b, rows, n_rows, ctrl_fixed, sdf_out, states_mode, s);
#define MPPI_TC_ACTS(HH, GG) MPPI_TC_CASE(HH, GG, 0) MPPI_TC_CASE(HH, GG, 1) MPPI_TC_CASE(HH, GG, 2)
    MPPI_TC_ACTS(128, 1) MPPI_TC_ACTS(128, 2) MPPI_TC_ACTS(128, 3)
    MPPI_TC_ACTS(256, 1) MPPI_TC_ACTS(256, 2) MPPI_TC_ACTS(256, 3)
#undef MPPI_TC_ACTS
#undef MPPI_TC_CASE
    return cudaErrorInvalidValue;
}

}  // namespace mppi
