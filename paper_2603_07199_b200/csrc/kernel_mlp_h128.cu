// Fused Gate-SDF MLP at hidden width 128 (configs[1], configs[4]; the H = 128 positional-encoding variant of
// SURVEY §8f F3) on 5th-generation tensor cores (sm_100a). Round-2 design, replacing the H = 128 form of
// kernel_mlp_tc.cu, whose time per tile was dominated by layer 1 on the CUDA cores (timeline trace: ~2.6 k of
// ~3.4 k cycles per tile per CTA at configs[1]) with only two tiles in flight.
//
// Method ("query the decoder for every predicted position"; the latent concatenated with every
// state, folded into the per-frame bias b1' = W1[:,3:] z + b1; Eq. 10 stage term with the
// BASELINE configs[1] terms, reading R12; quantisation contract R15):
//   a1  = bf16(act(W1p . PE(p_c) + b1'))      layer 1 on the TENSOR cores: an exact-split MMA (below)
//   a_l = bf16(act(W_l a_{l-1} + b_l))        hidden layers, bf16 x bf16 -> fp32 in TMEM (bias by an MMA)
//   s   = w_out . a_L + b_out                 fused into the last epilogue (fp32 FFMA2)
//   term = w_sdf exp(min(-s/scale, emax)) - w_guide |v| (s(p_c + h d) - s(p_c)) / h
//
// Layer 1 as an MMA keeps fp32 accuracy (R15: "layer 1 fully fp32"): every fp32 position coordinate x and
// weight w is split exactly into bf16 parts x = x_h + x_m + x_l (+ <= 2^-25 |x|), and the K = 32 operand rows
// carry the six products x_h w_h, x_h w_m, x_m w_h, x_h w_l, x_m w_m, x_l w_h per coordinate (18 columns;
// the dropped ones are <= 2^-24 |x w|); bf16 x bf16 products are exact in the fp32 accumulator. With the
// positional encoding (4 bands, reading E1) each sin/cos feature f adds f_h w_h, f_h w_l, f_l w_h (a two-part
// split: <= 2^-16 relative, ~1e-5 absolute on a pre-activation, far below the 2^-9 bf16 ulp of a1; DESIGN.md
// reading E2) -> K = 96. The folded bias b1' (fp32, per controller) is added in the layer-1 epilogue.
//
// Layout: one CTA per SM (persistent), tiles of 128 query rows (64 states x {p_c, p_c + h d} with guidance).
// NSLOT tiles in flight per CTA (4 for the configs[1]/[4] MLP): each slot owns a 128-column fp32 accumulator D
// in TMEM and a 32 KB shared-memory A operand (SW128 K-major, the layout of the resident weight images), so
// every MMA is the SS form and TMEM holds accumulators only. Per tile and slot the tensor pipe runs the units
// L1 (K = 32/96), GEMM 1..G (bias MMA + K = 128), each followed by that slot's epilogue; the issuer walks the
// slots round-robin, so while one slot's epilogue drains D the other slots' MMAs run.
// Warp roles: warp 0 = TMEM allocator + MMA issuer (lane 0), warp 1 = weight loader, warps 2-3 idle;
// epilogue warps 4.. in groups of 4 (one per TMEM lane quarter / SMSP), group s owns slot s: thread = row.
#include <cuda_bf16.h>
#include <stdint.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "../../include/mppi.h"
#include "mppi_internal.cuh"
#include "rollout_dev.cuh"
#include "tc_ptx.cuh"

namespace mppi {
namespace h128 {
using namespace mppi::tc;

constexpr int H = 128;
constexpr int kRows = 128;      // rows per tile = MMA M
constexpr int kCW = 16;         // TMEM columns per epilogue load
#ifndef H128_NB
#define H128_NB 1
#endif
#ifndef H128_WPS
#define H128_WPS 4      // epilogue warps per tile slot (8: 2 column groups, fewer slots)
#endif
#ifndef H128_REGS_CTL
#define H128_REGS_CTL 56
#endif
#ifndef H128_REGS_CTL_FUSE
#define H128_REGS_CTL_FUSE 88
#endif
#ifndef H128_A1_HELPER
#define H128_A1_HELPER 0   // 1: warps 2-3 build the layer-1 operands (measured +3% at configs[4]: off)
#endif
#ifndef H128_DYN
#define H128_DYN 0   // 1: ready-first issue order over the slots (non-blocking probes)
#endif
#ifndef H128_STAG
#define H128_STAG 0   // > 0: staggered issue order (slot s starts H128_STAG * s visits late)
#endif
#ifndef H128_L1LAG
#define H128_L1LAG 4   // issue order: the next round's layer-1 unit of slot s follows the last GEMM of slot s + LAG
#endif
#ifndef H128_DESC_ADD
#define H128_DESC_ADD 1   // GEMM K-step descriptors by one 32-bit add on the address field (0: rebuilt per MMA;
                          // measured -1.7% at configs[4], -1.6% at configs[1]: the issuer shares SMSP 0 with 4 busy
                          // epilogue warps, so its instruction count per unit is on the MMA hand-off path)
#endif
#ifndef H128_WAIT_FIRST
#define H128_WAIT_FIRST 1   // the issuer probes a barrier once (test_wait) before its try_wait loop (A/B: configs[4]
                            // -1.1%, configs[1] -0.4%; 0: the loop alone)
#endif
#ifndef H128_ISSUER_WAIT
#define H128_ISSUER_WAIT 0   // 0: try_wait loop (no sleep); 1: try_wait with the 100 ns suspend hint (NANOSLEEP in SASS)
#endif
constexpr int kNB = H128_NB;    // 16-column loads per tcgen05.wait::ld

constexpr int kSmemMax = 232448;

template <int G, int PEB, bool FUSE = false>
struct Cfg {
    static constexpr int NPE = 3 + 6 * PEB;                   // position features (raw p, PE bands)
    static constexpr int K1_USED = 18 + 18 * PEB;             // layer-1 operand columns (split products)
    static constexpr int K1 = (K1_USED + 15) / 16 * 16;       // 32, or 96 with 4 PE bands
    static constexpr int K1C = K1 / 8;                        // 16-B K core matrices per row
    static constexpr int W_BYTES = G * H * H * 2;             // hidden weights, SW128 K-major per layer
    static constexpr int BIAS_UNIT = H * 32;                  // per layer: H rows x 16 bf16 [b_hi, b_lo, 0...]
    static constexpr int BIAS_BYTES = G * BIAS_UNIT;
    static constexpr int B1_BYTES = H * K1 * 2;               // layer-1 B operand, no-swizzle K-major
    static constexpr int IMG_BYTES = W_BYTES + BIAS_BYTES + B1_BYTES;
    static constexpr int A_BYTES = kRows * H * 2;             // per slot: A operand (32 KB)
    static constexpr int WPS = H128_WPS;                      // epilogue warps per slot (4 lane quarters x COLG)
    static constexpr int COLG = WPS / 4;                      // column groups: a thread owns QW columns of its row
    static constexpr int QW = H / COLG;
    static constexpr int NCH = QW / kCW;                      // 16-column TMEM loads per thread per unit
    static constexpr int FIXED = IMG_BYTES + 256 + 4 * H + 8 * 32 + 16 + 1024;
    // A1 helper (no PE, not fused): warps 2-3 build every tile's layer-1 operand as soon as the slot's last GEMM
    // has read A, and keep |v| per row in a double-buffered slot array for the output epilogue
    static constexpr bool HELPER = !FUSE && PEB == 0 && H128_A1_HELPER;
    static constexpr int PER_SLOT = A_BYTES + 16 * kRows + 4 * H + 4 * COLG * kRows + 8 * kRows;
    static constexpr int fits(int n) { return FIXED + n * PER_SLOT <= kSmemMax && 4 + WPS * n <= 32; }
#ifdef H128_NSLOT
    static constexpr int NSLOT = H128_NSLOT;
#else
    static constexpr int NSLOT = fits(4) ? 4 : fits(3) ? 3 : 2;
#endif
    static constexpr int OFF_BIAS = W_BYTES;
    static constexpr int OFF_B1 = OFF_BIAS + BIAS_BYTES;
    static constexpr int OFF_A = OFF_B1 + B1_BYTES;           // 1024-aligned (SW128 atoms)
    static constexpr int OFF_ONES = OFF_A + NSLOT * A_BYTES;  // 8 rows x [1, 1, 0 x 14] bf16 (read with SBO = 0)
    static constexpr int OFF_ROWS = OFF_ONES + 256;           // [NSLOT][128] float4 query rows
    static constexpr int OFF_WO = OFF_ROWS + NSLOT * 16 * kRows;
    static constexpr int OFF_B1S = OFF_WO + 4 * H;            // [NSLOT][H] staged b1' (x kPre)
    static constexpr int OFF_PART = OFF_B1S + NSLOT * 4 * H;  // [NSLOT][COLG][128] partial output dots
    static constexpr int OFF_NV = OFF_PART + NSLOT * 4 * COLG * kRows;   // [NSLOT][2][128] |v| per row (HELPER)
    static constexpr int OFF_BAR = OFF_NV + NSLOT * 8 * kRows;
    static constexpr int OFF_TMEM = OFF_BAR + 8 * 32;
    static constexpr int SMEM = 1024 + OFF_TMEM + 16;
    static constexpr int EPI_WARPS = WPS * NSLOT;
    static constexpr int THREADS = 32 * (4 + EPI_WARPS);
    // setmaxnreg split of the launch register pool (65536 / THREADS rounded to 8 per thread)
    static constexpr int REGS_LAUNCH = (65536 / THREADS) / 8 * 8;
    // the issuer loop spills below ~48; FUSE: warps 2-3 of the same warpgroup run the rollout (~80 registers)
    static constexpr int REGS_CTL = REGS_LAUNCH >= 96 ? (FUSE ? H128_REGS_CTL_FUSE : H128_REGS_CTL) : 24;
    static constexpr int REGS_EPI_RAW = (REGS_LAUNCH * THREADS - 128 * REGS_CTL) / (32 * EPI_WARPS) / 8 * 8;
    static constexpr int REGS_EPI = REGS_EPI_RAW > 232 ? 232 : REGS_EPI_RAW;
    static constexpr int TMEM_COLS = NSLOT * 128 <= 256 ? 256 : 512;
    static_assert(SMEM <= kSmemMax, "shared memory budget");
    static_assert(WPS % 4 == 0 && QW % kCW == 0 && (K1C % COLG) == 0, "epilogue partition");
    static_assert(OFF_A % 1024 == 0, "SW128 A tiles need 1024-B alignment");
};

#ifdef MPPI_TC_TRACE
// Debug-only timeline (clock64) of the first 2 CTAs: role 0 = MMA issuer, 1..4 = slot epilogue leaders;
// code = [11:8] event, [7:4] unit (0 = layer 1, 1.. = GEMMs), [3:0] local tile index & 15.
constexpr int kTraceCap = 2048;
__device__ unsigned long long g_h128_trace[2][5][kTraceCap];
#define H_TRACE(role, ev, u, t)                                                                                 \
    do {                                                                                                        \
        if (blockIdx.x < 2 && trace_n < kTraceCap) {                                                            \
            const unsigned long long _c = ((unsigned long long)(ev) << 8) | (((u) & 15) << 4) | ((t) & 15);     \
            g_h128_trace[blockIdx.x][role][trace_n++] = (_c << 48) | ((unsigned long long)clock64() & 0xFFFFFFFFFFFFull); \
        }                                                                                                       \
    } while (0)
#define H_TRACE_DECL int trace_n = 0
#else
#define H_TRACE(role, ev, u, t) \
    do {                        \
    } while (0)
#define H_TRACE_DECL
#endif

// barrier slots (8 B each)
enum { BAR_ROWS = 0, BAR_SA1 = 4, BAR_AREADY = 8, BAR_DFREE = 12, BAR_MMA = 16, BAR_W = 20, BAR_RFREE = 21,
       BAR_AFREE = 25 /*[slots]: the tile's last GEMM has read A (HELPER)*/ };

__device__ __forceinline__ uint32_t bf16_bits(float v) {
    return (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(v));
}
__device__ __forceinline__ float bf16_val(uint32_t b) { return __uint_as_float(b << 16); }
// issuer wait: the suspend-hint form compiles to a NANOSLEEP of the whole hint whenever the first probe
// fails, which adds up to ~200 cycles to every MMA hand-off (timeline trace); the plain try_wait loop does not
__device__ __forceinline__ void issuer_wait(uint32_t bar, uint32_t parity) {
#if H128_ISSUER_WAIT == 1
    mbar_wait_issuer(bar, parity);
#else
#if H128_WAIT_FIRST
    if (mbar_test(bar, parity)) return;   // ready: no loop head (YIELD) on the issuer's path
#endif
    uint32_t n = 0;
    while (!mbar_try_wait<false>(bar, parity))
        if (++n > (1u << 26)) __trap();
#endif
}

// FUSE (the fused rollout, configs[4]-sized problems): the rows are not read from HBM. Warps 2-3 of the control
// warpgroup roll out 64 samples (a "block": one controller, samples k0..k0+63) over the whole horizon with the
// same device code as k_rollout (rollout_dev.cuh) and write each step's 128 query rows straight into the next
// slot's shared-memory row buffer; the CTA's tiles are (block, t) for its blocks in turn. The noise (for
// k_softmin), the shifted nominal and the non-SDF partial costs go to HBM as k_rollout writes them.
template <int G, int ACT, int PEB, bool FUSE>
__global__ void __launch_bounds__(Cfg<G, PEB, FUSE>::THREADS, 1)
    k_mlp_h128(Params p, const float4* __restrict__ rows, long long n_rows, int ctrl_fixed, int states_mode,
               const uint8_t* __restrict__ wimg, const float* __restrict__ w_out, const float* __restrict__ b_out,
               const float* __restrict__ b1f, float* __restrict__ sdf_out, float* __restrict__ terms, Buffers bufs) {
    using C = Cfg<G, PEB, FUSE>;
    constexpr int NS = C::NSLOT;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const uint32_t sbase = smem_u32(smem);
    const uint32_t bar0 = sbase + C::OFF_BAR;
    auto bar = [&](int i) { return bar0 + 8u * (uint32_t)i; };
    uint32_t* s_tmem = reinterpret_cast<uint32_t*>(smem + C::OFF_TMEM);
    float* s_wo = reinterpret_cast<float*>(smem + C::OFF_WO);
    constexpr float kP = kPre<ACT>;
    H_TRACE_DECL;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long group = blockIdx.x, n_groups = gridDim.x;
    // FUSE: blocks of 64 samples (K % 64 == 0, guidance on: 128 rows per (block, t) tile)
    const long long kb_per_ctrl = FUSE ? p.K / 64 : 1;
    const long long n_units = FUSE ? (long long)p.n_ctrl * kb_per_ctrl : (n_rows + kRows - 1) / kRows;
    const long long n_my_units = group < n_units ? (n_units - group + n_groups - 1) / n_groups : 0;
    const long long n_my = FUSE ? n_my_units * p.T : n_my_units;   // local tiles
    const long long rows_per_ctrl = states_mode ? (long long)p.T * p.K * p.rps : (1ll << 62);
    // controller of a step row (states mode): rows < 2^31 (validated), so a 32-bit division -- a 64-bit one is
    // ~10x the instructions, and this runs twice per tile and thread
    auto ctrl_of = [&](long long row) -> long long { return (long long)((uint32_t)row / (uint32_t)rows_per_ctrl); };
    // first global row of local tile i (FUSE: tile = (block j, step t); rows of a state are adjacent)
    auto row0_of = [&](long long i) -> long long {
        if constexpr (FUSE) {   // 32-bit divisions (a 64-bit one is ~10x the instructions, per tile and thread)
            const uint32_t ii = (uint32_t)i, T = (uint32_t)p.T, kb = (uint32_t)kb_per_ctrl;
            const uint32_t j = ii / T, t = ii - j * T, blk = (uint32_t)group + j * (uint32_t)n_groups;
            const uint32_t bb = blk / kb, k0 = (blk - bb * kb) * 64u;
            return (((long long)bb * p.T + t) * p.K + k0) * 2;
        } else {
            return (group + i * n_groups) * kRows;
        }
    };

    // ---- setup: the ones operand of the bias MMA (one 8-row group, every group reads it: SBO = 0)
    if (threadIdx.x < 16) {
        uint32_t* o = reinterpret_cast<uint32_t*>(smem + C::OFF_ONES + threadIdx.x * 16);
        o[0] = threadIdx.x < 8 ? 0x3F803F80u : 0u;   // K core 0: row = [1, 1, 0 x 6]; K core 1: zeros
        o[1] = o[2] = o[3] = 0u;
    }
    for (int i = threadIdx.x; i < H; i += blockDim.x) s_wo[i] = w_out[i];
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(bar(BAR_ROWS + s), FUSE ? 2 : 1);   // FUSE: the two rollout warps
            mbar_init(bar(BAR_RFREE + s), 1);
            mbar_init(bar(BAR_AFREE + s), 1);
            mbar_init(bar(BAR_SA1 + s), C::HELPER ? 2 : C::WPS);
            mbar_init(bar(BAR_AREADY + s), C::WPS);
            mbar_init(bar(BAR_DFREE + s), C::WPS);
            mbar_init(bar(BAR_MMA + s), 1);
        }
        mbar_init(bar(BAR_W), 1);
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

    if (warp < 4) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(C::REGS_CTL));
        if (warp == 1 && lane == 0 && n_my > 0) {
            // ================= weight loader: the whole image (hidden W, hidden biases, layer-1 B), once
            mbar_expect_tx(bar(BAR_W), (uint32_t)C::IMG_BYTES);
            for (int off = 0; off < C::IMG_BYTES; off += 32768) {
                const int nb = C::IMG_BYTES - off < 32768 ? C::IMG_BYTES - off : 32768;
                bulk_g2s(sbase + (uint32_t)off, wimg + off, (uint32_t)nb, bar(BAR_W));
            }
        } else if (C::HELPER && (warp == 2 || warp == 3) && n_my > 0) {
            // ================= layer-1 operand builder: tile i of slot i % NS as soon as the slot's last GEMM of
            // tile i - NS has read A (BAR_AFREE, one commit per tile: it cannot run a phase ahead, because the
            // slot's next MMA is this tile's layer 1, which waits for this builder), two rows per thread
            const int tid = threadIdx.x - 64;
            auto issue_rows_h = [&](long long i) {
                if (i >= n_my) return;
                const int s2 = (int)(i % NS);
                const long long r0 = row0_of(i);
                const long long nr = min((long long)kRows, n_rows - r0);
                mbar_expect_tx(bar(BAR_ROWS + s2), (uint32_t)(16 * nr));
                bulk_g2s(sbase + (uint32_t)(C::OFF_ROWS + s2 * 16 * kRows), rows + r0, (uint32_t)(16 * nr), bar(BAR_ROWS + s2));
            };
            if (tid == 0)
                for (int s2 = 0; s2 < NS; ++s2) issue_rows_h(s2);
            for (long long i = 0; i < n_my; ++i) {
                const int sl = (int)(i % NS);
                const uint32_t rnd = (uint32_t)(i / NS);
                if (rnd > 0) mbar_wait(bar(BAR_AFREE + sl), (rnd - 1) & 1u);
                mbar_wait(bar(BAR_ROWS + sl), rnd & 1u);
                const float4* s_rows = reinterpret_cast<const float4*>(smem + C::OFF_ROWS + sl * 16 * kRows);
                float* s_nv = reinterpret_cast<float*>(smem + C::OFF_NV + (sl * 2 + (int)(rnd & 1u)) * 4 * kRows);
                const uint32_t aA = sbase + (uint32_t)(C::OFF_A + sl * C::A_BYTES);
#pragma unroll
                for (int hf = 0; hf < 2; ++hf) {
                    const int r = tid + 64 * hf;
                    const long long row = row0_of(i) + r;
                    const float4 q = row < n_rows ? s_rows[r] : make_float4(0.f, 0.f, 0.f, 0.f);
                    s_nv[r] = q.w;
                    uint32_t col[C::K1];
#pragma unroll
                    for (int k = 0; k < C::K1; ++k) col[k] = 0u;
                    const float pv[3] = {q.x, q.y, q.z};
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        const uint32_t h = bf16_bits(pv[c]);
                        const float r1 = pv[c] - bf16_val(h);
                        const uint32_t m = bf16_bits(r1);
                        const uint32_t lo = bf16_bits(r1 - bf16_val(m));
                        col[0 + c] = h; col[3 + c] = h; col[6 + c] = m; col[9 + c] = h; col[12 + c] = m; col[15 + c] = lo;
                    }
                    const uint32_t rb = aA + (uint32_t)((r / 8) * (C::K1C * 128) + (r % 8) * 16);
#pragma unroll
                    for (int kc = 0; kc < C::K1C; ++kc)
                        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(rb + (uint32_t)(kc * 128)),
                                     "r"(col[8 * kc] | (col[8 * kc + 1] << 16)), "r"(col[8 * kc + 2] | (col[8 * kc + 3] << 16)),
                                     "r"(col[8 * kc + 4] | (col[8 * kc + 5] << 16)), "r"(col[8 * kc + 6] | (col[8 * kc + 7] << 16))
                                     : "memory");
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes -> MMA operand reads
                named_bar_sync(7, 64);   // both builder warps have read the row buffer
                if (tid == 0) issue_rows_h(i + NS);
                __syncwarp();
                if (lane == 0) mbar_arrive_local(bar(BAR_SA1 + sl));
            }
        } else if (FUSE && (warp == 2 || warp == 3) && n_my > 0) {
            // ================= fused rollout producer: thread = one sample of the current block
            const int tid = threadIdx.x - 64;
            const unsigned long long step = *bufs.step;
            const int sh = step > 0 ? 1 : 0;
            const bool dev_noise = p.noise_device != 0;
            const long long NK = (long long)p.n_ctrl * p.K;
            const float inv_mass = 1.f / p.mass;
            for (long long j = 0; j < n_my_units; ++j) {
                const long long blk = group + j * n_groups;
                const int bb = (int)(blk / kb_per_ctrl);
                const int k = (int)((blk % kb_per_ctrl) * 64) + tid;
                const bool first_block = blk % kb_per_ctrl == 0;
                float x[10];
#pragma unroll
                for (int q = 0; q < 10; ++q) x[q] = __ldg(bufs.x0 + bb * 10 + q);
                float R[9], tq[3], gc[3];
#pragma unroll
                for (int q = 0; q < 9; ++q) R[q] = __ldg(bufs.Tq + bb * 12 + q);
#pragma unroll
                for (int q = 0; q < 3; ++q) { tq[q] = __ldg(bufs.Tq + bb * 12 + 9 + q); gc[q] = __ldg(bufs.goal + bb * 3 + q); }
                const long long col = (long long)bb * p.K + k;
                const unsigned long long gidx = global_sample(p, bb, k);
                const float4* Uo = reinterpret_cast<const float4*>(bufs.U_out) + (long long)bb * p.T;
                float part = 0.f;
                for (int t = 0; t < p.T; ++t) {
                    const long long i = j * p.T + t;
                    const int sl = (int)(i % NS);
                    const uint32_t use = (uint32_t)(i / NS);
                    const float4 U = Uo[min(t + sh, p.T - 1)];   // warm-start shift
                    if (first_block && tid == 0) reinterpret_cast<float4*>(bufs.U_nom)[(long long)bb * p.T + t] = U;
                    float4 n;
                    if (dev_noise) {
                        n = philox_normals(gidx, t, step, p.seed);
                        bufs.noise[(long long)t * NK + col] = n;   // for k_softmin
                    } else {
                        n = bufs.noise[(long long)t * NK + col];
                    }
                    float4 row0, row1;
                    ctbr_step(p, x, U, n, R, tq, gc, inv_mass, row0, row1, part);
                    if (use > 0) mbar_wait(bar(BAR_RFREE + sl), (use - 1) & 1u);   // the slot has read its rows
                    float4* dst = reinterpret_cast<float4*>(smem + C::OFF_ROWS + sl * 16 * kRows);
                    dst[2 * tid] = row0;
                    dst[2 * tid + 1] = row1;
                    __syncwarp();
                    if (lane == 0) mbar_arrive_local(bar(BAR_ROWS + sl));
                }
                bufs.partial[col] = part;
            }
        } else if (warp == 0 && n_my > 0) {
            // ================= MMA issuer: per round of NS tiles, unit u = 0 (layer 1), 1..G (GEMMs), slots
            // round-robin. Barrier phases follow from (round n, unit): SA1 / DFREE once per tile, AREADY G times.
            // The whole warp walks the schedule with warp-uniform values (descriptors in uniform registers) and one
            // elected lane issues. (A ready-first order over the slots, with non-blocking probes, measured 30%
            // slower at configs[4].)
            constexpr uint32_t idesc = idesc_bf16(128, 128);
            mbar_wait(bar(BAR_W), 0);
            // unit u of slot sl's n-th tile (local tile i0 + sl, i0 = n NS): wait for its operands, issue, commit
            auto issue_unit = [&](int sl, int u, uint32_t n, long long i0) {
                const uint32_t d_t = tmem + (uint32_t)(sl * 128);
                const uint32_t a0 = sbase + (uint32_t)(C::OFF_A + sl * C::A_BYTES);
                if (lane == 0) H_TRACE(0, 0, u, i0 + sl);
                if (u == 0) {
                    if (n > 0) issuer_wait(bar(BAR_DFREE + sl), (n - 1) & 1u);
                    issuer_wait(bar(BAR_SA1 + sl), n & 1u);
                } else {
                    issuer_wait(bar(BAR_AREADY + sl), (n * (uint32_t)G + (uint32_t)(u - 1)) & 1u);
                }
                tc_fence_after();
                if (lane == 0) H_TRACE(0, 1, u, i0 + sl);
                if (elect_one()) {
                    if (u == 0) {
                        const uint32_t b0 = sbase + (uint32_t)C::OFF_B1;
#pragma unroll
                        for (int j = 0; j < C::K1 / 16; ++j)
                            tc_mma_ss<1>(d_t, smem_desc_noswz(a0 + (uint32_t)(j * 256), 128, C::K1C * 128),
                                         smem_desc_noswz(b0 + (uint32_t)(j * 256), 128, C::K1C * 128), idesc,
                                         j > 0 ? 1u : 0u);
                    } else {
                        const int l = u - 1;
                        // D = bias (ones x [b_hi, b_lo]), then D += A W_l^T over K = 128
#ifndef H128_NO_BIAS_MMA
                        tc_mma_ss<1>(d_t, smem_desc_noswz(sbase + (uint32_t)C::OFF_ONES, 128, 0),
                                     smem_desc_noswz(sbase + (uint32_t)(C::OFF_BIAS + l * C::BIAS_UNIT), 128, 256),
                                     idesc, 0u);
#endif
                        const uint32_t w0 = sbase + (uint32_t)(l * H * H * 2);
#if H128_DESC_ADD
                        // K step j: the descriptors' 14-bit address fields advance by off / 16 (no carry: shared
                        // addresses < 256 KB), so one 32-bit add per operand instead of a descriptor rebuild
                        const uint64_t ad = smem_desc_sw128(a0), wd = smem_desc_sw128(w0);
                        const uint32_t ad_lo = (uint32_t)ad, ad_hi = (uint32_t)(ad >> 32);
                        const uint32_t wd_lo = (uint32_t)wd, wd_hi = (uint32_t)(wd >> 32);
#pragma unroll
                        for (int j = 0; j < H / 16; ++j) {
                            const uint32_t o16 = (uint32_t)((j / 4) * (kRows * 128) + (j % 4) * 32) >> 4;
                            tc_mma_ss<1>(d_t, ((uint64_t)ad_hi << 32) | (ad_lo + o16), ((uint64_t)wd_hi << 32) | (wd_lo + o16),
                                         idesc, 1u);
                        }
#else
#pragma unroll
                        for (int j = 0; j < H / 16; ++j) {
                            const uint32_t off = (uint32_t)((j / 4) * (kRows * 128) + (j % 4) * 32);
                            tc_mma_ss<1>(d_t, smem_desc_sw128(a0 + off), smem_desc_sw128(w0 + off), idesc, 1u);
                        }
#endif
                    }
                    tc_commit<1>(bar(BAR_MMA + sl));
                    // a second commit of the last GEMM for the layer-1 builder (its own barrier: waiting on
                    // BAR_MMA's parity could alias a phase two commits back)
                    if (C::HELPER && u == G) tc_commit<1>(bar(BAR_AFREE + sl));
                }
                __syncwarp();
                if (lane == 0) H_TRACE(0, 2, u, i0 + sl);
            };
#if H128_DYN
            // ready-first order: each round the issuer takes, among the slots whose next unit's operands are ready
            // (non-blocking mbarrier probes), the one earliest in the round-robin order (key = units issued x NS +
            // slot), so a slot still in its epilogue never holds back a ready one
            uint32_t cnt[NS], lim[NS];
#pragma unroll
            for (int s2 = 0; s2 < NS; ++s2) {
                cnt[s2] = 0u;
                lim[s2] = (uint32_t)((n_my > s2 ? (n_my - s2 + NS - 1) / NS : 0) * (G + 1));
            }
            uint32_t spins = 0;
            for (;;) {
                int pick = -1;
                uint32_t best = 0xFFFFFFFFu;
                bool pending = false;
#pragma unroll
                for (int s2 = 0; s2 < NS; ++s2) {
                    if (cnt[s2] >= lim[s2]) continue;
                    pending = true;
                    const uint32_t key = cnt[s2] * (uint32_t)NS + (uint32_t)s2;
                    if (key >= best) continue;
                    const uint32_t n = cnt[s2] / (uint32_t)(G + 1);
                    const uint32_t u = cnt[s2] - n * (uint32_t)(G + 1);
                    const bool rdy = u == 0 ? ((n == 0 || mbar_test(bar(BAR_DFREE + s2), (n - 1) & 1u)) &&
                                               mbar_test(bar(BAR_SA1 + s2), n & 1u))
                                            : mbar_test(bar(BAR_AREADY + s2), (n * (uint32_t)G + u - 1) & 1u);
                    if (rdy) {
                        best = key;
                        pick = s2;
                    }
                }
                if (!pending) break;
                if (pick < 0) {
                    if (++spins > (1u << 28)) __trap();
                    continue;
                }
#pragma unroll
                for (int s2 = 0; s2 < NS; ++s2)
                    if (s2 == pick) {
                        const uint32_t n = cnt[s2] / (uint32_t)(G + 1);
                        issue_unit(s2, (int)(cnt[s2] - n * (uint32_t)(G + 1)), n, (long long)n * NS);
                        ++cnt[s2];
                    }
            }
#elif H128_STAG > 0
            // staggered order: the issuer visits the slots round-robin and each visit issues the slot's next unit;
            // slot s joins H128_STAG * s visits late, so the slots' epilogue phases (layer 1, GEMM, output) do not
            // all coincide. Per-slot unit counters, compile-time indexed (the visit loop is unrolled over the slots)
            uint32_t cnt[NS], lim[NS];
#pragma unroll
            for (int s2 = 0; s2 < NS; ++s2) {
                cnt[s2] = 0u;
                lim[s2] = (uint32_t)((n_my > s2 ? (n_my - s2 + NS - 1) / NS : 0) * (G + 1));
            }
            for (uint32_t round = 0;; ++round) {
                bool any = false;
#pragma unroll
                for (int sl = 0; sl < NS; ++sl) {
                    if (cnt[sl] < lim[sl]) any = true;
                    if (round < (uint32_t)(H128_STAG * sl) || cnt[sl] >= lim[sl]) continue;
                    const uint32_t n = cnt[sl] / (uint32_t)(G + 1);
                    issue_unit(sl, (int)(cnt[sl] - n * (uint32_t)(G + 1)), n, (long long)n * NS);
                    ++cnt[sl];
                }
                if (!any) break;
            }
#else
            // lockstep rounds: per round of NS tiles, unit u of every slot before unit u + 1. The next round's
            // layer-1 units are interleaved into this round's last GEMM units, slot s's right after the last GEMM
            // of slot s + H128_L1LAG (H128_L1LAG >= NS: all of them after the last GEMMs, the plain order), so the
            // small layer-1 MMAs and their epilogues overlap the other slots' last GEMMs
            constexpr int kLag = H128_L1LAG;
            {
                const int ns0 = (int)min((long long)NS, n_my);
                for (int sl = 0; sl < ns0; ++sl) issue_unit(sl, 0, 0u, 0);
            }
            for (long long i0 = 0; i0 < n_my; i0 += NS) {
                const uint32_t n = (uint32_t)(i0 / NS);
                const int ns = (int)min((long long)NS, n_my - i0);
                const int ns_next = (int)max(0ll, min((long long)NS, n_my - i0 - NS));
                for (int u = 1; u < G; ++u)
                    for (int sl = 0; sl < ns; ++sl) issue_unit(sl, u, n, i0);
                for (int j = 0; j < ns || j - kLag < ns_next; ++j) {
                    if (j < ns) issue_unit(j, G, n, i0);
                    if (j - kLag >= 0 && j - kLag < ns_next) issue_unit(j - kLag, 0, n + 1, i0 + NS);
                }
            }
#endif
        }
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(C::REGS_EPI));
        // ================= epilogue group sl: warps 4 + WPS sl ..; thread = QW columns of one row of the slot's tiles
        constexpr int kNBatch = C::NCH / kNB;
        const int sl = (warp - 4) / C::WPS;
        const int e = (warp - 4) % C::WPS;
        const int gq = warp & 3;                          // TMEM lane quarter
        const int ch = e >> 2;                            // column group: columns [ch QW, ch QW + QW)
        const int r = gq * 32 + lane;                     // row of the tile
        const int gtid = e * 32 + lane;
        const uint32_t t_row = tmem + ((uint32_t)(gq * 32) << 16) + (uint32_t)(sl * 128 + ch * C::QW);
        const uint32_t aA = sbase + (uint32_t)(C::OFF_A + sl * C::A_BYTES);
        const float4* s_rows = reinterpret_cast<const float4*>(smem + C::OFF_ROWS + sl * 16 * kRows);
        float* b1s = reinterpret_cast<float*>(smem + C::OFF_B1S + sl * 4 * H);
        float* part = reinterpret_cast<float*>(smem + C::OFF_PART + sl * 4 * C::COLG * kRows);
        const bool leader = e == 0 && lane == 0;
        auto group_sync = [&]() { named_bar_sync(1 + sl, 32 * C::WPS); };
        auto issue_rows = [&](long long i) {   // query rows of local tile i -> this slot's row buffer (TMA engine)
            if (FUSE || !leader || i >= n_my) return;   // FUSE: the rollout warps write the rows
            const long long r0 = row0_of(i);
            const long long nv = min((long long)kRows, n_rows - r0);
            mbar_expect_tx(bar(BAR_ROWS + sl), (uint32_t)(16 * nv));
            bulk_g2s(sbase + (uint32_t)(C::OFF_ROWS + sl * 16 * kRows), rows + r0, (uint32_t)(16 * nv),
                     bar(BAR_ROWS + sl));
        };
        // 16 activations (bf16x2 x 8) of neurons j0..j0+15 -> the slot's A tile (SW128 K-major)
        auto store_a = [&](int j0, const uint32_t* packed) {
            const int kc = j0 / 64, c0 = (j0 % 64) / 8;
            const uint32_t rb = aA + (uint32_t)(kc * (kRows * 128) + r * 128);
#ifdef H128_NO_STORE_A
            if (p.K != -12345) return;   // timing probe only (wrong results): the epilogue's A stores skipped
#endif
#pragma unroll
            for (int c = 0; c < 2; ++c)
                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(rb + (uint32_t)((((c0 + c) ^ (r & 7))) * 16)),
                             "r"(packed[4 * c]), "r"(packed[4 * c + 1]), "r"(packed[4 * c + 2]), "r"(packed[4 * c + 3])
                             : "memory");
        };
        // layer-1 operand row of local tile i (exact bf16 splits, see the header) -> A; returns |v| of the row
        const bool tracer = leader;   // trace roles 1..4 = slots 0..3
        auto build_a1 = [&](long long i) -> float {
            if (tracer) H_TRACE(1 + sl, 6, 0, i);
            const uint32_t rnd = (uint32_t)((i - sl) / NS);
            mbar_wait(bar(BAR_ROWS + sl), rnd & 1u);
            const long long row = row0_of(i) + r;
            const float4 q = row < n_rows ? s_rows[r] : make_float4(0.f, 0.f, 0.f, 0.f);
            uint32_t col[C::K1];
#pragma unroll
            for (int k = 0; k < C::K1; ++k) col[k] = 0u;
            const float pv[3] = {q.x, q.y, q.z};
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const uint32_t h = bf16_bits(pv[c]);
                const float r1 = pv[c] - bf16_val(h);
                const uint32_t m = bf16_bits(r1);
                const uint32_t lo = bf16_bits(r1 - bf16_val(m));
                // terms t = 0..5: x_h w_h, x_h w_m, x_m w_h, x_h w_l, x_m w_m, x_l w_h
                col[0 + c] = h; col[3 + c] = h; col[6 + c] = m; col[9 + c] = h; col[12 + c] = m; col[15 + c] = lo;
            }
            if constexpr (PEB > 0) {
                // PE(p) = [sin(2^b pi p), cos(2^b pi p)]_{b < PEB} after p (reading E1; sincospif: exact range
                // reduction), each feature split f = f_h + f_l: columns f_h w_h, f_h w_l, f_l w_h
#pragma unroll
                for (int bnd = 0; bnd < PEB; ++bnd) {
                    const float sc = (float)(1 << bnd);
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        float sv, cv;
                        sincospif(pv[c] * sc, &sv, &cv);
                        const int js = 6 * bnd + c, jc = 6 * bnd + 3 + c;
                        const uint32_t sh = bf16_bits(sv), ch = bf16_bits(cv);
                        const uint32_t sl2 = bf16_bits(sv - bf16_val(sh)), cl2 = bf16_bits(cv - bf16_val(ch));
                        col[18 + 3 * js] = sh; col[18 + 3 * js + 1] = sh; col[18 + 3 * js + 2] = sl2;
                        col[18 + 3 * jc] = ch; col[18 + 3 * jc + 1] = ch; col[18 + 3 * jc + 2] = cl2;
                    }
                }
            }
            const uint32_t rb = aA + (uint32_t)((r / 8) * (C::K1C * 128) + (r % 8) * 16);
            // the COLG threads of a row each store their share of the row's K cores
#pragma unroll
            for (int kc = 0; kc < C::K1C; ++kc)
                if (kc / (C::K1C / C::COLG) == ch)
                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(rb + (uint32_t)(kc * 128)),
                             "r"(col[8 * kc] | (col[8 * kc + 1] << 16)), "r"(col[8 * kc + 2] | (col[8 * kc + 3] << 16)),
                             "r"(col[8 * kc + 4] | (col[8 * kc + 5] << 16)), "r"(col[8 * kc + 6] | (col[8 * kc + 7] << 16))
                             : "memory");
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes -> MMA operand reads
            __syncwarp();
            if (lane == 0) mbar_arrive_local(bar(BAR_SA1 + sl));
            group_sync();                 // every warp of the group has read the row buffer
            if (FUSE && leader) mbar_arrive_local(bar(BAR_RFREE + sl));
            issue_rows(i + NS);
            if (tracer) H_TRACE(1 + sl, 7, 0, i);
            return q.w;
        };
        // D of the slot in batches of kNB x 16 columns: one tcgen05.wait::ld per batch (its cost, not the load,
        // dominates a 16-column chunk), the next batch in flight while this one is computed
        auto load_batch = [&](int kb, uint32_t (&a)[kNB][kCW]) {
#pragma unroll
            for (int cb = 0; cb < kNB; ++cb) tmem_ld16(t_row + (uint32_t)((kb * kNB + cb) * kCW), a[cb]);
        };
        auto wait_batch = [&](uint32_t (&a)[kNB][kCW]) {
            tmem_wait_ld_regs(a[0]);
#pragma unroll
            for (int cb = 1; cb < kNB; ++cb) tmem_tie_regs(a[cb]);
        };
        auto arrive_sched = [&](int b) {   // all of this warp's tcgen05 / shared accesses done -> issuer
            __syncwarp();
            if (lane == 0) mbar_arrive_local(bar(b + sl));
        };

        uint32_t mma_cnt = 0;
        long long staged = -1;             // controller whose b1' is in b1s
        float nv = 0.f;                    // |v| of this thread's row of the current tile
        if constexpr (!C::HELPER) {
            issue_rows(sl);
            if (sl < n_my) nv = build_a1(sl);
        }
        const float bo = __ldg(b_out);
        for (long long i = sl; i < n_my; i += NS) {
            const long long row0 = row0_of(i);
            // ---- layer-1 epilogue: x = D + b1' (per controller, x kPre), act, bf16 -> A of the first GEMM
            {
                const long long lo = states_mode ? ctrl_of(min(row0, n_rows - 1)) : ctrl_fixed;
                if (lo != staged) {   // uniform across the group
                    group_sync();
                    for (int j = gtid; j < H; j += 32 * C::WPS) b1s[j] = lo < p.n_ctrl ? b1f[(size_t)lo * H + j] * kP : 0.f;
                    staged = lo;
                    group_sync();
                }
                const long long row = row0 + r;
                const long long bb = states_mode ? ctrl_of(min(row, n_rows - 1)) : ctrl_fixed;
                const float* bfar = bb != lo ? b1f + (size_t)bb * H : nullptr;   // rows of a later controller
                const bool any_far = __any_sync(0xFFFFFFFFu, bfar != nullptr);
                if (tracer) H_TRACE(1 + sl, 3, 0, i);
                mbar_wait(bar(BAR_MMA + sl), (mma_cnt++) & 1u);
                tc_fence_after();
                if (tracer) H_TRACE(1 + sl, 4, 0, i);
                uint32_t accb[2][kNB][kCW];
                load_batch(0, accb[0]);
#pragma unroll
                for (int kb = 0; kb < kNBatch; ++kb) {
                    wait_batch(accb[kb & 1]);
                    if (kb + 1 < kNBatch) load_batch(kb + 1, accb[(kb + 1) & 1]);
#pragma unroll
                    for (int cb = 0; cb < kNB; ++cb) {
                    const int k = kb * kNB + cb;
                    uint32_t(&acc)[kCW] = accb[kb & 1][cb];
                    uint32_t packed[kCW / 2];
                    const int j0 = ch * C::QW + k * kCW;
                    if (!any_far) {   // every row of the tile belongs to the staged controller (the common case)
#pragma unroll
                        for (int i2 = 0; i2 < kCW; i2 += 4) {
#ifdef H128_NO_BIAS_LDS
                            const float4 bv = make_float4(b1s[0], b1s[1], b1s[2], b1s[3]);   // timing experiment only
#else
                            const float4 bv = *reinterpret_cast<const float4*>(b1s + j0 + i2);
#endif
                            const float2 x0 = ffma2(make_float2(__uint_as_float(acc[i2]), __uint_as_float(acc[i2 + 1])),
                                                    make_float2(1.f, 1.f), make_float2(bv.x, bv.y));
                            const float2 x1 = ffma2(make_float2(__uint_as_float(acc[i2 + 2]), __uint_as_float(acc[i2 + 3])),
                                                    make_float2(1.f, 1.f), make_float2(bv.z, bv.w));
                            packed[i2 / 2] = act_pack<ACT>(x0.x, x0.y);
                            packed[i2 / 2 + 1] = act_pack<ACT>(x1.x, x1.y);
                        }
                    } else {          // rare: the tile crosses into a later controller
#pragma unroll
                        for (int i2 = 0; i2 < kCW; i2 += 2) {
                            const int j = j0 + i2;
                            const float b0 = bfar ? __ldg(bfar + j) * kP : b1s[j];
                            const float b1 = bfar ? __ldg(bfar + j + 1) * kP : b1s[j + 1];
                            packed[i2 / 2] = act_pack<ACT>(__uint_as_float(acc[i2]) + b0, __uint_as_float(acc[i2 + 1]) + b1);
                        }
                    }
                    store_a(ch * C::QW + k * kCW, packed);
                    }
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                tc_fence_before();
                arrive_sched(BAR_AREADY);
                if (tracer) H_TRACE(1 + sl, 5, 0, i);
            }
            // ---- hidden GEMM epilogues; the last one computes the output layer and the stage term
            float2 sdot = make_float2(0.f, 0.f);
            float nv_next = 0.f;
#pragma unroll 1
            for (int l = 0; l < G; ++l) {
                const bool last = l == G - 1;
                if (tracer) H_TRACE(1 + sl, 3, l + 1, i);
                mbar_wait(bar(BAR_MMA + sl), (mma_cnt++) & 1u);
                tc_fence_after();
                if (tracer) H_TRACE(1 + sl, 4, l + 1, i);
                if (!C::HELPER && last && i + NS < n_my) nv_next = build_a1(i + NS);   // the last GEMM has read A: next layer 1
                uint32_t accb[2][kNB][kCW];
                load_batch(0, accb[0]);
#pragma unroll
                for (int kb = 0; kb < kNBatch; ++kb) {
                    wait_batch(accb[kb & 1]);
                    if (kb + 1 < kNBatch) {
                        load_batch(kb + 1, accb[(kb + 1) & 1]);
                    } else if (last) {   // D of the slot may be overwritten (next tile's layer 1)
                        tc_fence_before();
                        arrive_sched(BAR_DFREE);
                    }
#pragma unroll
                    for (int cb = 0; cb < kNB; ++cb) {
                    const int k = kb * kNB + cb;
                    uint32_t(&acc)[kCW] = accb[kb & 1][cb];
                    if (!last) {
                        uint32_t packed[kCW / 2];
#pragma unroll
                        for (int i2 = 0; i2 < kCW; i2 += 2)
                            packed[i2 / 2] = act_pack<ACT>(__uint_as_float(acc[i2]), __uint_as_float(acc[i2 + 1]));
                        store_a(ch * C::QW + k * kCW, packed);
                    } else {
#pragma unroll
                        for (int i2 = 0; i2 < kCW; i2 += 4) {
#ifdef H128_NO_WOUT_LDS
                            const float4 wv = make_float4(0.01f * i2, 0.02f, 0.03f, 0.04f * k);   // timing experiment only
#else
                            const float4 wv = *reinterpret_cast<const float4*>(s_wo + ch * C::QW + k * kCW + i2);
#endif
                            const uint32_t p0 = act_pack<ACT>(__uint_as_float(acc[i2]), __uint_as_float(acc[i2 + 1]));
                            const uint32_t p1 = act_pack<ACT>(__uint_as_float(acc[i2 + 2]), __uint_as_float(acc[i2 + 3]));
                            sdot = ffma2(make_float2(__uint_as_float(p0 << 16), __uint_as_float(p0 & 0xFFFF0000u)),
                                         make_float2(wv.x, wv.y), sdot);
                            sdot = ffma2(make_float2(__uint_as_float(p1 << 16), __uint_as_float(p1 & 0xFFFF0000u)),
                                         make_float2(wv.z, wv.w), sdot);
                        }
                    }
                    }
                }
                if (!last) {
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    tc_fence_before();
                    arrive_sched(BAR_AREADY);
                }
                if (tracer) H_TRACE(1 + sl, 5, l + 1, i);
            }
            if constexpr (C::HELPER)   // |v| of this row, kept by the layer-1 builder
                nv = reinterpret_cast<const float*>(smem + C::OFF_NV + (sl * 2 + (int)(((i - sl) / NS) & 1)) * 4 * kRows)[r];
            // ---- output of this tile: combine the column groups' partial dots, FD pair (adjacent lanes), term
            float sv = sdot.x + sdot.y;
            if constexpr (C::COLG > 1) {
                part[ch * kRows + r] = sv;
                group_sync();
                sv = bo;
#pragma unroll
                for (int q2 = 0; q2 < C::COLG; ++q2) sv += part[q2 * kRows + r];
            } else {
                sv += bo;
            }
            const long long row = row0 + r;
            if (ch == 0 && row < n_rows && sdf_out) sdf_out[row] = sv;
            if (ch == 0 && states_mode) {
                if (p.rps == 2) {
                    const float s1 = __shfl_xor_sync(0xFFFFFFFFu, sv, 1);
                    const float term = p.w_sdf * __expf(fminf(-sv * p.inv_sdf_scale, p.sdf_exp_max)) -
                                       p.w_guide * nv * (s1 - sv) * p.inv_fd_h;
                    if ((lane & 1) == 0 && row < n_rows) terms[row >> 1] = term;
                } else {
                    const float term = p.model == MPPI_MODEL_PAPER
                                           ? p.q_sdf * fmaxf(p.d_safe - sv, 0.f)   // Eq. 8 hinge
                                           : p.w_sdf * __expf(fminf(-sv * p.inv_sdf_scale, p.sdf_exp_max));
                    if (row < n_rows) terms[row] = term;
                }
            }
            if constexpr (C::COLG > 1) group_sync();   // part[] is reused by the next tile
            nv = nv_next;
        }
    }
    // ---- teardown
    __syncwarp();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::TMEM_COLS));
}

template <int G, int ACT, int PEB, bool FUSE>
cudaError_t launch_t(const Params& p, const Buffers& b, const float4* rows, long long n_rows, int ctrl_fixed,
                     float* sdf_out, bool states_mode, cudaStream_t s) {
    using C = Cfg<G, PEB, FUSE>;
    constexpr int kMaxDev = 64;
    static int n_ctas[kMaxDev] = {};   // persistent grid per device (one CTA per SM); 0 = not set up
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDev) return cudaErrorInvalidDevice;
    if (n_ctas[dev] == 0) {
        cudaError_t e = cudaFuncSetAttribute(k_mlp_h128<G, ACT, PEB, FUSE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             C::SMEM);
        if (e != cudaSuccess) return e;
        int n_sm = 0, per_sm = 0;
        cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_mlp_h128<G, ACT, PEB, FUSE>, C::THREADS, C::SMEM);
        if (e != cudaSuccess) return e;
        if (per_sm < 1) return cudaErrorInvalidConfiguration;
        n_ctas[dev] = n_sm;
        if (getenv("MPPI_VERBOSE"))
            fprintf(stderr, "[mppi] k_mlp_h128<G=%d,ACT=%d,PEB=%d,FUSE=%d> dev %d: %d CTAs x %d threads, %d tiles in flight, smem %d B\n",
                    G, ACT, PEB, (int)FUSE, dev, n_sm, C::THREADS, C::NSLOT, C::SMEM);
    }
    const long long units = FUSE ? (long long)p.n_ctrl * (p.K / 64) : (n_rows + kRows - 1) / kRows;
    if (units == 0) return cudaSuccess;
    const unsigned grid = (unsigned)(units < n_ctas[dev] ? units : n_ctas[dev]);
    k_mlp_h128<G, ACT, PEB, FUSE><<<grid, C::THREADS, C::SMEM, s>>>(p, rows, n_rows, ctrl_fixed, states_mode ? 1 : 0,
                                                                      (const uint8_t*)b.hid_wbf, b.w_out, b.b_out, b.b1f,
                                                                      sdf_out, b.terms, b);
    return cudaGetLastError();
}

}  // namespace h128

int mlp_h128_trace_copy(unsigned long long* host, int max_entries) {
#ifdef MPPI_TC_TRACE
    const int n = 2 * 5 * h128::kTraceCap;
    if (max_entries < n) return 0;
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(host, h128::g_h128_trace, sizeof(unsigned long long) * n);
    static unsigned long long zeros[2 * 5 * h128::kTraceCap];
    cudaMemcpyToSymbol(h128::g_h128_trace, zeros, sizeof(zeros));
    return n;
#else
    (void)host;
    (void)max_entries;
    return 0;
#endif
}

bool mlp_h128_supported(int G, int pe_bands) { return G >= 1 && G <= 3 && (pe_bands == 0 || pe_bands == 4); }

// Image bytes: the hidden part (same layout as mlp_tc_pack_weights at H = 128) + the layer-1 B operand.
size_t mlp_h128_image_bytes(int G, int pe_bands) {
    const int k1 = ((18 + 18 * pe_bands) + 15) / 16 * 16;
    return (size_t)G * 128 * 128 * 2 + (size_t)G * 128 * 32 + (size_t)128 * k1 * 2;
}

// Layer-1 B operand (appended after the hidden image): row n = neuron, K-major without swizzle
// ([n / 8][K core][n % 8][8 bf16]); the columns pair with the A columns the kernel builds:
// position terms t = 0..5 per coordinate c (column 3 t + c): w_h, w_m, w_h, w_l, w_m, w_h; PE feature j
// (column 18 + 3 j + t): w_h, w_l, w_h. Weights are scaled by kPre (x1/2 for SiLU: exact).
// w1pos: [128][3 + 6 pe_bands] fp32 (the position columns of W1, nn.Linear order).
void mlp_h128_pack_l1(int pe_bands, int act, const float* w1pos, uint8_t* out) {
    const int npe = 3 + 6 * pe_bands;
    const int k1 = ((18 + 18 * pe_bands) + 15) / 16 * 16, k1c = k1 / 8;
    const float kp = act == MPPI_ACT_SILU ? 0.5f : 1.0f;
    auto rne = [](float v) {
        uint32_t u;
        std::memcpy(&u, &v, 4);
        u = (u + 0x7FFFu + ((u >> 16) & 1u)) & 0xFFFF0000u;
        float r;
        std::memcpy(&r, &u, 4);
        return r;
    };
    auto bits = [](float v) {
        uint32_t u;
        std::memcpy(&u, &v, 4);
        return (uint16_t)(u >> 16);
    };
    std::memset(out, 0, (size_t)128 * k1 * 2);
    auto put = [&](int n, int k, float v) {
        const uint16_t b = bits(v);
        std::memcpy(out + (size_t)(n / 8) * (k1c * 128) + (size_t)(k / 8) * 128 + (size_t)(n % 8) * 16 + (size_t)(k % 8) * 2,
                    &b, 2);
    };
    for (int n = 0; n < 128; ++n) {
        for (int f = 0; f < npe; ++f) {
            const float w = w1pos[(size_t)n * npe + f] * kp;
            const float wh = rne(w), wm = rne(w - wh), wl = rne(w - wh - wm);
            if (f < 3) {
                const float part[6] = {wh, wm, wh, wl, wm, wh};
                for (int t = 0; t < 6; ++t) put(n, 3 * t + f, part[t]);
            } else {
                const int j = f - 3;
                const float wlo = rne(w - wh);
                put(n, 18 + 3 * j, wh);
                put(n, 18 + 3 * j + 1, wlo);
                put(n, 18 + 3 * j + 2, wh);
            }
        }
    }
}

cudaError_t launch_mlp_h128(const Params& p, const Buffers& b, const float4* rows, long long n_rows, int ctrl_fixed,
                            float* sdf_out, bool states_mode, cudaStream_t s, bool fuse) {
#define MPPI_H128_CASE(GG, AA)                                                                                  \
    if (p.n_gemm == GG && p.act == AA) {                                                                        \
        if (fuse) return h128::launch_t<GG, AA, 0, true>(p, b, rows, n_rows, ctrl_fixed, sdf_out, states_mode, s); \
        return p.pe_bands == 4 ? h128::launch_t<GG, AA, 4, false>(p, b, rows, n_rows, ctrl_fixed, sdf_out, states_mode, s) \
                               : h128::launch_t<GG, AA, 0, false>(p, b, rows, n_rows, ctrl_fixed, sdf_out, states_mode, s); \
    }
#ifdef MPPI_TC_QUICK
    MPPI_H128_CASE(2, 1)
#else
    MPPI_H128_CASE(1, 0) MPPI_H128_CASE(1, 1) MPPI_H128_CASE(1, 2)
    MPPI_H128_CASE(2, 0) MPPI_H128_CASE(2, 1) MPPI_H128_CASE(2, 2)
    MPPI_H128_CASE(3, 0) MPPI_H128_CASE(3, 1) MPPI_H128_CASE(3, 2)
#endif
#undef MPPI_H128_CASE
    return cudaErrorInvalidValue;
}

}  // namespace mppi
