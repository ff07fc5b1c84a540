// Fused Gate-SDF MLP on 5th-generation tensor cores (sm_100a): tcgen05.mma with the activation
// operand A and the accumulator D both in tensor memory (TMEM), the weights B resident in shared
// memory (loaded once per persistent CTA by cp.async.bulk, i.e. the TMA engine), bias + activation +
// bf16 pack in the epilogue, the output layer and the finite-difference guidance combine fused into
// the last epilogue.
//
// Method (PAPER.md:168 "query the decoder for every predicted position", :40 latent concatenated with
// every sampled state, folded here into the per-frame bias b1' = W1[:,3:] z + b1; Eq. 10
// with the BASELINE configs[1] terms 50 exp(-s/0.1) - 0.5 grad(s).v, reading R12):
//   a1 = bf16(act(W1[:, :3] p_c + b1'))                     layer 1 on CUDA cores (fp32), K = 3
//   a_l = bf16(act(W_l a_{l-1} + b_l)), l = 2..n_hidden     tensor cores, bf16 x bf16 -> fp32 (TMEM)
//   s = w_out . a_L + b_out                                 fused into the last epilogue (fp32)
//   term = w_sdf exp(min(-s/scale, emax)) - w_guide |v| (s(p_c + h d) - s(p_c)) / h
//
// Work unit: a tile of 128 query rows per CTA (64 states x {p_c, p_c + h d} with guidance).
// H = 256 (configs[2,3]) runs as CTA pairs (cluster of 2, tcgen05 cta_group::2, MMA M = 256): each
// CTA keeps HALF of every weight matrix resident (192 KB for 3 GEMM layers) and its own 128 rows in
// TMEM; only the pair's leader issues MMAs. H = 128 (configs[1,4]) runs one CTA per tile (cta_group::1,
// M = 128) with all weights resident (<= 96 KB).
// Two tiles in flight per CTA (TMEM slots X, Y: D = 128 fp32 columns + A = H/2 bf16x2 columns each).
// Per layer the MMA work is one full-K unit per N-half h (N = 128) and slot, issued X(h0) Y(h0) X(h1)
// Y(h1): the epilogue of one slot overlaps the MMAs of the other. D is released as soon as the epilogue
// has loaded it; the N-half-0 activations wait in registers until the layer's last MMA has read A. At
// H = 256 the next layer's N-half-0 unit is issued in two K halves: K-half 0 as soon as those kept
// activations are stored (and D is free), K-half 1 after the N-half-1 epilogue.
// H = 128: layer 1 writes a shared-memory A tile and the first GEMM runs as SS MMAs, so each slot
// computes layer 1 of its next tile while its last GEMM runs.
// Warp roles: warp 0 = TMEM allocator + MMA issuer (the leader CTA; H = 256: the whole warp, one
// elected lane issues); warp 1 = weight loader; warps 4..19 = epilogue, two groups of 8 (one per
// slot; warp w owns TMEM lanes 32 (w%4)..+31 and one column half of a unit).
#include <cuda_bf16.h>
#include <stdint.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "../../include/mppi.h"
#include "mppi_internal.cuh"
#include "rollout_dev.cuh"
#include "tc_ptx.cuh"

namespace mppi {
namespace tc {

#ifdef MPPI_TC_TRACE
// Debug-only timeline (clock64 per SM) of the first CTAs; each (block, role) appends to its own slice,
// no atomics: code = [11:8] event, [7:6] layer, [5] half, [4] chunk, [3:0] tile & 15.
constexpr int kTraceCap = 2048;
__device__ unsigned long long g_tc_trace[4][3][kTraceCap];
#define TC_TRACE(role, ev, l, h, c, t)                                                                        \
    do {                                                                                                      \
        if (blockIdx.x < 4 && trace_n < kTraceCap) {                                                          \
            const unsigned long long _code = ((ev) << 8) | (((l) & 3) << 6) | (((h) & 1) << 5) |              \
                                             (((c) & 1) << 4) | ((t) & 15);                                    \
            g_tc_trace[blockIdx.x][role][trace_n++] = (_code << 48) | ((unsigned long long)clock64() & 0xFFFFFFFFFFFFull); \
        }                                                                                                     \
    } while (0)
#define TC_TRACE_DECL int trace_n = 0
#else
#define TC_TRACE(role, ev, l, h, c, t) \
    do {                               \
    } while (0)
#define TC_TRACE_DECL
#endif

constexpr int kEpiWarps = 16;   // 4 per SMSP
constexpr int kEpiWarp0 = 4;    // epilogue warp w reads TMEM lanes 32 (w % 4)
constexpr int kThreads = 32 * (kEpiWarp0 + kEpiWarps);   // warp 0 MMA, warp 1 weight loader, 2-3 idle
// setmaxnreg split of the CTA register pool (640 threads launched at 96 registers): warpgroup 0
// (issuer, loader) 32, the four epilogue warpgroups 112: 128 x 32 + 512 x 112 = 640 x 96
#ifndef MPPI_REGS_CTL
#define MPPI_REGS_CTL 56   // the issuer spills below ~56 (measured c3 -1.2% vs 32)
#endif
constexpr int kRegsCtl = MPPI_REGS_CTL, kRegsEpi = ((96 * 640 - 128 * MPPI_REGS_CTL) / 512) / 8 * 8;
constexpr int kCW = 16;         // TMEM columns per epilogue load
#ifndef MPPI_ISSUER_WARP
#define MPPI_ISSUER_WARP -1   // -1: per configuration (see the issuer); 0 / 1 force lane 0 / the warp form
#endif
#ifndef MPPI_EPI_PIPE
#define MPPI_EPI_PIPE -1   // -1: per configuration (see the epilogue); 0 / 1 force off / on
#endif
#ifndef MPPI_EPI_ALL
#define MPPI_EPI_ALL -1   // -1: per configuration (H = 256 on); 0 / 1 force off / on
#endif
#ifndef MPPI_SPLITK
#define MPPI_SPLITK 1
#endif
#ifndef MPPI_L1_SMEM
#define MPPI_L1_SMEM 1
#endif
#ifndef MPPI_L1_MMA
#define MPPI_L1_MMA 0   // H = 256: layer 1 as a K = 32 MMA on exact bf16 splits (see Cfg::L1M; A/B: +28% at configs[2])
#endif
#ifndef MPPI_L1M_ALL
#define MPPI_L1M_ALL 0   // L1M: the GEMM layers' epilogues load the whole D share at once (kAll), layer 1 pipelined
#endif
#ifndef MPPI_DESC_ADD
#define MPPI_DESC_ADD -1   // TS-form K-step B descriptors by one 32-bit add on the address field: -1 = with PE only
                          // (A/B: configs[2]+PE -1.5%, configs[2] +0.3%, configs[3] -0.2%), 0 / 1 = off / on
#endif
#ifndef MPPI_FUSE_CTL
#define MPPI_FUSE_CTL 80   // FUSE: registers of the control warpgroup (the rollout producers); the epilogue gets the rest
#endif
#ifndef MPPI_BIAS_EPI
#define MPPI_BIAS_EPI 0   // 1: hidden biases added in the epilogue (FFMA2) instead of one K = 16 ones x bias MMA per unit
#endif
#ifndef MPPI_PE_MMA
#define MPPI_PE_MMA 1   // H = 256 with PE: the 27 position features as a K = 96 exact-split MMA (Cfg::L1PE)
#endif
constexpr int kTileRows = 128;

// ------------------------------------------------------------------ configuration
template <int H, int G, int PEB = 0>
struct Cfg {
    static constexpr int NPE = 3 + 6 * PEB;                  // layer-1 position features (raw p + PE bands)
    static constexpr int CG = H == 256 ? 2 : 1;              // CTAs per MMA (cta_group)
    // A TS-form MMA (A in TMEM) streams 4 KB of A per K=16 step per CTA (M = 128): below N = 128 it runs
    // at the A-read rate, not the math rate, so units are N = 128 (two per layer for H = 256, one for 128)
    static constexpr int NH = H / 128;                       // MMA units (N blocks) per GEMM layer
    static constexpr int UN = H / NH;                        // N of one unit (128)
    static constexpr int RB = UN / CG;                       // weight rows (N) of a unit held per CTA
    static constexpr int UNIT_BYTES = RB * H * 2;            // bf16 B block of one unit in one CTA
    static constexpr int W_BYTES = G * NH * UNIT_BYTES;      // resident weights per CTA
    static constexpr int A_OFF = UN;                         // per slot: D [0, UN) fp32, A [UN, UN + H/2) bf16x2
    static constexpr int SLOT_COLS = 256;
    static constexpr int NSLOT = 512 / SLOT_COLS;            // tiles in flight per CTA: 2
    static constexpr int TMEM_COLS = NSLOT * SLOT_COLS;      // = 512
    static constexpr int GW = kEpiWarps / NSLOT;             // epilogue warps per slot group (8)
    static constexpr int COLG = GW / 4;                      // column groups per TMEM lane quarter in a group
    // H = 256: layer 1 runs on the tensor cores like the hidden layers (two N-half units of K = 32: the exact
    // three-part bf16 splits of p_c and W1p, six cross products per coordinate, as kernel_mlp_h128.cu), so its
    // epilogue is a GEMM epilogue (D + b1', act, pack) instead of a CUDA-core 3-wide dot per neuron pair
    static constexpr bool L1M = CG == 2 && (PEB == 0 ? MPPI_L1_MMA : MPPI_PE_MMA);
    // L1PE (H = 256 with PE, reading E2): layer 1 is one MMA unit per N-half over K1 = 96 operand columns -- raw p
    // in the six-product split (18), each of the 24 sin/cos features as f_h w_h, f_h w_l, f_l w_h (72), 6 zero.
    // Its B operand (24 KB per CTA) takes the shared memory of the bias MMA images and the row buffers: the
    // hidden biases are added in the epilogue (FFMA2) and each thread loads its query row itself, one tile ahead.
    static constexpr bool L1PE = L1M && PEB > 0;
    static constexpr int K1_USED = 18 + 18 * PEB;                     // layer-1 operand columns in use
    static constexpr int K1 = (K1_USED + 15) / 16 * 16;              // 32, or 96 with 4 PE bands
    static constexpr int K1S = K1 / 16;                              // K = 16 MMA steps of layer 1
    static constexpr bool BIAS_MMA = !MPPI_BIAS_EPI;                 // hidden biases by a ones x bias MMA
    // L1PE: the bias operands in compact form, built at kernel start: per layer l an 8-row ones tile with the ones
    // in K columns 2l, 2l+1, read with SBO = 0 (every 8-row group the same rows), and per N-half ONE bias image
    // holding all layers, b_hi / b_lo of layer l in columns 2l, 2l+1 -- 4.8 KB instead of 16 KB (the 24 KB layer-1
    // B operand needs the rest). Biases in the epilogue instead (MPPI_BIAS_EPI) measured +7% / +10.6% at H = 256.
    static constexpr bool BIAS_COMPACT = L1PE && BIAS_MMA;
    static constexpr int NROWBUF = L1PE ? 0 : L1M ? NSLOT : 2 * NSLOT;   // query-row buffers (L1M: |v| in registers)
    static constexpr int QW = UN / COLG;                     // epilogue columns per warp per unit
    static constexpr int NCH = QW / kCW;                     // TMEM loads per warp per unit
    static constexpr int MMA_M = 128 * CG;
    // H = 256: the first unit of a layer (N-half 0) is issued in two K halves. K-half 0 of A (the previous
    // layer's N-half 0, kept in registers) is written as soon as the previous layer's last MMA has read A,
    // so those 8 MMAs start when D is free instead of after the whole epilogue of N-half 1.
    static constexpr bool SPLITK = NH == 2 && MPPI_SPLITK;
    // H = 128 (one CTA per tile, weights 64 KB): layer 1 writes its activations to a shared-memory A tile
    // per slot and the first GEMM runs as SS MMAs, so a slot computes layer 1 of its NEXT tile while it
    // waits for the last GEMM of the current one (layer 1 leaves the tile's MMA <-> epilogue chain)
    static constexpr bool A1S = CG == 1 && MPPI_L1_SMEM;
    static_assert(A_OFF + H / 2 <= SLOT_COLS && QW % kCW == 0 && RB % 8 == 0, "TMEM / unit layout");
    // smem carve-up (offsets from the 1024-aligned base)
    // hidden-layer biases enter the accumulator through one extra K = 16 MMA per unit: A = a constant
    // "ones" tile [128 rows][1, 1, 0 x 14], B = [b_hi, b_lo, 0 x 14] per output row (bf16 split of the
    // kP-scaled fp32 bias), both no-swizzle K-major -- so the epilogue adds nothing
    static constexpr int BIAS_UNIT = RB * 32;                        // RB rows x 16 bf16
    static constexpr int IMG_BYTES = W_BYTES + G * NH * BIAS_UNIT;   // weight image per CTA (rank), global stride
    static constexpr int BIAS_BYTES = BIAS_MMA ? (BIAS_COMPACT ? NH : G * NH) * BIAS_UNIT : 0;   // bias images (smem)
    static constexpr int OFF_BIAS = W_BYTES;
    static constexpr int OFF_ONES = OFF_BIAS + BIAS_BYTES;           // [128 rows][16] bf16 ones tile (compact: [G][8][16])
    static constexpr int ONES_BYTES = BIAS_COMPACT ? G * 256 : kTileRows * 32;
    static constexpr int OFF_HB = OFF_ONES + (BIAS_MMA ? ONES_BYTES : 0);   // !BIAS_MMA: [G][H] kP b (fp32)
    static constexpr int OFF_WO = OFF_HB + (BIAS_MMA ? 0 : 4 * G * H);         // [H] output weights
    static constexpr int OFF_W1XY = OFF_WO + 4 * H;                  // [H/2] (w0x, w1x, w0y, w1y) layer-1 positions, scaled
    static constexpr int OFF_W1Z = OFF_W1XY + (L1M ? 0 : 8 * H);     // [H/2] (w0z, w1z)
    static constexpr int BL1_TILE = RB * 32;                         // L1M: per (unit, K step) RB rows x 16 bf16
    static constexpr int OFF_BL1 = OFF_W1Z + (L1M ? 0 : 4 * H);      // L1M: [NH][2 K steps] no-swizzle K-major
    static constexpr int OFF_B1 = OFF_BL1 + (L1M ? NH * K1S * BL1_TILE : 0);   // [NSLOT groups][H] folded bias b1', scaled
    // PEB > 0: [H/2][NPE] float2 PE weights (scaled) in shared memory at H = 128; at H = 256 the resident hidden
    // weights leave no room, so layer 1 reads the same pair-major image from global memory (L1-cached,
    // warp-uniform addresses)
    static constexpr bool PE_SMEM = PEB > 0 && CG == 1;
    static constexpr int OFF_PE = OFF_B1 + NSLOT * 4 * H;
    static constexpr int OFF_PART = OFF_PE + (PE_SMEM ? (H / 2) * NPE * 8 : 0);   // [NSLOT][COLG][128] partial dots
    static constexpr int OFF_ROWS = OFF_PART + 4 * NSLOT * COLG * kTileRows;  // [NROWBUF][128] float4 query rows
    static constexpr int OFF_SA = A1S ? (OFF_ROWS + NROWBUF * 16 * kTileRows + 1023) / 1024 * 1024 : 0;
    static constexpr int SA_BYTES = kTileRows * H * 2;               // [K/64][128 rows][128 B] SW128 K-major
    static constexpr int OFF_BAR = A1S ? OFF_SA + NSLOT * SA_BYTES : OFF_ROWS + NROWBUF * 16 * kTileRows;
    static constexpr int OFF_TMEM = OFF_BAR + 8 * (L1PE ? 28 : 32);   // L1PE: no FUSE barriers (<= BAR_AK0 + 1)
    static constexpr int SMEM = 1024 + OFF_TMEM + 16;
    static_assert(SMEM <= 232448, "shared memory budget");
};

// Barrier slots (8 B each): per tile slot (up to 4) and per query-row buffer (up to 8)
enum { BAR_AREADY = 0 /*[slots]*/, BAR_DFREE = 4 /*[slots]*/, BAR_MMA = 8 /*[slots]*/, BAR_WLOCAL = 12,
       BAR_WREADY = 13, BAR_ROWS = 14 /*[row buffers]*/, BAR_SREADY = 22 /*[slots]: smem layer-1 A tile*/,
       BAR_AK0 = 26 /*[slots]: K-half 0 of A written (SPLITK)*/, BAR_RFREE = 28 /*[row buffers]: FUSE, consumed*/ };

// H = 256 with positional encoding: the pair-major layer-1 weights travel as a kernel parameter (27 KB of the
// 32 KB parameter space, a per-launch copy in the constant bank): every epilogue thread reads the same weight at
// the same time, which is the constant cache's broadcast case, and shared memory has no room left for them
template <int NPAIR, int NPE>
struct PEWeights {
    float2 w[NPAIR * NPE];
};
struct NoPEWeights {};
// MPPI_L1_PARAM=1: without PE too, the H = 256 kernel takes its 3 x 256 position weights from the launch parameters
// instead of two shared-memory loads per neuron pair (which share the MIO queue with the MUFU work). FFMA2 has no
// constant-bank operand, so each weight pair becomes an LDC.64: measured +13% (configs[2]) / +8% (configs[3]); off.
#ifndef MPPI_L1_PARAM
#define MPPI_L1_PARAM 0
#endif
template <int H, int G, int PEB>
using PEArg = typename std::conditional<(H == 256 && ((PEB > 0 && !MPPI_PE_MMA) || MPPI_L1_PARAM)), PEWeights<H / 2, 3 + 6 * PEB>,
                                        NoPEWeights>::type;

// FUSE (H = 256 CTA pairs, configs[3]-sized problems): the rows are not read from HBM. Warps 2-3 of each CTA
// roll out its 64 samples of the pair's 128-sample block over the whole horizon with the device code of
// k_rollout (rollout_dev.cuh) and write each step's 128 query rows into the next row buffer; the pair's tiles
// are (block, t). Noise (for k_softmin), the shifted nominal and the non-SDF partial costs go to HBM as
// k_rollout writes them.
template <int H, int G, int ACT, int PEB, bool FUSE>
__global__ void __launch_bounds__(kThreads, 1)
    k_mlp_tc(const __grid_constant__ PEArg<H, G, PEB> pew, Params p, const float4* __restrict__ rows, long long n_rows,
             int ctrl_fixed, int states_mode,
             const uint8_t* __restrict__ wimg, const float* __restrict__ hid_b, const float* __restrict__ w_out,
             const float* __restrict__ b_out, const float4* __restrict__ w1p, const float* __restrict__ b1f,
             float* __restrict__ sdf_out, float* __restrict__ terms, const float2* __restrict__ w1pe2, Buffers bufs) {
    using C = Cfg<H, G, PEB>;
    static_assert(!FUSE || (H == 256 && PEB == 0 && !C::L1M), "fused rollout: H = 256 CTA pairs, CUDA-core layer 1");
    // FUSE: the producer warps share warpgroup 0 with the issuer and need ~80 registers (no epilogue spills at 96)
    constexpr int kCtl = FUSE ? MPPI_FUSE_CTL : kRegsCtl;
    constexpr int kEpi = ((96 * 640 - 128 * kCtl) / 512) / 8 * 8;
    constexpr int CG = C::CG;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    const uint32_t raw_u32 = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + ((1024u - (raw_u32 & 1023u)) & 1023u);
    const uint32_t sbase = smem_u32(smem);
    float4* s_w1xy = reinterpret_cast<float4*>(smem + C::OFF_W1XY);
    float2* s_w1z = reinterpret_cast<float2*>(smem + C::OFF_W1Z);
    float* s_wo = reinterpret_cast<float*>(smem + C::OFF_WO);
    float* s_b1 = reinterpret_cast<float*>(smem + C::OFF_B1);
    float* s_part = reinterpret_cast<float*>(smem + C::OFF_PART);
    const float* s_hb = reinterpret_cast<const float*>(smem + C::OFF_HB);   // !BIAS_MMA
    const uint32_t bar0 = sbase + C::OFF_BAR;
    auto bar = [&](int i) { return bar0 + 8u * (uint32_t)i; };
    uint32_t* s_tmem = reinterpret_cast<uint32_t*>(smem + C::OFF_TMEM);
    constexpr float kP = kPre<ACT>;
    TC_TRACE_DECL;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = CG == 2 ? cluster_ctarank() : 0u;
    const bool leader = rank == 0;
    const long long group = blockIdx.x / CG, n_groups = gridDim.x / CG;
    // work units of the CTA group: pair tiles of 256 rows, or (FUSE) blocks of 128 samples (T tiles each)
    const long long kb_per_ctrl = FUSE ? p.K / 128 : 1;
    const long long n_units = FUSE ? (long long)p.n_ctrl * kb_per_ctrl
                                   : (n_rows + (long long)kTileRows * CG - 1) / ((long long)kTileRows * CG);
    const long long n_my_units = group < n_units ? (n_units - group + n_groups - 1) / n_groups : 0;
    const long long n_tiles = FUSE ? (n_my_units > 0 ? n_units : 0) : n_units;   // "this group has work" below
    const long long n_my_all = FUSE ? n_my_units * p.T : n_my_units;               // local tiles of the group
    const long long rows_per_ctrl = states_mode ? (long long)p.T * p.K * p.rps : (1ll << 62);
    // controller of a step row (states mode): rows < 2^31 (validated), so a 32-bit division -- a 64-bit one is
    // ~10x the instructions, and this runs twice per tile and thread
    auto ctrl_of = [&](long long row) -> long long { return (long long)((uint32_t)row / (uint32_t)rows_per_ctrl); };

    // ---- setup
    if constexpr (C::L1M) {
        // layer-1 B operand of this CTA: rows = its RB neurons of each N-half unit, K = 32 columns pairing with
        // the A columns (t = 0..5 per coordinate c, column 3 t + c): w_h, w_m, w_h, w_l, w_m, w_h (x kP)
        // L1PE: then per PE feature f (columns 18 + 3 f + {0, 1, 2}) the two-part split w_h, w_l, w_h (weights from
        // the kP-scaled pair-major copy w1pe2)
        for (int idx = threadIdx.x; idx < C::NH * C::RB; idx += kThreads) {
            const int q = idx / C::RB, nn = idx % C::RB;
            const int n = q * C::UN + (int)rank * C::RB + nn;   // neuron
            auto wpe = [&](int f) {   // kP W1[n][f], f < NPE
                const float2 w2 = w1pe2[(n / 2) * C::NPE + f];
                return (n & 1) ? w2.y : w2.x;
            };
            float wc[3];
            if constexpr (C::L1PE) {
                wc[0] = wpe(0); wc[1] = wpe(1); wc[2] = wpe(2);
            } else {
                const float4 w = w1p[n];
                wc[0] = w.x * kP; wc[1] = w.y * kP; wc[2] = w.z * kP;
            }
            uint16_t part[3][3];   // [h, m, l][c]
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const __nv_bfloat16 hb = __float2bfloat16_rn(wc[c]);
                const float r1 = wc[c] - __bfloat162float(hb);
                const __nv_bfloat16 mb = __float2bfloat16_rn(r1);
                const __nv_bfloat16 lb = __float2bfloat16_rn(r1 - __bfloat162float(mb));
                part[0][c] = __bfloat16_as_ushort(hb);
                part[1][c] = __bfloat16_as_ushort(mb);
                part[2][c] = __bfloat16_as_ushort(lb);
            }
            constexpr int kB[6] = {0, 1, 0, 2, 1, 0};   // B part of term t
            for (int k = 0; k < C::K1; ++k) {
                uint16_t v = 0;
                if (k < 18) {
                    v = part[kB[k / 3]][k % 3];
                } else if (k < C::K1_USED) {
                    const float w = wpe(3 + (k - 18) / 3);
                    const __nv_bfloat16 hb = __float2bfloat16_rn(w);
                    v = (k - 18) % 3 == 1 ? __bfloat16_as_ushort(__float2bfloat16_rn(w - __bfloat162float(hb)))
                                          : __bfloat16_as_ushort(hb);
                }
                const int st = k / 16, kk = k % 16;
                *reinterpret_cast<uint16_t*>(smem + C::OFF_BL1 + (q * C::K1S + st) * C::BL1_TILE + (nn / 8) * 256 +
                                             (kk / 8) * 128 + (nn % 8) * 16 + (kk % 8) * 2) = v;
            }
        }
    } else
    for (int jp = threadIdx.x; jp < H / 2; jp += kThreads) {
        const float4 w0 = w1p[2 * jp], w1 = w1p[2 * jp + 1];
        s_w1xy[jp] = make_float4(w0.x * kP, w1.x * kP, w0.y * kP, w1.y * kP);
        s_w1z[jp] = make_float2(w0.z * kP, w1.z * kP);
    }
    if constexpr (C::PE_SMEM) {   // [pair jp][feature f] = (W1[2jp][f], W1[2jp+1][f]) kP
        float2* s_pe = reinterpret_cast<float2*>(smem + C::OFF_PE);
        for (int i = threadIdx.x; i < (H / 2) * C::NPE; i += kThreads) s_pe[i] = w1pe2[i];
    }
    if constexpr (!C::BIAS_MMA) {   // hidden biases for the epilogue, kP-scaled fp32
        float* s_hb = reinterpret_cast<float*>(smem + C::OFF_HB);
        for (int i = threadIdx.x; i < G * H; i += kThreads) s_hb[i] = hid_b[i] * kP;
    }
    if constexpr (C::BIAS_COMPACT) {
        uint32_t* zb = reinterpret_cast<uint32_t*>(smem + C::OFF_BIAS);   // bias images and ones tiles are adjacent
        for (int i = threadIdx.x; i < (C::BIAS_BYTES + C::ONES_BYTES) / 4; i += kThreads) zb[i] = 0u;
        __syncthreads();
        for (int i = threadIdx.x; i < G * 8; i += kThreads)   // ones tile l, row r: K columns 2l, 2l+1
            *reinterpret_cast<uint32_t*>(smem + C::OFF_ONES + (i / 8) * 256 + (i % 8) * 16 + (i / 8) * 4) = 0x3F803F80u;
        for (int idx = threadIdx.x; idx < C::NH * C::RB; idx += kThreads) {   // bias image of N-half q, neuron nn
            const int q = idx / C::RB, nn = idx % C::RB;
            const int n = q * C::UN + (int)rank * C::RB + nn;
            for (int l = 0; l < G; ++l) {   // the bf16 split of kP b (as the global image's, mlp_tc_pack_weights)
                const float bv = hid_b[l * H + n] * kP;
                const __nv_bfloat16 hi = __float2bfloat16_rn(bv);
                const __nv_bfloat16 lo = __float2bfloat16_rn(bv - __bfloat162float(hi));
                *reinterpret_cast<uint32_t*>(smem + C::OFF_BIAS + q * C::BIAS_UNIT + (nn / 8) * 256 + ((2 * l) / 8) * 128 +
                                             (nn % 8) * 16 + ((2 * l) % 8) * 2) =
                    (uint32_t)__bfloat16_as_ushort(hi) | ((uint32_t)__bfloat16_as_ushort(lo) << 16);
            }
        }
    } else if constexpr (C::BIAS_MMA)
    for (int r = threadIdx.x; r < kTileRows; r += kThreads) {   // ones tile: row r = [1, 1, 0 x 14] (bf16)
        uint32_t* o = reinterpret_cast<uint32_t*>(smem + C::OFF_ONES + (r / 8) * 256 + (r % 8) * 16);
        o[0] = 0x3F803F80u;
        o[1] = o[2] = o[3] = 0u;
        o[32] = o[33] = o[34] = o[35] = 0u;   // K core 1 (128 B further)
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes -> MMA operand reads
    for (int i = threadIdx.x; i < H; i += kThreads) s_wo[i] = w_out[i];
    if (threadIdx.x == 0) {
        for (int i = 0; i < C::NSLOT; ++i) {
            mbar_init(bar(BAR_AREADY + i), C::GW * CG);
            mbar_init(bar(BAR_DFREE + i), C::GW * CG);
            mbar_init(bar(BAR_MMA + i), 1);
            mbar_init(bar(BAR_SREADY + i), C::GW * CG);
            mbar_init(bar(BAR_AK0 + i), C::GW * CG);
        }
        mbar_init(bar(BAR_WLOCAL), 1);
        mbar_init(bar(BAR_WREADY), CG);
        for (int i = 0; i < C::NROWBUF; ++i) {
            mbar_init(bar(BAR_ROWS + i), FUSE ? 2 : 1);   // FUSE: the two rollout warps
            if (FUSE) mbar_init(bar(BAR_RFREE + i), 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        if constexpr (CG == 1) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(s_tmem)),
                         "r"(C::TMEM_COLS));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        } else {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(s_tmem)),
                         "r"(C::TMEM_COLS));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        }
    }
    tc_fence_before();
    __syncthreads();
    if constexpr (CG == 2) cluster_sync();   // peer barriers initialised before any remote arrive
    tc_fence_after();
    const uint32_t tmem = *s_tmem;
    // leader-CTA addresses of the scheduling barriers (the MMA issuer waits on them)
    const uint32_t lbar0 = CG == 2 ? map_to_rank(bar0, 0) : bar0;
    auto lbar = [&](int i) { return lbar0 + 8u * (uint32_t)i; };

    if (warp < kEpiWarp0) {
      asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kCtl));
      if (warp == 1) {
        // ================= weight loader: this CTA's share of every unit, once
        if (lane == 0 && group < n_tiles) {
            mbar_expect_tx(bar(BAR_WLOCAL), (uint32_t)(C::W_BYTES + (C::BIAS_COMPACT ? 0 : C::BIAS_BYTES)));
            const uint8_t* src = wimg + (size_t)rank * C::IMG_BYTES;
            for (int u = 0; u < G * C::NH; ++u)
                bulk_g2s(sbase + (uint32_t)(u * C::UNIT_BYTES), src + (size_t)u * C::UNIT_BYTES, C::UNIT_BYTES,
                         bar(BAR_WLOCAL));
            if constexpr (C::BIAS_MMA && !C::BIAS_COMPACT)
                bulk_g2s(sbase + (uint32_t)C::OFF_BIAS, src + C::W_BYTES, C::BIAS_BYTES, bar(BAR_WLOCAL));
            mbar_wait(bar(BAR_WLOCAL), 0);
            if constexpr (CG == 2) mbar_arrive_cluster(lbar(BAR_WREADY));
            else mbar_arrive_local(bar(BAR_WREADY));
        }
      } else if (FUSE && (warp == 2 || warp == 3) && n_my_all > 0) {
        // ================= fused rollout producer (FUSE): thread = one of this CTA's 64 samples of the block
        const int tid = threadIdx.x - 64;
        const unsigned long long step = *bufs.step;
        const int sh = step > 0 ? 1 : 0;
        const bool dev_noise = p.noise_device != 0;
        const long long NK = (long long)p.n_ctrl * p.K;
        const float inv_mass = 1.f / p.mass;
        for (long long j = 0; j < n_my_units; ++j) {
            const long long blk = group + j * n_groups;
            const int bb = (int)(blk / kb_per_ctrl);
            const int k = (int)((blk % kb_per_ctrl) * 128) + (int)rank * 64 + tid;
            const bool first = blk % kb_per_ctrl == 0 && rank == 0 && tid == 0;
            float x[10];
#pragma unroll
            for (int q = 0; q < 10; ++q) x[q] = __ldg(bufs.x0 + bb * 10 + q);
            float Rm[9], tq[3], gc[3];
#pragma unroll
            for (int q = 0; q < 9; ++q) Rm[q] = __ldg(bufs.Tq + bb * 12 + q);
#pragma unroll
            for (int q = 0; q < 3; ++q) { tq[q] = __ldg(bufs.Tq + bb * 12 + 9 + q); gc[q] = __ldg(bufs.goal + bb * 3 + q); }
            const long long col = (long long)bb * p.K + k;
            const unsigned long long gidx = global_sample(p, bb, k);
            const float4* Uo = reinterpret_cast<const float4*>(bufs.U_out) + (long long)bb * p.T;
            float part = 0.f;
            for (int t = 0; t < p.T; ++t) {
                const long long i = j * p.T + t;
                constexpr int kNRB = C::NROWBUF > 0 ? C::NROWBUF : 1;
                const int rb = (int)(i % kNRB);
                const uint32_t use = (uint32_t)(i / kNRB);
                const float4 U = Uo[min(t + sh, p.T - 1)];   // warm-start shift
                if (first) reinterpret_cast<float4*>(bufs.U_nom)[(long long)bb * p.T + t] = U;
                float4 n;
                if (dev_noise) {
                    n = philox_normals(gidx, t, step, p.seed);
                    bufs.noise[(long long)t * NK + col] = n;   // for k_softmin
                } else {
                    n = bufs.noise[(long long)t * NK + col];
                }
                float4 row0, row1;
                ctbr_step(p, x, U, n, Rm, tq, gc, inv_mass, row0, row1, part);
                if (use > 0) mbar_wait(bar(BAR_RFREE + rb), (use - 1) & 1u);   // tile i - NROWBUF has been output
                float4* dst = reinterpret_cast<float4*>(smem + C::OFF_ROWS) + rb * kTileRows;
                dst[2 * tid] = row0;
                dst[2 * tid + 1] = row1;
                __syncwarp();
                if (lane == 0) mbar_arrive_local(bar(BAR_ROWS + rb));
            }
            bufs.partial[col] = part;
        }
      } else if (warp == 0) {
        // ================= MMA issuer (one thread of the leader CTA)
        // NSLOT tiles in flight (TMEM slots). Per layer and N-half h, one full-K unit per slot, issued slot by
        // slot (X(h0) Y(h0) .. X(h1) Y(h1) ..): while the epilogue drains one slot the tensor pipe works on
        // the others.
        // H = 256 (CTA pairs): the whole warp walks the schedule and one elected lane issues, so the operands
        // stay in uniform registers (A/B at configs[2]: -5%); H = 128: lane 0 alone (the warp form +4% at [4])
        constexpr bool kWarpIssuer = MPPI_ISSUER_WARP < 0 ? CG == 2 : MPPI_ISSUER_WARP != 0;
        if ((kWarpIssuer || lane == 0) && leader && group < n_tiles) {
            constexpr uint32_t idesc = idesc_bf16(C::MMA_M, C::UN);
            const long long n_my = n_my_all;
            // Barrier phases. H = 256: every slot sees the same sequence per tile (AREADY once per layer, DFREE
            // before every unit but the first), so they follow from (tile n, l, h) and nothing spills from the
            // issuer's 32 registers (configs[2] -1.3%). H = 128: per-slot counters (the closed form measured
            // +15% at configs[1,4] with the lane-0 issuer).
            constexpr uint32_t kAPerTile = C::A1S ? G - 1 : C::L1M ? G + 1 : G;
            constexpr uint32_t kLay = C::L1M ? G + 1 : G;   // MMA layers per tile (L1M: layer 1 is one)
            uint32_t a_cnt[C::NSLOT] = {}, u_cnt[C::NSLOT] = {}, s_cnt[C::NSLOT] = {};
            mbar_wait<CG == 2>(bar(BAR_WREADY), 0);
            for (long long i0 = 0; i0 < n_my; i0 += C::NSLOT) {
                const int ns = (int)min((long long)C::NSLOT, n_my - i0);
                const uint32_t n = (uint32_t)(i0 / C::NSLOT);   // this slot-tile's index: barrier phases below
                for (int l = C::L1M ? -1 : 0; l < G; ++l)
                    for (int h = 0; h < C::NH; ++h)
                        for (int sl = 0; sl < ns; ++sl) {
                            TC_TRACE(0, 0, l, h, sl, i0);
                            const bool a_smem = C::A1S && l == 0;
                            // layer index within the tile's A-ready sequence (L1M: the A1 operand is step 0)
                            const uint32_t lp = (uint32_t)(C::L1M ? l + 1 : l);
                            if constexpr (CG == 2) {
                                if (h == 0) {
                                    if (C::SPLITK && l >= 0) mbar_wait_issuer(bar(BAR_AK0 + sl), (n * G + (uint32_t)l) & 1u);
                                    else mbar_wait_issuer(bar(BAR_AREADY + sl), (n * kAPerTile + lp) & 1u);
                                }
                                const uint32_t u = (n * kLay + lp) * C::NH + (uint32_t)h;
                                if (u > 0) mbar_wait_issuer(bar(BAR_DFREE + sl), (u - 1) & 1u);
                            } else {
                                if (a_smem) mbar_wait_issuer(bar(BAR_SREADY + sl), (s_cnt[sl]++) & 1);
                                else if (h == 0) mbar_wait_issuer(bar(BAR_AREADY + sl), (a_cnt[sl]++) & 1);
                                if (u_cnt[sl] > 0) mbar_wait_issuer(bar(BAR_DFREE + sl), (u_cnt[sl] - 1) & 1);
                                ++u_cnt[sl];
                            }
                            tc_fence_after();
                            TC_TRACE(0, 1, l, h, sl, i0);
                            const uint32_t d_t = tmem + (uint32_t)(sl * C::SLOT_COLS);
                            const uint32_t a_t = d_t + (uint32_t)C::A_OFF;
                            const uint32_t b_unit = sbase + (uint32_t)((l * C::NH + h) * C::UNIT_BYTES);
                            // the B descriptor of K step j is the unit's with its 14-bit address field advanced by the byte
                            // offset / 16 (no carry: shared addresses < 256 KB): one 32-bit add instead of a rebuild
                            constexpr bool kDescAdd = MPPI_DESC_ADD < 0 ? C::L1PE : MPPI_DESC_ADD != 0;
                            const uint64_t bd0 = smem_desc_sw128(b_unit);
                            const uint32_t bd_lo = (uint32_t)bd0, bd_hi = (uint32_t)(bd0 >> 32);
                            auto issue_k = [&](int j_lo, int j_hi) {   // K steps [16 j_lo, 16 j_hi) of the unit
#pragma unroll
                                for (int j = 0; j < H / 16; ++j) {
                                    if (j < j_lo || j >= j_hi) continue;
                                    const int kk = j * 16;
                                    const uint32_t b_addr = b_unit + (uint32_t)((kk / 64) * (C::RB * 128) + (kk % 64) * 2);
                                    if (kDescAdd && !a_smem) {
                                        const uint32_t o16 = (uint32_t)((kk / 64) * (C::RB * 128) + (kk % 64) * 2) >> 4;
                                        tc_mma_ts<CG>(d_t, a_t + (uint32_t)(kk / 2), ((uint64_t)bd_hi << 32) | (bd_lo + o16), idesc,
                                                      (C::BIAS_MMA || j > 0) ? 1u : 0u);
                                        continue;
                                    }
                                    if (a_smem) {
                                        const uint32_t a_addr = sbase + (uint32_t)(C::OFF_SA + sl * C::SA_BYTES +
                                                                                   (kk / 64) * (kTileRows * 128) + (kk % 64) * 2);
                                        tc_mma_ss<CG>(d_t, smem_desc_sw128(a_addr), smem_desc_sw128(b_addr), idesc, 1u);
                                    } else {
                                        tc_mma_ts<CG>(d_t, a_t + (uint32_t)(kk / 2), smem_desc_sw128(b_addr), idesc,
                                                  (C::BIAS_MMA || j > 0) ? 1u : 0u);
                                    }
                                }
                            };
                            if (C::L1M && l < 0) {   // layer 1: D = A1 (TMEM) x B1^T, K = K1 (bias b1' in the epilogue)
                                if (!kWarpIssuer || elect_one()) {
#pragma unroll
                                    for (int st = 0; st < C::K1S; ++st)
                                        tc_mma_ts<CG>(d_t, a_t + (uint32_t)(st * 8),
                                                      smem_desc_kmajor_noswz(sbase + (uint32_t)(C::OFF_BL1 + (h * C::K1S + st) * C::BL1_TILE)),
                                                      idesc, st > 0 ? 1u : 0u);
                                    tc_commit<CG>(bar(BAR_MMA + sl));
                                }
                                if constexpr (kWarpIssuer) __syncwarp();
                                TC_TRACE(0, 2, l, h, sl, i0);
                                continue;
                            }
                            // SPLITK: N-half 0 starts on K-half 0 of A; K-half 1 waits for the whole epilogue
                            const int j_mid = C::SPLITK && h == 0 ? H / 32 : H / 16;
                            if (!kWarpIssuer || elect_one()) {
                                // D = bias (ones x [b_hi, b_lo]), then D += A W^T over K = H
                                if constexpr (C::BIAS_COMPACT)
                                    tc_mma_ss<CG>(d_t, smem_desc_noswz(sbase + (uint32_t)(C::OFF_ONES + l * 256), 128, 0),
                                                  smem_desc_kmajor_noswz(sbase + (uint32_t)(C::OFF_BIAS + h * C::BIAS_UNIT)),
                                                  idesc, 0u);
                                else if constexpr (C::BIAS_MMA)
                                    tc_mma_ss<CG>(d_t, smem_desc_kmajor_noswz(sbase + (uint32_t)C::OFF_ONES),
                                                  smem_desc_kmajor_noswz(sbase + (uint32_t)(C::OFF_BIAS + (l * C::NH + h) * C::BIAS_UNIT)),
                                                  idesc, 0u);
                                issue_k(0, j_mid);
                            }
                            if (C::SPLITK && h == 0) {
                                if constexpr (kWarpIssuer) __syncwarp();
                                mbar_wait_issuer(bar(BAR_AREADY + sl), (n * kAPerTile + lp) & 1u);
                                tc_fence_after();
                            }
                            if (!kWarpIssuer || elect_one()) {
                                issue_k(j_mid, H / 16);
                                tc_commit<CG>(bar(BAR_MMA + sl));
                            }
                            if constexpr (kWarpIssuer) __syncwarp();
                            TC_TRACE(0, 2, l, h, sl, i0);
                        }
            }
        }
      }
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kEpi));
        // ================= epilogue: NSLOT groups of GW warps, group sl owns TMEM slot sl and the CTA's
        // tiles i = sl, sl + NSLOT, ... (one group computes while the others wait for their MMA units)
        constexpr int kColGroups = C::COLG;
        const int e = warp - kEpiWarp0;
        const int sl = e / C::GW;                  // tile slot of this group
        const int eg = e % C::GW;
        const int g = warp & 3;                    // TMEM lane quarter
        const int cgi = eg >> 2;                   // column group of each N-half (QW columns)
        const int row_in_tile = g * 32 + lane;
        const uint32_t lane_addr = (uint32_t)(g * 32) << 16;
        const int gthreads = C::GW * 32;
        const int gtid = eg * 32 + lane;
        const bool tracer = lane == 0 && eg == 0 && sl < 2;   // trace roles 1, 2 = slots 0, 1
        const int trole = 1 + sl;
        const long long n_my = n_my_all;
        uint32_t mma_cnt = 0;
        long long staged = -1;                     // controller whose b1' sits in this group's b1g
        float* b1g = s_b1 + sl * H;
        float* part = s_part + sl * kColGroups * kTileRows;
        auto arrive_sched = [&](int i) {           // epilogue -> MMA issuer (leader CTA)
            if constexpr (CG == 2) mbar_arrive_cluster(lbar(i));
            else mbar_arrive_local(bar(i));
        };
        auto tile_of = [&](long long i) { return group + i * n_groups; };
        auto tile_row0 = [&](long long t) { return t * (kTileRows * CG) + (long long)rank * kTileRows; };
        // first global row of this CTA's part of local tile i (FUSE: tile = (block, step t); the CTA's 64
        // samples are rank * 64 .. + 63 of the 128-sample block; the two rows of a state are adjacent)
        auto row0_of = [&](long long i) -> long long {
            if constexpr (FUSE) {   // 32-bit divisions (a 64-bit one is ~10x the instructions, per tile and thread)
                const uint32_t ii = (uint32_t)i, T = (uint32_t)p.T, kb = (uint32_t)kb_per_ctrl;
                const uint32_t j = ii / T, t = ii - j * T, blk = (uint32_t)group + j * (uint32_t)n_groups;
                const uint32_t bb = blk / kb, k0 = (blk - bb * kb) * 128u + rank * 64u;
                return (((long long)bb * p.T + t) * p.K + k0) * 2;
            } else {
                return tile_row0(tile_of(i));
            }
        };
        // query rows of this CTA's part of tile i -> smem buffer i % NROWBUF by one bulk-async copy (TMA
        // engine), issued one tile of this slot (NSLOT tiles) ahead by one elected thread of the group
        const float4* s_rows = reinterpret_cast<const float4*>(smem + C::OFF_ROWS);
        constexpr int kNRB = C::NROWBUF > 0 ? C::NROWBUF : 1;   // (no row buffers with L1PE: never used)
        const bool row_issuer = eg == 0 && lane == 0;
        auto issue_rows = [&](long long i) {
            if (FUSE || C::NROWBUF == 0 || !row_issuer || i >= n_my) return;   // FUSE: the rollout warps write the rows
            const long long r0 = row0_of(i);
            const long long nv = min((long long)kTileRows, n_rows - r0);
            if (nv <= 0) {
                mbar_arrive_local(bar(BAR_ROWS + (int)(i % kNRB)));
                return;
            }
            mbar_expect_tx(bar(BAR_ROWS + (int)(i % kNRB)), (uint32_t)(16 * nv));
            bulk_g2s(sbase + C::OFF_ROWS + (uint32_t)((i % kNRB) * 16 * kTileRows), rows + r0, (uint32_t)(16 * nv),
                     bar(BAR_ROWS + (int)(i % kNRB)));
        };
        auto row_of = [&](long long i) {   // this thread's query row of tile i (after its buffer landed)
            const long long row = row0_of(i) + row_in_tile;
            return row < n_rows ? s_rows[(i % kNRB) * kTileRows + row_in_tile] : make_float4(0.f, 0.f, 0.f, 0.f);
        };
        // 16 layer-1 activations (bf16x2) of this thread's row, neurons j0..j0+15 -> the slot's A operand:
        // TMEM, or (A1S) the shared-memory tile in the SW128 K-major layout of the weight images
        auto store_a1 = [&](int j0, const uint32_t* packed) {
            if constexpr (C::A1S) {
                const int kc = j0 / 64, c0 = (j0 % 64) / 8;
                const uint32_t rbase = sbase + (uint32_t)(C::OFF_SA + sl * C::SA_BYTES + kc * (kTileRows * 128) + row_in_tile * 128);
#pragma unroll
                for (int c = 0; c < 2; ++c)
                    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(rbase + (uint32_t)((((c0 + c) ^ (row_in_tile & 7))) * 16)),
                                 "r"(packed[4 * c]), "r"(packed[4 * c + 1]), "r"(packed[4 * c + 2]), "r"(packed[4 * c + 3])
                                 : "memory");
            } else {
                tmem_st8(tmem + lane_addr + (uint32_t)(sl * C::SLOT_COLS + C::A_OFF) + (uint32_t)(j0 / 2), packed);
            }
        };
        // layer 1 (CUDA cores): a1 = act(W1p p + b1') -> bf16 -> A operand of this slot, for tile index i
        auto layer1 = [&](long long i) {
            const long long t1 = tile_of(i);
            if (tracer) TC_TRACE(trole, 6, 0, 0, sl, t1);
            mbar_wait(bar(BAR_ROWS + (int)(i % kNRB)), (uint32_t)((i / kNRB) & 1));
            if (tracer) TC_TRACE(trole, 11, 0, 0, sl, t1);
            const float4 q = row_of(i);
            const float2 qx2 = make_float2(q.x, q.x), qy2 = make_float2(q.y, q.y), qz2 = make_float2(q.z, q.z);
            if constexpr (!C::A1S) issue_rows(i + C::NSLOT);   // buffer last read by tile i - NSLOT (behind its bar)
            const long long row0 = row0_of(i);
            const long long lo = states_mode ? ctrl_of(min(row0, n_rows - 1)) : ctrl_fixed;
            if (lo != staged) {   // uniform across the group
                named_bar_sync(1 + C::NSLOT + sl, gthreads);   // nobody in the group still reads the old staging
                for (int j = gtid; j < H; j += gthreads) b1g[j] = lo < p.n_ctrl ? b1f[(size_t)lo * H + j] * kP : 0.f;
                staged = lo;
                named_bar_sync(1 + C::NSLOT + sl, gthreads);
            }
            const long long row = row0 + row_in_tile;
            const long long bb = states_mode ? ctrl_of(min(row, n_rows - 1)) : ctrl_fixed;
            const float* bfar = bb != lo ? b1f + (size_t)bb * H : nullptr;   // rows of a later controller
            const bool any_far = __any_sync(0xFFFFFFFFu, bfar != nullptr);
            if constexpr (PEB > 0) {
                // PE(p_c) = [p, sin(2^i pi p), cos(2^i pi p)]_{i < PEB} in fp32 (sincospif: exact range
                // reduction), then the NPE-wide layer-1 dot on FFMA2 (reading E1)
                float feat[C::NPE];
                feat[0] = q.x;
                feat[1] = q.y;
                feat[2] = q.z;
#pragma unroll
                for (int bnd = 0; bnd < PEB; ++bnd) {
                    const float sc = (float)(1 << bnd);
                    sincospif(q.x * sc, &feat[3 + 6 * bnd + 0], &feat[3 + 6 * bnd + 3]);
                    sincospif(q.y * sc, &feat[3 + 6 * bnd + 1], &feat[3 + 6 * bnd + 4]);
                    sincospif(q.z * sc, &feat[3 + 6 * bnd + 2], &feat[3 + 6 * bnd + 5]);
                }
                const float2* s_pe = reinterpret_cast<const float2*>(smem + C::OFF_PE);
                auto pe_w = [&](int idx) -> float2 {
                    if constexpr (C::PE_SMEM) return s_pe[idx];
                    else if constexpr (sizeof(pew) > 1) return pew.w[idx];
                    else return make_float2(0.f, 0.f);   // L1PE: layer 1 is prep() + an MMA (never called)
                };
#pragma unroll
                for (int c = 0; c < C::NH; ++c) {
#pragma unroll
                    for (int k = 0; k < C::NCH; ++k) {
                        const int j0 = c * C::UN + cgi * C::QW + k * kCW;
                        uint32_t packed[kCW / 2];
#pragma unroll
                        for (int i2 = 0; i2 < kCW; i2 += 2) {
                            const int jp = (j0 + i2) / 2;
                            float2 x = *reinterpret_cast<const float2*>(b1g + j0 + i2);
                            if (any_far && bfar) x = make_float2(__ldg(bfar + j0 + i2) * kP, __ldg(bfar + j0 + i2 + 1) * kP);
#pragma unroll
                            for (int f = 0; f < C::NPE; ++f) x = ffma2(pe_w(jp * C::NPE + f), make_float2(feat[f], feat[f]), x);
                            packed[i2 / 2] = act_pack<ACT>(x.x, x.y);
                        }
                        store_a1(j0, packed);
                    }
                    if (C::SPLITK && c == 0) {   // K-half 0 of the first GEMM's A is complete
                        tmem_wait_st();
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) arrive_sched(BAR_AK0 + sl);
                    }
                }
            } else
#pragma unroll
            for (int c = 0; c < C::NH; ++c) {
#pragma unroll
                for (int k = 0; k < C::NCH; ++k) {
                    const int j0 = c * C::UN + cgi * C::QW + k * kCW;
                    uint32_t packed[kCW / 2];
                    if (!any_far) {
#pragma unroll
                        for (int i2 = 0; i2 < kCW; i2 += 2) {
                            const int jp = (j0 + i2) / 2;   // neuron pair (j0+i2, j0+i2+1)
                            float2 wx, wy, wz;
                            if constexpr (sizeof(pew) > 1) {   // weights in the launch parameters (H = 256)
                                wx = pew.w[jp * 3]; wy = pew.w[jp * 3 + 1]; wz = pew.w[jp * 3 + 2];
                            } else {
                                const float4 wa = s_w1xy[jp];
                                wx = make_float2(wa.x, wa.y); wy = make_float2(wa.z, wa.w); wz = s_w1z[jp];
                            }
                            const float2 x = ffma2(wx, qx2, ffma2(wy, qy2, ffma2(wz, qz2, *reinterpret_cast<const float2*>(b1g + j0 + i2))));
                            packed[i2 / 2] = act_pack<ACT>(x.x, x.y);
                        }
                    } else {   // rare: the tile crosses a controller boundary
#pragma unroll
                        for (int i2 = 0; i2 < kCW; i2 += 2) {
                            const int jp = (j0 + i2) / 2;
                            const float4 wa = s_w1xy[jp];
                            const float b0 = bfar ? __ldg(bfar + j0 + i2) * kP : b1g[j0 + i2];
                            const float b1 = bfar ? __ldg(bfar + j0 + i2 + 1) * kP : b1g[j0 + i2 + 1];
                            const float2 x = ffma2(make_float2(wa.x, wa.y), qx2,
                                                   ffma2(make_float2(wa.z, wa.w), qy2, ffma2(s_w1z[jp], qz2, make_float2(b0, b1))));
                            packed[i2 / 2] = act_pack<ACT>(x.x, x.y);
                        }
                    }
                    store_a1(j0, packed);
                }
                if (C::SPLITK && c == 0) {   // K-half 0 of the first GEMM's A is complete
                    tmem_wait_st();
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) arrive_sched(BAR_AK0 + sl);
                }
            }
            if (tracer) TC_TRACE(trole, 12, 0, 0, sl, t1);
            if constexpr (C::A1S) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes -> MMA operand reads
                __syncwarp();
                if (lane == 0) arrive_sched(BAR_SREADY + sl);
            } else {
                tmem_wait_st();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) arrive_sched(BAR_AREADY + sl);
            }
            if (tracer) TC_TRACE(trole, 7, 0, 0, sl, t1);
        };

        // L1M: the layer-1 MMA operand of tile i (exact bf16 splits of p_c, K = 32 or 96) -> the slot's A columns in
        // TMEM. Nothing of the tile is kept in registers across its layers (the epilogue is at its register limit):
        // the far-controller state is recomputed in the layer-1 epilogue and |v| re-read at the output.
        // L1PE: no row buffers -- each thread loads its query row itself (an L2 prefetch is issued a tile ahead)
        auto row_ptr = [&](long long i) -> const float4* {
            const long long row = row0_of(i) + row_in_tile;
            return i < n_my && row < n_rows ? rows + row : nullptr;
        };
        auto prep = [&](long long i) {
            const long long t1 = tile_of(i);
            if (tracer) TC_TRACE(trole, 6, 0, 0, sl, t1);
            float4 q;
            if constexpr (C::L1PE) {
                const float4* rp = row_ptr(i);
                q = rp ? __ldg(rp) : make_float4(0.f, 0.f, 0.f, 0.f);
            } else {
                mbar_wait(bar(BAR_ROWS + (int)(i % kNRB)), (uint32_t)((i / kNRB) & 1));
                q = row_of(i);
            }
            const long long row0 = tile_row0(t1);
            const long long lo = states_mode ? ctrl_of(min(row0, n_rows - 1)) : ctrl_fixed;
            if (lo != staged) {   // uniform across the group; b1g of the previous tile is no longer read
                named_bar_sync(1 + C::NSLOT + sl, gthreads);
                for (int j = gtid; j < H; j += gthreads) b1g[j] = lo < p.n_ctrl ? b1f[(size_t)lo * H + j] * kP : 0.f;
                staged = lo;
            }
            uint32_t hv[3], mv[3], lv[3];
            const float pc[3] = {q.x, q.y, q.z};
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const __nv_bfloat16 hb = __float2bfloat16_rn(pc[c]);
                const float r1 = pc[c] - __bfloat162float(hb);
                const __nv_bfloat16 mb = __float2bfloat16_rn(r1);
                const __nv_bfloat16 lb = __float2bfloat16_rn(r1 - __bfloat162float(mb));
                hv[c] = __bfloat16_as_ushort(hb);
                mv[c] = __bfloat16_as_ushort(mb);
                lv[c] = __bfloat16_as_ushort(lb);
            }
            // columns 3 t + c, t = 0..5: x_h, x_h, x_m, x_h, x_m, x_l (pairs with B: w_h, w_m, w_h, w_l, w_m, w_h);
            // compile-time indices only (a runtime index sends the arrays to local memory)
            uint32_t kv[16];
#pragma unroll
            for (int w2 = 0; w2 < 16; ++w2) {
                uint32_t v2[2];
#pragma unroll
                for (int e2 = 0; e2 < 2; ++e2) {
                    const int k = 2 * w2 + e2, t = k / 3, c = k % 3;
                    v2[e2] = k >= 18 ? 0u : (t == 2 || t == 4) ? mv[c] : t == 5 ? lv[c] : hv[c];
                }
                kv[w2] = v2[0] | (v2[1] << 16);
            }
            const uint32_t a_base = tmem + lane_addr + (uint32_t)(sl * C::SLOT_COLS + C::A_OFF);
            if constexpr (C::L1PE) {
                // columns 18 + 3 f + {0, 1, 2} = f_h, f_h, f_l per PE feature f (pairs with B: w_h, w_l, w_h); f = 6 b + c
                // (sin), 6 b + 3 + c (cos); each of the row's two threads writes 24 of the 48 TMEM columns
                auto feat = [&](int f) -> float {   // PE feature f (compile-time): sin / cos(2^b pi p_c), f = 6 b + 3 cos + c
                    float sv, cv;
                    sincospif(pc[f % 3] * (float)(1 << (f / 6)), &sv, &cv);
                    return (f % 6) >= 3 ? cv : sv;
                };
                auto colv = [&](int k) -> uint32_t {   // bf16 bits of operand column k (compile-time k)
                    if (k < 18) {
                        const int t = k / 3, c = k % 3;
                        return (t == 2 || t == 4) ? mv[c] : t == 5 ? lv[c] : hv[c];
                    }
                    if (k >= C::K1_USED) return 0u;
                    const float fv = feat((k - 18) / 3);
                    const __nv_bfloat16 fh = __float2bfloat16_rn(fv);
                    if ((k - 18) % 3 < 2) return __bfloat16_as_ushort(fh);
                    return __bfloat16_as_ushort(__float2bfloat16_rn(fv - __bfloat162float(fh)));
                };
                constexpr int kHalf = C::K1 / 4;   // TMEM columns (bf16 pairs) per thread: 24
                auto store_half = [&](auto cg_c) {   // this thread's 24 columns, 8 at a time (features computed per store)
                    constexpr int cg = decltype(cg_c)::value;
#pragma unroll
                    for (int s8 = 0; s8 < kHalf / 8; ++s8) {
                        uint32_t a8[8];
#pragma unroll
                        for (int w2 = 0; w2 < 8; ++w2) {
                            const int k = 2 * (kHalf * cg + 8 * s8 + w2);
                            a8[w2] = colv(k) | (colv(k + 1) << 16);
                        }
                        tmem_st8(a_base + (uint32_t)(kHalf * cg + 8 * s8), a8);
                    }
                };
                if (cgi == 0) store_half(std::integral_constant<int, 0>{});
                else store_half(std::integral_constant<int, 1>{});
            } else {
                uint32_t a[8];
#pragma unroll
                for (int w2 = 0; w2 < 8; ++w2) a[w2] = cgi == 0 ? kv[w2] : kv[8 + w2];
                tmem_st8(a_base + (uint32_t)(8 * cgi), a);
            }
            named_bar_sync(1 + C::NSLOT + sl, gthreads);   // every warp has read the row buffer (and b1g is staged)
            issue_rows(i + C::NSLOT);
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) arrive_sched(BAR_AREADY + sl);
            if (tracer) TC_TRACE(trole, 7, 0, 0, sl, t1);
        };
        issue_rows(sl);
        if constexpr (C::L1M) {
            if (sl < n_my) prep(sl);
        } else {
            if constexpr (C::A1S) issue_rows(sl + C::NSLOT);
            if (sl < n_my) layer1(sl);
        }
        for (long long i = sl; i < n_my; i += C::NSLOT) {
            uint32_t keep[C::NH > 1 ? C::QW / 2 : 1];   // unit-0 activations (bf16x2) until unit 1 is done
            float2 sdot2 = make_float2(0.f, 0.f);
            if constexpr (C::L1PE) {   // the row prep(i + NSLOT) reads, into L2 a tile ahead
                const float4* rp = row_ptr(i + C::NSLOT);
                if (rp) asm volatile("prefetch.global.L2 [%0];" ::"l"(rp));
            }
            // one layer's units; layer 1 (L1M) is a separate instantiation (kL1), so its epilogue's registers are
            // allocated apart from the GEMM layers' rolled loop
            auto run_layer = [&](auto l1c, const int l) {
                constexpr bool kL1 = decltype(l1c)::value;
                const bool last = !kL1 && (l == G - 1);
#pragma unroll
                for (int h = 0; h < C::NH; ++h) {
                    if (tracer) TC_TRACE(trole, 3, l, h, sl, i);
                    mbar_wait(bar(BAR_MMA + sl), (mma_cnt++) & 1);
                    tc_fence_after();
                    if (tracer) TC_TRACE(trole, 4, l, h, sl, i);
                    const uint32_t d_col = (uint32_t)(sl * C::SLOT_COLS + cgi * C::QW);
                    const uint32_t a_col = (uint32_t)(sl * C::SLOT_COLS + C::A_OFF);
                    if (C::SPLITK && !last && h == C::NH - 1) {
                        // the layer's last MMA has read A: N-half 0's activations -> K-half 0 of the next A now
#pragma unroll
                        for (int k = 0; k < C::NCH; ++k)
                            tmem_st8(tmem + lane_addr + a_col + (uint32_t)((cgi * C::QW + k * kCW) / 2), &keep[k * (kCW / 2)]);
                        tmem_wait_st();
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) arrive_sched(BAR_AK0 + sl);
                    }
                    // L1M: the tile's last MMA has read A -> next tile's layer-1 operand into the dead A columns (after
                    // the keep[] store above, so keep[] is dead here: prep's registers do not spill it)
                    if (C::L1M && last && h == C::NH - 1 && i + C::NSLOT < n_my) prep(i + C::NSLOT);
                    // H = 256: chunk k + 1's TMEM load is in flight while chunk k is computed (configs[2] -2%;
                    // H = 128 +2%: load, wait, compute)
                    // kAll (H = 256): the whole D share of the warp (NCH x 16 columns) loaded at once, one wait, and
                    // D released before any of it is computed, so the slot's next unit can start ~1 k cycles
                    // earlier (the N-half-0 activations kept in registers are already stored at h = 1)
                    // (L1M: off -- with layer 1's epilogue and prep in the same loop, kAll's 64 live accumulator registers
                    // spill the tile state; the pipelined form has no spills)
                    constexpr bool kAll = MPPI_EPI_ALL < 0 ? CG == 2 && (!C::L1M || (MPPI_L1M_ALL && !kL1)) : MPPI_EPI_ALL != 0;
                    constexpr bool kPipe = !kAll && (MPPI_EPI_PIPE < 0 ? CG == 2 : MPPI_EPI_PIPE != 0);
                    uint32_t accb[kAll ? C::NCH : kPipe ? 2 : 1][kCW];
                    if constexpr (kAll) {
#pragma unroll
                        for (int k = 0; k < C::NCH; ++k) tmem_ld16(tmem + lane_addr + d_col + (uint32_t)(k * kCW), accb[k]);
                        tmem_wait_ld_regs(accb[0]);
#pragma unroll
                        for (int k = 1; k < C::NCH; ++k) tmem_tie_regs(accb[k]);
                    }
                    if constexpr (kPipe) tmem_ld16(tmem + lane_addr + d_col, accb[0]);
#pragma unroll
                    for (int k = 0; k < C::NCH; ++k) {
                        uint32_t(&acc)[kCW] = accb[kAll ? k : kPipe ? (k & 1) : 0];
                        if constexpr (kAll) {
                        } else if constexpr (kPipe) {
                            tmem_wait_ld_regs(acc);
                            if (k + 1 < C::NCH)
                                tmem_ld16(tmem + lane_addr + d_col + (uint32_t)((k + 1) * kCW), accb[(k + 1) & 1]);
                        } else {
                            tmem_ld16(tmem + lane_addr + d_col + (uint32_t)(k * kCW), acc);
                            tmem_wait_ld_regs(acc);
                        }
                        if (kAll ? k == 0 : k == C::NCH - 1) {   // D of the slot may be overwritten now
                            tc_fence_before();
                            __syncwarp();
                            if (lane == 0) arrive_sched(BAR_DFREE + sl);
                            if (tracer) TC_TRACE(trole, 10, l, h, sl, i);
                        }
                        const int j0 = h * C::UN + cgi * C::QW + k * kCW;   // output neuron index
                        if (!last) {
                            uint32_t packed[kCW / 2];
                            if (kL1) {   // layer 1: D + kP b1' (per controller), fast path for one controller
                                // rows of a controller after the staged one (the tile crosses a controller boundary)
                                const long long row = row0_of(i) + row_in_tile;
                                const long long bb = states_mode ? ctrl_of(min(row, n_rows - 1)) : ctrl_fixed;
                                const float* bfar_t = bb != staged ? b1f + (size_t)bb * H : nullptr;
                                const bool any_far_t = __any_sync(0xFFFFFFFFu, bfar_t != nullptr);
                                if (!any_far_t) {
#pragma unroll
                                    for (int i2 = 0; i2 < kCW; i2 += 4) {
                                        const float4 bv = *reinterpret_cast<const float4*>(b1g + j0 + i2);
                                        const float2 x0 = ffma2(make_float2(__uint_as_float(acc[i2]), __uint_as_float(acc[i2 + 1])),
                                                                make_float2(1.f, 1.f), make_float2(bv.x, bv.y));
                                        const float2 x1 = ffma2(make_float2(__uint_as_float(acc[i2 + 2]), __uint_as_float(acc[i2 + 3])),
                                                                make_float2(1.f, 1.f), make_float2(bv.z, bv.w));
                                        packed[i2 / 2] = act_pack<ACT>(x0.x, x0.y);
                                        packed[i2 / 2 + 1] = act_pack<ACT>(x1.x, x1.y);
                                    }
                                } else {
#pragma unroll
                                    for (int i2 = 0; i2 < kCW; i2 += 2) {
                                        const float b0 = bfar_t ? __ldg(bfar_t + j0 + i2) * kP : b1g[j0 + i2];
                                        const float b1 = bfar_t ? __ldg(bfar_t + j0 + i2 + 1) * kP : b1g[j0 + i2 + 1];
                                        packed[i2 / 2] = act_pack<ACT>(__uint_as_float(acc[i2]) + b0, __uint_as_float(acc[i2 + 1]) + b1);
                                    }
                                }
                            } else if constexpr (!C::BIAS_MMA) {
#pragma unroll
                            for (int i2 = 0; i2 < kCW; i2 += 4) {   // D = kP W a; + kP b (fp32) here
                                const float4 bv = *reinterpret_cast<const float4*>(s_hb + l * H + j0 + i2);
                                const float2 x0 = ffma2(make_float2(__uint_as_float(acc[i2]), __uint_as_float(acc[i2 + 1])),
                                                        make_float2(1.f, 1.f), make_float2(bv.x, bv.y));
                                const float2 x1 = ffma2(make_float2(__uint_as_float(acc[i2 + 2]), __uint_as_float(acc[i2 + 3])),
                                                        make_float2(1.f, 1.f), make_float2(bv.z, bv.w));
                                packed[i2 / 2] = act_pack<ACT>(x0.x, x0.y);
                                packed[i2 / 2 + 1] = act_pack<ACT>(x1.x, x1.y);
                            }
                            } else {
#pragma unroll
                            for (int i2 = 0; i2 < kCW; i2 += 4) {
                                // D = kP (W a + b): bias and pre-scale are already in the accumulator
                                packed[i2 / 2] = act_pack<ACT>(__uint_as_float(acc[i2]), __uint_as_float(acc[i2 + 1]));
                                packed[i2 / 2 + 1] = act_pack<ACT>(__uint_as_float(acc[i2 + 2]), __uint_as_float(acc[i2 + 3]));
                            }
                            }
                            if (h < C::NH - 1) {
#pragma unroll
                                for (int i2 = 0; i2 < kCW / 2; ++i2) keep[k * (kCW / 2) + i2] = packed[i2];
                            } else {
                                // every unit of this layer done: A of the slot is dead -> next input
                                if constexpr (C::NH > 1 && !C::SPLITK)
                                    tmem_st8(tmem + lane_addr + a_col + (uint32_t)((j0 - C::UN) / 2), &keep[k * (kCW / 2)]);
                                tmem_st8(tmem + lane_addr + a_col + (uint32_t)(j0 / 2), packed);
                            }
                        } else {
#pragma unroll
                            for (int i2 = 0; i2 < kCW; i2 += 4) {
                                const float4 wv = *reinterpret_cast<const float4*>(s_wo + j0 + i2);
                                float4 xv = make_float4(__uint_as_float(acc[i2]), __uint_as_float(acc[i2 + 1]),
                                                        __uint_as_float(acc[i2 + 2]), __uint_as_float(acc[i2 + 3]));
                                if constexpr (!C::BIAS_MMA) {   // + kP b of the last hidden layer
                                    const float4 bv = *reinterpret_cast<const float4*>(s_hb + l * H + j0 + i2);
                                    const float2 x0 = ffma2(make_float2(xv.x, xv.y), make_float2(1.f, 1.f), make_float2(bv.x, bv.y));
                                    const float2 x1 = ffma2(make_float2(xv.z, xv.w), make_float2(1.f, 1.f), make_float2(bv.z, bv.w));
                                    xv = make_float4(x0.x, x0.y, x1.x, x1.y);
                                }
                                const uint32_t p0 = act_pack<ACT>(xv.x, xv.y);
                                const uint32_t p1 = act_pack<ACT>(xv.z, xv.w);
                                // output dot in two interleaved partial sums (even / odd neurons)
                                sdot2 = ffma2(make_float2(__uint_as_float(p0 << 16), __uint_as_float(p0 & 0xFFFF0000u)),
                                              make_float2(wv.x, wv.y), sdot2);
                                sdot2 = ffma2(make_float2(__uint_as_float(p1 << 16), __uint_as_float(p1 & 0xFFFF0000u)),
                                              make_float2(wv.z, wv.w), sdot2);
                            }
                        }
                    }
                    if (!last && h == C::NH - 1) {
                        tmem_wait_st();
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) arrive_sched(BAR_AREADY + sl);
                    }
                    if (tracer) TC_TRACE(trole, 5, l, h, sl, i);
                }
            };
            if constexpr (C::L1M) run_layer(std::true_type{}, -1);
#pragma unroll 1
            for (int l = 0; l < G; ++l) {
                run_layer(std::false_type{}, l);
                if constexpr (C::A1S)   // the first GEMM has read the smem A tile: next tile's layer 1
                    if (l == 0 && i + C::NSLOT < n_my) layer1(i + C::NSLOT);
            }
            // ---- output of this tile: combine column groups, FD pair, write
            (void)tile_of;
            part[cgi * kTileRows + row_in_tile] = sdot2.x + sdot2.y;
            named_bar_sync(1 + sl, gthreads);
            if (cgi == 0) {
                float sv = __ldg(b_out);
#pragma unroll
                for (int q2 = 0; q2 < kColGroups; ++q2) sv += part[q2 * kTileRows + row_in_tile];
                const long long row = row0_of(i) + row_in_tile;
                if (row < n_rows && sdf_out) sdf_out[row] = sv;
                if (states_mode) {
                    if (p.rps == 2) {
                        const float s1 = __shfl_xor_sync(0xFFFFFFFFu, sv, 1);
                        const float term = p.w_sdf * __expf(fminf(-sv * p.inv_sdf_scale, p.sdf_exp_max)) -
                                           p.w_guide *
                                               (C::L1M ? (row < n_rows ? __ldg(reinterpret_cast<const float*>(rows + row) + 3) : 0.f)
                                                       : row_of(i).w) *
                                               (s1 - sv) * p.inv_fd_h;
                        if ((lane & 1) == 0 && row < n_rows) terms[row >> 1] = term;
                    } else {
                        const float term = p.model == MPPI_MODEL_PAPER
                                               ? p.q_sdf * fmaxf(p.d_safe - sv, 0.f)   // Eq. 8 hinge
                                               : p.w_sdf * __expf(fminf(-sv * p.inv_sdf_scale, p.sdf_exp_max));
                        if (row < n_rows) terms[row] = term;
                    }
                }
            }
            named_bar_sync(1 + sl, gthreads);   // part[] and the row buffer are reused by this group
            if (FUSE && row_issuer) mbar_arrive_local(bar(BAR_RFREE + (int)(i % kNRB)));   // to the rollout warps
            if (tracer) TC_TRACE(trole, 8, 0, 0, sl, i);
            if constexpr (C::L1M) {
            } else if constexpr (C::A1S) issue_rows(i + 2 * C::NSLOT);   // this tile's row buffer is free now
            else if (i + C::NSLOT < n_my) layer1(i + C::NSLOT);   // next tile of this slot; overlaps the others' MMAs
        }
    }
    // ---- teardown
    __syncwarp();
    tc_fence_before();
    __syncthreads();
    if constexpr (CG == 2) cluster_sync();   // the leader's MMAs wrote into this CTA's TMEM
    tc_fence_after();
    if (warp == 0) {
        if constexpr (CG == 1)
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::TMEM_COLS));
        else
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::TMEM_COLS));
    }
}

template <int H, int G, int ACT, int PEB, bool FUSE = false>
cudaError_t launch_t(const Params& p, const Buffers& b, const float4* rows, long long n_rows, int ctrl_fixed,
                     float* sdf_out, bool states_mode, cudaStream_t s) {
    using C = Cfg<H, G, PEB>;
    // per device (a process may drive several): the dynamic-smem opt-in and the persistent grid size
    constexpr int kMaxDev = 64;
    static int max_groups[kMaxDev] = {};   // co-resident CTA groups (clusters) on the device; 0 = not set up
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDev) return cudaErrorInvalidDevice;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C::CG;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = C::SMEM;
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (max_groups[dev] == 0) {
        cudaError_t e = cudaFuncSetAttribute(k_mlp_tc<H, G, ACT, PEB, FUSE>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
        if (e != cudaSuccess) return e;
        int n_sm = 0;
        cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
        int groups = n_sm / C::CG;
        // with clusters, GPC/TPC floor-sweeping can leave fewer pairs co-resident than SMs/2: a static
        // round-robin over more groups than fit would serialise a second wave
        int clusters = 0;
        cfg.gridDim = dim3((unsigned)(groups * C::CG));
        if (cudaOccupancyMaxActiveClusters(&clusters, k_mlp_tc<H, G, ACT, PEB, FUSE>, &cfg) == cudaSuccess && clusters > 0)
            groups = clusters < groups ? clusters : groups;
        cudaGetLastError();
        if (groups < 1) return cudaErrorInvalidConfiguration;
        max_groups[dev] = groups;
        if (getenv("MPPI_VERBOSE"))
            fprintf(stderr, "[mppi] k_mlp_tc<%d,%d,%d> dev %d: %d SMs, %d co-resident groups of %d CTAs, smem %d B\n", H, G,
                    ACT, dev, n_sm, groups, C::CG, C::SMEM);
    }
    const long long tiles = FUSE ? (long long)p.n_ctrl * (p.K / 128)   // 128-sample blocks
                                 : (n_rows + (long long)kTileRows * C::CG - 1) / ((long long)kTileRows * C::CG);
    if (tiles == 0) return cudaSuccess;
    const long long groups = tiles < max_groups[dev] ? tiles : max_groups[dev];
    cfg.gridDim = dim3((unsigned)(groups * C::CG));
    PEArg<H, G, PEB> pew{};
    if constexpr (sizeof(PEArg<H, G, PEB>) > 1) {
        if (!b.w1pe2_host) return cudaErrorInvalidValue;
        std::memcpy(pew.w, b.w1pe2_host, sizeof(pew.w));
    }
    return cudaLaunchKernelEx(&cfg, k_mlp_tc<H, G, ACT, PEB, FUSE>, pew, p, rows, n_rows, ctrl_fixed, states_mode ? 1 : 0,
                              (const uint8_t*)b.hid_wbf, (const float*)b.hid_b, (const float*)b.w_out,
                              (const float*)b.b_out, (const float4*)b.w1p, (const float*)b.b1f, sdf_out, b.terms,
                              (const float2*)b.w1pe2, b);
}

}  // namespace tc

int mlp_tc_trace_copy(unsigned long long* host, int max_entries) {
#ifdef MPPI_TC_TRACE
    const int n = 4 * 3 * tc::kTraceCap;
    if (max_entries < n) return 0;
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(host, tc::g_tc_trace, sizeof(unsigned long long) * n);
    static unsigned long long zeros[4 * 3 * tc::kTraceCap];
    cudaMemcpyToSymbol(tc::g_tc_trace, zeros, sizeof(zeros));
    return n;
#else
    (void)host;
    (void)max_entries;
    return 0;
#endif
}

bool mlp_tc_supported(int H, int G, int act) {
    return (H == 128 || H == 256) && G >= 1 && G <= 3 && act >= 0 && act <= 2;
}

size_t mlp_tc_weight_bytes(int H, int G) { return (size_t)G * H * H * 2 + (size_t)G * H * 32; }

// Global image = the shared-memory images of the CTA(s) of one MMA group, per rank r:
//  * hidden layers: [layer][unit q] blocks of RB x H bf16 (rank r holds rows [q UN + r RB, +RB) of W_l,
//    UN = 128, RB = UN/CG), scaled by kPre<act> (exact: a power of two); inside a block, [64-wide K chunk]
//    [row n][128 B] with the 16-byte groups of row n XOR-swizzled by (n % 8) (UMMA SWIZZLE_128B, K-major);
//  * hidden biases: [layer][unit q] blocks of RB rows x 16 bf16, row n = [b_hi, b_lo, 0 x 14] with
//    b_hi + b_lo = kPre b (bf16 split of the fp32 value), no swizzle: [n / 8][K core][n % 8][8 bf16].
void mlp_tc_pack_weights(int H, int G, int act, const float* W, const float* hb, uint8_t* out) {
    const int CG = H == 256 ? 2 : 1, NH = H / 128;
    const int UN = H / NH, RB = UN / CG;
    const float kp = act == MPPI_ACT_SILU ? 0.5f : 1.0f;
    const size_t unit = (size_t)RB * H * 2, bunit = (size_t)RB * 32;
    const size_t hidden = (size_t)G * NH * unit;
    const size_t per_rank = hidden + (size_t)G * NH * bunit;
    auto bits_of = [](float v) {
        uint32_t u;
        std::memcpy(&u, &v, 4);
        return (uint16_t)(u >> 16);
    };
    auto bf16_rne = [](float v) {
        uint32_t u;
        std::memcpy(&u, &v, 4);
        u = (u + 0x7FFFu + ((u >> 16) & 1u)) & 0xFFFF0000u;
        float r;
        std::memcpy(&r, &u, 4);
        return r;
    };
    std::memset(out, 0, per_rank * CG);
    for (int r = 0; r < CG; ++r)
        for (int l = 0; l < G; ++l)
            for (int q = 0; q < NH; ++q) {
                uint8_t* blk = out + (size_t)r * per_rank + (size_t)(l * NH + q) * unit;
                uint8_t* bblk = out + (size_t)r * per_rank + hidden + (size_t)(l * NH + q) * bunit;
                for (int nn = 0; nn < RB; ++nn) {
                    const int n = q * UN + r * RB + nn;
                    for (int k = 0; k < H; ++k) {
                        const uint16_t b = bits_of(W[(size_t)l * H * H + (size_t)n * H + k] * kp);   // bf16 value
                        const int kc = k / 64, w = k % 64;
                        const size_t off = (size_t)kc * RB * 128 + (size_t)nn * 128 +
                                           (size_t)(((w / 8) ^ (nn % 8)) * 16) + (size_t)(w % 8) * 2;
                        std::memcpy(blk + off, &b, 2);
                    }
                    const float bv = hb[(size_t)l * H + n] * kp;
                    const float hi = bf16_rne(bv), lo = bf16_rne(bv - hi);
                    const uint16_t pair[2] = {bits_of(hi), bits_of(lo)};
                    std::memcpy(bblk + (size_t)(nn / 8) * 256 + (size_t)(nn % 8) * 16, pair, 4);
                }
            }
}

bool mlp_tc_pe_supported(int H, int n_gemm, int pe_bands) {
    return pe_bands == 0 || (pe_bands == 4 && (H == 128 || H == 256) && n_gemm >= 1 && n_gemm <= 3);
}


cudaError_t launch_mlp_tc(const Params& p, const Buffers& b, const float4* rows, long long n_rows, int ctrl_fixed,
                          float* sdf_out, bool states_mode, cudaStream_t s, bool fuse) {
    if (p.H == 128 && !p.mlp_legacy) return launch_mlp_h128(p, b, rows, n_rows, ctrl_fixed, sdf_out, states_mode, s, fuse);
    if (fuse) {   // H = 256 fused rollout: the configs[2]/[3] MLP shape (ReLU / SiLU), no PE
#define MPPI_TC_FUSE(GG, AA) \
        if (p.H == 256 && p.n_gemm == GG && p.act == AA && p.pe_bands == 0) \
            return tc::launch_t<256, GG, AA, 0, true>(p, b, rows, n_rows, ctrl_fixed, sdf_out, states_mode, s);
#if MPPI_L1_MMA   // (the fused producer runs beside the CUDA-core layer 1 only)
#elif defined(MPPI_TC_QUICK)
        MPPI_TC_FUSE(3, 2)
#else
        MPPI_TC_FUSE(3, 1) MPPI_TC_FUSE(3, 2)
#endif
#undef MPPI_TC_FUSE
        return cudaErrorInvalidValue;
    }
#define MPPI_TC_CASE(HH, GG, AA) \
    if (p.H == HH && p.n_gemm == GG && p.act == AA) \
        return p.pe_bands == 0 ? tc::launch_t<HH, GG, AA, 0>(p, b, rows, n_rows, ctrl_fixed, sdf_out, states_mode, s) \
                               : tc::launch_t<HH, GG, AA, 4>(p, b, rows, n_rows, ctrl_fixed, sdf_out, states_mode, s);
#define MPPI_TC_CASE0(HH, GG, AA) \
    if (p.H == HH && p.n_gemm == GG && p.act == AA && p.pe_bands == 0) \
        return tc::launch_t<HH, GG, AA, 0>(p, b, rows, n_rows, ctrl_fixed, sdf_out, states_mode, s);
#define MPPI_TC_ACTS(HH, GG) MPPI_TC_CASE(HH, GG, 0) MPPI_TC_CASE(HH, GG, 1) MPPI_TC_CASE(HH, GG, 2)
    // H = 128 runs kernel_mlp_h128.cu; its round-1 form here stays for A/B (MPPI_H128_LEGACY=1, configs[1]/[4] MLP)
    MPPI_TC_CASE0(128, 2, 1)
#ifdef MPPI_TC_QUICK   // development builds: the configs[2..3] instantiations only
    MPPI_TC_CASE(256, 3, 2)
#else
    MPPI_TC_ACTS(256, 1) MPPI_TC_ACTS(256, 2) MPPI_TC_ACTS(256, 3)
#endif
#undef MPPI_TC_ACTS
#undef MPPI_TC_CASE
#undef MPPI_TC_CASE0
    return cudaErrorInvalidValue;
}

}  // namespace mppi
