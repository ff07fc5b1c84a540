// Internal declarations shared by the host orchestrator and the kernels of the B200 MPPI path.
// Nothing here is shared with oracle/ (the CPU checker is independent by construction).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace mppi {

// Softmin record: (m, S, S2, SJ, N, 0, 0, 0, V[T][4]) per controller -- min cost, sum of weights relative
// to m, sum of squared weights, sum and count of the finite costs, weighted control deviations.
constexpr int kRecHead = 8;

// Per-step constants, passed by value to every kernel.
struct Params {
    int n_ctrl, K, T;
    int rps;              // query rows per state: 2 with FD guidance (p_c, p_c + h d), else 1
    int H, L, n_gemm;     // hidden width, latent dim, hidden->hidden GEMM layers (n_hidden - 1)
    int act;              // MPPI_ACT_*
    int K_global;
    long long k_offset;
    long long ctrl_offset;   // global index of this context's first controller (noise counters)
    float dt, inv_lambda, mass, gravity;
    float u_lo[4], u_hi[4], sigma[4];
    float w_goal, w_sdf, inv_sdf_scale, sdf_exp_max, w_u, w_guide, fd_h, inv_fd_h;
    unsigned long long seed;
    // MPPI_MODEL_PAPER (reading P1-P6)
    int model;
    float arm_d, kappa;              // arm / sqrt(2) (rotor offset along each body axis), yaw moment per thrust
    float Jx, Jy, Jz, inv_Jx, inv_Jy, inv_Jz;
    float thrust_max, rate_max, q_gate, q_vis, q_sdf, d_safe;
    // MPPI_SDF_GATE
    int sdf_provider;
    float gate_c, gate_tana;
    int pe_bands;         // positional encoding bands (0 or 4)
    int mlp_legacy;       // 1: H = 128 runs the round-1 kernel_mlp_tc form (A/B only, env MPPI_H128_LEGACY=1)
    int noise_device;     // MPPI_NOISE_DEVICE: the rollout generates the noise (and stores it for k_softmin)
};

// Device buffers of one context (all inside the workspace).
struct Buffers {
    // MLP weights
    float4* w1p;          // [H] (W1[j][0..2], unused) layer-1 position columns
    float* w1pe;          // [H][3 + 6 pe_bands] layer-1 positional-encoding columns (pe_bands > 0)
    float2* w1pe2;        // [H/2][3 + 6 pe_bands] the same, neuron-pair major, x kPre (H = 256 PE layer 1)
    const float2* w1pe2_host;   // HOST copy of w1pe2 (launch-time kernel parameter of the H = 256 PE kernel)
    float* w1z;           // [H][L] layer-1 latent columns (for the fold)
    float* b1;            // [H]
    float* b1f;           // [n_ctrl][H] folded bias b1' = W1z z + b1
    float* hid_w32;       // fp32 mode: [n_gemm][H][H]
    uint8_t* hid_wbf;     // bf16 mode: [n_gemm] swizzled UMMA B images (see kernel_mlp_tc.cu)
    float* hid_b;         // [n_gemm][H]
    float* w_out;         // [H] (bf16-rounded values in bf16 mode)
    float* b_out;         // [1]
    // controller state
    float* z;             // [n_ctrl][L]
    float* Tq;            // [n_ctrl][12]
    float* x0;            // [n_ctrl][10]
    float* goal;          // [n_ctrl][3]
    unsigned long long* step;  // [1] step index of the current step
    float* U_out;         // [n_ctrl][T][4] latest nominal (result of the last update)
    float* U_nom;         // [n_ctrl][T][4] nominal used by the current step (shifted U_out)
    float4* noise;        // [T][n_ctrl*K] standard normals
    float4* rows;         // [n_ctrl*T*K*rps] query rows
    float* sdf_rows;      // [n_ctrl*T*K*rps] s per row (debug)
    float* terms;         // [n_ctrl*T*K] SDF-dependent stage cost
    float* partial;       // [n_ctrl*K] non-SDF cost sums
    float* J;             // [n_ctrl*K]
    unsigned* tickets;    // [n_ctrl] + [n_ctrl][groups] k_softmin arrivals this step (reset by the last block)
    float* blkrec;        // [n_ctrl][softmin blocks][kRecHead + 4T] per-block records, then [n_ctrl][groups][...]
    float* record;        // [n_ctrl][kRecHead + 4T]  this rank's record
    float* gathered;      // [world][n_ctrl][kRecHead + 4T]
    float* weights;       // [n_ctrl][K] normalised softmin weights (debug, on demand)
    float* diag;          // [n_ctrl][4]
    int* flags;           // [n_ctrl]
};

// Launchers (kernels_simt.cu)
void launch_noise_shift(const Params& p, const Buffers& b, bool gen_noise, cudaStream_t s);
void launch_rollout(const Params& p, const Buffers& b, bool device_noise, cudaStream_t s);   // + noise + shift
void launch_mlp_simt(const Params& p, const Buffers& b, const float4* rows, long long n_rows, int ctrl_fixed,
                     float* sdf_out, bool states_mode, cudaStream_t s);
void launch_softmin(const Params& p, const Buffers& b, bool write_record, cudaStream_t s);
int softmin_blocks(int K);
int softmin_group_count(int K);   // group records / tickets of the two-level combine (0: one level)
void launch_combine(const Params& p, const Buffers& b, const float* recs, int R, cudaStream_t s);
void launch_fold(const Params& p, const Buffers& b, int ctrl_begin, int ctrl_count, cudaStream_t s);
void launch_weights(const Params& p, const Buffers& b, cudaStream_t s);   // debug: normalised softmin weights
// analytic Gate-SDF (Eq. 2) on the step's query rows -> SDF stage terms (replaces the MLP launch)
void launch_sdf_gate(const Params& p, const Buffers& b, float* sdf_out, cudaStream_t s);

// tcgen05 / TMEM SDF-MLP (kernel_mlp_tc.cu)
bool mlp_tc_supported(int H, int n_gemm, int act);
int mlp_tc_trace_copy(unsigned long long* host, int max_entries);   // debug builds (MPPI_TC_TRACE) only
size_t mlp_tc_weight_bytes(int H, int n_gemm);
// Lay out bf16 weights of the n_gemm hidden layers (host, [l][H][H] fp32 nn.Linear order, already
// bf16-representable) in the swizzled UMMA image the kernel copies to shared memory.
// The hidden biases hb [n_gemm][H] go into the same image (added by the tensor cores).
void mlp_tc_pack_weights(int H, int n_gemm, int act, const float* W, const float* hb, uint8_t* out);
// rows_mode: rows are per-state query rows of the step (writes per-state SDF terms) when states_mode,
// else arbitrary rows for mppi_sdf_eval (writes s per row only).
// fuse: the rollout runs inside the kernel (states mode, CTBR model, guidance on; H = 128: K % 64 == 0,
// H = 256: K % 128 == 0 and the configs[2]/[3] MLP shape); rows are then unused
cudaError_t launch_mlp_tc(const Params& p, const Buffers& b, const float4* rows, long long n_rows, int ctrl_fixed,
                          float* sdf_out, bool states_mode, cudaStream_t s, bool fuse = false);
bool mlp_tc_pe_supported(int H, int n_gemm, int pe_bands);

// H = 128 tcgen05 SDF-MLP with shared-memory A operands and layer 1 on the tensor cores (kernel_mlp_h128.cu)
bool mlp_h128_supported(int n_gemm, int pe_bands);
int mlp_h128_trace_copy(unsigned long long* host, int max_entries);   // debug builds (MPPI_TC_TRACE) only
int softmin_trace_copy(unsigned long long* host, int max_entries);   // debug builds (MPPI_TC_TRACE) only
size_t mlp_h128_image_bytes(int n_gemm, int pe_bands);   // hidden image (as mlp_tc_pack_weights) + layer-1 B
void mlp_h128_pack_l1(int pe_bands, int act, const float* w1pos, uint8_t* out);
// fuse: the rollout runs inside the kernel (CTBR model, guidance on, K % 64 == 0, states_mode): rows unused
cudaError_t launch_mlp_h128(const Params& p, const Buffers& b, const float4* rows, long long n_rows, int ctrl_fixed,
                            float* sdf_out, bool states_mode, cudaStream_t s, bool fuse = false);

}  // namespace mppi
