/*
 * mppi.h — C ABI of the B200 (sm_100a) MPPI + Gate-SDF hot path (arxiv 2603.07199).
 *
 * One call of mppi_step() is one MPPI iteration (§IV-A, Eq. 5) per controller:
 *   sample   u_{k,t} = clamp(U*_t + sigma (.) n_{k,t})
 *   rollout  x_{k,t+1} = RK4(x_{k,t}, u_{k,t}) (CTBR quadrotor)             PAPER.md:146; BASELINE configs[0]
 *   query    s = g_phi(z, p_c), p_c = R_q p + t_q in the cached frame
 *   cost     J_k = sum_t w_goal|p-g_c|^2 + w_sdf e^{-s/scale} + w_u|u|^2
 *                        - w_guide grad(s).v                                 PAPER.md:185 (Eq. 10 structure);
 *                                                                            BASELINE configs[0..1] terms
 *   update   U* <- sum_k softmax(-J/lambda)_k u_k                            PAPER.md:141 (Eq. 5)
 * The latent code z enters only through a per-frame first-layer bias b1' = W1[:,3:] z + b1
 * ("latent duplicated M x K times and concatenated", folded; "encode ... once").
 *
 * Conventions: all arrays are little-endian, row-major, fp32 unless stated. State x = [p(3), v(3),
 * q(w,x,y,z)]; control u = [c (N), wx, wy, wz (rad/s, body frame)] (MPPI_MODEL_PAPER: see below; the
 * state dimension is 17 and u is the rotor thrust rates); MLP weights in nn.Linear order
 * W[out][in], layer-1 input columns [p_c(3) | z(L)]. Units: m, s, N, rad.
 *
 * Ownership: the caller owns the device workspace (>= mppi_workspace_bytes()) and must keep it alive
 * until mppi_destroy(); pass NULL to let the library cudaMalloc it. Setters copy their host arrays
 * before returning. mppi_step() enqueues work on cfg.stream and returns immediately (x0/goal are staged
 * in pinned memory, so the caller may reuse them). mppi_get_controls() synchronises the stream and is
 * where asynchronous failures surface.
 *
 * Errors: every call returns an mppi_status. Invalid arguments leave the context untouched. A CUDA or
 * NCCL error poisons the context: every later call except mppi_destroy() returns MPPI_ERR_POISONED.
 * mppi_last_error() returns a thread-local message for the last failure on this thread.
 * A context is single-caller; distinct contexts are independent.
 */
#ifndef MPPI_B200_H
#define MPPI_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MPPI_ABI_VERSION 3

typedef struct mppi_ctx mppi_ctx;
typedef int32_t mppi_status;

enum {
    MPPI_OK = 0,
    MPPI_ERR_INVALID = -1,     /* bad argument / config; context untouched                       */
    MPPI_ERR_CUDA = -2,        /* CUDA runtime error; context poisoned                            */
    MPPI_ERR_NCCL = -3,        /* NCCL error; context poisoned                                    */
    MPPI_ERR_NOT_READY = -4,   /* step before weights and every latent were set                   */
    MPPI_ERR_NONFINITE = -5,   /* every J of some controller was non-finite; its U* is unchanged  */
    MPPI_ERR_OOM = -6,         /* workspace too small / allocation failed                         */
    MPPI_ERR_POISONED = -7,    /* an earlier CUDA/NCCL error poisoned this context                */
    MPPI_ERR_UNSUPPORTED = -8  /* valid config this build has no kernel for       */
};
enum { MPPI_ACT_SOFTPLUS = 0, MPPI_ACT_RELU = 1, MPPI_ACT_SILU = 2 };
enum { MPPI_MLP_FP32 = 0, MPPI_MLP_BF16 = 1 };
enum { MPPI_NOISE_DEVICE = 0, MPPI_NOISE_EXTERNAL = 1 };
/* MPPI_MODEL_BASELINE: the CTBR dynamics and cost terms of BASELINE configs[0..4] (above).
 * MPPI_MODEL_PAPER: the paper's own model (SURVEY.md §8f F1 + F2; readings P1-P7):
 *   state x = [p(3), v(3), q(w,x,y,z)(4), w(3) body rates, T(4) rotor thrusts] (17 floats),
 *   control u = [T1dot..T4dot] (N/s), X-configuration rigid body, RK4 with T clamped to
 *   [0, thrust_max] and w to +-rate_max after each step;
 *   J = sum_{k=0}^{T-1} q_gate (|p_{k+1} - g|^2 - |p_k - g|^2) + q_vis (1 - cos(psi_k - psi_gate,k))
 *       + q_sdf max(0, d_safe - s(p_k))                      (Eqs. 6-10),
 *   so the SDF is queried at x_0..x_{T-1}; w_goal, w_sdf, sdf_scale, w_u are unused and w_guide must be 0. */
enum { MPPI_MODEL_BASELINE = 0, MPPI_MODEL_PAPER = 1 };
/* SDF provider. MPPI_SDF_MLP: the neural Gate-SDF g_phi(z, p_c) (weights + latents).
 * MPPI_SDF_GATE: the analytic Gate-SDF of Eq. 2, s = gate_c + |x| gate_tana - max(|y|, |z|)
 * with p_c = (x, y, z) in the query frame, which must then be the gate frame (gate plane x = 0); no
 * weights are needed and mppi_set_latent only sets T_q (z is ignored). */
enum { MPPI_SDF_MLP = 0, MPPI_SDF_GATE = 1 };

typedef struct {
    int32_t abi_version;       /* MPPI_ABI_VERSION                                                 */
    int32_t n_ctrl;            /* controllers in this context (configs[4]: drones on this GPU), >=1 */
    int32_t K, T;              /* K: samples per controller ON THIS RANK; T: horizon steps          */
    int32_t K_global;          /* samples per controller over all ranks (== K when world_size==1)   */
    int64_t k_offset;          /* this rank's first global sample index (rank * K in configs[3])    */
    float dt, lambda, mass, gravity;            /* configs[0]: 0.02, 1.0, 1.0, 9.81                 */
    float u_lo[4], u_hi[4];                     /* [0,-6,-6,-6], [4 m g, 6, 6, 6]                   */
    float sigma[4];                             /* [2, 1, 1, 1]                                      */
    float w_goal, w_sdf, sdf_scale, sdf_exp_max, w_u, w_guide, fd_h;  /* 1, 50, 0.1, 80, 0.01, 0.5|0, 0.1 */
    int32_t latent_dim, hidden, n_hidden;       /* L; width H; hidden layers incl. layer 1          */
    int32_t activation, mlp_dtype;              /* MPPI_ACT_*, MPPI_MLP_*                           */
    int32_t noise_mode;                         /* MPPI_NOISE_*                                     */
    uint64_t seed;                              /* Philox key (device noise)                        */
    int32_t world_size, rank;                   /* sample sharding over ranks (configs[3])          */
    const void* nccl_unique_id;                 /* 128-byte ncclUniqueId; NULL: no NCCL (split-phase).
                                                   Non-NULL also with world_size 1 (exercises the path) */
    int32_t device;                             /* CUDA device ordinal                              */
    void* stream;                               /* cudaStream_t all work is enqueued on (0: legacy) */
    /* ABI 2 */
    int32_t model;                              /* MPPI_MODEL_*                                     */
    float arm, kappa;                           /* MPPI_MODEL_PAPER: rotor arm (m), yaw moment per thrust (m) */
    float inertia[3];                           /* MPPI_MODEL_PAPER: diag(J) (kg m^2)               */
    float thrust_max, rate_max;                 /* MPPI_MODEL_PAPER: rotor thrust (N), body-rate (rad/s) limits */
    float q_gate, q_vis, q_sdf, d_safe;         /* MPPI_MODEL_PAPER: Eq. 10 weights, Eq. 8 clearance (m) */
    int32_t sdf_provider;                       /* MPPI_SDF_*                                       */
    float gate_c, gate_tana;                    /* MPPI_SDF_GATE: inner half-width c (m), tan(alpha) */
    int32_t pe_bands;                           /* positional encoding of the SDF input:
                                                   0, or 4 (bf16 MLP, hidden 128 or 256): layer 1 reads
                                                   [p, sin(2^i pi p), cos(2^i pi p) (i < 4) | z], i.e.
                                                   in_dim[0] = 3 + 6 pe_bands + latent_dim (E1) */
    /* ABI 3 */
    int64_t ctrl_offset;                        /* global index of this context's first controller when the
                                                   controllers of one job are split over contexts/ranks
                                                   (configs[4]); keys the device noise, so the split job draws
                                                   the unsplit job's samples. 0 otherwise */
} mppi_config;

/* Bytes of device workspace mppi_create() needs for this config (0 if the config is invalid). */
size_t mppi_workspace_bytes(const mppi_config* cfg);

/* Validate cfg, bind the workspace (NULL: library-allocated), create the context: one MPPI controller
 * state (U*, weights, latent cache) per controller of the batch. With
 * world_size > 1 and a non-NULL nccl_unique_id this is collective over all ranks (ncclCommInitRank).
 * Errors: MPPI_ERR_INVALID / MPPI_ERR_UNSUPPORTED (bad or unbuilt config; *out = NULL), MPPI_ERR_OOM,
 * MPPI_ERR_CUDA, MPPI_ERR_NCCL. */
mppi_status mppi_create(const mppi_config* cfg, void* d_workspace, size_t ws_bytes, mppi_ctx** out);
/* Wait for the context's queued work, then release everything it owns (not a caller workspace).
 * NULL is a no-op. Always MPPI_OK; also valid on a poisoned context. */
mppi_status mppi_destroy(mppi_ctx* ctx);

/* Fill out128 with a fresh ncclUniqueId (rank 0; the caller broadcasts it, e.g. torch.distributed). */
mppi_status mppi_get_nccl_unique_id(void* out128);

/* Dense layers of g_phi: n_layers = n_hidden + 1; layer l has shape
 * W[l]: [out_dim[l]][in_dim[l]] and b[l]: [out_dim[l]], host fp32. Layer 0 is [H][3+L]; layers
 * 1..n_hidden-1 are [H][H]; the last is [1][H]. In MPPI_MLP_BF16 mode the hidden and output weights
 * are rounded once to bf16 (RNE) here; layer 0 and every bias stay fp32 (reading R15).
 * Invalidates every latent fold (mppi_set_latent must be called again). */
mppi_status mppi_set_sdf_weights(mppi_ctx* ctx, int32_t n_layers, const int32_t* in_dim, const int32_t* out_dim,
                                 const float* const* W, const float* const* b);

/* Per-frame latent code z [L] and cached world->query-frame transform T_q = (R row-major 3x3, t[3])
 * for controller ctrl. Folds b1' = W1[:,3:] z + b1 on the device. ctrl = -1 sets every
 * controller from arrays z [n_ctrl][L] and T_q [n_ctrl][12]. Requires weights. */
mppi_status mppi_set_latent(mppi_ctx* ctx, int32_t ctrl, const float* z, const float* T_q);

/* Latent cache with object permanence (§IV-B3: "we cache the latest valid latent code
 * and its corresponding camera pose ... under visual occlusion the SDF is queried in the cached frame").
 * valid != 0: a valid depth frame -- as mppi_set_latent, and t_frame (caller's clock, s) is recorded.
 * valid == 0: an invalid/occluded frame -- nothing is uploaded; the cached (z, T_q) of the last valid
 * frame stays in use (z / T_q may be NULL). Either way the frame is counted. Before the first valid frame
 * of a controller, stepping returns MPPI_ERR_NOT_READY. ctrl = -1: every controller (arrays as above). */
mppi_status mppi_set_latent_frame(mppi_ctx* ctx, int32_t ctrl, const float* z, const float* T_q, double t_frame,
                                  int32_t valid);
/* Cache status per controller: out_t [n_ctrl] = t_frame of the cached (last valid) frame (NaN when it came
 * from mppi_set_latent), out_steps [n_ctrl] = mppi_step calls since it was set (the latent's age in
 * iterations), out_invalid [n_ctrl] = invalid frames seen since then. Any pointer may be NULL. */
mppi_status mppi_get_latent_status(mppi_ctx* ctx, double* out_t, int64_t* out_steps, int64_t* out_invalid);

/* Nominal sequence U* [T][4] for controller ctrl (ctrl = -1: [n_ctrl][T][4]); resets the warm start. */
mppi_status mppi_set_nominal(mppi_ctx* ctx, int32_t ctrl, const float* U);

/* MPPI_NOISE_EXTERNAL: standard normals n [T][n_ctrl*K][4] (device pointer, fp32), copied on the stream.
 * Each step uses the last noise set (sigma is applied inside the step). */
mppi_status mppi_set_noise(mppi_ctx* ctx, const float* d_noise);

/* One MPPI iteration. x0 [n_ctrl][10] (MPPI_MODEL_PAPER: [n_ctrl][17]), goal g_c [n_ctrl][3] (the
 * paper model's waypoint p_wp) are HOST arrays. If step_index > 0 the
 * nominal is first shifted (U*_t <- U*_{t+1}, last repeated). step_index also keys the
 * device noise. world_size > 1 with NCCL: includes the all-gather + combine; without NCCL the caller
 * uses mppi_step_local / mppi_step_finish. Async; returns MPPI_ERR_NOT_READY before weights/latents. */
mppi_status mppi_step(mppi_ctx* ctx, const float* x0, const float* goal, uint64_t step_index);
/* Same, with x0 / goal already resident in device memory. */
mppi_status mppi_step_device(mppi_ctx* ctx, const float* d_x0, const float* d_goal, uint64_t step_index);

/* Split-phase sharded step (configs[3] without an NCCL communicator, e.g. emulated ranks):
 * mppi_step_local runs sample..cost and writes this rank's record (m_r, S_r, S2_r, SJ_r, N_r, 0, 0, 0,
 * V_r[T][4]) per controller (S2 = sum of squared weights, for the ESS diagnostic; SJ / N = sum / count of
 * the finite costs, for the mean cost); mppi_record_size() is the record length in floats per controller
 * (8 + 4T); mppi_get_record_device()
 * returns the device pointer of [n_ctrl][record]; mppi_step_finish combines R gathered records
 * (device [R][n_ctrl][record], rank order) into U*. */
mppi_status mppi_step_local(mppi_ctx* ctx, const float* x0, const float* goal, uint64_t step_index);
int32_t mppi_record_size(const mppi_ctx* ctx);
const float* mppi_get_record_device(const mppi_ctx* ctx);
mppi_status mppi_step_finish(mppi_ctx* ctx, const float* d_records, int32_t R);

/* Synchronise and copy the updated U* [n_ctrl][T][4] (Eq. 5) and u0 = U*[:,0,:] [n_ctrl][4]
 * (if non-NULL; "only the first action ... is applied") to host. Returns
 * MPPI_ERR_NONFINITE if every J of some controller was non-finite in the last step (that controller's U*
 * is left unchanged); MPPI_ERR_NCCL (context poisoned) if the communicator reports an asynchronous error. */
mppi_status mppi_get_controls(mppi_ctx* ctx, float* U_out, float* u0_out);

/* Synchronise; out [n_ctrl][4] = (J_min, S = sum w~, ESS = S^2 / sum w~^2, mean of the finite J; +inf if
 * none) of the last step (SPEC.md:349 per-step diagnostics). */
mppi_status mppi_get_diagnostics(mppi_ctx* ctx, float* out);

/* Test support: copy an internal buffer of the last step to host (synchronises).
 * MPPI_DBG_QUERIES: [n_ctrl][T][K][rps][4] query rows (p_c, |v|) / (p_c + h d, 0), rps = 2 if w_guide != 0
 * MPPI_DBG_SDF:     [n_ctrl][T][K][rps] s per row     MPPI_DBG_COSTS: [n_ctrl][K] J
 * MPPI_DBG_NOISE:   [T][n_ctrl*K][4] standard normals used   MPPI_DBG_TERMS: [n_ctrl][T][K] SDF stage terms
 * MPPI_DBG_PARTIAL: [n_ctrl][K] non-SDF cost sums   MPPI_DBG_RECORD: [n_ctrl][8 + 4T] this rank's record
 * MPPI_DBG_WEIGHTS: [n_ctrl][K] normalised softmin weights w_k = e^{-(J_k - J_min)/lambda} / S of the last
 *                   full step (Eq. 5; computed on the device on demand) */
enum { MPPI_DBG_QUERIES = 0, MPPI_DBG_SDF = 1, MPPI_DBG_COSTS = 2, MPPI_DBG_NOISE = 3, MPPI_DBG_TERMS = 4,
       MPPI_DBG_PARTIAL = 5, MPPI_DBG_RECORD = 6, MPPI_DBG_WEIGHTS = 7 };
mppi_status mppi_debug_copy(mppi_ctx* ctx, int32_t what, void* host_dst, size_t bytes);

/* Test support: on != 0 makes every later step also write s per query row (the buffer behind
 * MPPI_DBG_SDF, 4 B per row of extra HBM traffic); off by default, when MPPI_DBG_SDF returns
 * MPPI_ERR_NOT_READY. Takes effect from the next step (the step graph is re-captured). */
mppi_status mppi_set_debug_outputs(mppi_ctx* ctx, int32_t on);

/* Test support: run the production SDF-MLP kernel of this context on n query-frame rows
 * d_rows [n][4] (x, y, z, unused; device fp32) with controller ctrl's folded latent, writing s [n]
 * (device fp32) to d_out. Asynchronous on cfg.stream. */
mppi_status mppi_sdf_eval(mppi_ctx* ctx, int32_t ctrl, const float* d_rows, int64_t n, float* d_out);

/* Profiling: level 1 records CUDA events (captured in the step graph) around the SDF-MLP launch only;
 * level 2 around every stage (each event node costs ~2 us of step time); 0 off.
 * mppi_get_kernel_times() synchronises and returns the last step's per-stage device times in ms:
 * out[0] (noise + shift, fused into the rollout: ~0), [1] rollout, [2] SDF-MLP, [3] softmin (cost + min +
 * weights + update or record), [4] NCCL exchange + combine; stages not measured at level 1 read 0. */
mppi_status mppi_set_profiling(mppi_ctx* ctx, int32_t level);
mppi_status mppi_get_kernel_times(mppi_ctx* ctx, float* out, int32_t n_out);
/* Number of kernels this library launches per mppi_step (for the bench's gpu_launches count). */
int32_t mppi_kernels_per_step(const mppi_ctx* ctx);
/* 1 if the step runs the rollout inside the SDF-MLP kernel (opt-in: env MPPI_FUSED=1 at mppi_create; CTBR model,
 * guidance on; H = 128 with K % 64 == 0, H = 256 with K % 128 == 0; off while debug outputs are on):
 * the query rows then never reach HBM and MPPI_DBG_QUERIES returns MPPI_ERR_NOT_READY. */
int32_t mppi_fused_rollout(const mppi_ctx* ctx);

/* Debug builds only (compiled with -DMPPI_TC_TRACE): copy up to max_entries timeline records to host_out and
 * return the count (0 in release builds). Which log: env MPPI_TRACE_H128=1 the H = 128 SDF-MLP kernel
 * (clock64 records of its first CTAs), MPPI_TRACE_SOFTMIN=1 k_softmin ([1024 blocks][10] %globaltimer stamps of
 * controller 0), else the H = 256 SDF-MLP kernel. Test tooling (tests/trace_*.py); not part of the method. */
int32_t mppi_debug_trace(uint64_t* host_out, int32_t max_entries);

const char* mppi_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* MPPI_B200_H */
