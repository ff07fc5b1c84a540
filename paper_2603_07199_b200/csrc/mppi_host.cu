// Host side of the C ABI declared in include/mppi.h: validation, workspace layout, weight packing,
// latent fold, CUDA-graph capture of the per-step launch sequence, NCCL exchange, profiling events.
#include <cuda_runtime.h>
#include <nccl.h>

#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/mppi.h"
#include "mppi_internal.cuh"

using namespace mppi;

namespace {

thread_local std::string g_err;

mppi_status fail(mppi_status st, const std::string& msg) {
    g_err = msg;
    return st;
}

constexpr int kStaging = 4;
// the fused rollout is opt-in (MPPI_FUSED=1); these switch it on by default for large problems
constexpr bool kFuse128Default = true;    // configs[4]: -0.35% device, -1.2% end to end, -1.68 GB DRAM per step
constexpr bool kFuse256Default = false;
constexpr int kNumStages = 5;   // noise+shift, rollout, mlp, cost, update

struct Layout {
    size_t off[32];
    size_t total;
};

enum BufId {
    B_W1P, B_W1PE, B_W1PE2, B_W1Z, B_B1, B_B1F, B_HW32, B_HWBF, B_HB, B_WOUT, B_BOUT, B_Z, B_TQ, B_X0, B_GOAL, B_STEP, B_UOUT,
    B_UNOM, B_NOISE, B_ROWS, B_SDF, B_TERMS, B_PART, B_J, B_TICK, B_BLKREC, B_REC, B_GATH, B_DIAG, B_FLAGS, B_WGT,
    B_COUNT
};

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

int state_dim_of(const mppi_config* c) { return c->model == MPPI_MODEL_PAPER ? 17 : 10; }
// bytes of x0 [n][sd] + goal [n][3], rounded up to 8 (the step index follows)
size_t step_inputs_bytes(const mppi_config* c) { return ((size_t)4 * c->n_ctrl * (state_dim_of(c) + 3) + 7) / 8 * 8; }
size_t step_block_bytes(const mppi_config* c) { return step_inputs_bytes(c) + 8; }

bool compute_layout(const mppi_config* c, Layout* L) {
    const size_t n = (size_t)c->n_ctrl, K = (size_t)c->K, T = (size_t)c->T, H = (size_t)c->hidden;
    const size_t Ld = (size_t)c->latent_dim, G = (size_t)(c->n_hidden - 1);
    const size_t rps = c->w_guide != 0.f ? 2 : 1;
    const size_t world = (size_t)(c->world_size > 0 ? c->world_size : 1);
    const size_t recw = kRecHead + 4 * T;
    size_t sz[B_COUNT];
    sz[B_W1P] = 16 * H;
    sz[B_W1PE] = 4 * H * (size_t)(3 + 6 * c->pe_bands);
    sz[B_W1PE2] = 4 * H * (size_t)(3 + 6 * c->pe_bands);
    sz[B_W1Z] = 4 * H * Ld;
    sz[B_B1] = 4 * H;
    sz[B_B1F] = 4 * n * H;
    sz[B_HW32] = c->mlp_dtype == MPPI_MLP_FP32 ? 4 * G * H * H : 0;
    sz[B_HWBF] = c->mlp_dtype == MPPI_MLP_BF16 ? mlp_tc_weight_bytes((int)H, (int)G) : 0;
    if (c->mlp_dtype == MPPI_MLP_BF16 && H == 128) sz[B_HWBF] = mlp_h128_image_bytes((int)G, c->pe_bands);
    sz[B_HB] = 4 * G * H;
    sz[B_WOUT] = 4 * H;
    sz[B_BOUT] = 16;
    sz[B_Z] = 4 * n * Ld;
    sz[B_TQ] = 4 * n * 12;
    // x0, goal and the step index are one contiguous block (one H2D copy per step): [x0 | goal | pad | step]
    sz[B_X0] = step_block_bytes(c);
    sz[B_GOAL] = 0;
    sz[B_STEP] = 0;
    sz[B_UOUT] = 16 * n * T;
    sz[B_UNOM] = 16 * n * T;
    sz[B_NOISE] = 16 * T * n * K;
    sz[B_ROWS] = 16 * n * T * K * rps + 16 * 128;   // + one tile of slack for tile-granular loads
    sz[B_SDF] = 4 * n * T * K * rps + 4 * 128;
    sz[B_TERMS] = 4 * n * T * K;
    sz[B_PART] = 4 * n * K;
    sz[B_J] = 4 * n * K;
    sz[B_TICK] = 4 * n * (1 + (size_t)softmin_group_count(c->K));
    sz[B_BLKREC] = 4 * n * (size_t)(softmin_blocks(c->K) + softmin_group_count(c->K)) * recw;
    sz[B_REC] = 4 * n * recw;
    sz[B_GATH] = 4 * world * n * recw;
    sz[B_DIAG] = 16 * n;
    sz[B_FLAGS] = 4 * n;
    sz[B_WGT] = 4 * n * K;
    size_t o = 0;
    for (int i = 0; i < B_COUNT; ++i) {
        o = align_up(o, 1024);
        L->off[i] = o;
        o += sz[i];
    }
    L->total = align_up(o, 1024);
    return true;
}

uint16_t bf16_bits_rne(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    if ((u & 0x7F800000u) == 0x7F800000u) return (uint16_t)((u >> 16) | ((u & 0x007FFFFFu) ? 0x40 : 0));
    u += 0x7FFFu + ((u >> 16) & 1u);
    return (uint16_t)(u >> 16);
}
float bf16_value(float f) {
    uint32_t u = (uint32_t)bf16_bits_rne(f) << 16;
    float r;
    std::memcpy(&r, &u, 4);
    return r;
}

}  // namespace

struct mppi_ctx {
    mppi_config cfg{};
    Params p{};
    Buffers b{};
    Layout lay{};
    void* ws = nullptr;
    bool own_ws = false;
    cudaStream_t stream = nullptr;   // caller's stream (cfg.stream; may be the legacy default stream)
    cudaStream_t work = nullptr;     // internal non-blocking stream the step graph is captured/launched on
    cudaEvent_t ev_in = nullptr, ev_out = nullptr;
    bool poisoned = false;
    bool weights = false;
    std::vector<char> latent_set;
    bool use_tc = false;
    bool fused = false;              // the step runs the rollout inside the H = 128 SDF-MLP kernel
    bool last_fused = false;
    // pinned staging ring for x0 / goal / step
    float* h_stage[kStaging] = {};
    float* h_out = nullptr;          // pinned readback of U* [n_ctrl][T][4] and the flags [n_ctrl]
    cudaEvent_t stage_ev[kStaging] = {};
    int stage_i = 0;
    // graphs: [0] full step, [1] local (record) step
    cudaGraphExec_t graph[2] = {nullptr, nullptr};
    int profiling = 0;   // 0 off, 1 events around the SDF-MLP launch only, 2 every stage boundary
    int debug_outputs = 0;   // write s per query row in the step (MPPI_DBG_SDF)
    cudaEvent_t prof_ev[kNumStages + 1] = {};
    bool prof_valid = false;
    ncclComm_t comm = nullptr;
    ncclResult_t nccl_err = ncclSuccess;   // last NCCL call's result inside the step capture
    int last_mode = -1;
    // latent cache status per controller: frame time, steps and invalid frames since
    std::vector<double> latent_t;
    std::vector<int64_t> latent_steps, latent_invalid;
    std::vector<float> w1pe2_host;   // pair-major kPre-scaled layer-1 position/PE weights (kernel parameter)
};

// Every entry point that touches the device runs on the context's device and restores the caller's.
struct DeviceGuard {
    int prev = -1;
    bool changed = false;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) == cudaSuccess && prev != dev) changed = cudaSetDevice(dev) == cudaSuccess;
    }
    ~DeviceGuard() {
        if (changed) cudaSetDevice(prev);
    }
};

#define CUDA_TRY(ctx, expr)                                                                             \
    do {                                                                                                \
        cudaError_t _e = (expr);                                                                        \
        if (_e != cudaSuccess) {                                                                        \
            if (ctx) (ctx)->poisoned = true;                                                            \
            return fail(MPPI_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));             \
        }                                                                                               \
    } while (0)

#define NCCL_TRY(ctx, expr)                                                                             \
    do {                                                                                                \
        ncclResult_t _r = (expr);                                                                       \
        if (_r != ncclSuccess) {                                                                        \
            if (ctx) (ctx)->poisoned = true;                                                            \
            return fail(MPPI_ERR_NCCL, std::string(#expr) + ": " + ncclGetErrorString(_r));             \
        }                                                                                               \
    } while (0)

static int state_dim(const mppi_config* c) { return c->model == MPPI_MODEL_PAPER ? 17 : 10; }

static mppi_status validate(const mppi_config* c) {
    if (!c) return fail(MPPI_ERR_INVALID, "cfg is NULL");
    if (c->abi_version != MPPI_ABI_VERSION) return fail(MPPI_ERR_INVALID, "abi_version mismatch");
    if (c->n_ctrl < 1 || c->K < 1 || c->T < 1) return fail(MPPI_ERR_INVALID, "n_ctrl, K, T must be >= 1");
    if (c->K_global < c->K) return fail(MPPI_ERR_INVALID, "K_global < K");
    if (c->k_offset < 0 || c->k_offset + c->K > c->K_global) return fail(MPPI_ERR_INVALID, "k_offset out of range");
    if (c->ctrl_offset < 0) return fail(MPPI_ERR_INVALID, "ctrl_offset < 0");
    if (!(c->dt > 0.f) || !(c->lambda > 0.f) || !(c->mass > 0.f)) return fail(MPPI_ERR_INVALID, "dt, lambda, mass > 0");
    if (!(c->sdf_scale > 0.f)) return fail(MPPI_ERR_INVALID, "sdf_scale > 0");
    if (c->w_guide != 0.f && !(c->fd_h > 0.f)) return fail(MPPI_ERR_INVALID, "fd_h > 0 with guidance");
    if (c->model != MPPI_MODEL_BASELINE && c->model != MPPI_MODEL_PAPER) return fail(MPPI_ERR_INVALID, "bad model");
    if (c->sdf_provider != MPPI_SDF_MLP && c->sdf_provider != MPPI_SDF_GATE) return fail(MPPI_ERR_INVALID, "bad sdf_provider");
    if (c->pe_bands != 0 && c->pe_bands != 4) return fail(MPPI_ERR_UNSUPPORTED, "pe_bands must be 0 or 4");
    if (c->pe_bands && (c->mlp_dtype != MPPI_MLP_BF16 || !mlp_tc_pe_supported(c->hidden, c->n_hidden - 1, c->pe_bands)))
        return fail(MPPI_ERR_UNSUPPORTED, "positional encoding: bf16 tcgen05 MLP (hidden 128 or 256) only");
    if (c->sdf_provider == MPPI_SDF_GATE && (!std::isfinite(c->gate_c) || !(c->gate_tana >= 0.f) || !std::isfinite(c->gate_tana)))
        return fail(MPPI_ERR_INVALID, "gate_c finite, gate_tana >= 0");
    if (c->model == MPPI_MODEL_PAPER) {
        if (c->w_guide != 0.f) return fail(MPPI_ERR_INVALID, "the paper model has no guidance term (w_guide must be 0)");
        if (!(c->inertia[0] > 0.f) || !(c->inertia[1] > 0.f) || !(c->inertia[2] > 0.f) || !(c->arm > 0.f))
            return fail(MPPI_ERR_INVALID, "inertia and arm must be > 0");
        if (!(c->thrust_max > 0.f) || !(c->rate_max > 0.f)) return fail(MPPI_ERR_INVALID, "thrust_max, rate_max > 0");
        if (!std::isfinite(c->q_gate) || !std::isfinite(c->q_vis) || !std::isfinite(c->q_sdf) || !std::isfinite(c->d_safe))
            return fail(MPPI_ERR_INVALID, "non-finite cost weight");
    }
    for (int i = 0; i < 4; ++i)
        if (!(c->u_lo[i] <= c->u_hi[i])) return fail(MPPI_ERR_INVALID, "u_lo > u_hi");
    if (c->latent_dim < 0 || c->hidden < 1 || c->n_hidden < 1) return fail(MPPI_ERR_INVALID, "bad MLP dims");
    if (c->activation < 0 || c->activation > 2) return fail(MPPI_ERR_INVALID, "bad activation");
    if (c->noise_mode != MPPI_NOISE_DEVICE && c->noise_mode != MPPI_NOISE_EXTERNAL)
        return fail(MPPI_ERR_INVALID, "bad noise_mode");
    if (c->world_size < 1 || c->rank < 0 || c->rank >= c->world_size) return fail(MPPI_ERR_INVALID, "bad rank/world");
    if (c->mlp_dtype == MPPI_MLP_FP32) {
        if (c->hidden != 32 && c->hidden != 64)
            return fail(MPPI_ERR_UNSUPPORTED, "fp32 MLP kernel supports hidden 32 or 64");
    } else if (c->mlp_dtype == MPPI_MLP_BF16) {
        if (!mlp_tc_supported(c->hidden, c->n_hidden - 1, c->activation))
            return fail(MPPI_ERR_UNSUPPORTED, "bf16 tcgen05 MLP kernel: unsupported hidden width / depth");
    } else {
        return fail(MPPI_ERR_INVALID, "bad mlp_dtype");
    }
    const double rows = (double)c->n_ctrl * c->K * c->T * (c->w_guide != 0.f ? 2 : 1);
    if (rows > 2147483647.0 * 0.5) return fail(MPPI_ERR_INVALID, "problem too large");
    return MPPI_OK;
}

extern "C" {

const char* mppi_last_error(void) { return g_err.c_str(); }

size_t mppi_workspace_bytes(const mppi_config* cfg) {
    if (validate(cfg) != MPPI_OK) return 0;
    Layout L;
    compute_layout(cfg, &L);
    return L.total;
}

mppi_status mppi_get_nccl_unique_id(void* out128) {
    if (!out128) return fail(MPPI_ERR_INVALID, "out is NULL");
    ncclUniqueId id;
    ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) return fail(MPPI_ERR_NCCL, ncclGetErrorString(r));
    std::memcpy(out128, &id, sizeof(id));
    return MPPI_OK;
}

mppi_status mppi_create(const mppi_config* cfg, void* d_ws, size_t ws_bytes, mppi_ctx** out) {
    if (!out) return fail(MPPI_ERR_INVALID, "out is NULL");
    *out = nullptr;
    mppi_status st = validate(cfg);
    if (st != MPPI_OK) return st;
    Layout L;
    compute_layout(cfg, &L);
    if (d_ws && ws_bytes < L.total) return fail(MPPI_ERR_OOM, "workspace too small");
    mppi_ctx* ctx = new mppi_ctx();
    ctx->cfg = *cfg;
    ctx->lay = L;
    ctx->stream = (cudaStream_t)cfg->stream;
    int n_dev = 0;
    if (cudaGetDeviceCount(&n_dev) != cudaSuccess || cfg->device < 0 || cfg->device >= n_dev) {
        delete ctx;
        return fail(MPPI_ERR_INVALID, "cfg.device is not a CUDA device of this process");
    }
    DeviceGuard dg(cfg->device);
    cudaError_t e;
    if (!d_ws) {
        e = cudaMalloc(&ctx->ws, L.total);
        if (e != cudaSuccess) { delete ctx; return fail(MPPI_ERR_OOM, cudaGetErrorString(e)); }
        ctx->own_ws = true;
    } else {
        if (((uintptr_t)d_ws) % 1024) { delete ctx; return fail(MPPI_ERR_INVALID, "workspace must be 1024-B aligned"); }
        ctx->ws = d_ws;
    }
    char* base = (char*)ctx->ws;
    Buffers& b = ctx->b;
    b.w1p = (float4*)(base + L.off[B_W1P]);
    b.w1pe = (float*)(base + L.off[B_W1PE]);
    b.w1pe2 = (float2*)(base + L.off[B_W1PE2]);
    b.w1z = (float*)(base + L.off[B_W1Z]);
    b.b1 = (float*)(base + L.off[B_B1]);
    b.b1f = (float*)(base + L.off[B_B1F]);
    b.hid_w32 = (float*)(base + L.off[B_HW32]);
    b.hid_wbf = (uint8_t*)(base + L.off[B_HWBF]);
    b.hid_b = (float*)(base + L.off[B_HB]);
    b.w_out = (float*)(base + L.off[B_WOUT]);
    b.b_out = (float*)(base + L.off[B_BOUT]);
    b.z = (float*)(base + L.off[B_Z]);
    b.Tq = (float*)(base + L.off[B_TQ]);
    b.x0 = (float*)(base + L.off[B_X0]);
    b.goal = b.x0 + (size_t)cfg->n_ctrl * state_dim_of(cfg);
    b.step = (unsigned long long*)(base + L.off[B_X0] + step_inputs_bytes(cfg));
    b.U_out = (float*)(base + L.off[B_UOUT]);
    b.U_nom = (float*)(base + L.off[B_UNOM]);
    b.noise = (float4*)(base + L.off[B_NOISE]);
    b.rows = (float4*)(base + L.off[B_ROWS]);
    b.sdf_rows = (float*)(base + L.off[B_SDF]);
    b.terms = (float*)(base + L.off[B_TERMS]);
    b.partial = (float*)(base + L.off[B_PART]);
    b.J = (float*)(base + L.off[B_J]);
    b.tickets = (unsigned*)(base + L.off[B_TICK]);
    b.blkrec = (float*)(base + L.off[B_BLKREC]);
    b.record = (float*)(base + L.off[B_REC]);
    b.gathered = (float*)(base + L.off[B_GATH]);
    b.diag = (float*)(base + L.off[B_DIAG]);
    b.flags = (int*)(base + L.off[B_FLAGS]);
    b.weights = (float*)(base + L.off[B_WGT]);

    Params& p = ctx->p;
    p.n_ctrl = cfg->n_ctrl; p.K = cfg->K; p.T = cfg->T;
    p.rps = cfg->w_guide != 0.f ? 2 : 1;
    p.H = cfg->hidden; p.L = cfg->latent_dim; p.n_gemm = cfg->n_hidden - 1; p.act = cfg->activation;
    p.K_global = cfg->K_global; p.k_offset = cfg->k_offset; p.ctrl_offset = cfg->ctrl_offset;
    p.dt = cfg->dt; p.inv_lambda = 1.f / cfg->lambda; p.mass = cfg->mass; p.gravity = cfg->gravity;
    for (int i = 0; i < 4; ++i) { p.u_lo[i] = cfg->u_lo[i]; p.u_hi[i] = cfg->u_hi[i]; p.sigma[i] = cfg->sigma[i]; }
    p.w_goal = cfg->w_goal; p.w_sdf = cfg->w_sdf; p.inv_sdf_scale = 1.f / cfg->sdf_scale;
    p.sdf_exp_max = cfg->sdf_exp_max; p.w_u = cfg->w_u; p.w_guide = cfg->w_guide; p.fd_h = cfg->fd_h;
    p.inv_fd_h = cfg->fd_h > 0.f ? 1.f / cfg->fd_h : 0.f;
    p.seed = cfg->seed;
    p.model = cfg->model;
    p.arm_d = cfg->arm / sqrtf(2.f);
    p.kappa = cfg->kappa;
    p.Jx = cfg->inertia[0]; p.Jy = cfg->inertia[1]; p.Jz = cfg->inertia[2];
    p.inv_Jx = 1.f / cfg->inertia[0]; p.inv_Jy = 1.f / cfg->inertia[1]; p.inv_Jz = 1.f / cfg->inertia[2];
    p.thrust_max = cfg->thrust_max; p.rate_max = cfg->rate_max;
    p.q_gate = cfg->q_gate; p.q_vis = cfg->q_vis; p.q_sdf = cfg->q_sdf; p.d_safe = cfg->d_safe;
    p.sdf_provider = cfg->sdf_provider; p.gate_c = cfg->gate_c; p.gate_tana = cfg->gate_tana;
    p.pe_bands = cfg->pe_bands;
    p.noise_device = cfg->noise_mode == MPPI_NOISE_DEVICE ? 1 : 0;
    {
        const char* lg = getenv("MPPI_H128_LEGACY");
        p.mlp_legacy = lg && lg[0] == '1' ? 1 : 0;
    }
    ctx->use_tc = cfg->mlp_dtype == MPPI_MLP_BF16;
    {   // fused rollout (FUSE in kernel_mlp_h128.cu / kernel_mlp_tc.cu): the rollout runs inside the SDF-MLP
        // kernel, so the query rows never reach HBM; MPPI_FUSED=0/1 overrides the default below
        const bool common = ctx->use_tc && cfg->pe_bands == 0 && cfg->model == MPPI_MODEL_BASELINE &&
                            cfg->sdf_provider == MPPI_SDF_MLP && cfg->w_guide != 0.f;
        const bool e128 = common && cfg->hidden == 128 && cfg->K % 64 == 0 && !p.mlp_legacy;
        const bool e256 = common && cfg->hidden == 256 && cfg->K % 128 == 0 && cfg->n_hidden == 4 &&
                          (cfg->activation == MPPI_ACT_SILU || cfg->activation == MPPI_ACT_RELU);
        // default: on for large H = 128 problems (configs[4]: -0.35% step, -1.2% end to end, 1.68 GB less DRAM
        // traffic per step; final round-2 session A/B), off at H = 256 (configs[3] 2% slower) and for
        // small problems (configs[1]: 35% slower -- too few blocks to hide the producer); the large-problem test is
        // >= 8 blocks per SM / CTA pair
        int n_sm = 148;
        cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, cfg->device);
        const bool auto128 = e128 && (long long)cfg->n_ctrl * (cfg->K / 64) >= 8LL * n_sm && kFuse128Default;
        const bool auto256 = e256 && (long long)cfg->n_ctrl * (cfg->K / 128) >= 8LL * (n_sm / 2) && kFuse256Default;
        const char* fe = getenv("MPPI_FUSED");
        ctx->fused = (e128 || e256) && (fe ? fe[0] == '1' : auto128 || auto256);
    }
    ctx->latent_set.assign(cfg->n_ctrl, 0);
    ctx->latent_t.assign(cfg->n_ctrl, NAN);
    ctx->latent_steps.assign(cfg->n_ctrl, 0);
    ctx->latent_invalid.assign(cfg->n_ctrl, 0);

    auto cleanup = [&](mppi_status s, const std::string& m) {
        mppi_destroy(ctx);
        return fail(s, m);
    };
    const size_t stage_floats = step_block_bytes(cfg) / 4 + 2;
    for (int i = 0; i < kStaging; ++i) {
        if (cudaHostAlloc((void**)&ctx->h_stage[i], stage_floats * sizeof(float), cudaHostAllocDefault) != cudaSuccess)
            return cleanup(MPPI_ERR_OOM, "cudaHostAlloc staging");
        if (cudaEventCreateWithFlags(&ctx->stage_ev[i], cudaEventDisableTiming) != cudaSuccess)
            return cleanup(MPPI_ERR_CUDA, "cudaEventCreate");
    }
    if (cudaHostAlloc((void**)&ctx->h_out, sizeof(float) * cfg->n_ctrl * cfg->T * 4 + sizeof(int) * cfg->n_ctrl,
                      cudaHostAllocDefault) != cudaSuccess)
        return cleanup(MPPI_ERR_OOM, "cudaHostAlloc readback");
    for (int i = 0; i <= kNumStages; ++i)
        if (cudaEventCreate(&ctx->prof_ev[i]) != cudaSuccess) return cleanup(MPPI_ERR_CUDA, "cudaEventCreate");
    if (cudaStreamCreateWithFlags(&ctx->work, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->ev_in, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->ev_out, cudaEventDisableTiming) != cudaSuccess)
        return cleanup(MPPI_ERR_CUDA, "work stream / events");
    // zero-init the small state (U, diag, flags, step) so debug reads are defined
    if (cudaMemsetAsync(base, 0, L.off[B_NOISE], ctx->stream) != cudaSuccess ||
        cudaMemsetAsync(b.tickets, 0, 4 * (size_t)cfg->n_ctrl * (1 + softmin_group_count(cfg->K)), ctx->stream) != cudaSuccess ||
        cudaMemsetAsync(b.diag, 0, 16 * (size_t)cfg->n_ctrl, ctx->stream) != cudaSuccess ||
        cudaMemsetAsync(b.flags, 0, 4 * (size_t)cfg->n_ctrl, ctx->stream) != cudaSuccess)
        return cleanup(MPPI_ERR_CUDA, "memset");
    if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) return cleanup(MPPI_ERR_CUDA, "sync");
    // A communicator is created whenever an id is given (also for world_size 1: the record ->
    // ncclAllGather -> combine path then runs inside the step graph on a single GPU)
    if (cfg->nccl_unique_id) {
        ncclUniqueId id;
        std::memcpy(&id, cfg->nccl_unique_id, sizeof(id));
        ncclResult_t r = ncclCommInitRank(&ctx->comm, cfg->world_size, id, cfg->rank);
        if (r != ncclSuccess) return cleanup(MPPI_ERR_NCCL, ncclGetErrorString(r));
    }
    *out = ctx;
    return MPPI_OK;
}

mppi_status mppi_destroy(mppi_ctx* ctx) {
    if (!ctx) return MPPI_OK;
    DeviceGuard dg(ctx->cfg.device);
    // a step may still be in flight: nothing is released before the context's work has drained
    if (ctx->work) cudaStreamSynchronize(ctx->work);
    if (ctx->stream || ctx->work) cudaStreamSynchronize(ctx->stream);
    cudaGetLastError();
    for (auto& g : ctx->graph)
        if (g) cudaGraphExecDestroy(g);
    for (int i = 0; i < kStaging; ++i) {
        if (ctx->h_stage[i]) cudaFreeHost(ctx->h_stage[i]);
        if (ctx->stage_ev[i]) cudaEventDestroy(ctx->stage_ev[i]);
    }
    if (ctx->h_out) cudaFreeHost(ctx->h_out);
    for (auto& e : ctx->prof_ev)
        if (e) cudaEventDestroy(e);
    if (ctx->comm) ncclCommDestroy(ctx->comm);
    if (ctx->work) cudaStreamDestroy(ctx->work);
    if (ctx->ev_in) cudaEventDestroy(ctx->ev_in);
    if (ctx->ev_out) cudaEventDestroy(ctx->ev_out);
    if (ctx->own_ws && ctx->ws) cudaFree(ctx->ws);
    delete ctx;
    return MPPI_OK;
}

#define CHECK_CTX(ctx)                                                        \
    do {                                                                      \
        if (!(ctx)) return fail(MPPI_ERR_INVALID, "ctx is NULL");             \
        if ((ctx)->poisoned) return fail(MPPI_ERR_POISONED, "context poisoned by an earlier CUDA/NCCL error"); \
    } while (0)
// CHECK_CTX + run the rest of the entry point on the context's device
#define ENTER_CTX(ctx)                       \
    CHECK_CTX(ctx);                          \
    DeviceGuard _dev_guard((ctx)->cfg.device)

static void invalidate_graphs(mppi_ctx* ctx) {
    for (auto& g : ctx->graph)
        if (g) { cudaGraphExecDestroy(g); g = nullptr; }
}

mppi_status mppi_set_sdf_weights(mppi_ctx* ctx, int32_t n_layers, const int32_t* in_dim, const int32_t* out_dim,
                                 const float* const* W, const float* const* bvec) {
    ENTER_CTX(ctx);
    const mppi_config& c = ctx->cfg;
    const int H = c.hidden, Ld = c.latent_dim, G = c.n_hidden - 1;
    if (n_layers != c.n_hidden + 1 || !in_dim || !out_dim || !W || !bvec)
        return fail(MPPI_ERR_INVALID, "n_layers must be n_hidden + 1");
    const int npe = 3 + 6 * c.pe_bands;   // layer-1 position features (raw p, then the PE bands)
    for (int l = 0; l < n_layers; ++l) {
        const int ei = l == 0 ? npe + Ld : H, eo = l == n_layers - 1 ? 1 : H;
        if (in_dim[l] != ei || out_dim[l] != eo) return fail(MPPI_ERR_INVALID, "layer dims do not match the config");
        if (!W[l] || !bvec[l]) return fail(MPPI_ERR_INVALID, "NULL weight pointer");
    }
    const bool bf = c.mlp_dtype == MPPI_MLP_BF16;
    std::vector<float4> w1p(H);
    std::vector<float> w1z((size_t)H * Ld), b1(H), hb((size_t)G * H), wo(H), bo(4, 0.f);
    std::vector<float> w1pe((size_t)H * npe);
    for (int j = 0; j < H; ++j) {
        const float* r = W[0] + (size_t)j * (npe + Ld);
        w1p[j] = make_float4(r[0], r[1], r[2], 0.f);
        for (int f = 0; f < npe; ++f) w1pe[(size_t)j * npe + f] = r[f];
        for (int l = 0; l < Ld; ++l) w1z[(size_t)j * Ld + l] = r[npe + l];
        b1[j] = bvec[0][j];
    }
    std::vector<float> hw((size_t)G * H * H);
    for (int l = 0; l < G; ++l) {
        for (size_t i = 0; i < (size_t)H * H; ++i) hw[(size_t)l * H * H + i] = bf ? bf16_value(W[1 + l][i]) : W[1 + l][i];
        for (int i = 0; i < H; ++i) hb[(size_t)l * H + i] = bvec[1 + l][i];
    }
    for (int j = 0; j < H; ++j) wo[j] = bf ? bf16_value(W[n_layers - 1][j]) : W[n_layers - 1][j];
    bo[0] = bvec[n_layers - 1][0];
    cudaStream_t s = ctx->stream;
    CUDA_TRY(ctx, cudaStreamSynchronize(s));
    CUDA_TRY(ctx, cudaMemcpy(ctx->b.w1p, w1p.data(), sizeof(float4) * H, cudaMemcpyHostToDevice));
    CUDA_TRY(ctx, cudaMemcpy(ctx->b.w1pe, w1pe.data(), sizeof(float) * w1pe.size(), cudaMemcpyHostToDevice));
    {   // neuron-pair-major, kPre-scaled copy of the position / PE columns (layer 1 of the H = 256 PE kernel)
        const float kp = c.activation == MPPI_ACT_SILU ? 0.5f : 1.0f;
        std::vector<float> w2((size_t)H * npe);
        for (int jp = 0; jp < H / 2; ++jp)
            for (int f = 0; f < npe; ++f) {
                w2[((size_t)jp * npe + f) * 2] = w1pe[(size_t)(2 * jp) * npe + f] * kp;
                w2[((size_t)jp * npe + f) * 2 + 1] = w1pe[(size_t)(2 * jp + 1) * npe + f] * kp;
            }
        CUDA_TRY(ctx, cudaMemcpy(ctx->b.w1pe2, w2.data(), sizeof(float) * w2.size(), cudaMemcpyHostToDevice));
        ctx->w1pe2_host = std::move(w2);
        ctx->b.w1pe2_host = reinterpret_cast<const float2*>(ctx->w1pe2_host.data());
        invalidate_graphs(ctx);   // the H = 256 PE kernel carries these weights in its launch parameters
    }
    CUDA_TRY(ctx, cudaMemcpy(ctx->b.w1z, w1z.data(), sizeof(float) * w1z.size(), cudaMemcpyHostToDevice));
    CUDA_TRY(ctx, cudaMemcpy(ctx->b.b1, b1.data(), sizeof(float) * H, cudaMemcpyHostToDevice));
    if (G > 0) CUDA_TRY(ctx, cudaMemcpy(ctx->b.hid_b, hb.data(), sizeof(float) * hb.size(), cudaMemcpyHostToDevice));
    CUDA_TRY(ctx, cudaMemcpy(ctx->b.w_out, wo.data(), sizeof(float) * H, cudaMemcpyHostToDevice));
    CUDA_TRY(ctx, cudaMemcpy(ctx->b.b_out, bo.data(), sizeof(float) * 4, cudaMemcpyHostToDevice));
    if (G > 0) {
        if (bf) {
            std::vector<uint8_t> img(H == 128 ? mlp_h128_image_bytes(G, c.pe_bands) : mlp_tc_weight_bytes(H, G));
            mlp_tc_pack_weights(H, G, c.activation, hw.data(), hb.data(), img.data());
            // H = 128: the layer-1 B operand (exact bf16 splits of the position / PE columns) follows
            if (H == 128) mlp_h128_pack_l1(c.pe_bands, c.activation, w1pe.data(), img.data() + mlp_tc_weight_bytes(H, G));
            CUDA_TRY(ctx, cudaMemcpy(ctx->b.hid_wbf, img.data(), img.size(), cudaMemcpyHostToDevice));
        } else {
            CUDA_TRY(ctx, cudaMemcpy(ctx->b.hid_w32, hw.data(), sizeof(float) * hw.size(), cudaMemcpyHostToDevice));
        }
    }
    ctx->weights = true;
    std::fill(ctx->latent_set.begin(), ctx->latent_set.end(), 0);
    return MPPI_OK;
}

static mppi_status set_latent_impl(mppi_ctx* ctx, int32_t ctrl, const float* z, const float* T_q, double t_frame,
                                   int32_t valid) {
    ENTER_CTX(ctx);
    const mppi_config& c = ctx->cfg;
    const bool gate = c.sdf_provider == MPPI_SDF_GATE;
    if (ctrl < -1 || ctrl >= c.n_ctrl) return fail(MPPI_ERR_INVALID, "bad ctrl");
    const int c0 = ctrl < 0 ? 0 : ctrl, cnt = ctrl < 0 ? c.n_ctrl : 1;
    if (!valid) {   // occluded / invalid frame: the cached (z, T_q) stays in use
        for (int i = 0; i < cnt; ++i) ++ctx->latent_invalid[c0 + i];
        return MPPI_OK;
    }
    if (!ctx->weights && !gate) return fail(MPPI_ERR_NOT_READY, "set weights before latents");
    if ((!z && c.latent_dim > 0) || !T_q) return fail(MPPI_ERR_INVALID, "NULL z / T_q");
    for (int i = 0; i < cnt * 12; ++i)
        if (!std::isfinite(T_q[i])) return fail(MPPI_ERR_INVALID, "non-finite T_q");
    for (int i = 0; i < cnt * c.latent_dim; ++i)
        if (!std::isfinite(z[i])) return fail(MPPI_ERR_INVALID, "non-finite z");
    cudaStream_t s = ctx->stream;
    if (c.latent_dim > 0)
        CUDA_TRY(ctx, cudaMemcpyAsync(ctx->b.z + (size_t)c0 * c.latent_dim, z, sizeof(float) * cnt * c.latent_dim,
                                      cudaMemcpyHostToDevice, s));
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->b.Tq + (size_t)c0 * 12, T_q, sizeof(float) * cnt * 12, cudaMemcpyHostToDevice, s));
    if (!gate) launch_fold(ctx->p, ctx->b, c0, cnt, s);   // the analytic provider uses T_q only
    CUDA_TRY(ctx, cudaGetLastError());
    CUDA_TRY(ctx, cudaStreamSynchronize(s));   // host arrays may be reused on return
    for (int i = 0; i < cnt; ++i) {
        ctx->latent_set[c0 + i] = 1;
        ctx->latent_t[c0 + i] = t_frame;
        ctx->latent_steps[c0 + i] = 0;
        ctx->latent_invalid[c0 + i] = 0;
    }
    return MPPI_OK;
}

mppi_status mppi_set_latent(mppi_ctx* ctx, int32_t ctrl, const float* z, const float* T_q) {
    return set_latent_impl(ctx, ctrl, z, T_q, NAN, 1);
}

mppi_status mppi_set_latent_frame(mppi_ctx* ctx, int32_t ctrl, const float* z, const float* T_q, double t_frame,
                                  int32_t valid) {
    return set_latent_impl(ctx, ctrl, z, T_q, t_frame, valid);
}

mppi_status mppi_get_latent_status(mppi_ctx* ctx, double* out_t, int64_t* out_steps, int64_t* out_invalid) {
    CHECK_CTX(ctx);
    const int n = ctx->cfg.n_ctrl;
    for (int i = 0; i < n; ++i) {
        if (out_t) out_t[i] = ctx->latent_t[i];
        if (out_steps) out_steps[i] = ctx->latent_steps[i];
        if (out_invalid) out_invalid[i] = ctx->latent_invalid[i];
    }
    return MPPI_OK;
}

mppi_status mppi_set_nominal(mppi_ctx* ctx, int32_t ctrl, const float* U) {
    ENTER_CTX(ctx);
    const mppi_config& c = ctx->cfg;
    if (ctrl < -1 || ctrl >= c.n_ctrl || !U) return fail(MPPI_ERR_INVALID, "bad ctrl / NULL");
    const int c0 = ctrl < 0 ? 0 : ctrl, cnt = ctrl < 0 ? c.n_ctrl : 1;
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->b.U_out + (size_t)c0 * c.T * 4, U, sizeof(float) * cnt * c.T * 4,
                                  cudaMemcpyHostToDevice, ctx->stream));
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    return MPPI_OK;
}

mppi_status mppi_set_noise(mppi_ctx* ctx, const float* d_noise) {
    ENTER_CTX(ctx);
    if (ctx->cfg.noise_mode != MPPI_NOISE_EXTERNAL) return fail(MPPI_ERR_INVALID, "context is not in external-noise mode");
    if (!d_noise) return fail(MPPI_ERR_INVALID, "NULL noise");
    const mppi_config& c = ctx->cfg;
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->b.noise, d_noise, sizeof(float4) * (size_t)c.T * c.n_ctrl * c.K,
                                  cudaMemcpyDeviceToDevice, ctx->stream));
    return MPPI_OK;
}

static cudaError_t launch_mlp_states(mppi_ctx* ctx, cudaStream_t s) {
    const Params& p = ctx->p;
    const long long n_states = (long long)p.n_ctrl * p.T * p.K;
    if (ctx->use_tc)
        return launch_mlp_tc(p, ctx->b, ctx->b.rows, n_states * p.rps, -1, ctx->debug_outputs ? ctx->b.sdf_rows : nullptr,
                             true, s);
    launch_mlp_simt(p, ctx->b, ctx->b.rows, n_states, -1, ctx->debug_outputs ? ctx->b.sdf_rows : nullptr, true, s);
    return cudaGetLastError();
}

// The per-step launch sequence (captured once into a CUDA graph). mode 0: full step with update
// (and NCCL exchange + combine when a communicator exists); mode 1: local step writing the record.
static cudaError_t enqueue_step(mppi_ctx* ctx, int mode, cudaStream_t s) {
    const Params& p = ctx->p;
    const int prof = ctx->profiling;
    auto mark = [&](int i) {
        if (prof >= 2 || (prof == 1 && (i == 2 || i == 3)))
            cudaEventRecordWithFlags(ctx->prof_ev[i], s, cudaEventRecordExternal);
    };
    mark(0);
    const bool fused = ctx->fused && !ctx->debug_outputs;   // debug outputs need the query rows in HBM
    mark(1);   // noise generation and the warm-start shift are fused into the rollout kernel
    if (!fused) launch_rollout(p, ctx->b, ctx->cfg.noise_mode == MPPI_NOISE_DEVICE, s);
    mark(2);
    cudaError_t e;
    if (fused) {   // rollout + SDF-MLP in one kernel: the query rows never leave shared memory
        const long long n_states = (long long)p.n_ctrl * p.T * p.K;
        e = launch_mlp_tc(p, ctx->b, nullptr, n_states * p.rps, -1, nullptr, true, s, true);
    } else if (ctx->cfg.sdf_provider == MPPI_SDF_GATE) {
        launch_sdf_gate(p, ctx->b, ctx->debug_outputs ? ctx->b.sdf_rows : nullptr, s);
        e = cudaGetLastError();
    } else {
        e = launch_mlp_states(ctx, s);
    }
    if (e != cudaSuccess) return e;
    mark(3);
    if (mode == 1 || ctx->comm) {
        launch_softmin(p, ctx->b, true, s);
        mark(4);
        if (mode == 0) {
            const size_t recn = (size_t)p.n_ctrl * (kRecHead + 4 * p.T);
            ctx->nccl_err = ncclAllGather(ctx->b.record, ctx->b.gathered, recn, ncclFloat, ctx->comm, s);
            if (ctx->nccl_err != ncclSuccess) return cudaErrorUnknown;   // reported as MPPI_ERR_NCCL
            launch_combine(p, ctx->b, ctx->b.gathered, ctx->cfg.world_size, s);
        }
    } else {
        launch_softmin(p, ctx->b, false, s);
        mark(4);
    }
    mark(5);
    return cudaGetLastError();
}

static mppi_status run_step(mppi_ctx* ctx, const float* x0, const float* goal, uint64_t step, bool device_inputs,
                            int mode) {
    ENTER_CTX(ctx);
    if (!ctx->weights && ctx->cfg.sdf_provider != MPPI_SDF_GATE) return fail(MPPI_ERR_NOT_READY, "weights not set");
    for (char v : ctx->latent_set)
        if (!v) return fail(MPPI_ERR_NOT_READY, "latent not set for every controller");
    if (!x0 || !goal) return fail(MPPI_ERR_INVALID, "NULL x0/goal");
    if (mode == 0 && ctx->cfg.world_size > 1 && !ctx->comm)
        return fail(MPPI_ERR_INVALID, "sharded context without NCCL: use mppi_step_local / mppi_step_finish");
    const int n = ctx->cfg.n_ctrl, sd = state_dim(&ctx->cfg);
    // The graph runs on the internal stream, ordered after everything already queued on the caller's
    // stream; the caller's stream then waits for the step (so setters, debug copies and
    // get_controls on cfg.stream see its results).
    cudaStream_t s = ctx->work;
    CUDA_TRY(ctx, cudaEventRecord(ctx->ev_in, ctx->stream));
    CUDA_TRY(ctx, cudaStreamWaitEvent(s, ctx->ev_in, 0));
    if (device_inputs) {
        CUDA_TRY(ctx, cudaMemcpyAsync(ctx->b.x0, x0, sizeof(float) * n * sd, cudaMemcpyDeviceToDevice, s));
        CUDA_TRY(ctx, cudaMemcpyAsync(ctx->b.goal, goal, sizeof(float) * n * 3, cudaMemcpyDeviceToDevice, s));
        unsigned long long* hs =
            reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(ctx->h_stage[ctx->stage_i]) + step_inputs_bytes(&ctx->cfg));
        CUDA_TRY(ctx, cudaEventSynchronize(ctx->stage_ev[ctx->stage_i]));
        *hs = step;
        CUDA_TRY(ctx, cudaMemcpyAsync(ctx->b.step, hs, 8, cudaMemcpyHostToDevice, s));
    } else {
        float* h = ctx->h_stage[ctx->stage_i];
        CUDA_TRY(ctx, cudaEventSynchronize(ctx->stage_ev[ctx->stage_i]));   // previous use of this slot done
        std::memcpy(h, x0, sizeof(float) * n * sd);
        std::memcpy(h + (size_t)n * sd, goal, sizeof(float) * n * 3);
        std::memcpy(reinterpret_cast<char*>(h) + step_inputs_bytes(&ctx->cfg), &step, 8);
        // one H2D copy of [x0 | goal | pad | step] (pinned staging ring; the device block has the same layout)
        CUDA_TRY(ctx, cudaMemcpyAsync(ctx->b.x0, h, step_block_bytes(&ctx->cfg), cudaMemcpyHostToDevice, s));
    }
    CUDA_TRY(ctx, cudaEventRecord(ctx->stage_ev[ctx->stage_i], s));
    ctx->stage_i = (ctx->stage_i + 1) % kStaging;
    if (!ctx->graph[mode]) {
        cudaGraph_t g;
        CUDA_TRY(ctx, cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        ctx->nccl_err = ncclSuccess;
        cudaError_t e = enqueue_step(ctx, mode, s);
        cudaError_t e2 = cudaStreamEndCapture(s, &g);
        if (e != cudaSuccess) {
            if (e2 == cudaSuccess) cudaGraphDestroy(g);
            ctx->poisoned = true;
            if (ctx->nccl_err != ncclSuccess)
                return fail(MPPI_ERR_NCCL, std::string("step capture: ncclAllGather: ") + ncclGetErrorString(ctx->nccl_err));
            return fail(MPPI_ERR_CUDA, std::string("step capture: ") + cudaGetErrorString(e));
        }
        CUDA_TRY(ctx, e2);
        cudaError_t e3 = cudaGraphInstantiate(&ctx->graph[mode], g, 0);
        cudaGraphDestroy(g);
        CUDA_TRY(ctx, e3);
    }
    CUDA_TRY(ctx, cudaGraphLaunch(ctx->graph[mode], s));
    for (auto& a : ctx->latent_steps) ++a;
    CUDA_TRY(ctx, cudaEventRecord(ctx->ev_out, s));
    CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->stream, ctx->ev_out, 0));
    ctx->prof_valid = ctx->profiling > 0;
    ctx->last_mode = mode;
    ctx->last_fused = ctx->fused && !ctx->debug_outputs;
    return MPPI_OK;
}

mppi_status mppi_step(mppi_ctx* ctx, const float* x0, const float* goal, uint64_t step_index) {
    return run_step(ctx, x0, goal, step_index, false, 0);
}

mppi_status mppi_step_device(mppi_ctx* ctx, const float* d_x0, const float* d_goal, uint64_t step_index) {
    return run_step(ctx, d_x0, d_goal, step_index, true, 0);
}

mppi_status mppi_step_local(mppi_ctx* ctx, const float* x0, const float* goal, uint64_t step_index) {
    return run_step(ctx, x0, goal, step_index, false, 1);
}

int32_t mppi_record_size(const mppi_ctx* ctx) { return ctx ? kRecHead + 4 * ctx->cfg.T : 0; }

const float* mppi_get_record_device(const mppi_ctx* ctx) { return ctx ? ctx->b.record : nullptr; }

mppi_status mppi_step_finish(mppi_ctx* ctx, const float* d_records, int32_t R) {
    ENTER_CTX(ctx);
    if (!d_records || R < 1) return fail(MPPI_ERR_INVALID, "bad records");
    launch_combine(ctx->p, ctx->b, d_records, R, ctx->stream);
    CUDA_TRY(ctx, cudaGetLastError());
    return MPPI_OK;
}

mppi_status mppi_get_controls(mppi_ctx* ctx, float* U_out, float* u0_out) {
    ENTER_CTX(ctx);
    if (!U_out) return fail(MPPI_ERR_INVALID, "NULL U_out");
    const mppi_config& c = ctx->cfg;
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    if (ctx->comm) {   // asynchronous communicator failures surface here
        ncclResult_t ar = ncclSuccess;
        NCCL_TRY(ctx, ncclCommGetAsyncError(ctx->comm, &ar));
        if (ar != ncclSuccess && ar != ncclInProgress) {
            ctx->poisoned = true;
            return fail(MPPI_ERR_NCCL, std::string("communicator async error: ") + ncclGetErrorString(ar));
        }
    }
    // U* and the non-finite flags into pinned memory by two async copies on the stream, one synchronisation
    const size_t u_bytes = sizeof(float) * c.n_ctrl * c.T * 4;
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->h_out, ctx->b.U_out, u_bytes, cudaMemcpyDeviceToHost, ctx->stream));
    int* h_flags = reinterpret_cast<int*>(reinterpret_cast<char*>(ctx->h_out) + u_bytes);
    CUDA_TRY(ctx, cudaMemcpyAsync(h_flags, ctx->b.flags, sizeof(int) * c.n_ctrl, cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    std::memcpy(U_out, ctx->h_out, u_bytes);
    if (u0_out)
        for (int i = 0; i < c.n_ctrl; ++i) std::memcpy(u0_out + 4 * i, U_out + (size_t)i * c.T * 4, 16);
    for (int i = 0; i < c.n_ctrl; ++i)
        if (h_flags[i]) return fail(MPPI_ERR_NONFINITE, "every J was non-finite for some controller; its U* is unchanged");
    return MPPI_OK;
}

mppi_status mppi_get_diagnostics(mppi_ctx* ctx, float* out) {
    ENTER_CTX(ctx);
    if (!out) return fail(MPPI_ERR_INVALID, "NULL out");
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    CUDA_TRY(ctx, cudaMemcpy(out, ctx->b.diag, sizeof(float) * 4 * ctx->cfg.n_ctrl, cudaMemcpyDeviceToHost));
    return MPPI_OK;
}

mppi_status mppi_debug_copy(mppi_ctx* ctx, int32_t what, void* host_dst, size_t bytes) {
    ENTER_CTX(ctx);
    const Params& p = ctx->p;
    const size_t states = (size_t)p.n_ctrl * p.T * p.K;
    const void* src = nullptr;
    size_t need = 0;
    switch (what) {
        case MPPI_DBG_QUERIES:
            if (ctx->last_fused) return fail(MPPI_ERR_NOT_READY, "query rows are not stored by the fused rollout (debug outputs off)");
            src = ctx->b.rows;
            need = 16 * states * p.rps;
            break;
        case MPPI_DBG_SDF:
            if (!ctx->debug_outputs) return fail(MPPI_ERR_NOT_READY, "MPPI_DBG_SDF needs mppi_set_debug_outputs(ctx, 1)");
            src = ctx->b.sdf_rows;
            need = 4 * states * p.rps;
            break;
        case MPPI_DBG_COSTS: src = ctx->b.J; need = 4 * (size_t)p.n_ctrl * p.K; break;
        case MPPI_DBG_NOISE: src = ctx->b.noise; need = 16 * states; break;
        case MPPI_DBG_TERMS: src = ctx->b.terms; need = 4 * states; break;
        case MPPI_DBG_PARTIAL: src = ctx->b.partial; need = 4 * (size_t)p.n_ctrl * p.K; break;
        case MPPI_DBG_RECORD: src = ctx->b.record; need = 4 * (size_t)p.n_ctrl * (kRecHead + 4 * p.T); break;
        case MPPI_DBG_WEIGHTS:
            if (ctx->last_mode != 0) return fail(MPPI_ERR_NOT_READY, "MPPI_DBG_WEIGHTS needs a full mppi_step first");
            launch_weights(p, ctx->b, ctx->stream);
            CUDA_TRY(ctx, cudaGetLastError());
            src = ctx->b.weights;
            need = 4 * (size_t)p.n_ctrl * p.K;
            break;
        default: return fail(MPPI_ERR_INVALID, "bad debug id");
    }
    if (!host_dst || bytes < need) return fail(MPPI_ERR_INVALID, "destination too small");
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    CUDA_TRY(ctx, cudaMemcpy(host_dst, src, need, cudaMemcpyDeviceToHost));
    return MPPI_OK;
}

mppi_status mppi_sdf_eval(mppi_ctx* ctx, int32_t ctrl, const float* d_rows, int64_t n, float* d_out) {
    ENTER_CTX(ctx);
    if (!ctx->weights) return fail(MPPI_ERR_NOT_READY, "weights not set");
    if (ctrl < 0 || ctrl >= ctx->cfg.n_ctrl || !ctx->latent_set[ctrl]) return fail(MPPI_ERR_NOT_READY, "latent not set");
    if (n < 0 || (n > 0 && (!d_rows || !d_out))) return fail(MPPI_ERR_INVALID, "bad rows/out");
    if (n == 0) return MPPI_OK;
    if (((uintptr_t)d_rows) % 16) return fail(MPPI_ERR_INVALID, "rows must be 16-B aligned");
    cudaError_t e;
    if (ctx->use_tc) {
        e = launch_mlp_tc(ctx->p, ctx->b, (const float4*)d_rows, n, ctrl, d_out, false, ctx->stream);
    } else {
        launch_mlp_simt(ctx->p, ctx->b, (const float4*)d_rows, n, ctrl, d_out, false, ctx->stream);
        e = cudaGetLastError();
    }
    CUDA_TRY(ctx, e);
    return MPPI_OK;
}

mppi_status mppi_set_debug_outputs(mppi_ctx* ctx, int32_t on) {
    ENTER_CTX(ctx);
    if ((on != 0) != (ctx->debug_outputs != 0)) {
        ctx->debug_outputs = on != 0;
        invalidate_graphs(ctx);
    }
    return MPPI_OK;
}

mppi_status mppi_set_profiling(mppi_ctx* ctx, int32_t level) {
    ENTER_CTX(ctx);
    if (level < 0 || level > 2) return fail(MPPI_ERR_INVALID, "profiling level must be 0, 1 or 2");
    if (level != ctx->profiling) {
        ctx->profiling = level;
        invalidate_graphs(ctx);
    }
    return MPPI_OK;
}

mppi_status mppi_get_kernel_times(mppi_ctx* ctx, float* out, int32_t n_out) {
    ENTER_CTX(ctx);
    if (!out || n_out < 1 || n_out > kNumStages) return fail(MPPI_ERR_INVALID, "bad out");
    if (!ctx->prof_valid) return fail(MPPI_ERR_NOT_READY, "no profiled step yet");
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    for (int i = 0; i < n_out; ++i) {
        out[i] = 0.f;
        if (ctx->profiling >= 2 || i == 2) CUDA_TRY(ctx, cudaEventElapsedTime(out + i, ctx->prof_ev[i], ctx->prof_ev[i + 1]));
    }
    return MPPI_OK;
}

int32_t mppi_debug_trace(uint64_t* host_out, int32_t max_entries) {
    if (!host_out || max_entries <= 0) return 0;
    // H = 128 kernel (kernel_mlp_h128.cu) when MPPI_TRACE_H128=1, else the kernel_mlp_tc.cu timeline
    const char* h = getenv("MPPI_TRACE_H128");
    if (h && h[0] == '1') return mlp_h128_trace_copy(reinterpret_cast<unsigned long long*>(host_out), max_entries);
    const char* sm = getenv("MPPI_TRACE_SOFTMIN");
    if (sm && sm[0] == '1') return softmin_trace_copy(reinterpret_cast<unsigned long long*>(host_out), max_entries);
    return mlp_tc_trace_copy(reinterpret_cast<unsigned long long*>(host_out), max_entries);
}

int32_t mppi_kernels_per_step(const mppi_ctx* ctx) {
    if (!ctx) return 0;
    // rollout (+ noise + shift), mlp, softmin (cost + min + weights + update) (+ combine when sharded with NCCL);
    // the fused rollout runs inside the mlp kernel
    return (ctx->fused && !ctx->debug_outputs ? 2 : 3) + (ctx->comm ? 1 : 0);
}

int32_t mppi_fused_rollout(const mppi_ctx* ctx) { return ctx && ctx->fused && !ctx->debug_outputs ? 1 : 0;
}

}  // extern "C"
