// CUDA-core kernels of the MPPI hot path (sm_100a): noise + warm-start shift (K0), rollout (K1),
// fp32 SDF-MLP (K2f, configs[0]), cost + min reduction (K3), softmin weights + update (K4),
// shard combine, latent fold (K5). The bf16 SDF-MLP on tcgen05 tensor cores is kernel_mlp_tc.cu.
//
// Paper map (PAPER.md line, section/equation):
//   K0  dU ~ N(0, Sigma)                                     PAPER.md:139 (§IV-A); generator: reading R24
//   K1  U^m = U* + dU^m, clamp; rollout xdot = f(x,u)        PAPER.md:139, :146 (CTBR per BASELINE configs[0])
//       query in the cached frame p_c = R p + t
//   K2f s = g_phi(z, p_c) with the latent folded into b1'
//   K3  J = sum of stage costs (Eq. 10 structure)            PAPER.md:185    } fused: k_softmin
//   K4  U* = sum_m w_m U^m, w = softmax(-J/lambda)           PAPER.md:141 (Eq. 5)
#include <math.h>
#include <stdint.h>

#include "../../include/mppi.h"
#include "mppi_internal.cuh"
#include "rollout_dev.cuh"

namespace mppi {

// ------------------------------------------------------------------ helpers (rollout_dev.cuh: Philox, dynamics)
__device__ __forceinline__ float act_f32(int a, float x) {
    if (a == MPPI_ACT_RELU) return fmaxf(x, 0.f);
    if (a == MPPI_ACT_SOFTPLUS) return fmaxf(x, 0.f) + log1pf(expf(-fabsf(x)));
    return x / (1.f + expf(-x));  // SiLU
}

// ------------------------------------------------------------------ K0: noise + warm-start shift
// (debug / standalone form; the step graph fuses both into k_rollout)
// Thread i < n_ctrl*T: U_nom[b][t] = U_out[b][min(t + (step>0), T-1)] (PAPER.md:144 shift).
// Thread i < T*n_ctrl*K (gen): Philox4x32-10(key = seed, ctr = (g, t, step_lo, step_hi)), g = global
// sample index global_sample(b, k); u = ((x >> 9) + 0.5) 2^-23; Box-Muller -> 4 normals.
__global__ void __launch_bounds__(256) k_noise_shift(Params p, Buffers b, int gen) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const unsigned long long step = *b.step;
    if (i < (long long)p.n_ctrl * p.T) {
        const int bb = (int)(i / p.T), t = (int)(i % p.T);
        const int src = step > 0 ? min(t + 1, p.T - 1) : t;
        reinterpret_cast<float4*>(b.U_nom)[i] = reinterpret_cast<const float4*>(b.U_out)[(long long)bb * p.T + src];
    }
    const long long NK = (long long)p.n_ctrl * p.K;
    if (gen && i < NK * p.T) {
        const int t = (int)(i / NK);
        const long long j = i - (long long)t * NK;
        const int bb = (int)(j / p.K), k = (int)(j - (long long)bb * p.K);
        const unsigned long long g = global_sample(p, bb, k);
        b.noise[i] = philox_normals(g, t, step, p.seed);
    }
}

void launch_noise_shift(const Params& p, const Buffers& b, bool gen, cudaStream_t s) {
    long long n = (long long)p.n_ctrl * p.T;
    if (gen) n = max(n, (long long)p.n_ctrl * p.K * p.T);
    const int bs = 256;
    k_noise_shift<<<(unsigned)((n + bs - 1) / bs), bs, 0, s>>>(p, b, gen ? 1 : 0);
}

// ------------------------------------------------------------------ K1: rollout
// K1 rollout: one thread per (controller, sample); state in registers; time-major noise read as float4.
#ifndef MPPI_RO_BLOCK
#define MPPI_RO_BLOCK 64
#endif
constexpr int kRolloutBlock = MPPI_RO_BLOCK;   // small blocks: K/64 blocks spread the latency-bound rollout over all SMs

// Device-noise producer warps of a rollout block (DEV): they generate the Philox normals of step t+1
// (and store them for k_softmin) while the consumer warps integrate step t, handing them over through a
// two-slot shared-memory buffer with one named barrier per step -- the Philox + Box-Muller chain is
// off the rollout's dependency chain (measured: the inline form cost ~10 us per step at configs[1..2]).
__device__ __forceinline__ void named_sync_rollout() {
    asm volatile("bar.sync 1, %0;" ::"r"(2 * kRolloutBlock) : "memory");
}
__device__ void rollout_noise_producer(const Params& p, const Buffers& b, int bb, int lt, int k,
                                       unsigned long long step, float4 (*s_n)[kRolloutBlock]) {
    const bool valid = k < p.K;
    const long long NK = (long long)p.n_ctrl * p.K, col = (long long)bb * p.K + k;
    const unsigned long long gidx = global_sample(p, bb, k);
    if (valid) {
        const float4 n = philox_normals(gidx, 0, step, p.seed);
        s_n[0][lt] = n;
        b.noise[col] = n;
    }
    named_sync_rollout();
    for (int t = 0; t < p.T; ++t) {
        if (valid && t + 1 < p.T) {
            const float4 n = philox_normals(gidx, t + 1, step, p.seed);
            s_n[(t + 1) & 1][lt] = n;
            b.noise[(long long)(t + 1) * NK + col] = n;
        }
        named_sync_rollout();
    }
}

// DEV: generate the noise in registers (Philox, one step ahead) and store it for k_softmin; otherwise
// read the externally set noise. The warm-start shift is fused: the nominal is read from U_out at the
// shifted index, and block 0 of each controller writes the shifted copy U_nom for k_softmin.
constexpr int kMaxTStaged = 128;   // nominal staged in shared memory up to this horizon

template <bool DEV>
#ifndef MPPI_RO_MINB
#define MPPI_RO_MINB 7   // resident rollout blocks per SM: 72 registers (measured r02: 6 -> 7 raises issue-active)
#endif
__global__ void __launch_bounds__(2 * kRolloutBlock, MPPI_RO_MINB) k_rollout(Params p, Buffers b) {
    __shared__ float4 s_n[2][kRolloutBlock];   // DEV: normals of steps t (read) and t + 1 (being written)
    __shared__ float4 s_U[kMaxTStaged];   // the shifted nominal U*_t of this controller (L1-latency reads)
    const int bb = blockIdx.y;
    const int lt = threadIdx.x % kRolloutBlock;
    const int k = blockIdx.x * kRolloutBlock + lt;
    const unsigned long long step = *b.step;
    const int sh = step > 0 ? 1 : 0;
    for (int t = threadIdx.x; t < p.T; t += blockDim.x) {
        const float4 u = reinterpret_cast<const float4*>(b.U_out)[(long long)bb * p.T + min(t + sh, p.T - 1)];
        if (t < kMaxTStaged) s_U[t] = u;
        if (blockIdx.x == 0) reinterpret_cast<float4*>(b.U_nom)[(long long)bb * p.T + t] = u;
    }
    __syncthreads();
    if (DEV && threadIdx.x >= kRolloutBlock) {
        rollout_noise_producer(p, b, bb, lt, k, step, s_n);
        return;
    }
    const bool valid = k < p.K;   // DEV: threads past K still meet every barrier (no stores)
    if (!DEV && !valid) return;
    const float* x0 = b.x0 + bb * 10;
    float x[10];
#pragma unroll
    for (int i = 0; i < 10; ++i) x[i] = __ldg(x0 + i);
    const float* Tq = b.Tq + bb * 12;
    float R[9], tq[3], gc[3];
#pragma unroll
    for (int i = 0; i < 9; ++i) R[i] = __ldg(Tq + i);
#pragma unroll
    for (int i = 0; i < 3; ++i) { tq[i] = __ldg(Tq + 9 + i); gc[i] = __ldg(b.goal + bb * 3 + i); }
    const float4* Uo = reinterpret_cast<const float4*>(b.U_out) + (long long)bb * p.T;
    const long long NK = (long long)p.n_ctrl * p.K;
    const long long col = (long long)bb * p.K + k;
    const unsigned long long gidx = global_sample(p, bb, k);
    const float inv_mass = 1.f / p.mass;
    float part = 0.f;
    // software pipelining: the noise / nominal of step t+1 are produced while step t integrates
    float4 n_next = DEV ? make_float4(0.f, 0.f, 0.f, 0.f) : b.noise[col];
    if (DEV) named_sync_rollout();   // slot 0 written
    auto nominal = [&](int t) { return t < kMaxTStaged ? s_U[t] : Uo[min(t + sh, p.T - 1)]; };
    float4 U_next = nominal(0);
    for (int t = 0; t < p.T; ++t) {
        const float4 n = DEV ? s_n[t & 1][lt] : n_next;
        const float4 U = U_next;
        if (t + 1 < p.T) {
            if (!DEV) n_next = b.noise[(long long)(t + 1) * NK + col];
            U_next = nominal(t + 1);
        }
        float4 row0, row1;
        ctbr_step(p, x, U, n, R, tq, gc, inv_mass, row0, row1, part);
        const long long s = ((long long)bb * p.T + t) * p.K + k;
        if (!valid) {
        } else if (p.rps == 2) {
            b.rows[2 * s] = row0;
            b.rows[2 * s + 1] = row1;
        } else {
            b.rows[s] = row0;
        }
        if (DEV) named_sync_rollout();   // slot t & 1 consumed; slot (t + 1) & 1 written
    }
    if (valid) b.partial[col] = part;
}

// ------------------------------------------------------------------ K1 (paper model): rotor rollout
// MPPI_MODEL_PAPER (SURVEY.md §8f F1 + F2; readings P1-P6): x = [p, v, q, w, T], u = Tdot;
// pdot = v; vdot = (sum T / m) b3(q) - g e_z; qdot = 1/2 q (x) (0, w); wdot = J^-1 (tau - w x J w); Tdot = u
// (PAPER.md:146), X mixer tau = (d(-T1 + T2 + T3 - T4), -d(T1 - T2 + T3 - T4), kappa (T1 + T2 - T3 - T4)).
__device__ __forceinline__ void dyn_rotor(const Params& p, const float* x, const float* u, float* xd) {
    const float qw = x[6], qx = x[7], qy = x[8], qz = x[9];
    const float wx = x[10], wy = x[11], wz = x[12];
    const float T1 = x[13], T2 = x[14], T3 = x[15], T4 = x[16];
    const float fm = (T1 + T2 + T3 + T4) / p.mass;
    xd[0] = x[3]; xd[1] = x[4]; xd[2] = x[5];
    xd[3] = fm * (2.f * (qx * qz + qw * qy));
    xd[4] = fm * (2.f * (qy * qz - qw * qx));
    xd[5] = fm * (1.f - 2.f * (qx * qx + qy * qy)) - p.gravity;
    xd[6] = 0.5f * (-qx * wx - qy * wy - qz * wz);
    xd[7] = 0.5f * (qw * wx + qy * wz - qz * wy);
    xd[8] = 0.5f * (qw * wy + qz * wx - qx * wz);
    xd[9] = 0.5f * (qw * wz + qx * wy - qy * wx);
    const float tx = p.arm_d * (-T1 + T2 + T3 - T4);
    const float ty = -p.arm_d * (T1 - T2 + T3 - T4);
    const float tz = p.kappa * (T1 + T2 - T3 - T4);
    xd[10] = (tx - (wy * (p.Jz * wz) - wz * (p.Jy * wy))) * p.inv_Jx;
    xd[11] = (ty - (wz * (p.Jx * wx) - wx * (p.Jz * wz))) * p.inv_Jy;
    xd[12] = (tz - (wx * (p.Jy * wy) - wy * (p.Jx * wx))) * p.inv_Jz;
    xd[13] = u[0]; xd[14] = u[1]; xd[15] = u[2]; xd[16] = u[3];
}

// One thread per (controller, sample). Per step k = 0..T-1 (the sums of Eqs. 6-9 run over the states
// x_0..x_{T-1}): the query row of x_k (p_c = R p_k + t, |v_k|), the yaw-alignment term of x_k, the RK4
// step to x_{k+1} (then q renormalised, w and T clamped; reading P4) and the progress term
// |p_{k+1} - g|^2 - |p_k - g|^2. The SDF hinge term q_sdf max(0, d_safe - s) is added by the MLP kernel.
template <bool DEV>
__global__ void __launch_bounds__(2 * kRolloutBlock) k_rollout_paper(Params p, Buffers b) {
    __shared__ float4 s_n[2][kRolloutBlock];   // DEV: normals of steps t (read) and t + 1 (being written)
    __shared__ float4 s_U[kMaxTStaged];
    const int bb = blockIdx.y;
    const int lt = threadIdx.x % kRolloutBlock;
    const int k = blockIdx.x * kRolloutBlock + lt;
    const unsigned long long step = *b.step;
    const int sh = step > 0 ? 1 : 0;
    for (int t = threadIdx.x; t < p.T; t += blockDim.x) {
        const float4 u = reinterpret_cast<const float4*>(b.U_out)[(long long)bb * p.T + min(t + sh, p.T - 1)];
        if (t < kMaxTStaged) s_U[t] = u;
        if (blockIdx.x == 0) reinterpret_cast<float4*>(b.U_nom)[(long long)bb * p.T + t] = u;
    }
    __syncthreads();
    if (DEV && threadIdx.x >= kRolloutBlock) {
        rollout_noise_producer(p, b, bb, lt, k, step, s_n);
        return;
    }
    const bool valid = k < p.K;   // DEV: threads past K still meet every barrier (no stores)
    if (!DEV && !valid) return;
    float x[17];
#pragma unroll
    for (int i = 0; i < 17; ++i) x[i] = __ldg(b.x0 + bb * 17 + i);
    const float* Tq = b.Tq + bb * 12;
    float R[9], tq[3], gc[3];
#pragma unroll
    for (int i = 0; i < 9; ++i) R[i] = __ldg(Tq + i);
#pragma unroll
    for (int i = 0; i < 3; ++i) { tq[i] = __ldg(Tq + 9 + i); gc[i] = __ldg(b.goal + bb * 3 + i); }
    const float4* Uo = reinterpret_cast<const float4*>(b.U_out) + (long long)bb * p.T;
    auto nominal = [&](int t) { return t < kMaxTStaged ? s_U[t] : Uo[min(t + sh, p.T - 1)]; };
    const long long NK = (long long)p.n_ctrl * p.K;
    const long long col = (long long)bb * p.K + k;
    const unsigned long long gidx = global_sample(p, bb, k);
    const float dt = p.dt, hdt = 0.5f * p.dt, dt6 = p.dt / 6.f;
    float part = 0.f;
    float4 n_next = DEV ? make_float4(0.f, 0.f, 0.f, 0.f) : b.noise[col];
    if (DEV) named_sync_rollout();   // slot 0 written
    float4 U_next = nominal(0);
    for (int t = 0; t < p.T; ++t) {
        const float4 n = DEV ? s_n[t & 1][lt] : n_next;
        const float4 U = U_next;
        if (t + 1 < p.T) {
            if (!DEV) n_next = b.noise[(long long)(t + 1) * NK + col];
            U_next = nominal(t + 1);
        }
        float u[4];
        u[0] = clampf(U.x + p.sigma[0] * n.x, p.u_lo[0], p.u_hi[0]);
        u[1] = clampf(U.y + p.sigma[1] * n.y, p.u_lo[1], p.u_hi[1]);
        u[2] = clampf(U.z + p.sigma[2] * n.z, p.u_lo[2], p.u_hi[2]);
        u[3] = clampf(U.w + p.sigma[3] * n.w, p.u_lo[3], p.u_hi[3]);
        // ---- query row and yaw alignment of x_k
        float pc[3];
#pragma unroll
        for (int r = 0; r < 3; ++r) pc[r] = R[3 * r] * x[0] + R[3 * r + 1] * x[1] + R[3 * r + 2] * x[2] + tq[r];
        const float nv = sqrtf(x[3] * x[3] + x[4] * x[4] + x[5] * x[5]);
        if (valid) b.rows[((long long)bb * p.T + t) * p.K + k] = make_float4(pc[0], pc[1], pc[2], nv);
        // cos(psi - psi_gate) as the dot of unit heading and line-of-sight vectors (atan2(0,0) = 0 -> (1,0))
        const float hx = 1.f - 2.f * (x[8] * x[8] + x[9] * x[9]), hy = 2.f * (x[6] * x[9] + x[7] * x[8]);
        const float lx = gc[0] - x[0], ly = gc[1] - x[1];
        const float h2 = hx * hx + hy * hy, l2 = lx * lx + ly * ly;
        const float hi = h2 > 0.f ? rsqrtf(h2) : 0.f, li = l2 > 0.f ? rsqrtf(l2) : 0.f;
        const float chx = h2 > 0.f ? hx * hi : 1.f, chy = hy * hi, clx = l2 > 0.f ? lx * li : 1.f, cly = ly * li;
        const float vis = 1.f - (chx * clx + chy * cly);
        const float d0 = (x[0] - gc[0]) * (x[0] - gc[0]) + (x[1] - gc[1]) * (x[1] - gc[1]) + (x[2] - gc[2]) * (x[2] - gc[2]);
        // ---- RK4 step (input held), running sum of the stage derivatives
        float kk[17], acc[17], xt[17];
        dyn_rotor(p, x, u, kk);
#pragma unroll
        for (int i = 0; i < 17; ++i) { acc[i] = kk[i]; xt[i] = x[i] + hdt * kk[i]; }
        dyn_rotor(p, xt, u, kk);
#pragma unroll
        for (int i = 0; i < 17; ++i) { acc[i] += 2.f * kk[i]; xt[i] = x[i] + hdt * kk[i]; }
        dyn_rotor(p, xt, u, kk);
#pragma unroll
        for (int i = 0; i < 17; ++i) { acc[i] += 2.f * kk[i]; xt[i] = x[i] + dt * kk[i]; }
        dyn_rotor(p, xt, u, kk);
#pragma unroll
        for (int i = 0; i < 17; ++i) x[i] = x[i] + dt6 * (acc[i] + kk[i]);
        const float qinv = rsqrtf(x[6] * x[6] + x[7] * x[7] + x[8] * x[8] + x[9] * x[9]);
#pragma unroll
        for (int i = 6; i < 10; ++i) x[i] *= qinv;
#pragma unroll
        for (int i = 10; i < 13; ++i) x[i] = clampf(x[i], -p.rate_max, p.rate_max);
#pragma unroll
        for (int i = 13; i < 17; ++i) x[i] = clampf(x[i], 0.f, p.thrust_max);
        const float d1 = (x[0] - gc[0]) * (x[0] - gc[0]) + (x[1] - gc[1]) * (x[1] - gc[1]) + (x[2] - gc[2]) * (x[2] - gc[2]);
        part += p.q_gate * (d1 - d0) + p.q_vis * vis;
        if (DEV) named_sync_rollout();
    }
    if (valid) b.partial[col] = part;
}

void launch_rollout(const Params& p, const Buffers& b, bool device_noise, cudaStream_t s) {
    dim3 grid((p.K + kRolloutBlock - 1) / kRolloutBlock, p.n_ctrl);
    if (p.model == MPPI_MODEL_PAPER) {
        if (device_noise) k_rollout_paper<true><<<grid, 2 * kRolloutBlock, 0, s>>>(p, b);
        else k_rollout_paper<false><<<grid, kRolloutBlock, 0, s>>>(p, b);
        return;
    }
    if (device_noise) k_rollout<true><<<grid, 2 * kRolloutBlock, 0, s>>>(p, b);   // + noise producer warps
    else k_rollout<false><<<grid, kRolloutBlock, 0, s>>>(p, b);
}

// ------------------------------------------------------------------ K2f: fp32 SDF-MLP on CUDA cores
// Used for MPPI_MLP_FP32 (configs[0]: 35 -> 64 -> 64 -> 1 softplus). Thread per state (states mode:
// evaluates its rps rows and writes the SDF stage term) or per row (mppi_sdf_eval).
template <int H>
__device__ float mlp_row_f32(const Params& p, const float4* w1p, const float* b1f, const float* hw, const float* hb,
                             const float* wo, float bo, float x, float y, float z) {
    float a[H], an[H];
#pragma unroll
    for (int j = 0; j < H; ++j) {
        const float4 w = w1p[j];
        a[j] = act_f32(p.act, w.x * x + w.y * y + w.z * z + b1f[j]);
    }
    for (int l = 0; l < p.n_gemm; ++l) {
        const float* W = hw + (size_t)l * H * H;
#pragma unroll 4
        for (int i = 0; i < H; ++i) {
            float acc = 0.f;
#pragma unroll
            for (int j = 0; j < H; ++j) acc = fmaf(W[i * H + j], a[j], acc);
            an[i] = act_f32(p.act, acc + hb[l * H + i]);
        }
#pragma unroll
        for (int j = 0; j < H; ++j) a[j] = an[j];
    }
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < H; ++j) s = fmaf(wo[j], a[j], s);
    return s + bo;
}

template <int H>
__global__ void __launch_bounds__(128) k_mlp_simt(Params p, Buffers b, const float4* rows, long long n_items,
                                                   int ctrl_fixed, float* sdf_out, int states_mode) {
    extern __shared__ float smem[];
    float* hw = smem;                                   // [n_gemm][H][H]
    float* hb = hw + (size_t)p.n_gemm * H * H;          // [n_gemm][H]
    float* wo = hb + p.n_gemm * H;                      // [H]
    float4* w1p = reinterpret_cast<float4*>(wo + H);    // [H]
    for (int i = threadIdx.x; i < p.n_gemm * H * H; i += blockDim.x) hw[i] = b.hid_w32[i];
    for (int i = threadIdx.x; i < p.n_gemm * H; i += blockDim.x) hb[i] = b.hid_b[i];
    for (int i = threadIdx.x; i < H; i += blockDim.x) { wo[i] = b.w_out[i]; w1p[i] = b.w1p[i]; }
    __syncthreads();
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_items) return;
    const int rps = states_mode ? p.rps : 1;
    const int bb = states_mode ? (int)(i / ((long long)p.T * p.K)) : ctrl_fixed;
    const float* b1f = b.b1f + (size_t)bb * H;
    const float bo = b.b_out[0];
    float sv[2] = {0.f, 0.f};
    float nv = 0.f;
    for (int r = 0; r < rps; ++r) {
        const float4 q = rows[i * rps + r];
        if (r == 0) nv = q.w;
        sv[r] = mlp_row_f32<H>(p, w1p, b1f, hw, hb, wo, bo, q.x, q.y, q.z);
        if (sdf_out) sdf_out[i * rps + r] = sv[r];
    }
    if (states_mode) {
        float term;
        if (p.model == MPPI_MODEL_PAPER) {
            term = p.q_sdf * fmaxf(p.d_safe - sv[0], 0.f);   // Eq. 8 hinge
        } else {
            term = p.w_sdf * expf(fminf(-sv[0] * p.inv_sdf_scale, p.sdf_exp_max));
            if (rps == 2) term -= p.w_guide * nv * (sv[1] - sv[0]) * p.inv_fd_h;
        }
        b.terms[i] = term;
    }
}

void launch_mlp_simt(const Params& p, const Buffers& b, const float4* rows, long long n_items, int ctrl_fixed,
                     float* sdf_out, bool states_mode, cudaStream_t s) {
    const size_t smem = sizeof(float) * ((size_t)p.n_gemm * p.H * p.H + (size_t)p.n_gemm * p.H + p.H) +
                        sizeof(float4) * p.H;
    const unsigned grid = (unsigned)((n_items + 127) / 128);
    if (grid == 0) return;
    if (p.H == 32) {
        cudaFuncSetAttribute(k_mlp_simt<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_mlp_simt<32><<<grid, 128, smem, s>>>(p, b, rows, n_items, ctrl_fixed, sdf_out, states_mode);
    } else {
        cudaFuncSetAttribute(k_mlp_simt<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_mlp_simt<64><<<grid, 128, smem, s>>>(p, b, rows, n_items, ctrl_fixed, sdf_out, states_mode);
    }
}

// ------------------------------------------------------------------ K3+K4: cost, softmin weights, update
// One kernel, grid (sample chunks of 256, controllers). Per block (chunk of samples):
//   J_k = partial_k + sum_t term[t][k] (non-finite -> +inf)                         PAPER.md:185 (Eq. 10)
//   m_b = min_k J_k; w_k = exp((m_b - J_k)/lambda); S_b = sum w; S2_b = sum w^2;
//   V_b[t] = sum_k w_k (clamp(U*_t + sigma n_{t,k}) - U*_t)   (clamped samples, reading R5)
// -> block record (m_b, S_b, S2_b, SJ_b, N_b, 0, 0, 0, V_b) with SJ_b / N_b the sum / count of the finite J
// (mean-cost diagnostic). The last block of the controller (atomic ticket) combines the
// records in block order: m = min m_b, f_b = exp((m - m_b)/lambda), S = sum S_b f_b, V = sum V_b f_b,
// U* <- U* + V/S (Eq. 5) -- the shard-combine identity, so the result is deterministic.
// write_record: the combined record is this rank's record for the cross-rank combine (configs[3]).
constexpr int kSoftminThreads = 512;   // 512/SPB threads per sample in phase 1, 16 warps over t in phase 2
// samples per block: 256, or 512 from K = 65536 on (configs[3]: 256 blocks, one wave at 2 blocks per SM)
#ifndef MPPI_SOFTMIN_K512
#define MPPI_SOFTMIN_K512 65536
#endif
__host__ __device__ constexpr int softmin_spb(int K) { return K >= MPPI_SOFTMIN_K512 ? 512 : 256; }
// two-level record combine from 33 sample blocks on: groups of kSoftminGroup (0 = one level)
constexpr int kSoftminGroup = 16;
__host__ __device__ constexpr int softmin_groups(int nblk) { return nblk > 32 ? (nblk + kSoftminGroup - 1) / kSoftminGroup : 0; }

__device__ __forceinline__ float block_reduce(float v, float* red, bool is_min) {
    #pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const float u = __shfl_xor_sync(0xFFFFFFFFu, v, o);
        v = is_min ? fminf(v, u) : v + u;
    }
    const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[w] = v;
    __syncthreads();
    float r = red[0];
    for (int i = 1; i < nw; ++i) r = is_min ? fminf(r, red[i]) : r + red[i];   // fixed order
    return r;
}

#ifdef MPPI_TC_TRACE
// Debug-only timeline of k_softmin (controller 0, T slice 0, first 1024 blocks): %globaltimer at block start,
// after phase 1, after the reductions, after phase 2, after the combine (last block only), and the SM id
__device__ unsigned long long g_sm_trace[1024][10];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define SM_TRACE(i)                                                                                    \
    do {                                                                                               \
        if (blockIdx.y == 0 && blockIdx.z == 0 && blockIdx.x < 1024 && threadIdx.x == 0) {             \
            g_sm_trace[blockIdx.x][i] = gtimer();                                                      \
            if ((i) == 0) { unsigned s_; asm("mov.u32 %0, %%smid;" : "=r"(s_)); g_sm_trace[blockIdx.x][5] = s_; } \
        }                                                                                              \
    } while (0)
int softmin_trace_copy(unsigned long long* host, int max_entries) {
    const int n = max_entries < 1024 * 10 ? max_entries : 1024 * 10;
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(host, g_sm_trace, (size_t)n * 8);
    return n;
}
#else
#define SM_TRACE(i) do {} while (0)
int softmin_trace_copy(unsigned long long*, int) { return 0; }
#endif

// four sums with the tree of block_reduce per component (same results as four block_reduce calls)
__device__ __forceinline__ float4 block_reduce4(float4 v, float4* red4) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        v.x += __shfl_xor_sync(0xFFFFFFFFu, v.x, o);
        v.y += __shfl_xor_sync(0xFFFFFFFFu, v.y, o);
        v.z += __shfl_xor_sync(0xFFFFFFFFu, v.z, o);
        v.w += __shfl_xor_sync(0xFFFFFFFFu, v.w, o);
    }
    const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red4[w] = v;
    __syncthreads();
    float4 r = red4[0];
    for (int i = 1; i < nw; ++i) {
        const float4 q = red4[i];
        r.x += q.x; r.y += q.y; r.z += q.z; r.w += q.w;
    }
    return r;
}

// Record combine of k_softmin (the softmin shard-combine identity; records in order): m = min m_b,
// f_b = exp((m - m_b)/lambda), S = sum S_b f_b, S2 = sum S2_b f_b^2, V = sum V_b f_b; final: U* = U + V/S (or this
// rank's record) and the diagnostics, else the group record out_rec. It runs once per step on one SM, so its code
// is cold in the instruction caches (trace build: ~5 us per phase of an unrolled, thrice-inlined form whatever
// the record count); hence one out-of-line copy (the final level runs right after the same SM's group level, so
// warm) of short rolled loops: record heads staged in shared memory (one record per thread), per-thread sums.
struct CombineOut {   // by value: a reference to the kernel's Params would copy them to every thread's stack
    int T, bb, W;
    float inv_lambda;
    float* record;
    const float* U_nom;
    float* U_out;
    float* diag;
    int* flags;
};
__device__ __noinline__ void softmin_combine(const CombineOut o, const float* recs, int n, bool final_level,
                                             float* out_rec, int write_record, float (*s_hd)[kSoftminThreads],
                                             float* s_f) {
    const int W = o.W, bb = o.bb;
    const int nh = min(n, kSoftminThreads);
    if (threadIdx.x < nh) {
        const float* r = recs + (long long)threadIdx.x * W;
        const float h0 = __ldcg(r), h1 = __ldcg(r + 1), h2 = __ldcg(r + 2), h3 = __ldcg(r + 3), h4 = __ldcg(r + 4);
        s_hd[0][threadIdx.x] = h0; s_hd[1][threadIdx.x] = h1; s_hd[2][threadIdx.x] = h2;
        s_hd[3][threadIdx.x] = h3; s_hd[4][threadIdx.x] = h4;
    }
    __syncthreads();
    float mg = INFINITY;
#pragma unroll 1
    for (int i = 0; i < nh; ++i) mg = fminf(mg, s_hd[0][i]);
#pragma unroll 1
    for (int i = nh; i < n; ++i) mg = fminf(mg, __ldcg(recs + (long long)i * W));
    const bool ok = mg < INFINITY;
    if (threadIdx.x < nh) {
        const float mi = s_hd[0][threadIdx.x];
        s_f[threadIdx.x] = (ok && mi < INFINITY) ? expf((mg - mi) * o.inv_lambda) : 0.f;
    }
    __syncthreads();
    auto fscale_far = [&](int i) {   // records past the first 512
        const float mi = __ldcg(recs + (long long)i * W);
        return (ok && mi < INFINITY) ? expf((mg - mi) * o.inv_lambda) : 0.f;
    };
    float Sg = 0.f, S2g = 0.f, SJg = 0.f, NJg = 0.f;
#pragma unroll 1
    for (int i = 0; i < nh; ++i) {
        const float f = s_f[i];
        Sg = fmaf(s_hd[1][i], f, Sg);
        S2g = fmaf(s_hd[2][i] * f, f, S2g);
        SJg += s_hd[3][i];
        NJg += s_hd[4][i];
    }
#pragma unroll 1
    for (int i = nh; i < n; ++i) {
        const float f = fscale_far(i);
        const float* r = recs + (long long)i * W;
        Sg = fmaf(__ldcg(r + 1), f, Sg);
        S2g = fmaf(__ldcg(r + 2) * f, f, S2g);
        SJg += __ldcg(r + 3);
        NJg += __ldcg(r + 4);
    }
#pragma unroll 1
    for (int tc = threadIdx.x; tc < 4 * o.T; tc += blockDim.x) {
        float V = 0.f;
        if (ok) {
#pragma unroll 8
            for (int i = 0; i < nh; ++i) V = fmaf(__ldcg(recs + (long long)i * W + kRecHead + tc), s_f[i], V);
#pragma unroll 1
            for (int i = nh; i < n; ++i) V = fmaf(__ldcg(recs + (long long)i * W + kRecHead + tc), fscale_far(i), V);
        }
        const int t = tc >> 2, c = tc & 3;
        if (!final_level) {
            out_rec[kRecHead + tc] = V;
        } else if (write_record) {
            o.record[(long long)bb * W + kRecHead + tc] = V;
        } else {
            const float Uv = o.U_nom[((long long)bb * o.T + t) * 4 + c];
            o.U_out[((long long)bb * o.T + t) * 4 + c] = (ok && Sg > 0.f) ? Uv + V / Sg : Uv;
        }
    }
    if (threadIdx.x == 0) {
        float* out = !final_level ? out_rec : write_record ? o.record + (long long)bb * W : nullptr;
        if (out) {
            out[0] = mg; out[1] = Sg; out[2] = S2g; out[3] = SJg;
            out[4] = NJg; out[5] = out[6] = out[7] = 0.f;
        } else {
            float* d = o.diag + bb * 4;
            d[0] = mg;
            d[1] = Sg;
            d[2] = S2g > 0.f ? Sg * Sg / S2g : 0.f;
            d[3] = NJg > 0.f ? SJg / NJg : INFINITY;
            o.flags[bb] = ok ? 0 : 1;
        }
    }
}

// resident blocks per SM: 256-sample blocks two (64 registers), 512-sample blocks one
template <int kSoftminBlock>
__host__ __device__ constexpr int kSoftminMinBlocks() { return kSoftminBlock == 256 ? 2 : 1; }

template <int kSoftminBlock>
__global__ void __launch_bounds__(kSoftminThreads, kSoftminMinBlocks<kSoftminBlock>()) k_softmin(Params p, Buffers b, int write_record) {
    __shared__ float s_w[kSoftminBlock];
    // phase 1 partition: a thread sums the terms of 4 consecutive samples (float4 loads, 16 in flight: 256 B per
    // thread, enough bytes in flight per SM to stream the terms at HBM rate) over one of NSL time slices
    constexpr int QB = kSoftminBlock / 4, NSL = kSoftminThreads / QB;
    __shared__ float s_part[NSL][kSoftminBlock];
    __shared__ float red[kSoftminThreads / 32];
    __shared__ float4 red4[kSoftminThreads / 32];
    __shared__ bool s_last;
    // grid (sample blocks, controllers, T slices): every T slice recomputes the sample block's J, m, S
    // (identically) and accumulates V only over its own time steps, so the noise-bound phase 2 runs on
    // gridDim.z times more SMs without adding block records
    const int bb = blockIdx.y, nblk = gridDim.x, tz = blockIdx.z, nz_t = gridDim.z;
    const int kk = threadIdx.x % kSoftminBlock, half = threadIdx.x / kSoftminBlock;
    const int k = blockIdx.x * kSoftminBlock + kk;
    const int W = kRecHead + 4 * p.T;   // m, S, S2, SJ, N, pad x3, V[T][4] (16-B aligned)
    // ---- phase 1: J_k = partial_k + sum over the NSL slices (in order) of each slice's terms summed in t order
    SM_TRACE(0);
    float J = INFINITY;
    {
        const int q = threadIdx.x % QB, sl = threadIdx.x / QB;
        const int kq = blockIdx.x * kSoftminBlock + 4 * q;
        const int th = (p.T + NSL - 1) / NSL, t0 = sl * th, t1 = min(p.T, t0 + th);
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        if (kq < p.K) {
            const float* tp = b.terms + (long long)bb * p.T * p.K + kq;
            if ((p.K & 3) == 0) {   // 16-B aligned quads (every config; ragged K takes the scalar form)
                const long long st4 = p.K / 4;
                const float4* tp4 = reinterpret_cast<const float4*>(tp);
                constexpr int PB = kSoftminMinBlocks<kSoftminBlock>() == 2 ? 8 : 16;   // loads in flight (64 registers: 8)
                int t = t0;
                for (; t + PB <= t1; t += PB) {
                    float4 v[PB];
#pragma unroll
                    for (int i = 0; i < PB; ++i) v[i] = __ldcs(tp4 + (long long)(t + i) * st4);
#pragma unroll
                    for (int i = 0; i < PB; ++i) {
                        acc.x += v[i].x; acc.y += v[i].y; acc.z += v[i].z; acc.w += v[i].w;
                    }
                }
                for (; t < t1; ++t) {
                    const float4 v = __ldcs(tp4 + (long long)t * st4);
                    acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
                }
            } else {
                const int nq = min(4, p.K - kq);
                for (int t = t0; t < t1; ++t) {
                    const float* r = tp + (long long)t * p.K;
                    acc.x += __ldcs(r);
                    if (nq > 1) acc.y += __ldcs(r + 1);
                    if (nq > 2) acc.z += __ldcs(r + 2);
                    if (nq > 3) acc.w += __ldcs(r + 3);
                }
            }
        }
        *reinterpret_cast<float4*>(&s_part[sl][4 * q]) = acc;
        __syncthreads();
        if (half == 0 && k < p.K) {
            float tsum = s_part[0][kk];
#pragma unroll
            for (int i = 1; i < NSL; ++i) tsum += s_part[i][kk];
            const float a = b.partial[(long long)bb * p.K + k] + tsum;
            J = isfinite(a) ? a : INFINITY;
            if (tz == 0) b.J[(long long)bb * p.K + k] = J;
        }
    }
    SM_TRACE(1);
    const float m = block_reduce(J, red, true);
    const float w = (J < INFINITY) ? expf((m - J) * p.inv_lambda) : 0.f;   // 0 for the second half
    if (half == 0) s_w[kk] = w;
    // S, S2 and the mean-cost diagnostic (sum and count of the finite costs) in one reduction
    const float4 sums = block_reduce4(make_float4(w, w * w, J < INFINITY ? J : 0.f, J < INFINITY ? 1.f : 0.f), red4);
    const float S = sums.x;
    float* rec = b.blkrec + ((long long)bb * nblk + blockIdx.x) * W;
    if (tz == 0 && threadIdx.x == 0) {
        rec[0] = m; rec[1] = S; rec[2] = sums.y; rec[3] = sums.z;
        rec[4] = sums.w; rec[5] = rec[6] = rec[7] = 0.f;
    }
    // ---- phase 2: warp per time step (coalesced over the block's samples), fixed shuffle tree
    const int kn = min(kSoftminBlock, p.K - (int)blockIdx.x * kSoftminBlock);
    const long long NK = (long long)p.n_ctrl * p.K;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const int tsl = (p.T + nz_t - 1) / nz_t, tb = tz * tsl, te = min(p.T, tb + tsl);
    SM_TRACE(2);
    // this lane's softmin weights (samples lane + 32 r) in registers for every t of the warp
    constexpr int PER = kSoftminBlock / 32;
    float wr[PER];
#pragma unroll
    for (int r = 0; r < PER; ++r) {
        const int i = lane + 32 * r;
        wr[r] = i < kn ? s_w[i] : 0.f;
    }
    // V[t] partial of one half (PH float4 per lane) of the block's samples, in sample order
    // parts per t: 512-sample blocks (one block per SM): 2 x 8 float4, each part's loads in flight while the
    // previous part is summed (measured configs[3]: the same time at two blocks per SM with 4 x 4); 256-sample
    // blocks (two per SM, 64 registers): one part of 8 (the ping-pong form spills there: configs[4] 0.20 -> 0.23 ms)
    constexpr int PH = 8, NH = PER / PH;
    auto v_load = [&](int t, int h, float4 (&nv)[PH]) {
        const float4* nz = b.noise + (long long)t * NK + (long long)bb * p.K + (long long)blockIdx.x * kSoftminBlock;
#pragma unroll
        for (int r = 0; r < PH; ++r) {
            const int i = lane + 32 * (h * PH + r);
            nv[r] = i < kn ? __ldcs(nz + i) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
    };
    auto v_acc = [&](const float4& U, int h, const float4 (&nv)[PH], float4& v) {
#pragma unroll
        for (int r = 0; r < PH; ++r) {
            const int i = lane + 32 * (h * PH + r);
            if (i < kn) {
                const float wi = wr[h * PH + r];
                const float4 n = nv[r];
                v.x = fmaf(wi, clampf(U.x + p.sigma[0] * n.x, p.u_lo[0], p.u_hi[0]) - U.x, v.x);
                v.y = fmaf(wi, clampf(U.y + p.sigma[1] * n.y, p.u_lo[1], p.u_hi[1]) - U.y, v.y);
                v.z = fmaf(wi, clampf(U.z + p.sigma[2] * n.z, p.u_lo[2], p.u_hi[2]) - U.z, v.z);
                v.w = fmaf(wi, clampf(U.w + p.sigma[3] * n.w, p.u_lo[3], p.u_hi[3]) - U.w, v.w);
            }
        }
    };
    auto v_store = [&](int t, float4 v) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            v.x += __shfl_xor_sync(0xFFFFFFFFu, v.x, o);
            v.y += __shfl_xor_sync(0xFFFFFFFFu, v.y, o);
            v.z += __shfl_xor_sync(0xFFFFFFFFu, v.z, o);
            v.w += __shfl_xor_sync(0xFFFFFFFFu, v.w, o);
        }
        if (lane == 0) reinterpret_cast<float4*>(rec + kRecHead)[t] = v;
    };
    const bool live = m < INFINITY;
    if constexpr (NH == 1) {
        for (int t = tb + warp; t < te; t += nw) {
            const float4 U = reinterpret_cast<const float4*>(b.U_nom)[(long long)bb * p.T + t];
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (live) {   // all of this lane's loads for step t first, then the sums in sample order
                float4 nv[PH];
                v_load(t, 0, nv);
                v_acc(U, 0, nv, v);
            }
            v_store(t, v);
        }
    } else {
        static_assert(NH % 2 == 0, "ping-pong over an even number of parts");
        float4 A[PH], B[PH];
        int t = tb + warp;
        if (live && t < te) v_load(t, 0, A);
        for (; t < te; t += nw) {
            const float4 U = reinterpret_cast<const float4*>(b.U_nom)[(long long)bb * p.T + t];
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (live) {
#pragma unroll
                for (int h = 0; h < NH; ++h) {
                    float4(&cur)[PH] = (h & 1) ? B : A;
                    float4(&nxt)[PH] = (h & 1) ? A : B;
                    if (h + 1 < NH) v_load(t, h + 1, nxt);
                    else if (t + nw < te) v_load(t + nw, 0, nxt);
                    v_acc(U, h, cur, v);
                }
            }
            v_store(t, v);
        }
    }
    SM_TRACE(3);
    // ---- combine the block records in order (the softmin shard-combine identity, so the result is exact up to
    // rounding and deterministic): m = min m_b, f_b = exp((m - m_b)/lambda), S = sum S_b f_b, V = sum V_b f_b.
    // Up to 32 sample blocks: the last block of the controller (atomic ticket) combines them all. More (configs[3]:
    // 256): two levels -- the last block of each group of kSoftminGroup sample blocks combines the group into a
    // group record, the last group combiner combines the group records -- so the single-SM tail reads
    // kSoftminGroup + n_groups records instead of nblk (measured configs[3]: 18 us of a 69 us kernel flat).
    __shared__ float s_hd[5][kSoftminThreads];   // record heads of a combine (softmin_combine)
    __shared__ float s_f[kSoftminThreads];
    auto combine = [&](const float* recs, int n, bool final_level, float* out_rec) {
        const CombineOut o{p.T, bb, W, p.inv_lambda, b.record, b.U_nom, b.U_out, b.diag, b.flags};
        softmin_combine(o, recs, n, final_level, out_rec, write_record, s_hd, s_f);
    };
    // arrive on a ticket; true for the block that completes it (which resets it for the next step). The block's
    // record writes reach thread 0 through the barrier and the device through its fence (the grid-barrier
    // pattern: one fence per block, not one per thread -- 512 MEMBAR.SC.GPU cost microseconds on the tail)
    auto last_arrival = [&](unsigned* ticket, unsigned count) {
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            s_last = atomicAdd(ticket, 1u) == count - 1u;
            if (s_last) {
                *ticket = 0u;   // every arrival of this step is in (the kernel boundary orders the next step)
                __threadfence();
            }
        }
        __syncthreads();
        return s_last;
    };
    const int ngrp = softmin_groups(nblk);
    if (ngrp == 0) {
        if (!last_arrival(b.tickets + bb, (unsigned)(nblk * nz_t))) return;
        SM_TRACE(6);
        combine(b.blkrec + (long long)bb * nblk * W, nblk, true, nullptr);
    } else {
        const int g = blockIdx.x / kSoftminGroup, members = min(kSoftminGroup, nblk - g * kSoftminGroup);
        float* grec = b.blkrec + (long long)p.n_ctrl * nblk * W + ((long long)bb * ngrp + g) * W;
        if (!last_arrival(b.tickets + p.n_ctrl + (long long)bb * ngrp + g, (unsigned)(members * nz_t))) return;
        combine(b.blkrec + ((long long)bb * nblk + (long long)g * kSoftminGroup) * W, members, false, grec);
        if (!last_arrival(b.tickets + bb, (unsigned)ngrp)) return;
        SM_TRACE(6);
        combine(b.blkrec + (long long)p.n_ctrl * nblk * W + (long long)bb * ngrp * W, ngrp, true, nullptr);
    }
    SM_TRACE(4);
}

void launch_softmin(const Params& p, const Buffers& b, bool write_record, cudaStream_t s) {
    const int spb = softmin_spb(p.K);
    const int nblk = (p.K + spb - 1) / spb;
    // T slices so that about 128 blocks run (c1: 8, c2: 2, configs[4]: 1); a slice is >= 8 steps
    int tsplit = 1;
    while (tsplit < 8 && (long long)nblk * p.n_ctrl * tsplit * 2 <= 128 && p.T / (tsplit * 2) >= 8) tsplit *= 2;
    dim3 grid(nblk, p.n_ctrl, tsplit);
    if (spb == 512) k_softmin<512><<<grid, kSoftminThreads, 0, s>>>(p, b, write_record ? 1 : 0);
    else k_softmin<256><<<grid, kSoftminThreads, 0, s>>>(p, b, write_record ? 1 : 0);
}

int softmin_blocks(int K) { return (K + softmin_spb(K) - 1) / softmin_spb(K); }
int softmin_group_count(int K) { return softmin_groups(softmin_blocks(K)); }

// ------------------------------------------------------------------ shard combine (configs[3])
// m = min_r m_r; S = sum_r S_r e^{-(m_r - m)/lambda}; V = sum_r V_r e^{...}; U* = U + V/S.
// Every rank combines in rank order, so every rank gets bitwise-identical U*.
__global__ void k_combine(Params p, Buffers b, const float* recs, int R) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= p.n_ctrl * p.T) return;
    const int bb = i / p.T, t = i % p.T;
    const int W = kRecHead + 4 * p.T;   // m, S, S2, SJ, N, pad x3, V[T][4] (16-B aligned)
    float m = INFINITY;
    for (int r = 0; r < R; ++r) m = fminf(m, recs[((long long)r * p.n_ctrl + bb) * W]);
    const float4 U = reinterpret_cast<const float4*>(b.U_nom)[(long long)bb * p.T + t];
    float4 Un = U;
    float S = 0.f, S2 = 0.f, SJ = 0.f, NJ = 0.f, v[4] = {0.f, 0.f, 0.f, 0.f};
    for (int r = 0; r < R; ++r) {
        const float* rec = recs + ((long long)r * p.n_ctrl + bb) * W;
        SJ += rec[3];
        NJ += rec[4];
    }
    if (isfinite(m)) {
        for (int r = 0; r < R; ++r) {
            const float* rec = recs + ((long long)r * p.n_ctrl + bb) * W;
            if (!(rec[0] < INFINITY)) continue;
            const float f = expf((m - rec[0]) * p.inv_lambda);
            S += rec[1] * f;
            S2 += rec[2] * f * f;
            for (int c = 0; c < 4; ++c) v[c] += rec[kRecHead + 4 * t + c] * f;
        }
        if (S > 0.f) {
            Un.x = U.x + v[0] / S; Un.y = U.y + v[1] / S; Un.z = U.z + v[2] / S; Un.w = U.w + v[3] / S;
        }
    }
    reinterpret_cast<float4*>(b.U_out)[(long long)bb * p.T + t] = Un;
    if (t == 0) {
        float* d = b.diag + bb * 4;
        d[0] = m;
        d[1] = S;
        d[2] = S2 > 0.f ? S * S / S2 : 0.f;
        d[3] = NJ > 0.f ? SJ / NJ : INFINITY;
        b.flags[bb] = isfinite(m) ? 0 : 1;
    }
}

void launch_combine(const Params& p, const Buffers& b, const float* recs, int R, cudaStream_t s) {
    const int n = p.n_ctrl * p.T;
    k_combine<<<(n + 127) / 128, 128, 0, s>>>(p, b, recs, R);
}

// ------------------------------------------------------------------ debug: normalised softmin weights
// w_k = exp(-(J_k - J_min)/lambda) / S (Eq. 5) of the last step, from its costs and the
// (J_min, S) the update used (diag); on demand for mppi_debug_copy(MPPI_DBG_WEIGHTS), not on the step path.
__global__ void k_weights(Params p, Buffers b) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (long long)p.n_ctrl * p.K) return;
    const int bb = (int)(i / p.K);
    const float m = b.diag[bb * 4], S = b.diag[bb * 4 + 1], J = b.J[i];
    b.weights[i] = (J < INFINITY && m < INFINITY && S > 0.f) ? expf((m - J) * p.inv_lambda) / S : 0.f;
}

void launch_weights(const Params& p, const Buffers& b, cudaStream_t s) {
    const long long n = (long long)p.n_ctrl * p.K;
    k_weights<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(p, b);
}

// ------------------------------------------------------------------ analytic Gate-SDF provider (F4)
// s_guide(p) = c + |x| tan(alpha) - max(|y|, |z|) in the gate frame (Eqs. 1-2), on the
// step's query rows; writes the same SDF stage term the MLP epilogue would (model 0: 50 e^{-s/0.1} and the
// forward-difference guidance; model 1: the Eq. 8 hinge). Thread per state.
__device__ __forceinline__ float gate_sdf(const Params& p, float4 q) {
    return p.gate_c + fabsf(q.x) * p.gate_tana - fmaxf(fabsf(q.y), fabsf(q.z));
}

__global__ void k_sdf_gate(Params p, Buffers b, float* sdf_out) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long n = (long long)p.n_ctrl * p.T * p.K;
    if (i >= n) return;
    const float4 q0 = b.rows[i * p.rps];
    const float s0 = gate_sdf(p, q0);
    float s1 = s0;
    if (p.rps == 2) s1 = gate_sdf(p, b.rows[i * 2 + 1]);
    if (sdf_out) {
        sdf_out[i * p.rps] = s0;
        if (p.rps == 2) sdf_out[i * 2 + 1] = s1;
    }
    float term;
    if (p.model == MPPI_MODEL_PAPER) {
        term = p.q_sdf * fmaxf(p.d_safe - s0, 0.f);
    } else {
        term = p.w_sdf * expf(fminf(-s0 * p.inv_sdf_scale, p.sdf_exp_max));
        if (p.rps == 2) term -= p.w_guide * q0.w * (s1 - s0) * p.inv_fd_h;
    }
    b.terms[i] = term;
}

void launch_sdf_gate(const Params& p, const Buffers& b, float* sdf_out, cudaStream_t s) {
    const long long n = (long long)p.n_ctrl * p.T * p.K;
    k_sdf_gate<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(p, b, sdf_out);
}

// ------------------------------------------------------------------ K5: latent fold
// b1'[b][j] = sum_l W1[j][3+l] z_b[l] + b1[j]: the latent concat of PAPER.md:40 folded into a bias.
__global__ void k_fold(Params p, Buffers b, int c0) {
    const int bb = c0 + blockIdx.x;
    for (int j = threadIdx.x; j < p.H; j += blockDim.x) {
        float acc = b.b1[j];
        const float* w = b.w1z + (size_t)j * p.L;
        const float* z = b.z + (size_t)bb * p.L;
        for (int l = 0; l < p.L; ++l) acc = fmaf(w[l], z[l], acc);
        b.b1f[(size_t)bb * p.H + j] = acc;
    }
}

void launch_fold(const Params& p, const Buffers& b, int c0, int count, cudaStream_t s) {
    k_fold<<<count, 256, 0, s>>>(p, b, c0);
}

}  // namespace mppi
