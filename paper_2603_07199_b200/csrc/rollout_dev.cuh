// Device code of the CTBR rollout shared by k_rollout (kernels_simt.cu) and the fused rollout producer of
// the H = 128 SDF-MLP kernel (kernel_mlp_h128.cu): the noise generator (reading R24'), the dynamics
// (PAPER.md:146 in the CTBR form of BASELINE configs[0]; readings R1-R4) and one rollout step. Nothing here is
// shared with oracle/.
#pragma once
#include <math.h>
#include <stdint.h>

#include "../../include/mppi.h"
#include "mppi_internal.cuh"

namespace mppi {

__device__ __forceinline__ void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        const uint32_t lo0 = 0xD2511F53u * c[0], hi0 = __umulhi(0xD2511F53u, c[0]);
        const uint32_t lo1 = 0xCD9E8D57u * c[2], hi1 = __umulhi(0xCD9E8D57u, c[2]);
        const uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
        c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
    }
}

__device__ __forceinline__ float clampf(float v, float lo, float hi) { return fminf(fmaxf(v, lo), hi); }

// Standard normals of (global sample g, step t, iteration step): Philox4x32-10 (key = seed, counter =
// (g, t, step_lo, step_hi)), u = ((x >> 9) + 0.5) 2^-23, Box-Muller on (u0,u1), (u2,u3) (reading R24').
__device__ __forceinline__ float4 philox_normals(unsigned long long g, int t, unsigned long long step,
                                                 unsigned long long seed) {
    uint32_t c[4] = {(uint32_t)g, (uint32_t)t, (uint32_t)step, (uint32_t)(step >> 32)};
    philox4x32_10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
    const float s23 = 1.1920928955078125e-07f;  // 2^-23
    const float u0 = ((float)(c[0] >> 9) + 0.5f) * s23, u1 = ((float)(c[1] >> 9) + 0.5f) * s23;
    const float u2 = ((float)(c[2] >> 9) + 0.5f) * s23, u3 = ((float)(c[3] >> 9) + 0.5f) * s23;
    // fast SFU forms (MUFU.LG2 / SIN / COS, abs error ~2^-21 on these ranges):
    // cos(2 pi u) = -cos(theta), sin(2 pi u) = -sin(theta), theta = 2 pi (u - 1/2) in [-pi, pi)
    const float r0 = sqrtf(-2.f * __logf(u0)), r1 = sqrtf(-2.f * __logf(u2));
    float s0, c0, s1, c1;
    __sincosf(6.283185307179586f * (u1 - 0.5f), &s0, &c0);
    __sincosf(6.283185307179586f * (u3 - 0.5f), &s1, &c1);
    return make_float4(-r0 * c0, -r0 * s0, -r1 * c1, -r1 * s1);
}

// Global sample index keying the noise (reading R24'): controller ctrl_offset + b of the whole job, sample
// k_offset + k of its K_global, so every sharding (samples over ranks, configs[3]; controllers over ranks,
// configs[4]) draws exactly the samples of the unsharded job.
__device__ __forceinline__ unsigned long long global_sample(const Params& p, int bb, int k) {
    return (unsigned long long)(p.ctrl_offset + bb) * (unsigned long long)p.K_global + (unsigned long long)p.k_offset +
           (unsigned long long)k;
}

// CTBR dynamics xdot = f(x, u): x = [p, v, q(w,x,y,z)], com = c/m, body rates (wx, wy, wz).
__device__ __forceinline__ void dyn_ctbr(const float* x, float com, float wx, float wy, float wz, float g, float* xd) {
    const float qw = x[6], qx = x[7], qy = x[8], qz = x[9];
    xd[0] = x[3]; xd[1] = x[4]; xd[2] = x[5];
    xd[3] = com * (2.f * (qx * qz + qw * qy));
    xd[4] = com * (2.f * (qy * qz - qw * qx));
    xd[5] = com * (1.f - 2.f * (qx * qx + qy * qy)) - g;
    xd[6] = 0.5f * (-qx * wx - qy * wy - qz * wz);
    xd[7] = 0.5f * (qw * wx + qy * wz - qz * wy);
    xd[8] = 0.5f * (qw * wy + qz * wx - qx * wz);
    xd[9] = 0.5f * (qw * wz + qx * wy - qy * wx);
}


// One CTBR rollout step of one sample (readings R4, R5, R7, R11, R12): the clamped
// input u = clamp(U*_t + sigma n), classic RK4 with u held, q renormalised; then the query rows of x_{t+1}
// in the cached frame (p_c = R p + t_q, |v|) and (p_c + h v_c/|v|, 0), and the non-SDF
// stage cost w_goal |p - g_c|^2 + w_u |u|^2 added to part. Shared by k_rollout and the fused rollout producer
// of kernel_mlp_h128.cu, so both produce the same rows.
__device__ __forceinline__ void ctbr_step(const Params& p, float (&x)[10], float4 U, float4 n, const float (&R)[9],
                                          const float (&tq)[3], const float (&gc)[3], float inv_mass, float4& row0,
                                          float4& row1, float& part) {
    const float dt = p.dt, hdt = 0.5f * p.dt, dt6 = p.dt / 6.f, g = p.gravity;
    const float u0 = clampf(U.x + p.sigma[0] * n.x, p.u_lo[0], p.u_hi[0]);
    const float u1 = clampf(U.y + p.sigma[1] * n.y, p.u_lo[1], p.u_hi[1]);
    const float u2 = clampf(U.z + p.sigma[2] * n.z, p.u_lo[2], p.u_hi[2]);
    const float u3 = clampf(U.w + p.sigma[3] * n.w, p.u_lo[3], p.u_hi[3]);
    const float com = u0 * inv_mass;
    float k1[10], k2[10], k3[10], k4[10], xt[10];
    dyn_ctbr(x, com, u1, u2, u3, g, k1);
#pragma unroll
    for (int i = 0; i < 10; ++i) xt[i] = x[i] + hdt * k1[i];
    dyn_ctbr(xt, com, u1, u2, u3, g, k2);
#pragma unroll
    for (int i = 0; i < 10; ++i) xt[i] = x[i] + hdt * k2[i];
    dyn_ctbr(xt, com, u1, u2, u3, g, k3);
#pragma unroll
    for (int i = 0; i < 10; ++i) xt[i] = x[i] + dt * k3[i];
    dyn_ctbr(xt, com, u1, u2, u3, g, k4);
#pragma unroll
    for (int i = 0; i < 10; ++i) x[i] = x[i] + dt6 * (k1[i] + 2.f * k2[i] + 2.f * k3[i] + k4[i]);
    const float qinv = rsqrtf(x[6] * x[6] + x[7] * x[7] + x[8] * x[8] + x[9] * x[9]);   // MUFU, ~2 ulp
#pragma unroll
    for (int i = 6; i < 10; ++i) x[i] = x[i] * qinv;
    // query-frame position and direction, scored at x_{t+1} (reading R7)
    float pc[3], dv[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
        pc[r] = R[3 * r] * x[0] + R[3 * r + 1] * x[1] + R[3 * r + 2] * x[2] + tq[r];
        dv[r] = R[3 * r] * x[3] + R[3 * r + 1] * x[4] + R[3 * r + 2] * x[5];
    }
    const float nv = sqrtf(x[3] * x[3] + x[4] * x[4] + x[5] * x[5]);
    const float sc = nv >= 1e-6f ? __fdividef(p.fd_h, nv) : 0.f;
    row0 = make_float4(pc[0], pc[1], pc[2], nv);
    row1 = make_float4(pc[0] + sc * dv[0], pc[1] + sc * dv[1], pc[2] + sc * dv[2], 0.f);
    const float dx = x[0] - gc[0], dy = x[1] - gc[1], dz = x[2] - gc[2];
    part += p.w_goal * (dx * dx + dy * dy + dz * dz) + p.w_u * (u0 * u0 + u1 * u1 + u2 * u2 + u3 * u3);
}

}  // namespace mppi
