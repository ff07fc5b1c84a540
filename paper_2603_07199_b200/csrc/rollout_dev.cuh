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

__device__ __forceinline__ float sqrt_approx(float v) {
    float r;
    asm("sqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(v));
    return r;
}

// Standard normals of (global sample g, step t, iteration step): Philox4x32-10 (key = seed, counter =
// (g, t, step_lo, step_hi)), u = ((x >> 9) + 0.5) 2^-23, Box-Muller on (u0,u1), (u2,u3) (reading R24').
__device__ __forceinline__ float4 philox_normals(unsigned long long g, int t, unsigned long long step,
                                                 unsigned long long seed) {
    uint32_t c[4] = {(uint32_t)g, (uint32_t)t, (uint32_t)step, (uint32_t)(step >> 32)};
    philox4x32_10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
    const float s23 = 1.1920928955078125e-07f;  // 2^-23
    const float u0 = ((float)(c[0] >> 9) + 0.5f) * s23, u1 = ((float)(c[1] >> 9) + 0.5f) * s23;
    const float u2 = ((float)(c[2] >> 9) + 0.5f) * s23, u3 = ((float)(c[3] >> 9) + 0.5f) * s23;
    // fast SFU forms (MUFU.LG2 / SQRT / SIN / COS, abs error ~2^-21 on these ranges):
    // cos(2 pi u) = -cos(theta), sin(2 pi u) = -sin(theta), theta = 2 pi (u - 1/2) in [-pi, pi)
    const float r0 = sqrt_approx(-2.f * __logf(u0)), r1 = sqrt_approx(-2.f * __logf(u2));
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

// One CTBR rollout step of one sample (readings R4, R5, R7, R11, R12): the clamped
// input u = clamp(U*_t + sigma n), classic RK4 with u held, q renormalised; then the query rows of x_{t+1}
// in the cached frame (p_c = R p + t_q, |v|) and (p_c + h v_c/|v|, 0), and the non-SDF
// stage cost w_goal |p - g_c|^2 + w_u |u|^2 added to part. Shared by k_rollout and the fused rollout producers
// of the SDF-MLP kernels, so all produce the same rows.
// Issue-bound at configs[3..4] (one thread per sample, T dependent steps): the state updates run as f32x2
// pairs (FFMA2 / FADD2 on (px,py), (vx,vy), (qw,qx), (qy,qz); pz and vz scalar), the quaternion rates use the
// half body rates, |v| is MUFU.SQRT (sqrt.approx, ~1 ulp) -- about 200 instructions per step instead of ~300.
// The CTBR step splits into an attitude half and a translational half: q evolves on its own (q' = 1/2 q (x) w,
// w = the held body rates), and the translational dynamics read q only through the thrust direction terms of
// the four RK4 stage attitudes. ctbr_att_step computes the clamped input, the attitude RK4 step (q renormalised)
// and those stage terms; ctbr_trans_step the velocity / position RK4 step from them, the query rows and the
// stage cost. ctbr_step runs both in one thread (k_rollout, the fused producers). Running the two halves on two
// warps of a three-stage pipeline (noise / attitude / translation, 32 samples per block) was measured for the
// small configurations and does not shorten the chain (configs[1] rollout 19.3 vs 19.5 us, configs[2] 25 vs
// 27 us): within one thread the halves already overlap.
struct CtbrStage {   // per step: thrust-direction terms of the 4 stage attitudes, u0, |u|^2
    float bx[4], by[4], bz[4];
    float u0, uu;
};

// (bx, by, bz) of one attitude: a = (c/m) 2 (bx, by), az = (c/m)(1 - 2 bz) - g
__device__ __forceinline__ void ctbr_b3(float2 q01, float2 q23, float& bx, float& by, float& bz) {
    const float qw = q01.x, qx = q01.y, qy = q23.x, qz = q23.y;
    bx = fmaf(qx, qz, qw * qy);
    by = fmaf(qy, qz, -qw * qx);
    bz = fmaf(qx, qx, qy * qy);
}
// q' = 1/2 q (x) (0, w) with the half body rates hw
__device__ __forceinline__ void ctbr_dq(float2 q01, float2 q23, float hwx, float hwy, float hwz, float2& dq01,
                                       float2& dq23) {
    const float qw = q01.x, qx = q01.y, qy = q23.x, qz = q23.y;
    dq01.x = fmaf(-qx, hwx, fmaf(-qy, hwy, -qz * hwz));
    dq01.y = fmaf(qw, hwx, fmaf(qy, hwz, -qz * hwy));
    dq23.x = fmaf(qw, hwy, fmaf(qz, hwx, -qx * hwz));
    dq23.y = fmaf(qw, hwz, fmaf(qx, hwy, -qy * hwx));
}

// attitude half: u = clamp(U*_t + sigma n) (R5), RK4 of q with u held (q renormalised), stage terms
__device__ __forceinline__ void ctbr_att_step(const Params& p, float2& Q01, float2& Q23, float4 U, float4 n,
                                              CtbrStage& st) {
    const float dt = p.dt, hdt = 0.5f * p.dt, dt6 = p.dt * (1.f / 6.f);
    const float u0 = clampf(fmaf(p.sigma[0], n.x, U.x), p.u_lo[0], p.u_hi[0]);
    const float u1 = clampf(fmaf(p.sigma[1], n.y, U.y), p.u_lo[1], p.u_hi[1]);
    const float u2 = clampf(fmaf(p.sigma[2], n.z, U.z), p.u_lo[2], p.u_hi[2]);
    const float u3 = clampf(fmaf(p.sigma[3], n.w, U.w), p.u_lo[3], p.u_hi[3]);
    const float hwx = 0.5f * u1, hwy = 0.5f * u2, hwz = 0.5f * u3;
    const float2 H2 = make_float2(hdt, hdt), D2 = make_float2(dt, dt);
    float2 d01_1, d23_1, d01_2, d23_2, d01_3, d23_3, d01_4, d23_4;
    ctbr_b3(Q01, Q23, st.bx[0], st.by[0], st.bz[0]);
    ctbr_dq(Q01, Q23, hwx, hwy, hwz, d01_1, d23_1);
    const float2 q01_2 = __ffma2_rn(H2, d01_1, Q01), q23_2 = __ffma2_rn(H2, d23_1, Q23);
    ctbr_b3(q01_2, q23_2, st.bx[1], st.by[1], st.bz[1]);
    ctbr_dq(q01_2, q23_2, hwx, hwy, hwz, d01_2, d23_2);
    const float2 q01_3 = __ffma2_rn(H2, d01_2, Q01), q23_3 = __ffma2_rn(H2, d23_2, Q23);
    ctbr_b3(q01_3, q23_3, st.bx[2], st.by[2], st.bz[2]);
    ctbr_dq(q01_3, q23_3, hwx, hwy, hwz, d01_3, d23_3);
    const float2 q01_4 = __ffma2_rn(D2, d01_3, Q01), q23_4 = __ffma2_rn(D2, d23_3, Q23);
    ctbr_b3(q01_4, q23_4, st.bx[3], st.by[3], st.bz[3]);
    ctbr_dq(q01_4, q23_4, hwx, hwy, hwz, d01_4, d23_4);
    const float2 T2 = make_float2(2.f, 2.f), S6 = make_float2(dt6, dt6);
    const float2 s01 = __fadd2_rn(__ffma2_rn(T2, __fadd2_rn(d01_2, d01_3), d01_1), d01_4);
    const float2 s23 = __fadd2_rn(__ffma2_rn(T2, __fadd2_rn(d23_2, d23_3), d23_1), d23_4);
    float2 q01 = __ffma2_rn(S6, s01, Q01), q23 = __ffma2_rn(S6, s23, Q23);
    const float qinv = rsqrtf(fmaf(q01.x, q01.x, fmaf(q01.y, q01.y, fmaf(q23.x, q23.x, q23.y * q23.y))));  // MUFU
    const float2 QI = make_float2(qinv, qinv);
    Q01 = __fmul2_rn(q01, QI);
    Q23 = __fmul2_rn(q23, QI);
    st.u0 = u0;
    st.uu = fmaf(u0, u0, fmaf(u1, u1, fmaf(u2, u2, u3 * u3)));
}

// translational half: RK4 of (p, v) with the stage accelerations a_s = (c/m)(2 bx, 2 by, 1 - 2 bz) - g e_z,
// then the query rows of x_{t+1} in the cached frame (p_c = R p + t_q, |v|) and (p_c + h v_c/|v|, 0)
// (reading R7) and the non-SDF stage cost w_goal |p - g_c|^2 + w_u |u|^2
__device__ __forceinline__ void ctbr_trans_step(const Params& p, float2& P, float& pz, float2& V, float& vz,
                                                const CtbrStage& st, const float (&R)[9], const float (&tq)[3],
                                                const float (&gc)[3], float inv_mass, float4& row0, float4& row1,
                                                float& part) {
    const float dt = p.dt, hdt = 0.5f * p.dt, dt6 = p.dt * (1.f / 6.f), g = p.gravity;
    const float com = st.u0 * inv_mass, com2 = 2.f * com, comg = com - g;
    const float2 H2 = make_float2(hdt, hdt), D2 = make_float2(dt, dt);
    float2 a[4];
    float az[4];
#pragma unroll
    for (int s2 = 0; s2 < 4; ++s2) {
        a[s2] = make_float2(com2 * st.bx[s2], com2 * st.by[s2]);
        az[s2] = fmaf(-com2, st.bz[s2], comg);
    }
    const float2 V2 = __ffma2_rn(H2, a[0], V);
    const float vz2 = fmaf(hdt, az[0], vz);
    const float2 V3 = __ffma2_rn(H2, a[1], V);
    const float vz3 = fmaf(hdt, az[1], vz);
    const float2 V4 = __ffma2_rn(D2, a[2], V);
    const float vz4 = fmaf(dt, az[2], vz);
    // x + dt/6 (k1 + 2 k2 + 2 k3 + k4); the position rates k_i are the stage velocities V, V2, V3, V4
    const float2 T2 = make_float2(2.f, 2.f), S6 = make_float2(dt6, dt6);
    const float2 sP = __fadd2_rn(__ffma2_rn(T2, __fadd2_rn(V2, V3), V), V4);
    const float2 sV = __fadd2_rn(__ffma2_rn(T2, __fadd2_rn(a[1], a[2]), a[0]), a[3]);
    P = __ffma2_rn(S6, sP, P);
    const float vz0 = vz;
    V = __ffma2_rn(S6, sV, V);
    pz = fmaf(dt6, fmaf(2.f, vz2 + vz3, vz0) + vz4, pz);
    vz = fmaf(dt6, fmaf(2.f, az[1] + az[2], az[0]) + az[3], vz0);
    const float x[6] = {P.x, P.y, pz, V.x, V.y, vz};
    float pc[3], dv[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
        pc[r] = fmaf(R[3 * r], x[0], fmaf(R[3 * r + 1], x[1], fmaf(R[3 * r + 2], x[2], tq[r])));
        dv[r] = fmaf(R[3 * r], x[3], fmaf(R[3 * r + 1], x[4], R[3 * r + 2] * x[5]));
    }
    const float nv = sqrt_approx(fmaf(x[3], x[3], fmaf(x[4], x[4], x[5] * x[5])));
    const float sc = nv >= 1e-6f ? __fdividef(p.fd_h, nv) : 0.f;
    row0 = make_float4(pc[0], pc[1], pc[2], nv);
    row1 = make_float4(fmaf(sc, dv[0], pc[0]), fmaf(sc, dv[1], pc[1]), fmaf(sc, dv[2], pc[2]), 0.f);
    const float dx = x[0] - gc[0], dy = x[1] - gc[1], dz = x[2] - gc[2];
    part += p.w_goal * fmaf(dx, dx, fmaf(dy, dy, dz * dz)) + p.w_u * st.uu;
}

// One CTBR rollout step of one sample in one thread (readings R4, R5, R7, R11, R12): the
// attitude half then the translational half. Shared by k_rollout and the fused rollout producers of the SDF-MLP
// kernels, so all produce the same rows.
// Issue-bound at configs[3..4]: the state updates run as f32x2 pairs (FFMA2 / FADD2 on (px,py), (vx,vy),
// (qw,qx), (qy,qz); pz and vz scalar), the quaternion rates use the half body rates, |v| is MUFU.SQRT
// (sqrt.approx, ~1 ulp).
__device__ __forceinline__ void ctbr_step(const Params& p, float (&x)[10], float4 U, float4 n, const float (&R)[9],
                                          const float (&tq)[3], const float (&gc)[3], float inv_mass, float4& row0,
                                          float4& row1, float& part) {
    float2 P = make_float2(x[0], x[1]), V = make_float2(x[3], x[4]);
    float pz = x[2], vz = x[5];
    float2 Q01 = make_float2(x[6], x[7]), Q23 = make_float2(x[8], x[9]);
    CtbrStage st;
    ctbr_att_step(p, Q01, Q23, U, n, st);
    ctbr_trans_step(p, P, pz, V, vz, st, R, tq, gc, inv_mass, row0, row1, part);
    x[0] = P.x; x[1] = P.y; x[2] = pz; x[3] = V.x; x[4] = V.y; x[5] = vz;
    x[6] = Q01.x; x[7] = Q01.y; x[8] = Q23.x; x[9] = Q23.y;
}

}  // namespace mppi
