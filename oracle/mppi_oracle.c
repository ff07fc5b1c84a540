/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation of one MPPI iteration with a Gate-SDF cost
 * (arxiv 2603.07199), written step by step in the paper's order. Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it. It shares no code, header, table
 * or constant generator with the CUDA path under paper_2603_07199_b200/.
 *
 * Precision: every floating-point step is fp64, except the bf16 quantisation contract of BASELINE
 * configs[1..4] ("bf16, fp32 accumulate"; SURVEY.md §8c reading R15), which is emulated exactly:
 * hidden/output weights rounded once to bf16 (RNE), hidden activations rounded to bf16 after the
 * activation. Those rounding decisions are taken on the fp32 value of the activation (the kernel's
 * precision, as the task's rule for float-decides-integer asks).
 *
 * Citations (PAPER.md line, section/equation):
 *   sampling      U^m = U* + dU^m, dU ~ N(0, Sigma)                PAPER.md:139 (§IV-A)
 *   update        U* = sum w_m U^m, w = softmax(-J/lambda)         PAPER.md:140-144 (Eq. 5)
 *   dynamics      xdot = f(x,u)                                    PAPER.md:146 (§IV-A), CTBR form of
 *                 BASELINE configs[0] (state p,v,q; input thrust + body rates; RK4)
 *   SDF query     s_k = g_phi(z, p_k), latent once per frame      PAPER.md:168 (§IV-B3)
 *   cached frame  world -> cached camera transform                 PAPER.md:181 (§IV-B3)
 *   total cost    J = sum of weighted stage costs                  PAPER.md:185 (Eq. 10), with the
 *                 BASELINE configs[0..1] terms (||p-g_c||^2, 50 exp(-s/0.1), 0.01||u||^2, -0.5 grad s.v)
 *   analytic SDF  s_guide = c + |x| tan(a) - max(|y|,|z|)          PAPER.md:64-72 (Eqs. 1-2)
 *   PE            g_phi(z, PE(p)), PE(p) = [p, sin(2^i pi p), cos(2^i pi p)]_{i<B}  PAPER.md:121 (reading E1)
 *   paper model   (model 1; SURVEY.md §8f F1 + F2, readings P1-P7)
 *                 x = [p, v, q, w, T], u = [T1dot..T4dot]            PAPER.md:146 (§IV-A)
 *                 J_gate = sum_k |p_{k+1}-p_wp|^2 - |p_k-p_wp|^2   PAPER.md:153 (Eq. 6)
 *                 J_vis  = sum_k 1 - cos(psi_k - psi_gate,k)        PAPER.md:161 (Eq. 7)
 *                 C_sdf  = max(0, d_safe - s_k), J_sdf = sum_k C   PAPER.md:172, :177 (Eqs. 8-9)
 *                 J = Q_gate J_gate + Q_vis J_vis + Q_sdf J_sdf     PAPER.md:185 (Eq. 10); Table I
 *   noise RNG     Philox4x32-10 + Box-Muller (reading R24)        — parity unpinned against the paper
 *                 (the paper draws N(0,Sigma) without naming a generator); pinned to the Random123 KAT.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ACT_SOFTPLUS 0
#define ACT_RELU 1
#define ACT_SILU 2

typedef struct {
    int32_t n_ctrl, K, T;
    double dt, lambda, mass, gravity;
    double u_lo[4], u_hi[4], sigma[4];
    double w_goal, w_sdf, sdf_scale, sdf_exp_max, w_u, w_guide, fd_h;
    int32_t latent_dim, hidden, n_hidden, activation, mlp_bf16;
    int32_t sdf_mode;            /* 0: MLP g_phi; 1: analytic Gate-SDF (Eq. 2) in the query frame */
    double gate_c, gate_tana;    /* analytic-SDF parameters (sdf_mode 1) */
    int32_t model;               /* 0: BASELINE CTBR dynamics + configs[0..1] terms; 1: the paper's model */
    double arm, kappa;           /* model 1: rotor arm (m), yaw moment per unit thrust (m)           */
    double inertia[3];           /* model 1: diag(J) (kg m^2)                                         */
    double thrust_max, rate_max; /* model 1: T_i in [0, thrust_max] (N); |w_i| <= rate_max (rad/s)    */
    double q_gate, q_vis, q_sdf, d_safe;   /* model 1: Eq. 10 weights, Eq. 8 clearance               */
    int32_t pe_bands;            /* positional encoding PE(p) on the MLP input (reading E1) */
} oracle_cfg;

/* ------------------------------------------------------------------ Philox4x32-10 (Salmon et al.) */
static void philox_round(uint32_t c[4], const uint32_t k[2]) {
    uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
    uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c[1] ^ k[0];
    uint32_t n2 = hi0 ^ c[3] ^ k[1];
    c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
}

void oracle_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    uint32_t c[4] = {ctr[0], ctr[1], ctr[2], ctr[3]};
    uint32_t k[2] = {key[0], key[1]};
    for (int r = 0; r < 10; ++r) {
        if (r > 0) { k[0] += 0x9E3779B9u; k[1] += 0xBB67AE85u; }
        philox_round(c, k);
    }
    memcpy(out, c, sizeof(c));
}

/* Standard normals for global samples g0..g0+nK-1 (R24): key = seed, counter = (g, t, step_lo, step_hi);
 * u_i = ((x_i >> 9) + 0.5) * 2^-23 in (0,1) (24 significant bits: exact in fp32 as well as fp64);
 * Box-Muller on (u0,u1) -> n0,n1 and (u2,u3) -> n2,n3.
 * out: [T][nK][4]. */
void oracle_noise(uint64_t seed, uint64_t step, int64_t g0, int32_t nK, int32_t T, double* out) {
    const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    const double two_pi = 6.283185307179586476925286766559;
    for (int t = 0; t < T; ++t)
        for (int i = 0; i < nK; ++i) {
            uint64_t g = (uint64_t)(g0 + i);
            uint32_t ctr[4] = {(uint32_t)g, (uint32_t)t, (uint32_t)step, (uint32_t)(step >> 32)};
            uint32_t x[4];
            oracle_philox4x32_10(ctr, key, x);
            double u[4];
            for (int j = 0; j < 4; ++j) u[j] = ((double)(x[j] >> 9) + 0.5) * (1.0 / 8388608.0);
            double r0 = sqrt(-2.0 * log(u[0])), r1 = sqrt(-2.0 * log(u[2]));
            double* o = out + ((size_t)t * nK + i) * 4;
            o[0] = r0 * cos(two_pi * u[1]);
            o[1] = r0 * sin(two_pi * u[1]);
            o[2] = r1 * cos(two_pi * u[3]);
            o[3] = r1 * sin(two_pi * u[3]);
        }
}

/* ------------------------------------------------------------------ bf16 round-to-nearest-even */
static double bf16_round(double v) {
    float f = (float)v;                       /* decision taken on the fp32 value (kernel precision) */
    uint32_t u;
    memcpy(&u, &f, 4);
    if ((u & 0x7F800000u) == 0x7F800000u) {   /* inf / nan pass through (nan quieted) */
        if (u & 0x007FFFFFu) u |= 0x00400000u;
        u &= 0xFFFF0000u;
    } else {
        u += 0x7FFFu + ((u >> 16) & 1u);
        u &= 0xFFFF0000u;
    }
    memcpy(&f, &u, 4);
    return (double)f;
}

double oracle_bf16_round(double v) { return bf16_round(v); }

/* ------------------------------------------------------------------ dynamics (CTBR, R1-R4) */
/* x = [p(3), v(3), q(w,x,y,z)]; u = [c (N), wx, wy, wz (rad/s, body frame)].
 * pdot = v; vdot = (c/m) b3(q) - g e_z with b3(q) = R(q) e_z; qdot = 1/2 q (x) (0, w). */
static void dyn_f(const double* x, const double* u, double m, double g, double* xd) {
    const double qw = x[6], qx = x[7], qy = x[8], qz = x[9];
    const double c = u[0], wx = u[1], wy = u[2], wz = u[3];
    xd[0] = x[3]; xd[1] = x[4]; xd[2] = x[5];
    const double b3x = 2.0 * (qx * qz + qw * qy);
    const double b3y = 2.0 * (qy * qz - qw * qx);
    const double b3z = 1.0 - 2.0 * (qx * qx + qy * qy);
    xd[3] = c / m * b3x;
    xd[4] = c / m * b3y;
    xd[5] = c / m * b3z - g;
    /* Hamilton product q (x) (0, w) */
    xd[6] = 0.5 * (-qx * wx - qy * wy - qz * wz);
    xd[7] = 0.5 * (qw * wx + qy * wz - qz * wy);
    xd[8] = 0.5 * (qw * wy + qz * wx - qx * wz);
    xd[9] = 0.5 * (qw * wz + qx * wy - qy * wx);
}

/* Classic RK4 with the input held over the step; q renormalised after the full step only (R4). */
void oracle_rk4_step(const double* x, const double* u, double dt, double m, double g, double* out) {
    double k1[10], k2[10], k3[10], k4[10], xt[10];
    dyn_f(x, u, m, g, k1);
    for (int i = 0; i < 10; ++i) xt[i] = x[i] + 0.5 * dt * k1[i];
    dyn_f(xt, u, m, g, k2);
    for (int i = 0; i < 10; ++i) xt[i] = x[i] + 0.5 * dt * k2[i];
    dyn_f(xt, u, m, g, k3);
    for (int i = 0; i < 10; ++i) xt[i] = x[i] + dt * k3[i];
    dyn_f(xt, u, m, g, k4);
    for (int i = 0; i < 10; ++i) out[i] = x[i] + dt / 6.0 * (k1[i] + 2.0 * k2[i] + 2.0 * k3[i] + k4[i]);
    double qn = sqrt(out[6] * out[6] + out[7] * out[7] + out[8] * out[8] + out[9] * out[9]);
    for (int i = 6; i < 10; ++i) out[i] /= qn;
}

/* ------------------------------------------------------------------ dynamics (paper model, reading P1-P3) */
/* x = [p(3), v(3), q(w,x,y,z)(4), w(3) body rates, T(4) rotor thrusts], u = [T1dot..T4dot] (N/s).
 * pdot = v; vdot = (sum T / m) b3(q) - g e_z; qdot = 1/2 q (x) (0, w); wdot = J^-1 (tau - w x J w);
 * Tdot = u. X configuration, d = arm / sqrt(2), rotors at body (x, y):
 * 1 (+d, -d), 2 (-d, +d), 3 (+d, +d), 4 (-d, -d); 1, 2 spin one way and 3, 4 the other:
 * tau = (sum y_i T_i, -sum x_i T_i, kappa (T1 + T2 - T3 - T4)). */
void oracle_rotor_deriv(const oracle_cfg* cfg, const double* x, const double* u, double* xd) {
    const double qw = x[6], qx = x[7], qy = x[8], qz = x[9];
    const double wx = x[10], wy = x[11], wz = x[12];
    const double T1 = x[13], T2 = x[14], T3 = x[15], T4 = x[16];
    const double F = T1 + T2 + T3 + T4;
    const double d = cfg->arm / sqrt(2.0);
    xd[0] = x[3]; xd[1] = x[4]; xd[2] = x[5];
    xd[3] = F / cfg->mass * 2.0 * (qx * qz + qw * qy);
    xd[4] = F / cfg->mass * 2.0 * (qy * qz - qw * qx);
    xd[5] = F / cfg->mass * (1.0 - 2.0 * (qx * qx + qy * qy)) - cfg->gravity;
    xd[6] = 0.5 * (-qx * wx - qy * wy - qz * wz);
    xd[7] = 0.5 * (qw * wx + qy * wz - qz * wy);
    xd[8] = 0.5 * (qw * wy + qz * wx - qx * wz);
    xd[9] = 0.5 * (qw * wz + qx * wy - qy * wx);
    const double tx = d * (-T1 + T2 + T3 - T4);
    const double ty = -d * (T1 - T2 + T3 - T4);
    const double tz = cfg->kappa * (T1 + T2 - T3 - T4);
    const double Jx = cfg->inertia[0], Jy = cfg->inertia[1], Jz = cfg->inertia[2];
    /* w x (J w) */
    const double cx = wy * (Jz * wz) - wz * (Jy * wy);
    const double cy = wz * (Jx * wx) - wx * (Jz * wz);
    const double cz = wx * (Jy * wy) - wy * (Jx * wx);
    xd[10] = (tx - cx) / Jx;
    xd[11] = (ty - cy) / Jy;
    xd[12] = (tz - cz) / Jz;
    for (int i = 0; i < 4; ++i) xd[13 + i] = u[i];
}

/* RK4 with the input held over the step; then q renormalised, T clamped to [0, thrust_max], w clamped to
 * +-rate_max (reading P4). */
void oracle_rotor_step(const oracle_cfg* cfg, const double* x, const double* u, double* out) {
    const double dt = cfg->dt;
    double k1[17], k2[17], k3[17], k4[17], xt[17];
    oracle_rotor_deriv(cfg, x, u, k1);
    for (int i = 0; i < 17; ++i) xt[i] = x[i] + 0.5 * dt * k1[i];
    oracle_rotor_deriv(cfg, xt, u, k2);
    for (int i = 0; i < 17; ++i) xt[i] = x[i] + 0.5 * dt * k2[i];
    oracle_rotor_deriv(cfg, xt, u, k3);
    for (int i = 0; i < 17; ++i) xt[i] = x[i] + dt * k3[i];
    oracle_rotor_deriv(cfg, xt, u, k4);
    for (int i = 0; i < 17; ++i) out[i] = x[i] + dt / 6.0 * (k1[i] + 2.0 * k2[i] + 2.0 * k3[i] + k4[i]);
    double qn = sqrt(out[6] * out[6] + out[7] * out[7] + out[8] * out[8] + out[9] * out[9]);
    for (int i = 6; i < 10; ++i) out[i] /= qn;
    for (int i = 10; i < 13; ++i) out[i] = out[i] < -cfg->rate_max ? -cfg->rate_max : (out[i] > cfg->rate_max ? cfg->rate_max : out[i]);
    for (int i = 13; i < 17; ++i) out[i] = out[i] < 0.0 ? 0.0 : (out[i] > cfg->thrust_max ? cfg->thrust_max : out[i]);
}

/* ------------------------------------------------------------------ SDF providers */
static double act_fn(int a, double v) {
    switch (a) {
        case ACT_SOFTPLUS: return (v > 0.0 ? v : 0.0) + log1p(exp(-fabs(v)));
        case ACT_RELU: return v > 0.0 ? v : 0.0;
        default: return v / (1.0 + exp(-v));   /* SiLU */
    }
}

/* Positional encoding ("a positional encoding applied to the spatial coordinates before
 * concatenation"; reading E1): the raw coordinates, then per band i = 0..B-1 the six values
 * sin(2^i pi x), sin(2^i pi y), sin(2^i pi z), cos(2^i pi x), cos(2^i pi y), cos(2^i pi z). out: 3 + 6B. */
void oracle_pe(int bands, const double* p, double* out) {
    const double pi = 3.14159265358979323846264338327950288;
    for (int c = 0; c < 3; ++c) out[c] = p[c];
    for (int i = 0; i < bands; ++i)
        for (int c = 0; c < 3; ++c) {
            const double a = ldexp(pi * p[c], i);
            out[3 + 6 * i + c] = sin(a);
            out[3 + 6 * i + 3 + c] = cos(a);
        }
}

/* s = g_phi(z, p): layer 1 on [PE(p) | z] (PE(p) = p without PE; full dot, fp64, NOT folded); hidden
 * layers; linear output. W: all layers concatenated, each [out][in] row-major (nn.Linear); b likewise.
 * acts (may be NULL): [n_hidden][H] post-activation values of every hidden layer, after the bf16
 * rounding of the quantisation contract (R15) when mlp_bf16 -- test support for the R15 pin. */
static double mlp_forward(const oracle_cfg* cfg, const float* W, const float* b, const float* z, const double* p,
                          double* acts) {
    const int L = cfg->latent_dim, H = cfg->hidden;
    double* a = (double*)malloc(sizeof(double) * (size_t)H);
    double* an = (double*)malloc(sizeof(double) * (size_t)H);
    const float* Wl = W;
    const float* bl = b;
    const int npe = 3 + 6 * cfg->pe_bands;
    double feat[3 + 6 * 16];
    oracle_pe(cfg->pe_bands, p, feat);
    const int in1 = npe + L;
    for (int i = 0; i < H; ++i) {
        double acc = 0.0;
        for (int j = 0; j < npe; ++j) acc += (double)Wl[(size_t)i * in1 + j] * feat[j];
        for (int j = 0; j < L; ++j) acc += (double)Wl[(size_t)i * in1 + npe + j] * (double)z[j];
        acc += (double)bl[i];
        double v = act_fn(cfg->activation, acc);
        a[i] = cfg->mlp_bf16 ? bf16_round(v) : v;
    }
    if (acts) memcpy(acts, a, sizeof(double) * (size_t)H);
    Wl += (size_t)H * in1;
    bl += H;
    for (int l = 1; l < cfg->n_hidden; ++l) {
        for (int i = 0; i < H; ++i) {
            double acc = 0.0;
            for (int j = 0; j < H; ++j) {
                double w = (double)Wl[(size_t)i * H + j];
                if (cfg->mlp_bf16) w = bf16_round(w);
                acc += w * a[j];
            }
            acc += (double)bl[i];
            double v = act_fn(cfg->activation, acc);
            an[i] = cfg->mlp_bf16 ? bf16_round(v) : v;
        }
        memcpy(a, an, sizeof(double) * (size_t)H);
        if (acts) memcpy(acts + (size_t)l * H, a, sizeof(double) * (size_t)H);
        Wl += (size_t)H * H;
        bl += H;
    }
    double s = 0.0;
    for (int j = 0; j < H; ++j) {
        double w = (double)Wl[j];
        if (cfg->mlp_bf16) w = bf16_round(w);
        s += w * a[j];
    }
    s += (double)bl[0];
    free(a);
    free(an);
    return s;
}

double oracle_mlp(const oracle_cfg* cfg, const float* W, const float* b, const float* z, const double* p) {
    return mlp_forward(cfg, W, b, z, p, NULL);
}

/* The same forward, also returning every hidden layer's activations acts [n_hidden][H] (test support). */
double oracle_mlp_trace(const oracle_cfg* cfg, const float* W, const float* b, const float* z, const double* p,
                        double* acts) {
    return mlp_forward(cfg, W, b, z, p, acts);
}

/* Eq. 1-2: r(p) = max(|y|,|z|); s_guide = c + |x| tan(alpha) - r(p). */
double oracle_sdf_analytic(double c, double tana, const double* p) {
    double r = fabs(p[1]) > fabs(p[2]) ? fabs(p[1]) : fabs(p[2]);
    return c + fabs(p[0]) * tana - r;
}

static double sdf_eval(const oracle_cfg* cfg, const float* W, const float* b, const float* z, const double* p) {
    if (cfg->sdf_mode == 1) return oracle_sdf_analytic(cfg->gate_c, cfg->gate_tana, p);
    return oracle_mlp(cfg, W, b, z, p);
}

/* MLP on externally given query-frame rows [n][4] (x,y,z,_) -> s[n] (test support). */
void oracle_sdf_rows(const oracle_cfg* cfg, const float* W, const float* b, const float* z,
                     const float* rows, int64_t n, double* out) {
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t i = 0; i < n; ++i) {
        double p[3] = {rows[i * 4 + 0], rows[i * 4 + 1], rows[i * 4 + 2]};
        out[i] = sdf_eval(cfg, W, b, z, p);
    }
}

/* ------------------------------------------------------------------ rollout + cost of one sample */
static double oracle_rollout_paper(const oracle_cfg* cfg, const float* W, const float* b, const float* z,
                                   const float* Tq, const float* x0, const float* goal, const float* U,
                                   const double* noise, int64_t nstride, double* states, double* queries,
                                   double* sdf, double* stage);
static double clampd(double v, double lo, double hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* One sample: u_t = clamp(U*_t + sigma * n_t) (clamp per R5); x_{t+1} = RK4(x_t, u_t);
 * query at x_{t+1} (R7) in the cached frame p_c = R p + t; SDF s = g_phi(z, p_c)
 * (PAPER.md:168); guidance by directional forward difference along d = R v / |v| (R12);
 * stage cost c_t = w_goal |p - g_c|^2 + w_sdf exp(min(-s/scale, emax)) + w_u |u|^2
 *                 - w_guide |v| (s(p_c + h d) - s(p_c)) / h       (Eq. 10 structure; BASELINE terms);
 * J = sum_t c_t, non-finite -> +inf.
 * noise: [T] x 4 with element stride `nstride` between time steps. Outputs may be NULL:
 * states [T+1][10], queries [T][8] (p_c, |v|, p_c + h d, 0), sdf [T][2], stage [T]. */
double oracle_rollout(const oracle_cfg* cfg, const float* W, const float* b, const float* z, const float* Tq,
                      const float* x0, const float* goal, const float* U, const double* noise, int64_t nstride,
                      double* states, double* queries, double* sdf, double* stage) {
    if (cfg->model == 1)
        return oracle_rollout_paper(cfg, W, b, z, Tq, x0, goal, U, noise, nstride, states, queries, sdf, stage);
    const int T = cfg->T;
    double x[10], xn[10], u[4];
    for (int i = 0; i < 10; ++i) x[i] = x0[i];
    if (states) memcpy(states, x, sizeof(x));
    double J = 0.0;
    const int guide = cfg->w_guide != 0.0;
    for (int t = 0; t < T; ++t) {
        const double* n = noise + (size_t)t * nstride;
        for (int c = 0; c < 4; ++c) u[c] = clampd((double)U[t * 4 + c] + cfg->sigma[c] * n[c], cfg->u_lo[c], cfg->u_hi[c]);
        oracle_rk4_step(x, u, cfg->dt, cfg->mass, cfg->gravity, xn);
        memcpy(x, xn, sizeof(x));
        if (states) memcpy(states + (size_t)(t + 1) * 10, x, sizeof(x));
        const double* p = x;
        const double* v = x + 3;
        double pc[3], dv[3], pc2[3];
        for (int r = 0; r < 3; ++r) {
            pc[r] = (double)Tq[r * 3 + 0] * p[0] + (double)Tq[r * 3 + 1] * p[1] + (double)Tq[r * 3 + 2] * p[2] + (double)Tq[9 + r];
            dv[r] = (double)Tq[r * 3 + 0] * v[0] + (double)Tq[r * 3 + 1] * v[1] + (double)Tq[r * 3 + 2] * v[2];
        }
        const double nv = sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
        for (int r = 0; r < 3; ++r) pc2[r] = pc[r] + cfg->fd_h * (nv >= 1e-6 ? dv[r] / nv : 0.0);
        const double s0 = sdf_eval(cfg, W, b, z, pc);
        const double s1 = guide ? sdf_eval(cfg, W, b, z, pc2) : s0;
        double dg = 0.0;
        for (int r = 0; r < 3; ++r) dg += (p[r] - (double)goal[r]) * (p[r] - (double)goal[r]);
        double un = u[0] * u[0] + u[1] * u[1] + u[2] * u[2] + u[3] * u[3];
        double ex = -s0 / cfg->sdf_scale;
        if (ex > cfg->sdf_exp_max) ex = cfg->sdf_exp_max;
        double ct = cfg->w_goal * dg + cfg->w_sdf * exp(ex) + cfg->w_u * un;
        if (guide) ct -= cfg->w_guide * nv * (s1 - s0) / cfg->fd_h;
        if (queries) {
            double* q = queries + (size_t)t * 8;
            q[0] = pc[0]; q[1] = pc[1]; q[2] = pc[2]; q[3] = nv;
            q[4] = pc2[0]; q[5] = pc2[1]; q[6] = pc2[2]; q[7] = 0.0;
        }
        if (sdf) { sdf[t * 2] = s0; sdf[t * 2 + 1] = s1; }
        if (stage) stage[t] = ct;
        J += ct;
    }
    if (!isfinite(J)) J = INFINITY;
    return J;
}

/* One sample of the paper's model (reading P5-P6): u_k = clamp(U*_k + sigma n_k, +-Tdot_max);
 * for k = 0..T-1 (the sums of Eqs. 6-9 run over k = 0..K-1 of the current trajectory):
 *   query the state x_k: p_c = R p_k + t; s_k = g_phi(z, p_c)
 *   psi_k = yaw of q_k = atan2(2(qw qz + qx qy), 1 - 2(qy^2 + qz^2)); psi_gate,k = atan2(g_y - p_y, g_x - p_x)
 *   x_{k+1} = step(x_k, u_k)
 *   c_k = Q_gate (|p_{k+1} - g|^2 - |p_k - g|^2) + Q_vis (1 - cos(psi_k - psi_gate,k)) + Q_sdf max(0, d_safe - s_k)
 * J = sum_k c_k (non-finite -> +inf). goal = p_wp = the gate centre. Outputs as oracle_rollout, states
 * [T+1][17]; queries [T][8] = (p_c, |v_k|, 0, 0, 0, 0); sdf [T][2] = (s_k, s_k). */
static double oracle_rollout_paper(const oracle_cfg* cfg, const float* W, const float* b, const float* z,
                                   const float* Tq, const float* x0, const float* goal, const float* U,
                                   const double* noise, int64_t nstride, double* states, double* queries,
                                   double* sdf, double* stage) {
    const int T = cfg->T;
    double x[17], xn[17], u[4];
    for (int i = 0; i < 17; ++i) x[i] = x0[i];
    if (states) memcpy(states, x, sizeof(x));
    double J = 0.0;
    for (int t = 0; t < T; ++t) {
        const double* n = noise + (size_t)t * nstride;
        for (int c = 0; c < 4; ++c) u[c] = clampd((double)U[t * 4 + c] + cfg->sigma[c] * n[c], cfg->u_lo[c], cfg->u_hi[c]);
        const double* p = x;
        const double* v = x + 3;
        double pc[3];
        for (int r = 0; r < 3; ++r)
            pc[r] = (double)Tq[r * 3 + 0] * p[0] + (double)Tq[r * 3 + 1] * p[1] + (double)Tq[r * 3 + 2] * p[2] + (double)Tq[9 + r];
        const double nv = sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
        const double s0 = sdf_eval(cfg, W, b, z, pc);
        const double qw = x[6], qx = x[7], qy = x[8], qz = x[9];
        const double psi = atan2(2.0 * (qw * qz + qx * qy), 1.0 - 2.0 * (qy * qy + qz * qz));
        const double psig = atan2((double)goal[1] - p[1], (double)goal[0] - p[0]);
        double d0 = 0.0;
        for (int r = 0; r < 3; ++r) d0 += (p[r] - (double)goal[r]) * (p[r] - (double)goal[r]);
        oracle_rotor_step(cfg, x, u, xn);
        double d1 = 0.0;
        for (int r = 0; r < 3; ++r) d1 += (xn[r] - (double)goal[r]) * (xn[r] - (double)goal[r]);
        const double hinge = cfg->d_safe - s0 > 0.0 ? cfg->d_safe - s0 : 0.0;
        const double ct = cfg->q_gate * (d1 - d0) + cfg->q_vis * (1.0 - cos(psi - psig)) + cfg->q_sdf * hinge;
        memcpy(x, xn, sizeof(x));
        if (states) memcpy(states + (size_t)(t + 1) * 17, x, sizeof(x));
        if (queries) {
            double* q = queries + (size_t)t * 8;
            q[0] = pc[0]; q[1] = pc[1]; q[2] = pc[2]; q[3] = nv;
            q[4] = q[5] = q[6] = q[7] = 0.0;
        }
        if (sdf) { sdf[t * 2] = s0; sdf[t * 2 + 1] = s0; }
        if (stage) stage[t] = ct;
        J += ct;
    }
    if (!isfinite(J)) J = INFINITY;
    return J;
}

/* ------------------------------------------------------------------ softmin update (Eq. 5) */
/* For one controller: J[K]; U[T][4]; noise with element stride nstride between t and 4 between k.
 * Jmin = min J; w_k = exp(-(J_k - Jmin)/lambda); S = sum w; V_t = sum_k w_k (u_{k,t} - U_t);
 * U_new = U + V/S. All J infinite -> U_new = U, flag 1 (SPEC.md:341 reading). */
int oracle_softmin(const oracle_cfg* cfg, int32_t K, const double* J, const float* U, const double* noise,
                   int64_t nstride, double* Jmin_o, double* S_o, double* V, double* U_new, double* ess_o) {
    const int T = cfg->T;
    double Jmin = INFINITY;
    for (int k = 0; k < K; ++k) if (J[k] < Jmin) Jmin = J[k];
    for (int i = 0; i < T * 4; ++i) V[i] = 0.0;
    if (!(Jmin < INFINITY)) {
        for (int i = 0; i < T * 4; ++i) U_new[i] = U[i];
        if (Jmin_o) *Jmin_o = INFINITY;
        if (S_o) *S_o = 0.0;
        if (ess_o) *ess_o = 0.0;
        return 1;
    }
    double S = 0.0, S2 = 0.0;
    for (int k = 0; k < K; ++k) {
        double w = (J[k] < INFINITY) ? exp(-(J[k] - Jmin) / cfg->lambda) : 0.0;
        S += w;
        S2 += w * w;
        if (w == 0.0) continue;
        for (int t = 0; t < T; ++t)
            for (int c = 0; c < 4; ++c) {
                double uk = clampd((double)U[t * 4 + c] + cfg->sigma[c] * noise[(size_t)t * nstride + (size_t)k * 4 + c],
                                   cfg->u_lo[c], cfg->u_hi[c]);
                V[t * 4 + c] += w * (uk - (double)U[t * 4 + c]);
            }
    }
    for (int i = 0; i < T * 4; ++i) U_new[i] = (double)U[i] + V[i] / S;
    if (Jmin_o) *Jmin_o = Jmin;
    if (S_o) *S_o = S;
    if (ess_o) *ess_o = S * S / S2;
    return 0;
}

/* Shard record (configs[3]): m_r = min J over the shard; S_r, V_r relative to m_r. */
int oracle_shard_record(const oracle_cfg* cfg, int32_t Kr, const double* J, const float* U, const double* noise,
                        int64_t nstride, double* rec /* [2 + T*4]: m, S, V */) {
    double U_new_dummy[4096];
    double* Un = cfg->T * 4 <= 4096 ? U_new_dummy : (double*)malloc(sizeof(double) * (size_t)cfg->T * 4);
    int flag = oracle_softmin(cfg, Kr, J, U, noise, nstride, &rec[0], &rec[1], rec + 2, Un, NULL);
    if (Un != U_new_dummy) free(Un);
    return flag;
}

/* Combine R shard records: m = min m_r; S = sum S_r e^{-(m_r-m)/lambda}; V likewise; U_new = U + V/S. */
int oracle_combine(const oracle_cfg* cfg, int32_t R, const double* recs, const float* U, double* U_new) {
    const int T = cfg->T, W = 2 + T * 4;
    double m = INFINITY;
    for (int r = 0; r < R; ++r) if (recs[r * W] < m) m = recs[r * W];
    if (!(m < INFINITY)) {
        for (int i = 0; i < T * 4; ++i) U_new[i] = U[i];
        return 1;
    }
    double S = 0.0;
    double* V = (double*)calloc((size_t)T * 4, sizeof(double));
    for (int r = 0; r < R; ++r) {
        const double* rec = recs + (size_t)r * W;
        if (!(rec[0] < INFINITY)) continue;
        double f = exp(-(rec[0] - m) / cfg->lambda);
        S += rec[1] * f;
        for (int i = 0; i < T * 4; ++i) V[i] += rec[2 + i] * f;
    }
    for (int i = 0; i < T * 4; ++i) U_new[i] = (double)U[i] + V[i] / S;
    free(V);
    return 0;
}

/* ------------------------------------------------------------------ full iteration */
/* One MPPI iteration for every controller b (already-shifted nominal U). noise: [T][n_ctrl*K][4].
 * Per-controller inputs: z [n][L], Tq [n][12], x0 [n][10] (model 1: [n][17]), goal [n][3], U [n][T][4].
 * Optional outputs (NULL to skip): queries [n][K][T][8], sdf [n][K][T][2], stage [n][K][T],
 * J [n][K], Jmin/S/ess [n], V/U_new [n][T][4], flags [n]. */
void oracle_step(const oracle_cfg* cfg, const float* W, const float* b, const float* z, const float* Tq,
                 const float* x0, const float* goal, const float* U, const double* noise,
                 double* queries, double* sdf, double* stage, double* J, double* Jmin, double* S, double* ess,
                 double* V, double* U_new, int32_t* flags) {
    const int n = cfg->n_ctrl, K = cfg->K, T = cfg->T, L = cfg->latent_dim;
    const int sd = cfg->model == 1 ? 17 : 10;   /* state dimension */
    const int64_t nstride = (int64_t)n * K * 4;
    double* Jl = J ? J : (double*)malloc(sizeof(double) * (size_t)n * K);
#pragma omp parallel for schedule(dynamic, 4) collapse(2)
    for (int bb = 0; bb < n; ++bb)
        for (int k = 0; k < K; ++k) {
            size_t sk = (size_t)bb * K + k;
            Jl[sk] = oracle_rollout(cfg, W, b, z + (size_t)bb * L, Tq + (size_t)bb * 12, x0 + (size_t)bb * sd,
                                    goal + (size_t)bb * 3, U + (size_t)bb * T * 4, noise + sk * 4, nstride, NULL,
                                    queries ? queries + sk * T * 8 : NULL, sdf ? sdf + sk * T * 2 : NULL,
                                    stage ? stage + sk * T : NULL);
        }
    double* Vt = (double*)malloc(sizeof(double) * (size_t)T * 4);
    double* Ut = (double*)malloc(sizeof(double) * (size_t)T * 4);
    for (int bb = 0; bb < n; ++bb) {
        double jm, ss, es;
        int f = oracle_softmin(cfg, K, Jl + (size_t)bb * K, U + (size_t)bb * T * 4, noise + (size_t)bb * K * 4, nstride,
                               &jm, &ss, Vt, Ut, &es);
        if (Jmin) Jmin[bb] = jm;
        if (S) S[bb] = ss;
        if (ess) ess[bb] = es;
        if (V) memcpy(V + (size_t)bb * T * 4, Vt, sizeof(double) * (size_t)T * 4);
        if (U_new) memcpy(U_new + (size_t)bb * T * 4, Ut, sizeof(double) * (size_t)T * 4);
        if (flags) flags[bb] = f;
    }
    free(Vt);
    free(Ut);
    if (!J) free(Jl);
}

/* Warm-start shift ("the sequence initializes the next control cycle"):
 * U_t <- U_{t+1}, last entry repeated. In place on [n][T][4]. */
void oracle_shift(int32_t n, int32_t T, float* U) {
    for (int bb = 0; bb < n; ++bb) {
        float* u = U + (size_t)bb * T * 4;
        for (int t = 0; t + 1 < T; ++t)
            for (int c = 0; c < 4; ++c) u[t * 4 + c] = u[(t + 1) * 4 + c];
    }
}
