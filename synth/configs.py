"""BASELINE.json configs[0..4] as plain data, plus reduced parity variants.

Values come from /root/repo/BASELINE.json `configs` (cited per field below) and the readings of
SURVEY.md §8(c) (R-numbers). Nothing here computes anything.
"""
from __future__ import annotations

import dataclasses
from dataclasses import dataclass, field

ACT_SOFTPLUS, ACT_RELU, ACT_SILU = 0, 1, 2
MLP_FP32, MLP_BF16 = 0, 1


@dataclass
class MPPIConfig:
    name: str
    n_ctrl: int = 1              # controllers (drones) on one device (configs[4]: 1024)
    K: int = 256                 # samples per controller (paper's M)
    T: int = 20                  # horizon (paper's K)
    dt: float = 0.02             # configs[0..2] dt=0.02 s; configs[3] dt=0.01 s
    lam: float = 1.0             # temperature: configs[0] 1.0, configs[1..] 0.5
    mass: float = 1.0            # configs[0] m = 1 kg
    gravity: float = 9.81        # R3
    rate_max: float = 6.0        # configs[0] body rates in +-6 rad/s
    sigma: tuple = (2.0, 1.0, 1.0, 1.0)   # configs[0] sigma = (2 N, 1 rad/s x3)
    w_goal: float = 1.0          # configs[0] 1.0*||p - g_c||^2
    w_sdf: float = 50.0          # configs[0] 50*exp(-sdf/0.1)
    sdf_scale: float = 0.1
    sdf_exp_max: float = 80.0    # R9 overflow guard
    w_u: float = 0.01            # configs[0] 0.01*||u||^2
    w_guide: float = 0.0         # configs[1] -0.5*grad(sdf).v  (0 in configs[0])
    fd_h: float = 0.1            # R12 directional forward difference step (m)
    latent_dim: int = 32         # configs[0] 32, [1] 64, [2..3] 128, [4] 64
    hidden: int = 64             # hidden width
    n_hidden: int = 2            # hidden layers incl. the first (latent-conditioned) layer
    activation: int = ACT_SOFTPLUS
    mlp_dtype: int = MLP_FP32
    seed: int = 0
    steps: int = 1               # closed-loop steps the config asks for (configs[1..]: 100)
    latent_every: int = 0        # redraw latent every N steps (configs[1]: 5)
    per_drone_gates: bool = False  # configs[4]
    # the paper's own model (model 1; SURVEY.md §8f F1 + F2; readings P1-P7)
    model: int = 0               # 0: BASELINE CTBR + configs terms; 1: per-rotor thrust-rate model + Eq. 6-10
    arm: float = 0.15            # P3: rotor arm (m) -- the paper gives no airframe
    kappa: float = 0.016         # P3: yaw moment per unit thrust (m)
    inertia: tuple = (0.0025, 0.0025, 0.0045)   # P3: diag(J) (kg m^2)
    thrust_max: float = 10.0     # Table I "T_s [N] [0, 10]"
    tdot_max: float = 10.0       # Table I "Tdot_s [-10, 10]"
    q_gate: float = 1.0          # P6: Eq. 10 weights (the paper gives none)
    q_vis: float = 2.0
    q_sdf: float = 10.0
    d_safe: float = 1.0          # Table I "d_safe 1.0"
    # SDF provider: 0 the neural g_phi, 1 the analytic Gate-SDF of Eq. 2
    sdf_provider: int = 0
    gate_c: float = 0.5          # inner half-width: inner diameter 1.0 m
    gate_tana: float = 0.36397023426620234   # tan(20 deg): alpha unstated; SURVEY/SPEC.md:139-141 golden values
    # positional encoding of the query position (reading E1): 0 = none
    pe_bands: int = 0

    @property
    def u_lo(self):
        if self.model == 1:
            return (-self.tdot_max,) * 4
        return (0.0, -self.rate_max, -self.rate_max, -self.rate_max)

    @property
    def u_hi(self):
        if self.model == 1:
            return (self.tdot_max,) * 4
        return (4.0 * self.mass * self.gravity, self.rate_max, self.rate_max, self.rate_max)

    @property
    def state_dim(self) -> int:
        return 17 if self.model == 1 else 10

    @property
    def fd(self) -> bool:
        return self.w_guide != 0.0

    @property
    def layer_dims(self):
        """[(in, out)] for every dense layer, nn.Linear order ([out][in] weights). Layer 1 reads
        [PE(p) (3 + 6 pe_bands) | z (L)]."""
        dims = [(3 + 6 * self.pe_bands + self.latent_dim, self.hidden)]
        dims += [(self.hidden, self.hidden)] * (self.n_hidden - 1)
        dims += [(self.hidden, 1)]
        return dims

    def replace(self, **kw) -> "MPPIConfig":
        return dataclasses.replace(self, **kw)


CONFIGS = {
    # configs[0]: tiny fp32 PR1 reference.
    "c0": MPPIConfig(name="c0", K=256, T=20, dt=0.02, lam=1.0, latent_dim=32, hidden=64,
                     n_hidden=2, activation=ACT_SOFTPLUS, mlp_dtype=MLP_FP32, w_guide=0.0),
    # configs[1]: paper-scale single controller, 67->128->128->128->1 ReLU bf16, guidance.
    "c1": MPPIConfig(name="c1", K=4096, T=50, dt=0.02, lam=0.5, latent_dim=64, hidden=128,
                     n_hidden=3, activation=ACT_RELU, mlp_dtype=MLP_BF16, w_guide=0.5,
                     steps=100, latent_every=5),
    # configs[2]: large-sample single GPU, 131->256x4->1 SiLU bf16.
    "c2": MPPIConfig(name="c2", K=16384, T=50, dt=0.02, lam=0.5, latent_dim=128, hidden=256,
                     n_hidden=4, activation=ACT_SILU, mlp_dtype=MLP_BF16, w_guide=0.5,
                     steps=100, latent_every=5),
    # configs[3]: sharded large-K, K=131072 (global), T=100, dt=0.01, configs[2] MLP.
    "c3": MPPIConfig(name="c3", K=131072, T=100, dt=0.01, lam=0.5, latent_dim=128, hidden=256,
                     n_hidden=4, activation=ACT_SILU, mlp_dtype=MLP_BF16, w_guide=0.5,
                     steps=100, latent_every=5),
    # configs[4]: 1024 independent drones, K=1024, T=50, configs[1] MLP shared.
    "c4": MPPIConfig(name="c4", n_ctrl=1024, K=1024, T=50, dt=0.02, lam=0.5, latent_dim=64,
                     hidden=128, n_hidden=3, activation=ACT_RELU, mlp_dtype=MLP_BF16,
                     w_guide=0.5, steps=100, per_drone_gates=True),
}

# The paper's configuration (SURVEY.md §8f F1 + F2): Table I M=8192, K=20, dt=0.03,
# lambda in [0.01, 0.1], Tdot in [-10, 10], T in [0, 10] N, w in [-10, 10] rad/s, d_safe = 1; latent
# z in R^128; the per-rotor thrust-rate model and Eq. 6-10 costs; MLP size unstated ->
# the configs[2] MLP; no guidance term (Eq. 10 has none).
CONFIGS["c5"] = MPPIConfig(name="c5", model=1, K=8192, T=20, dt=0.03, lam=0.05, rate_max=10.0,
                           sigma=(5.0, 5.0, 5.0, 5.0), latent_dim=128, hidden=256, n_hidden=4,
                           activation=ACT_SILU, mlp_dtype=MLP_BF16, w_guide=0.0, steps=100, latent_every=5)

# Reduced parity variants: same MLP/cost/dynamics structure, sizes the oracle finishes in seconds
# while still spanning several 128-row tiles and a ragged tail.
CONFIGS["c1s"] = CONFIGS["c1"].replace(name="c1s", K=200, T=7, steps=1)
CONFIGS["c2s"] = CONFIGS["c2"].replace(name="c2s", K=136, T=5, steps=1)
CONFIGS["c3s"] = CONFIGS["c3"].replace(name="c3s", K=256, T=6, steps=1)
CONFIGS["c4s"] = CONFIGS["c4"].replace(name="c4s", n_ctrl=6, K=64, T=4, steps=1)
CONFIGS["c5s"] = CONFIGS["c5"].replace(name="c5s", K=200, T=6, steps=1)
# The analytic Gate-SDF provider on the configs[1] / configs[4] / paper-model paths
CONFIGS["c1g"] = CONFIGS["c1"].replace(name="c1g", sdf_provider=1)
CONFIGS["c1gs"] = CONFIGS["c1s"].replace(name="c1gs", sdf_provider=1)
CONFIGS["c4gs"] = CONFIGS["c4s"].replace(name="c4gs", sdf_provider=1)
CONFIGS["c5gs"] = CONFIGS["c5s"].replace(name="c5gs", sdf_provider=1)
# Positional encoding on the configs[1] MLP: 4 bands (27 position features)
CONFIGS["c1pe"] = CONFIGS["c1"].replace(name="c1pe", pe_bands=4)
CONFIGS["c1pes"] = CONFIGS["c1s"].replace(name="c1pes", pe_bands=4)
# ... and on the configs[2]/[3] MLP (H = 256)
CONFIGS["c2pe"] = CONFIGS["c2"].replace(name="c2pe", pe_bands=4)
CONFIGS["c2pes"] = CONFIGS["c2s"].replace(name="c2pes", pe_bands=4)


def get_config(name: str, **overrides) -> MPPIConfig:
    cfg = CONFIGS[name]
    return cfg.replace(**overrides) if overrides else cfg
