"""Seeded synthetic inputs shared by the oracle tests, the CUDA parity tests and bench.py.

This module holds NO arithmetic of the MPPI method (no dynamics, no MLP, no cost, no softmin).
It only draws the inputs the method consumes: configs (BASELINE.json configs[0..4] as data),
MLP weights, latent codes, gate poses / query-frame transforms, initial states, nominal
controls and standard-normal noise for the external-noise parity mode.

Input recipe:
  * weights: Kaiming-uniform U(+-sqrt(6/fan_in)) (BASELINE configs[0] "Kaiming-uniform init from
    a seed"); biases U(+-1/sqrt(fan_in)) (the nn.Linear default; BASELINE is silent on biases).
  * latent z ~ N(0, 1) (BASELINE configs[0..4]).
  * gate centre g_c ~ U([2,6] x [-2,2] x [-1,1]) m (reading R17 of SURVEY.md §8c).
  * per-drone gate pose (configs[4]): yaw ~ U(-pi, pi), pitch ~ U(-30deg, 30deg) (R22).
  * x0 = hover at the origin, U* = hover thrust m*g with zero rates (R18).
  * noise: i.i.d. standard normals, time-major [T][n_ctrl*K][4] (parity mode uploads these).
"""
from .configs import MPPIConfig, CONFIGS, get_config  # noqa: F401
from .inputs import (  # noqa: F401
    rng_for, make_weights, make_latents, make_goals, make_query_transforms, make_gate_poses,
    make_x0, make_nominal, make_noise, constructed_gate_net, camera_transform, make_query_rows,
)
