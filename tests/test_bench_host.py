"""Host-side pins of bench.py (no GPU): the algorithmic work it divides by, the scaling key, and the
reference arm's rank handling."""
import argparse
import os
import sys

import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402
import synth  # noqa: E402


@pytest.mark.parametrize("name,flop", [
    ("c0", 8704),      # flop / eval, latent folded
    ("c1", 66560),
    ("c2", 395264),
    ("c3", 395264),
    ("c4", 66560),
])
def test_mlp_flops_per_row_matches_survey_table(name, flop):
    assert bench.mlp_flops_per_row(synth.get_config(name)) == flop


def test_positional_encoding_widens_layer_one():
    cfg = synth.get_config("c1pe")   # 4 bands: 3 + 24 position features
    H = cfg.hidden
    assert bench.mlp_flops_per_row(cfg) - bench.mlp_flops_per_row(synth.get_config("c1")) == 2 * 24 * H


@pytest.mark.parametrize("name,scaling", [("c3", "strong"), ("c4", "strong"), ("c2", "weak"), ("c1", "weak")])
def test_scaling_key_follows_the_partition(name, scaling):
    assert bench.scaling_of(synth.get_config(name)) == scaling


def test_reference_arm_only_runs_on_rank_zero(capsys):
    args = argparse.Namespace(config="auto", steps=1, warmup=0)
    assert bench.run_reference(args, world=2, rank=1) is None
    assert capsys.readouterr().out == ""


def test_default_workload_is_configs3():
    cfg = bench.pick_config("auto", 1)
    assert (cfg.name, cfg.K, cfg.T, cfg.hidden) == ("c3", 131072, 100, 256)
    assert "c3" in bench.workload_name(cfg, 1) and "sharded" in bench.workload_name(cfg, 8)
