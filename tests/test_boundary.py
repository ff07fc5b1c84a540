"""C-ABI boundary checks that need no GPU (-m "not gpu"): the library loads, exports every symbol
include/mppi.h declares, and validates configs without touching the device."""
import ctypes as C
import os
import re

import pytest

import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2603_07199_b200 import build
    build.build()
    from paper_2603_07199_b200 import _lib
    return _lib.load()


def _declared():
    txt = open(os.path.join(ROOT, "include", "mppi.h")).read()
    return sorted(set(re.findall(r"\b(mppi_[a-z_0-9]+)\s*\(", txt)))


def test_header_matches_binding_exports():
    from paper_2603_07199_b200 import _lib
    assert _declared() == sorted(_lib.EXPORTS)


def test_library_exports_every_declared_symbol(lib):
    for name in _declared():
        assert hasattr(lib, name), name


def test_workspace_bytes_and_validation(lib):
    from paper_2603_07199_b200._lib import make_config
    for name in ("c0", "c1", "c2", "c3", "c4", "c1s", "c2s", "c4s"):
        cfg = synth.get_config(name)
        c = make_config(cfg)
        nb = lib.mppi_workspace_bytes(C.byref(c))
        assert nb > 0, name
        # noise + rows dominate: at least 16 B noise + 16 B per query row per state
        states = cfg.n_ctrl * cfg.K * cfg.T
        assert nb >= states * (16 + 16 * (2 if cfg.fd else 1))
    c2 = synth.get_config("c2")
    assert lib.mppi_workspace_bytes(C.byref(make_config(c2))) < 8 * 2 ** 30   # fits easily in 180 GB
    bad = [
        synth.get_config("c0").replace(K=0),
        synth.get_config("c0").replace(T=0),
        synth.get_config("c0").replace(lam=0.0),
        synth.get_config("c0").replace(hidden=96),                        # fp32 SIMT: 32/64 only
        synth.get_config("c2").replace(hidden=192),                       # tcgen05: 128/256 only
        synth.get_config("c0").replace(dt=-1.0),
    ]
    for cfg in bad:
        assert lib.mppi_workspace_bytes(C.byref(make_config(cfg))) == 0
        ctx = C.c_void_p()
        st = lib.mppi_create(C.byref(make_config(cfg)), None, 0, C.byref(ctx))
        assert st in (-1, -8) and not ctx.value
        assert lib.mppi_last_error()
    c = make_config(synth.get_config("c0"))
    c.abi_version = 99
    assert lib.mppi_workspace_bytes(C.byref(c)) == 0
    c = make_config(synth.get_config("c0"), world_size=2, rank=2)
    assert lib.mppi_workspace_bytes(C.byref(c)) == 0


def test_null_context_is_rejected(lib):
    assert lib.mppi_step(None, None, None, 0) == -1
    assert lib.mppi_get_controls(None, None, None) == -1
    assert lib.mppi_destroy(None) == 0
    assert lib.mppi_record_size(None) == 0


def test_product_package_does_not_import_oracle():
    """The product path must not route through the CPU oracle (no CPU fallback)."""
    pkg = os.path.join(ROOT, "paper_2603_07199_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"(#|//).*", "", src).lower().replace("oracle/", ""), f


def test_largest_problem_boundary(lib):
    """The index space of a context: query rows n_ctrl K T (2 with guidance) up to 2^30 (32-bit tile / row
    arithmetic in the kernels) -- the largest accepted size is sized, one step above it is rejected."""
    from paper_2603_07199_b200._lib import make_config
    top = synth.get_config("c1").replace(K=1 << 22, T=127)          # 1.065e9 rows
    nb = lib.mppi_workspace_bytes(C.byref(make_config(top)))
    assert nb > 0 and nb < 64 * 2 ** 30                              # ~33 GB of the 180 GB
    assert lib.mppi_workspace_bytes(C.byref(make_config(top.replace(T=128)))) == 0   # 2^30 + ... rows
    assert lib.mppi_workspace_bytes(C.byref(make_config(top.replace(T=128, w_guide=0.0)))) > 0
