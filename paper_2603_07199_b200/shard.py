"""Host-side partitioning of the MPPI iteration over ranks (one process per GPU).

configs[3]: the K samples of every controller are split evenly; rank r owns global samples
[r K/R, (r+1) K/R) and keys its noise by global index, so the union of the shards is the unsharded
iteration. The one exchange is the all-gather of the per-controller softmin record (m, S, S2, SJ, N, 0, 0, 0, V);
every rank combines the records in rank order (k_combine / mppi_step_finish), so all ranks agree.
configs[4]: the controllers are split evenly and nothing is exchanged (replicas of the data path).
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class ShardPlan:
    mode: str            # "samples" (configs[3]), "controllers" (configs[4]) or "replica"
    world: int
    rank: int
    K_local: int
    K_global: int
    k_offset: int
    n_ctrl_local: int
    ctrl_offset: int

    @property
    def sharded(self) -> bool:
        return self.mode == "samples" and self.world > 1


def plan(cfg, world: int, rank: int, mode: str | None = None) -> ShardPlan:
    """Partition cfg over `world` ranks. mode defaults to samples for configs[3] ("c3"), controllers
    for configs[4] ("c4") and independent replicas otherwise."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    if mode is None:
        mode = {"c3": "samples", "c4": "controllers"}.get(getattr(cfg, "name", "")[:2], "replica")
    if world == 1 or mode == "replica":
        return ShardPlan("replica", world, rank, cfg.K, cfg.K, 0, cfg.n_ctrl, 0)
    if mode == "samples":
        if cfg.K % world:
            raise ValueError(f"K={cfg.K} not divisible by world={world}")
        Kl = cfg.K // world
        return ShardPlan("samples", world, rank, Kl, cfg.K, rank * Kl, cfg.n_ctrl, 0)
    if mode == "controllers":
        if cfg.n_ctrl % world:
            raise ValueError(f"n_ctrl={cfg.n_ctrl} not divisible by world={world}")
        nl = cfg.n_ctrl // world
        return ShardPlan("controllers", world, rank, cfg.K, cfg.K, 0, nl, rank * nl)
    raise ValueError(f"unknown mode {mode}")
