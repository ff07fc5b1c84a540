"""N>1 host logic on CPU (-m "not gpu"): world_size-2 gloo process groups run the sharding plan of
paper_2603_07199_b200.shard with the oracle as the per-rank compute, exchange the softmin records with
all_gather (the collective the NCCL path uses), combine in rank order, and must reproduce the unsharded
oracle iteration (configs[3] identity) and the controller partition (configs[4])."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth
from paper_2603_07199_b200 import shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank_samples(rank, world, port, out_q):
    import oracle
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = synth.get_config("c3s").replace(K=64, T=4, n_ctrl=2)
    plan = shard.plan(cfg, world, rank)
    Ws, bs = synth.make_weights(cfg)
    z, Tq, x0, goal, U = (synth.make_latents(cfg), synth.make_query_transforms(cfg), synth.make_x0(cfg),
                          synth.make_goals(cfg), synth.make_nominal(cfg))
    lcfg = cfg.replace(K=plan.K_local)
    oc = oracle.make_cfg(lcfg)
    recs = []
    for b in range(cfg.n_ctrl):
        # global noise counter g = b*K_global + k_offset + k (what the device generator uses)
        nz = oracle.noise(cfg.seed, 0, b * plan.K_global + plan.k_offset, plan.K_local, cfg.T)
        J = [oracle.rollout(oc, Ws, bs, z[b], Tq[b], x0[b], goal[b], U[b], nz[:, k])["J"] for k in range(plan.K_local)]
        recs.append(oracle.shard_record(oc, np.array(J), U[b], nz))
    mine = torch.tensor(np.stack(recs))
    gathered = [torch.zeros_like(mine) for _ in range(world)]
    dist.all_gather(gathered, mine)
    U_new = np.stack([oracle.combine(oc, np.stack([g[b].numpy() for g in gathered]), U[b])[0]
                      for b in range(cfg.n_ctrl)])
    out_q.put((rank, U_new))
    dist.destroy_process_group()


def _rank_controllers(rank, world, port, out_q):
    import oracle
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = synth.get_config("c4s").replace(n_ctrl=4, K=16, T=3)
    plan = shard.plan(cfg, world, rank)
    sl = slice(plan.ctrl_offset, plan.ctrl_offset + plan.n_ctrl_local)
    Ws, bs = synth.make_weights(cfg)
    full = dict(z=synth.make_latents(cfg), Tq=synth.make_query_transforms(cfg), x0=synth.make_x0(cfg),
                goal=synth.make_goals(cfg), U=synth.make_nominal(cfg))
    noise = oracle.noise(cfg.seed, 0, plan.ctrl_offset * cfg.K, plan.n_ctrl_local * cfg.K, cfg.T)
    lcfg = cfg.replace(n_ctrl=plan.n_ctrl_local)
    out = oracle.step(oracle.make_cfg(lcfg), Ws, bs, full["z"][sl], full["Tq"][sl], full["x0"][sl],
                      full["goal"][sl], full["U"][sl], noise, want_queries=False)
    mine = torch.tensor(out["U_new"])
    gathered = [torch.zeros_like(mine) for _ in range(world)]
    dist.all_gather(gathered, mine)   # only to compare; the data path itself exchanges nothing
    out_q.put((rank, torch.cat(gathered).numpy()))
    dist.destroy_process_group()


def _run(fn, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=fn, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def test_plan_partitions():
    c3 = synth.get_config("c3")
    ps = [shard.plan(c3, 8, r) for r in range(8)]
    assert all(p.sharded and p.K_local == 16384 for p in ps)
    assert [p.k_offset for p in ps] == [r * 16384 for r in range(8)]
    c4 = synth.get_config("c4")
    ps = [shard.plan(c4, 8, r) for r in range(8)]
    assert all(p.mode == "controllers" and p.n_ctrl_local == 128 and not p.sharded for p in ps)
    assert shard.plan(synth.get_config("c2"), 4, 1).mode == "replica"
    with pytest.raises(ValueError):
        shard.plan(c3.replace(K=100), 3, 0)


def test_gloo_sample_sharding_matches_unsharded_oracle():
    import oracle
    res = _run(_rank_samples)
    np.testing.assert_array_equal(res[0], res[1])      # every rank combines to the same U*
    cfg = synth.get_config("c3s").replace(K=64, T=4, n_ctrl=2)
    Ws, bs = synth.make_weights(cfg)
    ref = oracle.step(oracle.make_cfg(cfg), Ws, bs, synth.make_latents(cfg), synth.make_query_transforms(cfg),
                      synth.make_x0(cfg), synth.make_goals(cfg), synth.make_nominal(cfg),
                      oracle.noise(cfg.seed, 0, 0, cfg.n_ctrl * cfg.K, cfg.T), want_queries=False)
    np.testing.assert_allclose(res[0], ref["U_new"], rtol=1e-12, atol=1e-12)


def test_gloo_controller_partition_matches_single_process():
    import oracle
    res = _run(_rank_controllers)
    cfg = synth.get_config("c4s").replace(n_ctrl=4, K=16, T=3)
    Ws, bs = synth.make_weights(cfg)
    ref = oracle.step(oracle.make_cfg(cfg), Ws, bs, synth.make_latents(cfg), synth.make_query_transforms(cfg),
                      synth.make_x0(cfg), synth.make_goals(cfg), synth.make_nominal(cfg),
                      oracle.noise(cfg.seed, 0, 0, cfg.n_ctrl * cfg.K, cfg.T), want_queries=False)
    np.testing.assert_allclose(res[0], ref["U_new"], rtol=1e-12, atol=1e-12)
