"""Host logic of the multi-GPU path, on CPU:

* LPT object sharding (parallel.py) -- balance and determinism;
* the Reptile orchestration (meta.py) run by 2 gloo ranks with a CPU engine
  built on the oracle: the all-reduced update equals the single-process one
  and equals reptile_update(theta, mean_i theta_i, beta) (meta.cpp:83-92,
  SPEC.md:323 linearity);
* the meta-step task schedule (round-robin over per-epoch shuffles,
  meta.cpp:104-110), equal to the compiled reference's order.
"""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2503_01582_b200 import FieldArch, TrainConfig, scenes
from paper_2503_01582_b200.meta import Engine, MetaConfig, meta_train, task_schedule
from paper_2503_01582_b200.parallel import imbalance, shard_lpt, step_cost


def test_lpt_sharding_balanced_and_complete():
    rng = np.random.default_rng(0)
    archs = [FieldArch(hash_levels=int(rng.choice([8, 12, 16])), log2_table_size=int(rng.integers(14, 20)),
                       hidden_width=int(rng.choice([32, 64])), hidden_layers=int(rng.choice([1, 2])))
             for _ in range(32)]
    costs = [step_cost(a, 2048, 96) for a in archs]
    for world in (1, 2, 4, 8):
        sh = shard_lpt(costs, world)
        assert sorted(i for s in sh for i in s) == list(range(32))
        assert imbalance(costs, sh) < 1.25
        assert sh == shard_lpt(costs, world)  # deterministic


def test_task_schedule_round_robin_epochs():
    s = task_schedule(5, 7, 2, seed=3)
    flat = [t for b in s for t in b]
    assert sorted(flat[:5]) == list(range(5)) and sorted(flat[5:10]) == list(range(5))
    assert task_schedule(5, 7, 2, seed=3) == s


@pytest.mark.ref
@pytest.mark.parametrize("n_tasks", [1, 2, 7, 512, 513, 70001])
def test_task_schedule_equals_reference_meta_train_order(ref, n_tasks):
    """meta_train's schedule (meta.cpp:101-112: order reshuffled in place each epoch by
    std::shuffle over mt19937(derive_seed(seed, 0xE9C6 + epoch))) is index work: the
    restated libstdc++ shuffle reproduces the compiled reference's order exactly, for 3 epochs,
    on both of libstdc++'s paths (paired draws while n^2 < 2^32, single draws beyond)."""
    for seed in (0, 9, 2**40 + 5):
        want = ref.meta_task_order(n_tasks, seed, 3)
        steps = 3 * n_tasks if n_tasks < 1000 else n_tasks + 5
        got = [b[0] for b in task_schedule(n_tasks, steps, 1, seed)]
        flat = want.reshape(-1)[:steps]
        assert got == flat.tolist()


class OracleEngine(Engine):
    """CPU engine for the orchestration tests (test infrastructure)."""

    def __init__(self, orc, arch, theta, tasks, cfg):
        self.orc, self.arch, self.theta, self.tasks, self.cfg = orc, arch, theta.copy(), tasks, cfg
        self.adapted = {}

    def adapt(self, task, q, seed):
        sc = self.tasks[task]
        ob = self.orc.object_create(self.arch, self.theta, None, 8, seed, self.cfg.to_c(), sc.box_min, sc.box_max)
        ob.set_frames(sc.cams, sc.rgb, sc.depth, sc.mask, 1, sc.obj_pose)
        ob.train_step(q)
        self.adapted[task] = ob.params()

    def delta_sum(self, tasks):
        acc = np.zeros_like(self.theta)
        for t in tasks:
            acc += self.adapted[t] - self.theta
        return torch.from_numpy(acc)

    def apply(self, buf, n, beta):
        d = buf.numpy().astype(np.float32)
        keep = np.float32(1) - np.float32(beta)
        adapted = self.theta + d * np.float32(1.0 / n)
        self.theta = (keep * self.theta + np.float32(beta) * adapted).astype(np.float32)

    def update_exact(self, task, beta):
        self.theta = self.orc.reptile_update(self.theta, self.adapted[task], beta)


ARCH = FieldArch(hash_levels=3, features_per_level=2, log2_table_size=8, base_resolution=4, per_level_scale=1.5,
                 hidden_width=8, hidden_layers=1)
CFG = TrainConfig(rays_per_iter=16, samples_per_ray=8, prior_sampling=0, grid_refresh_every=0)


def make_tasks():
    return [scenes.box_union_scene(n_views=3, res=24, seed=100 + i) for i in range(4)]


def _rank_main(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.pyoracle import Oracle

    orc = Oracle()
    theta = (np.random.default_rng(5).standard_normal(ARCH.param_count()) * 0.1).astype(np.float32)
    eng = OracleEngine(orc, ARCH, theta, make_tasks(), CFG)
    meta_train(eng, 4, MetaConfig(N=2, q=2, beta=0.3, seed=9, tasks_per_step=4), world=world, rank=rank,
               allreduce=lambda b: dist.all_reduce(b))
    if rank == 0:
        np.save(out_path, eng.theta)
    dist.barrier()
    dist.destroy_process_group()


def test_reptile_allreduce_two_gloo_ranks(oracle, tmp_path):
    out = str(tmp_path / "theta2.npy")
    port = 29500 + os.getpid() % 1000
    mp.spawn(_rank_main, args=(2, port, out), nprocs=2, join=True)
    theta2 = np.load(out)
    # single process, same schedule and draws
    theta = (np.random.default_rng(5).standard_normal(ARCH.param_count()) * 0.1).astype(np.float32)
    eng = OracleEngine(oracle, ARCH, theta, make_tasks(), CFG)
    meta_train(eng, 4, MetaConfig(N=2, q=2, beta=0.3, seed=9, tasks_per_step=4))
    np.testing.assert_allclose(theta2, eng.theta, rtol=1e-5, atol=1e-7)
    # linearity: one meta-step == reptile_update(theta, mean adapted, beta)
    eng1 = OracleEngine(oracle, ARCH, theta, make_tasks(), CFG)
    meta_train(eng1, 4, MetaConfig(N=1, q=2, beta=0.3, seed=9, tasks_per_step=4))
    mean_adapted = np.mean([eng1.adapted[t] for t in range(4)], axis=0).astype(np.float32)
    np.testing.assert_allclose(eng1.theta, oracle.reptile_update(theta, mean_adapted, 0.3), rtol=1e-5, atol=1e-7)


def test_bench_gpus_flag_spawns_ranks(monkeypatch):
    """`bench.py --gpus N` outside torchrun re-executes itself under torch.distributed.run with N
    ranks on 127.0.0.1; inside a launch the rank count must equal --gpus (fails loudly)."""
    import subprocess
    import sys

    import bench

    calls = []
    monkeypatch.setattr(subprocess, "call", lambda cmd: calls.append(cmd) or 0)
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.delenv("TORCHELASTIC_RUN_ID", raising=False)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--workload", "cfg4", "--steps", "3"])
    with pytest.raises(SystemExit) as e:
        bench.main()
    assert e.value.code == 0 and len(calls) == 1
    cmd = calls[0]
    assert cmd[1:3] == ["-m", "torch.distributed.run"] and "--nproc-per-node=4" in cmd
    assert "--master-addr=127.0.0.1" in cmd and cmd[-6:] == ["--gpus", "4", "--workload", "cfg4", "--steps", "3"]
    monkeypatch.setenv("WORLD_SIZE", "2")
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4"])
    with pytest.raises(SystemExit, match="WORLD_SIZE=2"):
        bench.main()


def _objects_rank_main(rank, world, port, out_path):
    """One rank of the object-sharded path (cfg3/cfg5): LPT shard of the objects, each trained
    independently (oracle objects stand in for the GPU ones), per-object losses gathered."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.pyoracle import Oracle

    orc = Oracle()
    tasks = make_tasks()
    archs = [ARCH, FieldArch(hash_levels=4, log2_table_size=9, hidden_width=8, hidden_layers=2), ARCH,
             FieldArch(hash_levels=2, log2_table_size=7, hidden_width=4, hidden_layers=1)]
    mine = shard_lpt([step_cost(a, CFG.rays_per_iter, CFG.samples_per_ray) for a in archs], world)[rank]
    losses = torch.zeros(len(archs), 3, dtype=torch.float64)
    for i in mine:
        sc = tasks[i]
        theta = (np.random.default_rng(40 + i).standard_normal(archs[i].param_count()) * 0.1).astype(np.float32)
        ob = orc.object_create(archs[i], theta, None, 8, 70 + i, CFG.to_c(), sc.box_min, sc.box_max)
        ob.set_frames(sc.cams, sc.rgb, sc.depth, sc.mask, 1, sc.obj_pose)
        losses[i] = torch.tensor([s["total"] for s in ob.train_step(3)], dtype=torch.float64)
    dist.all_reduce(losses)  # every object lives on exactly one rank: the sum is a gather
    if rank == 0:
        np.save(out_path, losses.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_object_sharding_two_gloo_ranks(oracle, tmp_path):
    """Objects are independent (mapper.cpp:572-585): LPT-sharding them over 2 ranks and gathering
    their losses gives exactly the single-process per-object losses -- no data-path collective."""
    out = str(tmp_path / "losses.npy")
    port = 30500 + os.getpid() % 1000
    mp.spawn(_objects_rank_main, args=(2, port, out), nprocs=2, join=True)
    got = np.load(out)
    tasks = make_tasks()
    archs = [ARCH, FieldArch(hash_levels=4, log2_table_size=9, hidden_width=8, hidden_layers=2), ARCH,
             FieldArch(hash_levels=2, log2_table_size=7, hidden_width=4, hidden_layers=1)]
    assert sorted(i for s in shard_lpt([step_cost(a, 16, 8) for a in archs], 2) for i in s) == [0, 1, 2, 3]
    for i, sc in enumerate(tasks):
        theta = (np.random.default_rng(40 + i).standard_normal(archs[i].param_count()) * 0.1).astype(np.float32)
        ob = oracle.object_create(archs[i], theta, None, 8, 70 + i, CFG.to_c(), sc.box_min, sc.box_max)
        ob.set_frames(sc.cams, sc.rgb, sc.depth, sc.mask, 1, sc.obj_pose)
        want = [s["total"] for s in ob.train_step(3)]
        assert np.array_equal(got[i], want), (i, got[i], want)
