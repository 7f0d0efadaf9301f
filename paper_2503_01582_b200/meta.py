"""Reptile meta-learning of category priors (BASELINE config 4).

Reference: meta.cpp:24-120 -- inner_adapt (q Adam steps on one task with
midpoint sampling and a FRESH Adam, meta.cpp:31-34), reptile_update
(meta.cpp:83-92), meta_train (round-robin over a per-epoch reshuffled task
order, meta.cpp:94-120; inner stream mt19937(derive_seed(seed, step)),
meta.cpp:111).

B200 design: each rank adapts its share of a meta-batch of tasks on its GPU
(one ObjectTrainer per task holds the task's views; the meta parameters live
in a frames-less ObjectTrainer), sums the deltas theta_i - theta, and the
ranks all-reduce that sum over NCCL (torch.distributed) -- the only
collective of the whole path. Then

    theta <- (1 - beta) theta + beta (theta + sum_i delta_i / T),

i.e. reptile_update(theta, mean_i theta_i, beta) by linearity.
With one task per meta-step on one rank the exact reference update
reptile_update(theta, theta_1, beta) is applied instead.

The orchestration below only talks to an `Engine`; the product engine is
`CudaEngine` (C-ABI calls). Tests drive the same orchestration with a CPU
engine built on the oracle (tests/test_meta_gloo.py).
"""
from __future__ import annotations

import random
from dataclasses import dataclass, field

from .trainer import derive_seed


@dataclass
class MetaConfig:
    """noma::MetaConfig (meta.hpp:22-29) + the batching of this build."""

    N: int = 300  # meta-steps
    q: int = 40  # inner iterations per task
    eta: float = 1e-2  # inner Adam lr
    beta: float = 0.1  # Reptile interpolation
    seed: int = 0
    tasks_per_step: int = 1  # T (1 = reference meta_train)
    log: list = field(default_factory=list)


def task_schedule(n_tasks: int, n_steps: int, tasks_per_step: int, seed: int) -> list[list[int]]:
    """Task indices of each meta-step: round-robin over an order reshuffled at
    every epoch (meta.cpp:104-110). The shuffle is Python's (seeded by
    derive_seed(seed, 0xE9C6 + epoch)), not libstdc++'s std::shuffle."""
    order = list(range(n_tasks))
    out, k = [], 0
    for _step in range(n_steps):
        batch = []
        for _ in range(tasks_per_step):
            slot = k % n_tasks
            if slot == 0:
                random.Random(derive_seed(seed, 0xE9C6 + k // n_tasks)).shuffle(order)
            batch.append(order[slot])
            k += 1
        out.append(batch)
    return out


class Engine:
    """What the Reptile orchestration needs from a compute backend."""

    def adapt(self, task: int, q: int, seed: int) -> None:  # inner_adapt into the task's worker
        raise NotImplementedError

    def delta_sum(self, tasks: list[int]):  # sum_i (theta_i - theta), a reducible buffer
        raise NotImplementedError

    def apply(self, delta_sum, n_tasks: int, beta: float) -> None:
        raise NotImplementedError

    def update_exact(self, task: int, beta: float) -> None:  # reptile_update(theta, theta_task, beta)
        raise NotImplementedError


def meta_train(engine: Engine, n_tasks: int, cfg: MetaConfig, world: int = 1, rank: int = 0, allreduce=None):
    """Run cfg.N meta-steps. `allreduce(buf)` sums buf over ranks in place
    (None on a single rank). Each rank adapts the tasks of the meta-batch
    with index % world == rank."""
    sched = task_schedule(n_tasks, cfg.N, cfg.tasks_per_step, cfg.seed)
    for step, batch in enumerate(sched):
        mine = [t for i, t in enumerate(batch) if i % world == rank]
        for j, t in enumerate(batch):
            if j % world == rank:
                # inner stream per (meta-step, slot): derive_seed(seed, step) for slot 0 (meta.cpp:111)
                engine.adapt(t, cfg.q, derive_seed(cfg.seed, step * max(cfg.tasks_per_step, 1) + j))
        if world == 1 and len(batch) == 1:
            engine.update_exact(batch[0], cfg.beta)
            continue
        buf = engine.delta_sum(mine)
        if allreduce is not None:
            stream = getattr(engine, "stream", None)
            if stream is not None:
                import torch

                with torch.cuda.stream(stream):
                    allreduce(buf)
            else:
                allreduce(buf)
        engine.apply(buf, len(batch), cfg.beta)


class CudaEngine(Engine):
    """Product engine: tasks are ObjectTrainers (views on the device), the
    meta parameters a frames-less ObjectTrainer; deltas are device buffers
    (torch tensors). Every torch op -- and the caller's NCCL all-reduce, run
    inside `with torch.cuda.stream(engine.stream)` -- is ordered on the
    library's own stream, so a meta-step needs no host synchronization."""

    def __init__(self, meta, workers):
        import torch

        self.meta, self.workers = meta, workers
        self.P = meta.arch.param_count()
        dev = f"cuda:{meta.ctx.device}"
        self.stream = torch.cuda.ExternalStream(meta.ctx.stream, device=dev)
        self.buf = torch.empty(self.P, dtype=torch.float32, device=dev)
        self.tmp = torch.empty(self.P, dtype=torch.float32, device=dev)

    def adapt(self, task, q, seed):
        w = self.workers[task]
        w.copy_params_from(self.meta)  # params = theta; fresh Adam (meta.cpp:31-34)
        w.set_seed(seed)
        w.train_step(q, stats=False)

    def delta_sum(self, tasks):
        import torch

        from .trainer import reptile_delta

        with torch.cuda.stream(self.stream):
            if len(tasks) == 1:
                reptile_delta(self.meta, self.workers[tasks[0]], self.buf.data_ptr())
            else:
                self.buf.zero_()
                for t in tasks:
                    reptile_delta(self.meta, self.workers[t], self.tmp.data_ptr())
                    self.buf += self.tmp
        return self.buf

    def apply(self, delta_sum, n_tasks, beta):
        from .trainer import reptile_apply

        reptile_apply(self.meta, delta_sum.data_ptr(), n_tasks, beta)

    def update_exact(self, task, beta):
        self.meta.reptile_update(self.workers[task], beta)
