"""Reptile meta-learning of category priors (BASELINE config 4).

Reference: meta.cpp:24-120 -- inner_adapt (q Adam steps on one task with
midpoint sampling and a FRESH Adam, meta.cpp:31-34), reptile_update
(meta.cpp:83-92), meta_train (round-robin over a per-epoch reshuffled task
order, meta.cpp:94-120; inner stream mt19937(derive_seed(seed, step)),
meta.cpp:111).

B200 design: each rank adapts its share of a meta-batch of tasks on its GPU
(one ObjectTrainer per task holds the task's views; the meta parameters live
in a frames-less ObjectTrainer), sums the deltas theta_i - theta, and the
ranks all-reduce that sum over NCCL inside the C ABI (prenom_reptile_step, the
communicator bound to the context) -- the only collective of the whole path.
Then

    theta <- (1 - beta) theta + beta (theta + sum_i delta_i / T),

i.e. reptile_update(theta, mean_i theta_i, beta) by linearity.
With one task per meta-step on one rank the exact reference update
reptile_update(theta, theta_1, beta) is applied instead.

The orchestration below only talks to an `Engine`; the product engine is
`CudaEngine` (C-ABI calls). Tests drive the same orchestration with a CPU
engine built on the oracle (tests/test_meta_parallel.py).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

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


class _Mt19937:
    """std::mt19937(seed32): raw 32-bit outputs (numpy's MT19937 with init_genrand seeding)."""

    def __init__(self, seed32: int):
        self.bg = np.random.MT19937()
        self.bg._legacy_seeding(int(seed32) & 0xFFFFFFFF)

    def __call__(self) -> int:
        return int(self.bg.random_raw())


def _uniform_int(g: _Mt19937, a: int, b: int) -> int:
    """libstdc++ (GCC 13) std::uniform_int_distribution<size_t>{a, b}(mt19937): the
    generator's range is exactly 2^32 - 1, so downscaling takes Lemire's nearly
    divisionless path (_S_nd<uint64_t>: product = g() * range, reject low < -range % range)."""
    rng = b - a + 1
    assert 0 < rng <= 0xFFFFFFFF
    prod = g() * rng
    low = prod & 0xFFFFFFFF
    if low < rng:
        thresh = ((1 << 32) - rng) % rng
        while low < thresh:
            prod = g() * rng
            low = prod & 0xFFFFFFFF
    return a + (prod >> 32)


def std_shuffle(order: list, g: _Mt19937) -> None:
    """libstdc++ (GCC 13) std::shuffle(first, last, mt19937&) in place: while n^2 fits the
    generator's range, swap positions come two at a time from one draw
    (__gen_two_uniform_ints: x in [0, b0*b1), positions x / b1 and x % b1), after a lone
    first swap when n is even; otherwise one uniform_int_distribution draw per element."""
    n = len(order)
    if n < 2:
        return
    if 0xFFFFFFFF // n >= n:
        i = 1
        if n % 2 == 0:
            j = _uniform_int(g, 0, 1)
            order[i], order[j] = order[j], order[i]
            i += 1
        while i != n:
            r = i + 1  # swap range of element i
            x = _uniform_int(g, 0, r * (r + 1) - 1)
            j0, j1 = x // (r + 1), x % (r + 1)
            order[i], order[j0] = order[j0], order[i]
            i += 1
            order[i], order[j1] = order[j1], order[i]
            i += 1
        return
    for i in range(1, n):
        j = _uniform_int(g, 0, i)
        order[i], order[j] = order[j], order[i]


def task_schedule(n_tasks: int, n_steps: int, tasks_per_step: int, seed: int) -> list[list[int]]:
    """Task indices of each meta-step: round-robin over an order reshuffled in place at every
    epoch, std::shuffle over std::mt19937(derive_seed(seed, 0xE9C6 + epoch)) exactly as
    meta.cpp:104-110 runs it (libstdc++ algorithm restated above; pinned against the compiled
    reference by tests/test_meta_parallel.py). With tasks_per_step = 1 this is meta_train's
    order step for step."""
    order = list(range(n_tasks))
    out, k = [], 0
    for _step in range(n_steps):
        batch = []
        for _ in range(tasks_per_step):
            slot = k % n_tasks
            if slot == 0:
                std_shuffle(order, _Mt19937(derive_seed(seed, 0xE9C6 + k // n_tasks)))
            batch.append(order[slot])
            k += 1
        out.append(batch)
    return out


class Engine:
    """What the Reptile orchestration needs from a compute backend."""

    def adapt(self, task: int, q: int, seed: int) -> None:  # inner_adapt into the task's worker
        raise NotImplementedError

    def update_exact(self, task: int, beta: float) -> None:  # reptile_update(theta, theta_task, beta)
        raise NotImplementedError

    def reptile_step(self, tasks: list[int], n_tasks: int, beta: float, allreduce=None) -> None:
        """theta <- reptile_update(theta, mean over the meta-batch, beta); `tasks` are this
        rank's. Default: delta_sum -> allreduce(buf) (in place, None on one rank) -> apply."""
        buf = self.delta_sum(tasks)
        if allreduce is not None:
            allreduce(buf)
        self.apply(buf, n_tasks, beta)

    def delta_sum(self, tasks: list[int]):  # sum_i (theta_i - theta), a reducible buffer
        raise NotImplementedError

    def apply(self, delta_sum, n_tasks: int, beta: float) -> None:
        raise NotImplementedError


def meta_train(engine: Engine, n_tasks: int, cfg: MetaConfig, world: int = 1, rank: int = 0, allreduce=None):
    """Run cfg.N meta-steps. Each rank adapts the tasks of the meta-batch with
    index % world == rank; the engine's reptile_step sums them across ranks
    (CudaEngine: NCCL inside the C call; CPU engines: `allreduce(buf)`, which
    sums buf over ranks in place)."""
    sched = task_schedule(n_tasks, cfg.N, cfg.tasks_per_step, cfg.seed)
    for step, batch in enumerate(sched):
        mine = [t for i, t in enumerate(batch) if i % world == rank]
        for j, t in enumerate(batch):
            if j % world == rank:
                # inner stream per (meta-step, slot): derive_seed(seed, step) for slot 0 (meta.cpp:111)
                engine.adapt(t, cfg.q, derive_seed(cfg.seed, step * max(cfg.tasks_per_step, 1) + j))
        if world == 1 and len(batch) == 1:
            engine.update_exact(batch[0], cfg.beta)
        else:
            engine.reptile_step(mine, len(batch), cfg.beta, allreduce)


class CudaEngine(Engine):
    """Product engine: tasks are ObjectTrainers (views on the device), the meta parameters a
    frames-less ObjectTrainer. A meta-step is C-ABI calls only, all ordered on the library's
    stream with no host synchronisation: inner loops (prenom_train_step), then
    prenom_reptile_step -- delta-sum kernel, ncclAllReduce over the context's communicator
    (bound with Context.init_comm when world > 1), interpolation kernel."""

    def __init__(self, meta, workers):
        self.meta, self.workers = meta, workers

    def adapt(self, task, q, seed):
        w = self.workers[task]
        w.copy_params_from(self.meta)  # params = theta; fresh Adam (meta.cpp:31-34)
        w.set_seed(seed)
        w.train_step(q, stats=False)

    def reptile_step(self, tasks, n_tasks, beta, allreduce=None):
        from .trainer import reptile_step

        reptile_step(self.meta, [self.workers[t] for t in tasks], n_tasks, beta)

    def update_exact(self, task, beta):
        self.meta.reptile_update(self.workers[task], beta)
