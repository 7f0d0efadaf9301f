"""GPU-backed genome evaluation: the fitness function the
reference's NSGA-II architecture search calls per genome, with every training
and extraction step on the B200 path.

Reference: search.cpp:138-161 (arch_of, meta_config_of), 214-228
(iter_cost_model), 230-270 (evaluate_genome):

    time_per_iter = time_scale * iter_cost_model(arch, inner)
    theta = meta_train(train_tasks, arch, meta_config_of(g, inner, seed))    -> Reptile on the GPU
    for each test task i:
        adapted = inner_adapt(theta, arch, task, adapt_iters, g.eta, ...)    -> train steps on the GPU
        grid = refresh_grid(arch, adapted, grid_resolution)                 -> device density query
        mesh = marching_cubes(grid, choose_iso(grid))                       -> device marching cubes
        cd_i = chamfer(sample_surface(transformed(mesh, gt_size, box.min)),
                       sample_surface(gt_mesh))                              -> device NN search
    cd = mean_i cd_i (non-finite -> 1e6)

The NSGA-II loop itself (non_dominated_sort, crowding, evolve) is host
bookkeeping over these evaluations and stays out of scope.
Randomness: meta-training and adaptation draw from Philox (G3);
surface sampling is the reference's own mt19937 stream (metrics.py), so given
the same meshes the metric is bit-exact.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import metrics as M
from ._capi import MLP_FP32
from .meta import CudaEngine, MetaConfig, meta_train
from .prior import Genome
from .trainer import DataError, FieldArch, NumericError, ObjectTrainer, TrainConfig

PENALTY_CD = 1e6  # search.cpp:17


def search_mix_seed(base: int, salt: int) -> int:
    """search.cpp:19-25 (its own salt multiplier, unlike mapper.cpp's)."""
    M64 = (1 << 64) - 1
    s = (base * 0x9E3779B97F4A7C15 + salt * 0xD1B54A32D192ED03 + 1) & M64
    s ^= s >> 31
    s = (s * 0x94D049BB133111EB) & M64
    s ^= s >> 29
    return (s ^ (s >> 32)) & 0xFFFFFFFF


def arch_of(g: Genome) -> FieldArch:
    """search.cpp:138-148 (base_resolution keeps the FieldArch default)."""
    return FieldArch(hash_levels=g.hash_levels, features_per_level=g.features_per_level,
                     log2_table_size=g.log2_table_size, per_level_scale=g.per_level_scale,
                     hidden_width=g.hidden_width, hidden_layers=g.hidden_layers,
                     density_activation=g.density_activation)


@dataclass
class SearchConfig:
    """The evaluation keys of noma::SearchConfig (search.hpp:75-88)."""

    rays_per_iter: int = 64  # inner{64, 0.25, 16, {}}
    bg_fraction: float = 0.25
    samples_per_ray: int = 16
    adapt_iters: int = 60
    grid_resolution: int = 32
    metric_samples: int = 2048
    time_scale: float = 2.5e-10
    mlp_precision: int = MLP_FP32


@dataclass
class Evaluation:
    """noma::Evaluation (search.hpp:70-73); both objectives minimised."""

    time_per_iter: float = 0.0
    cd: float = 0.0
    per_task_cd: list = field(default_factory=list)


@dataclass
class EvalTask:
    """A task as evaluate_genome reads it (task.hpp:23-36): views + camera poses, the
    object box (gt_center +- gt_size/2, object frame = scene frame here), and the
    ground-truth mesh in metric units."""

    scene: object  # scenes.Scene: cams, rgb, depth, mask, obj_pose
    gt_vertices: np.ndarray
    gt_triangles: np.ndarray
    gt_size: np.ndarray = field(default_factory=lambda: np.ones(3, np.float32))
    gt_center: np.ndarray = field(default_factory=lambda: np.zeros(3, np.float32))

    @property
    def box_min(self):
        return (np.asarray(self.gt_center, np.float32) - np.asarray(self.gt_size, np.float32) * np.float32(0.5))

    @property
    def box_max(self):
        return (np.asarray(self.gt_center, np.float32) + np.asarray(self.gt_size, np.float32) * np.float32(0.5))


def iter_cost_model(arch: FieldArch, rays_per_iter: int, samples_per_ray: int) -> float:
    """search.cpp:214-228 (modelled arithmetic ops of one inner iteration)."""
    L, F = float(arch.hash_levels), float(arch.features_per_level)
    W, H = float(arch.hidden_width), float(arch.hidden_layers)
    inp = L * F
    encode = L * 8.0 * (2.0 * F + 10.0)
    mlp = 2.0 * (inp * W + max(H - 1.0, 0.0) * W * W + 4.0 * W) + H * W
    per_point = 3.0 * (encode + mlp)
    points = float(rays_per_iter) * samples_per_ray
    adam = 10.0 * float(arch.param_count())
    return points * per_point + adam


def _inner_cfg(g: Genome, cfg: SearchConfig) -> TrainConfig:
    """meta_config_of's InnerOptions (search.cpp:150-161) as the worker's train config:
    midpoint sampling over the object box (meta.cpp:57), no grid refresh."""
    return TrainConfig(rays_per_iter=cfg.rays_per_iter, bg_fraction=cfg.bg_fraction,
                       samples_per_ray=cfg.samples_per_ray, lambda_d=g.lambda_d, lambda_sigma=g.lambda_sigma,
                       prior_sampling=0, grid_refresh_every=0, eta=g.eta, mlp_precision=cfg.mlp_precision)


def _worker(ctx, arch, tcfg, task: EvalTask):
    w = ObjectTrainer.create(ctx, arch, theta=None, grid_res=8, seed=1, cfg=tcfg, box_min=task.box_min,
                             box_max=task.box_max)
    sc = task.scene
    w.set_frames(sc.cams, sc.rgb, sc.depth, sc.mask, 1, sc.obj_pose)
    return w


def evaluate_genome(ctx, g: Genome, train_tasks: list, test_tasks: list, eval_seed: int,
                    cfg: SearchConfig | None = None) -> Evaluation:
    """search.cpp:230-270 on the GPU."""
    cfg = cfg or SearchConfig()
    if not train_tasks or not test_tasks:
        raise DataError("evaluate_genome: empty task set")
    arch = arch_of(g)
    ev = Evaluation(time_per_iter=cfg.time_scale * iter_cost_model(arch, cfg.rays_per_iter, cfg.samples_per_ray))
    tcfg = _inner_cfg(g, cfg)
    objs = []
    try:
        # meta_train (meta.cpp:94-120): theta = init_params(arch, seed), Reptile over the train split
        meta = ObjectTrainer.create(ctx, arch, theta=None, grid_res=8, seed=eval_seed, cfg=tcfg)
        objs.append(meta)
        workers = [_worker(ctx, arch, tcfg, t) for t in train_tasks]
        objs += workers
        meta_train(CudaEngine(meta, workers), len(workers),
                   MetaConfig(N=g.meta_steps, q=g.inner_iters, eta=g.eta, beta=g.beta, seed=eval_seed))
        theta = meta.get_params()
        if not np.all(np.isfinite(theta)):
            ev.cd = PENALTY_CD
            return ev
        cd_sum = 0.0
        for i, task in enumerate(test_tasks):
            w = _worker(ctx, arch, tcfg, task)
            objs.append(w)
            w.copy_params_from(meta)  # inner_adapt: params = theta, fresh Adam (meta.cpp:31-34)
            w.set_seed(search_mix_seed(eval_seed, 0x7E57 + i))
            task_cd = PENALTY_CD
            try:
                w.train_step(cfg.adapt_iters, stats=False)
                w.check()
                finite = np.all(np.isfinite(w.get_params()))
            except NumericError:
                finite = False
            if finite:
                v, t, _ = w.extract_mesh(cfg.grid_resolution)  # refresh_grid + choose_iso + marching_cubes
                if len(t):
                    metric = M.transformed(v, task.gt_size, task.box_min)  # Pose{{}, box.min}
                    rec = M.sample_surface(metric, t, cfg.metric_samples, search_mix_seed(eval_seed, 0xAB1 + i))
                    gt = M.sample_surface(task.gt_vertices, task.gt_triangles, cfg.metric_samples,
                                          search_mix_seed(eval_seed, 0xCB1 + i))
                    task_cd = M.chamfer(ctx, rec, gt)
            ev.per_task_cd.append(task_cd)
            cd_sum += task_cd
        ev.cd = cd_sum / len(test_tasks)
        if not math.isfinite(ev.cd):
            ev.cd = PENALTY_CD
        return ev
    finally:
        for o in objs:
            o.close()
