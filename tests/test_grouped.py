"""GPU: grouped multi-object launches (prenom_train_step_many with same-arch objects).

run_mapper trains one object per worker (mapper.cpp:572-585); the B200 scheduler trains the
objects of one architecture and batch shape through ONE launch per stage (k_sample_grp,
k_fwd_wx<GRP>, k_composite_grp, k_bwd_tc<GRP> + k_mlp_grad_reduce_grp, k_adam_grp) over a
per-object descriptor table. Each object's step must be the one prenom_train_step runs: the
same samples and keyframes (bit-exact), the same first-step loss (bit-exact: the forward and
compositing do the same arithmetic per sample), and then the same training up to the
summation order of the gradient atomics / MLP-gradient partials.
"""
import numpy as np
import pytest

from paper_2503_01582_b200 import FieldArch, ObjectTrainer, TrainConfig, scenes
from paper_2503_01582_b200 import trainer as T
from paper_2503_01582_b200._capi import MLP_BF16, MLP_BF16X3

pytestmark = pytest.mark.gpu

ARCH_A = FieldArch(hash_levels=8, features_per_level=2, log2_table_size=13, base_resolution=8, per_level_scale=1.4,
                   hidden_width=32, hidden_layers=2)
ARCH_B = FieldArch(hash_levels=16, features_per_level=2, log2_table_size=12, base_resolution=8, per_level_scale=1.3,
                   hidden_width=64, hidden_layers=1)


def make(ctx, arch, i, mlp, refresh=5, rays=256, prior=1):
    sc = scenes.box_union_scene(n_views=5, res=48, seed=300 + i)
    cfg = TrainConfig(rays_per_iter=rays, samples_per_ray=48, coarse_samples=16, prior_sampling=prior,
                      grid_refresh_every=refresh, mlp_precision=mlp)
    o = ObjectTrainer.create(ctx, arch, grid=scenes.occupancy_prior(sc.boxes, R=16), seed=40 + i, cfg=cfg,
                             box_min=sc.box_min, box_max=sc.box_max)
    o.set_frames(sc.cams, sc.rgb, sc.depth, sc.mask, 1, sc.obj_pose)
    return o


@pytest.fixture(autouse=True)
def grouping_off_after(ctx):
    yield
    ctx.set_grouping(False)  # the library default


def pairs(ctx, mlp, n=3, **kw):
    """n objects of ARCH_A (a group) + one of ARCH_B, twice: grouped run and reference run."""
    mk = lambda: [make(ctx, ARCH_A, i, mlp, **kw) for i in range(n)] + [make(ctx, ARCH_B, 9, mlp, **kw)]
    return mk(), mk()


@pytest.mark.parametrize("mlp", [MLP_BF16X3, MLP_BF16])
def test_grouped_steps_equal_per_object_steps(ctx, mlp):
    grouped, alone = pairs(ctx, mlp)
    ctx.set_grouping(True)
    steps = 12
    T.train_many(grouped, steps)
    for o in alone:
        o.train_step(steps, stats=False)
    for a, b in zip(grouped, alone):
        la, lb = a.last_stats(steps), b.last_stats(steps)
        assert la[0] == lb[0]  # same samples, same forward and compositing arithmetic: bit-exact
        for k, (x, y) in enumerate(zip(la, lb)):
            assert x["frame"] == y["frame"]
            if k < 5:  # before the first grid refresh the samples do not depend on the weights
                assert x["n_samples"] == y["n_samples"] and x["escaped"] == y["escaped"]
            assert abs(x["total"] - y["total"]) <= 2e-3 * abs(y["total"]), (k, x, y)
        pa, pb = a.get_params(), b.get_params()
        assert np.linalg.norm(pa - pb) <= 2e-3 * np.linalg.norm(pb)
        assert a.step() == b.step() == steps  # step counters advanced by the call


def test_grouping_launches_one_kernel_per_stage(ctx):
    """3 same-arch objects + 1 other: per step 6 grouped launches + the single object's 5 (its
    MLP-gradient reduction runs inside its Adam launch)."""
    grouped, _ = pairs(ctx, MLP_BF16X3, refresh=0)
    ctx.set_grouping(True)
    T.train_many(grouped, 1)
    ctx.synchronize()
    n0 = ctx.launch_count()
    T.train_many(grouped, 4)
    ctx.synchronize()
    assert ctx.launch_count() - n0 == 4 * (6 + 5)
    ctx.set_grouping(False)
    n0 = ctx.launch_count()
    T.train_many(grouped, 4)
    ctx.synchronize()
    assert ctx.launch_count() - n0 == 4 * 4 * 5


def test_grouped_first_step_matches_oracle(ctx, oracle):
    """Split-bf16 grouped step vs the CPU oracle: loss terms within 1e-5 (the north_star fp32 bar)."""
    objs = [make(ctx, ARCH_A, i, MLP_BF16X3, refresh=0) for i in range(4)]
    refs = []
    for i, o in enumerate(objs):
        sc = scenes.box_union_scene(n_views=5, res=48, seed=300 + i)
        cfg = TrainConfig(rays_per_iter=256, samples_per_ray=48, coarse_samples=16, prior_sampling=1,
                          grid_refresh_every=0)
        ob = oracle.object_create(ARCH_A, o.get_params(), scenes.occupancy_prior(sc.boxes, R=16), 16, 40 + i,
                                  cfg.to_c(), sc.box_min, sc.box_max)
        ob.set_frames(sc.cams, sc.rgb, sc.depth, sc.mask, 1, sc.obj_pose)
        refs.append(ob)
    ctx.set_grouping(True)
    T.train_many(objs, 1)
    for o, ob in zip(objs, refs):
        g, r = o.last_stats(1)[0], ob.train_step(1)[0]
        assert g["frame"] == r["frame"] and g["n_samples"] == r["n_samples"]
        for k in ("total", "color", "depth", "sigma"):
            assert abs(g[k] - r[k]) <= 1e-5 * abs(r[k]) + 1e-9, (k, g, r)


def test_grouped_ragged_tiles_and_one_ray(ctx):
    """Batches that are not a multiple of the 128-sample tile (333 x 48) and a 1-ray group."""
    for rays in (333, 1):
        grouped = [make(ctx, ARCH_A, i, MLP_BF16X3, refresh=0, rays=rays) for i in range(3)]
        alone = [make(ctx, ARCH_A, i, MLP_BF16X3, refresh=0, rays=rays) for i in range(3)]
        ctx.set_grouping(True)
        T.train_many(grouped, 3)
        for o in alone:
            o.train_step(3, stats=False)
        for a, b in zip(grouped, alone):
            la, lb = a.last_stats(3), b.last_stats(3)
            assert la[0] == lb[0]
            for x, y in zip(la, lb):
                assert abs(x["total"] - y["total"]) <= 2e-3 * abs(y["total"]) + 1e-9


def test_grouped_long_call_spans_job_chunks(ctx):
    """A 70-step call (job arrays uploaded 64 steps at a time): same keyframes and samples as
    per-object training for every step, step counters advanced by 70, losses close."""
    grouped = [make(ctx, ARCH_A, i, MLP_BF16X3, refresh=0, rays=64) for i in range(2)]
    alone = [make(ctx, ARCH_A, i, MLP_BF16X3, refresh=0, rays=64) for i in range(2)]
    ctx.set_grouping(True)
    T.train_many(grouped, 70)
    for o in alone:
        o.train_step(70, stats=False)
    for a, b in zip(grouped, alone):
        assert a.step() == b.step() == 70
        la, lb = a.last_stats(70), b.last_stats(70)
        assert la[0] == lb[0]
        for x, y in zip(la, lb):
            assert x["frame"] == y["frame"] and x["n_samples"] == y["n_samples"]
            assert abs(x["total"] - y["total"]) <= 2e-2 * abs(y["total"]) + 1e-9


def test_grouped_objects_at_different_steps_and_cadences(ctx):
    """A group whose objects are at different steps (Adam bias corrections, keyframe picks,
    Philox streams per object) and refresh their grids on different cadences."""
    def pair(i, pre, refresh):
        a = make(ctx, ARCH_A, i, MLP_BF16X3, refresh=refresh, rays=96)
        b = make(ctx, ARCH_A, i, MLP_BF16X3, refresh=refresh, rays=96)
        if pre:
            a.train_step(pre, stats=False)
            b.train_step(pre, stats=False)
        return a, b
    pairs_ = [pair(0, 0, 3), pair(1, 5, 4), pair(2, 2, 0)]
    ctx.set_grouping(True)
    T.train_many([a for a, _ in pairs_], 6)
    for (a, b), pre in zip(pairs_, (0, 5, 2)):
        b.train_step(6, stats=False)
        assert a.step() == b.step() == pre + 6
        la, lb = a.last_stats(6), b.last_stats(6)
        assert la[0]["frame"] == lb[0]["frame"] and la[0]["n_samples"] == lb[0]["n_samples"]
        assert abs(la[0]["total"] - lb[0]["total"]) <= 1e-5 * abs(lb[0]["total"])
        for x, y in zip(la, lb):
            assert x["frame"] == y["frame"]
            assert abs(x["total"] - y["total"]) <= 5e-3 * abs(y["total"]) + 1e-9


@pytest.mark.parametrize("mlp", [MLP_BF16X3, MLP_BF16])
def test_two_groups_of_different_archs(ctx, mlp):
    """Two groups in one call (W32 H2 INP16 and W64 H1 INP32: the latter's split backward has no
    feature overlay), on two lanes, each equal to per-object training."""
    mk = lambda: ([make(ctx, ARCH_A, i, mlp, refresh=4) for i in range(2)]
                  + [make(ctx, ARCH_B, 5 + i, mlp, refresh=4) for i in range(3)])
    grouped, alone = mk(), mk()
    ctx.set_grouping(True)
    T.train_many(grouped, 6)
    for o in alone:
        o.train_step(6, stats=False)
    for a, b in zip(grouped, alone):
        la, lb = a.last_stats(6), b.last_stats(6)
        assert la[0] == lb[0]
        for x, y in zip(la, lb):
            assert x["frame"] == y["frame"]
            assert abs(x["total"] - y["total"]) <= 2e-3 * abs(y["total"]) + 1e-9
