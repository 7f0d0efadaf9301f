"""GPU: Reptile meta-training (CudaEngine) and multi-object training vs the oracle."""
import numpy as np
import pytest
import torch

from paper_2503_01582_b200 import FieldArch, ObjectTrainer, TrainConfig, scenes
from paper_2503_01582_b200 import trainer as T
from paper_2503_01582_b200.meta import CudaEngine, MetaConfig, meta_train

from test_meta_parallel import OracleEngine

pytestmark = pytest.mark.gpu

ARCH = FieldArch(hash_levels=6, features_per_level=2, log2_table_size=11, base_resolution=6, per_level_scale=1.5,
                 hidden_width=16, hidden_layers=2)
CFG = TrainConfig(rays_per_iter=64, samples_per_ray=16, prior_sampling=0, grid_refresh_every=0)


def tasks():
    return [scenes.box_union_scene(n_views=4, res=32, seed=200 + i) for i in range(3)]


@pytest.mark.parametrize("tps", [1, 3])
def test_reptile_cuda_engine_matches_oracle_engine(ctx, oracle, tps):
    ts = tasks()
    theta = (np.random.default_rng(1).standard_normal(ARCH.param_count()) * 0.05).astype(np.float32)
    meta = ObjectTrainer.create(ctx, ARCH, theta=theta, grid_res=8, cfg=CFG)
    workers = []
    for sc in ts:
        w = ObjectTrainer.create(ctx, ARCH, theta=theta, grid_res=8, cfg=CFG, box_min=sc.box_min, box_max=sc.box_max)
        w.set_frames(sc.cams, sc.rgb, sc.depth, sc.mask, 1, sc.obj_pose)
        workers.append(w)
    mc = MetaConfig(N=3, q=4, beta=0.2, seed=7, tasks_per_step=tps)
    meta_train(CudaEngine(meta, workers), len(ts), mc)
    ref = OracleEngine(oracle, ARCH, theta, ts, CFG)
    meta_train(ref, len(ts), mc)
    got = meta.get_params()
    # Same draws (bit-exact samples); parameters differ only by gradient summation order.
    moved = np.abs(ref.theta - theta) > 1e-6
    assert moved.mean() > 0.01
    err = np.abs(got - ref.theta)
    assert np.quantile(err, 0.999) < 2e-3, np.quantile(err, 0.999)


def test_train_many_equals_individual_training(ctx):
    """prenom_train_step_many (objects concurrently on lane streams) == training each alone."""
    ts = tasks()
    objs_a, objs_b = [], []
    for i, sc in enumerate(ts):
        for lst in (objs_a, objs_b):
            o = ObjectTrainer.create(ctx, ARCH, grid_res=8, seed=10 + i, cfg=CFG, box_min=sc.box_min, box_max=sc.box_max)
            o.set_frames(sc.cams, sc.rgb, sc.depth, sc.mask, 1, sc.obj_pose)
            lst.append(o)
    T.train_many(objs_a, 5)
    for o in objs_b:
        o.train_step(5, stats=False)
    for a, b in zip(objs_a, objs_b):
        la, lb = a.last_stats(5), b.last_stats(5)
        for x, y in zip(la, lb):
            assert x["n_samples"] == y["n_samples"] and x["frame"] == y["frame"]
            assert abs(x["total"] - y["total"]) <= 1e-4 * abs(y["total"])


def test_reptile_delta_apply_linearity(ctx, rng):
    """prenom_reptile_delta + NCCL-style sum + prenom_reptile_apply == reptile_update(theta, mean)."""
    P = ARCH.param_count()
    th = rng.standard_normal(P).astype(np.float32)
    meta = ObjectTrainer.create(ctx, ARCH, theta=th, grid_res=8, cfg=CFG)
    ads = [rng.standard_normal(P).astype(np.float32) for _ in range(3)]
    objs = [ObjectTrainer.create(ctx, ARCH, theta=a, grid_res=8, cfg=CFG) for a in ads]
    acc = torch.zeros(P, device="cuda")
    tmp = torch.empty(P, device="cuda")
    for o in objs:
        T.reptile_delta(meta, o, tmp.data_ptr())
        ctx.synchronize()  # stream-ordered on the library stream; torch reads it next
        acc += tmp
    torch.cuda.synchronize()
    T.reptile_apply(meta, acc.data_ptr(), 3, 0.1)
    mean = np.mean(ads, axis=0)
    want = (np.float32(0.9) * th + np.float32(0.1) * mean).astype(np.float32)
    np.testing.assert_allclose(meta.get_params(), want, rtol=1e-5, atol=1e-6)
    # exact single-task update (meta.cpp:83-92)
    meta.set_params(th)
    meta.reptile_update(objs[0], 0.1)
    assert np.array_equal(meta.get_params(), (np.float32(0.9) * th + np.float32(0.1) * ads[0]).astype(np.float32))


def test_streaming_async_steps_equal_train_step(ctx):
    """prenom_train_step_async + prenom_wait_stats with a keyframe upload before every
    step (the e2e streaming loop of bench.py) == prenom_train_step on a twin object."""
    import torch

    sc = tasks()[0]
    a = ObjectTrainer.create(ctx, ARCH, grid_res=8, seed=21, cfg=CFG, box_min=sc.box_min, box_max=sc.box_max)
    b = ObjectTrainer.create(ctx, ARCH, grid_res=8, seed=21, cfg=CFG, box_min=sc.box_min, box_max=sc.box_max)
    for o in (a, b):
        o.set_frames(sc.cams, sc.rgb, sc.depth, sc.mask, 1, sc.obj_pose)
    want = a.train_step(6)
    rgb = torch.from_numpy(np.ascontiguousarray(sc.rgb)).pin_memory()
    dep = torch.from_numpy(np.ascontiguousarray(sc.depth)).pin_memory()
    got, prev = [], None
    for i in range(6):
        f = b.frame_at(i)
        assert f == want[i]["frame"]
        b.upload_frame(f, rgb[f].numpy(), dep[f].numpy(), None)
        tk = b.train_step_async(1, prefetch_next=i < 5)
        if prev is not None:
            got += b.wait_stats(prev)
        prev = tk
    got += b.wait_stats(prev)
    for x, y in zip(got, want):
        assert x["n_samples"] == y["n_samples"] and x["frame"] == y["frame"]
        assert abs(x["total"] - y["total"]) <= 1e-4 * abs(y["total"])
    with pytest.raises(Exception, match="ticket"):
        b.wait_stats(12345)


@pytest.mark.parametrize("mutation", ["upload_new_pixels", "set_seed", "restore", "set_grid", "render"])
def test_pending_prefetch_is_dropped_by_state_changes(ctx, mutation):
    """A step enqueued with prefetch_next samples step t+1 ahead on the sampling stream. A call
    that changes what step t+1 must sample -- new pixels for its keyframe, a new seed, a
    checkpoint restore, a new sampling grid -- drops that prefetch, so the step equals the same
    sequence run without any prefetch; so does a render, which reuses the sample buffers."""
    sc = tasks()[1]
    grid = scenes.occupancy_prior(sc.boxes, R=16)
    cfg = TrainConfig(rays_per_iter=128, samples_per_ray=32, prior_sampling=1, grid_refresh_every=0)

    def make():
        o = ObjectTrainer.create(ctx, ARCH, grid=grid, seed=5, cfg=cfg, box_min=sc.box_min, box_max=sc.box_max)
        o.set_frames(sc.cams, sc.rgb, sc.depth, sc.mask, 1, sc.obj_pose)
        return o

    a, b = make(), make()
    ck = a.checkpoint()
    f1 = a.frame_at(1)
    new_rgb = np.ascontiguousarray(1.0 - sc.rgb[f1]).astype(np.float32)
    new_grid = np.ascontiguousarray(grid[::-1]).astype(np.float32)

    def mutate(o):
        if mutation == "upload_new_pixels":
            o.upload_frame(f1, new_rgb, np.ascontiguousarray(sc.depth[f1]), None)
        elif mutation == "set_seed":
            o.set_seed(99)
        elif mutation == "restore":
            o.restore(ck)
        elif mutation == "render":  # reuses the sample buffers; must not leave the prefetch corrupted
            orig = np.array([[0.0, 0.0, -2.0], [0.3, -0.2, 2.0]], np.float32)
            dirs = np.array([[0.0, 0.0, 1.0], [0.0, 0.0, -1.0]], np.float32)
            o.render(orig, dirs)
        else:
            o.set_grid(new_grid)

    a.wait_stats(a.train_step_async(1, prefetch_next=True))  # leaves step 1's samples prefetched
    mutate(a)
    got = a.train_step(1)[0]
    b.train_step(1)  # no prefetch
    mutate(b)
    want = b.train_step(1)[0]
    assert got["frame"] == want["frame"] and got["n_samples"] == want["n_samples"]
    assert got["escaped"] == want["escaped"]
    assert abs(got["total"] - want["total"]) <= 1e-4 * abs(want["total"]), (got, want)


@pytest.mark.parametrize("mlp", [0, 1])
def test_checkpoint_resume_continues_the_same_run(ctx, mlp):
    """Checkpoint after 7 steps (θ, Adam m/v/step, sampling grid), restore into a fresh
    object, train 5 more: the same frames, sample counts and losses as the uninterrupted
    run (the step keys the Philox draws; sums differ only by atomic order)."""
    sc = tasks()[1]
    grid = scenes.occupancy_prior(sc.boxes, R=16)
    cfg = TrainConfig(rays_per_iter=128, samples_per_ray=32, prior_sampling=1, grid_refresh_every=4,
                      mlp_precision=mlp)

    arch = FieldArch(hash_levels=6, features_per_level=2, log2_table_size=11, base_resolution=6, per_level_scale=1.5,
                     hidden_width=32, hidden_layers=2)  # tensor-core-eligible for the bf16 case

    def make():
        o = ObjectTrainer.create(ctx, arch, grid=grid, seed=77, cfg=cfg, box_min=sc.box_min, box_max=sc.box_max)
        o.set_frames(sc.cams, sc.rgb, sc.depth, sc.mask, 1, sc.obj_pose)
        return o

    a = make()
    a.train_step(7, stats=False)
    ck = a.checkpoint()
    want = a.train_step(5)
    b = make()
    b.restore(ck)
    assert b.step() == 7
    got = b.train_step(5)
    for x, y in zip(got, want):
        assert x["frame"] == y["frame"] and x["n_samples"] == y["n_samples"]
        assert abs(x["total"] - y["total"]) <= 1e-3 * abs(y["total"])


def test_reptile_step_nccl_one_rank(oracle):
    """prenom_reptile_step with an NCCL communicator bound to the context (1 rank: the
    ncclAllReduce runs for real and is the identity): delta-sum kernel -> all-reduce ->
    interpolation equals the fp32 formula bit for bit, and reptile_update(theta, mean theta_i,
    beta) of the reference restatement to fp32 rounding (meta.cpp:83-92)."""
    from paper_2503_01582_b200 import Context, UsageError

    c = Context(0)
    try:
        c.init_comm(1, 0, T.comm_unique_id())
        n, r, ver = c.comm_info()
        assert (n, r) == (1, 0) and ver > 0
        rng = np.random.default_rng(5)
        P = ARCH.param_count()
        theta = rng.standard_normal(P).astype(np.float32)
        thetas = [(theta + rng.standard_normal(P).astype(np.float32) * 0.1).astype(np.float32) for _ in range(3)]
        meta = ObjectTrainer.create(c, ARCH, theta=theta, grid_res=8, cfg=CFG)
        ws = [ObjectTrainer.create(c, ARCH, theta=t, grid_res=8, cfg=CFG) for t in thetas]
        beta = np.float32(0.1)
        T.reptile_step(meta, ws, 3, float(beta))
        got = meta.get_params()
        acc = np.zeros(P, np.float32)
        for t in thetas:
            acc = (acc + (t - theta)).astype(np.float32)
        inv = np.float32(1.0) / np.float32(3.0)
        adapted = (theta + acc * inv).astype(np.float32)
        want = ((np.float32(1.0) - beta) * theta + beta * adapted).astype(np.float32)
        assert np.array_equal(got, want)
        ref = oracle.reptile_update(theta, np.mean(np.stack(thetas), 0).astype(np.float32), float(beta))
        np.testing.assert_allclose(got, ref, rtol=1e-6, atol=1e-6)
        # a rank with no task in this meta-step still joins the all-reduce
        before = meta.get_params()
        T.reptile_step(meta, [], 2, float(beta))
        np.testing.assert_allclose(meta.get_params(), before, rtol=1e-6, atol=1e-7)
    finally:
        c.close()
    # without a communicator the other ranks' tasks cannot be summed
    c2 = Context(0)
    try:
        meta = ObjectTrainer.create(c2, ARCH, grid_res=8, cfg=CFG)
        w = ObjectTrainer.create(c2, ARCH, grid_res=8, cfg=CFG)
        with pytest.raises(UsageError):
            T.reptile_step(meta, [w], 2, 0.1)
        T.reptile_step(meta, [w], 1, 0.1)  # one task, no communicator: the exact reference update
    finally:
        c2.close()
