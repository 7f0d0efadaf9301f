"""Small end-to-end run for compute-sanitizer: bf16 and fp32 train steps,
render, density query, debug stages (no oracle, no torch)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_01582_b200 import Context, FieldArch, ObjectTrainer, TrainConfig, scenes  # noqa: E402
from paper_2503_01582_b200 import trainer as T  # noqa: E402

ctx = Context(0)
sc = scenes.box_union_scene(n_views=3, res=32, seed=1)
grid = scenes.occupancy_prior(sc.boxes, R=16)
for prec, arch in ((1, scenes.cfg1_arch()), (0, FieldArch(hash_levels=6, log2_table_size=11, hidden_width=16))):
    cfg = TrainConfig(rays_per_iter=300, samples_per_ray=40, prior_sampling=1, grid_refresh_every=2,
                      mlp_precision=prec)
    o = ObjectTrainer.create(ctx, arch, grid=grid, seed=3, cfg=cfg, box_min=sc.box_min, box_max=sc.box_max)
    o.set_frames(sc.cams, sc.rgb, sc.depth, sc.mask, 1, sc.obj_pose)
    print(o.train_step(3)[-1])
    rng = np.random.default_rng(0)
    orig = rng.uniform(-1, 1, (50, 3)).astype(np.float32)
    dirs = (-orig / np.linalg.norm(orig, axis=1, keepdims=True)).astype(np.float32)
    print(o.render(orig, dirs)[0].sum(), o.density_query(9).sum())
    xyz = rng.uniform(0, 1, (130, 3)).astype(np.float32)
    p = o.get_params()
    g = T.debug_field_backward(ctx, arch, p, xyz, rng.standard_normal(130).astype(np.float32),
                               rng.standard_normal((130, 3)).astype(np.float32), precision=prec)
    print(np.abs(g).sum())
# multi-object lanes, streaming API with keyframe uploads, device frames, mesh, metric NN
from paper_2503_01582_b200 import metrics as M  # noqa: E402

cfg = TrainConfig(rays_per_iter=200, samples_per_ray=24, prior_sampling=1, grid_refresh_every=0, mlp_precision=1)
objs = []
for i in range(3):
    o = ObjectTrainer.create(ctx, scenes.cfg1_arch(), grid=grid, seed=10 + i, cfg=cfg, box_min=sc.box_min,
                             box_max=sc.box_max)
    o.set_frames(sc.cams, sc.rgb, sc.depth, sc.mask, 1, sc.obj_pose)
    objs.append(o)
T.train_many(objs, 2)
o = objs[0]
for i in range(3):
    f = o.frame_at(o.step())
    o.upload_frame(f, np.ascontiguousarray(sc.rgb[f]), np.ascontiguousarray(sc.depth[f]), None)
    print(o.wait_stats(o.train_step_async(1, prefetch_next=True))[0]["total"])
o.synth_frames(sc.cams, sc.boxes, depth_noise=0.01, missing_frac=0.05, seed=2)
o.train_step(2)
v, t, iso = o.extract_mesh(24, iso=0.5)
print("mesh", len(v), len(t), o.get_mesh_grid().shape)
a = np.random.default_rng(1).uniform(0, 1, (300, 3)).astype(np.float32)
print("chamfer", M.chamfer(ctx, a, a[::-1] + 0.01))
ctx.synchronize()
print("sanitize run ok")
