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
print("sanitize run ok")
