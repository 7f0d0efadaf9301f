"""cfg5 tail on one object: a few train steps, then extract_mesh(256) (density query +
choose_iso + marching cubes); run under ncu for the per-kernel split."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2503_01582_b200 import Context, ObjectTrainer, TrainConfig, scenes  # noqa: E402

ctx = Context(0)
arch = bench.mixed_category_archs()[int(sys.argv[1]) if len(sys.argv) > 1 else 0]
rng = np.random.default_rng(3)
boxes = scenes.random_boxes(rng)
cfg = TrainConfig(rays_per_iter=1366, samples_per_ray=96, coarse_samples=32, prior_sampling=1, grid_refresh_every=50,
                  mlp_precision=1)
o = ObjectTrainer.create(ctx, arch, grid=scenes.occupancy_prior(boxes, R=128), seed=5, cfg=cfg,
                         box_min=np.full(3, -0.5, np.float32), box_max=np.full(3, 0.5, np.float32))
o.synth_frames(scenes.fibonacci_cameras(20, 1.5, 512, 512, 512.0), boxes, 0.01, 0.05, seed=1)
o.train_step(60, stats=False)
ctx.synchronize()
for rep in range(3):
    t = time.perf_counter()
    nt = o.extract_mesh_counts(256)
    ctx.synchronize()
    print(f"extract_mesh(256): {1e3 * (time.perf_counter() - t):.2f} ms, {nt} triangles")
