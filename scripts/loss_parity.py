"""North-star evidence at a BASELINE config's full size: loss after N steps, GPU (fp32 and
bf16 MLP) vs the CPU oracle on the same seeded inputs, θ and Philox draws.

  python scripts/loss_parity.py cfg1 200     (~4 min: single-threaded oracle)
  PO_THREADS=16 python scripts/loss_parity.py cfg2 200   (oracle threaded, see prenom_oracle.c)

Writes profiles/loss_parity_<cfg>.json."""
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from oracle import pyoracle  # noqa: E402
from paper_2503_01582_b200 import Context, ObjectTrainer, TrainConfig, scenes  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
STEPS = int(sys.argv[2]) if len(sys.argv) > 2 else 200
if which == "cfg1":
    sc = scenes.sphere_scene()
    arch = scenes.cfg1_arch()
    grid = np.zeros((8, 8, 8), np.float32)
    kw = dict(rays_per_iter=4096, samples_per_ray=64, prior_sampling=0, grid_refresh_every=0)
    desc = "cfg1 full size: sphere, 24 views 128^2, L8 T2^15 W32 H2, 4096 rays x 64 midpoints"
else:
    sc = scenes.box_union_scene(n_views=50, res=256, seed=1000)
    arch = scenes.cfg2_arch(64)
    grid = scenes.occupancy_prior(sc.boxes, R=32)
    kw = dict(rays_per_iter=8192, samples_per_ray=96, coarse_samples=32, prior_sampling=1, grid_refresh_every=50)
    desc = ("cfg2 full size: box union, 50 views 256^2, 32^3 prior, L16 T2^19 W64 H2, 8192 rays x 32 -> 96 "
            "prior samples, refresh every 50")
rng = np.random.default_rng(0)
P, nh = arch.param_count(), arch.hash_param_count()
theta = np.empty(P, np.float32)
theta[:nh] = rng.uniform(-1e-4, 1e-4, nh)  # BASELINE: tables U(-1e-4, 1e-4)
theta[nh:] = (rng.standard_normal(P - nh) * np.sqrt(2.0 / arch.hidden_width)).astype(np.float32)
R = grid.shape[0]
out = {"config": f"{desc}, Adam 1e-2, {STEPS} steps, seed 0", "steps": STEPS,
       "oracle_threads": int(os.environ.get("PO_THREADS", "1"))}
ctx = Context(0)
for name, mlp in (("gpu_fp32", 0), ("gpu_bf16", 1)):
    cfg = TrainConfig(mlp_precision=mlp, **kw)
    o = ObjectTrainer.create(ctx, arch, theta=theta, grid=grid, seed=0, cfg=cfg, box_min=sc.box_min, box_max=sc.box_max)
    o.set_frames(sc.cams, sc.rgb, sc.depth, sc.mask, 1, sc.obj_pose)
    t = time.perf_counter()
    out[name] = [s["total"] for s in o.train_step(STEPS)]
    out[name + "_s"] = time.perf_counter() - t
    o.close()
orc = pyoracle.Oracle()
ob = orc.object_create(arch, theta, grid, R, 0, TrainConfig(**kw).to_c(), sc.box_min, sc.box_max)
ob.set_frames(sc.cams, sc.rgb, sc.depth, sc.mask, 1, sc.obj_pose)
t = time.perf_counter()
out["oracle"] = [s["total"] for s in ob.train_step(STEPS)]
out["oracle_s"] = time.perf_counter() - t
last = lambda k: float(np.mean(out[k][-20:]))  # noqa: E731
out["final_loss_mean_last20"] = {k: last(k) for k in ("oracle", "gpu_fp32", "gpu_bf16")}
out["ratio_fp32_vs_oracle"] = last("gpu_fp32") / last("oracle")
out["ratio_bf16_vs_oracle"] = last("gpu_bf16") / last("oracle")
out["first_step_rel_diff_fp32"] = abs(out["gpu_fp32"][0] - out["oracle"][0]) / out["oracle"][0]
(ROOT / "profiles" / f"loss_parity_{which}.json").write_text(json.dumps(out))
print(json.dumps({k: v for k, v in out.items() if not isinstance(v, list)}, indent=1))
