"""North-star evidence at a BASELINE config's full size: loss after N steps, GPU MLP modes vs the
CPU oracle on the same seeded inputs, θ and Philox draws.

  python scripts/loss_parity.py cfg1 200                       (oracle single-threaded, ~4 min)
  PO_THREADS=16 python scripts/loss_parity.py cfg2 200         (oracle threaded, see prenom_oracle.c)
  python scripts/loss_parity.py cfg2 200 --oracle-cache profiles/r1/loss_parity_cfg2.json \
      --modes fp32,bf16,bf16x3,x3m1,x3m2,x3m4 --repeats 2 --tag r2a

Modes: fp32 (SIMT), bf16, bf16x3 (split bf16, all products split), x3m<mask> (split bf16 with
only the PRENOM_SPLIT_MASK bits <mask> of the cross products enabled: 1 forward, 2 backward data
products, 4 weight gradients; run in a child process because the mask is read once per process).
--oracle-cache takes the oracle's per-step curve from an earlier run's JSON (the oracle is
deterministic at a fixed PO_THREADS). Writes profiles/loss_parity_<cfg>[_<tag>].json."""
import argparse
import json
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

ap = argparse.ArgumentParser()
ap.add_argument("which", nargs="?", default="cfg1")
ap.add_argument("steps", nargs="?", type=int, default=200)
ap.add_argument("--modes", default="fp32,bf16,bf16x3")
ap.add_argument("--repeats", type=int, default=1)
ap.add_argument("--oracle-cache", default=None)
ap.add_argument("--tag", default="")
ap.add_argument("--child", default=None, help=argparse.SUPPRESS)  # internal: one GPU mode, curve to stdout
args = ap.parse_args()
STEPS = args.steps

from paper_2503_01582_b200 import Context, ObjectTrainer, TrainConfig, scenes  # noqa: E402


def workload(which):
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
    return sc, arch, grid, kw, desc, theta


sc, arch, grid, kw, desc, theta = workload(args.which)
MODE_ID = {"fp32": 0, "bf16": 1, "bf16x3": 2}


def run_gpu(mlp):
    ctx = Context(0)
    cfg = TrainConfig(mlp_precision=mlp, **kw)
    o = ObjectTrainer.create(ctx, arch, theta=theta, grid=grid, seed=0, cfg=cfg, box_min=sc.box_min, box_max=sc.box_max)
    o.set_frames(sc.cams, sc.rgb, sc.depth, sc.mask, 1, sc.obj_pose)
    t = time.perf_counter()
    curve = [s["total"] for s in o.train_step(STEPS)]
    dt = time.perf_counter() - t
    o.close()
    return curve, dt


if args.child:
    curve, dt = run_gpu(MODE_ID[args.child])
    print(json.dumps({"curve": curve, "s": dt}))
    sys.exit(0)

out = {"config": f"{desc}, Adam 1e-2, {STEPS} steps, seed 0", "steps": STEPS}
last = lambda c: float(np.mean(c[-20:]))  # noqa: E731
if args.oracle_cache:
    cache = json.loads(Path(args.oracle_cache).read_text())
    out["oracle"] = cache["oracle"][:STEPS]
    out["oracle_from"] = args.oracle_cache
    out["oracle_threads"] = cache.get("oracle_threads", 1)
else:
    from oracle import pyoracle  # noqa: E402  (checker only)
    orc = pyoracle.Oracle()
    ob = orc.object_create(arch, theta, grid, grid.shape[0], 0, TrainConfig(**kw).to_c(), sc.box_min, sc.box_max)
    ob.set_frames(sc.cams, sc.rgb, sc.depth, sc.mask, 1, sc.obj_pose)
    t = time.perf_counter()
    out["oracle"] = [s["total"] for s in ob.train_step(STEPS)]
    out["oracle_s"] = time.perf_counter() - t
    out["oracle_threads"] = int(os.environ.get("PO_THREADS", "1"))
ref = last(out["oracle"])
out["ratios"] = {}
for mode in args.modes.split(","):
    for r in range(args.repeats):
        name = f"gpu_{mode}" + (f"_{r}" if args.repeats > 1 else "")
        env = dict(os.environ)
        child = mode
        if mode.startswith("x3m"):
            env["PRENOM_SPLIT_MASK"] = mode[3:]
            child = "bf16x3"
        res = subprocess.run([sys.executable, __file__, args.which, str(STEPS), "--child", child], env=env,
                             capture_output=True, text=True, check=True)
        d = json.loads(res.stdout.strip().splitlines()[-1])
        out[name] = d["curve"]
        out[name + "_s"] = d["s"]
        out["ratios"][name] = last(d["curve"]) / ref
        out.setdefault("first_step_rel_diff", {})[name] = abs(d["curve"][0] - out["oracle"][0]) / out["oracle"][0]
        print(name, out["ratios"][name], flush=True)
out["final_loss_mean_last20_oracle"] = ref
fn = ROOT / "profiles" / (f"loss_parity_{args.which}" + (f"_{args.tag}" if args.tag else "") + ".json")
fn.write_text(json.dumps(out))
print(json.dumps({k: v for k, v in out.items() if not isinstance(v, list)}, indent=1))
