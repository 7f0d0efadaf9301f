"""Phase timeline of the tensor-core backward (k_bwd_tc) on the cfg2 workload: clock64 stamps of
CTA 0's first 64 tiles (MLP issuing thread and first scatter thread), via prenom_debug_bwd_trace.

  PRENOM_BWD_WAIT=8 python scripts/bwd_trace.py [bf16x3|bf16] [out.json]
"""
import ctypes as C
import json
import os
import sys

import numpy as np

os.environ["PRENOM_BWD_WAIT"] = str(int(os.environ.get("PRENOM_BWD_WAIT", "0")) | 8)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2503_01582_b200 import Context, ObjectTrainer  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "bf16x3"
out_path = sys.argv[2] if len(sys.argv) > 2 else None
group = int(os.environ.get("TRACE_GROUP", "0"))  # > 0: that many cfg4 objects through grouped launches
sys.argv = ["bench.py", "--mlp", mode]
args = bench.parse()
ctx = Context(0)
if group:
    from paper_2503_01582_b200 import TrainConfig, scenes
    from paper_2503_01582_b200.trainer import train_many

    objs = []
    for i in range(group):
        sc = scenes.box_union_scene(n_views=20, res=128, seed=7000 + i)
        cfg = TrainConfig(rays_per_iter=4096, samples_per_ray=64, prior_sampling=0, grid_refresh_every=0,
                          mlp_precision=bench.mlp_id(mode))
        o = ObjectTrainer.create(ctx, scenes.cfg4_arch(), theta=None, grid_res=8, seed=1 + i, cfg=cfg,
                                 box_min=sc.box_min, box_max=sc.box_max)
        o.set_frames(sc.cams, sc.rgb, sc.depth, sc.mask, 1, sc.obj_pose)
        objs.append(o)
    ctx.set_grouping(True)
    train_many(objs, 10)
else:
    sc, grid, arch, cfg = bench.make_workload(args, 0)
    o = ObjectTrainer.create(ctx, arch, theta=None, grid=grid, seed=7, cfg=cfg, box_min=sc.box_min, box_max=sc.box_max)
    o.set_frames(sc.cams, sc.rgb, sc.depth, sc.mask, 1, sc.obj_pose)
    o.train_step(20, stats=False)
ctx.synchronize()
mlp = np.zeros((64, 16), np.int64)
sca = np.zeros((64, 4), np.int64)
cta = np.zeros((1024, 5), np.int64)
P64 = C.POINTER(C.c_int64)
ctx.lib.prenom_debug_bwd_trace(ctx.h, mlp.ctypes.data_as(P64), sca.ctypes.data_as(P64), cta.ctypes.data_as(P64))
GHZ = 1.965
names = ["start", "X in", "L0", "L1", "out", "G ready", "dWo+dH1", "dW1+dH0", "dW0+dX", "X re-fetched", "slot free"]
order = [0, 1, 2, 3, 4, 5, 6, 7, 9, 10, 8]
n = 0
while n < 64 and mlp[n, 0] and mlp[n, 8]:
    n += 1
rows = mlp[:n]
res = {"tiles": int(n), "mode": mode, "phase_us": {}, "tile_us": None}
prev = rows[:, 0]
for sl in order[1:]:
    d = (rows[:, sl] - prev) / GHZ / 1e3
    res["phase_us"][names[sl]] = round(float(np.median(d)), 3)
    prev = rows[:, sl]
res["x_in_us_per_tile"] = [round(float(v), 2) for v in (rows[:, 1] - rows[:, 0]) / GHZ / 1e3]
tile = (rows[1:, 0] - rows[:-1, 0]) / GHZ / 1e3
res["tile_us_per_tile"] = [round(float(v), 2) for v in tile]
res["tile_us"] = round(float(np.median(tile)), 3)
ns = 0
while ns < 64 and sca[ns, 0] and sca[ns, 2]:
    ns += 1
s = sca[:ns]
res["scatter_us"] = {"wait_slot_to_release": round(float(np.median((s[:, 1] - s[:, 0]) / GHZ / 1e3)), 3),
                     "scatter": round(float(np.median((s[:, 2] - s[:, 1]) / GHZ / 1e3)), 3),
                     "idle_before_next": round(float(np.median((s[1:, 0] - s[:-1, 2]) / GHZ / 1e3)), 3)}
nc = int(np.sum(cta[:, 3] > 0))
c = cta[:nc]
t0 = c[:, 0].min()
res["ctas"] = {"n": nc, "kernel_us": round((c[:, 3].max() - t0) / 1e3, 2),
               "prologue_us_median": round(float(np.median(c[:, 1] - c[:, 0])) / 1e3, 2),
               "first_entry_to_last_entry_us": round((c[:, 0].max() - t0) / 1e3, 2),
               "loop_end_us": {"min": round((c[:, 2].min() - t0) / 1e3, 2), "median": round(float(np.median(c[:, 2] - t0)) / 1e3, 2),
                               "max": round((c[:, 2].max() - t0) / 1e3, 2)},
               "flush_us_median": round(float(np.median(c[:, 3] - c[:, 2])) / 1e3, 2),
               "tiles_per_cta": {"min": int(c[:, 4].min()), "max": int(c[:, 4].max()), "mean": round(float(c[:, 4].mean()), 2)},
               "tile_us_mean": round(float(np.mean((c[:, 2] - c[:, 1]) / np.maximum(c[:, 4], 1))) / 1e3, 3)}
line = json.dumps(res)
print(line)
if out_path:
    open(out_path, "w").write(line)
