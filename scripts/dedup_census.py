"""Census of the backward scatter's atomics on one cfg2 step's samples: per level,
float2 atomics with the kernel's run-level de-duplication (one set of 8 per run
of equal cells in a warp of 32 consecutive samples) vs the ideal vertex-level
de-duplication inside the warp (one per distinct table row) vs merging only the
vertices that consecutive runs share. Sizes the payoff of a vertex-level scheme
before building one. Needs a GPU (the sampler runs through the C ABI)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2503_01582_b200 import Context, ObjectTrainer  # noqa: E402
from paper_2503_01582_b200.trainer import debug_sample_rays  # noqa: E402

args = bench.parse()
ctx = Context(0)
sc, grid, arch, cfg = bench.make_workload(args, 0)
obj = ObjectTrainer.create(ctx, arch, theta=None, grid=grid, seed=7, cfg=cfg, box_min=sc.box_min, box_max=sc.box_max)
obj.set_frames(sc.cams, sc.rgb, sc.depth, sc.mask, 1, sc.obj_pose)
step = 5
r = obj.debug_generate_rays(obj.frame_at(step), step)
g = obj.get_grid()
s = debug_sample_rays(ctx, r["origins"], r["dirs"], sc.box_min, sc.box_max, True, g, cfg.coarse_samples,
                      cfg.samples_per_ray, 1e-4, 7, step)
S = cfg.samples_per_ray
pos = np.clip(s["positions"].reshape(-1, 3), 0.0, 1.0)
valid = np.repeat(s["count"] > 0, S)
n = len(pos) // 32 * 32
pos, valid = pos[:n], valid[:n]
T = arch.log2_table_size
tot = {"run": 0, "pair": 0, "ideal": 0, "hop": 0}
print(f"{n} samples, {valid.mean():.3f} valid")
print("level res dense  run-atomics  pair-merge  ideal   one-hop (per valid sample)")
for l in range(arch.hash_levels):
    res = arch.level_resolution(l)
    V = res + 1
    dense = V ** 3 <= (1 << T)
    c = np.minimum((pos * np.float32(res)).astype(np.int64), res - 1)
    corners = np.array([[(k >> 0) & 1, (k >> 1) & 1, (k >> 2) & 1] for k in range(8)])
    v = c[:, None, :] + corners[None]  # [n, 8, 3]
    if dense:
        rows = v[..., 0] + V * (v[..., 1] + V * v[..., 2])
    else:
        rows = ((v[..., 0] * 1) ^ (v[..., 1] * 2654435761) ^ (v[..., 2] * 805459861)) & ((1 << T) - 1)
    key = (c[:, 2] * res + c[:, 1]) * res + c[:, 0]
    key = np.where(valid, key, -1 - np.arange(n) % 32)
    kw, rw, vw = key.reshape(-1, 32), rows.reshape(-1, 32, 8), valid.reshape(-1, 32)
    head = np.ones_like(kw, bool)
    head[:, 1:] = kw[:, 1:] != kw[:, :-1]
    head &= vw
    run = int(head.sum()) * 8
    ideal = pair = hop = 0
    for w in range(len(kw)):
        hs = np.nonzero(head[w])[0]
        if len(hs) == 0:
            continue
        sets = [set(rw[w, h].tolist()) for h in hs]
        ideal += len(set().union(*sets))
        pair += 8 * len(sets) - sum(len(a & b) for a, b in zip(sets[:-1], sets[1:]))
        # one hop, no chains: head i hands a shared vertex to head i-1 unless
        # head i-1 hands that same vertex on to head i-2
        gives = [set()] + [a & b for a, b in zip(sets[:-1], sets[1:])]  # gives[i]: i -> i-1
        hop += 8 * len(sets) - sum(len(gives[i] - gives[i - 1]) for i in range(1, len(sets)))
    nv = int(valid.sum())
    tot["run"] += run
    tot["pair"] += pair
    tot["ideal"] += ideal
    tot["hop"] += hop
    print(f"{l:5d} {res:4d} {int(dense):5d}  {run / nv:11.3f}  {pair / nv:10.3f}  {ideal / nv:6.3f}  {hop / nv:6.3f}")
nv = int(valid.sum())
print(f"total per valid sample: run {tot['run'] / nv:.2f}  pair {tot['pair'] / nv:.2f}  ideal {tot['ideal'] / nv:.2f}"
      f"  -> pair saves {1 - tot['pair'] / tot['run']:.1%}, ideal {1 - tot['ideal'] / tot['run']:.1%}, "
      f"one-hop {1 - tot['hop'] / tot['run']:.1%}")

# ---- shuffle census of the run reduction (warp-uniform strategy per level-warp)
print("\nshuffles per warp-level: current (pull<=4 else tree) vs best of {pull, tree, per-cell butterfly}")
cur_tot = best_tot = 0
nwl = 0
for l in range(arch.hash_levels):
    res = arch.level_resolution(l)
    c = np.minimum((pos * np.float32(res)).astype(np.int64), res - 1)
    key = (c[:, 2] * res + c[:, 1]) * res + c[:, 0]
    key = np.where(valid, key, -1 - np.arange(n) % 32)
    kw = key.reshape(-1, 32)
    head = np.ones_like(kw, bool)
    head[:, 1:] = kw[:, 1:] != kw[:, :-1]
    cur = best = 0
    for w in range(len(kw)):
        hs = np.nonzero(head[w])[0]
        ends = np.append(hs[1:], 32)
        rmax = int((ends - hs).max())
        pull = 5 * (rmax - 1)
        tree = 16 * int(np.ceil(np.log2(rmax))) if rmax > 1 else 0
        bfly = 18 * len(hs)
        cur += pull if rmax <= 4 else tree
        best += min(pull, tree, bfly)
    cur_tot += cur
    best_tot += best
    nwl += len(kw)
    print(f"{l:5d} cur {cur / len(kw):6.1f}  best {best / len(kw):6.1f}")
print(f"all levels: cur {cur_tot / nwl:.1f} best {best_tot / nwl:.1f} per warp-level")
