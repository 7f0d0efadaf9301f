"""Multi-object scheduler modes: K objects of one arch trained by prenom_train_step_many with
per-object launches on lane streams (grouping off) and with grouped launches (one launch per
stage for all K), against ONE object carrying K times the rays (--same-state: and K times the
table, i.e. the parameter / Adam state of K objects).

    python scripts/group_probe.py [--arch cfg4|cfg3a] [--k 1 2 4 8] [--steps 64]

Wall clock around ctx.synchronize() (host enqueue is ~20 us/step, far below the device time).
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2503_01582_b200 import Context, FieldArch, ObjectTrainer, TrainConfig, scenes  # noqa: E402
from paper_2503_01582_b200._capi import MLP_BF16X3  # noqa: E402
from paper_2503_01582_b200.trainer import train_many  # noqa: E402


def arch_of(name):
    if name == "cfg4":
        return scenes.cfg4_arch(), 4096, 64
    if name == "cfg1":
        return scenes.cfg1_arch(), 4096, 64
    if name == "cfg3a":  # the largest cfg3 category
        return FieldArch(hash_levels=12, features_per_level=2, log2_table_size=19, base_resolution=16,
                         per_level_scale=1.5, hidden_width=32, hidden_layers=1), 2048, 64
    raise SystemExit(name)


def make(ctx, arch, rays, S, seed):
    sc = scenes.box_union_scene(n_views=20, res=128, seed=seed)
    cfg = TrainConfig(rays_per_iter=rays, samples_per_ray=S, prior_sampling=0, grid_refresh_every=0,
                      mlp_precision=MLP_BF16X3 if not os.environ.get('PROBE_BF16') else 1)
    o = ObjectTrainer.create(ctx, arch, theta=None, grid_res=8, seed=seed, cfg=cfg, box_min=sc.box_min,
                             box_max=sc.box_max)
    o.set_frames(sc.cams, sc.rgb, sc.depth, sc.mask, 1, sc.obj_pose)
    return o


def timed(fn, steps):
    fn(4)
    ctx.synchronize()
    t0 = time.perf_counter()
    fn(steps)
    ctx.synchronize()
    return time.perf_counter() - t0


def kernel_times(ctx, fn, steps):
    """Per-stage device time (prenom_ctx_profile: serial launches, CUDA events per launch)."""
    import ctypes as C
    lib = ctx.lib
    fn(2)
    ctx.synchronize()
    lib.prenom_ctx_profile(ctx.h, 1)
    fn(steps)
    kms, kn = (C.c_double * 7)(), (C.c_int64 * 7)()
    lib.prenom_ctx_kernel_times(ctx.h, kms, kn)
    lib.prenom_ctx_profile(ctx.h, 0)
    names = ["sample", "fwd", "composite", "mlp_bwd", "encode_bwd", "adam", "refresh"]
    return {names[i]: (round(kms[i] / steps, 4), kn[i]) for i in range(7) if kn[i]}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--arch", default="cfg4")
    ap.add_argument("--k", type=int, nargs="+", default=[1, 2, 4, 8])
    ap.add_argument("--steps", type=int, default=64)
    ap.add_argument("--kernels", action="store_true", help="per-stage device times (serialised)")
    ap.add_argument("--same-state", action="store_true",
                    help="give the one big object k times the table (the parameter/Adam state of k objects)")
    args = ap.parse_args()
    ctx = Context(0)
    arch, rays, S = arch_of(args.arch)
    res = []
    for k in args.k:
        objs = [make(ctx, arch, rays, S, 100 + i) for i in range(k)]
        if k == 1:
            t = timed(lambda n: objs[0].train_step(n, stats=False), args.steps)
            tg = t
        else:
            ctx.set_grouping(False)
            t = timed(lambda n: train_many(objs, n), args.steps)
            ctx.set_grouping(True)
            tg = timed(lambda n: train_many(objs, n), args.steps)
        import dataclasses, math
        barch = dataclasses.replace(arch, log2_table_size=arch.log2_table_size + int(math.log2(k))) if args.same_state else arch
        big = make(ctx, barch, rays * k, S, 999)
        tb = timed(lambda n: big.train_step(n, stats=False), args.steps)
        n = k * rays * S * args.steps
        row = {"arch": args.arch, "k": k, "lanes_samples_per_s": n / t, "grouped_samples_per_s": n / tg,
               "one_object_samples_per_s": n / tb, "lanes_ms_per_step": 1e3 * t / args.steps,
               "grouped_ms_per_step": 1e3 * tg / args.steps, "one_object_ms_per_step": 1e3 * tb / args.steps}
        if args.kernels and k > 1:
            ctx.set_grouping(False)
            row["kernels_lanes_ms_per_step"] = kernel_times(ctx, lambda n: train_many(objs, n), args.steps)
            ctx.set_grouping(True)
            row["kernels_grouped_ms_per_step"] = kernel_times(ctx, lambda n: train_many(objs, n), args.steps)
        print(json.dumps(row), flush=True)
        res.append(row)
        for o in objs + [big]:
            o.close()
