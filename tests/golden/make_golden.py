"""Generate tests/golden/ref_golden.npz from the REFERENCE ITSELF.

Runs the unmodified reference sources (oracle/_ref/libnoma_ref.so, built by
oracle/Makefile from /root/reference/proj/core/src) on small seeded inputs
and stores inputs + outputs. tests/test_golden.py checks the C oracle and
(on a GPU box) the CUDA path against these fixtures, so the pin survives
where /root/reference is absent. Re-run: python tests/golden/make_golden.py
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import pyoracle  # noqa: E402
from paper_2503_01582_b200 import FieldArch  # noqa: E402

ARCHS = {
    "cfg1": dict(hash_levels=8, features_per_level=2, log2_table_size=13, base_resolution=16,
                 per_level_scale=1.4859943389892578, hidden_width=32, hidden_layers=2, density_activation=0),
    "l16w64": dict(hash_levels=16, features_per_level=2, log2_table_size=12, base_resolution=16,
                   per_level_scale=1.3195079565048218, hidden_width=64, hidden_layers=2, density_activation=0),
    "tiny_sp": dict(hash_levels=3, features_per_level=1, log2_table_size=6, base_resolution=3,
                    per_level_scale=1.5, hidden_width=8, hidden_layers=1, density_activation=1),
}


def main():
    pyoracle.build_oracle(ref=True)
    ref = pyoracle.Ref()
    rng = np.random.default_rng(20261019)
    out = {}
    for name, kw in ARCHS.items():
        a = FieldArch(**kw)
        out[f"{name}/arch"] = np.array([kw[k] for k in ("hash_levels", "features_per_level", "log2_table_size",
                                                        "base_resolution", "per_level_scale", "hidden_width",
                                                        "hidden_layers", "density_activation")], np.float64)
        params = ref.init_params(a, 11)  # noma::init_params (field.cpp:150-166)
        nh = a.hash_param_count()
        params[:nh] *= 2000.0  # O(0.2) table entries so features are not ~1e-4
        xyz = rng.uniform(-0.02, 1.02, (96, 3)).astype(np.float32)
        xyz[:3] = [[0, 0, 0], [1, 1, 1], [0.25, 0.5, 0.75]]
        sg, rgb, cache = ref.field_eval(a, params, xyz, cache=True)
        ds = rng.standard_normal(96).astype(np.float32)
        dr = rng.standard_normal((96, 3)).astype(np.float32)
        out[f"{name}/params"] = params
        out[f"{name}/xyz"] = xyz
        out[f"{name}/features"] = ref.hash_encode(a, params, xyz)
        out[f"{name}/raw"] = cache["raw"]
        out[f"{name}/sigma"] = sg
        out[f"{name}/rgb"] = rgb
        out[f"{name}/d_sigma"] = ds
        out[f"{name}/d_rgb"] = dr
        out[f"{name}/grad"] = ref.field_backward(a, params, xyz, ds, dr)
        out[f"{name}/refresh9"] = ref.refresh_grid(a, params, 9)
    # samplers (render.cpp:104-132, density_grid.cpp:20-117)
    o = rng.uniform(-1.5, 2.5, (64, 3)).astype(np.float32)
    d = (rng.uniform(0.2, 0.8, (64, 3)) - o)
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    d = d.astype(np.float32)
    b0, b1 = np.zeros(3, np.float32), np.ones(3, np.float32)
    grid = (rng.uniform(0, 50, (10, 10, 10)) * (rng.random((10, 10, 10)) < 0.4)).astype(np.float32)
    us_d, us_esc, cdf_all, fine_d, fine_u, fine_pos = [], [], [], [], [], []
    for i in range(64):
        u = ref.uniform_samples(o[i], d[i], b0, b1, 24)
        us_esc.append(u["escaped"])
        us_d.append(u["depths"])
        st, tp, cdf = ref.build_ray_cdf(grid, o[i], d[i], b0, b1, 16, 1e-4)
        cdf_all.append(cdf if st == 0 else np.full(16, np.nan, np.float32))
        if st == 0:
            r = ref.inverse_transform_sample(o[i], d[i], b0, b1, 16, cdf, 40, seed=i)
            fine_d.append(r["depths"])
            fine_u.append(r["uniforms"])
            fine_pos.append(r["positions"])
        else:
            fine_d.append(np.full(40, np.nan, np.float32))
            fine_u.append(np.full(80, np.nan, np.float32))
            fine_pos.append(np.full((40, 3), np.nan, np.float32))
    out.update({"rays/o": o, "rays/d": d, "rays/grid": grid, "rays/uniform_depths": np.array(us_d),
                "rays/escaped": np.array(us_esc), "rays/cdf16": np.array(cdf_all), "rays/fine_depths": np.array(fine_d),
                "rays/fine_uniforms": np.array(fine_u), "rays/fine_positions": np.array(fine_pos)})
    # compositing + loss (render.cpp:134-243) with the reference's own background draws
    B, S = 24, 12
    kind = (rng.random(B) < 0.3).astype(np.int32)
    esc = (rng.random(B) < 0.1).astype(np.int32)
    cnt = np.where(esc == 1, 0, S)
    off = np.concatenate([[0], np.cumsum(cnt)]).astype(np.int32)
    ns = off[-1]
    dl = rng.uniform(1e-3, 0.1, ns).astype(np.float32)
    dp = np.cumsum(dl).astype(np.float32)
    sgm = rng.uniform(0, 30, ns).astype(np.float32)
    col = rng.uniform(0, 1, (ns, 3)).astype(np.float32)
    trgb = rng.uniform(0, 1, (B, 3)).astype(np.float32)
    tdep = np.where(rng.random(B) < 0.2, -1.0, rng.uniform(0.5, 2, B)).astype(np.float32)
    bl = ref.batch_loss(kind, trgb, tdep, esc, off, dl, dp, sgm, col, 0.1, 1e-4, seed=77)
    out.update({"loss/kind": kind, "loss/escaped": esc, "loss/offsets": off, "loss/deltas": dl, "loss/depths": dp,
                "loss/sigma": sgm, "loss/rgb": col, "loss/target_rgb": trgb, "loss/target_depth": tdep,
                "loss/bg_colors": bl["bg_colors"], "loss/terms": bl["terms"], "loss/d_sigma": bl["d_sigma"],
                "loss/d_rgb": bl["d_rgb"]})
    # Adam (field.cpp:295-310), three steps
    p = rng.standard_normal(257).astype(np.float32)
    m = np.zeros(257, np.float32)
    v = np.zeros(257, np.float32)
    gs = rng.standard_normal((3, 257)).astype(np.float32)
    gs[:, ::5] = 0
    pp, mm, vv, st = p, m, v, 0
    for k in range(3):
        pp, mm, vv, st = ref.adam_step(pp, gs[k], mm, vv, st)
    out.update({"adam/p0": p, "adam/grads": gs, "adam/p3": pp, "adam/m3": mm, "adam/v3": vv})
    np.savez_compressed(Path(__file__).with_name("ref_golden.npz"), **out)
    print("wrote", Path(__file__).with_name("ref_golden.npz"), len(out), "arrays")


if __name__ == "__main__":
    main()
