"""Golden vectors produced by the reference itself (tests/golden/make_golden.py
runs the unmodified reference sources): the C oracle must reproduce them
(CPU), and so must the CUDA path (GPU), without /root/reference present."""
from pathlib import Path

import numpy as np
import pytest

from paper_2503_01582_b200 import FieldArch

G = np.load(Path(__file__).with_name("golden") / "ref_golden.npz")
ARCHS = ["cfg1", "l16w64", "tiny_sp"]
B0, B1 = np.zeros(3, np.float32), np.ones(3, np.float32)


def arch(name):
    v = G[f"{name}/arch"]
    return FieldArch(hash_levels=int(v[0]), features_per_level=int(v[1]), log2_table_size=int(v[2]),
                     base_resolution=int(v[3]), per_level_scale=float(np.float32(v[4])), hidden_width=int(v[5]),
                     hidden_layers=int(v[6]), density_activation=int(v[7]))


# ------------------------------------------------------------------ CPU
@pytest.mark.parametrize("name", ARCHS)
def test_oracle_field_matches_reference_golden(oracle, name):
    a = arch(name)
    p, x = G[f"{name}/params"], G[f"{name}/xyz"]
    f, _, _ = oracle.hash_encode(a, p, x)
    assert np.array_equal(f, G[f"{name}/features"])
    s, c, k = oracle.field_eval(a, p, x, cache=True)
    assert np.array_equal(k["raw"], G[f"{name}/raw"])
    assert np.array_equal(s, G[f"{name}/sigma"]) and np.array_equal(c, G[f"{name}/rgb"])
    g = oracle.field_backward(a, p, x, G[f"{name}/d_sigma"], G[f"{name}/d_rgb"])
    assert np.array_equal(g, G[f"{name}/grad"])
    assert np.array_equal(oracle.refresh_grid(a, p, 9), G[f"{name}/refresh9"])


def test_oracle_samplers_match_reference_golden(oracle):
    from oracle.pyoracle import fptr, zeros

    o, d, grid = G["rays/o"], G["rays/d"], G["rays/grid"]
    for i in range(len(o)):
        u = oracle.uniform_samples(o[i], d[i], B0, B1, 24)
        assert u["escaped"] == bool(G["rays/escaped"][i])
        if not u["escaped"]:
            assert np.array_equal(u["depths"], G["rays/uniform_depths"][i])
        if np.isnan(G["rays/cdf16"][i][0]):
            continue
        cs = oracle.uniform_samples(o[i], d[i], B0, B1, 16)
        esc, _, cdf = oracle.build_ray_cdf(grid, cs["deltas"], cs["positions"], 1e-4)
        assert not esc
        np.testing.assert_allclose(cdf, G["rays/cdf16"][i], rtol=1e-6, atol=1e-7)
        dep, dl, pos = zeros(40), zeros(40), zeros(40, 3)
        ref_cdf = np.ascontiguousarray(G["rays/cdf16"][i])
        oracle.lib.po_inverse_transform_sample(fptr(o[i]), fptr(d[i]), fptr(B0), fptr(B1), float(cs["t_entry"]),
                                               float(cs["t_exit"]), 16, fptr(cs["depths"]), fptr(cs["deltas"]),
                                               fptr(ref_cdf), 40, fptr(np.ascontiguousarray(G["rays/fine_uniforms"][i])),
                                               fptr(dep), fptr(dl), fptr(pos))
        assert np.array_equal(dep, G["rays/fine_depths"][i])
        assert np.array_equal(pos, G["rays/fine_positions"][i])


def test_oracle_loss_and_adam_match_reference_golden(oracle):
    r = oracle.batch_loss(G["loss/kind"], G["loss/target_rgb"], G["loss/target_depth"], G["loss/escaped"],
                          G["loss/offsets"], G["loss/deltas"], G["loss/depths"], G["loss/sigma"], G["loss/rgb"],
                          G["loss/bg_colors"], 0.1, 1e-4)
    assert np.array_equal(r["terms"], G["loss/terms"])
    assert np.array_equal(r["d_sigma"], G["loss/d_sigma"]) and np.array_equal(r["d_rgb"], G["loss/d_rgb"])
    p, m, v, s = G["adam/p0"], np.zeros(257, np.float32), np.zeros(257, np.float32), 0
    for k in range(3):
        p, m, v, s = oracle.adam_step(p, G["adam/grads"][k], m, v, s)
    assert np.array_equal(p, G["adam/p3"]) and np.array_equal(m, G["adam/m3"]) and np.array_equal(v, G["adam/v3"])


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
@pytest.mark.parametrize("name", ARCHS)
def test_cuda_field_matches_reference_golden(ctx, name):
    from paper_2503_01582_b200 import trainer as T

    a = arch(name)
    p, x = G[f"{name}/params"], G[f"{name}/xyz"]
    assert np.array_equal(T.debug_hash_encode(ctx, a, p, x), G[f"{name}/features"])
    s, c, raw = T.debug_field_eval(ctx, a, p, x, precision=0)
    assert np.array_equal(raw, G[f"{name}/raw"])
    np.testing.assert_allclose(s, G[f"{name}/sigma"], rtol=1e-6)
    np.testing.assert_allclose(c, G[f"{name}/rgb"], rtol=1e-6, atol=1e-7)
    g = T.debug_field_backward(ctx, a, p, x, G[f"{name}/d_sigma"], G[f"{name}/d_rgb"])
    ref = G[f"{name}/grad"]
    np.testing.assert_allclose(g, ref, rtol=1e-4, atol=1e-5 * np.abs(ref).max())


@pytest.mark.gpu
def test_cuda_uniform_samples_and_adam_match_reference_golden(ctx):
    from paper_2503_01582_b200 import trainer as T

    o, d = G["rays/o"], G["rays/d"]
    g = T.debug_sample_rays(ctx, o, d, B0, B1, False, None, 16, 24, 1e-4, seed=0, step=0)
    for i in range(len(o)):
        assert (g["count"][i] == 0) == bool(G["rays/escaped"][i])
        if g["count"][i]:
            assert np.array_equal(g["depths"][i], G["rays/uniform_depths"][i])
    p, m, v, s = G["adam/p0"], np.zeros(257, np.float32), np.zeros(257, np.float32), 0
    for k in range(3):
        p, m, v, s = T.debug_adam(ctx, p, G["adam/grads"][k], m, v, s)
    assert np.array_equal(p, G["adam/p3"]) and np.array_equal(m, G["adam/m3"]) and np.array_equal(v, G["adam/v3"])


@pytest.mark.gpu
def test_cuda_batch_loss_matches_reference_golden(ctx):
    from paper_2503_01582_b200 import trainer as T

    S = 12
    esc = G["loss/escaped"]
    B = len(esc)
    cnt = np.where(esc == 1, 0, S).astype(np.int32)
    # re-pack the flat per-sample arrays into B x S slots
    dl, dp, sg, rgb = (np.zeros((B, S), np.float32) for _ in range(4))
    rgb = np.zeros((B, S, 3), np.float32)
    off = G["loss/offsets"]
    for r in range(B):
        if cnt[r]:
            sl = slice(off[r], off[r + 1])
            dl[r], dp[r], sg[r], rgb[r] = G["loss/deltas"][sl], G["loss/depths"][sl], G["loss/sigma"][sl], G["loss/rgb"][sl]
    out = T.debug_batch_loss(ctx, S, G["loss/kind"], G["loss/target_rgb"], G["loss/target_depth"], cnt, dl, dp, sg,
                             rgb, np.nan_to_num(G["loss/bg_colors"]))
    np.testing.assert_allclose(out["terms"], G["loss/terms"], rtol=1e-9)
    valid = np.repeat(cnt > 0, S)
    np.testing.assert_allclose(out["d_sigma"][valid], G["loss/d_sigma"], rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(out["d_rgb"][valid], G["loss/d_rgb"], rtol=1e-5, atol=1e-7)
