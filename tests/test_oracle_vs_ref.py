"""Pins the C oracle (oracle/prenom_oracle.c) to the reference itself
(oracle/_ref/libnoma_ref.so = the untouched reference sources).

* deterministic reference math -> bit-exact (np.array_equal),
* RNG consumers -> the reference's own mt19937 draws are replayed into the
  oracle, which must then reproduce the reference output bit-exactly,
* build_ray_cdf -> tolerance (det_exp vs glibc exp), bins/flags identical.
"""
import numpy as np
import pytest

from conftest import grad_params, tiny_arch
from paper_2503_01582_b200 import Camera, FieldArch, Pose
from paper_2503_01582_b200 import scenes

pytestmark = pytest.mark.ref

BOX0, BOX1 = np.zeros(3, np.float32), np.ones(3, np.float32)


def big_archs():
    return [scenes.cfg1_arch(), FieldArch(hash_levels=16, features_per_level=2, log2_table_size=12,
                                          base_resolution=16, per_level_scale=scenes.cfg2_arch().per_level_scale,
                                          hidden_width=64, hidden_layers=2)]


def test_param_count_and_level_resolution(oracle, ref, rng):
    for _ in range(30):
        a = tiny_arch(rng, hash_levels=int(rng.integers(1, 9)), log2_table_size=int(rng.integers(0, 11)),
                      hidden_layers=int(rng.integers(1, 4)))
        assert oracle.param_count(a) == ref.param_count(a) == a.param_count()
        for l in range(a.hash_levels):
            assert oracle.level_resolution(a, l) == ref.level_resolution(a, l) == a.level_resolution(l)
    # the per-level scales reach exactly the BASELINE max resolutions.
    assert scenes.cfg1_arch().level_resolution(7) == 256 == ref.level_resolution(scenes.cfg1_arch(), 7)
    assert scenes.cfg2_arch().level_resolution(15) == 1024 == ref.level_resolution(scenes.cfg2_arch(), 15)


def test_vertex_table_row_bit_exact(oracle, ref, rng):
    for a in big_archs() + [tiny_arch(rng) for _ in range(5)]:
        for l in range(a.hash_levels):
            res = a.level_resolution(l)
            for _ in range(20):
                x, y, z = (int(v) for v in rng.integers(0, res + 1, 3))
                assert oracle.vertex_table_row(a, l, x, y, z) == ref.vertex_table_row(a, l, x, y, z)


def test_hash_encode_bit_exact(oracle, ref, rng):
    for a in big_archs() + [tiny_arch(rng) for _ in range(5)]:
        params = ref.init_params(a, 7) * 1000.0
        xyz = rng.uniform(-0.05, 1.05, (64, 3)).astype(np.float32)
        xyz[:4] = [[0, 0, 0], [1, 1, 1], [0.25, 0.5, 0.75], [1, 0, 1]]
        ours, _, _ = oracle.hash_encode(a, params, xyz)
        assert np.array_equal(ours, ref.hash_encode(a, params, xyz))


def test_field_eval_bit_exact(oracle, ref, rng):
    for a in big_archs() + [tiny_arch(rng) for _ in range(6)]:
        params = grad_params(a, rng)
        xyz = rng.uniform(0, 1, (48, 3)).astype(np.float32)
        s1, c1, k1 = oracle.field_eval(a, params, xyz, cache=True)
        s2, c2, k2 = ref.field_eval(a, params, xyz, cache=True)
        assert np.array_equal(k1["features"], k2["features"])
        assert np.array_equal(k1["raw"], k2["raw"])
        assert np.array_equal(s1, s2) and np.array_equal(c1, c2)


def test_field_backward_bit_exact(oracle, ref, rng):
    for a in big_archs()[:1] + [tiny_arch(rng) for _ in range(6)]:
        params = grad_params(a, rng)
        n = 32
        xyz = rng.uniform(0, 1, (n, 3)).astype(np.float32)
        ds = rng.standard_normal(n).astype(np.float32)
        dr = rng.standard_normal((n, 3)).astype(np.float32)
        assert np.array_equal(oracle.field_backward(a, params, xyz, ds, dr), ref.field_backward(a, params, xyz, ds, dr))


def test_adam_bit_exact(oracle, ref, rng):
    n = 4096
    p = rng.standard_normal(n).astype(np.float32)
    m = np.zeros(n, np.float32)
    v = np.zeros(n, np.float32)
    s1 = s2 = 0
    p1, m1, v1 = p.copy(), m.copy(), v.copy()
    p2, m2, v2 = p.copy(), m.copy(), v.copy()
    for _ in range(5):
        g = rng.standard_normal(n).astype(np.float32)
        g[::7] = 0
        p1, m1, v1, s1 = oracle.adam_step(p1, g, m1, v1, s1)
        p2, m2, v2, s2 = ref.adam_step(p2, g, m2, v2, s2)
        assert s1 == s2
        assert np.array_equal(p1, p2) and np.array_equal(m1, m2) and np.array_equal(v1, v2)
    # test_nfcore.cpp:329-336 hand step
    hp, _, _, _ = oracle.adam_step(np.ones(1, np.float32), np.ones(1, np.float32), np.zeros(1, np.float32),
                                   np.zeros(1, np.float32), 0, lr=0.1)
    assert abs(hp[0] - 0.9) < 1e-6


def random_rays(rng, n, inside_frac=0.1):
    o = rng.uniform(-2, 3, (n, 3)).astype(np.float32)
    k = int(n * inside_frac)
    o[:k] = rng.uniform(0.1, 0.9, (k, 3))
    tgt = rng.uniform(0.2, 0.8, (n, 3)).astype(np.float32)
    d = tgt - o
    d[: n // 10] = rng.standard_normal((n // 10, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    d[-3] = [0, 0, 1]
    d[-2] = [1, 0, 0]
    o[-3] = [0.5, 0.5, -1]
    o[-2] = [-1, 5, 0.5]
    return o, d.astype(np.float32)


def test_uniform_samples_bit_exact(oracle, ref, rng):
    o, d = random_rays(rng, 300)
    for i in range(len(o)):
        for n in (1, 4, 32):
            a = oracle.uniform_samples(o[i], d[i], BOX0, BOX1, n)
            b = ref.uniform_samples(o[i], d[i], BOX0, BOX1, n)
            assert a["escaped"] == b["escaped"]
            if not a["escaped"]:
                for k in ("depths", "deltas", "positions", "t_entry", "t_exit"):
                    assert np.array_equal(a[k], b[k]), k
    # test_render.cpp:197-216 known answer
    s = oracle.uniform_samples([0.5, 0.5, -1], [0, 0, 1], BOX0, BOX1, 4)
    assert np.allclose(s["depths"], [1.125, 1.375, 1.625, 1.875], rtol=1e-6)


def test_trilerp_bit_exact(oracle, ref, rng):
    g = rng.uniform(0, 5, (9, 9, 9)).astype(np.float32)
    for p in rng.uniform(-0.1, 1.1, (500, 3)).astype(np.float32):
        assert oracle.trilerp(g, p) == ref.trilerp(g, p)


def test_build_ray_cdf_pinned(oracle, ref, rng):
    """det_exp vs glibc exp: cdf within 1e-6, escape flags identical."""
    o, d = random_rays(rng, 200)
    n_flag_agree = 0
    for i in range(len(o)):
        R = int(rng.integers(2, 12))
        g = (rng.uniform(0, 30, (R, R, R)) * (rng.random() < 0.8)).astype(np.float32)
        st, tp_r, cdf_r = ref.build_ray_cdf(g, o[i], d[i], BOX0, BOX1, 32, 1e-4)
        if st == 2:
            continue
        s = oracle.uniform_samples(o[i], d[i], BOX0, BOX1, 32)
        esc, tp_o, cdf_o = oracle.build_ray_cdf(g, s["deltas"], s["positions"], 1e-4)
        assert esc == (st == 1)
        n_flag_agree += 1
        np.testing.assert_allclose(tp_o, tp_r, rtol=1e-6, atol=1e-12)
        if not esc:
            np.testing.assert_allclose(cdf_o, cdf_r, rtol=1e-6, atol=1e-7)
            assert cdf_o[-1] == 1.0
    assert n_flag_agree > 50


def test_inverse_transform_replay_bit_exact(oracle, ref, rng):
    """Feed the oracle the reference's own mt19937 draws: outputs must match bitwise."""
    o, d = random_rays(rng, 120)
    checked = 0
    for i in range(len(o)):
        R = 6
        g = rng.uniform(0, 40, (R, R, R)).astype(np.float32)
        st, tp, cdf = ref.build_ray_cdf(g, o[i], d[i], BOX0, BOX1, 16, 1e-4)
        if st:
            continue
        nf = int(rng.integers(1, 40))
        r = ref.inverse_transform_sample(o[i], d[i], BOX0, BOX1, 16, cdf, nf, seed=i)
        cs = ref.uniform_samples(o[i], d[i], BOX0, BOX1, 16)
        from oracle.pyoracle import fptr, zeros

        dep, dl, pos = zeros(nf), zeros(nf), zeros(nf, 3)
        oracle.lib.po_inverse_transform_sample(
            fptr(o[i]), fptr(d[i]), fptr(BOX0), fptr(BOX1), float(cs["t_entry"]), float(cs["t_exit"]), 16,
            fptr(cs["depths"]), fptr(cs["deltas"]), fptr(np.ascontiguousarray(cdf)), nf, fptr(r["uniforms"]),
            fptr(dep), fptr(dl), fptr(pos))
        assert np.array_equal(dep, r["depths"]) and np.array_equal(dl, r["deltas"])
        assert np.array_equal(pos, r["positions"])
        checked += 1
    assert checked > 30


def test_sample_ray_uniform_fallback_matches_reference(oracle, ref, rng):
    """test_priorgrid.cpp:229-243: zero grid -> exactly the uniform set."""
    g = np.zeros((8, 8, 8), np.float32)
    a = oracle.sample_ray(g, [0.5, 0.5, -0.5], [0, 0, 1], BOX0, BOX1, 32, 24, 1e-4, seed=3)
    b = ref.sample_ray(g, [0.5, 0.5, -0.5], [0, 0, 1], BOX0, BOX1, 32, 24, 1e-4, seed=3)
    u = ref.uniform_samples([0.5, 0.5, -0.5], [0, 0, 1], BOX0, BOX1, 24)
    for k in ("depths", "deltas", "positions"):
        assert np.array_equal(a[k], b[k]) and np.array_equal(a[k], u[k])


def test_composite_and_backward(oracle, ref, rng):
    for n in (1, 2, 8, 33, 96):
        sg = rng.uniform(0, 20, n).astype(np.float32)
        sg[:: max(1, n // 4)] = 0
        rgb = rng.uniform(0, 1, (n, 3)).astype(np.float32)
        dl = rng.uniform(1e-3, 0.3, n).astype(np.float32)
        dp = np.cumsum(dl).astype(np.float32)
        c1, d1, t1 = oracle.composite(sg, rgb, dl, dp)
        c2, d2, t2 = ref.composite(sg, rgb, dl, dp)
        assert np.array_equal(c1, c2) and d1 == d2 and np.array_equal(t1, t2)
        dc = rng.standard_normal(3).astype(np.float32)
        g1 = oracle.composite_backward(sg, rgb, dl, dp, dc, 0.3)
        g2 = ref.composite_backward(sg, rgb, dl, dp, dc, 0.3)
        assert np.array_equal(g1[0], g2[0]) and np.array_equal(g1[1], g2[1])


def make_batch(rng, n_rays, S):
    kind = (rng.random(n_rays) < 0.3).astype(np.int32)
    esc = (rng.random(n_rays) < 0.1).astype(np.int32)
    cnt = np.where(esc == 1, 0, S)
    off = np.concatenate([[0], np.cumsum(cnt)]).astype(np.int32)
    ns = off[-1]
    dl = rng.uniform(1e-3, 0.1, ns).astype(np.float32)
    dp = np.cumsum(dl).astype(np.float32)
    sg = rng.uniform(0, 30, ns).astype(np.float32)
    rgb = rng.uniform(0, 1, (ns, 3)).astype(np.float32)
    trgb = rng.uniform(0, 1, (n_rays, 3)).astype(np.float32)
    tdep = np.where(rng.random(n_rays) < 0.2, -1.0, rng.uniform(0.5, 2, n_rays)).astype(np.float32)
    return kind, trgb, tdep, esc, off, dl, dp, sg, rgb


def test_batch_loss_replay_bit_exact(oracle, ref, rng):
    for trial in range(5):
        kind, trgb, tdep, esc, off, dl, dp, sg, rgb = make_batch(rng, 40, 12)
        r = ref.batch_loss(kind, trgb, tdep, esc, off, dl, dp, sg, rgb, 0.1, 1e-4, seed=trial)
        o = oracle.batch_loss(kind, trgb, tdep, esc, off, dl, dp, sg, rgb, r["bg_colors"], 0.1, 1e-4)
        assert o["status"] == 0 and r["status"] == 0
        assert np.array_equal(o["terms"], r["terms"])
        assert np.array_equal(o["d_sigma"], r["d_sigma"]) and np.array_equal(o["d_rgb"], r["d_rgb"])


def test_dilation_band_bit_exact(oracle, ref, rng):
    for _ in range(5):
        m = (rng.random((40, 50)) < 0.02).astype(np.uint8)
        m[10:20, 12:30] = 1
        for b in (1, 3, 8):
            assert np.array_equal(oracle.dilation_band(m, 1, b), ref.dilation_band(m, 1, b))


def test_generate_rays_replay_bit_exact(oracle, ref, rng):
    sc = scenes.sphere_scene(n_views=3, res=48, fx=48.0)
    pose = Pose(R=np.array([[0.6, -0.8, 0], [0.8, 0.6, 0], [0, 0, 1]], np.float32), t=np.array([0.1, -0.2, 0.05], np.float32))
    for f in range(3):
        r = ref.generate_rays(sc.cams[f], sc.rgb[f], sc.depth[f], sc.mask[f], 1, pose, 200, 0.25, seed=f)
        # the oracle's pick indices: position of each picked pixel in its list
        m = sc.mask[f]
        obj = np.flatnonzero(m.reshape(-1) == 1)
        band = np.flatnonzero(oracle.dilation_band(m, 1, 8).reshape(-1))
        n_bg = int(np.round(200 * 0.25))
        picks = np.concatenate([np.searchsorted(obj, r["pick_px"][: 200 - n_bg]),
                                np.searchsorted(band, r["pick_px"][200 - n_bg:])]).astype(np.uint32)
        o = oracle.generate_rays(sc.cams[f], sc.rgb[f], sc.depth[f], m, 1, pose, 200, 0.25, 8, picks=picks)
        assert o["status"] == 0
        for k in ("origins", "dirs", "kinds", "target_rgb", "target_depth", "pick_px"):
            assert np.array_equal(o[k], r[k]), k


def test_refresh_grid_bit_exact(oracle, ref, rng):
    a = tiny_arch(rng)
    params = grad_params(a, rng)
    assert np.array_equal(oracle.refresh_grid(a, params, 9), ref.refresh_grid(a, params, 9))


def test_reptile_update_bit_exact(oracle, ref, rng):
    m = rng.standard_normal(1000).astype(np.float32)
    a = rng.standard_normal(1000).astype(np.float32)
    for beta in (0.0, 0.1, 1.0):
        assert np.array_equal(oracle.reptile_update(m, a, beta), ref.reptile_update(m, a, beta))


def test_train_step_matches_reference_loss_curve(oracle, ref):
    """Same math, different RNG: the Philox oracle and the mt19937 reference
    train the same scene; their mean loss over the last steps agrees."""
    from paper_2503_01582_b200 import TrainConfig

    sc = scenes.sphere_scene(n_views=6, res=32, fx=32.0, depth_noise=0.0)
    a = FieldArch(hash_levels=4, features_per_level=2, log2_table_size=10, base_resolution=4,
                  per_level_scale=1.5, hidden_width=16, hidden_layers=1)
    cfg = TrainConfig(rays_per_iter=64, samples_per_ray=16, prior_sampling=0, grid_refresh_every=0)
    theta = ref.init_params(a, 5)
    iters = 150
    _, _, lr, _ = ref.train_object(a, theta, None, 8, sc.cams, sc.rgb, sc.depth, sc.mask, 1, sc.obj_pose,
                                   sc.box_min, sc.box_max, cfg.to_c(), 11, iters)
    ob = oracle.object_create(a, theta, None, 8, 11, cfg.to_c(), sc.box_min, sc.box_max)
    ob.set_frames(sc.cams, sc.rgb, sc.depth, sc.mask, 1, sc.obj_pose)
    lo = np.array([s["total"] for s in ob.train_step(iters)])
    assert lo[-30:].mean() < 0.5 * lo[:10].mean()
    assert lr[-30:, 0].mean() < 0.5 * lr[:10, 0].mean()
    assert abs(lo[-30:].mean() / lr[-30:, 0].mean() - 1) < 0.3
