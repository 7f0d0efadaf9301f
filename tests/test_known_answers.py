"""Known-answer and property tests of the reference's own suite,
restated and run on BOTH the C oracle (CPU) and the CUDA path (GPU, marked).

Each test cites the reference test it restates. The reference checks its
library against hand arithmetic, a 64-bit "shadow" and product-form oracles;
here the same checks run against the oracle and the CUDA entry points of the
C ABI, with an independent float64 numpy shadow where the reference uses one.

Deliberate difference: the reference's batch_loss draws background colours
from one sequential mt19937 stream, so "escaped rays consume no draws"
(test_render.cpp:453-472) is a property of that stream. The B200 build draws
each ray's colours from a counter-based Philox stream keyed by the ray index,
so no ray's draws depend on any other ray at all; the loss tests below inject
the background colours, as shadow::batch_loss does (shadow.hpp:38-48).
"""
import math

import numpy as np
import pytest

from conftest import grad_params, tiny_arch
from paper_2503_01582_b200 import FieldArch

B0, B1 = np.zeros(3, np.float32), np.ones(3, np.float32)


# --------------------------------------------------------------- backends
class OracleBackend:
    name = "oracle"

    def __init__(self, orc):
        self.o = orc

    def hash_encode(self, arch, params, xyz):
        return self.o.hash_encode(arch, params, np.asarray(xyz, np.float32).reshape(-1, 3))[0]

    def field_eval(self, arch, params, xyz):
        s, c = self.o.field_eval(arch, params, np.asarray(xyz, np.float32).reshape(-1, 3))[:2]
        return s, c

    def field_backward(self, arch, params, xyz, ds, dr):
        return self.o.field_backward(arch, params, np.asarray(xyz, np.float32).reshape(-1, 3),
                                     np.asarray(ds, np.float32), np.asarray(dr, np.float32).reshape(-1, 3))

    def adam(self, p, g, m, v, step, lr):
        return self.o.adam_step(p, g, m, v, step, lr=lr)

    def uniform_samples(self, o, d, n):
        return self.o.uniform_samples(np.float32(o), np.float32(d), B0, B1, n)

    def sample_rays(self, grid, O, D, n_c, n_f, eps=1e-4, seed=0):
        out = []
        for i in range(len(O)):
            r = self.o.sample_ray(grid, np.float32(O[i]), np.float32(D[i]), B0, B1, n_c, n_f, eps, seed=seed,
                                  tag=3, step=0, ray=i)
            out.append(r)
        return out

    def composite(self, sigma, rgb, deltas, depths):
        col, dep, _ = self.o.composite(sigma, rgb, deltas, depths)
        return col, dep

    def batch_loss(self, kind, trgb, tdep, count, S, deltas, depths, sigma, rgb, bg, lambda_d, lambda_sigma):
        esc = (np.asarray(count) == 0).astype(np.int32)
        off = np.concatenate([[0], np.cumsum(count)]).astype(np.int32)
        sel = [np.arange(S) < c for c in count]
        flat = lambda a, k=1: np.concatenate([np.asarray(a, np.float32).reshape(len(count), S, k)[i][sel[i]]
                                              for i in range(len(count))]).reshape(-1, k).squeeze()
        r = self.o.batch_loss(kind, trgb, tdep, esc, off, np.atleast_1d(flat(deltas)), np.atleast_1d(flat(depths)),
                              np.atleast_1d(flat(sigma)), flat(rgb, 3).reshape(-1, 3), bg, lambda_d, lambda_sigma)
        return r["terms"]

    def refresh_grid(self, arch, params, R):
        return self.o.refresh_grid(arch, params, R)


class CudaBackend:
    name = "cuda"

    def __init__(self, ctx):
        from paper_2503_01582_b200 import trainer as T

        self.ctx, self.T = ctx, T

    def hash_encode(self, arch, params, xyz):
        return self.T.debug_hash_encode(self.ctx, arch, params, xyz)

    def field_eval(self, arch, params, xyz):
        s, c, _ = self.T.debug_field_eval(self.ctx, arch, params, xyz, precision=0)
        return s, c

    def field_backward(self, arch, params, xyz, ds, dr):
        return self.T.debug_field_backward(self.ctx, arch, params, xyz, ds, dr)

    def adam(self, p, g, m, v, step, lr):
        return self.T.debug_adam(self.ctx, p, g, m, v, step, lr=lr)

    def uniform_samples(self, o, d, n):
        g = self.T.debug_sample_rays(self.ctx, np.float32([o]), np.float32([d]), B0, B1, False, None, 16, n, 1e-4,
                                     seed=0, step=0)
        return dict(escaped=g["count"][0] == 0, depths=g["depths"][0], deltas=g["deltas"][0],
                    positions=g["positions"][0], t_entry=g["t_entry"][0], t_exit=g["t_exit"][0])

    def sample_rays(self, grid, O, D, n_c, n_f, eps=1e-4, seed=0):
        g = self.T.debug_sample_rays(self.ctx, O, D, B0, B1, True, grid, n_c, n_f, eps, seed=seed, step=0)
        return [dict(escaped=g["count"][i] == 0, depths=g["depths"][i], deltas=g["deltas"][i],
                     positions=g["positions"][i], t_entry=g["t_entry"][i], t_exit=g["t_exit"][i])
                for i in range(len(O))]

    def composite(self, sigma, rgb, deltas, depths):
        n = len(sigma)
        out = self.T.debug_batch_loss(self.ctx, n, [0], [[0.0, 0.0, 0.0]], [-1.0], [n], [deltas], [depths],
                                      [sigma], np.float32(rgb).reshape(1, n, 3), np.zeros((1, 3), np.float32))
        return out["color"][0], out["depth"][0]

    def batch_loss(self, kind, trgb, tdep, count, S, deltas, depths, sigma, rgb, bg, lambda_d, lambda_sigma):
        out = self.T.debug_batch_loss(self.ctx, S, kind, trgb, tdep, count, deltas, depths, sigma,
                                      np.float32(rgb).reshape(len(kind), S, 3), bg, lambda_d, lambda_sigma)
        return out["terms"]

    def refresh_grid(self, arch, params, R):
        from paper_2503_01582_b200 import ObjectTrainer

        obj = ObjectTrainer.create(self.ctx, arch, theta=params, grid_res=8)
        try:
            return obj.density_query(R)
        finally:
            obj.close()


@pytest.fixture(params=["oracle", pytest.param("cuda", marks=pytest.mark.gpu)])
def be(request, oracle):
    if request.param == "oracle":
        return OracleBackend(oracle)
    return CudaBackend(request.getfixturevalue("ctx"))


# ------------------------------------------------------ float64 shadow field
def _res(a, l):
    return max(1, int(a.base_resolution * math.pow(float(np.float32(a.per_level_scale)), l)))


def _row(a, l, x, y, z):
    v = _res(a, l) + 1
    if v ** 3 <= (1 << a.log2_table_size):
        return x + v * (y + v * z)
    return ((x * 1) ^ ((y * 2654435761) & 0xFFFFFFFF) ^ ((z * 805459861) & 0xFFFFFFFF)) & ((1 << a.log2_table_size) - 1)


def shadow_encode(a, params, p):
    """encode_point in float64 (field.cpp:64-99); returns (features, touched rows per level)."""
    L, F, rows = a.hash_levels, a.features_per_level, 1 << a.log2_table_size
    p = np.clip(np.float64(p), 0.0, 1.0)
    feat, touched = np.zeros(L * F), []
    for l in range(L):
        r = _res(a, l)
        g = p * r
        c = np.minimum(g.astype(np.int64), r - 1)
        f = g - c
        tl = set()
        for k in range(8):
            d = ((k >> 0) & 1, (k >> 1) & 1, (k >> 2) & 1)
            w = float(np.prod([f[i] if d[i] else 1 - f[i] for i in range(3)]))
            row = _row(a, l, int(c[0] + d[0]), int(c[1] + d[1]), int(c[2] + d[2]))
            tl.add(row)
            base = l * F * rows + row * F
            feat[l * F:(l + 1) * F] += w * params[base:base + F].astype(np.float64)
        touched.append(tl)
    return feat, touched


def shadow_field(a, params, p, pre_out=None):
    """field_eval in float64 (field.cpp:174-217): (sigma, rgb[3]); pre_out collects the
    hidden pre-activations and the raw outputs."""
    x, _ = shadow_encode(a, params, p)
    off = a.hash_param_count()
    W = a.hidden_width
    n_in = x.size
    for _l in range(a.hidden_layers):
        Wm = np.float64(params[off:off + W * n_in]).reshape(W, n_in)
        off += W * n_in
        b = np.float64(params[off:off + W])
        off += W
        pre = Wm @ x + b
        if pre_out is not None:
            pre_out.extend(pre)
        x = np.maximum(pre, 0.0)
        n_in = W
    Wo = np.float64(params[off:off + 4 * n_in]).reshape(4, n_in)
    bo = np.float64(params[off + 4 * n_in:off + 4 * n_in + 4])
    raw = Wo @ x + bo
    if pre_out is not None:
        pre_out.append(("raw0", raw[0]))
    if a.density_activation == 0:
        sg = min(math.exp(min(raw[0], 10.0)), 1e4)
    else:
        sg = raw[0] + math.log1p(math.exp(-raw[0])) if raw[0] > 0 else math.log1p(math.exp(raw[0]))
    return sg, 1.0 / (1.0 + np.exp(-raw[1:]))


# ---------------------------------------------------------------- encoding
def test_param_count_equals_slot_enumeration(oracle):
    """test_nfcore.cpp:73-106: param_count == an independent enumeration of the layout slots."""
    rng = np.random.default_rng(0)
    for _ in range(50):
        a = FieldArch(hash_levels=int(rng.integers(1, 9)), features_per_level=int(rng.integers(1, 5)),
                      log2_table_size=int(rng.integers(0, 11)), base_resolution=4, per_level_scale=1.5,
                      hidden_width=int(rng.integers(1, 65)), hidden_layers=int(rng.integers(1, 4)))
        slots = a.hash_levels * a.features_per_level * (1 << a.log2_table_size)
        fan = a.hash_levels * a.features_per_level
        for _l in range(a.hidden_layers):
            slots += a.hidden_width * fan + a.hidden_width
            fan = a.hidden_width
        slots += 4 * fan + 4
        assert a.param_count() == slots == oracle.param_count(a)


def test_vertex_feature_equals_table_row(be, oracle):
    """test_nfcore.cpp:121-136: at an exact level-0 lattice vertex the level-0 features are that row."""
    a = FieldArch(hash_levels=2, features_per_level=2, log2_table_size=4, base_resolution=4,
                  per_level_scale=2.0, hidden_width=8, hidden_layers=1)
    p = grad_params(a, np.random.default_rng(5))
    f = be.hash_encode(a, p, [[0.25, 0.5, 0.75]])[0]
    row = oracle.vertex_table_row(a, 0, 1, 2, 3)
    assert f[0] == p[row * 2] and f[1] == p[row * 2 + 1]


def test_encoder_matches_float64_shadow(be):
    """test_nfcore.cpp:138-150: encoder within 1e-5 (relative) of the float64 shadow."""
    rng = np.random.default_rng(7)
    for _ in range(10):
        a = tiny_arch(rng)
        p = grad_params(a, rng)
        x = rng.uniform(0.02, 0.98, (4, 3)).astype(np.float32)
        got = be.hash_encode(a, p, x)
        for i in range(4):
            want, _ = shadow_encode(a, p, x[i])
            np.testing.assert_allclose(got[i], want, rtol=1e-5, atol=1e-7)


def test_encoding_is_continuous(be):
    """test_nfcore.cpp:293-309: a 1e-5 nudge moves every feature by at most 200 * 1e-5."""
    rng = np.random.default_rng(31)
    for _ in range(10):
        a = tiny_arch(rng)
        p = grad_params(a, rng)
        x = rng.uniform(0.1, 0.9, (1, 3)).astype(np.float32)
        q = np.repeat(x, 3, axis=0)
        q[np.arange(3), np.arange(3)] += np.float32(1e-5)
        f = be.hash_encode(a, p, np.concatenate([x, q]))
        assert np.abs(f[1:] - f[0]).max() <= 200 * 1e-5


# ------------------------------------------------------------------- field
def test_field_outputs_in_range(be):
    """test_nfcore.cpp:152-169: sigma >= 0 and rgb in [0, 1] for 3x-scaled random parameters."""
    rng = np.random.default_rng(11)
    for _ in range(8):
        a = tiny_arch(rng)
        p = grad_params(a, rng) * np.float32(3)
        s, c = be.field_eval(a, p, rng.uniform(0, 1, (32, 3)).astype(np.float32))
        assert (s >= 0).all() and (c >= 0).all() and (c <= 1).all()


def test_field_batch_equals_per_point_and_params_untouched(be):
    """test_nfcore.cpp:171-187: batched evaluation == one point at a time; parameters unchanged."""
    rng = np.random.default_rng(13)
    a = tiny_arch(rng)
    p = grad_params(a, rng)
    before = p.copy()
    x = rng.uniform(0, 1, (16, 3)).astype(np.float32)
    s, c = be.field_eval(a, p, x)
    for i in range(16):
        s1, c1 = be.field_eval(a, p, x[i:i + 1])
        assert s1[0] == s[i] and np.array_equal(c1[0], c[i])
    assert np.array_equal(p, before)


def test_field_matches_float64_shadow(be):
    """test_nfcore.cpp:189-202: sigma within 2e-4 and rgb within 2e-5 (relative) of the float64 shadow."""
    rng = np.random.default_rng(17)
    for _ in range(12):
        a = tiny_arch(rng)
        p = grad_params(a, rng)
        x = rng.uniform(0.02, 0.98, (1, 3)).astype(np.float32)
        s, c = be.field_eval(a, p, x)
        ws, wc = shadow_field(a, p, x[0])
        assert s[0] == pytest.approx(ws, rel=2e-4)
        np.testing.assert_allclose(c[0], wc, rtol=2e-5)


# ---------------------------------------------------------------- backward
def test_zero_upstream_gives_zero_gradient(be):
    """test_nfcore.cpp:204-213."""
    rng = np.random.default_rng(19)
    a = tiny_arch(rng)
    g = be.field_backward(a, grad_params(a, rng), [[0.3, 0.6, 0.2]], [0.0], [[0.0, 0.0, 0.0]])
    assert not g.any()


def test_untouched_rows_keep_zero_gradient(be):
    """test_nfcore.cpp:215-240: table rows no corner touched get exactly zero gradient."""
    rng = np.random.default_rng(23)
    a = tiny_arch(rng, log2_table_size=8)
    p = grad_params(a, rng)
    x = np.float32([[0.4, 0.2, 0.7]])
    g = be.field_backward(a, p, x, [1.0], [[0.5, -0.5, 0.25]])
    _, touched = shadow_encode(a, p, x[0])
    rows, F = 1 << a.log2_table_size, a.features_per_level
    tab = g[:a.hash_param_count()].reshape(a.hash_levels, rows, F)
    for l in range(a.hash_levels):
        mask = np.ones(rows, bool)
        mask[list(touched[l])] = False
        assert not tab[l][mask].any()


def clean_point(a, p, rng):
    """A point whose hidden pre-activations are all >= 2e-2 away from the ReLU kink (and, for
    exp-clamped density, raw sigma <= 8.5 away from the clamp): test_nfcore.cpp:47-61."""
    for _ in range(200):
        x = rng.uniform(0.05, 0.95, 3).astype(np.float32)
        pre = []
        shadow_field(a, p, x, pre)
        raw0 = pre.pop()[1]
        if all(abs(v) >= 2e-2 for v in pre) and not (a.density_activation == 0 and raw0 > 8.5):
            return x
    raise AssertionError("no clean evaluation point")


def test_pointwise_gradient_matches_central_differences(be):
    """test_nfcore.cpp:242-279: analytic gradient vs float64 central differences (h = 1e-4), rel < 1e-3."""
    rng = np.random.default_rng(29)
    for _ in range(4):
        a = tiny_arch(rng)
        p = grad_params(a, rng)
        x = clean_point(a, p, rng)
        ds = np.float32(rng.uniform(-1, 1))
        dr = rng.uniform(-1, 1, 3).astype(np.float32)
        g = be.field_backward(a, p, x[None], [ds], dr[None])
        checked = 0
        for i in range(len(p)):
            up, dn = p.copy(), p.copy()
            up[i] = np.float32(np.float64(p[i]) + 1e-4)
            dn[i] = np.float32(np.float64(p[i]) - 1e-4)
            shi, chi = shadow_field(a, up, x)
            slo, clo = shadow_field(a, dn, x)
            phi = lambda s, c: float(ds) * s + float(np.dot(np.float64(dr), c))
            fd = (phi(shi, chi) - phi(slo, clo)) / (np.float64(up[i]) - np.float64(dn[i]))
            if abs(fd) <= 1e-6:
                continue
            checked += 1
            assert abs(g[i] - fd) / abs(fd) < 1e-3, (i, g[i], fd)
        assert checked > 10


# -------------------------------------------------------------------- Adam
def test_adam_zero_gradient_and_zero_lr_leave_params(be):
    """test_nfcore.cpp:311-327."""
    p = np.float32([0.5, -1.25, 3.0])
    z = np.zeros(3, np.float32)
    p1, *_ = be.adam(p, z, z, z, 0, 1e-2)
    assert np.array_equal(p1, p)
    p2, *_ = be.adam(p, np.float32([1.0, -2.0, 0.5]), z, z, 0, 0.0)
    assert np.array_equal(p2, p)


def test_adam_hand_step(be):
    """test_nfcore.cpp:329-336: p=1, g=1, lr=0.1 -> 1 - 0.1/(1+eps) ~ 0.9 after one step."""
    z = np.zeros(1, np.float32)
    p, _, _, step = be.adam(np.float32([1.0]), np.float32([1.0]), z, z, 0, 0.1)
    assert p[0] == pytest.approx(0.9, rel=1e-6) and step == 1


# ----------------------------------------------------------------- samples
def test_uniform_samples_axis_ray_midpoints(be):
    """test_render.cpp:197-216: z-axis ray entering at t=1, exiting at t=2, n=4."""
    s = be.uniform_samples([0.5, 0.5, -1.0], [0.0, 0.0, 1.0], 4)
    assert not s["escaped"]
    want = np.float32([1.125, 1.375, 1.625, 1.875])
    np.testing.assert_allclose(s["depths"], want, rtol=1e-6)
    np.testing.assert_allclose(s["deltas"], 0.25, rtol=1e-6)
    np.testing.assert_allclose(s["positions"][:, :2], 0.5, rtol=1e-6)
    np.testing.assert_allclose(s["positions"][:, 2], want - 1, rtol=1e-5)
    assert s["t_entry"] == pytest.approx(1.0) and s["t_exit"] == pytest.approx(2.0)


def test_uniform_samples_diagonal(be):
    """test_render.cpp:218-237: diagonal ray, n=32: span sqrt(3), equal deltas, positions in the box."""
    d = np.float32([1, 1, 1]) / np.float32(math.sqrt(3))
    s = be.uniform_samples([-0.5, -0.5, -0.5], d, 32)
    assert not s["escaped"]
    span = s["t_exit"] - s["t_entry"]
    assert span == pytest.approx(math.sqrt(3), rel=1e-5)
    np.testing.assert_allclose(s["deltas"], span / 32, rtol=1e-6)
    assert (s["positions"] >= 0).all() and (s["positions"] <= 1).all()


def test_uniform_samples_escape_cases(be):
    """test_render.cpp:239-250: a ray missing the box and one pointing away escape."""
    assert be.uniform_samples([-1.0, 5.0, 0.5], [1.0, 0.0, 0.0], 8)["escaped"]
    assert be.uniform_samples([0.5, 0.5, 2.0], [0.0, 0.0, 1.0], 8)["escaped"]


def test_uniform_samples_origin_inside(be):
    """test_render.cpp:252-263: origin inside the box clamps the span start to 0."""
    s = be.uniform_samples([0.5, 0.5, 0.5], [0.0, 0.0, 1.0], 4)
    assert not s["escaped"] and s["t_entry"] == 0.0 and s["t_exit"] == pytest.approx(0.5)
    np.testing.assert_allclose(s["depths"], [0.0625, 0.1875, 0.3125, 0.4375], rtol=1e-5)


# --------------------------------------------------------------- composite
def test_composite_zero_density(be):
    """test_render.cpp:265-276."""
    col, dep = be.composite(np.zeros(5, np.float32), np.tile(np.float32([0.9, 0.8, 0.7]), (5, 1)),
                            np.full(5, 0.2, np.float32), np.float32([1, 1.2, 1.4, 1.6, 1.8]))
    assert not np.any(col) and dep == 0.0


def test_composite_half_termination(be):
    """test_render.cpp:278-287: sigma * delta = ln 2 terminates with probability 1/2."""
    col, dep = be.composite(np.float32([math.log(2.0)]), np.float32([[0.8, 0.4, 0.2]]), np.float32([1.0]),
                            np.float32([1.7]))
    np.testing.assert_allclose(col, [0.4, 0.2, 0.1], rtol=1e-6)
    assert dep == pytest.approx(0.85, rel=1e-6)


def test_composite_matches_product_form(be):
    """test_render.cpp:289-317 (200 random 8-sample rays) + the mass identity of 319-339."""
    rng = np.random.default_rng(5)
    for _ in range(200):
        sg = rng.uniform(0, 8, 8).astype(np.float32)
        dl = rng.uniform(0.01, 0.4, 8).astype(np.float32)
        dp = (np.float32(rng.uniform(0.5, 1.0)) + np.cumsum(dl)).astype(np.float32)
        c = rng.uniform(0, 1, (8, 3)).astype(np.float32)
        a = 1 - np.exp(-np.float64(sg) * np.float64(dl))
        T = np.concatenate([[1.0], np.cumprod(1 - a)[:-1]])
        rho = T * a
        col, dep = be.composite(sg, c, dl, dp)
        np.testing.assert_allclose(col, rho @ np.float64(c), atol=1e-6)
        assert abs(dep - rho @ np.float64(dp)) < 1e-5
        # white colours: the composited colour is the total termination mass
        wcol, _ = be.composite(sg, np.ones((8, 3), np.float32), dl, dp)
        assert abs(wcol[0] - (1 - np.prod(1 - a))) < 1e-6


def test_composite_order_matters(be):
    """test_render.cpp:341-350: reversing asymmetric densities changes the first sample's weight."""
    red = np.zeros((3, 3), np.float32)
    red[0, 0] = 1.0  # colour.x = rho_0
    dl, dp = np.full(3, 0.3, np.float32), np.float32([1.0, 1.3, 1.6])
    f, _ = be.composite(np.float32([4.0, 0.5, 0.1]), red, dl, dp)
    b, _ = be.composite(np.float32([0.1, 0.5, 4.0]), red, dl, dp)
    assert abs(f[0] - b[0]) > 1e-3


# -------------------------------------------------------------------- loss
def _composite_np(sg, c, dl, dp):
    a = 1 - np.exp(-np.float64(sg) * np.float64(dl))
    T = np.concatenate([[1.0], np.cumprod(1 - a)[:-1]])
    rho = T * a
    return (rho @ np.float64(c)).astype(np.float32), np.float32(rho @ np.float64(dp)), rho.sum()


def test_loss_zero_when_prediction_equals_target(be):
    """test_render.cpp:352-385: targets set to the composited prediction give exactly zero loss."""
    rng = np.random.default_rng(11)
    S, B = 5, 3
    sg = rng.uniform(0, 5, (B, S)).astype(np.float32)
    c = rng.uniform(0, 1, (B, S, 3)).astype(np.float32)
    dl = np.full((B, S), 0.2, np.float32)
    dp = (1 + np.cumsum(dl, axis=1)).astype(np.float32)
    trgb, tdep = np.zeros((B, 3), np.float32), np.zeros(B, np.float32)
    for r in range(B):  # the backend's own composite is the target (bit-identical prediction)
        trgb[r], tdep[r] = be.composite(sg[r], c[r], dl[r], dp[r])
    terms = be.batch_loss(np.zeros(B, np.int32), trgb, tdep, np.full(B, S, np.int32), S, dl, dp, sg, c,
                          np.zeros((B, 3), np.float32), 0.3, 1e-3)
    assert np.array_equal(terms, np.zeros(4))


def test_loss_background_hand_case(be):
    """test_render.cpp:387-410: one background ray, sigma {0.3, 0.7}, lambda_sigma = 1, the colour
    arranged to composite onto the (injected) random target: total = sigma term = 1."""
    bg = np.float32([[0.3, 0.55, 0.8]])
    a1, a2 = 1 - math.exp(-0.3 * 0.25), 1 - math.exp(-0.7 * 0.25)
    mass = a1 + (1 - a1) * a2
    col = (bg[0] / np.float32(mass)).astype(np.float32)
    terms = be.batch_loss([1], [[0, 0, 0]], [-1.0], [2], 2, [[0.25, 0.25]], [[1.0, 1.25]], [[0.3, 0.7]],
                          np.stack([col, col])[None], bg, 0.5, 1.0)
    total, color, depth, sigma = terms
    assert sigma == pytest.approx(1.0, rel=1e-6) and color < 1e-5 and depth == 0.0
    assert total == pytest.approx(1.0, rel=1e-4)


def test_loss_depth_weight_linearity(be):
    """test_render.cpp:412-432: doubling lambda_d adds exactly one more weighted depth term."""
    kw = dict(kind=[0, 0], trgb=[[0.2, 0.3, 0.4]] * 2, tdep=[2.0, 3.0], count=[2, 2], S=2,
              deltas=[[0.5, 0.5]] * 2, depths=[[1.0, 1.5]] * 2, sigma=[[1.2, 0.4]] * 2,
              rgb=np.float32([[[0.9, 0.1, 0.3], [0.2, 0.8, 0.5]]] * 2), bg=np.zeros((2, 3), np.float32))
    base = be.batch_loss(lambda_d=0.25, lambda_sigma=0.0, **kw)
    twice = be.batch_loss(lambda_d=0.5, lambda_sigma=0.0, **kw)
    assert base[2] > 0.1 and twice[2] == base[2]
    assert twice[0] - base[0] == pytest.approx(0.25 * base[2], rel=1e-9)


def test_loss_background_target_depth_ignored(be):
    """test_render.cpp:434-451."""
    kw = dict(kind=[0, 1], trgb=[[0.5, 0.5, 0.5], [0, 0, 0]], count=[2, 2], S=2, deltas=[[0.5, 0.5]] * 2,
              depths=[[1.0, 1.5]] * 2, sigma=[[1.0, 0.5], [0.2, 0.1]],
              rgb=np.float32([[[0.9, 0.1, 0.3], [0.2, 0.8, 0.5]], [[0.4] * 3, [0.6] * 3]]),
              bg=np.float32([[0, 0, 0], [0.1, 0.7, 0.3]]), lambda_d=0.3, lambda_sigma=1e-2)
    a = be.batch_loss(tdep=[2.0, 2.0], **kw)
    b = be.batch_loss(tdep=[2.0, 5.0], **kw)
    assert a[0] == b[0]


# ------------------------------------------------------- grid and sampler (oracle: trilerp/CDF internals)
def test_trilerp_vertices_constant_and_linear(oracle):
    """test_priorgrid.cpp:48-80: exact at vertices, constant grids, linear fields (1e-5)."""
    rng = np.random.default_rng(1)
    g = rng.uniform(0, 10, (5, 5, 5)).astype(np.float32)  # [z][y][x]
    for k in range(5):
        for j in range(5):
            for i in range(5):
                assert oracle.trilerp(g, np.float32([i / 4, j / 4, k / 4])) == g[k, j, i]
    c = np.full((7, 7, 7), 3.25, np.float32)
    for _ in range(50):
        assert oracle.trilerp(c, rng.uniform(0, 1, 3).astype(np.float32)) == pytest.approx(3.25, rel=1e-6)
    r = 9
    ax = np.arange(r, dtype=np.float32) / np.float32(r - 1)
    lin = (2 * ax[None, None, :] + 3 * ax[None, :, None] + 5 * ax[:, None, None]).astype(np.float32)
    for _ in range(100):
        p = rng.uniform(0, 1, 3).astype(np.float32)
        assert oracle.trilerp(lin, p) == pytest.approx(2 * p[0] + 3 * p[1] + 5 * p[2], rel=1e-5, abs=1e-6)


def test_trilerp_continuous_across_cells(oracle):
    """test_priorgrid.cpp:82-96."""
    rng = np.random.default_rng(3)
    g = rng.uniform(0, 20, (8, 8, 8)).astype(np.float32)
    for _ in range(100):
        p = rng.uniform(0.05, 0.95, 3).astype(np.float32)
        ax = int(rng.integers(0, 3))
        p[ax] = np.float32(int(rng.integers(1, 7)) / 7)
        lo, hi = p.copy(), p.copy()
        lo[ax] -= np.float32(1e-6)
        hi[ax] += np.float32(1e-6)
        assert abs(oracle.trilerp(g, lo) - oracle.trilerp(g, hi)) < 1e-3


def _z_coarse(oracle, n):
    return oracle.uniform_samples(np.float32([0.5, 0.5, -0.5]), np.float32([0, 0, 1]), B0, B1, n)


def test_ray_cdf_zero_grid_escapes_and_geometric_case(oracle):
    """test_priorgrid.cpp:98-134: zero grid escapes; constant density 1 gives geometric term probs."""
    cs = _z_coarse(oracle, 16)
    esc, _, _ = oracle.build_ray_cdf(np.zeros((8, 8, 8), np.float32), cs["deltas"], cs["positions"], 1e-4)
    assert esc
    dl = np.full(4, 0.1, np.float32)
    pos = np.float32([[0.5, 0.5, 0.05 + 0.1 * i] for i in range(4)])
    esc, tp, cdf = oracle.build_ray_cdf(np.ones((8, 8, 8), np.float32), dl, pos, 1e-4)
    assert not esc
    rho = 1 - math.exp(-0.1)
    want = np.array([rho * (1 - rho) ** i for i in range(4)])
    np.testing.assert_allclose(tp, want, rtol=1e-6)
    np.testing.assert_allclose(cdf, np.cumsum(np.float64(tp)) / np.float64(tp).sum(), rtol=1e-6)
    assert cdf[3] == 1.0


def test_ray_cdf_monotone_and_escape_iff_mass(oracle):
    """test_priorgrid.cpp:136-158."""
    rng = np.random.default_rng(5)
    cs = _z_coarse(oracle, 12)
    for _ in range(20):
        esc, _, cdf = oracle.build_ray_cdf(rng.uniform(0, 5, (6, 6, 6)).astype(np.float32), cs["deltas"],
                                           cs["positions"], 1e-4)
        if esc:
            continue
        assert (np.diff(cdf) >= 0).all() and cdf[-1] == pytest.approx(1.0, rel=1e-6)
    cs = _z_coarse(oracle, 16)
    c = 1e-6
    while c < 1e-2:
        esc, tp, _ = oracle.build_ray_cdf(np.full((4, 4, 4), c, np.float32), cs["deltas"], cs["positions"], 1e-4)
        assert esc == (np.float64(tp).sum() < 1e-4)
        c *= 1.7


def test_inverse_transform_single_bin_confinement(oracle):
    """test_priorgrid.cpp:160-173: all CDF mass in bin 2 confines every fine sample to that bin."""
    from oracle.pyoracle import fptr, zeros

    cs = _z_coarse(oracle, 8)
    cdf = np.float32([0, 0, 1, 1, 1, 1, 1, 1])
    n = 64
    u = np.random.default_rng(7).uniform(0, 1, 2 * n).astype(np.float32)
    dep, dl, pos = zeros(n), zeros(n), zeros(n, 3)
    o, d = np.float32([0.5, 0.5, -0.5]), np.float32([0, 0, 1])
    oracle.lib.po_inverse_transform_sample(fptr(o), fptr(d), fptr(B0), fptr(B1), float(cs["t_entry"]),
                                           float(cs["t_exit"]), 8, fptr(cs["depths"]), fptr(cs["deltas"]),
                                           fptr(cdf), n, fptr(u), fptr(dep), fptr(dl), fptr(pos))
    lo = cs["depths"][2] - 0.5 * cs["deltas"][2]
    hi = cs["depths"][2] + 0.5 * cs["deltas"][2]
    assert (dep >= lo - 1e-5).all() and (dep <= hi + 1e-5).all()


# -------------------------------------------------- guided sampler (both backends)
def _z_rays(n):
    return np.tile(np.float32([0.5, 0.5, -0.5]), (n, 1)), np.tile(np.float32([0, 0, 1]), (n, 1))


def test_guided_samples_sorted_in_span_with_forward_deltas(be):
    """test_priorgrid.cpp:175-198 (+273-280): deterministic, strictly increasing, inside the span,
    delta_i = d_{i+1} - d_i, positions on the ray."""
    O, D = _z_rays(4)
    g = np.full((6, 6, 6), 2.0, np.float32)
    a = be.sample_rays(g, O, D, 8, 32, seed=11)
    b = be.sample_rays(g, O, D, 8, 32, seed=11)
    for ra, rb in zip(a, b):
        assert not ra["escaped"] and np.array_equal(ra["depths"], rb["depths"])
        d = ra["depths"]
        assert (np.diff(d) > 0).all()
        assert (d >= ra["t_entry"]).all() and (d <= ra["t_exit"]).all()
        np.testing.assert_allclose(ra["deltas"][:-1], np.diff(d), rtol=1e-6)
        np.testing.assert_allclose(ra["positions"][:, 0], 0.5, rtol=1e-6)
        np.testing.assert_allclose(ra["positions"][:, 2], d - 0.5, rtol=1e-5, atol=1e-7)
    s = be.sample_rays(np.full((16, 16, 16), 0.5, np.float32), O[:1], D[:1], 32, 32, seed=23)[0]
    assert not s["escaped"] and len(s["depths"]) == 32 and (np.diff(s["depths"]) > 0).all()


def test_guided_bin_frequencies_chi_square(be, oracle):
    """test_priorgrid.cpp:200-227: fine-sample bin frequencies follow the term probabilities
    (chi-square p > 0.01, 1e5 draws: here 1000 rays x 100 samples, each ray its own Philox stream)."""
    from scipy.stats import chi2

    O, D = _z_rays(1000)
    g = np.ones((6, 6, 6), np.float32)
    rays = be.sample_rays(g, O, D, 8, 100, seed=13)
    cs = _z_coarse(oracle, 8)
    _, tp, _ = oracle.build_ray_cdf(g, cs["deltas"], cs["positions"], 1e-4)
    d = np.concatenate([r["depths"] for r in rays])
    assert d.size == 100000
    edge0, width = cs["depths"][0] - 0.5 * cs["deltas"][0], cs["deltas"][0]
    bins = np.clip(((d - edge0) / width).astype(np.int64), 0, 7)
    counts = np.bincount(bins, minlength=8)
    expect = d.size * np.float64(tp) / np.float64(tp).sum()
    assert (expect > 100).all()
    stat = ((counts - expect) ** 2 / expect).sum()
    assert chi2.sf(stat, 7) > 0.01, (stat, counts, expect)


def test_guided_slab_captures_80_percent(be):
    """test_priorgrid.cpp:245-271: a dense slab z in [0.4, 0.5] draws >= 80% of the guided samples."""
    r = 101
    g = np.zeros((r, r, r), np.float32)
    z = np.arange(r, dtype=np.float32) / np.float32(r - 1)
    g[(z >= np.float32(0.4)) & (z <= np.float32(0.5))] = 50.0
    O, D = _z_rays(100)
    rays = be.sample_rays(g, O, D, 32, 100, seed=19)
    d = np.concatenate([x["depths"] for x in rays])
    assert d.size == 10000
    smear = 1 / (r - 1) + 1 / 32
    assert ((d >= 0.9 - smear) & (d <= 1.0 + smear)).sum() >= 8000


def test_guided_zero_grid_is_uniform(be):
    """test_priorgrid.cpp:229-243: a zero grid falls back to exactly the uniform sample set."""
    O, D = _z_rays(1)
    s = be.sample_rays(np.zeros((8, 8, 8), np.float32), O, D, 32, 24, seed=17)[0]
    u = be.uniform_samples(O[0], D[0], 24)
    assert not s["escaped"]
    assert np.array_equal(s["depths"], u["depths"]) and np.array_equal(s["deltas"], u["deltas"])
    assert np.array_equal(s["positions"], u["positions"])


# ------------------------------------------------------------ density query
def test_refresh_grid_equals_pointwise_eval(be):
    """test_priorgrid.cpp:282-298: vertex (i,j,k)/(R-1) values == field_eval sigma, bit for bit."""
    rng = np.random.default_rng(29)
    a = tiny_arch(rng)
    p = grad_params(a, rng)
    g = be.refresh_grid(a, p, 17)
    assert g.shape == (17, 17, 17)
    ijk = rng.integers(0, 17, (50, 3))
    s, _ = be.field_eval(a, p, (ijk / np.float32(16)).astype(np.float32))
    assert np.array_equal(g[ijk[:, 2], ijk[:, 1], ijk[:, 0]], s)


def test_refresh_grid_constant_for_zero_params_and_full_size(be):
    """test_priorgrid.cpp:300-321: zero parameters -> constant grid; a 64^3 query has 64^3 values."""
    rng = np.random.default_rng(31)
    a = tiny_arch(rng)
    p = np.zeros(a.param_count(), np.float32)
    g = be.refresh_grid(a, p, 8)
    c, _ = be.field_eval(a, p, [[0.3, 0.7, 0.1]])
    assert (g == c[0]).all()
    a1 = FieldArch(hash_levels=1, features_per_level=1, log2_table_size=4, hidden_width=8, hidden_layers=1)
    p1 = (np.random.default_rng(1).standard_normal(a1.param_count()) * 0.1).astype(np.float32)
    assert be.refresh_grid(a1, p1, 64).size == 64 ** 3


# ----------------------------------------------------------------- Reptile
@pytest.mark.gpu
def test_reptile_endpoints_and_exact_interpolation(ctx, oracle):
    """test_metalearn.cpp:112-134: beta 0 / 1 endpoints, the hand case, exact (1-b)*m + b*a."""
    from paper_2503_01582_b200 import ObjectTrainer

    a = FieldArch(hash_levels=1, features_per_level=1, log2_table_size=4, hidden_width=8, hidden_layers=1)
    P = a.param_count()
    rng = np.random.default_rng(11)
    meta_v = rng.uniform(-3, 3, P).astype(np.float32)
    ad_v = rng.uniform(-3, 3, P).astype(np.float32)
    meta = ObjectTrainer.create(ctx, a, theta=meta_v, grid_res=8)
    ad = ObjectTrainer.create(ctx, a, theta=ad_v, grid_res=8)
    for beta, want in ((0.0, meta_v), (1.0, ad_v),
                       (0.37, (np.float32(1 - np.float32(0.37)) * meta_v + np.float32(0.37) * ad_v))):
        meta.set_params(meta_v)
        meta.reptile_update(ad, beta)
        assert np.array_equal(meta.get_params(), want.astype(np.float32))
        assert np.array_equal(oracle.reptile_update(meta_v, ad_v, beta), want.astype(np.float32))
    meta.close()
    ad.close()
