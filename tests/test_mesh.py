"""Mesh extraction: marching_cubes after the density query,
on the device, against the reference itself (marching_cubes.cpp:125-180 incl.
cleanup_mesh, mesh.cpp:30-54; choose_iso, density_grid.cpp:134-136).

Bar: bit-exact -- identical vertex coordinates, identical triangles in the
identical order (vertices numbered by first use), for grids that exercise
every configuration family, ambiguous faces, values exactly at the iso level
(coincident vertices, zero-area triangles dropped by cleanup_mesh), empty and
full grids. Fixtures: tests/golden/ref_mesh_golden.npz (made by
tests/golden/make_golden_mesh.py from the compiled reference)."""
from pathlib import Path

import numpy as np
import pytest

from mesh_grids import GRIDS

G = np.load(Path(__file__).with_name("golden") / "ref_mesh_golden.npz")
NAMES = list(GRIDS().keys())


# ------------------------------------------------------------------ CPU
def test_case_table_matches_reference_golden():
    """The library's case table (generated from the reference's fixture, scripts/gen_mc_table.py)
    equals cube_case_triangles of the reference for all 256 configurations."""
    from paper_2503_01582_b200 import trainer as T

    counts = []
    for cfg in range(256):
        want = G["case_table"][cfg]
        want = want[want >= 0].reshape(-1, 3)
        got = T.mc_case_triangles(cfg)
        assert np.array_equal(got, want), cfg
        counts.append(len(got))
    assert counts[0] == counts[255] == 0 and max(counts) <= 16


@pytest.mark.ref
def test_golden_mesh_fixtures_match_live_reference(ref):
    for name, (grid, iso) in GRIDS().items():
        assert np.array_equal(G[f"{name}/grid"], grid)
        if iso is None:
            iso = ref.choose_iso(grid)
        assert np.float32(iso) == G[f"{name}/iso"]
        v, t = ref.marching_cubes(grid, iso)
        assert np.array_equal(v, G[f"{name}/vertices"]) and np.array_equal(t, G[f"{name}/triangles"])


def test_golden_meshes_are_nontrivial_and_welded():
    for name in NAMES:
        v, t = G[f"{name}/vertices"], G[f"{name}/triangles"]
        if name in ("empty", "full"):
            assert len(v) == 0 and len(t) == 0
            continue
        assert len(t) > 0
        # first-use numbering: vertex i first appears before vertex i+1
        flat = t.reshape(-1)
        first = np.full(len(v), -1)
        for q, idx in enumerate(flat):
            if first[idx] < 0:
                first[idx] = q
        assert (first >= 0).all() and (np.diff(first) > 0).all()
        assert (v >= 0).all() and (v <= 1).all()


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_cuda_marching_cubes_bit_exact(ctx, name):
    from paper_2503_01582_b200 import trainer as T

    v, t = T.debug_marching_cubes(ctx, G[f"{name}/grid"], float(G[f"{name}/iso"]))
    assert np.array_equal(t, G[f"{name}/triangles"]), name
    assert np.array_equal(v, G[f"{name}/vertices"]), name


@pytest.mark.gpu
def test_cuda_marching_cubes_repeatable_and_reusable(ctx):
    """Scratch re-use across calls (bigger, then smaller grid) does not leak state."""
    from paper_2503_01582_b200 import trainer as T

    a = T.debug_marching_cubes(ctx, G["blob24/grid"], float(G["blob24/iso"]))
    T.debug_marching_cubes(ctx, G["random10/grid"], 5.0)
    b = T.debug_marching_cubes(ctx, G["blob24/grid"], float(G["blob24/iso"]))
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


@pytest.mark.gpu
def test_extract_mesh_equals_reference_tail(ctx, oracle):
    """prenom_extract_mesh == refresh_grid -> choose_iso -> marching_cubes (mapper.cpp:186-187)."""
    from paper_2503_01582_b200 import FieldArch, ObjectTrainer

    a = FieldArch(hash_levels=6, features_per_level=2, log2_table_size=12, base_resolution=4, per_level_scale=1.5,
                  hidden_width=16, hidden_layers=2)
    rng = np.random.default_rng(3)
    theta = (rng.standard_normal(a.param_count()) * 0.3).astype(np.float32)
    nh = a.hash_param_count()
    theta[:nh] = rng.uniform(-1, 1, nh).astype(np.float32)
    theta[-4] = 2.5  # sigma bias: densities around exp(2.5) ~ 12, above the 5.0 iso floor
    obj = ObjectTrainer.create(ctx, a, theta=theta, grid_res=8)
    R = 40
    grid = obj.density_query(R)
    # density query: fp32 field_eval tolerance (device expf / sigmoid are not glibc's bits)
    np.testing.assert_allclose(grid, oracle.refresh_grid(a, theta, R), rtol=1e-6)
    mx = np.float32(grid.max())
    want_iso = max(np.float32(0.5) * mx, np.float32(5.0))
    v, t, iso = obj.extract_mesh(R)
    assert np.float32(iso) == want_iso
    from paper_2503_01582_b200 import trainer as T

    # given the same grid, the mesh is the reference's bit for bit
    from oracle import pyoracle

    if pyoracle.REF_SO.exists():
        ref = pyoracle.Ref()
        assert np.float32(ref.choose_iso(grid)) == want_iso
        wv, wt = ref.marching_cubes(grid, float(want_iso))
    else:
        wv, wt = T.debug_marching_cubes(ctx, grid, float(want_iso))
    assert np.array_equal(v, wv) and np.array_equal(t, wt)
    assert len(t) > 0
    # explicit iso
    v2, t2, iso2 = obj.extract_mesh(R, iso=float(want_iso) * 1.5)
    wv2, wt2 = T.debug_marching_cubes(ctx, grid, float(want_iso) * 1.5)
    assert iso2 == pytest.approx(float(want_iso) * 1.5) and np.array_equal(t2, wt2) and np.array_equal(v2, wv2)
    obj.close()


@pytest.mark.gpu
@pytest.mark.ref
def test_cuda_marching_cubes_matches_reference_at_128(ctx, ref):
    """A 128^3 smooth field with thin features, straight against the compiled reference."""
    from paper_2503_01582_b200 import trainer as T

    R = 128
    ax = np.arange(R, dtype=np.float32) / np.float32(R - 1)
    z, y, x = np.meshgrid(ax, ax, ax, indexing="ij")
    g = (30 * (np.sin(9 * x) * np.cos(7 * y) + np.sin(11 * z + 2 * x)) + 20).astype(np.float32)
    iso = ref.choose_iso(g)
    wv, wt = ref.marching_cubes(g, iso)
    v, t = T.debug_marching_cubes(ctx, g, iso)
    assert np.array_equal(t, wt) and np.array_equal(v, wv)
