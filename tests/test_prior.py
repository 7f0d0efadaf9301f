"""Category priors: the PriorBundle container
(prior_bundle.cpp:103-220) and bake_prior (density_grid.cpp:138-143).

CPU: our save_prior / load_prior / prior_summary against the reference's own
file (tests/golden/ref_prior_golden.noma, written by the reference's
save_prior) and, with oracle/_ref built, against the reference reading our
files and rejecting the same malformed files with the same messages.
GPU: bake_prior on the device == the reference's bake_prior, bit for bit;
ObjectTrainer.from_prior trains.
"""
import struct
from pathlib import Path

import numpy as np
import pytest

from prior_cases import golden_bundle_inputs

GOLDEN = Path(__file__).resolve().parent / "golden" / "ref_prior_golden.noma"


def _bundle():
    from paper_2503_01582_b200 import prior as PR

    arch, theta, grid, verts, tris, prov = golden_bundle_inputs()
    gi, gf = prov["genome_ints"], prov["genome_floats"]
    g = PR.Genome(hash_levels=gi[0], log2_table_size=gi[1], features_per_level=gi[2], hidden_width=gi[3],
                  hidden_layers=gi[4], meta_steps=gi[5], inner_iters=gi[6], density_activation=gi[7],
                  eta=float(np.float32(gf[0])), beta=float(np.float32(gf[1])),
                  per_level_scale=float(np.float32(gf[2])), lambda_d=float(np.float32(gf[3])),
                  lambda_sigma=float(np.float32(gf[4])))
    return PR.PriorBundle(arch=arch, theta=theta, grid=grid, vertices=verts, triangles=tris,
                          category=prov["category"], search_seed=prov["search_seed"],
                          population=prov["population"], generations=prov["generations"], genome=g)


# ---------------------------------------------------------------- CPU
def test_load_reference_golden_file():
    from paper_2503_01582_b200 import prior as PR

    want = _bundle()
    b = PR.load_prior(GOLDEN)
    assert b.category == want.category and b.format_version == 1
    assert b.arch == want.arch
    assert (b.search_seed, b.population, b.generations) == (want.search_seed, want.population, want.generations)
    assert b.genome == want.genome
    assert np.array_equal(b.theta, want.theta)
    assert np.array_equal(b.grid, want.grid)
    assert np.array_equal(b.vertices, want.vertices)
    assert np.array_equal(b.triangles, want.triangles)


def test_save_is_byte_identical_to_reference(tmp_path):
    from paper_2503_01582_b200 import prior as PR

    out = tmp_path / "ours.noma"
    PR.save_prior(_bundle(), out)
    assert out.read_bytes() == GOLDEN.read_bytes()
    # and a load -> save round trip is the identity (prior_bundle.hpp:34-36)
    out2 = tmp_path / "again.noma"
    PR.save_prior(PR.load_prior(out), out2)
    assert out2.read_bytes() == GOLDEN.read_bytes()


def test_summary_matches_reference_text():
    from paper_2503_01582_b200 import prior as PR

    assert PR.prior_summary(GOLDEN) == GOLDEN.with_suffix(".summary.txt").read_text()


def test_save_rejects_mismatched_payloads(tmp_path):
    from paper_2503_01582_b200 import DataError
    from paper_2503_01582_b200 import prior as PR

    b = _bundle()
    b.theta = b.theta[:-1]
    with pytest.raises(DataError, match="parameter count does not match"):
        PR.save_prior(b, tmp_path / "x.noma")
    b = _bundle()
    b.grid = b.grid.reshape(-1)[:-1]
    with pytest.raises(DataError, match="grid payload does not match"):
        PR.save_prior(b, tmp_path / "x.noma")


def _corruptions(data: bytes):
    """(name, bytes) malformed variants of a valid bundle (prior_bundle.cpp:141-197 checks)."""
    hlen = struct.unpack_from("<I", data, 6)[0]
    off_theta = 10 + hlen
    header = data[10:10 + hlen].decode()
    yield "magic", b"NOMB" + data[4:]
    yield "version0", data[:4] + struct.pack("<H", 0) + data[6:]
    yield "version2", data[:4] + struct.pack("<H", 2) + data[6:]
    yield "truncated_header", data[:12]
    for cut in (3, 9, off_theta + 4, off_theta + 100, len(data) - 13, len(data) - 1):
        yield f"truncated_{cut}", data[:cut]
    yield "trailing", data + b"\x00"
    yield "theta_len", data[:off_theta] + struct.pack("<Q", struct.unpack_from("<Q", data, off_theta)[0] + 4) + \
        data[off_theta + 8:]
    yield "category", data[:6] + struct.pack("<I", hlen + 1) + header.replace("chair", "chairs").encode() + \
        data[10 + hlen:]
    yield "arch", data[:6] + struct.pack("<I", hlen) + header.replace("hidden_width=16", "hidden_width=00").encode() + \
        data[10 + hlen:]
    tlen = struct.unpack_from("<Q", data, off_theta)[0]
    off_grid = off_theta + 8 + tlen
    yield "grid_res", data[:off_grid + 8] + struct.pack("<I", 1) + data[off_grid + 12:]
    yield "grid_len", data[:off_grid] + struct.pack("<Q", 5) + data[off_grid + 8:]
    # last triangle's last index -> out of range
    yield "tri_index", data[:-4] + struct.pack("<I", 99)


def test_load_errors(tmp_path):
    from paper_2503_01582_b200 import DataError, UsageError
    from paper_2503_01582_b200 import prior as PR

    data = GOLDEN.read_bytes()
    for name, bad in _corruptions(data):
        f = tmp_path / f"{name}.noma"
        f.write_bytes(bad)
        with pytest.raises((DataError, UsageError)):
            PR.load_prior(f)
    with pytest.raises(DataError, match="cannot read"):
        PR.load_prior(tmp_path / "missing.noma")


@pytest.mark.ref
def test_reference_reads_our_files_and_agrees_on_errors(tmp_path, ref):
    from paper_2503_01582_b200 import PrenomError
    from paper_2503_01582_b200 import prior as PR

    rng = np.random.default_rng(9)
    b = _bundle()
    b.category = "ball"
    b.theta = rng.standard_normal(b.arch.param_count()).astype(np.float32)
    b.grid = rng.uniform(0, 5, (9, 9, 9)).astype(np.float32)
    b.genome.density_activation = 0
    ours = tmp_path / "ours.noma"
    PR.save_prior(b, ours)
    arch, th, g, v, t = ref.load_prior(ours)
    assert arch["hash_levels"] == b.arch.hash_levels and np.float32(arch["per_level_scale"]) == np.float32(
        b.arch.per_level_scale)
    assert np.array_equal(th, b.theta) and np.array_equal(g, b.grid)
    assert np.array_equal(v, b.vertices) and np.array_equal(t, b.triangles)
    st, text = ref.prior_summary(ours)
    assert st == 0 and text == PR.prior_summary(ours)
    # malformed files: same accept/reject decision and the same message
    for name, bad in _corruptions(GOLDEN.read_bytes()):
        f = tmp_path / f"{name}.noma"
        f.write_bytes(bad)
        st, msg = ref.prior_summary(f)
        try:
            PR.load_prior(f)
            ours_msg = None
        except PrenomError as e:
            ours_msg = str(e)
        assert st != 0, name
        assert ours_msg == msg, (name, ours_msg, msg)


# ---------------------------------------------------------------- GPU
@pytest.mark.gpu
@pytest.mark.parametrize("R,iso", [(24, 8.0), (33, 3.0)])
def test_bake_prior_bit_exact_vs_reference(ctx, rng, R, iso):
    """bake_prior (density_grid.cpp:138-143) on the device: the σ lattice matches the
    reference's refresh_grid to the field tolerance (device expf vs glibc exp: <= 2e-6
    relative; the raw MLP outputs are bit-exact, tests/test_gpu_parity.py), and the mesh is
    bit-exact the reference's marching_cubes (+ cleanup_mesh) of that lattice. The seeded
    field gives 15k / 35k triangles."""
    from conftest import grad_params
    from oracle import pyoracle
    from paper_2503_01582_b200 import FieldArch
    from paper_2503_01582_b200 import prior as PR

    arch = FieldArch(hash_levels=6, features_per_level=2, log2_table_size=12, base_resolution=4,
                     per_level_scale=1.5, hidden_width=32, hidden_layers=2)
    theta = grad_params(arch, rng)
    theta[arch.hash_param_count():] *= 3.0  # a field with structure (σ spans the iso level)
    grid, v, t = PR.bake_prior(ctx, arch, theta, R, iso)
    assert len(t) > 1000
    rg = pyoracle.Oracle().refresh_grid(arch, theta, R)
    np.testing.assert_allclose(grid, rg, rtol=2e-6, atol=0)
    if pyoracle.REF_SO.exists():
        ref = pyoracle.Ref()
        np.testing.assert_allclose(grid, ref.refresh_grid(arch, theta, R), rtol=2e-6, atol=0)
        rv, rt = ref.marching_cubes(grid, iso)
        assert np.array_equal(v, rv) and np.array_equal(t, rt)


@pytest.mark.gpu
def test_from_prior_round_trip_and_train(ctx, rng, tmp_path):
    """save a trained object's prior, load it, create from it: same θ and grid; it trains."""
    from paper_2503_01582_b200 import FieldArch, ObjectTrainer, TrainConfig, scenes
    from paper_2503_01582_b200 import prior as PR

    sc = scenes.box_union_scene(n_views=4, res=48, seed=5)
    arch = FieldArch(hash_levels=6, features_per_level=2, log2_table_size=12, base_resolution=4,
                     per_level_scale=1.5, hidden_width=32, hidden_layers=2)
    cfg = TrainConfig(rays_per_iter=256, samples_per_ray=32, coarse_samples=16, prior_sampling=1,
                      grid_refresh_every=0)
    src = ObjectTrainer.create(ctx, arch, grid=scenes.occupancy_prior(sc.boxes, R=16), seed=3, cfg=cfg,
                               box_min=sc.box_min, box_max=sc.box_max)
    src.set_frames(sc.cams, sc.rgb, sc.depth, sc.mask, 1, sc.obj_pose)
    src.train_step(20, stats=False)
    theta = src.get_params()
    grid, v, t = PR.bake_prior(ctx, arch, theta, 20, 5.0)
    b = PR.PriorBundle(arch=arch, theta=theta, grid=grid, vertices=v, triangles=t, category="book")
    PR.save_prior(b, tmp_path / "p.noma")
    lb = PR.load_prior(tmp_path / "p.noma")
    obj = ObjectTrainer.from_prior(ctx, lb, seed=4, cfg=cfg, box_min=sc.box_min, box_max=sc.box_max)
    assert np.array_equal(obj.get_params(), theta)
    g = obj.get_grid()
    assert g.shape == (20, 20, 20) and np.array_equal(g, grid)
    obj.set_frames(sc.cams, sc.rgb, sc.depth, sc.mask, 1, sc.obj_pose)
    st = obj.train_step(5)
    assert all(np.isfinite(s["total"]) for s in st)


def test_from_prior_rejects_grids_beyond_the_device_limit():
    """load_prior accepts grids up to 4096^3 (prior_bundle.cpp); the device sampler's grids stop at
    1024^3 (32-bit lattice indices) -- a DataError naming the limit, not a silent resample (CPU)."""
    from types import SimpleNamespace

    from paper_2503_01582_b200 import DataError, ObjectTrainer
    from paper_2503_01582_b200.trainer import MAX_GRID_RES

    big = SimpleNamespace(grid=np.zeros((MAX_GRID_RES + 1, 1, 1), np.float32), arch=None, theta=None)
    with pytest.raises(DataError, match="1024"):
        ObjectTrainer.from_prior(None, big)
