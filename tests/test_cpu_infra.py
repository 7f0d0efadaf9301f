"""CPU-only checks: deterministic exp, Philox KAT (oracle), the C-ABI library
loads and exports every symbol include/prenom/prenom_gpu.h declares, host
helpers (arch math, scenes, seeds)."""
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2503_01582_b200 import FieldArch, derive_seed, mix_seed, scenes
from paper_2503_01582_b200 import _capi

ROOT = Path(__file__).resolve().parents[1]


def test_det_exp_close_to_libm(oracle):
    rng = np.random.default_rng(0)
    xs = np.concatenate([-rng.exponential(3.0, 20000), rng.uniform(-745, 709, 2000),
                         [-1e-300, 0.0, -5e-324, -745.2, -744.0, -708.5, 709.7, -1e-8]])
    worst = 0
    for x in xs:
        a = oracle.lib.po_det_exp(float(x))
        b = float(np.exp(x))
        if b == 0.0 or not np.isfinite(b):
            assert a == b or abs(a - b) <= 5e-324, x
            continue
        ulp = np.spacing(b)
        worst = max(worst, abs(a - b) / ulp)
    assert worst <= 2.0, worst


def test_philox_kat(oracle):
    assert list(oracle.philox([0, 0, 0, 0], [0, 0])) == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]
    assert list(oracle.philox([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2)) == [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]
    assert list(oracle.philox([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0])) == \
        [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]


def test_uniform_and_pick_ranges(oracle):
    assert oracle.lib.po_u01(0) == 0.0
    assert oracle.lib.po_u01(0xFFFFFFFF) < 1.0
    assert oracle.lib.po_pick(0xFFFFFFFF, 7) == 6 and oracle.lib.po_pick(0, 7) == 0


def test_library_exports_every_declared_symbol():
    header = (ROOT / "include" / "prenom" / "prenom_gpu.h").read_text()
    declared = set(re.findall(r"\b(prenom_[a-z0-9_]+)\s*\(", header)) - {"prenom_status"}
    assert declared == set(_capi.EXPORTED), declared ^ set(_capi.EXPORTED)
    lib = _capi.load()  # loads without a GPU; no compute is called
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.prenom_abi_version() == 1
    cfg = _capi.TrainCfgC()
    lib.prenom_default_train_cfg(cfg)
    assert cfg.rays_per_iter == 128 and cfg.samples_per_ray == 24 and abs(cfg.eta - 1e-2) < 1e-9


def test_host_param_count_matches_library():
    import ctypes as C

    lib = _capi.load()
    for a in (scenes.cfg1_arch(), scenes.cfg2_arch(), scenes.cfg4_arch(), FieldArch()):
        tot, hsh = C.c_size_t(), C.c_size_t()
        assert lib.prenom_param_count(C.byref(a.to_c()), C.byref(tot), C.byref(hsh)) == 0
        assert tot.value == a.param_count() and hsh.value == a.hash_param_count()
    # SURVEY §8 table param counts
    assert scenes.cfg1_arch().param_count() == 526020
    assert scenes.cfg2_arch(32).param_count() == 16779460
    assert scenes.cfg2_arch(64).param_count() == 16783748
    assert scenes.cfg4_arch().param_count() == 8395140


def test_no_context_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2503_01582_b200 import Context, CudaError, UsageError

    with pytest.raises((CudaError, UsageError)):
        Context(0)


def test_seed_helpers_match_reference_formulas():
    # mapper.cpp:20-26 / meta.cpp:14-20 re-derived independently
    def mix(b, s, k):
        M = (1 << 64) - 1
        v = (b * 0x9E3779B97F4A7C15 + s * k + 1) & M
        v ^= v >> 31
        v = (v * 0x94D049BB133111EB) & M
        v ^= v >> 29
        return (v ^ (v >> 32)) & 0xFFFFFFFF

    for b, s in [(0, 0), (1, 0x77AA), (12345, 0x1217 + 9)]:
        assert mix_seed(b, s) == mix(b, s, 0xC2B2AE3D27D4EB4F)
        assert derive_seed(b, s) == mix(b, s, 0xBF58476D1CE4E5B9)


def test_scenes_shapes_and_conventions():
    sc = scenes.sphere_scene(n_views=4, res=32, fx=32.0, depth_noise=0.0)
    assert sc.rgb.shape == (4, 32, 32, 3) and sc.depth.shape == (4, 32, 32) and sc.mask.dtype == np.uint8
    hit = sc.mask == 1
    assert hit.any() and (~hit).any()
    # depth = distance along the ray; camera at radius 1.5, sphere radius 0.35
    assert np.all(sc.depth[hit] >= 1.5 - 0.35 - 1e-4) and np.all(sc.depth[~hit] == 0)
    bu = scenes.box_union_scene(n_views=3, res=24, seed=1)
    assert 3 <= len(bu.boxes) <= 6
    g = scenes.occupancy_prior(bu.boxes, R=32)
    assert g.shape == (32, 32, 32) and g.max() <= scenes.SIGMA_PRIOR_SCALE + 1e-4 and g.max() > 0
