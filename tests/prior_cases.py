"""Seeded prior-bundle inputs shared by tests/golden/make_golden_prior.py and
tests/test_prior.py (the golden file is the reference's save_prior of these)."""
import numpy as np


def golden_bundle_inputs():
    from paper_2503_01582_b200 import FieldArch

    rng = np.random.default_rng(2503)
    arch = FieldArch(hash_levels=4, features_per_level=2, log2_table_size=8, base_resolution=4,
                     per_level_scale=float(np.float32(1.7)), hidden_width=16, hidden_layers=1,
                     density_activation=1)
    theta = rng.standard_normal(arch.param_count()).astype(np.float32)
    grid = rng.uniform(0.0, 40.0, (6, 6, 6)).astype(np.float32)
    verts = rng.uniform(0.0, 1.0, (5, 3)).astype(np.float32)
    tris = np.array([[0, 1, 2], [2, 3, 4]], np.int32)
    prov = dict(category="chair", search_seed=12345678901, population=24, generations=7,
                genome_ints=(12, 17, 2, 64, 1, 40, 9, 1), genome_floats=(3e-3, 0.25, 1.3819, 0.2, 3e-4))
    return arch, theta, grid, verts, tris, prov
