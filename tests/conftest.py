import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "ref: needs oracle/_ref/libnoma_ref.so (the compiled reference)")


@pytest.fixture(scope="session")
def oracle():
    from oracle import pyoracle

    if not pyoracle.ORACLE_SO.exists():
        pyoracle.build_oracle(ref=False)
    return pyoracle.Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle import pyoracle

    if not pyoracle.REF_SO.exists():
        if (pyoracle.REF_DIR / "core").exists():
            pyoracle.build_oracle(ref=True)
        else:
            pytest.skip("reference library not built and reference sources absent")
    return pyoracle.Ref()


@pytest.fixture(scope="session")
def ctx():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2503_01582_b200 import Context

    c = Context(0)
    yield c
    c.close()


@pytest.fixture
def rng():
    return np.random.default_rng(1234)


def tiny_arch(rng, **over):
    """testutil::random_tiny_arch analogue (testutil.hpp:74-87)."""
    from paper_2503_01582_b200 import FieldArch

    a = FieldArch(hash_levels=int(rng.integers(1, 4)), features_per_level=int(rng.integers(1, 3)),
                  log2_table_size=int(rng.integers(4, 7)), base_resolution=int(rng.integers(2, 5)),
                  per_level_scale=float(np.float32(rng.uniform(1.3, 1.6))),
                  hidden_width=int(rng.choice([4, 8])), hidden_layers=int(rng.integers(1, 3)),
                  density_activation=int(rng.integers(0, 2)))
    for k, v in over.items():
        setattr(a, k, v)
    return a


def grad_params(arch, rng):
    """testutil::random_params_for_gradients analogue (testutil.hpp:92-100)."""
    P, nh = arch.param_count(), arch.hash_param_count()
    p = np.empty(P, np.float32)
    p[:nh] = rng.uniform(-0.6, 0.6, nh)
    p[nh:] = 0.4 * rng.standard_normal(P - nh)
    return p
