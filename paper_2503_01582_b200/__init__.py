"""B200-native per-object NeRF train step (PRENOM, arXiv 2503.01582).

The product is the CUDA library ``_lib/libprenom_b200.so`` behind the C ABI in
``include/prenom/prenom_gpu.h``; this package is the reference-shaped host
API over it (see :mod:`.trainer`).
"""
from .trainer import (  # noqa: F401
    Camera,
    Context,
    CudaError,
    DataError,
    FieldArch,
    NumericError,
    ObjectTrainer,
    Pose,
    PrenomError,
    TrainConfig,
    UsageError,
    derive_seed,
    mix_seed,
)
