"""B200-native CodeGEMM decode GEMV (arXiv 2512.17970) behind the reference API.

The operator surface mirrors ``/root/reference/pkg/src/codegemm`` for the
decode hot path: the quantized-layer containers, ``codegemm_gemm`` and
``build_psumbook``, ``TileConfig`` / ``OpCounters`` and the error classes.
Compute runs in ``libcodegemm_b200.so`` (hand-written sm_100a CUDA behind a
C ABI, ``include/codegemm_b200.h``); there is no CPU path.
"""

from .engines import (
    DeviceLayer,
    OpCounters,
    Psumbook,
    StagedLaunch,
    TileConfig,
    build_psumbook,
    closed_form_counters,
    codegemm_gemm,
    gemm_group,
    gemm_stages,
    phase_split,
)
from .errors import (
    BadMagicError,
    CodeGemmError,
    ConfigError,
    CudaError,
    DimOverflowError,
    FormatError,
    IntegrityError,
    ShapeError,
    TruncatedFileError,
    UnsupportedVersionError,
)
from .quantizer import (
    Codebook,
    CodePlane,
    QuantConfig,
    QuantizedLayer,
    ScalePlane,
    pack_codes,
    random_layer,
    unpack_codes,
)
from .storage import deserialize, load_device_layer, serialize
from .tensors import Matrix, encode_f16_array

__version__ = "0.1.0"

__all__ = [
    "BadMagicError", "CodeGemmError", "Codebook", "CodePlane", "ConfigError", "CudaError",
    "DeviceLayer", "DimOverflowError", "FormatError", "IntegrityError", "Matrix", "OpCounters",
    "Psumbook", "QuantConfig", "QuantizedLayer", "ScalePlane", "ShapeError", "StagedLaunch",
    "TileConfig",
    "TruncatedFileError", "UnsupportedVersionError", "build_psumbook", "closed_form_counters",
    "deserialize", "load_device_layer", "serialize",
    "codegemm_gemm", "encode_f16_array", "gemm_group", "gemm_stages", "pack_codes", "phase_split", "random_layer",
    "unpack_codes",
]
