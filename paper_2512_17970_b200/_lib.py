"""ctypes binding of libcodegemm_b200.so (include/codegemm_b200.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (nvcc,
sm_100a).  There is no fallback: if the library is missing, importing the
compute entry points raises ``CudaError`` with the build instruction.
"""

from __future__ import annotations

import ctypes
import os

from .errors import CodeGemmError, ConfigError, CudaError, IntegrityError, ShapeError

LIB_NAME = "libcodegemm_b200.so"
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

CG_OK = 0
CG_ERR_CONFIG = 1
CG_ERR_SHAPE = 2
CG_ERR_INTEGRITY = 3
CG_ERR_CUDA = 4
CG_ERR_UNSUPPORTED = 5
CG_ERR_ARG = 6

CG_MODE_AUTO = 0
CG_MODE_FAST = 1
CG_MODE_STRICT = 2

CG_OPT_NO_PDL = 1
CG_OPT_NO_L2_PREFETCH = 2
CG_OPT_DETERMINISTIC = 4
CG_OPT_BATCH_EAGER = 8
CG_OPT_NO_BATCH = 16

MODES = {"auto": CG_MODE_AUTO, "fast": CG_MODE_FAST, "strict": CG_MODE_STRICT}

# Every symbol include/codegemm_b200.h declares (tests check the exports).
EXPORTS = (
    "cg_abi_version",
    "cg_last_error",
    "cg_device_count",
    "cg_layer_create",
    "cg_layer_create_packed",
    "cg_layer_destroy",
    "cg_layer_query",
    "cg_gemm_stages",
    "cg_gemm_stages_xchg",
    "cg_stages_prepare",
    "cg_stages_launch",
    "cg_stages_run_host",
    "cg_stages_set_mirror",
    "cg_stages_destroy",
    "cg_comm_create",
    "cg_comm_buffer",
    "cg_comm_ipc_handle",
    "cg_comm_open_peers",
    "cg_comm_set_peers",
    "cg_comm_destroy",
    "cg_layer_gemm",
    "cg_layer_gemm_host",
    "cg_gemm_group",
    "cg_layer_psumbook",
    "cg_layer_unpack_codes",
    "cg_psumbook_build",
    "cg_psumbook_build_f32",
)


class LayerOptions(ctypes.Structure):
    _fields_ = [
        ("u", ctypes.c_int),
        ("rg_per_task", ctypes.c_int),
        ("flags", ctypes.c_int),
        ("device", ctypes.c_int),
    ]


class LayerInfo(ctypes.Structure):
    _fields_ = [
        ("rows", ctypes.c_int64),
        ("cols", ctypes.c_int64),
        ("v", ctypes.c_int),
        ("m", ctypes.c_int),
        ("b", ctypes.c_int),
        ("g", ctypes.c_int64),
        ("fast_supported", ctypes.c_int),
        ("u", ctypes.c_int),
        ("rg_per_task", ctypes.c_int),
        ("n_slices", ctypes.c_int64),
        ("n_tasks", ctypes.c_int64),
        ("smem_bytes", ctypes.c_int),
        ("launches_fast", ctypes.c_int),
        ("device_bytes", ctypes.c_int64),
        ("algorithmic_bytes", ctypes.c_int64),
        ("batch_supported", ctypes.c_int),
        ("batch_ready", ctypes.c_int),
    ]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


_lib = None


def load() -> ctypes.CDLL:
    """Load (once) and type the library; raise CudaError if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise CudaError(
            f"{LIB_NAME} not found at {LIB_PATH}; build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'` (nvcc, sm_100a)"
        )
    lib = ctypes.CDLL(LIB_PATH)
    p, i, i64, vp = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_void_p
    u16pp = ctypes.POINTER(ctypes.c_void_p)
    lib.cg_abi_version.restype = i
    lib.cg_last_error.restype = ctypes.c_char_p
    lib.cg_device_count.restype = i
    lib.cg_layer_create.argtypes = [u16pp, u16pp, p, i64, i64, i, i, i, i64,
                                    ctypes.POINTER(LayerOptions), ctypes.POINTER(vp)]
    lib.cg_layer_create.restype = i
    lib.cg_layer_create_packed.argtypes = [u16pp, u16pp, p, i64, i64, i, i, i, i64,
                                    ctypes.POINTER(LayerOptions), ctypes.POINTER(vp)]
    lib.cg_layer_create_packed.restype = i
    lib.cg_layer_destroy.argtypes = [vp]
    lib.cg_layer_destroy.restype = i
    lib.cg_layer_query.argtypes = [vp, ctypes.POINTER(LayerInfo)]
    lib.cg_layer_query.restype = i
    lib.cg_layer_gemm.argtypes = [vp, p, i, p, i, vp]
    lib.cg_layer_gemm.restype = i
    lib.cg_gemm_group.argtypes = [ctypes.POINTER(vp), ctypes.POINTER(vp), ctypes.POINTER(vp), i,
                                  i, vp]
    lib.cg_gemm_group.restype = i
    lib.cg_gemm_stages.argtypes = [ctypes.POINTER(vp), ctypes.POINTER(vp),
                                   ctypes.POINTER(ctypes.c_int), ctypes.POINTER(vp),
                                   ctypes.POINTER(ctypes.c_int), i, i, vp]
    lib.cg_gemm_stages.restype = i
    lib.cg_gemm_stages_xchg.argtypes = [ctypes.POINTER(vp), ctypes.POINTER(vp),
                                        ctypes.POINTER(ctypes.c_int), ctypes.POINTER(vp),
                                        ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int),
                                        i, i, vp, vp]
    lib.cg_gemm_stages_xchg.restype = i
    lib.cg_stages_prepare.argtypes = [ctypes.POINTER(vp), ctypes.POINTER(vp),
                                      ctypes.POINTER(ctypes.c_int), ctypes.POINTER(vp),
                                      ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int),
                                      i, i, vp, ctypes.POINTER(vp)]
    lib.cg_stages_prepare.restype = i
    lib.cg_stages_launch.argtypes = [vp, vp]
    lib.cg_stages_launch.restype = i
    lib.cg_stages_run_host.argtypes = [vp, p, i64, p, p, p, i64, vp]
    lib.cg_stages_run_host.restype = i
    lib.cg_stages_set_mirror.argtypes = [vp, ctypes.POINTER(vp)]
    lib.cg_stages_set_mirror.restype = i
    lib.cg_stages_destroy.argtypes = [vp]
    lib.cg_stages_destroy.restype = i
    lib.cg_comm_create.argtypes = [i, i, ctypes.c_int64, i, i, i, ctypes.POINTER(vp)]
    lib.cg_comm_create.restype = i
    lib.cg_comm_buffer.argtypes = [vp, ctypes.POINTER(vp)]
    lib.cg_comm_buffer.restype = i
    lib.cg_comm_ipc_handle.argtypes = [vp, p]
    lib.cg_comm_ipc_handle.restype = i
    lib.cg_comm_open_peers.argtypes = [vp, p]
    lib.cg_comm_open_peers.restype = i
    lib.cg_comm_set_peers.argtypes = [vp, ctypes.POINTER(vp)]
    lib.cg_comm_set_peers.restype = i
    lib.cg_comm_destroy.argtypes = [vp]
    lib.cg_comm_destroy.restype = i
    lib.cg_layer_gemm_host.argtypes = [vp, p, i, p, i, vp]
    lib.cg_layer_gemm_host.restype = i
    lib.cg_layer_psumbook.argtypes = [vp, p, i, p, vp]
    lib.cg_layer_psumbook.restype = i
    lib.cg_layer_unpack_codes.argtypes = [vp, p, vp]
    lib.cg_layer_unpack_codes.restype = i
    lib.cg_psumbook_build.argtypes = [p, p, i, i, i, i64, i, p, vp]
    lib.cg_psumbook_build.restype = i
    lib.cg_psumbook_build_f32.argtypes = [p, p, i, i, i, i64, i, p, vp]
    lib.cg_psumbook_build_f32.restype = i
    _lib = lib
    return lib


_ERRORS = {
    CG_ERR_CONFIG: ConfigError,
    CG_ERR_SHAPE: ShapeError,
    CG_ERR_INTEGRITY: IntegrityError,
    CG_ERR_CUDA: CudaError,
    CG_ERR_UNSUPPORTED: ConfigError,
    CG_ERR_ARG: ValueError,
}


def check(rc: int) -> None:
    """Raise the reference-side exception class for a C status code."""
    if rc == CG_OK:
        return
    msg = load().cg_last_error().decode(errors="replace")
    raise _ERRORS.get(rc, CodeGemmError)(msg)
