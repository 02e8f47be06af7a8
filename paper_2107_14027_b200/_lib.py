"""ctypes binding of the C ABI in ``include/hexfuse_b200.h``.

The shared library is built in-tree by ``paper_2107_14027_b200/csrc/Makefile``
(``__graft_entry__.build()``) into ``paper_2107_14027_b200/lib/``.  There is no
fallback: if the library is missing, every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HEXFUSE_B200_LIB") or os.path.join(_HERE, "lib", "libhexfuse_b200.so")

HF_OK, HF_ERUNTIME, HF_EINVAL = 0, 1, 2
HF_FP32, HF_FP64 = 0, 1
HF_METHOD_AUTO, HF_METHOD_PLANAR, HF_METHOD_LINES, HF_METHOD_UNFUSED, HF_METHOD_PLANAR_MANAGED = 0, 1, 2, 3, 4


class hf_problem(C.Structure):
    _fields_ = [
        ("d", C.c_int),
        ("p", C.c_int),
        ("n_elem", C.c_int64),
        ("group", C.c_int),
        ("precision", C.c_int),
        ("nu", C.c_double),
        ("zeta", C.c_double),
        ("T", C.c_double),
        ("jac", C.c_double * 3),
        ("with_source", C.c_int),
        ("method", C.c_int),
    ]


class hf_kernel_info(C.Structure):
    _fields_ = [
        ("method", C.c_int),
        ("elems_per_cta", C.c_int),
        ("block_threads", C.c_int),
        ("shared_bytes", C.c_int),
        ("registers", C.c_int),
        ("grid", C.c_int64),
        ("bulk_path", C.c_int),
        ("blocks_per_sm", C.c_int),
        ("name", C.c_char * 96),
    ]


# Every symbol include/hexfuse_b200.h declares (checked by tests/test_capi.py).
EXPORTED = [
    "hf_n_vars", "hf_field_words", "hf_offset", "hf_validate", "hf_derivative_matrix",
    "hf_algorithmic_bytes_per_point", "hf_selected_method", "hf_preferred_group", "hf_kernel_info_get",
    "hf_fused_divergence", "hf_unfused_workspace_bytes", "hf_unfused_divergence", "hf_context_create",
    "hf_context_destroy", "hf_fused_divergence_host", "hf_fused_divergence_host_batch", "hf_partition", "hf_last_error", "hf_version",
    "hf_geometry_words", "hf_fused_divergence_mapped", "hf_mapped_kernel_info",
    "hf_face_words", "hf_fr_project", "hf_fr_correct", "hf_fr_divergence_faces", "hf_fr_residual",
    "hf_ipc_handle", "hf_ipc_open", "hf_ipc_close",
    "hf_blob_info", "hf_blob_read", "hf_blob_write", "hf_fused_divergence_blob",
]


class hf_mesh(C.Structure):
    _fields_ = [("dims", C.c_int * 3), ("e_begin", C.c_int64), ("n_local", C.c_int64), ("layer", C.c_int64)]

_lib = None


class HexfuseError(RuntimeError):
    """runtime_error analogue (HF_ERUNTIME)."""


class HexfuseInvalid(ValueError):
    """invalid_argument analogue (HF_EINVAL)."""


def load() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise HexfuseError(
            f"{LIB_PATH} is missing: the B200 kernels are not built. Run __graft_entry__.build() "
            "(there is no CPU fallback).")
    L = C.CDLL(LIB_PATH)
    P = C.POINTER(hf_problem)
    L.hf_n_vars.argtypes = [C.c_int]
    L.hf_field_words.argtypes = [P]
    L.hf_field_words.restype = C.c_int64
    L.hf_offset.argtypes = [P, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_int]
    L.hf_offset.restype = C.c_int64
    L.hf_validate.argtypes = [P]
    L.hf_derivative_matrix.argtypes = [C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double)]
    L.hf_algorithmic_bytes_per_point.argtypes = [P]
    L.hf_algorithmic_bytes_per_point.restype = C.c_int64
    L.hf_selected_method.argtypes = [P]
    L.hf_preferred_group.argtypes = [P]
    L.hf_kernel_info_get.argtypes = [P, C.POINTER(hf_kernel_info)]
    L.hf_fused_divergence.argtypes = [P, C.c_void_p, C.c_void_p, C.c_void_p]
    L.hf_unfused_workspace_bytes.argtypes = [P]
    L.hf_unfused_workspace_bytes.restype = C.c_size_t
    L.hf_unfused_divergence.argtypes = [P, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    L.hf_context_create.argtypes = [C.c_int]
    L.hf_context_create.restype = C.c_void_p
    L.hf_context_destroy.argtypes = [C.c_void_p]
    L.hf_context_destroy.restype = None
    L.hf_fused_divergence_host.argtypes = [C.c_void_p, P, C.c_void_p, C.c_void_p]
    L.hf_fused_divergence_host_batch.argtypes = [C.c_void_p, C.c_int, P, C.POINTER(C.c_void_p),
                                                 C.POINTER(C.c_void_p)]
    L.hf_partition.argtypes = [P, C.c_int, C.c_int, C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                               C.POINTER(C.c_int64)]
    L.hf_last_error.restype = C.c_char_p
    L.hf_version.restype = C.c_char_p
    L.hf_fused_divergence_variant.argtypes = [P, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                              C.POINTER(hf_kernel_info)]
    L.hf_geometry_words.argtypes = [P]
    L.hf_geometry_words.restype = C.c_int64
    L.hf_fused_divergence_mapped.argtypes = [P, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    L.hf_mapped_kernel_info.argtypes = [P, C.POINTER(hf_kernel_info)]
    L.hf_face_words.argtypes = [P]
    L.hf_face_words.restype = C.c_int64
    L.hf_fr_project.argtypes = [P, C.c_void_p, C.c_void_p, C.c_void_p]
    L.hf_fr_correct.argtypes = [P, C.POINTER(hf_mesh), C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    L.hf_fr_divergence_faces.argtypes = [P, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    L.hf_fr_residual.argtypes = [P, C.POINTER(C.c_int), C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    L.hf_ipc_handle.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(C.c_int64)]
    L.hf_ipc_open.argtypes = [C.c_void_p, C.POINTER(C.c_void_p)]
    L.hf_ipc_close.argtypes = [C.c_void_p]
    # (bound when present, so that an older build can still be A/B-timed through this package;
    # tests/test_capi.py checks that the built library exports every declared symbol)
    if hasattr(L, "hf_blob_info"):
        L.hf_blob_info.argtypes = [C.c_char_p, P]
        L.hf_blob_read.argtypes = [C.c_char_p, P, C.c_void_p]
        L.hf_blob_write.argtypes = [C.c_char_p, P, C.c_void_p]
        L.hf_fused_divergence_blob.argtypes = [C.c_void_p, P, C.c_char_p, C.c_char_p]
    _lib = L
    return L


def check(rc: int, what: str) -> None:
    if rc == HF_OK:
        return
    msg = load().hf_last_error().decode()
    if rc == HF_EINVAL:
        raise HexfuseInvalid(f"{what}: {msg}")
    raise HexfuseError(f"{what}: {msg}")
