"""B200-native (sm_100a) fused flux-evaluation + flux-divergence kernels for
ACM-HD flux reconstruction on tensor-product elements (arXiv 2107.14027).

The compute path is ``lib/libhexfuse_b200.so`` (hand-written CUDA, C ABI in
``include/hexfuse_b200.h``).  This package is the host-side mirror of the
reference's interface (see :mod:`.hexfuse`) plus the multi-GPU driver
(:mod:`.multi_gpu`).  There is no CPU fallback.
"""
from .hexfuse import (  # noqa: F401
    Context,
    ElementConfig,
    HexfuseError,
    HexfuseInvalid,
    Method,
    PhysParams,
    Precision,
    StateField,
    derivative_matrix,
    export_blob,
    field_rel_error,
    field_sidecar,
    field_words,
    fused_divergence,
    fused_divergence_blob,
    fused_divergence_device,
    fused_divergence_mapped_device,
    face_words,
    fr_correct_device,
    fr_divergence_faces_device,
    fr_project_device,
    fr_residual_device,
    make_mesh,
    geometry_words,
    mapped_kernel_info,
    fused_divergence_variant,
    import_blob,
    kernel_info,
    make_problem,
    n_vars,
    partition,
    preferred_group,
    problem_for,
    selected_method,
    unfused_divergence_device,
    unfused_workspace_bytes,
    validate,
    variant_info,
    var_gradient,
    var_pressure,
    var_velocity,
    verify_tolerance,
    word_bytes,
)

__version__ = "0.1.0"
