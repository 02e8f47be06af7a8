"""Host-side mirror of the reference's hot-path interface (``hexfuse`` C++
headers, /root/reference/proj/include/hexfuse), over the B200 C ABI.

Same names, argument meaning and error behaviour as the reference:

=================================  ===========================================
reference                          here
=================================  ===========================================
``Precision`` (core.hpp:10)        :class:`Precision`
``PhysParams`` (equations.hpp:14)  :class:`PhysParams` (``validate`` raises ValueError)
``n_vars`` (equations.hpp:27)      :func:`n_vars`
``ElementConfig`` (layout.hpp:58)  :class:`ElementConfig`
``StateField`` (layout.hpp:104)    :class:`StateField` (float64 storage, AoSoA)
``export_blob/import_blob``        :func:`export_blob` / :func:`import_blob` (layout.hpp:155-200)
``oracle_divergence``              :func:`fused_divergence` -- same signature, runs
  (oracle.hpp:20-62)                 the hand-written sm_100a kernels
``field_rel_error`` (verify.hpp)   :func:`field_rel_error`
``verify_tolerance``               :func:`verify_tolerance`
=================================  ===========================================

``std::invalid_argument`` maps to :class:`HexfuseInvalid` (a ``ValueError``),
``std::runtime_error`` to :class:`HexfuseError`.
"""
from __future__ import annotations

import ctypes as C
import enum
import threading
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib
from ._lib import HexfuseError, HexfuseInvalid, check, hf_kernel_info, hf_problem


class Precision(enum.IntEnum):
    fp32 = _lib.HF_FP32
    fp64 = _lib.HF_FP64


def word_bytes(p: Precision) -> int:
    return 4 if p == Precision.fp32 else 8


class Method(enum.IntEnum):
    auto = _lib.HF_METHOD_AUTO
    planar = _lib.HF_METHOD_PLANAR
    lines = _lib.HF_METHOD_LINES
    unfused = _lib.HF_METHOD_UNFUSED
    planar_managed = _lib.HF_METHOD_PLANAR_MANAGED


def n_vars(d: int) -> int:
    """equations.hpp:27-30"""
    if d not in (2, 3):
        raise HexfuseInvalid("n_vars: dimension must be 2 or 3")
    return 1 + d + d * d


def var_pressure() -> int:
    return 0


def var_velocity(b: int) -> int:
    return 1 + b


def var_gradient(d: int, b: int, a: int) -> int:
    """equations.hpp:34-36"""
    return 1 + d + b * d + a


@dataclass
class PhysParams:
    """equations.hpp:14-24"""
    nu: float = 6.25e-4
    zeta: float = 2.5
    T: float = 1.0

    def validate(self) -> None:
        if not self.nu >= 0.0:
            raise HexfuseInvalid("PhysParams: nu must be >= 0")
        if not self.zeta > 0.0:
            raise HexfuseInvalid("PhysParams: zeta must be > 0")
        if not self.T > 0.0:
            raise HexfuseInvalid("PhysParams: T must be > 0")


@dataclass
class ElementConfig:
    """layout.hpp:58-100.  ``group`` is the AoSoA group (elements per CTA);
    ``None`` picks the B200 kernel's preferred group (``hf_preferred_group``)."""
    p: int = 3
    d: int = 3
    n_elem: int = 256
    precision: Precision = Precision.fp64
    method: Method = Method.auto
    group: Optional[int] = None

    def m(self) -> int:
        return self.p + 1

    def n_points(self) -> int:
        return self.m() ** self.d

    def nv(self) -> int:
        return n_vars(self.d)

    def validate(self) -> None:
        if self.d not in (2, 3):
            raise HexfuseInvalid("ElementConfig: d must be 2 or 3")
        pmax = 7 if self.d == 3 else 8
        if not 1 <= self.p <= pmax:
            raise HexfuseInvalid(f"ElementConfig: p must be in [1,{pmax}]")
        if self.n_elem <= 0:
            raise HexfuseInvalid("ElementConfig: n_elem must be positive")

    def elems_per_block(self) -> int:
        if self.group is not None:
            return int(self.group)
        pr = make_problem(self.d, self.p, self.n_elem, 1, self.precision, PhysParams(), method=self.method)
        return preferred_group(pr)


class StateField:
    """layout.hpp:104-153.  Storage is float64 (as the reference's
    std::vector<double>); fp32 fields hold float-representable values."""

    def __init__(self, d: int, p: int, n_elem: int, group: int, precision: Precision, data=None):
        self.d, self.p, self.n_elem, self.group = int(d), int(p), int(n_elem), int(group)
        self.precision = Precision(precision)
        if self.group < 1:
            raise HexfuseInvalid("StateField: group must be >= 1")
        n = self.n_groups() * self.group_words()
        if data is None:
            self.data = np.zeros(n, dtype=np.float64)
        else:
            self.data = np.ascontiguousarray(data, dtype=np.float64)
            if self.data.size != n:
                raise HexfuseInvalid(f"StateField: expected {n} words, got {self.data.size}")

    @staticmethod
    def like(cfg: ElementConfig) -> "StateField":
        return StateField(cfg.d, cfg.p, cfg.n_elem, cfg.elems_per_block(), cfg.precision)

    def copy(self) -> "StateField":
        return StateField(self.d, self.p, self.n_elem, self.group, self.precision, self.data.copy())

    def m(self) -> int:
        return self.p + 1

    def nv(self) -> int:
        return n_vars(self.d)

    def n_points(self) -> int:
        return self.m() ** self.d

    def n_groups(self) -> int:
        return (self.n_elem + self.group - 1) // self.group

    def group_words(self) -> int:
        return self.group * self.n_points() * self.nv()

    def total_words(self) -> int:
        return int(self.data.size)

    def offset(self, e: int, i: int, j: int, k: int, v: int) -> int:
        """layout.hpp:128-134"""
        eg, el = divmod(e, self.group)
        m = self.m()
        pt = i + m * j + m * m * k
        return eg * self.group_words() + el + self.group * (pt + self.n_points() * v)

    def at(self, e, i, j, k, v) -> float:
        return float(self.data[self.offset(e, i, j, k, v)])

    def set(self, e, i, j, k, v, x) -> None:
        self.data[self.offset(e, i, j, k, v)] = x

    def state_at(self, e, i, j, k) -> np.ndarray:
        return np.array([self.at(e, i, j, k, v) for v in range(self.nv())])

    def quantize(self) -> None:
        """layout.hpp:149-152"""
        if self.precision == Precision.fp32:
            self.data = self.data.astype(np.float32).astype(np.float64)

    def words(self) -> np.ndarray:
        """The field in its storable precision (what crosses the C ABI)."""
        return self.data.astype(np.float32) if self.precision == Precision.fp32 else self.data

    def view(self) -> np.ndarray:
        """[group][v][pt][e_l] view of the padded storage."""
        return self.data.reshape(self.n_groups(), self.nv(), self.n_points(), self.group)


def field_sidecar(f: StateField) -> dict:
    """layout.hpp:155-159"""
    return {"d": f.d, "p": f.p, "n_elem": f.n_elem, "group": f.group,
            "precision": f.precision.name, "words": f.total_words(), "byte_order": "little"}


def _shape_problem(f: StateField) -> hf_problem:
    return make_problem(f.d, f.p, f.n_elem, f.group, f.precision, PhysParams())


def export_blob(f: StateField, path: str) -> None:
    """layout.hpp:161-177 through hf_blob_write: flat little-endian words + <path>.json
    sidecar, byte-identical to the reference's export_blob."""
    words = np.ascontiguousarray(f.words())
    check(_lib.load().hf_blob_write(path.encode(), C.byref(_shape_problem(f)), words.ctypes.data), "export_blob")


def import_blob(path: str) -> StateField:
    """layout.hpp:179-200 through hf_blob_info / hf_blob_read."""
    pr = hf_problem()
    pr.zeta = pr.T = 1.0
    check(_lib.load().hf_blob_info(path.encode(), C.byref(pr)), "import_blob")
    f = StateField(pr.d, pr.p, pr.n_elem, pr.group, Precision(pr.precision))
    raw = np.zeros(f.total_words(), dtype=np.float32 if f.precision == Precision.fp32 else np.float64)
    check(_lib.load().hf_blob_read(path.encode(), C.byref(pr), raw.ctypes.data), "import_blob")
    f.data = raw.astype(np.float64)
    return f


def fused_divergence_blob(in_path: str, out_path: str, params: PhysParams, jac: Sequence[float] = (1.0, 1.0, 1.0),
                          with_source: bool = False, method: Method = Method.auto) -> None:
    """A state blob in, its divergence blob out (hf_fused_divergence_blob, the host path)."""
    params.validate()
    pr = make_problem(3, 1, 0, 1, Precision.fp64, params, jac, with_source, method)
    check(_lib.load().hf_fused_divergence_blob(_context()._h, C.byref(pr), in_path.encode(), out_path.encode()),
          "hf_fused_divergence_blob")


def field_rel_error(got: StateField, ref: StateField) -> float:
    """verify.hpp:19-33: max|got-ref| / max(1, max|ref|) over real elements."""
    a = got.view()
    b = ref.view()
    ng, nv, npt, g = b.shape
    mask = (np.arange(ng * g).reshape(ng, g) < ref.n_elem)[:, None, None, :]
    mask = np.broadcast_to(mask, b.shape)
    diff = np.abs(a - b)[mask]
    maxdiff = float(np.max(diff)) if diff.size else 0.0
    if np.isnan(diff).any():
        maxdiff = float("inf")
    maxref = float(np.max(np.abs(b[mask]))) if diff.size else 0.0
    return maxdiff / max(1.0, maxref)


def verify_tolerance(p: Precision) -> float:
    """verify.hpp:35"""
    return 1e-5 if p == Precision.fp32 else 1e-11


# ------------------------------------------------------------------------------------------------
# Problem descriptors and C-ABI calls
# ------------------------------------------------------------------------------------------------

def make_problem(d: int, p: int, n_elem: int, group: int, precision, params: PhysParams,
                 jac: Sequence[float] = (1.0, 1.0, 1.0), with_source: bool = False, method=Method.auto) -> hf_problem:
    pr = hf_problem()
    pr.d, pr.p, pr.n_elem, pr.group = int(d), int(p), int(n_elem), int(group)
    pr.precision = int(Precision(precision))
    pr.nu, pr.zeta, pr.T = float(params.nu), float(params.zeta), float(params.T)
    for a in range(3):
        pr.jac[a] = float(jac[a]) if a < len(jac) else 0.0
    pr.with_source = int(bool(with_source))
    pr.method = int(Method(method))
    return pr


def problem_for(U: StateField, params: PhysParams, jac=(1.0, 1.0, 1.0), with_source=False,
                method=Method.auto) -> hf_problem:
    return make_problem(U.d, U.p, U.n_elem, U.group, U.precision, params, jac, with_source, method)


def validate(pr: hf_problem) -> None:
    check(_lib.load().hf_validate(C.byref(pr)), "hf_validate")


def field_words(pr: hf_problem) -> int:
    return int(_lib.load().hf_field_words(C.byref(pr)))


def selected_method(pr: hf_problem) -> Method:
    r = _lib.load().hf_selected_method(C.byref(pr))
    if r < 0:
        check(-r, "hf_selected_method")
    return Method(r)


def preferred_group(pr: hf_problem) -> int:
    r = _lib.load().hf_preferred_group(C.byref(pr))
    if r < 0:
        check(-r, "hf_preferred_group")
    return int(r)


def kernel_info(pr: hf_problem) -> dict:
    ki = hf_kernel_info()
    check(_lib.load().hf_kernel_info_get(C.byref(pr), C.byref(ki)), "hf_kernel_info_get")
    return {"method": Method(ki.method).name, "elems_per_cta": ki.elems_per_cta, "block_threads": ki.block_threads,
            "shared_bytes": ki.shared_bytes, "registers": ki.registers, "grid": int(ki.grid),
            "bulk_path": bool(ki.bulk_path), "blocks_per_sm": ki.blocks_per_sm, "name": ki.name.decode()}


def derivative_matrix(m: int):
    """Gauss-Legendre nodes and D (operators.hpp:17-74) as the library builds them."""
    D = (C.c_double * (m * m))()
    x = (C.c_double * m)()
    check(_lib.load().hf_derivative_matrix(m, D, x), "hf_derivative_matrix")
    return np.array(list(x)), np.array(list(D)).reshape(m, m)


def partition(pr: hf_problem, n_parts: int, part: int):
    """Contiguous group-aligned slice (e_begin, n_elem, word_offset) of part `part`."""
    e0, ne, wo = C.c_int64(), C.c_int64(), C.c_int64()
    check(_lib.load().hf_partition(C.byref(pr), n_parts, part, C.byref(e0), C.byref(ne), C.byref(wo)),
          "hf_partition")
    return int(e0.value), int(ne.value), int(wo.value)


def _ptr(x) -> int:
    if x is None:
        return 0
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        return int(x.data_ptr())
    raise TypeError("expected a device pointer (int) or a torch tensor")


def _stream(stream) -> int:
    if stream is None:
        import torch
        return int(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return stream
    return int(stream.cuda_stream)


def fused_divergence_device(pr: hf_problem, u, out, stream=None) -> None:
    """(b3)/(b2): u, out are device buffers (torch CUDA tensors or raw pointers) of
    ``field_words(pr)`` words of the problem's precision.  Asynchronous on `stream`."""
    check(_lib.load().hf_fused_divergence(C.byref(pr), _ptr(u), _ptr(out), _stream(stream)), "hf_fused_divergence")


# ---- extension: elements with a non-constant Jacobian (include/hexfuse_b200.h)
def geometry_words(pr: hf_problem) -> int:
    """Words of the corner array: 2^d corners x d coordinates per element, AoSoA with the field's group."""
    return int(_lib.load().hf_geometry_words(C.byref(pr)))


def fused_divergence_mapped_device(pr: hf_problem, u, geom, out, stream=None) -> None:
    """Fused divergence on (bi/tri)linear elements given by their corners: out = -(1/|J|) sum_a D_a(adj(J)_a. F)
    (+ source); pr.jac and pr.method are ignored.  Device buffers, asynchronous on `stream`."""
    check(_lib.load().hf_fused_divergence_mapped(C.byref(pr), _ptr(u), _ptr(geom), _ptr(out), _stream(stream)),
          "hf_fused_divergence_mapped")


def mapped_kernel_info(pr: hf_problem) -> dict:
    ki = hf_kernel_info()
    check(_lib.load().hf_mapped_kernel_info(C.byref(pr), C.byref(ki)), "hf_mapped_kernel_info")
    return {"elems_per_cta": ki.elems_per_cta, "block_threads": ki.block_threads, "shared_bytes": ki.shared_bytes,
            "registers": ki.registers, "grid": int(ki.grid), "bulk_path": bool(ki.bulk_path),
            "blocks_per_sm": ki.blocks_per_sm, "name": ki.name.decode()}


# ---- extension: FR stages 1 / 4+5 around the fused kernel (include/hexfuse_b200.h)
def face_words(pr: hf_problem) -> int:
    """Words of the face array U_f: 2 d m^(d-1) n_v per element, AoSoA with the field's group."""
    return int(_lib.load().hf_face_words(C.byref(pr)))


def make_mesh(dims, d: int, e_begin: int = 0, n_local: int | None = None, layer: int = 0):
    ms = _lib.hf_mesh()
    for a in range(3):
        ms.dims[a] = int(dims[a]) if a < len(dims) else 1
    if d == 2:
        ms.dims[2] = 1
    n_mesh = ms.dims[0] * ms.dims[1] * ms.dims[2]
    ms.e_begin, ms.n_local, ms.layer = int(e_begin), int(n_mesh if n_local is None else n_local), int(layer)
    return ms


def fr_project_device(pr: hf_problem, u, uf, stream=None) -> None:
    """Stage 1: every a-line extrapolated to xi_a = -1, +1 into the face array."""
    check(_lib.load().hf_fr_project(C.byref(pr), _ptr(u), _ptr(uf), _stream(stream)), "hf_fr_project")


def fr_correct_device(pr: hf_problem, mesh, uf, out, ghost_lo=None, ghost_hi=None, stream=None) -> None:
    """Stages 4+5 in place on `out` (which holds the fused kernel's result)."""
    check(_lib.load().hf_fr_correct(C.byref(pr), C.byref(mesh), _ptr(uf),
                                    _ptr(ghost_lo) if ghost_lo is not None else None,
                                    _ptr(ghost_hi) if ghost_hi is not None else None, _ptr(out), _stream(stream)),
          "hf_fr_correct")


def fr_divergence_faces_device(pr: hf_problem, u, uf, out, stream=None) -> None:
    """Stages 1+2+3+6 in one pass: the fused divergence into `out` and the faces
    into `uf` (bit-identical to fused_divergence_device + fr_project_device)."""
    check(_lib.load().hf_fr_divergence_faces(C.byref(pr), _ptr(u), _ptr(uf), _ptr(out), _stream(stream)),
          "hf_fr_divergence_faces")


def fr_residual_device(pr: hf_problem, dims, u, uf, out, stream=None) -> None:
    """The FR right-hand side (stages 1-6) on the periodic dims mesh, one device."""
    d3 = (C.c_int * 3)(*(list(dims) + [1] * (3 - len(dims))))
    check(_lib.load().hf_fr_residual(C.byref(pr), d3, _ptr(u), _ptr(uf), _ptr(out), _stream(stream)),
          "hf_fr_residual")


def ipc_handle(dev) -> tuple[bytes, int]:
    """CUDA IPC handle (64 bytes) of the allocation holding `dev`, and dev's byte offset in it."""
    buf = (C.c_char * 64)()
    off = C.c_int64()
    check(_lib.load().hf_ipc_handle(_ptr(dev), buf, C.byref(off)), "hf_ipc_handle")
    return bytes(buf), int(off.value)


def ipc_open(handle: bytes) -> int:
    """Map a peer process's allocation; returns its device address in this process."""
    out = C.c_void_p()
    buf = (C.c_char * 64).from_buffer_copy(handle)
    check(_lib.load().hf_ipc_open(buf, C.byref(out)), "hf_ipc_open")
    return int(out.value)


def ipc_close(ptr: int) -> None:
    check(_lib.load().hf_ipc_close(C.c_void_p(ptr)), "hf_ipc_close")


def fused_divergence_variant(pr: hf_problem, method: Method, variant: int, u, out, stream=None) -> None:
    """Tuning hook: launch a specific method/variant, bypassing the selection table."""
    check(_lib.load().hf_fused_divergence_variant(C.byref(pr), int(method), int(variant), _ptr(u), _ptr(out),
                                                  _stream(stream), None), "hf_fused_divergence_variant")


def variant_info(pr: hf_problem, method: Method, variant: int) -> dict:
    ki = hf_kernel_info()
    check(_lib.load().hf_fused_divergence_variant(C.byref(pr), int(method), int(variant), 0, 0, 0, C.byref(ki)),
          "hf_fused_divergence_variant(info)")
    return {"method": Method(ki.method).name, "elems_per_cta": ki.elems_per_cta, "block_threads": ki.block_threads,
            "shared_bytes": ki.shared_bytes, "registers": ki.registers, "grid": int(ki.grid),
            "bulk_path": bool(ki.bulk_path), "blocks_per_sm": ki.blocks_per_sm, "name": ki.name.decode()}


def unfused_workspace_bytes(pr: hf_problem) -> int:
    return int(_lib.load().hf_unfused_workspace_bytes(C.byref(pr)))


def unfused_divergence_device(pr: hf_problem, u, out, ws, stream=None) -> None:
    check(_lib.load().hf_unfused_divergence(C.byref(pr), _ptr(u), _ptr(out), _ptr(ws), _stream(stream)),
          "hf_unfused_divergence")


class Context:
    """Owns device staging buffers and streams for the host-buffer path."""

    def __init__(self, device: int = 0):
        self._h = _lib.load().hf_context_create(int(device))
        if not self._h:
            raise HexfuseError("hf_context_create: " + _lib.load().hf_last_error().decode())

    def close(self) -> None:
        if self._h:
            _lib.load().hf_context_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def run(self, pr: hf_problem, u_host: np.ndarray, out_host: np.ndarray) -> None:
        """Host arrays (float32 for fp32, float64 for fp64), e.g. pinned torch CPU tensors' numpy views."""
        check(_lib.load().hf_fused_divergence_host(self._h, C.byref(pr), _host_ptr(u_host), _host_ptr(out_host)),
              "hf_fused_divergence_host")

    def run_batch(self, items) -> None:
        """[(problem, u_host, out_host), ...] through one copy pipeline (hf_fused_divergence_host_batch)."""
        items = list(items)
        n = len(items)
        prs = (hf_problem * n)(*[it[0] for it in items])
        us = (C.c_void_p * n)(*[_host_ptr(it[1]) for it in items])
        outs = (C.c_void_p * n)(*[_host_ptr(it[2]) for it in items])
        check(_lib.load().hf_fused_divergence_host_batch(self._h, n, prs, us, outs), "hf_fused_divergence_host_batch")


def _host_ptr(a) -> int:
    if hasattr(a, "data_ptr"):
        return int(a.data_ptr())
    return int(a.ctypes.data)


_tls = threading.local()


def _context() -> Context:
    c = getattr(_tls, "ctx", None)
    if c is None:
        import torch
        c = Context(torch.cuda.current_device() if torch.cuda.is_available() else 0)
        _tls.ctx = c
    return c


def fused_divergence(U: StateField, params: PhysParams, jac: Sequence[float] = (1.0, 1.0, 1.0),
                     with_source: bool = False, method: Method = Method.auto) -> StateField:
    """Drop-in for ``oracle_divergence(U, params, jac, with_source)`` (oracle.hpp:20-62):
    returns a new StateField of U's shape and group, padding zeroed, computed by the
    B200 kernels through the host-buffer C ABI."""
    params.validate()
    pr = problem_for(U, params, jac, with_source, method)
    validate(pr)
    out = StateField(U.d, U.p, U.n_elem, U.group, U.precision)
    if U.n_elem == 0:
        return out
    if method == Method.unfused:
        return _unfused_host(U, pr, out)
    src = U.words()
    dst = np.zeros_like(src)
    _context().run(pr, src, dst)
    out.data = dst.astype(np.float64)
    return out


def _unfused_host(U: StateField, pr: hf_problem, out: StateField) -> StateField:
    import torch
    dt = torch.float32 if U.precision == Precision.fp32 else torch.float64
    u = torch.from_numpy(U.words().copy()).to("cuda")
    o = torch.zeros_like(u)
    ws = torch.empty(unfused_workspace_bytes(pr) // u.element_size(), dtype=dt, device="cuda")
    unfused_divergence_device(pr, u, o, ws)
    out.data = o.cpu().numpy().astype(np.float64)
    return out
