"""ctypes front-end for the parity checkers.

TEST INFRASTRUCTURE ONLY.  Imported by tests/, ``__graft_entry__.smoke()`` and
``bench.py``'s cpu_baseline / ``--impl reference`` legs, and nowhere else.  The
product package ``paper_2107_14027_b200`` never imports this module.

Two libraries, both built by ``oracle/Makefile`` into ``oracle/_ref/``:

* ``libhexfuse_oracle.so`` -- the C restatement of the reference hot path
  (``oracle/hexfuse_oracle.c``), citing reference file:line per function.
* ``libhexfuse_ref.so`` -- the reference's own headers
  (``/root/reference/proj/include/hexfuse/oracle.hpp``, ``verify.hpp``)
  compiled in place through ``oracle/ref_shim.cpp``.  It travels to the GPU
  box prebuilt (``oracle/_ref`` is git-ignored, not gpurun-ignored).

All fields are flat float64 numpy arrays in the reference AoSoA order
(``StateField::offset``, layout.hpp:128-134), padded to ``n_groups*group_words``.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_REF_DIR = os.path.join(_HERE, "_ref")
_ORACLE_SO = os.path.join(_REF_DIR, "libhexfuse_oracle.so")
_REF_SO = os.path.join(_REF_DIR, "libhexfuse_ref.so")

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_i64 = C.c_int64


def build(quiet: bool = True) -> None:
    """Compile the restatement (always) and the reference shim (if /root/reference exists)."""
    out = subprocess.run(["make", "-C", _HERE, "all"], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)


def _load(path: str) -> C.CDLL:
    if not os.path.exists(path):
        build()
    return C.CDLL(path)


_lib = None
_ref = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        L = _load(_ORACLE_SO)
        L.hfo_n_vars.argtypes = [C.c_int]
        L.hfo_gauss_legendre_points.argtypes = [C.c_int, _dp]
        L.hfo_derivative_matrix.argtypes = [C.c_int, _dp, _dp]
        L.hfo_gl_derivative_matrix.argtypes = [C.c_int, _dp]
        L.hfo_flux.argtypes = [C.c_int, _dp, C.c_double, C.c_double, C.c_double, _dp]
        L.hfo_flux.restype = None
        L.hfo_source.argtypes = [C.c_int, _dp, C.c_double, _dp]
        L.hfo_source.restype = None
        L.hfo_flux_structural_nonzero.argtypes = [C.c_int, C.c_int, C.c_int]
        L.hfo_offset.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int]
        L.hfo_offset.restype = _i64
        L.hfo_field_words.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int]
        L.hfo_field_words.restype = _i64
        L.hfo_oracle_divergence.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, _dp, _dp, C.c_double,
                                            C.c_double, C.c_double, _dp, C.c_int]
        L.hfo_oracle_divergence_range.argtypes = [C.c_int, C.c_int, C.c_int, _dp, _dp, C.c_double,
                                                  C.c_double, C.c_double, _dp, C.c_int, C.c_int, C.c_int]
        L.hfo_mt19937_64_first.argtypes = [C.c_uint64, C.c_int]
        L.hfo_mt19937_64_first.restype = C.c_uint64
        L.hfo_random_field.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64, _dp]
        L.hfo_factor3.argtypes = [C.c_int, C.POINTER(C.c_int)]
        L.hfo_factor3.restype = None
        L.hfo_tgv_field.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_int), _dp, _dp, C.c_double, C.c_double,
                                    C.c_int, C.c_int, _dp]
        L.hfo_field_rel_error.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, _dp, _dp]
        L.hfo_field_rel_error.restype = C.c_double
        L.hfo_verify_tolerance.argtypes = [C.c_int]
        L.hfo_verify_tolerance.restype = C.c_double
        L.hfo_io_model.argtypes = [C.c_int, C.POINTER(C.c_int), C.c_int, C.POINTER(_i64), C.POINTER(_i64)]
        L.hfo_geometry_words.argtypes = [C.c_int, C.c_int, C.c_int]
        L.hfo_geometry_words.restype = _i64
        L.hfo_mapped_jacobian.argtypes = [C.c_int, _dp, _dp, _dp]
        L.hfo_mapped_jacobian.restype = None
        L.hfo_adjugate.argtypes = [C.c_int, _dp, _dp]
        L.hfo_adjugate.restype = C.c_double
        L.hfo_oracle_divergence_mapped.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, _dp, _dp, _dp, C.c_double,
                                                   C.c_double, C.c_double, C.c_int]
        L.hfo_face_words.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int]
        L.hfo_face_words.restype = _i64
        L.hfo_face_interp.argtypes = [C.c_int, _dp, _dp]
        L.hfo_correction_derivs.argtypes = [C.c_int, _dp, _dp]
        L.hfo_max_wavespeed.argtypes = [C.c_int, _dp, C.c_int, C.c_double, C.c_double, C.c_double]
        L.hfo_max_wavespeed.restype = C.c_double
        L.hfo_common_flux.argtypes = [C.c_int, _dp, _dp, C.c_int, C.c_double, C.c_double, C.c_double, _dp]
        L.hfo_common_flux.restype = None
        L.hfo_project_faces.argtypes = [C.c_int, C.c_int, C.c_int, _dp, _dp, C.c_int, C.c_int]
        L.hfo_fr_correct.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int), _dp, _dp, C.c_double, C.c_double,
                                     C.c_double, _dp, C.c_int, C.c_int]
        L.hfo_fr_residual.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_int), C.c_int, _dp, _dp, C.c_double,
                                      C.c_double, C.c_double, _dp, C.c_int]
        _lib = L
    return _lib


def ref_available() -> bool:
    return os.path.exists(_REF_SO)


def host_cpu() -> dict:
    """Model name, logical CPUs usable by this process and the ISA flags of the host."""
    model, flags = "unknown", set()
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name") and model == "unknown":
                    model = line.split(":", 1)[1].strip()
                elif line.startswith("flags") and not flags:
                    flags = set(line.split(":", 1)[1].split())
    except OSError:
        pass
    try:
        usable = len(os.sched_getaffinity(0))
    except AttributeError:
        usable = os.cpu_count() or 1
    return {"model": model, "logical_cpus": usable, "flags": flags}


_V3 = {"avx", "avx2", "bmi1", "bmi2", "f16c", "fma", "movbe", "xsave"}
_V4 = _V3 | {"avx512f", "avx512bw", "avx512cd", "avx512dq", "avx512vl"}
_timing = None


def ref_timing():
    """(library, build description) for TIMING the reference's oracle_divergence on this
    host: the -O3 -march=x86-64-v4 / -v3 build of the same shim (what -march=native gives
    on an AVX-512 / AVX2 host), else the portable parity build.  Never used for parity."""
    global _timing
    if _timing is None:
        flags = host_cpu()["flags"]
        path, desc = _REF_SO, "-O3 -ffp-contract=off (portable parity build)"
        for isa, need in (("x86-64-v4", _V4), ("x86-64-v3", _V3)):
            cand = os.path.join(_REF_DIR, f"libhexfuse_ref_{isa}.so")
            if need <= flags and os.path.exists(cand):
                path, desc = cand, f"-O3 -march={isa}"
                break
        if not os.path.exists(path):
            raise RuntimeError("oracle/_ref/libhexfuse_ref*.so missing (reference tree absent at build time)")
        R = C.CDLL(path)
        R.ref_last_error.restype = C.c_char_p
        R.ref_random_field.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_ulonglong, _dp]
        R.ref_time_oracle_mt.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _dp, _dp, C.c_double,
                                         C.c_double, C.c_double, _dp, C.c_int, C.c_int]
        R.ref_time_oracle_mt.restype = C.c_double
        _timing = (R, desc)
    return _timing


def ref() -> C.CDLL:
    """The reference's own oracle (compiled in place).  Raises if never built."""
    global _ref
    if _ref is None:
        if not os.path.exists(_REF_SO):
            build()
        if not os.path.exists(_REF_SO):
            raise RuntimeError("oracle/_ref/libhexfuse_ref.so missing (reference tree absent at build time)")
        R = C.CDLL(_REF_SO)
        R.ref_last_error.restype = C.c_char_p
        R.ref_random_field.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_ulonglong, _dp]
        R.ref_tgv_field.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, _dp]
        R.ref_factor3.argtypes = [C.c_int, C.POINTER(C.c_int)]
        R.ref_factor3.restype = None
        R.ref_oracle_divergence.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _dp, _dp, C.c_double,
                                            C.c_double, C.c_double, _dp, C.c_int]
        R.ref_field_rel_error.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, _dp, _dp]
        R.ref_field_rel_error.restype = C.c_double
        R.ref_gl_derivative.argtypes = [C.c_int, _dp, _dp]
        R.ref_derivative_matrix.argtypes = [C.c_int, _dp, _dp]
        R.ref_time_oracle_mt.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _dp, _dp, C.c_double,
                                         C.c_double, C.c_double, _dp, C.c_int, C.c_int]
        R.ref_time_oracle_mt.restype = C.c_double
        R.ref_export_blob.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _dp, C.c_char_p]
        R.ref_import_blob.argtypes = [C.c_char_p, C.POINTER(C.c_int), C.c_void_p, C.c_longlong]
        R.ref_import_blob.restype = C.c_longlong
        R.ref_max_abs_eigenvalue.argtypes = [C.c_int, _dp, C.c_int, C.c_double, C.c_double, C.c_double]
        R.ref_max_abs_eigenvalue.restype = C.c_double
        _ref = R
    return _ref


# ----------------------------------------------------------------------------------------------
# numpy wrappers over the restatement
# ----------------------------------------------------------------------------------------------

def n_vars(d: int) -> int:
    return 1 + d + d * d


def n_points(d: int, p: int) -> int:
    return (p + 1) ** d


def field_words(d: int, p: int, n_elem: int, group: int) -> int:
    return int(lib().hfo_field_words(d, p, n_elem, group))


def gl_nodes(m: int) -> np.ndarray:
    x = np.zeros(m)
    if lib().hfo_gauss_legendre_points(m, x) != 0:
        raise ValueError("gauss_legendre_points: m out of range")
    return x


def derivative_matrix(nodes: np.ndarray) -> np.ndarray:
    nodes = np.ascontiguousarray(nodes, dtype=np.float64)
    m = len(nodes)
    D = np.zeros(m * m)
    if lib().hfo_derivative_matrix(m, nodes, D) != 0:
        raise ValueError("derivative_matrix: duplicate nodes")
    return D.reshape(m, m)


def flux(d: int, s, nu: float, zeta: float, T: float) -> np.ndarray:
    s = np.ascontiguousarray(s, dtype=np.float64)
    f = np.zeros(d * n_vars(d))
    lib().hfo_flux(d, s, nu, zeta, T, f)
    return f.reshape(d, n_vars(d))


def source(d: int, s, T: float) -> np.ndarray:
    s = np.ascontiguousarray(s, dtype=np.float64)
    out = np.zeros(n_vars(d))
    lib().hfo_source(d, s, T, out)
    return out


def random_field(d: int, p: int, n_elem: int, group: int, fp32: bool, seed: int) -> np.ndarray:
    out = np.zeros(field_words(d, p, n_elem, group))
    lib().hfo_random_field(d, p, n_elem, group, int(fp32), seed, out)
    return out


def factor3(n: int):
    o = (C.c_int * 3)()
    lib().hfo_factor3(n, o)
    return [o[0], o[1], o[2]]


def tgv_field(p: int, n_elem: int, group: int, fp32: bool, width: float = 2.0, zero_mean_pressure: bool = True,
              elems=None, origin=(0.0, 0.0, 0.0)) -> np.ndarray:
    """oracle.hpp:116-151 on a factor3(n_elem) brick (verify.hpp:85-91 uses width 2)."""
    el = factor3(n_elem) if elems is None else list(elems)
    assert el[0] * el[1] * el[2] == n_elem
    out = np.zeros(field_words(3, p, n_elem, group))
    e3 = (C.c_int * 3)(*el)
    if lib().hfo_tgv_field(p, group, e3, np.array(origin, dtype=np.float64), np.array([width] * 3), 1.4, 0.08,
                           int(zero_mean_pressure), int(fp32), out) != 0:
        raise ValueError("tgv_field")
    return out


def oracle_divergence(d: int, p: int, n_elem: int, group: int, U: np.ndarray, nu: float, zeta: float, T: float,
                      jac=(1.0, 1.0, 1.0), with_source: bool = False) -> np.ndarray:
    U = np.ascontiguousarray(U, dtype=np.float64)
    assert U.size == field_words(d, p, n_elem, group)
    out = np.zeros_like(U)
    rc = lib().hfo_oracle_divergence(d, p, n_elem, group, U, out, nu, zeta, T,
                                     np.array(jac, dtype=np.float64), int(with_source))
    if rc != 0:
        raise ValueError("oracle_divergence: invalid arguments")
    return out


def oracle_divergence_elements(d: int, p: int, group: int, U: np.ndarray, out: np.ndarray, nu: float, zeta: float,
                               T: float, jac, with_source: bool, e_begin: int, e_end: int) -> None:
    """Compute only elements [e_begin, e_end) into ``out`` (used for sampled parity at scale)."""
    rc = lib().hfo_oracle_divergence_range(d, p, group, U, out, nu, zeta, T, np.array(jac, dtype=np.float64),
                                           int(with_source), e_begin, e_end)
    if rc != 0:
        raise ValueError("oracle_divergence_range: invalid arguments")


# ---- extension: (bi/tri)linear elements with a non-constant Jacobian (hexfuse_oracle.c)
def geometry_words(d: int, n_elem: int, group: int) -> int:
    return int(lib().hfo_geometry_words(d, n_elem, group))


def geom_offset(d: int, group: int, e: int, c: int, x: int) -> int:
    """AoSoA word of corner c (bit k = +xi_k side), coordinate x, of element e."""
    nc = 1 << d
    return (e // group) * group * nc * d + e % group + group * (x + d * c)


def box_geometry(d: int, n_elem: int, group: int, h, origin=None) -> np.ndarray:
    """Axis-aligned boxes of half-widths h (element e shifted by 2*h_0*e along x)."""
    G = np.zeros(geometry_words(d, n_elem, group))
    for e in range(n_elem):
        for c in range(1 << d):
            for x in range(d):
                s = 1.0 if (c >> x) & 1 else -1.0
                base = (origin[x] if origin is not None else 0.0) + (2.0 * h[0] * e if x == 0 else 0.0)
                G[geom_offset(d, group, e, c, x)] = base + s * h[x]
    return G


def random_geometry(d: int, n_elem: int, group: int, seed: int, h=(0.5, 0.7, 0.9), amp: float = 0.15,
                    fp32: bool = False) -> np.ndarray:
    """Boxes of half-widths h with every corner displaced by U(-amp, amp) * h (curved trilinear
    elements, positive Jacobian for amp < 1/3); quantised to float for FP32 problems."""
    rng = np.random.default_rng(seed)
    G = box_geometry(d, n_elem, group, h)
    for e in range(n_elem):
        for c in range(1 << d):
            for x in range(d):
                G[geom_offset(d, group, e, c, x)] += rng.uniform(-amp, amp) * h[x]
    if fp32:
        G = G.astype(np.float32).astype(np.float64)
    return G


def oracle_divergence_mapped(d: int, p: int, n_elem: int, group: int, U: np.ndarray, G: np.ndarray, nu: float,
                             zeta: float, T: float, with_source: bool = False) -> np.ndarray:
    U = np.ascontiguousarray(U, dtype=np.float64)
    G = np.ascontiguousarray(G, dtype=np.float64)
    assert U.size == field_words(d, p, n_elem, group) and G.size == geometry_words(d, n_elem, group)
    out = np.zeros_like(U)
    if lib().hfo_oracle_divergence_mapped(d, p, n_elem, group, U, G, out, nu, zeta, T, int(with_source)) != 0:
        raise ValueError("oracle_divergence_mapped: invalid arguments")
    return out


# ---- extension: the adjacent FR stages 1/4/5 on a periodic structured mesh
def face_words(d: int, p: int, n_elem: int, group: int) -> int:
    return int(lib().hfo_face_words(d, p, n_elem, group))


def face_interp(m: int):
    lm, lp = np.zeros(m), np.zeros(m)
    lib().hfo_face_interp(m, lm, lp)
    return lm, lp


def correction_derivs(m: int):
    gl, gr = np.zeros(m), np.zeros(m)
    lib().hfo_correction_derivs(m, gl, gr)
    return gl, gr


def max_wavespeed(d: int, s, a: int, nu: float, zeta: float, T: float) -> float:
    return float(lib().hfo_max_wavespeed(d, np.ascontiguousarray(s, dtype=np.float64), a, nu, zeta, T))


def common_flux(d: int, UL, UR, a: int, nu: float, zeta: float, T: float) -> np.ndarray:
    out = np.zeros(1 + d + d * d)
    lib().hfo_common_flux(d, np.ascontiguousarray(UL, dtype=np.float64), np.ascontiguousarray(UR, dtype=np.float64),
                          a, nu, zeta, T, out)
    return out


def project_faces(d: int, p: int, n_elem: int, group: int, U: np.ndarray) -> np.ndarray:
    Uf = np.zeros(face_words(d, p, n_elem, group))
    lib().hfo_project_faces(d, p, group, np.ascontiguousarray(U, dtype=np.float64), Uf, 0, n_elem)
    return Uf


def fr_correct(d: int, p: int, group: int, dims, Uf: np.ndarray, out: np.ndarray, nu: float, zeta: float, T: float,
               jac, e_begin: int, e_end: int) -> None:
    """Stages 4+5 in place on ``out`` for elements [e_begin, e_end) of the whole-mesh arrays."""
    dims3 = (C.c_int * 3)(*(list(dims) + [1] * (3 - len(dims))))
    if lib().hfo_fr_correct(d, p, group, dims3, Uf, out, nu, zeta, T, np.array(jac, dtype=np.float64),
                            e_begin, e_end) != 0:
        raise ValueError("fr_correct: invalid arguments")


def fr_residual(d: int, p: int, dims, group: int, U: np.ndarray, nu: float, zeta: float, T: float,
                jac=(1.0, 1.0, 1.0), with_source: bool = False) -> np.ndarray:
    """Stages 1-6 of PAPER.md Table 1 on the periodic nx x ny (x nz) mesh."""
    dims3 = (C.c_int * 3)(*(list(dims) + [1] * (3 - len(dims))))
    n = int(np.prod(dims[:d]))
    U = np.ascontiguousarray(U, dtype=np.float64)
    assert U.size == field_words(d, p, n, group)
    out = np.zeros_like(U)
    if lib().hfo_fr_residual(d, p, dims3, group, U, out, nu, zeta, T, np.array(jac, dtype=np.float64),
                             int(with_source)) != 0:
        raise ValueError("fr_residual: invalid arguments")
    return out


def ref_max_abs_eigenvalue(d: int, s, a: int, nu: float, zeta: float, T: float) -> float:
    return float(ref().ref_max_abs_eigenvalue(d, np.ascontiguousarray(s, dtype=np.float64), a, nu, zeta, T))


def field_rel_error(d: int, p: int, n_elem: int, group: int, got: np.ndarray, ref_: np.ndarray) -> float:
    return float(lib().hfo_field_rel_error(d, p, n_elem, group, np.ascontiguousarray(got, dtype=np.float64),
                                           np.ascontiguousarray(ref_, dtype=np.float64)))


def verify_tolerance(fp32: bool) -> float:
    return float(lib().hfo_verify_tolerance(int(fp32)))


def io_model(d: int, stages) -> tuple[int, int]:
    """stages: iterable of 'S2','S3','S6','Fused23','Fused236' (io_model.hpp:27-40)."""
    code = {"S2": 0, "S3": 1, "S6": 2, "Fused23": 3, "Fused236": 4}
    arr = (C.c_int * len(stages))(*[code[s] for s in stages])
    r, w = _i64(), _i64()
    if lib().hfo_io_model(d, arr, len(stages), C.byref(r), C.byref(w)) != 0:
        raise ValueError("io_model: bad dimension or stage")
    return int(r.value), int(w.value)


# ----------------------------------------------------------------------------------------------
# numpy wrappers over the reference itself
# ----------------------------------------------------------------------------------------------

def ref_random_field(d, p, n_elem, group, fp32, seed) -> np.ndarray:
    out = np.zeros(field_words(d, p, n_elem, group))
    if ref().ref_random_field(d, p, n_elem, group, int(fp32), seed, out) != 0:
        raise ValueError(ref().ref_last_error().decode())
    return out


def ref_tgv_field(p, n_elem, group, fp32, width=2.0, zero_mean_pressure=True) -> np.ndarray:
    out = np.zeros(field_words(3, p, n_elem, group))
    if ref().ref_tgv_field(p, n_elem, group, int(fp32), width, int(zero_mean_pressure), out) != 0:
        raise ValueError(ref().ref_last_error().decode())
    return out


def ref_oracle_divergence(d, p, n_elem, group, fp32, U, nu, zeta, T, jac=(1.0, 1.0, 1.0), with_source=False):
    U = np.ascontiguousarray(U, dtype=np.float64)
    out = np.zeros_like(U)
    rc = ref().ref_oracle_divergence(d, p, n_elem, group, int(fp32), U, out, nu, zeta, T,
                                     np.array(jac, dtype=np.float64), int(with_source))
    if rc != 0:
        raise ValueError(ref().ref_last_error().decode())
    return out


def ref_time_oracle_mt(d, p, n_elem, group, fp32, U, nu, zeta, T, jac=(1.0, 1.0, 1.0), with_source=False,
                       n_threads=1, timing_build=False):
    """Returns (seconds, out) for the reference oracle run on n_threads group-aligned sub-fields
    (timing_build: the -march build of ref_timing() instead of the parity build)."""
    R = ref_timing()[0] if timing_build else ref()
    U = np.ascontiguousarray(U, dtype=np.float64)
    out = np.zeros_like(U)
    t = R.ref_time_oracle_mt(d, p, n_elem, group, int(fp32), U, out, nu, zeta, T,
                             np.array(jac, dtype=np.float64), int(with_source), n_threads)
    if t < 0:
        raise RuntimeError(R.ref_last_error().decode())
    return t, out


def ref_random_field_timing(d, p, n_elem, group, fp32, seed) -> np.ndarray:
    """hexfuse::random_field through the timing build (no other library loaded)."""
    R = ref_timing()[0]
    nv = 1 + d + d * d
    words = -(-n_elem // group) * group * (p + 1) ** d * nv
    out = np.zeros(words)
    if R.ref_random_field(d, p, n_elem, group, int(fp32), seed, out) != 0:
        raise ValueError(R.ref_last_error().decode())
    return out


def ref_export_blob(d, p, n_elem, group, fp32, data, path: str) -> None:
    """hexfuse::export_blob (layout.hpp:161-177): flat little-endian words + <path>.json."""
    data = np.ascontiguousarray(data, dtype=np.float64)
    if ref().ref_export_blob(d, p, n_elem, group, int(fp32), data, path.encode()) != 0:
        raise RuntimeError(ref().ref_last_error().decode())


def ref_import_blob(path: str):
    """hexfuse::import_blob (layout.hpp:179-200) -> (d, p, n_elem, group, fp32, data float64)."""
    shape = (C.c_int * 5)()
    n = ref().ref_import_blob(path.encode(), shape, None, 0)
    if n < 0:
        raise RuntimeError(ref().ref_last_error().decode())
    out = np.zeros(n)
    ref().ref_import_blob(path.encode(), shape, out.ctypes.data, n)
    return shape[0], shape[1], shape[2], shape[3], bool(shape[4]), out


def ref_derivative_matrix(nodes) -> np.ndarray:
    """The reference's derivative_matrix (operators.hpp:49-74) on the given nodes."""
    x = np.ascontiguousarray(nodes, dtype=np.float64)
    D = np.zeros(x.size * x.size)
    if ref().ref_derivative_matrix(x.size, x, D) != 0:
        raise ValueError(ref().ref_last_error().decode())
    return D.reshape(x.size, x.size)


def ref_gl_derivative(m: int):
    x = np.zeros(m)
    D = np.zeros(m * m)
    if ref().ref_gl_derivative(m, x, D) != 0:
        raise ValueError(ref().ref_last_error().decode())
    return x, D.reshape(m, m)
