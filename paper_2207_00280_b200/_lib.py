"""Loader and thin typed wrappers for ``lib/libiga_b200.so`` (the C-ABI in
``include/iga_b200.h``).

The product path has no CPU fallback: if the library is missing or no CUDA
device is present, every entry point raises.  Status codes map to the
reference's exception conventions: invalid arguments -> ``ValueError``
(integrators.py:180-190, assembly.py:22-24), CUDA failures -> ``RuntimeError``.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
# IGA_LIB_PATH: load another build of the same ABI (tuning experiments: tools/gsf_variants.sh)
LIB_PATH = os.environ.get("IGA_LIB_PATH") or os.path.join(_HERE, "lib", "libiga_b200.so")
CSRC = os.path.join(_HERE, "csrc")

IGA_OK, IGA_EINVAL, IGA_ECUDA, IGA_EUNSUPPORTED, IGA_ENOCONV = 0, 1, 2, 3, 4
OPS = {"mass": 0, "stiffness": 1, "stiffness_mass": 2}
METHOD_CLASSICAL, METHOD_SUMFACT, METHOD_SUMFACT_ASSEMBLED, METHOD_SEPARABLE = 0, 1, 2, 3

# Every symbol include/iga_b200.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "iga_last_error",
    "iga_abi_version",
    "iga_mesh_tables",
    "iga_mesh_tables_general",
    "iga_band_tables",
    "iga_basis_eval",
    "iga_eval_basis",
    "iga_csr_nnz",
    "iga_csr_pattern",
    "iga_element_matrices",
    "iga_integrate_assemble",
    "iga_assemble_elements",
    "iga_axpy",
    "iga_spmv",
    "iga_apply",
    "iga_write_matrix_market",
    "iga_write_matrix_market_host",
    "iga_cg_work_size",
    "iga_cg",
)


class IgaProblem(ctypes.Structure):
    """Mirror of ``struct iga_problem`` (include/iga_b200.h)."""

    _fields_ = [
        ("dim", ctypes.c_int32),
        ("K", ctypes.c_int32),
        ("p", ctypes.c_int32),
        ("q", ctypes.c_int32),
        ("op", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
        ("jac", ctypes.c_double),
        ("coef_scalar", ctypes.c_double),
        ("coef", ctypes.c_void_p),
        ("weights", ctypes.c_void_p),
        ("tables_v", ctypes.c_void_p),
        ("tables_d", ctypes.c_void_p),
        ("band", ctypes.c_void_p),
        ("knots", ctypes.c_void_p),
        ("elem_weights", ctypes.c_void_p),
    ]


_lib = None


def build(force: bool = False) -> str:
    """Compile the sm_100a library in-tree with nvcc (csrc/Makefile)."""
    if force or not os.path.exists(LIB_PATH):
        subprocess.run(["make", "-s", "-j8", "-C", CSRC], check=True)
    return LIB_PATH


def load():
    """Load the shared library and declare argument types (no CUDA needed)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"libiga_b200.so not found at {LIB_PATH}; build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")
    L = ctypes.CDLL(LIB_PATH)
    vp, i32, i64, dp = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    L.iga_last_error.restype = ctypes.c_char_p
    L.iga_abi_version.restype = i32
    L.iga_mesh_tables.argtypes = [i32, i32, i32, vp, vp, vp, vp]
    L.iga_band_tables.argtypes = [ctypes.POINTER(IgaProblem), vp, vp, vp, vp, vp, vp]
    L.iga_mesh_tables_general.argtypes = [i32, i32, i32, vp, vp, vp, vp, vp, vp, vp]
    L.iga_basis_eval.argtypes = [i32, i32, vp, i64, vp, vp, vp, vp, vp]
    L.iga_eval_basis.argtypes = [vp, i32, i32, i64, vp, vp, vp, vp]
    L.iga_csr_nnz.argtypes = [i32, i32, i32, i64, i64]
    L.iga_csr_nnz.restype = i64
    L.iga_csr_pattern.argtypes = [i32, i32, i32, i64, i64, vp, vp, vp]
    L.iga_element_matrices.argtypes = [ctypes.POINTER(IgaProblem), i32, vp, vp, vp, vp, vp, i64,
                                       vp, vp]
    L.iga_integrate_assemble.argtypes = [ctypes.POINTER(IgaProblem), i32, i32, i32, i32, i32, vp,
                                         vp]
    L.iga_assemble_elements.argtypes = [i32, i32, i32, vp, i32, i32, vp, vp]
    L.iga_axpy.argtypes = [i64, vp, vp, vp]
    L.iga_spmv.argtypes = [i32, i32, i32, vp, vp, vp, vp]
    L.iga_apply.argtypes = [ctypes.POINTER(IgaProblem), dp, dp, vp, vp, vp]
    L.iga_write_matrix_market.argtypes = [i32, i32, i32, vp, ctypes.c_char_p, i32, vp]
    L.iga_write_matrix_market_host.argtypes = [i32, i32, i32, vp, ctypes.c_char_p, i32]
    L.iga_cg_work_size.argtypes = [i64]
    L.iga_cg_work_size.restype = i64
    L.iga_cg.argtypes = [i32, i32, i32, vp, ctypes.POINTER(IgaProblem), dp, dp, i64, vp, vp, vp, dp,
                         i64, i32, ctypes.POINTER(i64), vp]
    for name in ("iga_mesh_tables", "iga_mesh_tables_general", "iga_band_tables", "iga_basis_eval", "iga_eval_basis", "iga_csr_pattern", "iga_element_matrices",
                 "iga_integrate_assemble", "iga_assemble_elements", "iga_axpy", "iga_spmv",
                 "iga_apply", "iga_write_matrix_market", "iga_write_matrix_market_host", "iga_cg"):
        getattr(L, name).restype = i32
    if L.iga_abi_version() != 5:
        raise ImportError("libiga_b200.so ABI version mismatch")
    _lib = L
    return L


def check(rc: int) -> None:
    if rc == IGA_OK:
        return
    msg = load().iga_last_error().decode(errors="replace")
    if rc in (IGA_EINVAL, IGA_EUNSUPPORTED):
        raise ValueError(msg)
    if rc == IGA_ENOCONV:
        raise RuntimeError(msg)
    raise RuntimeError(f"CUDA failure in libiga_b200: {msg}")


def require_cuda():
    """The device path needs a CUDA device; there is no CPU fallback."""
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_2207_00280_b200 requires a CUDA device (B200, sm_100a); "
                           "no CPU fallback exists")
    load()
    return torch


def ptr(t) -> int | None:
    """Raw device pointer of a torch tensor (None for None)."""
    return None if t is None else t.data_ptr()


def stream_ptr(stream=None) -> int:
    import torch

    s = torch.cuda.current_stream() if stream is None else stream
    return s.cuda_stream
