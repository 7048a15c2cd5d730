"""Global CSR assembly (drop-in for igabench.assembly).

The global matrix lives on the device as a structured CSR (full symmetric,
sorted columns, the layout assembly.py:80-82 produces).  ``GlobalGram.matrix``
materialises the scipy ``csr_matrix`` lazily (one device->host copy);
``assemble`` scatters host element matrices on the device with a
deterministic lexicographic-element-order gather (kernel
``iga_assemble_elements``).
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .device import csr_nnz, csr_pattern, n_dofs as _n_dofs
from .integrators import ElementMatrix
from .mesh import ElementId, element_list, support_set


def dof_index(beta: tuple[int, int, int], K: int, p: int) -> int:
    """Lexicographic flat index over (K+p)^3 (assembly.py:19-25)."""
    n1d = K + p
    for c in beta:
        if not 0 <= c < n1d:
            raise ValueError(f"multi-index {beta} out of range for K={K}, p={p}")
    return (beta[0] * n1d + beta[1]) * n1d + beta[2]


def element_dofs(alpha: ElementId, K: int, p: int) -> np.ndarray:
    return np.array([dof_index(b, K, p) for b in support_set(alpha, p)], dtype=np.int64)


_PATTERN_CACHE: dict = {}


def host_pattern(dim: int, K: int, p: int):
    """Host copy of the structured pattern (K5 on the device, copied once and cached
    per (dim, K, p), like the reference caches canonical_pairs)."""
    key = (dim, K, p)
    if key not in _PATTERN_CACHE:
        pat = csr_pattern(dim, K, p)
        nnz = int(pat.indptr[-1].item())
        idx_dtype = np.int32 if nnz < 2**31 else np.int64
        indptr = pat.indptr.cpu().numpy().astype(idx_dtype)
        indices = pat.indices.cpu().numpy().astype(idx_dtype, copy=False)
        _PATTERN_CACHE[key] = (indptr, indices)
    return _PATTERN_CACHE[key]


class GlobalGram:
    """Assembled global matrix: device CSR values + lazily materialised scipy CSR.

    Fields match the reference dataclass (assembly.py:28-38): K, p, n_dofs, matrix.
    """

    def __init__(self, K: int, p: int, n_dofs: int, values=None, dim: int = 3, matrix=None,
                 shards=None):
        self.K, self.p, self.n_dofs, self.dim = K, p, n_dofs, dim
        self._values = values  # torch fp64 on the device, CSR order
        # multi-device result: the owned CSR value ranges of consecutive row slabs, one
        # tensor per device (concatenated in row order they are the whole CSR)
        self.shards = shards
        self._matrix = matrix

    @property
    def values(self):
        """Device CSR values; for a multi-device result the shards are gathered onto the
        first shard's device on first access."""
        if self._values is None and self.shards is not None:
            import torch

            dev = self.shards[0].device
            self._values = torch.cat([s.to(dev) for s in self.shards])
        return self._values

    @values.setter
    def values(self, v):
        self._values = v

    def host_values(self) -> np.ndarray:
        if self._values is None and self.shards is not None:
            return np.concatenate([s.cpu().numpy() for s in self.shards])
        return self.values.cpu().numpy()

    @property
    def matrix(self):
        if self._matrix is None:
            import scipy.sparse

            indptr, indices = host_pattern(self.dim, self.K, self.p)
            data = self.host_values()
            self._matrix = scipy.sparse.csr_matrix((data, indices, indptr),
                                                   shape=(self.n_dofs, self.n_dofs))
            self._matrix.has_sorted_indices = True
        return self._matrix

    def spmv(self, x: np.ndarray) -> np.ndarray:
        return spmv(self, x)

    def __repr__(self):
        return f"GlobalGram(K={self.K}, p={self.p}, n_dofs={self.n_dofs}, dim={self.dim})"


def assemble(elements, K: int, p: int) -> GlobalGram:
    """Assemble one ElementMatrix per element of the K^3 mesh (assembly.py:46-83).

    Element matrices are uploaded once and summed on the device into the
    structured CSR in lexicographic element order."""
    by_id: dict[ElementId, ElementMatrix] = {}
    for alpha, mat in elements:
        if alpha in by_id:
            raise ValueError(f"duplicate element {alpha}")
        by_id[alpha] = mat
    expected = element_list(K)
    if len(by_id) != len(expected) or set(by_id) != set(expected):
        raise ValueError(f"element set does not cover the {K}^3 mesh")
    n = (p + 1) ** 3
    host = np.empty((len(expected), n, n))
    for e, alpha in enumerate(expected):
        ent = np.asarray(by_id[alpha].entries)
        if ent.shape != (n, n):
            raise ValueError(f"element matrix for {alpha} has wrong shape")
        host[e] = ent
    torch = _lib.require_cuda()  # after the reference's ValueError checks
    mats = torch.from_numpy(host).cuda()
    nd = _n_dofs(3, K, p)
    values = torch.empty(csr_nnz(3, K, p), dtype=torch.float64, device=mats.device)
    _lib.check(_lib.load().iga_assemble_elements(3, K, p, mats.data_ptr(), 0, K + p,
                                                 values.data_ptr(), _lib.stream_ptr()))
    return GlobalGram(K=K, p=p, n_dofs=nd, values=values)


def spmv(gram: GlobalGram, x: np.ndarray) -> np.ndarray:
    """G x on the device over the structured CSR (assembly.py:86-91)."""
    torch = _lib.require_cuda()
    x = np.asarray(x)
    if x.shape != (gram.n_dofs,):
        raise ValueError(f"vector length {x.shape} does not match {gram.n_dofs} dofs")
    if gram.values is None:
        return gram.matrix @ x
    xd = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).to(gram.values.device)
    yd = torch.empty_like(xd)
    _lib.check(_lib.load().iga_spmv(gram.dim, gram.K, gram.p, gram.values.data_ptr(),
                                    xd.data_ptr(), yd.data_ptr(), _lib.stream_ptr()))
    return yd.cpu().numpy()


def sparsity_row_bound(p: int) -> int:
    return (2 * p + 1) ** 3


def symbolic_pattern(K: int, p: int):
    """Boolean CSR pattern (assembly.py:99-115), generated on the device (K5)."""
    import scipy.sparse

    indptr, indices = host_pattern(3, K, p)
    nd = _n_dofs(3, K, p)
    pat = scipy.sparse.csr_matrix((np.ones(len(indices), dtype=bool), indices, indptr),
                                  shape=(nd, nd))
    pat.has_sorted_indices = True
    return pat


def write_matrix_market(gram: GlobalGram, path, threads: int | None = None) -> None:
    """Symmetric Matrix Market coordinate file (assembly.py:118-120), byte-identical to
    ``scipy.io.mmwrite(path, gram.matrix.tocoo(), symmetry="symmetric")``.

    Device-resident values stream to the host in row blocks through the native writer
    (csrc/iga_mmio.cu: double-buffered copies, multi-threaded formatting); a gram that
    only has a host CSR is written by the same formatter from host memory."""
    import os

    L = _lib.load()
    path = os.fspath(path)
    nthr = int(threads or os.cpu_count() or 1)
    if gram.values is not None:
        _lib.require_cuda()
        vals = gram.values.contiguous()
        _lib.check(L.iga_write_matrix_market(gram.dim, gram.K, gram.p, _lib.ptr(vals),
                                             path.encode(), nthr, _lib.stream_ptr()))
        return
    m = gram.matrix
    indptr, indices = host_pattern(gram.dim, gram.K, gram.p)
    if not (np.array_equal(m.indptr, indptr) and np.array_equal(m.indices, indices)):
        raise ValueError("matrix does not have the structured IGA pattern")
    data = np.ascontiguousarray(m.data, dtype=np.float64)
    _lib.check(L.iga_write_matrix_market_host(gram.dim, gram.K, gram.p, data.ctypes.data,
                                              path.encode(), nthr))
