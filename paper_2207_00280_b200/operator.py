"""Matrix-free operators and the heat-step building blocks.

``MatrixFreeOperator(K, p).apply(x, alpha, beta)`` computes ``alpha M x + beta S x``
on the device without assembling (kernel ``iga_apply``); ``rhs(mu, dt)`` is the
device version of ``heat.HeatProblem.assemble_rhs`` (heat.py:131-158), i.e.
``M mu - dt S mu``.  ``cg`` solves ``G u = b`` with the assembled device CSR and
``iga_spmv`` (the solve of ``heat.HeatProblem._solve``, heat.py:168-175).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .device import MeshProblem


class MatrixFreeOperator:
    def __init__(self, K: int, p: int, q: int | None = None, coefficient=None, knots=None):
        if p < 1:
            raise ValueError("the gradient term requires degree >= 1")
        self.prob = MeshProblem(3, K, p, q, operator="stiffness", coefficient=coefficient,
                                knots=knots)
        self.n_dofs = self.prob.n_dofs

    def apply(self, x, alpha: float = 1.0, beta: float = 0.0, out=None, stream=None):
        torch = _lib.require_cuda()
        host = not isinstance(x, torch.Tensor)
        xd = torch.as_tensor(np.ascontiguousarray(x, dtype=np.float64)).cuda() if host else x
        if xd.numel() != self.n_dofs:
            raise ValueError(f"vector length {xd.numel()} does not match {self.n_dofs} dofs")
        yd = torch.empty_like(xd) if out is None else out
        s = self.prob.problem_struct()
        _lib.check(_lib.load().iga_apply(ctypes.byref(s), float(alpha), float(beta),
                                         xd.data_ptr(), yd.data_ptr(),
                                         _lib.stream_ptr(stream)))
        return yd.cpu().numpy() if host else yd

    def rhs(self, mu, dt: float):
        """``int U B - dt int grad U . grad B`` (heat.py:131-158)."""
        if dt < 0:
            raise ValueError("timestep must be >= 0")
        return self.apply(mu, 1.0, -float(dt))


def cg(A, b, x0=None, rtol: float = 1e-10, maxiter: int | None = None, alpha: float = 1.0,
       beta: float = 0.0, check_every: int = 16, stream=None):
    """Conjugate gradients on the device (HeatProblem._solve, heat.py:168-175: rtol 1e-10,
    maxiter 10 n), stopping at ``||b - A x|| <= rtol ||b||``.  ``A`` is an assembled
    GlobalGram (SpMV on the structured CSR) or a MatrixFreeOperator applied as
    ``alpha M + beta S`` (SPD for alpha > 0, beta >= 0).  The whole iteration runs in the
    library (``iga_cg``): stream-ordered launches with deterministic reductions, the host
    reading the solver state every ``check_every`` iterations.  Returns (x, iterations);
    device inputs give a device x, host inputs a numpy x."""
    torch = _lib.require_cuda()
    L = _lib.load()
    n = A.n_dofs
    host = not isinstance(b, torch.Tensor)

    def dev(v):
        if isinstance(v, torch.Tensor):
            return v.to(device="cuda", dtype=torch.float64).contiguous()
        return torch.as_tensor(np.ascontiguousarray(v, dtype=np.float64)).cuda()

    bd = dev(b)
    if bd.numel() != n:
        raise ValueError(f"right-hand side length {bd.numel()} does not match {n} dofs")
    x = torch.zeros_like(bd) if x0 is None else dev(x0).clone()
    if x.numel() != n:
        raise ValueError(f"x0 length {x.numel()} does not match {n} dofs")
    work = torch.empty(int(L.iga_cg_work_size(n)), dtype=torch.float64, device=bd.device)
    maxiter = 10 * n if maxiter is None else int(maxiter)
    iters = ctypes.c_int64(0)
    if isinstance(A, MatrixFreeOperator):
        s = A.prob.problem_struct()
        rc = L.iga_cg(3, 0, 0, None, ctypes.byref(s), float(alpha), float(beta), n, bd.data_ptr(),
                      x.data_ptr(), work.data_ptr(), float(rtol), maxiter, int(check_every),
                      ctypes.byref(iters), _lib.stream_ptr(stream))
    else:
        rc = L.iga_cg(A.dim, A.K, A.p, A.values.data_ptr(), None, 1.0, 0.0, n, bd.data_ptr(),
                      x.data_ptr(), work.data_ptr(), float(rtol), maxiter, int(check_every),
                      ctypes.byref(iters), _lib.stream_ptr(stream))
    _lib.check(rc)
    return (x.cpu().numpy() if host else x), int(iters.value)


def heat_step(op: MatrixFreeOperator, mu, dt: float, rtol: float = 1e-10):
    """One forward-Euler step of the heat demo on the device (HeatProblem.step,
    heat.py:101-107): L = M mu - dt S mu (assemble_rhs), then G mu' = L by CG from
    x0 = mu with the Gram (mass) operator applied matrix-free."""
    if dt < 0:
        raise ValueError("timestep must be >= 0")
    L = op.rhs(mu, dt)
    x, _ = cg(op, L, x0=mu, rtol=rtol, alpha=1.0, beta=0.0)
    return x
