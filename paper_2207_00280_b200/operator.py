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
       beta: float = 0.0):
    """Conjugate gradients on the device (HeatProblem._solve, heat.py:168-175: rtol 1e-10,
    maxiter 10 n).  ``A`` is an assembled GlobalGram (SpMV on the structured CSR) or a
    MatrixFreeOperator applied as ``alpha M + beta S`` (SPD for alpha > 0, beta >= 0)."""
    torch = _lib.require_cuda()
    L = _lib.load()
    n = A.n_dofs
    bd = torch.as_tensor(np.ascontiguousarray(b, dtype=np.float64)).cuda()
    x = torch.zeros_like(bd) if x0 is None else torch.as_tensor(
        np.ascontiguousarray(x0, dtype=np.float64)).cuda()
    Ap = torch.empty_like(bd)

    if isinstance(A, MatrixFreeOperator):
        def spmv(v, out):
            return A.apply(v, alpha, beta, out=out)
    else:
        def spmv(v, out):
            _lib.check(L.iga_spmv(A.dim, A.K, A.p, A.values.data_ptr(), v.data_ptr(),
                                  out.data_ptr(), _lib.stream_ptr()))
            return out

    r = bd - spmv(x, Ap)
    p = r.clone()
    rr = torch.dot(r, r)
    bnorm = torch.linalg.norm(bd)
    tol = rtol * bnorm
    maxiter = 10 * n if maxiter is None else maxiter
    for it in range(maxiter):
        if torch.sqrt(rr) <= tol:
            return x.cpu().numpy(), it
        spmv(p, Ap)
        step = rr / torch.dot(p, Ap)
        x += step * p
        r -= step * Ap
        rr_new = torch.dot(r, r)
        p = r + (rr_new / rr) * p
        rr = rr_new
    raise RuntimeError("conjugate gradient did not converge")


def heat_step(op: MatrixFreeOperator, mu, dt: float, rtol: float = 1e-10):
    """One forward-Euler step of the heat demo on the device (HeatProblem.step,
    heat.py:101-107): L = M mu - dt S mu (assemble_rhs), then G mu' = L by CG from
    x0 = mu with the Gram (mass) operator applied matrix-free."""
    if dt < 0:
        raise ValueError("timestep must be >= 0")
    L = op.rhs(mu, dt)
    x, _ = cg(op, L, x0=mu, rtol=rtol, alpha=1.0, beta=0.0)
    return x
