"""Dense LP solver on the GPU: the drop-in for the reference's ``harmonyep.simplex``
(``/root/reference/pkg/src/harmonyep/simplex.py``).

Same surface -- ``LinearProgram`` (:24-38), ``SimplexResult`` (:41-47), ``SimplexError``
(:20-21, a ``ContractViolation``) and ``simplex_solve(lp, basis=None, tol=1e-9,
max_iter=50000)`` (:99-192) -- but every pivot runs in one launch of the cluster kernel
``hep_lp_solve`` (``csrc/lp.cu``; include/hep.h).  The kernel follows the reference's
two-phase Bland's-rule tableau method operation for operation, so a cold solve returns
the reference's basis, pivot count and solution bit for bit; a warm start factorises the
previous basis by device Gauss-Jordan instead of LAPACK, which agrees to rounding.

Only the LP matrices (built on the host by ``scheduler._comm_aware_lp`` /
``_topology_aware_lp``, as in the reference) cross PCIe; the host reads back x, the basis
and the counters.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .core import ContractViolation

_STATUS = {1: "LP is infeasible", 2: "LP is unbounded", 3: "simplex exceeded {max_iter} pivots"}


class SimplexError(ContractViolation):
    """Infeasible / unbounded LP or pivot limit (reference simplex.py:20-21)."""


@dataclass
class LinearProgram:
    """min c.x  s.t.  a_eq x = b_eq,  a_ub x <= b_ub,  x >= 0 (fp64, dense)."""

    c: np.ndarray
    a_eq: np.ndarray
    b_eq: np.ndarray
    a_ub: np.ndarray
    b_ub: np.ndarray

    def __post_init__(self):
        f64 = np.float64
        self.c = np.asarray(self.c, dtype=f64)
        self.b_eq = np.asarray(self.b_eq, dtype=f64).reshape(-1)
        self.b_ub = np.asarray(self.b_ub, dtype=f64).reshape(-1)
        self.a_eq = np.asarray(self.a_eq, dtype=f64).reshape(self.b_eq.size, self.c.size) if self.b_eq.size \
            else np.zeros((0, self.c.size))
        self.a_ub = np.asarray(self.a_ub, dtype=f64).reshape(self.b_ub.size, self.c.size) if self.b_ub.size \
            else np.zeros((0, self.c.size))


@dataclass
class SimplexResult:
    x: np.ndarray
    objective: float
    basis: np.ndarray
    iterations: int
    status: str
    warm_started: bool = False
    device_us: float = 0.0


class _Workspace:
    """Device buffers of one LP shape, reused across solves of that shape."""

    def __init__(self, n: int, m_eq: int, m_ub: int, device):
        torch = _lib.require_cuda()
        self.key = (n, m_eq, m_ub)
        m = m_eq + m_ub
        self.bytes = int(_lib.lib().hep_lp_workspace(n, m_eq, m_ub))
        f64 = dict(dtype=torch.float64, device=device)
        self.work = torch.empty(max(self.bytes // 8, 1), **f64)
        self.x_full = torch.zeros(max(n + m_ub, 1), **f64)
        self.basis_out = torch.zeros(max(m, 1), dtype=torch.int64, device=device)
        self.basis_in = torch.zeros(max(m, 1), dtype=torch.int64, device=device)
        self.info = torch.zeros(8, dtype=torch.int64, device=device)


_WS: dict = {}


def _workspace(n: int, m_eq: int, m_ub: int):
    torch = _lib.require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device())
    key = (n, m_eq, m_ub, dev.index)
    ws = _WS.get(key)
    if ws is None:
        if len(_WS) > 16:
            _WS.clear()
        ws = _WS[key] = _Workspace(n, m_eq, m_ub, dev)
    return ws, dev


def simplex_solve(lp: LinearProgram, basis: np.ndarray | None = None, tol: float = 1e-9,
                  max_iter: int = 50000) -> SimplexResult:
    """Solve ``lp`` on the device (reference simplex.py:99-192).  ``basis``: a previous
    optimal basis to warm-start from; ignored unless it has one entry per constraint row
    and indexes only structural/slack columns (the reference's condition, :128)."""
    torch = _lib.require_cuda()
    n, m_eq, m_ub = lp.c.size, lp.b_eq.size, lp.b_ub.size
    m = m_eq + m_ub
    width = n + m_ub
    ws, dev = _workspace(n, m_eq, m_ub)
    d = {k: torch.from_numpy(np.ascontiguousarray(getattr(lp, k))).to(dev) for k in ("c", "a_eq", "b_eq", "a_ub", "b_ub")}
    d_basis = None
    if basis is not None:
        b = np.asarray(basis, dtype=np.int64).reshape(-1)
        if b.size == m and m > 0 and np.all(b < width) and np.all(b >= 0):
            ws.basis_in[:m].copy_(torch.from_numpy(b))
            d_basis = ws.basis_in
    stream = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    _lib.check(
        _lib.lib().hep_lp_solve(
            _lib.ptr(d["c"]), _lib.ptr(d["a_eq"]) if m_eq else None, _lib.ptr(d["b_eq"]) if m_eq else None,
            _lib.ptr(d["a_ub"]) if m_ub else None, _lib.ptr(d["b_ub"]) if m_ub else None,
            n, m_eq, m_ub, _lib.ptr(d_basis), float(tol), int(max_iter),
            _lib.ptr(ws.work), ctypes.c_size_t(ws.bytes), _lib.ptr(ws.x_full), _lib.ptr(ws.basis_out),
            _lib.ptr(ws.info), _lib.stream_handle(stream),
        ),
        "hep_lp_solve",
    )
    e1.record(stream)
    info = ws.info.cpu().tolist()
    status = int(info[1])
    if status:
        raise SimplexError(_STATUS.get(status, f"simplex status {status}").format(max_iter=max_iter))
    x = np.maximum(ws.x_full[:n].cpu().numpy(), 0.0)
    return SimplexResult(
        x=x,
        objective=float(lp.c @ x),
        basis=ws.basis_out[:m].cpu().numpy().copy(),
        iterations=int(info[0]),
        status="optimal",
        warm_started=bool(info[2]),
        device_us=1e3 * e0.elapsed_time(e1),
    )
