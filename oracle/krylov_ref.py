"""Vector operations (Eqs. (2)-(6)) and Krylov solvers -- TEST INFRASTRUCTURE
ONLY (see oracle/__init__.py).  The consumers of the SpMV in the paper
(SURVEY.md §8(f) NEXT-1 / NEXT-3):

  spmv_axpby  Eq. (2), P:164-167   y = alpha A x + beta y
  axpby       Eq. (3), P:169-172   y = alpha x + beta y
  axpbyz      Eq. (4), P:174-177   z = alpha x + beta y
  dot         Eq. (5), P:179-182   a = <x, y>           (plain left-to-right sum)
  norm2       Eq. (6), P:184-187   r = sqrt(<x, x>)
  bicgstab    Alg. 4, with M = I (no preconditioner), written line
              by line in the paper's order and notation
  cg          "CG ... implemented" (the algorithm of \\cite{saad}, Alg. 6.18)

Every product A v is O1 (oracle.csr_spmv).  Plain Python loops over the
iterations; numpy only for the vector arithmetic of one line at a time.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import csr_spmv


def spmv_axpby(A, alpha: float, x: np.ndarray, beta: float, y: np.ndarray) -> np.ndarray:
    return alpha * csr_spmv(A, x) + beta * y


def axpby(alpha: float, x: np.ndarray, beta: float, y: np.ndarray) -> np.ndarray:
    return alpha * x + beta * y


def axpbyz(alpha: float, x: np.ndarray, beta: float, y: np.ndarray) -> np.ndarray:
    return alpha * x + beta * y


def dot(x: np.ndarray, y: np.ndarray) -> float:
    s = 0.0
    for a, b in zip(x.tolist(), y.tolist()):
        s = s + a * b
    return s


def norm2(x: np.ndarray) -> float:
    return math.sqrt(dot(x, x))


@dataclass
class SolveRef:
    x: np.ndarray
    iterations: int
    converged: bool
    breakdown: int
    rel_residual: float
    history: list


def bicgstab(A, b: np.ndarray, x0: np.ndarray, tol: float, max_it: int) -> SolveRef:
    """Alg. 4 with M = I, so p* = p and s* = s.  Stopping tests:
    ||s||_2 <= tol ||r_0||_2 and ||r||_2 <= tol ||r_0||_2 (reading of 'is
    satisfied'); breakdown 1 when rho_{k-1} = 0 ('Fails'), 2 when omega_k = 0,
    3 when (r0, v) = 0 (alpha undefined; not tested by Alg. 4, reading A20),
    4 when (t, t) = 0 or omega_k is not finite (omega undefined; reading A20)."""
    x = x0.astype(np.float64).copy()
    r = b - csr_spmv(A, x)                      # r0 = b - A x0           (SpMV; vector update)
    r0 = r.copy()                               # shadow residual r~ = r0
    r0n = norm2(r)
    hist = [1.0 if r0n > 0 else 0.0]
    if r0n == 0.0:
        return SolveRef(x, 0, True, 0, 0.0, hist)
    rho_prev = alpha = omega = 0.0
    p = v = None
    for k in range(1, max_it + 1):
        rho = dot(r0, r)                        # rho_{k-1} = (r0, r)
        if rho == 0.0:
            return SolveRef(x, k, False, 1, hist[-1], hist)      # Fails
        if k == 1:
            p = r.copy()                        # p = r
        else:
            beta = (rho / rho_prev) * (alpha / omega)
            p = r + beta * (p - omega * v)      # p = r + beta (p - omega v)
        v = csr_spmv(A, p)                      # v = A p*               (SpMV)
        r0v = dot(r0, v)
        if r0v == 0.0:                          # not tested in Alg. 4 (reading A20): breakdown 3
            return SolveRef(x, k, False, 3, hist[-1], hist)
        alpha = rho / r0v                       # alpha_k = rho_{k-1} / (r0, v)
        s = r - alpha * v                       # s = r - alpha v
        sn = norm2(s)
        if sn <= tol * r0n:                     # ||s|| is satisfied
            x = x + alpha * p
            hist.append(sn / r0n)
            return SolveRef(x, k, True, 0, sn / r0n, hist)
        t = csr_spmv(A, s)                      # t = A s*               (SpMV)
        ts, tt = dot(t, s), dot(t, t)
        if tt == 0.0 or not math.isfinite(ts / tt):  # omega_k undefined (reading A20): breakdown 4
            return SolveRef(x, k, False, 4, hist[-1], hist)
        omega = ts / tt                         # omega_k = (t, s) / ||t||^2
        x = x + alpha * p + omega * s           # x = x + alpha p* + omega s*
        r = s - omega * t                       # r = s - omega t
        rn = norm2(r)
        hist.append(rn / r0n)
        if rn <= tol * r0n:                     # ||r|| is satisfied
            return SolveRef(x, k, True, 0, rn / r0n, hist)
        if omega == 0.0:
            return SolveRef(x, k, False, 2, rn / r0n, hist)
        rho_prev = rho
    return SolveRef(x, max_it, False, 0, hist[-1], hist)


def cg(A, b: np.ndarray, x0: np.ndarray, tol: float, max_it: int) -> SolveRef:
    """Conjugate gradients for SPD A (Saad, Alg. 6.18): stop when
    ||r_k||_2 <= tol ||r_0||_2; breakdown 4 when (p, A p) = 0 or alpha is not
    finite (A not SPD)."""
    x = x0.astype(np.float64).copy()
    r = b - csr_spmv(A, x)
    p = r.copy()
    rho = dot(r, r)
    r0n = math.sqrt(rho)
    hist = [1.0 if r0n > 0 else 0.0]
    if r0n == 0.0:
        return SolveRef(x, 0, True, 0, 0.0, hist)
    for k in range(1, max_it + 1):
        q = csr_spmv(A, p)
        pq = dot(p, q)
        if pq == 0.0 or not math.isfinite(rho / pq):   # alpha undefined (A not SPD): breakdown 4
            return SolveRef(x, k, False, 4, hist[-1], hist)
        alpha = rho / pq
        x = x + alpha * p
        r = r - alpha * q
        rho_new = dot(r, r)
        hist.append(math.sqrt(rho_new) / r0n)
        if math.sqrt(rho_new) <= tol * r0n:
            return SolveRef(x, k, True, 0, hist[-1], hist)
        p = r + (rho_new / rho) * p
        rho = rho_new
    return SolveRef(x, max_it, False, 0, hist[-1], hist)
