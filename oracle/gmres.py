"""Textbook restarted GMRES (oracle; test infrastructure only).

GMRES of Saad & Schultz [Saad86], cited at P:234-235: Arnoldi with modified
Gram-Schmidt, Givens rotations on the Hessenberg matrix, y = R^{-1} g at the end
of a cycle.  The caller forms the (left-preconditioned) operator K and right-hand
side c (the paper's one-sided system Eq.(one-sided)).

Stopping rule: stop at the first Arnoldi step j with
|g_{j+1}| <= tol * ||r_0||, r_0 = c - K x_0 of the *first* cycle of this solve.
At the restart length without convergence: x <- x_0 + V y, explicit residual,
next cycle.  max_iters caps the total Arnoldi steps (Q12).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable, List, Optional

import numpy as np


@dataclass
class GmresResult:
    x: np.ndarray
    iters: int
    converged: bool
    relres_est: float              # |g_{k+1}| / beta0 (Givens estimate)
    history: List[float] = field(default_factory=list)
    beta0: float = 0.0             # ||r_0|| of the first cycle (history * beta0 = ||r_j||)


def _dot(a, b):
    return float(np.dot(a.ravel(), b.ravel()))


def gmres(apply_K: Callable[[np.ndarray], np.ndarray], c: np.ndarray, x0: np.ndarray,
          restart: int, tol: float, max_iters: int,
          fixed_iters: Optional[int] = None) -> GmresResult:
    """Solve K x = c.  ``fixed_iters`` (replay mode) runs exactly that
    many Arnoldi steps (unless a lucky breakdown occurs) instead of testing tol."""
    x = np.array(x0, dtype=np.float64, copy=True)
    r = c - apply_K(x)
    beta0 = math.sqrt(_dot(r, r))
    hist = [1.0]
    if beta0 == 0.0 or (fixed_iters is not None and fixed_iters <= 0):
        return GmresResult(x, 0, True, 0.0, hist, beta0)
    total = 0
    while True:
        beta = math.sqrt(_dot(r, r))
        V = [r / beta]
        m = restart
        Hm = np.zeros((m + 1, m))
        cs = np.zeros(m)
        sn = np.zeros(m)
        g = np.zeros(m + 1)
        g[0] = beta
        k = 0
        stop = False
        breakdown = False
        for j in range(m):
            w = apply_K(V[j])
            for i in range(j + 1):                      # modified Gram-Schmidt
                Hm[i, j] = _dot(w, V[i])
                w = w - Hm[i, j] * V[i]
            hnext = math.sqrt(_dot(w, w))
            Hm[j + 1, j] = hnext
            for i in range(j):                          # previous rotations
                t = cs[i] * Hm[i, j] + sn[i] * Hm[i + 1, j]
                Hm[i + 1, j] = -sn[i] * Hm[i, j] + cs[i] * Hm[i + 1, j]
                Hm[i, j] = t
            den = math.hypot(Hm[j, j], Hm[j + 1, j])     # new rotation
            cs[j] = Hm[j, j] / den
            sn[j] = Hm[j + 1, j] / den
            Hm[j, j] = den
            Hm[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            total += 1
            k = j + 1
            hist.append(abs(g[j + 1]) / beta0)
            if fixed_iters is None:
                stop = abs(g[j + 1]) <= tol * beta0
            else:
                stop = total >= fixed_iters
            if hnext == 0.0:
                breakdown = True                        # lucky breakdown: exact solution
            if stop or breakdown or total >= max_iters:
                break
            V.append(w / hnext)
        # y = R^{-1} g (back substitution on the rotated upper-triangular R)
        y = np.zeros(k)
        for i in range(k - 1, -1, -1):
            y[i] = (g[i] - np.dot(Hm[i, i + 1:k], y[i + 1:k])) / Hm[i, i]
        for i in range(k):
            x = x + y[i] * V[i]
        # replay mode keeps restarting until exactly fixed_iters Arnoldi steps ran
        converged = stop if fixed_iters is None else total >= fixed_iters
        if breakdown:
            converged = True
        if converged or total >= max_iters:
            return GmresResult(x, total, converged, abs(g[k]) / beta0, hist, beta0)
        r = c - apply_K(x)                              # explicit residual, restart
