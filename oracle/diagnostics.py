"""Spectral and convergence diagnostics of the preconditioned systems (oracle; test infrastructure only).

SURVEY 8(f) NEXT-3, dense (Tier D) and therefore for small grids (N^d <= a few thousand):

* numerical range W(A) = {x* A x / x* x}: numerical radius r(A) = max |W(A)| and the
  distance v(A) = min |W(A)| of W(A) to the origin (Eq.(numrag)), by support functions:
  r(A) = max_theta lambda_max(Herm(e^{i theta} A)),  v(A) = max(0, max_theta lambda_min(Herm(e^{i theta} A)))
  (W(A) is compact and convex: Toeplitz-Hausdorff).
* Theorem 3.7 (proof P:342-414): for A_breve = P_alpha^{-1/2} A~ P_alpha^{-1/2},
  v(A_breve) >= min{2 e_check/(e_hat+e_check), (4-sqrt 6)/4},  r(A_breve) <= max{2 e_hat/(e_hat+e_check),
  (4+sqrt 6)/4}  (Eq.(Theq4)), and GMRES on the two-sided system satisfies
  ||r_k|| / ||r_0|| <= (2+c) c^k with c of P:333-337 (= sin(theta) at the two bounds, Lemma 3.6).
* eigenvalues of A~ and P_alpha^{-1} A~ (Figs 1-3): P^{-1} A~ is similar to A_breve, so its
  spectrum lies in W(A_breve).
"""
from __future__ import annotations

import math
from typing import Tuple

import numpy as np

from . import dense as D


def numerical_range_extremes(A: np.ndarray, n_theta: int = 1440) -> Tuple[float, float]:
    """(v(A), r(A)) of Eq.(numrag) from the support function of W(A) on n_theta angles, refined by a
    golden-section search around the best angle of each extreme."""
    A = np.asarray(A, dtype=np.complex128)

    def herm_eigs(th):
        B = np.exp(1j * th) * A
        w = np.linalg.eigvalsh(0.5 * (B + B.conj().T))
        return w[0], w[-1]

    ths = np.linspace(0.0, 2.0 * math.pi, n_theta, endpoint=False)
    lo = np.empty(n_theta)
    hi = np.empty(n_theta)
    for k, th in enumerate(ths):
        lo[k], hi[k] = herm_eigs(th)

    def refine(f, th0):
        a, b = th0 - 2 * math.pi / n_theta, th0 + 2 * math.pi / n_theta
        g = (math.sqrt(5) - 1) / 2
        for _ in range(40):
            c, d = b - g * (b - a), a + g * (b - a)
            if f(c) > f(d):
                b = d
            else:
                a = c
        return f(0.5 * (a + b))

    r = refine(lambda t: herm_eigs(t)[1], ths[int(np.argmax(hi))])
    v = refine(lambda t: herm_eigs(t)[0], ths[int(np.argmax(lo))])
    return max(0.0, v), r


def theorem37_bounds(ehat: float, echeck: float) -> Tuple[float, float, float]:
    """(lower bound of v, upper bound of r, c) of Theorem 3.7 (Eq.(Theq4) and P:333-337)."""
    s6 = math.sqrt(6.0)
    lo = min(2 * echeck / (ehat + echeck), (4 - s6) / 4)
    hi = max(2 * ehat / (ehat + echeck), (4 + s6) / 4)
    c = max(math.sqrt(1 - echeck ** 2 / ehat ** 2),
            math.sqrt(16 * s6 / (4 + s6) ** 2),
            math.sqrt(1 - (ehat + echeck) ** 2 * (11 - 4 * s6) / (32 * ehat ** 2)),
            math.sqrt(1 - 32 * echeck ** 2 / ((11 + 4 * s6) * (ehat + echeck) ** 2)))
    return lo, hi, c


def two_sided_matrix(Ds: D.DenseSystem, e_grid: np.ndarray, ebar: float) -> np.ndarray:
    """A_breve = P_alpha^{-1/2} A~ P_alpha^{-1/2} (Theorem 3.7's matrix)."""
    w, Q = np.linalg.eigh(Ds.P_alpha(ebar))
    Pmh = (Q / np.sqrt(w)) @ Q.T
    return Pmh @ Ds.A_tilde(e_grid) @ Pmh


def spectra(Ds: D.DenseSystem, e_grid: np.ndarray, ebar: float):
    """eigenvalues of A~ and of P_alpha^{-1} A~ (Figs 1-3)."""
    At = Ds.A_tilde(e_grid)
    return np.linalg.eigvals(At), np.linalg.eigvals(np.linalg.solve(Ds.P_alpha(ebar), At))
