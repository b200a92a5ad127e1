"""Tier D: dense assembly of every matrix of the scheme (oracle; test infrastructure only).

Grid functions are numpy arrays U of shape (n_1, ..., n_d) with U[j1-1,...,jd-1]
the value at x_J.  The paper's vector x_G orders the grid with axis 1 fastest
(Kronecker order H_{alpha_d} (x) ... (x) H_{alpha_1}), i.e.
``vec(U) = U.flatten(order="F")``.  Matrices here act on such vectors and are
assembled literally from the paper's formulas with ``np.kron``; only for
N^d <= ~4096.
"""
from __future__ import annotations

from functools import reduce
from typing import Sequence

import numpy as np

from . import fcd


def vec(U: np.ndarray) -> np.ndarray:
    """paper-order vector of a grid array (axis 1 fastest)."""
    return np.asarray(U).flatten(order="F")


def unvec(v: np.ndarray, n: Sequence[int]) -> np.ndarray:
    return np.asarray(v).reshape(tuple(n), order="F")


def kron_paper(mats: Sequence[np.ndarray]) -> np.ndarray:
    """mats[i] acts on axis i+1; returns mats[d-1] (x) ... (x) mats[0]."""
    return reduce(np.kron, list(mats)[::-1])


class DenseSystem:
    """All dense matrices of Eq.(tls), Eq.(equi), Eq.(Pa) for one problem."""

    def __init__(self, d, n, alpha, kappa, tau):
        self.d, self.n = d, tuple(n)
        self.alpha, self.kappa, self.tau = tuple(alpha), tuple(kappa), tau
        self.h = [1.0 / (ni + 1) for ni in self.n]
        self.eta = [fcd.eta(self.kappa[i], tau, self.h[i], self.alpha[i]) for i in range(d)]
        self.s = [fcd.fcd_coefficients(self.alpha[i], self.n[i]).astype(np.float64) for i in range(d)]
        self.H1 = [fcd.h_matrix(self.alpha[i], self.n[i]) for i in range(d)]
        self.S1 = [fcd.toeplitz_matrix(self.s[i]) for i in range(d)]
        self.tauS1 = [fcd.tau_matrix(self.s[i]) for i in range(d)]
        self.I1 = [np.eye(ni) for ni in self.n]
        self.Ntot = int(np.prod(self.n))

    # H_alpha = H_{alpha_d} (x) ... (x) H_{alpha_1}
    def H_alpha(self):
        return kron_paper(self.H1)

    def _sum_with(self, one_d):
        """sum_i eta_i (H (x) .. (x) one_d[i] (x) .. (x) H) as in Eq.(Salpha)/(tauSalpha)."""
        out = np.zeros((self.Ntot, self.Ntot))
        for i in range(self.d):
            mats = [self.H1[l] if l != i else one_d[i] for l in range(self.d)]
            out += self.eta[i] * kron_paper(mats)
        return out

    # S_alpha, Eq.(Salpha) P:104 (reading Q4 for the missing (x))
    def S_alpha(self):
        return self._sum_with(self.S1)

    # tau(S_alpha), Eq.(tauSalpha)
    def tau_S_alpha(self):
        return self._sum_with(self.tauS1)

    @staticmethod
    def E(e_grid: np.ndarray):
        """E^{(m+1/2)} = diag(e(x_G, t_{m+1/2}))."""
        return np.diag(vec(e_grid))

    # A = H_alpha E + S_alpha (Eq.(tls))
    def A(self, e_grid):
        return self.H_alpha() @ self.E(e_grid) + self.S_alpha()

    # b = (H_alpha E - S_alpha) u + tau F (Eq.(tls))
    def b(self, e_grid, u_vec, F_vec):
        return (self.H_alpha() @ self.E(e_grid) - self.S_alpha()) @ u_vec + self.tau * F_vec

    # A~ = E + H_alpha^{-1} S_alpha  (Eq.(equi))
    def A_tilde(self, e_grid):
        return self.E(e_grid) + np.linalg.solve(self.H_alpha(), self.S_alpha())

    # H_alpha^{-1/2} via the symmetric eigendecomposition (H_alpha is SPD, Lemma 3.5)
    def H_alpha_pow(self, p):
        w, Q = np.linalg.eigh(self.H_alpha())
        return (Q * w ** p) @ Q.T

    # P_alpha = ebar I + H^{-1/2} tau(S_alpha) H^{-1/2}  (Eq.(Pa))
    def P_alpha(self, ebar):
        Hm = self.H_alpha_pow(-0.5)
        return ebar * np.eye(self.Ntot) + Hm @ self.tau_S_alpha() @ Hm

    # P_hat = H_alpha P_alpha = ebar H_alpha + tau(S_alpha) (SURVEY 8 key identity)
    def P_hat(self, ebar):
        return ebar * self.H_alpha() + self.tau_S_alpha()

    def dst(self):
        """d-level orthonormal DST-I, S = S_d (x) ... (x) S_1."""
        return kron_paper([fcd.dst_matrix(ni) for ni in self.n])
