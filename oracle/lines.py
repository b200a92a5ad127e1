"""Tier L: per-line operators on grid arrays (oracle; test infrastructure only).

A grid function is an array U of shape (n_1, ..., n_d); array axis i-1 is the
paper's x_i.  Every 1-D operator is applied along one axis to every line:
Toeplitz and DST-I as dense n x n matrix products (numpy matmul is the only
library primitive used), H_alpha as the 3-point stencil with zero Dirichlet
values, H_alpha^{-1} as the dense inverse of that tridiagonal matrix.
No fast transform, no fusion.
"""
from __future__ import annotations

import numpy as np

from . import fcd


def along(M: np.ndarray, U: np.ndarray, axis: int) -> np.ndarray:
    """apply the n x n matrix M to every line of U along ``axis``."""
    return np.moveaxis(np.tensordot(M, U, axes=([1], [axis])), 0, axis)


def h_along(U: np.ndarray, alpha: float, axis: int) -> np.ndarray:
    """(H_alpha v)_j = (1 - alpha/12) v_j + alpha/24 (v_{j-1} + v_{j+1}), v_0 = v_{N+1} = 0."""
    V = np.moveaxis(U, axis, 0)
    out = (1.0 - alpha / 12.0) * V
    nb = np.zeros_like(V)
    nb[1:] += V[:-1]
    nb[:-1] += V[1:]
    out = out + (alpha / 24.0) * nb
    return np.moveaxis(out, 0, axis)


class LineSystem:
    """Per-line realisation of Eq.(tls)/(equi)/(Pa) for grids of any size."""

    def __init__(self, d, n, alpha, kappa, tau):
        self.d, self.n = d, tuple(n)
        self.alpha, self.kappa, self.tau = tuple(alpha), tuple(kappa), tau
        self.h = [1.0 / (ni + 1) for ni in self.n]
        self.eta = [fcd.eta(self.kappa[i], tau, self.h[i], self.alpha[i]) for i in range(d)]
        self.s = [fcd.fcd_coefficients(self.alpha[i], self.n[i]).astype(np.float64) for i in range(d)]
        self.T = [fcd.toeplitz_matrix(self.s[i]) for i in range(d)]
        self.Hinv = [np.linalg.inv(fcd.h_matrix(self.alpha[i], self.n[i])) for i in range(d)]
        self.S = [fcd.dst_matrix(ni) for ni in self.n]
        self.q = [fcd.tau_eigenvalues(fcd.fcd_coefficients(self.alpha[i], self.n[i])) for i in range(d)]
        self.lamH = [fcd.h_eigenvalues(self.alpha[i], self.n[i]) for i in range(d)]

    # ---- building blocks -------------------------------------------------
    def H_alpha(self, U):
        """H_alpha U = prod_l H_{alpha_l} along axis l."""
        for l in range(self.d):
            U = h_along(U, self.alpha[l], l)
        return U

    def H_alpha_inv(self, U):
        for l in range(self.d):
            U = along(self.Hinv[l], U, l)
        return U

    def S_alpha(self, U):
        """S_alpha U = sum_i eta_i (prod_{l != i} H_l) S_{alpha_i} U (Eq.(Salpha))."""
        out = np.zeros_like(U)
        for i in range(self.d):
            V = along(self.T[i], U, i)
            for l in range(self.d):
                if l != i:
                    V = h_along(V, self.alpha[l], l)
            out = out + self.eta[i] * V
        return out

    def A(self, e_grid, U):
        """A U = H_alpha (E U) + S_alpha U (Eq.(tls))."""
        return self.H_alpha(e_grid * U) + self.S_alpha(U)

    def A_tilde(self, e_grid, U):
        """A~ U = E U + H_alpha^{-1} S_alpha U (Eq.(equi))."""
        return e_grid * U + self.H_alpha_inv(self.S_alpha(U))

    def rhs(self, e_grid, U, F):
        """b = (H_alpha E - S_alpha) U + tau F (Eq.(tls))."""
        return self.H_alpha(e_grid * U) - self.S_alpha(U) + self.tau * F

    def dst(self, U):
        """d-level orthonormal DST-I: S along every axis."""
        for l in range(self.d):
            U = along(self.S[l], U, l)
        return U

    # ---- preconditioner spectra (Lemma 3.3) ---------
    def _outer(self, vals):
        out = vals[0]
        for v in vals[1:]:
            out = np.multiply.outer(out, v)
        return out

    def lambda_P(self, ebar):
        """Lambda_P(k) = ebar + sum_i eta_i q_i(k_i) / lambda^H_i(k_i): eigenvalues of P_alpha
        (Eq.(Pa), H^{-1/2} tau(S) H^{-1/2} = H^{-1} tau(S))."""
        out = np.full(self.n, float(ebar))
        for i in range(self.d):
            shape = [1] * self.d
            shape[i] = self.n[i]
            out = out + (self.eta[i] * self.q[i] / self.lamH[i]).reshape(shape)
        return out

    def lambda_H(self):
        """eigenvalues of H_alpha: prod_l lambda^H_l(k_l) (Lemma 3.3 + Lemma 3.5)."""
        return self._outer(self.lamH) if self.d > 1 else self.lamH[0].copy()

    def P_alpha_inv(self, ebar, U):
        """P_alpha^{-1} U = S Lambda_P^{-1} S U (Eq.(diag); Eq.(Pa))."""
        return self.dst(self.dst(U) / self.lambda_P(ebar))

    def P_alpha_inv_sqrt(self, ebar, U):
        return self.dst(self.dst(U) / np.sqrt(self.lambda_P(ebar)))

    def P_alpha_sqrt(self, ebar, U):
        """P_alpha^{1/2} U = S Lambda_P^{1/2} S U (maps u to the two-sided unknown u~)."""
        return self.dst(self.dst(U) * np.sqrt(self.lambda_P(ebar)))

    def P_hat_inv(self, ebar, U):
        """(H_alpha P_alpha)^{-1} U = S (Lambda_P Lambda_H)^{-1} S U (SURVEY 8 key identity)."""
        return self.dst(self.dst(U) / (self.lambda_P(ebar) * self.lambda_H()))
