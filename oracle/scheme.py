"""Right-hand side, e-bar and the CN time loop (oracle; test infrastructure only).

* F^{(m+1/2)}: Appendix P:660-697 literally for d = 1, 2; for any d the
  closed-grid compact stencil (prod_l H_l applied to f on the closed grid,
  restricted to the interior), which equals the Appendix for d = 1, 2 (pinned by
  tests) and is the reading for the garbled d = 3 Appendix.
* e-bar = (e-hat + e-check)/2 over the interior grid and all half levels
  (Eq.(bard), Eq.(dhat)).
* time loop: u^{(0)} = psi; per step the one-sided system
  P_alpha^{-1} A~ u^{(m+1)} = P_alpha^{-1} b~ (Eq.(one-sided)) with
  A~ = E + H^{-1} S_alpha, b~ = H^{-1} b (Eq.(equi)), b from Eq.(tls)
  (P:95-97); GMRES from x_0 = u^{(m)}.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import dense as D
from . import fcd
from .gmres import gmres
from .lines import LineSystem, h_along


# ---------------------------------------------------------------------------
# F^{(m+1/2)}
# ---------------------------------------------------------------------------
def compact_source(alpha, f_closed: np.ndarray) -> np.ndarray:
    """(prod_l calH_{alpha_l} f)|interior, calH_l g_j = (1-alpha_l/12) g_j + alpha_l/24 (g_{j-1}+g_{j+1})
    on the closed grid including boundary samples."""
    G = np.asarray(f_closed, dtype=np.float64)
    d = G.ndim
    for l in range(d):
        V = np.moveaxis(G, l, 0)
        out = (1.0 - alpha[l] / 12.0) * V[1:-1] + (alpha[l] / 24.0) * (V[:-2] + V[2:])
        G = np.moveaxis(out, 0, l)
    return G


def appendix_F_d1(alpha1: float, f_closed: np.ndarray) -> np.ndarray:
    """F = H_alpha f + alpha_1/24 f_0, f_0 = [f(a),0,...,0,f(b)]."""
    n = f_closed.size - 2
    H = fcd.h_matrix(alpha1, n)
    f0 = np.zeros(n)
    f0[0] += f_closed[0]
    f0[-1] += f_closed[-1]
    return H @ f_closed[1:-1] + alpha1 / 24.0 * f0


def appendix_F_d2(alpha1: float, alpha2: float, f_closed: np.ndarray) -> np.ndarray:
    """Literal d=2 Appendix, paper-order vector (axis 1 fastest).

    F = H_alpha f + (H_{alpha_2} (x) alpha_1/24 I) f_1 + alpha_2/24 [H_{alpha_1} g_1; 0; H_{alpha_1} g_2]
        + alpha_1 alpha_2/576 [g_3; 0; g_4].
    "N_1" at P:671 is read as N; n1 != n2 is allowed.
    """
    n1, n2 = f_closed.shape[0] - 2, f_closed.shape[1] - 2
    H1, H2 = fcd.h_matrix(alpha1, n1), fcd.h_matrix(alpha2, n2)
    # f(x_{1,j1}, x_{2,j2}) = f_closed[j1, j2]
    fG = D.vec(f_closed[1:-1, 1:-1])
    f1 = np.zeros((n1, n2))
    f1[0, :] += f_closed[0, 1:-1]
    f1[-1, :] += f_closed[-1, 1:-1]
    g1 = f_closed[1:-1, 0]
    g2 = f_closed[1:-1, -1]
    g3 = np.zeros(n1)
    g3[0] += f_closed[0, 0]
    g3[-1] += f_closed[-1, 0]
    g4 = np.zeros(n1)
    g4[0] += f_closed[0, -1]
    g4[-1] += f_closed[-1, -1]
    Halpha = np.kron(H2, H1)
    F = Halpha @ fG + np.kron(H2, alpha1 / 24.0 * np.eye(n1)) @ D.vec(f1)
    blk = np.zeros((n1, n2))
    blk[:, 0] += H1 @ g1
    blk[:, -1] += H1 @ g2
    F += alpha2 / 24.0 * D.vec(blk)
    blk = np.zeros((n1, n2))
    blk[:, 0] += g3
    blk[:, -1] += g4
    F += alpha1 * alpha2 / 576.0 * D.vec(blk)
    return F


# ---------------------------------------------------------------------------
# e-bar
# ---------------------------------------------------------------------------
def e_bar(prob):
    """(ebar, ehat, echeck): max/min of e over the interior grid x half levels."""
    ehat, echeck = -np.inf, np.inf
    for m in range(prob.M):
        e = prob.e_grid(prob.t_half(m))
        ehat = max(ehat, float(e.max()))
        echeck = min(echeck, float(e.min()))
    if echeck <= 0.0:
        raise ValueError("e must be positive (P:33)")
    return 0.5 * (ehat + echeck), ehat, echeck


def source_F(prob, m: int) -> np.ndarray:
    """F^{(m+1/2)} as a grid array (closed-grid compact stencil of f at t_{m+1/2})."""
    return compact_source(prob.alpha, prob.f_closed(prob.t_half(m)))


# ---------------------------------------------------------------------------
# time loop
# ---------------------------------------------------------------------------
@dataclass
class SolveReport:
    iters: List[int] = field(default_factory=list)
    relres: List[float] = field(default_factory=list)
    converged: List[bool] = field(default_factory=list)

    @property
    def mean_iters(self):
        return float(np.mean(self.iters)) if self.iters else 0.0


def solve(prob, steps: Optional[int] = None, u0: Optional[np.ndarray] = None,
          fixed_iters: Optional[List[int]] = None, restart: Optional[int] = None,
          tol: Optional[float] = None, max_iters: Optional[int] = None,
          ebar: Optional[float] = None, F_static: Optional[np.ndarray] = None,
          tier: str = "L", sided: int = 1):
    """March ``steps`` CN steps (default M) of Eq.(tls) with tau-preconditioned GMRES.

    sided=1: the one-sided system P^{-1} A~ u = P^{-1} b~ (Eq.(one-sided));
    sided=2: the two-sided system P^{-1/2} A~ P^{-1/2} u~ = P^{-1/2} b~, u = P^{-1/2} u~ (Eq.(Pls),
    P:223-232), started from u~_0 = P^{1/2} u^{(m)} (so that u_0 = u^{(m)}, Thm 3.9).
    Returns (u, report, ebar).  ``tier='D'`` uses dense matrices (tiny grids)."""
    steps = prob.M if steps is None else steps
    restart = prob.restart if restart is None else restart
    tol = prob.tol if tol is None else tol
    max_iters = 10 * restart if max_iters is None else max_iters
    if ebar is None:
        ebar = e_bar(prob)[0]
    u = prob.psi_interior() if u0 is None else np.array(u0, dtype=np.float64)
    rep = SolveReport()
    if tier == "D":
        Ds = D.DenseSystem(prob.d, prob.n, prob.alpha, prob.kappa, prob.tau)
        Pinv = np.linalg.inv(Ds.P_alpha(ebar))
        Hinv = np.linalg.inv(Ds.H_alpha())
        w, Q = np.linalg.eigh(Ds.P_alpha(ebar))
        Pmh = (Q / np.sqrt(w)) @ Q.T       # P^{-1/2}
        Pph = (Q * np.sqrt(w)) @ Q.T       # P^{1/2}
    else:
        Ls = LineSystem(prob.d, prob.n, prob.alpha, prob.kappa, prob.tau)
    for m in range(steps):
        e = prob.e_grid(prob.t_half(m))
        F = F_static if F_static is not None else source_F(prob, m)
        fx = None if fixed_iters is None else fixed_iters[m]
        if tier == "D":
            b = Ds.b(e, D.vec(u), D.vec(F))
            if sided == 1:
                Kmat = Pinv @ Ds.A_tilde(e)
                res = gmres(lambda v: Kmat @ v, Pinv @ (Hinv @ b), D.vec(u), restart, tol, max_iters, fx)
                u_new = D.unvec(res.x, prob.n)
            else:
                Kmat = Pmh @ Ds.A_tilde(e) @ Pmh
                res = gmres(lambda v: Kmat @ v, Pmh @ (Hinv @ b), Pph @ D.vec(u), restart, tol, max_iters, fx)
                u_new = D.unvec(Pmh @ res.x, prob.n)
        else:
            b = Ls.rhs(e, u, F)
            if sided == 1:
                c = Ls.P_alpha_inv(ebar, Ls.H_alpha_inv(b))
                K = lambda v: Ls.P_alpha_inv(ebar, Ls.A_tilde(e, v))
                res = gmres(K, c, u, restart, tol, max_iters, fx)
                u_new = res.x
            else:
                c = Ls.P_alpha_inv_sqrt(ebar, Ls.H_alpha_inv(b))
                K = lambda v: Ls.P_alpha_inv_sqrt(ebar, Ls.A_tilde(e, Ls.P_alpha_inv_sqrt(ebar, v)))
                res = gmres(K, c, Ls.P_alpha_sqrt(ebar, u), restart, tol, max_iters, fx)
                u_new = Ls.P_alpha_inv_sqrt(ebar, res.x)
        rep.iters.append(res.iters)
        rep.relres.append(res.relres_est)
        rep.converged.append(res.converged)
        u = u_new
    return u, rep, ebar
