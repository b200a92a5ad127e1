"""NEXT-3: spectral / convergence diagnostics (oracle side, dense, CPU).

Pins the numerical-range routine against closed forms and brute force, then checks Theorem 3.7
 on our operators: the numerical-range bounds of A_breve = P^{-1/2} A~ P^{-1/2}
(Eq.(Theq4)), the GMRES residual bound (2+c) c^k, that the spectrum of P^{-1} A~ lies in W(A_breve),
and the clustering that Figs 1-3 show."""
import math

import numpy as np
import pytest

from oracle import dense as D
from oracle import diagnostics as G
from oracle import scheme
from oracle.gmres import gmres
from paper_2404_10221_b200 import inputs as I


# ------------------------------------------------------------------ the numerical-range routine
def test_numerical_range_hermitian_is_the_eigenvalue_interval():
    rng = np.random.default_rng(3)
    B = rng.standard_normal((9, 9))
    A = B @ B.T + 0.5 * np.eye(9)
    w = np.linalg.eigvalsh(A)
    v, r = G.numerical_range_extremes(A)
    assert abs(v - w[0]) < 1e-9 * w[-1] and abs(r - w[-1]) < 1e-9 * w[-1]


def test_numerical_range_normal_matrix_is_the_hull_of_its_eigenvalues():
    # W(diag(l)) = conv{l}: brute force over convex combinations of the three eigenvalues
    lam = np.array([1 + 1j, 3 + 0j, 2 - 2j])
    v, r = G.numerical_range_extremes(np.diag(lam))
    t = np.linspace(0, 1, 401)
    a, b = np.meshgrid(t, t)
    ok = a + b <= 1
    z = (a[ok] * lam[0] + b[ok] * lam[1] + (1 - a[ok] - b[ok]) * lam[2])
    assert abs(r - np.abs(lam).max()) < 1e-9
    assert abs(v - np.abs(z).min()) < 2e-3          # grid resolution of the brute force
    assert v <= np.abs(z).min() + 1e-12               # v is the exact minimum


def test_numerical_range_contains_zero_gives_zero_distance():
    A = np.array([[0.0, 1.0], [-1.0, 0.0]])         # W = i[-1, 1]
    v, r = G.numerical_range_extremes(A)
    assert v == 0.0 and abs(r - 1.0) < 1e-9


def test_theorem37_constant_matches_sin_theta_at_the_bounds():
    # c of P:333-337 is the largest sin(theta) = sqrt(1 - (v/r)^2) over the bound pairs of Eq.(Theq4)
    for eh, ec in [(2.0, 1.0), (1.5, 1.49), (10.0, 1.0)]:
        lo_e, hi_e = 2 * ec / (eh + ec), 2 * eh / (eh + ec)
        lo_t, hi_t = (4 - math.sqrt(6)) / 4, (4 + math.sqrt(6)) / 4
        s = max(math.sqrt(1 - (v / r) ** 2) for v in (lo_e, lo_t) for r in (hi_e, hi_t))
        assert abs(G.theorem37_bounds(eh, ec)[2] - s) < 1e-14


# ------------------------------------------------------------------ Theorem 3.7 on our operators
def _cases():
    return [
        ("ex1", I.example(1, 15, 64, (1.3,))),
        ("ex1b", I.example(1, 31, 16, (1.9,))),
        ("ex2", I.example(2, 7, 16, (1.5, 1.7))),
        ("c2", I.config_c2(n=7, M=4)),
        ("ex3", I.example(3, 5, 8, (1.1, 1.3, 1.5))),
        ("c5", I.config_c5(M=4, nn=(5, 4, 6))),
    ]


@pytest.mark.parametrize("name,prob", _cases(), ids=[c[0] for c in _cases()])
def test_theorem37_numerical_range_bounds(name, prob):
    ebar, ehat, echeck = scheme.e_bar(prob)
    lo, hi, c = G.theorem37_bounds(ehat, echeck)
    Ds = D.DenseSystem(prob.d, prob.n, prob.alpha, prob.kappa, prob.tau)
    for m in (0, prob.M - 1):
        Ab = G.two_sided_matrix(Ds, prob.e_grid(prob.t_half(m)), ebar)
        v, r = G.numerical_range_extremes(Ab, n_theta=720)
        assert v >= lo * (1 - 1e-9) and r <= hi * (1 + 1e-9), (v, lo, r, hi)
        # the spectrum of P^{-1} A~ (similar to A_breve) lies in W(A_breve): v <= |lambda| <= r
        _, lam = G.spectra(Ds, prob.e_grid(prob.t_half(m)), ebar)
        assert np.all(np.abs(lam) >= v * (1 - 1e-8)) and np.all(np.abs(lam) <= r * (1 + 1e-8))
        assert np.all(lam.real > 0)


@pytest.mark.parametrize("name,prob", _cases()[::2], ids=[c[0] for c in _cases()[::2]])
def test_theorem37_gmres_residual_bound(name, prob):
    # two-sided GMRES from a random start: ||r_k|| / ||r_0|| <= (2 + c) c^k at every k
    ebar, ehat, echeck = scheme.e_bar(prob)
    _, _, c = G.theorem37_bounds(ehat, echeck)
    Ds = D.DenseSystem(prob.d, prob.n, prob.alpha, prob.kappa, prob.tau)
    Ab = G.two_sided_matrix(Ds, prob.e_grid(prob.t_half(0)), ebar)
    rng = np.random.default_rng(7)
    N = Ab.shape[0]
    res = gmres(lambda x: Ab @ x, rng.standard_normal(N), rng.standard_normal(N), restart=N, tol=1e-13,
                max_iters=N)
    for k, h in enumerate(res.history):
        assert h <= (2 + c) * c ** k * (1 + 1e-9) + 1e-15, (k, h, (2 + c) * c ** k)


@pytest.mark.parametrize("d,n,alpha", [(1, 15, (1.5,)), (2, 15, (1.5, 1.7)), (3, 7, (1.5, 1.7, 1.9))])
def test_preconditioned_spectrum_is_clustered(d, n, alpha):
    # Figs 1-3: the eigenvalues of P^{-1} A~ are far more tightly clustered than those of A~
    prob = I.example(d, n, 4096 if d < 3 else 1024, alpha)
    ebar, _, _ = scheme.e_bar(prob)
    Ds = D.DenseSystem(prob.d, prob.n, prob.alpha, prob.kappa, prob.tau)
    lam_a, lam_p = G.spectra(Ds, prob.e_grid(prob.t_half(prob.M - 1)), ebar)
    spread = lambda z: np.abs(z).max() / np.abs(z).min()
    assert spread(lam_p) < 3.0 and spread(lam_a) > 10 * spread(lam_p), (spread(lam_p), spread(lam_a))
