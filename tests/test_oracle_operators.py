"""Pins of the oracle's operators: Tier D (literal dense Kronecker assembly) vs Tier L
(per-line), the paper's identities, the RHS Appendix, e-bar and the seeded generator."""
import math

import numpy as np
import pytest

from oracle import dense as D
from oracle import fcd
from oracle import lines as L
from oracle import scheme
from paper_2404_10221_b200 import inputs as I

# anisotropic tiny grids: distinct n_i, alpha_i, kappa_i pin the axis <-> (alpha, kappa, n) association
CASES = [
    (1, (7,), (1.3,), (1.0,)),
    (1, (5,), (2.0,), (0.7,)),
    (2, (5, 4), (1.2, 1.8), (1.0, 0.5)),
    (2, (3, 6), (1.5, 1.1), (2.0, 1.0)),
    (3, (5, 4, 6), (1.2, 1.5, 1.9), (1.0, 0.5, 2.0)),
    (3, (3, 2, 4), (1.9, 1.1, 1.4), (0.3, 1.0, 1.7)),
]


def _sys(case, tau=0.25):
    d, n, a, k = case
    return D.DenseSystem(d, n, a, k, tau), L.LineSystem(d, n, a, k, tau)


def _rand(n, seed):
    return np.random.default_rng(seed).uniform(-1, 1, n)


@pytest.mark.parametrize("case", CASES)
def test_tier_d_equals_tier_l(case):
    Ds, Ls = _sys(case)
    n = case[1]
    x = _rand(n, 1)
    e = 1.0 + _rand(n, 2) ** 2
    F = _rand(n, 3)
    v = D.vec(x)
    def chk(dense_vec, arr):
        ref = D.unvec(dense_vec, n)
        assert np.max(np.abs(ref - arr)) <= 1e-13 * max(1.0, np.abs(ref).max())
    chk(Ds.H_alpha() @ v, Ls.H_alpha(x))
    chk(Ds.S_alpha() @ v, Ls.S_alpha(x))
    chk(Ds.A(e) @ v, Ls.A(e, x))
    chk(Ds.A_tilde(e) @ v, Ls.A_tilde(e, x))
    chk(Ds.b(e, v, D.vec(F)), Ls.rhs(e, x, F))
    chk(np.linalg.solve(Ds.H_alpha(), v), Ls.H_alpha_inv(x))
    ebar = 1.37
    chk(np.linalg.solve(Ds.P_alpha(ebar), v), Ls.P_alpha_inv(ebar, x))
    chk(np.linalg.solve(Ds.P_hat(ebar), v), Ls.P_hat_inv(ebar, x))
    w, Q = np.linalg.eigh(Ds.P_alpha(ebar))
    chk((Q / np.sqrt(w)) @ Q.T @ v, Ls.P_alpha_inv_sqrt(ebar, x))
    chk(Ds.dst() @ v, Ls.dst(x))


@pytest.mark.parametrize("case", CASES)
def test_key_identity_one_sided_equals_A_form(case):
    # P_alpha^{-1} A~ = (H P_alpha)^{-1} A = P_hat^{-1} A and P_alpha^{-1} b~ = P_hat^{-1} b
    # (tau matrices commute)
    Ds, _ = _sys(case)
    n = case[1]
    e = 1.0 + _rand(n, 5) ** 2
    ebar = 0.5 * (e.max() + e.min())
    K1 = np.linalg.solve(Ds.P_alpha(ebar), Ds.A_tilde(e))
    K2 = np.linalg.solve(Ds.P_hat(ebar), Ds.A(e))
    assert np.max(np.abs(K1 - K2)) < 1e-13 * np.abs(K1).max()
    b = _rand(Ds.Ntot, 6)
    c1 = np.linalg.solve(Ds.P_alpha(ebar), np.linalg.solve(Ds.H_alpha(), b))
    c2 = np.linalg.solve(Ds.P_hat(ebar), b)
    assert np.max(np.abs(c1 - c2)) < 1e-13 * np.abs(c1).max()


@pytest.mark.parametrize("case", CASES)
def test_preconditioner_spectrum_and_lemma_3_1(case):
    # P_alpha = S Lambda_P S with Lambda_P = ebar + sum eta_i q_i / lambda^H_i, built from the
    # literal P_alpha = ebar I + H^{-1/2} tau(S_alpha) H^{-1/2} (Eq.(Pa)); Lemma 3.1: SPD, Lambda_P > ebar
    Ds, Ls = _sys(case)
    ebar = 1.5
    S = Ds.dst()
    lamP = D.vec(Ls.lambda_P(ebar))
    P = Ds.P_alpha(ebar)
    assert np.max(np.abs(S @ np.diag(lamP) @ S - P)) < 1e-13 * np.abs(P).max()
    assert np.all(lamP > ebar)
    assert np.all(np.linalg.eigvalsh(P) > 0)
    lamHat = lamP * D.vec(Ls.lambda_H())
    Ph = Ds.P_hat(ebar)
    assert np.max(np.abs(S @ np.diag(lamHat) @ S - Ph)) < 1e-13 * np.abs(Ph).max()


@pytest.mark.parametrize("case", CASES[2:])
def test_commutativity_P198(case):
    # H^{-1/2} tau(S) H^{-1/2} = H^{-1} tau(S) = tau(S) H^{-1}
    Ds, _ = _sys(case)
    Hm = Ds.H_alpha_pow(-0.5)
    Hi = np.linalg.inv(Ds.H_alpha())
    T = Ds.tau_S_alpha()
    a, b, c = Hm @ T @ Hm, Hi @ T, T @ Hi
    assert np.max(np.abs(a - b)) < 1e-12 * np.abs(a).max()
    assert np.max(np.abs(a - c)) < 1e-12 * np.abs(a).max()


def test_kronecker_sum_of_H_inverse_S():
    # H_alpha^{-1} S_alpha = sum_i eta_i (I (x) .. (x) H_i^{-1} S_i (x) .. (x) I) (SURVEY VN-3)
    Ds, _ = _sys(CASES[4])
    lhs = np.linalg.solve(Ds.H_alpha(), Ds.S_alpha())
    rhs = np.zeros_like(lhs)
    for i in range(Ds.d):
        mats = [np.eye(Ds.n[l]) if l != i else np.linalg.solve(Ds.H1[i], Ds.S1[i]) for l in range(Ds.d)]
        rhs += Ds.eta[i] * D.kron_paper(mats)
    assert np.max(np.abs(lhs - rhs)) < 1e-13 * np.abs(lhs).max()


# ---------------------------------------------------------------- RHS F (Appendix)
def test_appendix_d1_equals_compact_stencil():
    f = np.random.default_rng(7).uniform(-1, 1, 11)
    assert np.max(np.abs(scheme.appendix_F_d1(1.3, f) - scheme.compact_source((1.3,), f))) < 1e-15


def test_appendix_d1_f_one_gives_one():
    # f = 1 gives F = 1 (row sums of H are 1 inside, the end corrections restore 1)
    F = scheme.appendix_F_d1(1.7, np.ones(9))
    assert np.max(np.abs(F - 1)) < 1e-15


@pytest.mark.parametrize("shape", [(5, 5), (4, 6)])
def test_appendix_d2_equals_compact_stencil(shape):
    f = np.random.default_rng(8).uniform(-1, 1, (shape[0] + 2, shape[1] + 2))
    lit = scheme.appendix_F_d2(1.2, 1.8, f)
    gen = D.vec(scheme.compact_source((1.2, 1.8), f))
    assert np.max(np.abs(lit - gen)) < 1e-14


def test_interior_only_source_is_H_alpha_f():
    # a source vanishing on the boundary gives F = H_alpha f (all boundary vectors vanish)
    n = (4, 3, 5)
    Ls = L.LineSystem(3, n, (1.2, 1.5, 1.9), (1, 1, 1), 0.1)
    r = np.random.default_rng(9).uniform(-1, 1, n)
    f = np.zeros([k + 2 for k in n])
    f[1:-1, 1:-1, 1:-1] = r
    assert np.max(np.abs(scheme.compact_source((1.2, 1.5, 1.9), f) - Ls.H_alpha(r))) < 1e-15


# ---------------------------------------------------------------- e-bar
def test_ebar_constant_and_scan():
    p = I.config_c1(n=15, M=8)
    eb, eh, ec = scheme.e_bar(p)
    ts = [(m + 0.5) / 8 for m in range(8)]
    x = np.arange(1, 16) / 16
    vals = [1 + 0.5 * np.sin(np.pi * x) * math.exp(-t) for t in ts]
    assert eh == max(v.max() for v in vals) and ec == min(v.min() for v in vals)
    assert eb == 0.5 * (eh + ec)


# ---------------------------------------------------------------- closed-form sources
def test_left_rl_printed_value():
    # left RL of x^4, alpha = 1.5, at x = 1 is Gamma(5)/Gamma(3.5) = 7.2216
    c = [0, 0, 0, 0, 1.0]
    assert abs(I.left_rl_poly(c, 1.5, np.array([1.0]))[0] - 7.2216) < 1e-4


@pytest.mark.parametrize("alpha", [1.2, 1.5, 1.9])
def test_fcd_approximates_riesz_derivative(alpha):
    # -h^{-alpha} S_alpha p -> d^alpha p for smooth p with zero extension: O(h^2) ([Celik]).
    # Pins sigma_alpha, the reflection and the sign of the source against the FCD operator.
    errs = []
    for N1 in (128, 256, 512):
        n = N1 - 1
        h = 1.0 / N1
        x = np.arange(1, N1) * h
        p = I.poly_eval(I.P4, x)
        s = fcd.fcd_coefficients(alpha, n).astype(float)
        approx = -h ** (-alpha) * (fcd.toeplitz_matrix(s) @ p)
        errs.append(np.max(np.abs(approx - I.riesz_poly(I.P4, alpha, x))))
    assert 3.7 < errs[0] / errs[1] < 4.3 and 3.9 < errs[1] / errs[2] < 4.1


# ---------------------------------------------------------------- seeded generator
def test_splitmix_numpy_equals_integer_reference():
    seed = I.SEED_BASE + 5
    cnt = np.array([0, 1, 2, 12345, 2 ** 40 + 3], dtype=np.uint64)
    got = I.splitmix64_uniform(seed, cnt)
    ref = [I.splitmix64_uniform_scalar(seed, int(c)) for c in cnt]
    assert np.array_equal(got, np.array(ref))
    f = I.seeded_field(seed, (7, 5, 3))
    # paper order: the counter of node (j1,j2,j3) is (j1-1) + 7 ((j2-1) + 5 (j3-1))
    assert f[2, 1, 2] == I.splitmix64_uniform_scalar(seed, 2 + 7 * (1 + 5 * 2))
    big = I.seeded_field(1, (200, 300))
    assert big.min() >= -1 and big.max() < 1 and abs(big.mean()) < 0.01
