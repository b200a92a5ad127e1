"""Pins of the 1-D oracle pieces (oracle/fcd.py) against what the paper and mathematics fix."""
import math
import os

import numpy as np
import pytest
import scipy.fft
import scipy.special

from oracle import fcd

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def spec_value(name):
    with open(os.path.join(GOLD, "spec_values.txt")) as f:
        for line in f:
            if line.startswith(name + " "):
                return float(line.split()[1])
    raise KeyError(name)


ALPHAS = [1.1, 1.3, 1.5, 1.7, 1.9]


# ---------------------------------------------------------------- FCD generator
def test_fcd_alpha2_is_second_difference():
    # alpha = 2: s = [2, -1, 0, ...] -- the centred second difference
    s = fcd.fcd_coefficients(2.0, 6).astype(float)
    assert np.allclose(s, [2, -1, 0, 0, 0, 0], atol=1e-15)


def test_fcd_s0_printed_value():
    assert abs(float(fcd.fcd_coefficients(1.5, 1)[0]) - spec_value("s0_alpha_1.5")) < 1e-9


@pytest.mark.parametrize("alpha", ALPHAS)
def test_fcd_gamma_closed_form(alpha):
    # s_k = (-1)^k Gamma(alpha+1) / (Gamma(alpha/2 - k + 1) Gamma(alpha/2 + k + 1)):
    # independent closed form of the FCD weights; only the reading alpha/2 + k (Q1) matches it
    n = 60
    s = fcd.fcd_coefficients(alpha, n).astype(float)
    k = np.arange(n)
    closed = (-1.0) ** k * scipy.special.gamma(alpha + 1) * scipy.special.rgamma(alpha / 2 - k + 1) \
        * scipy.special.rgamma(alpha / 2 + k + 1)
    assert np.max(np.abs(s - closed) / np.abs(closed)) < 1e-12


@pytest.mark.parametrize("alpha", ALPHAS)
def test_fcd_As1_sign_and_zero_sum(alpha):
    # (As1) P:130-135: s_0 > 0, s_k < 0, s_0 + 2 sum s_k = 0 (partial sums decrease to 0)
    s = fcd.fcd_coefficients(alpha, 4096).astype(float)
    assert s[0] > 0 and np.all(s[1:] < 0)
    partial = s[0] + 2 * np.cumsum(s[1:])
    assert np.all(partial > 0) and np.all(np.diff(partial) < 0)
    assert partial[-1] < 1e-2
    # the tail behaves like K^{-alpha}: doubling K shrinks the remainder by ~2^alpha
    r1, r2 = partial[1022], partial[4094]          # K = 1023 and 4095 terms
    assert 0.7 * 4 ** alpha < r1 / r2 < 1.3 * 4 ** alpha


def test_fcd_printed_denominator_violates_As1():
    # reading Q1: the printed constant denominator alpha/2+1 gives a geometric sequence whose
    # generator does not sum to zero, contradicting (As1) -- so the printed form cannot be meant
    alpha = 1.5
    ratio = 1 - (alpha + 1) / (alpha / 2 + 1)
    s0 = float(fcd.fcd_coefficients(alpha, 1)[0])
    printed_sum = s0 + 2 * s0 * ratio / (1 - ratio)
    assert abs(printed_sum) > 0.5


@pytest.mark.parametrize("alpha", [1.2, 1.5, 1.9])
def test_fcd_generating_function(alpha):
    # the FCD symbol: s_0 + 2 sum_k s_k cos(k theta) = (2 sin(theta/2))^alpha  ([Celik])
    K = 2_000_000
    k = np.arange(1, K)
    s0 = math.gamma(alpha + 1) / math.gamma(alpha / 2 + 1) ** 2
    s = s0 * np.cumprod(1 - (alpha + 1) / (alpha / 2 + k))
    for theta in (0.7, 2.0):
        val = s0 + 2 * np.sum(s * np.cos(k * theta))
        assert abs(val - (2 * math.sin(theta / 2)) ** alpha) < 1e-6


# ---------------------------------------------------------------- DST-I
@pytest.mark.parametrize("n", [1, 2, 3, 7, 31, 64])
def test_dst_symmetric_involution(n):
    S = fcd.dst_matrix(n)
    assert np.allclose(S, S.T, atol=0)
    assert np.max(np.abs(S @ S - np.eye(n))) < 1e-14


def test_dst_small_values():
    assert np.allclose(fcd.dst_matrix(1), [[1.0]], atol=1e-16)
    col = fcd.dst_matrix(3)[:, 0]
    ref = [spec_value("dst_n3_e1_0"), spec_value("dst_n3_e1_1"), spec_value("dst_n3_e1_2")]
    assert np.max(np.abs(col - ref)) < 1e-15


@pytest.mark.parametrize("n", [5, 16, 255])
def test_dst_matches_scipy(n):
    x = np.random.default_rng(n).standard_normal(n)
    ref = scipy.fft.dst(x, type=1, norm="ortho")
    assert np.max(np.abs(fcd.dst_matrix(n) @ x - ref)) < 1e-13


# ---------------------------------------------------------------- tau algebra
def test_hankel_small_cases():
    # n <= 2 -> zero (no t_2 exists).  SPEC S:126 claims n <= 3, but for N = 3 the list
    # [t_2, 0, 0, 0, t_2] puts t_2 in the corners, and only that H(T) makes tau(T) = S Q S
    # (test_tau_eigenvalues_bruteforce[n=3]); n=5 first column read off the antidiagonals
    for n in (1, 2):
        assert np.all(fcd.hankel_part(np.arange(1.0, n + 1)) == 0)
    assert np.array_equal(fcd.hankel_part(np.array([1.0, 2.0, 3.0])), np.diag([3.0, 0.0, 3.0]))
    t = np.array([5.0, -1.0, -0.5, -0.3, -0.2])
    assert np.allclose(fcd.hankel_part(t)[:, 0], [-0.5, -0.3, -0.2, 0, 0], atol=0)
    H = fcd.hankel_part(t)
    assert np.allclose(H, H.T) and np.allclose(H, H[::-1, ::-1])


@pytest.mark.parametrize("alpha", [1.1, 1.5, 1.9])
@pytest.mark.parametrize("n", [1, 2, 3, 5, 16, 31])
def test_tau_eigenvalues_bruteforce(alpha, n):
    s = fcd.fcd_coefficients(alpha, n)
    q = fcd.tau_eigenvalues(s)
    tau = fcd.tau_matrix(s.astype(float))
    # brute force: dense symmetric eigensolve of tau(T) = T - H(T)
    assert np.max(np.abs(np.sort(q) - np.linalg.eigvalsh(tau))) < 1e-13 * np.abs(q).max()
    # and tau(T) = S Q S (Eq.(diag)) with q in DST order
    S = fcd.dst_matrix(n)
    assert np.max(np.abs(S @ np.diag(q) @ S - tau)) < 1e-13 * np.abs(tau).max()


def test_tau_eigenvalue_divisor_N_is_wrong():
    # reading Q2: the printed divisor N does not diagonalise tau(T); N+1 does
    n, alpha = 16, 1.5
    s = fcd.fcd_coefficients(alpha, n).astype(float)
    i = np.arange(n)[:, None]
    j = np.arange(1, n)[None, :]
    q_printed = s[0] + 2 * np.sum(s[1:] * np.cos(np.pi * j * (i + 1) / n), axis=1)
    S = fcd.dst_matrix(n)
    err = np.max(np.abs(S @ np.diag(q_printed) @ S - fcd.tau_matrix(s)))
    assert err > 1e-3


@pytest.mark.parametrize("n", [1, 4, 31, 255])
def test_tau_laplacian_closed_form(n):
    t = np.zeros(n)
    t[0] = 2.0
    if n > 1:
        t[1] = -1.0
    k = np.arange(1, n + 1)
    assert np.max(np.abs(fcd.tau_eigenvalues(t) - 4 * np.sin(k * np.pi / (2 * n + 2)) ** 2)) < 1e-15


@pytest.mark.parametrize("alpha", [1.1, 1.5, 1.9])
@pytest.mark.parametrize("n", [4, 16, 31])
def test_lemma_3_4_hankel_bound(alpha, n):
    # Lemma 3.4: || tau(T)^{-1/2} H(T) tau(T)^{-1/2} ||_2 < 1/2
    s = fcd.fcd_coefficients(alpha, n).astype(float)
    w, Q = np.linalg.eigh(fcd.tau_matrix(s))
    R = (Q / np.sqrt(w)) @ Q.T
    assert np.linalg.norm(R @ fcd.hankel_part(s) @ R, 2) < 0.5


# ---------------------------------------------------------------- H_alpha
@pytest.mark.parametrize("alpha", [1.1, 1.5, 1.9, 2.0])
@pytest.mark.parametrize("n", [1, 4, 31])
def test_h_eigenvalues(alpha, n):
    lam = fcd.h_eigenvalues(alpha, n)
    H = fcd.h_matrix(alpha, n)
    assert np.max(np.abs(np.sort(lam) - np.linalg.eigvalsh(H))) < 1e-15
    S = fcd.dst_matrix(n)
    assert np.max(np.abs(S @ H @ S - np.diag(lam))) < 1e-14       # H is a tau matrix
    assert np.all(lam > 2 / 3) and np.all(lam < 1)                 # Lemma 3.5
    assert math.sqrt(lam.max() / lam.min()) <= math.sqrt(6) / 2     # cond(H^{1/2}) <= sqrt6/2


def test_h_eigenvalues_spec_example():
    # alpha=1.5, n=4 -> 1 - 0.25 sin^2(k pi/10)
    k = np.arange(1, 5)
    assert np.allclose(fcd.h_eigenvalues(1.5, 4), 1 - 0.25 * np.sin(k * np.pi / 10) ** 2, atol=1e-16)


# ---------------------------------------------------------------- extended-precision pin of q
def mp_tau_eigenvalues(alpha, n, ks, dps=30):
    """q(k) = s_0 + 2 sum_{j=1}^{n-1} s_j cos(pi j k/(n+1)) (Eq.(q), divisor n+1 per Q2) with
    s_j from the Gamma closed form (-1)^j Gamma(alpha+1) / (Gamma(alpha/2-j+1) Gamma(alpha/2+j+1))
    -- not the oracle's recurrence -- evaluated with 30 significant digits (mpmath)."""
    import mpmath as mp
    with mp.workdps(dps):
        a = mp.mpf(alpha)
        g = mp.gamma(a + 1)
        s = [(-1) ** j * g / (mp.gamma(a / 2 - j + 1) * mp.gamma(a / 2 + j + 1)) for j in range(n)]
        out = []
        for k in ks:
            acc = s[0]
            for j in range(1, n):
                acc += 2 * s[j] * mp.cos(mp.pi * j * k / (n + 1))
            out.append(acc)
        return [float(v) for v in out]


@pytest.mark.parametrize("alpha,n", [(1.1, 511), (1.5, 511), (1.9, 511), (1.2, 2047), (1.9, 2047)])
def test_tau_eigenvalues_match_30_digit_reference(alpha, n):
    # the small-k eigenvalues are heavily cancelling sums (condition up to ~1e6 at alpha=1.9,
    # n=2047): a plain FP64 sum is off by up to 2.5e-11 there (7e-12 at n=511), enough to move
    # P_hat^{-1} x by more than the 1e-12 parity bar; the oracle's long-double recurrence and sum
    # stay within 3e-14 (measured worst case: q(1) at alpha=1.9, n=2047) -- bar 1e-13
    ks = list(range(1, 9))
    ref = np.array(mp_tau_eigenvalues(alpha, n, ks))
    q = fcd.tau_eigenvalues(fcd.fcd_coefficients(alpha, n))[:8]
    assert np.max(np.abs(q - ref) / np.abs(ref)) < 1e-13, np.abs(q - ref) / np.abs(ref)
