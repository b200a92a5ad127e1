"""1-D structured operators of the scheme (oracle; test infrastructure only).

Every function follows PAPER.md (``P:n`` = line n) literally:

* FCD generator s_k^{(alpha)}            P:124-127, Eq.(eq0); reading Q1 (alpha/2 + k)
* H_alpha = I + alpha/24 tridiag(1,-2,1)  P:107-110, Eq.(Ha)
* S_alpha symmetric Toeplitz [s_|i-j|]
* eta_i = kappa_i tau / (2 h_i^alpha_i)
* Hankel H(T), antidiagonals [t2..t_{N-1},0,0,0,t_{N-1}..t2]
* tau(T) = T - H(T)                      P:141-145, Eq.(tau)
* q_i = t0 + 2 sum_j t_j cos(pi j (i+1)/(N+1))   P:155-159, Eq.(q); reading Q2 (N+1)
* S = [sqrt(2/(N+1)) sin(pi j k/(N+1))]
* lambda_k(H_alpha) = 1 - (alpha/6) sin^2(k pi/(2N+2))   P:305-314 (Lemma 3.5 proof)

Setup tables (s_k, q_i) are computed in x86 80-bit long double and rounded to
FP64 (the small-k q_i are heavily cancelling sums).
"""
from __future__ import annotations

import math

import numpy as np

LD = np.longdouble


def fcd_coefficients(alpha: float, n: int) -> np.ndarray:
    """s_0..s_{n-1} of the FCD generator, long double.

    s_0 = Gamma(alpha+1)/Gamma(alpha/2+1)^2,
    s_k = (1 - (alpha+1)/(alpha/2 + k)) s_{k-1}, k = 1..n-1.
    The printed denominator "alpha/2+1" is read as "alpha/2+k": the
    printed form violates the zero-sum property (As1).
    """
    if not (1.0 < alpha <= 2.0):
        raise ValueError("alpha must lie in (1, 2]")
    if n < 1:
        raise ValueError("n must be >= 1")
    a = LD(alpha)
    s = np.empty(n, dtype=LD)
    s[0] = LD(math.gamma(alpha + 1.0)) / LD(math.gamma(alpha / 2.0 + 1.0)) ** 2
    for k in range(1, n):
        s[k] = (LD(1) - (a + LD(1)) / (a / LD(2) + LD(k))) * s[k - 1]
    return s


def eta(kappa: float, tau: float, h: float, alpha: float) -> float:
    """eta_i = kappa_i tau / (2 h_i^alpha_i)."""
    return kappa * tau / (2.0 * h ** alpha)


def h_matrix(alpha: float, n: int) -> np.ndarray:
    """H_alpha = I_N + alpha/24 tridiag(1,-2,1)."""
    H = np.eye(n) * (1.0 - alpha / 12.0)
    i = np.arange(n - 1)
    H[i, i + 1] = alpha / 24.0
    H[i + 1, i] = alpha / 24.0
    return H


def toeplitz_matrix(t: np.ndarray) -> np.ndarray:
    """symmetric Toeplitz [T]_{ij} = t_{|i-j|}."""
    t = np.asarray(t, dtype=np.float64)
    n = t.size
    idx = np.abs(np.arange(n)[:, None] - np.arange(n)[None, :])
    return t[idx]


def hankel_part(t: np.ndarray) -> np.ndarray:
    """H(T): constant antidiagonals [t2,...,t_{N-1},0,0,0,t_{N-1},...,t2].

    Entry (i,j) (1-based) lies on antidiagonal number i+j-2 in 0..2N-2.
    """
    t = np.asarray(t, dtype=np.float64)
    n = t.size
    anti = np.concatenate([t[2:], np.zeros(3), t[2:][::-1]]) if n >= 2 else np.zeros(1)
    anti = anti[: 2 * n - 1]
    assert anti.size == 2 * n - 1
    ij = np.arange(n)[:, None] + np.arange(n)[None, :]
    return anti[ij]


def tau_matrix(t: np.ndarray) -> np.ndarray:
    """tau(T) = T - H(T)."""
    return toeplitz_matrix(t) - hankel_part(t)


def tau_eigenvalues(t: np.ndarray) -> np.ndarray:
    """q_i = t_0 + 2 sum_{j=1}^{N-1} t_j cos(pi j (i+1)/(N+1)), i=0..N-1 (Q2).

    Direct O(N^2) sum in long double; returns FP64.
    """
    t = np.asarray(t, dtype=LD)
    n = t.size
    j = np.arange(1, n, dtype=LD)
    q = np.empty(n, dtype=LD)
    # exact integer reduction of the angle: pi * (j (i+1) mod 2(N+1)) / (N+1)
    for i in range(n):
        r = (np.arange(1, n, dtype=np.int64) * (i + 1)) % (2 * (n + 1))
        ang = LD_PI * r.astype(LD) / LD(n + 1)
        q[i] = t[0] + LD(2) * np.sum(t[1:] * np.cos(ang))
    return q.astype(np.float64)


# pi to long-double precision (np.pi is a double; compute pi in long double)
LD_PI = LD(4) * np.arctan(LD(1))


def dst_matrix(n: int) -> np.ndarray:
    """S = [sqrt(2/(N+1)) sin(pi j k/(N+1))]_{j,k=1}^N."""
    jk = (np.arange(1, n + 1)[:, None] * np.arange(1, n + 1)[None, :]) % (2 * (n + 1))
    S = np.sqrt(LD(2) / LD(n + 1)) * np.sin(LD_PI * jk.astype(LD) / LD(n + 1))
    return S.astype(np.float64)


def h_eigenvalues(alpha: float, n: int) -> np.ndarray:
    """lambda_k(H_alpha) = 1 + alpha/24 * (-4 sin^2(k pi/(2N+2))), k=1..N.

    Ordered by k so that S H S = diag(lambda) with the DST-I of P:162.
    """
    k = np.arange(1, n + 1, dtype=LD)
    lam = LD(1) - LD(alpha) / LD(6) * np.sin(k * LD_PI / LD(2 * n + 2)) ** 2
    return lam.astype(np.float64)
