"""Seeded, synthetic problem inputs shared by the CPU oracle and the GPU harness.

This module holds *problem data only* -- grids, the coefficient function e(x,t),
the source f(x,t), the initial value psi, and the counter-based seeded field --
and none of the method's arithmetic (no FCD generator, no tau algebra, no
operators, no GMRES).  Both ``oracle/`` and the GPU harness draw their inputs
from here, as DESIGN.md section "Input recipe" states.

Citations: ``P:n`` = line n of /root/reference/PAPER.md (arXiv 2404.10221).

* Problem: e(x,t) d_t u = sum_i kappa_i d^{alpha_i} u + f on (0,1)^d,
  u = 0 on the boundary, u(x,0) = psi(x).
* Riesz derivative: d^alpha = sigma_alpha (left RL + right RL),
  sigma_alpha = -1/(2 cos(alpha pi/2)).  Used here only to build closed-form
  manufactured sources f (the continuous PDE, not the discrete method).
* Grid: h_i = 1/(n_i+1), x_{i,j} = j h_i, j = 0..n_i+1; time levels
  t_m = m tau, tau = T/M, half levels t_{m+1/2}.
* Configs C1..C5 are BASELINE.json ``configs[0..4]``; Examples 1-3 are
  P:523-526.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable, Optional, Sequence

import numpy as np

# ----------------------------------------------------------------------------
# Counter-based seeded field: SplitMix64 finaliser of a counter.
# r(J) = 2*((z >> 11) * 2^-53) - 1, z = mix64(seed + (l(J)+1) * GOLDEN), where
# l(J) is the paper-order linear index of the interior node J (axis 1 fastest,
# P:104 Kronecker order).  Exact in FP64, bit-identical on any platform.
# ----------------------------------------------------------------------------
GOLDEN = 0x9E3779B97F4A7C15
MIX1 = 0xBF58476D1CE4E5B9
MIX2 = 0x94D049BB133111EB
MASK64 = (1 << 64) - 1
SEED_BASE = 240410221


def splitmix64_uniform(seed: int, counters: np.ndarray) -> np.ndarray:
    """uniform[-1,1) values for uint64 ``counters`` (vectorised, wraps mod 2^64)."""
    c = np.asarray(counters, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed & MASK64) + (c + np.uint64(1)) * np.uint64(GOLDEN)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(MIX1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(MIX2)
        z = z ^ (z >> np.uint64(31))
    w = (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    return 2.0 * w - 1.0


def splitmix64_uniform_scalar(seed: int, counter: int) -> float:
    """Pure-Python integer version of :func:`splitmix64_uniform` (test pin)."""
    z = (seed + (counter + 1) * GOLDEN) & MASK64
    z = ((z ^ (z >> 30)) * MIX1) & MASK64
    z = ((z ^ (z >> 27)) * MIX2) & MASK64
    z ^= z >> 31
    return 2.0 * ((z >> 11) * 2.0 ** -53) - 1.0


def seeded_field(seed: int, n: Sequence[int]) -> np.ndarray:
    """Seeded uniform[-1,1) field on the interior grid, array shape ``tuple(n)``.

    Array index [j1-1, ..., jd-1] holds node J; the counter is the paper-order
    index l(J) = (j1-1) + n1*((j2-1) + n2*(j3-1)) (axis 1 fastest).
    """
    n = tuple(int(v) for v in n)
    d = len(n)
    # paper order: flatten with axis 1 fastest == Fortran order of shape n
    total = int(np.prod(n))
    out = np.empty(total, dtype=np.float64)
    chunk = 1 << 24
    for s in range(0, total, chunk):
        e = min(total, s + chunk)
        out[s:e] = splitmix64_uniform(seed, np.arange(s, e, dtype=np.uint64))
    return np.ascontiguousarray(out.reshape(n, order="F")) if d > 1 else out


def seeded_vector(seed: int, n: Sequence[int]) -> np.ndarray:
    """Seeded uniform test vector (same generator, used for operator parity)."""
    return seeded_field(seed, n)


# ----------------------------------------------------------------------------
# Riesz derivative of a polynomial on (0,1) in closed form.
# left RL of x^m: Gamma(m+1)/Gamma(m+1-alpha) x^(m-alpha); the right RL of p is
# the left RL of p(1-s) evaluated at 1-x.
# ----------------------------------------------------------------------------
def _poly_reflect(c: Sequence[float]) -> np.ndarray:
    """coefficients of q(s) = p(1-s) given p(x) = sum c_m x^m."""
    c = np.asarray(c, dtype=np.float64)
    deg = len(c) - 1
    q = np.zeros(deg + 1)
    for m, cm in enumerate(c):
        # (1-s)^m = sum_k C(m,k) (-s)^k
        for k in range(m + 1):
            q[k] += cm * math.comb(m, k) * (-1.0) ** k
    return q


def left_rl_poly(c: Sequence[float], alpha: float, x: np.ndarray) -> np.ndarray:
    """Left Riemann-Liouville derivative of order alpha of sum c_m x^m at x."""
    x = np.asarray(x, dtype=np.float64)
    out = np.zeros_like(x)
    for m, cm in enumerate(c):
        if cm == 0.0:
            continue
        if m < 2:
            raise ValueError("monomials of degree < 2 are singular at 0 for alpha in (1,2)")
        out += cm * math.gamma(m + 1) / math.gamma(m + 1 - alpha) * x ** (m - alpha)
    return out


def sigma_alpha(alpha: float) -> float:
    """sigma_alpha = -1/(2 cos(alpha pi / 2))."""
    return -1.0 / (2.0 * math.cos(alpha * math.pi / 2.0))


def riesz_poly(c: Sequence[float], alpha: float, x: np.ndarray) -> np.ndarray:
    """Riesz derivative d^alpha p on (0,1) of the polynomial p = sum c_m x^m."""
    x = np.asarray(x, dtype=np.float64)
    q = _poly_reflect(c)
    return sigma_alpha(alpha) * (left_rl_poly(c, alpha, x) + left_rl_poly(q, alpha, 1.0 - x))


# p2 = x^2 (1-x)^2 and p4 = x^4 (1-x)^4 as coefficient lists
P2 = [0.0, 0.0, 1.0, -2.0, 1.0]
P4 = [0.0] * 4 + [float(math.comb(4, k) * (-1) ** k) for k in range(5)]


def poly_eval(c: Sequence[float], x: np.ndarray) -> np.ndarray:
    x = np.asarray(x, dtype=np.float64)
    out = np.zeros_like(x)
    for m in range(len(c) - 1, -1, -1):
        out = out * x + c[m]
    return out


# ----------------------------------------------------------------------------
# Problem description
# ----------------------------------------------------------------------------
@dataclass
class SeparableCoeff:
    """e(x,t) = a(t) + b(t) * prod_i g_i(x_i) + sum_i k_i(x_i).

    ``g[i]``/``k[i]`` may be None (meaning 1 resp. 0)."""
    a: Callable[[float], float]
    b: Callable[[float], float]
    g: Sequence[Optional[Callable[[np.ndarray], np.ndarray]]]
    k: Sequence[Optional[Callable[[np.ndarray], np.ndarray]]]


@dataclass
class Problem:
    name: str
    d: int
    n: tuple
    alpha: tuple
    kappa: tuple
    M: int
    T: float
    coeff: SeparableCoeff
    # f(xs, t) on arrays broadcast over the closed grid
    source: Callable[[Sequence[np.ndarray], float], np.ndarray]
    # psi(xs) on the interior grid
    psi: Callable[[Sequence[np.ndarray]], np.ndarray]
    exact: Optional[Callable[[Sequence[np.ndarray], float], np.ndarray]] = None
    restart: int = 50
    tol: float = 1e-9
    seed: Optional[int] = None
    source_static: bool = False     # f independent of t (seeded fields)
    source_interior_only: bool = False  # f vanishes on the boundary of the closed grid
    notes: str = ""

    @property
    def tau(self) -> float:
        return self.T / self.M

    @property
    def N(self) -> int:
        return int(np.prod(self.n))

    def h(self, i: int) -> float:
        return 1.0 / (self.n[i] + 1)

    def x_interior(self, i: int) -> np.ndarray:
        """x_{i,j} = j h_i, j = 1..n_i."""
        return np.arange(1, self.n[i] + 1, dtype=np.float64) * self.h(i)

    def x_closed(self, i: int) -> np.ndarray:
        """x_{i,j} = j h_i, j = 0..n_i+1 (closed grid)."""
        return np.arange(0, self.n[i] + 2, dtype=np.float64) * self.h(i)

    def t_half(self, m: int) -> float:
        """t_{m+1/2}."""
        return (m + 0.5) * self.tau

    # --- grids as broadcastable coordinate arrays (array axis i == x_{i+1})
    def mesh(self, closed: bool = False):
        xs = []
        for i in range(self.d):
            x = self.x_closed(i) if closed else self.x_interior(i)
            shape = [1] * self.d
            shape[i] = x.size
            xs.append(x.reshape(shape))
        return xs

    # --- coefficient e on the grid
    def e_grid(self, t: float, closed: bool = False) -> np.ndarray:
        xs = self.mesh(closed)
        c = self.coeff
        prod = np.ones([x.size for x in xs]) if self.d > 1 else np.ones(xs[0].size)
        for i in range(self.d):
            if c.g[i] is not None:
                prod = prod * c.g[i](xs[i])
        out = c.a(t) + c.b(t) * prod
        for i in range(self.d):
            if c.k[i] is not None:
                out = out + c.k[i](xs[i])
        return np.asarray(out, dtype=np.float64)

    def e_tables(self):
        """Separable tables for the GPU ABI: a_half[M], b_half[M], g_i[n_i], k_i[n_i]."""
        c = self.coeff
        a_half = np.array([c.a(self.t_half(m)) for m in range(self.M)], dtype=np.float64)
        b_half = np.array([c.b(self.t_half(m)) for m in range(self.M)], dtype=np.float64)
        gs, ks = [], []
        for i in range(self.d):
            x = self.x_interior(i)
            gs.append(None if c.g[i] is None else np.ascontiguousarray(c.g[i](x), dtype=np.float64))
            ks.append(None if c.k[i] is None else np.ascontiguousarray(c.k[i](x), dtype=np.float64))
        return a_half, b_half, gs, ks

    def f_closed(self, t: float) -> np.ndarray:
        """source f(x, t) on the closed grid, array shape (n_i + 2)_i."""
        return np.asarray(self.source(self.mesh(closed=True), t), dtype=np.float64)

    def psi_interior(self) -> np.ndarray:
        return np.asarray(self.psi(self.mesh(closed=False)), dtype=np.float64) * np.ones(self.n)


def _interior_embed(field_int: np.ndarray) -> np.ndarray:
    """embed an interior array into the closed grid with zero boundary."""
    d = field_int.ndim
    out = np.zeros([s + 2 for s in field_int.shape])
    out[tuple(slice(1, -1) for _ in range(d))] = field_int
    return out


# ----------------------------------------------------------------------------
# BASELINE.json configs C1..C5 (SURVEY 8(d) with readings Q5-Q8)
# ----------------------------------------------------------------------------
def config_c1(n: int = 255, M: int = 64) -> Problem:
    """configs[0]: 1D, alpha=1.5, kappa=1, e=1+0.5 sin(pi x) e^{-t}, u=e^{-t}x^2(1-x)^2."""
    alpha, kappa = 1.5, 1.0

    def src(xs, t):
        x = xs[0]
        e = 1.0 + 0.5 * np.sin(np.pi * x) * math.exp(-t)
        u = math.exp(-t) * poly_eval(P2, x)
        return -e * u - kappa * math.exp(-t) * riesz_poly(P2, alpha, x)

    return Problem(
        name="C1", d=1, n=(n,), alpha=(alpha,), kappa=(kappa,), M=M, T=1.0,
        coeff=SeparableCoeff(a=lambda t: 1.0, b=lambda t: 0.5 * math.exp(-t),
                             g=[lambda x: np.sin(np.pi * x)], k=[None]),
        source=src, psi=lambda xs: poly_eval(P2, xs[0]),
        exact=lambda xs, t: math.exp(-t) * poly_eval(P2, xs[0]),
        restart=50, tol=1e-10,
        notes="manufactured u = exp(-t) x^2 (1-x)^2 with closed-form Riesz source")


def config_c2(n: int = 255, M: int = 32) -> Problem:
    """configs[1]: 2D, alpha=(1.3,1.7), kappa=(1,2), e=2+x y sin t, f = r(seed_2) + f_man (Q6, Q7)."""
    alpha = (1.3, 1.7)
    kappa = (1.0, 2.0)
    seed = SEED_BASE + 2
    r_int = seeded_field(seed, (n, n))
    r_closed = _interior_embed(r_int)

    def src(xs, t):
        x, y = xs
        e = 2.0 + x * y * math.sin(t)
        px, py = poly_eval(P2, x), poly_eval(P2, y)
        u = math.exp(-t) * px * py
        lap = kappa[0] * riesz_poly(P2, alpha[0], x) * py + kappa[1] * px * riesz_poly(P2, alpha[1], y)
        return r_closed - e * u - math.exp(-t) * lap

    return Problem(
        name="C2", d=2, n=(n, n), alpha=alpha, kappa=kappa, M=M, T=1.0,
        coeff=SeparableCoeff(a=lambda t: 2.0, b=lambda t: math.sin(t),
                             g=[lambda x: x, lambda y: y], k=[None, None]),
        source=src, psi=lambda xs: poly_eval(P2, xs[0]) * poly_eval(P2, xs[1]),
        restart=50, tol=1e-10, seed=seed,
        notes="seeded uniform field + manufactured term of u=exp(-t)p(x)p(y), p=x^2(1-x)^2")


def _seeded_static_source(seed, n):
    r_closed = _interior_embed(seeded_field(seed, n) if len(n) > 1 else seeded_field(seed, n))
    return lambda xs, t: r_closed


def config_c3(n: int = 2047, M: int = 16) -> Problem:
    """configs[2]: 2D, alpha=(1.2,1.9), e=1+0.9 exp(-10((x-1/2)^2+(y-1/2)^2))(1+t)."""
    seed = SEED_BASE + 3
    gfun = lambda x: np.exp(-10.0 * (x - 0.5) ** 2)
    return Problem(
        name="C3", d=2, n=(n, n), alpha=(1.2, 1.9), kappa=(1.0, 1.0), M=M, T=1.0,
        coeff=SeparableCoeff(a=lambda t: 1.0, b=lambda t: 0.9 * (1.0 + t), g=[gfun, gfun], k=[None, None]),
        source=_seeded_static_source(seed, (n, n)), psi=lambda xs: 0.0,
        restart=50, tol=1e-9, seed=seed, source_static=True, source_interior_only=True)


def config_c4(n: int = 255, M: int = 8) -> Problem:
    """configs[3]: 3D 255^3, alpha=1.5, e=1+0.5 prod sin(pi x_i) cos t, GMRES(30) tol 1e-9."""
    seed = SEED_BASE + 4
    s = lambda x: np.sin(np.pi * x)
    return Problem(
        name="C4", d=3, n=(n, n, n), alpha=(1.5, 1.5, 1.5), kappa=(1.0, 1.0, 1.0), M=M, T=1.0,
        coeff=SeparableCoeff(a=lambda t: 1.0, b=lambda t: 0.5 * math.cos(t), g=[s, s, s], k=[None] * 3),
        source=_seeded_static_source(seed, (n, n, n)), psi=lambda xs: 0.0,
        restart=30, tol=1e-9, seed=seed, source_static=True, source_interior_only=True)


def config_c5(n: int = 511, M: int = 4, nn: Optional[Sequence[int]] = None) -> Problem:
    """configs[4]: 3D 511^3, alpha=(1.1,1.5,1.9), kappa=(1,.5,2), e=1.5+0.5 tanh(5(x-1/2)) e^{-t}, GMRES(20) tol 1e-8."""
    seed = SEED_BASE + 5
    dims = tuple(nn) if nn is not None else (n, n, n)
    return Problem(
        name="C5", d=3, n=dims, alpha=(1.1, 1.5, 1.9), kappa=(1.0, 0.5, 2.0), M=M, T=1.0,
        coeff=SeparableCoeff(a=lambda t: 1.5, b=lambda t: 0.5 * math.exp(-t),
                             g=[lambda x: np.tanh(5.0 * (x - 0.5)), None, None], k=[None] * 3),
        source=_seeded_static_source(seed, dims), psi=lambda xs: 0.0,
        restart=20, tol=1e-8, seed=seed, source_static=True, source_interior_only=True)


CONFIGS = {"C1": config_c1, "C2": config_c2, "C3": config_c3, "C4": config_c4, "C5": config_c5}


# ----------------------------------------------------------------------------
# The paper's Examples 1-3 with the separable
# manufactured solution u = C e^{-t} prod p4(x_i) (SPEC's reading for Ex. 2/3).
# ----------------------------------------------------------------------------
def example(d: int, n: int, M: int, alpha: Sequence[float], tol: float = 1e-9,
            restart: int = 50) -> Problem:
    C = {1: 100.0, 2: 1e4, 3: 1e8}[d]
    kappa = {1: (100.0,), 2: (100.0, 100.0), 3: (100.0, 85.0, 103.0)}[d]
    div = 50.0 if d == 1 else 100.0
    alpha = tuple(float(a) for a in alpha)

    def u_exact(xs, t):
        out = C * math.exp(-t)
        for x in xs:
            out = out * poly_eval(P4, x)
        return out

    def src(xs, t):
        e = math.exp(-t) / div
        for x in xs:
            e = e + x * x / div
        u = u_exact(xs, t)
        lap = 0.0
        for i in range(d):
            term = C * math.exp(-t) * kappa[i] * riesz_poly(P4, alpha[i], xs[i])
            for l in range(d):
                if l != i:
                    term = term * poly_eval(P4, xs[l])
            lap = lap + term
        return -e * u - lap

    return Problem(
        name=f"Example{d}", d=d, n=(n,) * d, alpha=alpha, kappa=kappa, M=M, T=1.0,
        coeff=SeparableCoeff(a=lambda t: math.exp(-t) / div, b=lambda t: 0.0,
                             g=[None] * d, k=[(lambda x: x * x / div)] * d),
        source=src, psi=lambda xs: u_exact(xs, 0.0), exact=u_exact,
        restart=restart, tol=tol)
