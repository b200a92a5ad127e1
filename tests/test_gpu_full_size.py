"""GPU parity at the literal BASELINE.json sizes, and the ABI modes not covered elsewhere.

* Operators at full size: A^{(0)}, K = P_alpha^{-1} A~ (== P_hat^{-1} A) and P_hat^{-1}
  on the 255^2 (C2), 2047^2 (C3), 255^3 (C4) and 511^3 (C5) grids, one application each, against the
  oracle's per-line operators (Eq.(tls), Eq.(equi), Eq.(Pa)) at 1e-12.
* CN marches at full size: C2 all 32 steps, C3 / C4 the first two steps, C5 step 0 --
  iterations +-1, solution 1e-9 at matched counts (replay).  The system is Eq.(tls)
   solved through Eq.(one-sided).
* The generic (non on-chip) GMRES path with forced restarts in 2D and 3D, replay across restarts,
  RSFDE_COEF_GRID and RSFDE_X0_ZERO through the C ABI, each against the oracle (stopping rule and
  restart: P:513).

Inputs are the seeded synthetic fields of paper_2404_10221_b200.inputs.  The
oracle is plain numpy (FP64 BLAS per line); the 511^3 solve costs a few minutes of host time.
"""
import numpy as np
import pytest

from oracle import scheme
from oracle.gmres import gmres as oracle_gmres
from oracle.lines import LineSystem
from paper_2404_10221_b200 import inputs as I

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def _host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def relerr(got, ref):
    return float(np.max(np.abs(got - ref)) / max(np.max(np.abs(ref)), 1e-300))


def _solver(prob):
    from paper_2404_10221_b200.solver import RsfdeSolver
    return RsfdeSolver.from_problem(prob)


FULL = {"C2": I.config_c2, "C3": I.config_c3, "C4": I.config_c4, "C5": I.config_c5}


# ----------------------------------------------------------------------------- operators
@pytest.mark.parametrize("name", ["C2", "C3", "C4", "C5"])
def test_full_size_operator_parity(name):
    from paper_2404_10221_b200 import _lib as L
    p = FULL[name]()
    S = _solver(p)
    Ls = LineSystem(p.d, p.n, p.alpha, p.kappa, p.tau)
    ebar = scheme.e_bar(p)[0]
    assert abs(S.ebar()[0] - ebar) <= 4e-16 * ebar
    x = I.seeded_vector(2024, p.n)
    xd = _dev(x)
    e = p.e_grid(p.t_half(0))
    got = _host(S.matvec(L.OP_A, xd, m=0))
    assert relerr(got, Ls.A(e, x)) < 1e-12, ("A", relerr(got, Ls.A(e, x)))
    got = _host(S.precond(L.PHAT_INV, xd))
    ref = Ls.P_hat_inv(ebar, x)
    assert relerr(got, ref) < 1e-12, ("P_hat^-1", relerr(got, ref))
    del ref
    got = _host(S.matvec(L.OP_K, xd, m=0))
    ref = Ls.P_alpha_inv(ebar, Ls.A_tilde(e, x))          # the paper's literal one-sided operator
    assert relerr(got, ref) < 1e-12, ("K", relerr(got, ref))
    S.close()


# ----------------------------------------------------------------------------- marches
def _march_gpu(prob, steps, cfg_kw=None):
    S = _solver(prob)
    kw = {"restart": prob.restart, "tol": prob.tol}
    kw.update(cfg_kw or {})
    cfg = S.cfg(**kw)
    u = _dev(prob.psi_interior())
    if prob.source_static:
        F = S.compact_source(_dev(prob.f_closed(prob.t_half(0))))
        rep = S.solve_steps(u, F=F, F_static=True, m_begin=0, m_count=steps, cfg=cfg)
    else:
        F = torch.stack([S.compact_source(_dev(prob.f_closed(prob.t_half(m)))) for m in range(steps)])
        rep = S.solve_steps(u, F=F, F_static=False, m_begin=0, m_count=steps, cfg=cfg)
    out = _host(u)
    S.close()
    return out, rep


@pytest.mark.parametrize("name,steps", [("C2", 32), ("C3", 2), ("C4", 2), ("C5", 1)])
def test_full_size_march_parity(name, steps):
    prob = FULL[name]()
    u, rep = _march_gpu(prob, steps)
    Fst = scheme.source_F(prob, 0) if prob.source_static else None
    uo, ro, _ = scheme.solve(prob, steps=steps, F_static=Fst)
    assert all(rep["converged"]) and all(ro.converged)
    diffs = [abs(a - b) for a, b in zip(rep["iters"], ro.iters)]
    assert max(diffs) <= 1, (rep["iters"], ro.iters)
    if max(diffs) > 0:
        uo, ro, _ = scheme.solve(prob, steps=steps, F_static=Fst, fixed_iters=rep["iters"])
    assert relerr(u, uo) < 1e-9, relerr(u, uo)


# ----------------------------------------------------------------------------- generic path modes
def _small(d):
    if d == 2:
        p = I.config_c5(M=4, nn=(3, 3, 3))
        p.d, p.n = 2, (31, 63)
        p.alpha, p.kappa = (1.1, 1.5), (1.0, 0.5)
        p.coeff = I.SeparableCoeff(a=lambda t: 1.5, b=lambda t: 0.5 * np.exp(-t),
                                   g=[lambda x: np.tanh(5 * (x - 0.5)), None], k=[None, None])
        p.source = I._seeded_static_source(p.seed, p.n)
        return p
    return I.config_c5(M=4, nn=(15, 7, 31))


@pytest.mark.parametrize("d", [2, 3])
def test_generic_path_restart_parity(d):
    # restart = 3 forces several GMRES cycles per step on the generic (multi-kernel) path: explicit
    # residual, x <- x0 + V y, beta0 of the first cycle kept
    prob = _small(d)
    u, rep = _march_gpu(prob, prob.M, {"restart": 3})
    Fst = scheme.source_F(prob, 0)
    uo, ro, _ = scheme.solve(prob, F_static=Fst, restart=3)
    assert max(ro.iters) > 3                      # restarts really happened
    assert all(rep["converged"]) and max(abs(a - b) for a, b in zip(rep["iters"], ro.iters)) <= 1, \
        (rep["iters"], ro.iters)
    if rep["iters"] != ro.iters:
        uo, ro, _ = scheme.solve(prob, F_static=Fst, restart=3, fixed_iters=rep["iters"])
    assert relerr(u, uo) < 1e-9


def test_replay_across_restarts_gmres_step():
    # fixed_iters > restart: exactly fixed_iters Arnoldi steps over several cycles
    prob = _small(3)
    S = _solver(prob)
    Ls = LineSystem(prob.d, prob.n, prob.alpha, prob.kappa, prob.tau)
    ebar = scheme.e_bar(prob)[0]
    m = 1
    e = prob.e_grid(prob.t_half(m))
    b = I.seeded_vector(31, prob.n)
    x0 = 0.1 * I.seeded_vector(32, prob.n)
    K = lambda v: Ls.P_alpha_inv(ebar, Ls.A_tilde(e, v))
    c = Ls.P_alpha_inv(ebar, Ls.H_alpha_inv(b))
    for fixed in (5, 8):
        ref = oracle_gmres(K, c, x0, 3, 0.0, 100, fixed_iters=fixed)
        assert ref.iters == fixed
        xd = _dev(x0)
        its, rr, conv = S.gmres_step(m, _dev(b), xd, S.cfg(restart=3, tol=0.0, fixed_iters=fixed))
        assert its == fixed and conv
        assert relerr(_host(xd), ref.x) < 1e-9
    S.close()


def test_coef_grid_march_parity():
    # RSFDE_COEF_GRID: e(x, t_{m+1/2}) as a dense device field (M*N values), evaluated by the pass
    # kernels from HBM instead of the separable tables; the oracle uses the same e grid
    from paper_2404_10221_b200.solver import RsfdeSolver
    prob = _small(3)
    grid = _dev(np.stack([prob.e_grid(prob.t_half(m)) for m in range(prob.M)]))
    S = RsfdeSolver.from_problem_grid(prob, grid)
    Sref = _solver(prob)
    assert abs(S.ebar()[0] - Sref.ebar()[0]) <= 4e-16 * Sref.ebar()[0]
    cfg = S.cfg(restart=prob.restart, tol=prob.tol)
    F = S.compact_source(_dev(prob.f_closed(prob.t_half(0))))
    u = _dev(prob.psi_interior())
    rep = S.solve_steps(u, F=F, F_static=True, cfg=cfg)
    from paper_2404_10221_b200 import _lib as L
    x = I.seeded_vector(5, prob.n)
    e3 = prob.e_grid(prob.t_half(3))
    Ls = LineSystem(prob.d, prob.n, prob.alpha, prob.kappa, prob.tau)
    assert relerr(_host(S.matvec(L.OP_A, _dev(x), m=3)), Ls.A(e3, x)) < 1e-12
    Fst = scheme.source_F(prob, 0)
    uo, ro, _ = scheme.solve(prob, F_static=Fst)
    assert all(rep["converged"]) and max(abs(a - b) for a, b in zip(rep["iters"], ro.iters)) <= 1
    if rep["iters"] != ro.iters:
        uo, ro, _ = scheme.solve(prob, F_static=Fst, fixed_iters=rep["iters"])
    assert relerr(_host(u), uo) < 1e-9
    # time-constant grid (grid_static): e frozen at t_{1/2}
    S2 = RsfdeSolver.from_problem_grid(prob, _dev(prob.e_grid(prob.t_half(0))), grid_static=True)
    assert relerr(_host(S2.matvec(L.OP_A, _dev(x), m=3)), Ls.A(prob.e_grid(prob.t_half(0)), x)) < 1e-12
    for s in (S, S2, Sref):
        s.close()


def test_x0_zero_march_parity():
    # RSFDE_X0_ZERO: every step's GMRES starts from x_0 = 0 instead of u^{(m)}
    from paper_2404_10221_b200 import _lib as L
    prob = _small(3)
    prob.M = 3
    u, rep = _march_gpu(prob, prob.M, {"x0_policy": L.X0_ZERO})
    Ls = LineSystem(prob.d, prob.n, prob.alpha, prob.kappa, prob.tau)
    ebar = scheme.e_bar(prob)[0]
    F = scheme.source_F(prob, 0)
    uo = prob.psi_interior()
    its = []
    for m in range(prob.M):
        e = prob.e_grid(prob.t_half(m))
        c = Ls.P_alpha_inv(ebar, Ls.H_alpha_inv(Ls.rhs(e, uo, F)))
        K = lambda v, e=e: Ls.P_alpha_inv(ebar, Ls.A_tilde(e, v))
        fx = None
        ref = oracle_gmres(K, c, np.zeros(prob.n), prob.restart, prob.tol, 10 * prob.restart)
        assert abs(ref.iters - rep["iters"][m]) <= 1, (m, ref.iters, rep["iters"][m])
        if ref.iters != rep["iters"][m]:
            fx = rep["iters"][m]
            ref = oracle_gmres(K, c, np.zeros(prob.n), prob.restart, prob.tol, 10 * prob.restart, fixed_iters=fx)
        its.append(ref.iters)
        uo = ref.x
    assert relerr(u, uo) < 1e-9
    # the zero start needs more iterations than the warm start x_0 = u^{(m)}
    u2, rep2 = _march_gpu(prob, prob.M)
    assert sum(rep["iters"]) >= sum(rep2["iters"])


def test_x0_zero_gmres_step():
    from paper_2404_10221_b200 import _lib as L
    prob = _small(2)
    S = _solver(prob)
    Ls = LineSystem(prob.d, prob.n, prob.alpha, prob.kappa, prob.tau)
    ebar = scheme.e_bar(prob)[0]
    e = prob.e_grid(prob.t_half(2))
    b = I.seeded_vector(41, prob.n)
    K = lambda v: Ls.P_alpha_inv(ebar, Ls.A_tilde(e, v))
    c = Ls.P_alpha_inv(ebar, Ls.H_alpha_inv(b))
    ref = oracle_gmres(K, c, np.zeros(prob.n), 20, 1e-11, 200)
    xd = _dev(I.seeded_vector(42, prob.n))             # ignored: X0_ZERO
    its, rr, conv = S.gmres_step(2, _dev(b), xd, S.cfg(restart=20, tol=1e-11, x0_policy=L.X0_ZERO))
    assert conv and abs(its - ref.iters) <= 1
    if its != ref.iters:
        ref = oracle_gmres(K, c, np.zeros(prob.n), 20, 1e-11, 200, fixed_iters=its)
    assert relerr(_host(xd), ref.x) < 1e-9
    S.close()


# ----------------------------------------------------------------------------- T9 mesh independence
def test_mesh_independence_c5_gpu():
    # Theorem 3.7: iteration counts do not grow with n -- C5 at n = 127, 255, 511
    # (first two CN steps each); mean iterations within +-1
    means = []
    for n in (127, 255, 511):
        p = I.config_c5(n=n)
        _, rep = _march_gpu(p, 2)
        assert all(rep["converged"])
        means.append(float(np.mean(rep["iters"])))
    assert max(means) - min(means) <= 1.0, means


# ----------------------------------------------------------------------------- T1 at full n vs 30 digits
@pytest.mark.parametrize("name", ["C3", "C5"])
def test_library_tau_eigenvalues_vs_30_digits(name):
    # the library's host setup evaluates s_k and q_i in long double; pinned here against
    # an mpmath 30-digit evaluation through the Gamma closed form of s_k (tests/test_oracle_fcd.py)
    from test_oracle_fcd import mp_tau_eigenvalues
    p = FULL[name]()
    S = _solver(p)
    for i in range(p.d):
        ref = np.array(mp_tau_eigenvalues(p.alpha[i], p.n[i], range(1, 9)))
        q = S.table(i, 1)[:8]
        assert np.max(np.abs(q - ref) / np.abs(ref)) < 1e-13, (i, np.abs(q - ref) / np.abs(ref))
    S.close()
