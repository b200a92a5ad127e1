"""GPU parity: the CUDA path through the C ABI vs the CPU oracle on the same seeded inputs.

Bars (BASELINE.json north_star): operators and preconditioners 1e-12 relative (inf-norm),
final solutions 1e-9 relative, GMRES iteration counts within +-1.  Inputs are seeded
uniform[-1,1] (smooth inputs cancel and are not a fair parity input, VN-9).
"""
import numpy as np
import pytest

from oracle import fcd, scheme
from oracle.gmres import gmres as oracle_gmres
from oracle.lines import LineSystem
from paper_2404_10221_b200 import inputs as I

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _solver(prob):
    from paper_2404_10221_b200.solver import RsfdeSolver
    return RsfdeSolver.from_problem(prob)


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def _host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def relerr(got, ref):
    return float(np.max(np.abs(got - ref)) / max(np.max(np.abs(ref)), 1e-300))


def _prob(kind, shape, M=4):
    d = len(shape)
    if kind == "c5":
        p = I.config_c5(M=M, nn=shape if d == 3 else (3, 3, 3))
        if d != 3:
            p.d, p.n = d, tuple(shape)
            p.alpha, p.kappa = (1.1, 1.5, 1.9)[:d], (1.0, 0.5, 2.0)[:d]
            p.coeff = I.SeparableCoeff(a=lambda t: 1.5, b=lambda t: 0.5 * np.exp(-t),
                                       g=[lambda x: np.tanh(5 * (x - 0.5))] + [None] * (d - 1), k=[None] * d)
        return p
    if kind == "c1":
        return I.config_c1(n=shape[0], M=M)
    if kind == "ex":
        return I.example(d, shape[0], M, (1.3, 1.5, 1.7)[:d])
    raise ValueError(kind)


SHAPES = [("c1", (255,)), ("c1", (7,)), ("c1", (1,)), ("c5", (31, 63)), ("c5", (255, 15)),
          ("c5", (15, 7, 31)), ("c5", (63, 63, 63)), ("ex", (3, 3, 3)), ("c5", (1, 3, 1)),
          # long pencils: the three-stage FFT (L = 2048, 4096), strided and contiguous axes
          ("c5", (2047, 7)), ("c5", (7, 2047)), ("c5", (3, 1023, 3)), ("c1", (2047,)),
          # n = 511 pencils: the warp-specialised tile pipeline (strided tiles of 16 pencils, a
          # ragged last tile, the pad column, and contiguous 16-row tiles)
          ("c5", (511, 15, 31)), ("c5", (15, 511, 7)), ("c5", (7, 15, 511)), ("c5", (511, 511)), ("c1", (511,)),
          # n = 255 pencils: the tile pipeline with two 16-thread FFT groups per warp (L = 512, C4)
          ("c5", (255, 15, 31)), ("c5", (15, 255, 31)), ("c5", (7, 15, 255)), ("c5", (255, 255))]


@pytest.fixture(scope="module")
def cache():
    return {}


def _setup(cache, kind, shape):
    key = (kind, shape)
    if key not in cache:
        p = _prob(kind, shape)
        cache[key] = (p, _solver(p), LineSystem(p.d, p.n, p.alpha, p.kappa, p.tau), scheme.e_bar(p)[0])
    return cache[key]


# ----------------------------------------------------------------------- T1 setup tables
@pytest.mark.parametrize("kind,shape", SHAPES)
def test_setup_tables(cache, kind, shape):
    p, S, Ls, ebar = _setup(cache, kind, shape)
    for i in range(p.d):
        s = fcd.fcd_coefficients(p.alpha[i], p.n[i]).astype(float)
        assert relerr(S.table(i, 0), s) < 1e-14
        assert relerr(S.table(i, 1), Ls.q[i]) < 1e-14
        assert relerr(S.table(i, 2), Ls.lamH[i]) < 1e-14
        assert abs(S.table(i, 4)[0] - Ls.eta[i]) <= 1e-14 * Ls.eta[i]
    eb, eh, ec = S.ebar()
    ref = scheme.e_bar(p)
    assert abs(eb - ref[0]) <= 4e-16 * ref[0] and abs(eh - ref[1]) <= 4e-16 * ref[1]


# ----------------------------------------------------------------------- T3/T4 operators
@pytest.mark.parametrize("kind,shape", SHAPES)
@pytest.mark.parametrize("m", [0, 3])
def test_matvec_parity(cache, kind, shape, m):
    from paper_2404_10221_b200 import _lib as L
    p, S, Ls, ebar = _setup(cache, kind, shape)
    x = I.seeded_vector(1000 + m, p.n)
    e = p.e_grid(p.t_half(m))
    xd = _dev(x)
    cases = {
        L.OP_A: Ls.A(e, x),
        L.OP_S_ALPHA: Ls.S_alpha(x),
        L.OP_H_ALPHA: Ls.H_alpha(x),
        L.OP_H_ALPHA_INV: Ls.H_alpha_inv(x),
        L.OP_ATILDE: Ls.A_tilde(e, x),
        L.OP_K: Ls.P_alpha_inv(ebar, Ls.A_tilde(e, x)),
    }
    for op, ref in cases.items():
        got = _host(S.matvec(op, xd, m=m))
        assert relerr(got, ref) < 1e-12, (op, relerr(got, ref))


@pytest.mark.parametrize("kind,shape", SHAPES)
def test_precond_parity(cache, kind, shape):
    from paper_2404_10221_b200 import _lib as L
    p, S, Ls, ebar = _setup(cache, kind, shape)
    x = I.seeded_vector(77, p.n)
    xd = _dev(x)
    for kindp, ref in ((L.PHAT_INV, Ls.P_hat_inv(ebar, x)), (L.PALPHA_INV, Ls.P_alpha_inv(ebar, x)),
                       (L.PALPHA_INV_SQRT, Ls.P_alpha_inv_sqrt(ebar, x))):
        got = _host(S.precond(kindp, xd))
        assert relerr(got, ref) < 1e-12, (kindp, relerr(got, ref))


@pytest.mark.parametrize("kind,shape", SHAPES)
def test_compact_source_parity(cache, kind, shape):
    p, S, Ls, ebar = _setup(cache, kind, shape)
    f = np.random.default_rng(3).uniform(-1, 1, [v + 2 for v in p.n])
    got = _host(S.compact_source(_dev(f)))
    assert relerr(got, scheme.compact_source(p.alpha, f)) < 1e-14


# ----------------------------------------------------------------------- T5 one GMRES solve
@pytest.mark.parametrize("kind,shape", [("c1", (255,)), ("c5", (31, 63)), ("c5", (15, 7, 31))])
def test_gmres_step_parity(cache, kind, shape):
    p, S, Ls, ebar = _setup(cache, kind, shape)
    m = 1
    e = p.e_grid(p.t_half(m))
    b = I.seeded_vector(5, p.n)
    x0 = 0.1 * I.seeded_vector(6, p.n)
    # oracle: one-sided system P^{-1} A~ x = P^{-1} H^{-1} b (Eq.(one-sided))
    K = lambda v: Ls.P_alpha_inv(ebar, Ls.A_tilde(e, v))
    c = Ls.P_alpha_inv(ebar, Ls.H_alpha_inv(b))
    ref = oracle_gmres(K, c, x0, 20, 1e-11, 200)
    xd = _dev(x0)
    its, rr, conv = S.gmres_step(m, _dev(b), xd, S.cfg(restart=20, tol=1e-11))
    assert conv and abs(its - ref.iters) <= 1
    if its != ref.iters:   # replay at matched counts
        ref = oracle_gmres(K, c, x0, 20, 1e-11, 200, fixed_iters=its)
    assert relerr(_host(xd), ref.x) < 1e-9


# ----------------------------------------------------------------------- T6 time march
def _march(prob, restart=None, tol=None, form=0, host=False, solver_out=None):
    from paper_2404_10221_b200 import _lib as L
    S = _solver(prob)
    if solver_out is not None:
        solver_out.append(S)
    restart = restart or prob.restart
    tol = tol or prob.tol
    u0 = prob.psi_interior()
    # F^{(m+1/2)} is built on the GPU from the raw samples of f on the closed grid (inputs
    # module), so no oracle-computed value enters the CUDA path
    steps = [0] if prob.source_static else range(prob.M)
    F = torch.stack([S.compact_source(_dev(prob.f_closed(prob.t_half(m)))) for m in steps])
    Fs = bool(prob.source_static)
    if Fs:
        F = F[0].contiguous()
    if host:
        u = np.ascontiguousarray(u0)
        rep = S.solve_steps(u, F=np.ascontiguousarray(_host(F)), F_static=Fs,
                            cfg=S.cfg(restart=restart, tol=tol, form=form))
        return u, rep
    u = _dev(u0)
    rep = S.solve_steps(u, F=F, F_static=Fs, cfg=S.cfg(restart=restart, tol=tol, form=form))
    return _host(u), rep


@pytest.mark.parametrize("name", ["c1", "c2s", "c3s", "c4s", "c5s", "ex2"])
def test_solve_steps_parity(name):
    prob = {"c1": lambda: I.config_c1(n=255, M=64),
            "c3s": lambda: _c3_small(),
            "c2s": lambda: I.config_c2(n=63, M=8),
            "c4s": lambda: I.config_c4(n=31, M=4),
            "c5s": lambda: I.config_c5(M=4, nn=(31, 15, 63)),
            "ex2": lambda: I.example(2, 31, 16, (1.5, 1.7))}[name]()
    u, rep = _march(prob)
    Fst = scheme.source_F(prob, 0) if prob.source_static else None
    uo, ro, _ = scheme.solve(prob, F_static=Fst)
    assert all(rep["converged"]) and all(ro.converged)
    diffs = [abs(a - b) for a, b in zip(rep["iters"], ro.iters)]
    assert max(diffs) <= 1, (rep["iters"], ro.iters)
    if max(diffs) > 0:
        uo, ro, _ = scheme.solve(prob, F_static=Fst, fixed_iters=rep["iters"])
    assert relerr(u, uo) < 1e-9, relerr(u, uo)


def _c3_small():
    # C3's coefficients and orders on a 2047 x 63 grid (long contiguous-axis FFT), 3 steps
    p = I.config_c3(n=63, M=3)
    p.n = (63, 2047)
    p.source = lambda xs, t: I._interior_embed(I.seeded_field(p.seed, p.n))
    return p


def test_a_form_equals_atilde_form():
    from paper_2404_10221_b200 import _lib as L
    prob = I.config_c5(M=3, nn=(15, 31, 7))
    u1, r1 = _march(prob)
    u2, r2 = _march(prob, form=L.FORM_ATILDE)
    assert r1["iters"] == r2["iters"]
    assert relerr(u1, u2) < 1e-12


def test_host_pointer_path_equals_device_path():
    prob = I.config_c1(n=127, M=8)
    u1, r1 = _march(prob)
    u2, r2 = _march(prob, host=True)
    assert r1["iters"] == r2["iters"] and np.array_equal(u1, u2)


@pytest.mark.parametrize("shape", [(63,), (15, 31), (7, 15, 7)])
def test_exact_preconditioner_alpha_two(shape):
    # alpha = 2, constant e: P_hat = A exactly -> one iteration per step
    d = len(shape)
    prob = I.config_c5(M=3, nn=(3, 3, 3))
    prob.d, prob.n = d, shape
    prob.alpha, prob.kappa = (2.0,) * d, (1.0, 0.5, 2.0)[:d]
    prob.coeff = I.SeparableCoeff(a=lambda t: 1.5, b=lambda t: 0.0, g=[None] * d, k=[None] * d)
    prob.source = lambda xs, t: np.ones([x.size for x in xs])
    prob.source_static = False
    u, rep = _march(prob, restart=10, tol=1e-12)
    assert rep["iters"] == [1, 1, 1]


def test_zero_data_zero_iterations():
    # f = psi = 0 -> u stays exactly 0 with no Arnoldi step
    prob = I.config_c5(M=3, nn=(7, 7, 15))
    prob.source = lambda xs, t: np.zeros([x.size for x in xs])
    u, rep = _march(prob)
    assert rep["iters"] == [0, 0, 0] and np.all(u == 0)


def test_invalid_arguments_fail_loudly():
    from paper_2404_10221_b200 import _lib as L
    from paper_2404_10221_b200.solver import RsfdeSolver
    p = I.config_c1(n=100, M=4)   # n+1 = 101 is not a power of two
    with pytest.raises(L.RsfdeError) as ei:
        RsfdeSolver.from_problem(p)
    assert ei.value.status == L.E_DIM
    p = I.config_c1(n=31, M=4)
    p.alpha = (0.9,)
    with pytest.raises(L.RsfdeError) as ei:
        RsfdeSolver.from_problem(p)
    assert ei.value.status == L.E_DOMAIN


# ----------------------------------------------------------------------- two-sided system (NEXT-1)
@pytest.mark.parametrize("name", ["c1", "c5s", "ex2"])
def test_two_sided_march_parity(name):
    from paper_2404_10221_b200 import _lib as L
    prob = {"c1": lambda: I.config_c1(n=127, M=8),
            "c5s": lambda: I.config_c5(M=3, nn=(31, 15, 63)),
            "ex2": lambda: I.example(2, 31, 8, (1.5, 1.7))}[name]()
    u, rep = _march(prob, form=L.FORM_TWO_SIDED)
    Fst = scheme.source_F(prob, 0) if prob.source_static else None
    uo, ro, _ = scheme.solve(prob, F_static=Fst, sided=2)
    assert all(rep["converged"])
    assert max(abs(a - b) for a, b in zip(rep["iters"], ro.iters)) <= 1, (rep["iters"], ro.iters)
    if rep["iters"] != ro.iters:
        uo, ro, _ = scheme.solve(prob, F_static=Fst, sided=2, fixed_iters=rep["iters"])
    assert relerr(u, uo) < 1e-9
    # one- and two-sided solve the same linear systems
    u1, _ = _march(prob)
    assert relerr(u, u1) < 10 * prob.tol


def test_two_sided_gmres_step():
    from paper_2404_10221_b200 import _lib as L
    from paper_2404_10221_b200.solver import RsfdeSolver
    prob = I.config_c5(M=2, nn=(15, 7, 31))
    S = RsfdeSolver.from_problem(prob)
    Ls = LineSystem(prob.d, prob.n, prob.alpha, prob.kappa, prob.tau)
    ebar = scheme.e_bar(prob)[0]
    e = prob.e_grid(prob.t_half(1))
    b = I.seeded_vector(8, prob.n)
    x0 = 0.2 * I.seeded_vector(9, prob.n)
    K = lambda v: Ls.P_alpha_inv_sqrt(ebar, Ls.A_tilde(e, Ls.P_alpha_inv_sqrt(ebar, v)))
    c = Ls.P_alpha_inv_sqrt(ebar, Ls.H_alpha_inv(b))
    ref = oracle_gmres(K, c, Ls.P_alpha_sqrt(ebar, x0), 20, 1e-11, 200)
    xd = _dev(x0)
    its, rr, conv = S.gmres_step(1, _dev(b), xd, S.cfg(restart=20, tol=1e-11, form=L.FORM_TWO_SIDED))
    assert conv and abs(its - ref.iters) <= 1
    if its != ref.iters:
        ref = oracle_gmres(K, c, Ls.P_alpha_sqrt(ebar, x0), 20, 1e-11, 200, fixed_iters=its)
    assert relerr(_host(xd), Ls.P_alpha_inv_sqrt(ebar, ref.x)) < 1e-9


# ----------------------------------------------------------------------- batched marches (NEXT-4)
def test_batched_march_equals_separate_marches():
    # rsfde_solve_steps_batch: several independent systems (an alpha / N sweep as in Tables 1-3,
    # P:528-636) marched concurrently give exactly the results of separate rsfde_solve_steps calls
    from paper_2404_10221_b200 import solver as SV
    probs = [I.example(1, 31, 16, (1.3,)), I.example(1, 63, 16, (1.9,)), I.example(2, 15, 8, (1.5, 1.7)),
             I.config_c5(M=3, nn=(15, 7, 31))]
    sols = [_solver(p) for p in probs]
    Fs = []
    for S, p in zip(sols, probs):
        steps = [0] if p.source_static else range(p.M)
        F = torch.stack([S.compact_source(_dev(p.f_closed(p.t_half(m)))) for m in steps])
        Fs.append(F[0].contiguous() if p.source_static else F)
    fst = [bool(p.source_static) for p in probs]
    cfgs = [S.cfg(restart=p.restart, tol=p.tol) for S, p in zip(sols, probs)]
    u_sep = [_dev(p.psi_interior()) for p in probs]
    rep_sep = [S.solve_steps(u, F=F, F_static=f, cfg=c) for S, u, F, f, c in zip(sols, u_sep, Fs, fst, cfgs)]
    u_bat = [_dev(p.psi_interior()) for p in probs]
    rep_bat = SV.solve_steps_batch(sols, u_bat, Fs=Fs, F_static=fst, cfgs=cfgs)
    for a, b, ra, rb in zip(u_sep, u_bat, rep_sep, rep_bat):
        assert ra["iters"] == rb["iters"] and all(rb["converged"])
        assert torch.equal(a, b)                      # bit-identical: same kernels, deterministic sums
    for p, ub, rb in zip(probs, u_bat, rep_bat):      # and every system against the oracle
        _check_march_vs_oracle(p, _host(ub), rb)


def _check_march_vs_oracle(p, u, rep, restart=None):
    Fst = scheme.source_F(p, 0) if p.source_static else None
    uo, ro, _ = scheme.solve(p, F_static=Fst, restart=restart)
    assert all(rep["converged"]) and max(abs(a - b) for a, b in zip(rep["iters"], ro.iters)) <= 1, \
        (p.name, rep["iters"], ro.iters)
    if rep["iters"] != ro.iters:
        uo, ro, _ = scheme.solve(p, F_static=Fst, restart=restart, fixed_iters=rep["iters"])
    assert relerr(u, uo) < 1e-9, (p.name, relerr(u, uo))


def test_batched_onchip_kernel_sweep_vs_oracle(monkeypatch):
    # NEXT-4 as one launch: a Table-1-style alpha x N sweep of 1-D systems (Example 1, P:523-526,
    # alpha in {1.3, 1.5, 1.9}, N+1 in {16, 32, 64}) plus a C1-shaped system, one CTA per system;
    # every system is checked against the oracle and against its own separate march
    from paper_2404_10221_b200 import solver as SV
    probs = [I.example(1, n1 - 1, 32, (a,)) for a in (1.3, 1.5, 1.9) for n1 in (16, 32, 64)]
    probs.append(I.config_c1(n=255, M=16))
    sols = [_solver(p) for p in probs]
    Fs = [torch.stack([S.compact_source(_dev(p.f_closed(p.t_half(m)))) for m in range(p.M)])
          for S, p in zip(sols, probs)]
    cfgs = [S.cfg(restart=p.restart, tol=p.tol) for S, p in zip(sols, probs)]
    u_bat = [_dev(p.psi_interior()) for p in probs]
    n0 = [S.launch_count(reset=True) for S in sols]
    rep_bat = SV.solve_steps_batch(sols, u_bat, Fs=Fs, F_static=[False] * len(probs), cfgs=cfgs)
    # one batched launch accounted on the first context, nothing but pack/unpack on the others
    assert sols[0].launch_count() <= 2 * len(probs) + 1
    for p, ub, rb in zip(probs, u_bat, rep_bat):
        _check_march_vs_oracle(p, _host(ub), rb)
    # the same systems one by one (single-system on-chip kernel): identical results
    for S, p, F, c, ub, rb in zip(sols, probs, Fs, cfgs, u_bat, rep_bat):
        u1 = _dev(p.psi_interior())
        r1 = S.solve_steps(u1, F=F, F_static=False, cfg=c)
        assert r1["iters"] == rb["iters"] and torch.equal(u1, ub)
    # and the stream-per-system path agrees
    monkeypatch.setenv("RSFDE_NO_BATCH_KERNEL", "1")
    u_thr = [_dev(p.psi_interior()) for p in probs]
    rep_thr = SV.solve_steps_batch(sols, u_thr, Fs=Fs, F_static=[False] * len(probs), cfgs=cfgs)
    for a, b, ra, rb in zip(u_thr, u_bat, rep_thr, rep_bat):
        assert ra["iters"] == rb["iters"] and torch.equal(a, b)


def test_batched_march_rejects_duplicate_contexts():
    from paper_2404_10221_b200 import solver as SV
    p = I.example(1, 15, 4, (1.5,))
    S = _solver(p)
    with pytest.raises(Exception):
        SV.solve_steps_batch([S, S], [_dev(p.psi_interior()), _dev(p.psi_interior())])


# ----------------------------------------------------------------------- on-chip 1-D march
@pytest.mark.parametrize("restart", [50, 3])
def test_onchip_1d_march_matches_oracle_and_generic_path(restart, monkeypatch):
    # small 1-D problems march in one on-chip kernel (onchip_1d.cu); restart = 3 forces GMRES restarts
    prob = I.config_c1(n=127, M=12)
    u_on, rep_on = _march(prob, restart=restart)
    monkeypatch.setenv("RSFDE_NO_ONCHIP", "1")
    u_gen, rep_gen = _march(prob, restart=restart)
    monkeypatch.delenv("RSFDE_NO_ONCHIP")
    assert all(rep_on["converged"]) and all(rep_gen["converged"])
    assert max(abs(a - b) for a, b in zip(rep_on["iters"], rep_gen["iters"])) <= 1
    uo, ro, _ = scheme.solve(prob, restart=restart)
    assert max(abs(a - b) for a, b in zip(rep_on["iters"], ro.iters)) <= 1, (rep_on["iters"], ro.iters)
    if rep_on["iters"] != ro.iters:
        uo, ro, _ = scheme.solve(prob, restart=restart, fixed_iters=rep_on["iters"])
    assert relerr(u_on, uo) < 1e-9


@pytest.mark.parametrize("wide", ["1", "0"])
@pytest.mark.parametrize("kind,shape", [("c5", (511, 15, 31)), ("c5", (15, 511, 31)), ("c5", (511, 511)),
                                        ("c5", (31, 15, 511))])
def test_tile128_matvec_and_precond_parity(kind, shape, wide, monkeypatch, cache):
    # both tile widths of the L = 1024 pipeline on every axis kind: 8 pairs per CTA (the default: 128-byte
    # row pieces on strided axes, 16 rows on the contiguous axis) and 4 pairs per CTA (RSFDE_TILE128=0 /
    # RSFDE_TILE_CT8=0; still the fallback when the inner extent is not a multiple of 16)
    monkeypatch.setenv("RSFDE_TILE128", wide)
    monkeypatch.setenv("RSFDE_TILE_CT8", wide)
    test_matvec_parity(cache, kind, shape, 0)
    test_precond_parity(cache, kind, shape)


# ----------------------------------------------------------------------- Arnoldi variants
@pytest.mark.parametrize("name", ["c5s", "ex2", "c2s"])
def test_dcgs2_matches_cgs2_and_oracle(name, monkeypatch):
    # the default DCGS2 Arnoldi (delayed re-orthogonalisation, one dots + one update pass) and the
    # three-pass CGS2 (RSFDE_ORTHO=cgs2) are the same Krylov process: equal iteration counts and
    # solutions to rounding; the speculative one-ahead launches (RSFDE_NO_SPEC=1 disables them) do
    # not change a single bit
    prob = {"c5s": lambda: I.config_c5(M=4, nn=(31, 15, 63)),
            "ex2": lambda: I.example(2, 31, 8, (1.5, 1.7)),
            "c2s": lambda: I.config_c2(n=63, M=6)}[name]()
    u_d, r_d = _march(prob)
    monkeypatch.setenv("RSFDE_NO_SPEC", "1")
    u_ns, r_ns = _march(prob)
    monkeypatch.delenv("RSFDE_NO_SPEC")
    assert r_ns["iters"] == r_d["iters"] and np.array_equal(u_ns, u_d)
    monkeypatch.setenv("RSFDE_ORTHO", "cgs2")
    u_c, r_c = _march(prob)
    monkeypatch.delenv("RSFDE_ORTHO")
    assert max(abs(a - b) for a, b in zip(r_d["iters"], r_c["iters"])) <= 1
    if r_d["iters"] == r_c["iters"]:
        assert relerr(u_d, u_c) < 1e-11
    Fst = scheme.source_F(prob, 0) if prob.source_static else None
    uo, ro, _ = scheme.solve(prob, F_static=Fst)
    assert max(abs(a - b) for a, b in zip(r_d["iters"], ro.iters)) <= 1
    if r_d["iters"] != ro.iters:
        uo, ro, _ = scheme.solve(prob, F_static=Fst, fixed_iters=r_d["iters"])
    assert relerr(u_d, uo) < 1e-9


# ----------------------------------------------------------------------- graph-captured cycles
@pytest.mark.parametrize("name", ["c5s", "c2s", "ex2", "c4s_r3"])
def test_graph_cycle_bit_identical_to_stream_path(name, monkeypatch):
    # the first GMRES cycle of each CN step runs as one CUDA graph (r0, Arnoldi steps as conditional
    # IF nodes gated on the device convergence flag, SWITCH on the column count for y and x += V y):
    # the same kernels in the same order as the stream path (RSFDE_NO_GRAPH=1), so iteration counts
    # and solutions agree bit for bit; with restart 3 the later cycles of a step continue on the
    # stream path from the graph's state
    prob = {"c5s": lambda: I.config_c5(M=4, nn=(31, 15, 63)),
            "c2s": lambda: I.config_c2(n=63, M=6),
            "ex2": lambda: I.example(2, 31, 8, (1.5, 1.7)),
            "c4s_r3": lambda: I.config_c4(n=31, M=3)}[name]()
    restart = 3 if name.endswith("_r3") else None
    ss = []
    u_g, r_g = _march(prob, restart=restart, solver_out=ss)
    assert ss[0].graph_replays() == prob.M, ss[0].graph_replays()
    monkeypatch.setenv("RSFDE_NO_GRAPH", "1")
    ss = []
    u_s, r_s = _march(prob, restart=restart, solver_out=ss)
    assert ss[0].graph_replays() == 0
    monkeypatch.delenv("RSFDE_NO_GRAPH")
    assert r_g["iters"] == r_s["iters"], (r_g["iters"], r_s["iters"])
    assert np.array_equal(u_g, u_s)
    assert list(r_g["relres"]) == list(r_s["relres"])
    Fst = scheme.source_F(prob, 0) if prob.source_static else None
    uo, ro, _ = scheme.solve(prob, F_static=Fst, restart=restart)
    assert max(abs(a - b) for a, b in zip(r_g["iters"], ro.iters)) <= 1
    if r_g["iters"] != ro.iters:
        uo, ro, _ = scheme.solve(prob, F_static=Fst, restart=restart, fixed_iters=r_g["iters"])
    assert relerr(u_g, uo) < 1e-9


def test_graph_cycle_replay_mode_and_zero_residual():
    # fixed_iters (replay) caps the captured IF chain; a zero right-hand side converges at r0 = 0
    # with no Arnoldi step and no x update
    prob = I.config_c5(M=2, nn=(15, 7, 31))
    S = _solver(prob)
    F = S.compact_source(_dev(prob.f_closed(prob.t_half(0))))
    u = _dev(prob.psi_interior())
    rep = S.solve_steps(u, F=F, F_static=True, cfg=S.cfg(restart=prob.restart, fixed_iters=3))
    assert rep["iters"] == [3, 3] and S.graph_replays() == 2
    Fst = scheme.source_F(prob, 0)
    uo, ro, _ = scheme.solve(prob, F_static=Fst, fixed_iters=[3, 3])
    assert relerr(_host(u), uo) < 1e-9
    z = torch.zeros(prob.n, dtype=torch.float64, device="cuda")
    rep = S.solve_steps(z, F=torch.zeros_like(F), F_static=True, cfg=S.cfg(restart=prob.restart, tol=prob.tol))
    assert rep["iters"] == [0, 0] and all(rep["converged"]) and float(z.abs().max()) == 0.0
