"""GPU parity of the slab-sharded 3D path.

The ranks are emulated in one process on one device (nlocal == nranks: the transport is device
copies; decomposition, transposes, pads and the reductions are the production code), plus a
single-rank NCCL communicator that exercises the NCCL calls (send/recv groups, allreduce)."""
import numpy as np
import pytest

from oracle import scheme
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


@pytest.mark.parametrize("shape,P", [((15, 7, 31), 2), ((31, 15, 15), 4), ((63, 31, 7), 8), ((63, 63, 63), 4),
                                     # n = 511 / 255 axes: the tile pipelines in both slab layouts
                                     ((511, 15, 31), 2), ((15, 31, 511), 4), ((255, 15, 31), 2), ((31, 15, 255), 2)])
def test_sharded_operators_match_oracle(shape, P):
    from paper_2404_10221_b200 import _lib as L
    from paper_2404_10221_b200.solver import RsfdeTeam
    prob = I.config_c5(M=4, nn=shape)
    T = RsfdeTeam(prob, nranks=P)
    Ls = LineSystem(prob.d, prob.n, prob.alpha, prob.kappa, prob.tau)
    ebar = scheme.e_bar(prob)[0]
    x = I.seeded_vector(31, prob.n)
    for m in (0, 3):
        e = prob.e_grid(prob.t_half(m))
        got = _host(T.matvec(L.OP_K, _dev(x), m=m))
        assert relerr(got, Ls.P_alpha_inv(ebar, Ls.A_tilde(e, x))) < 1e-12
        got = _host(T.matvec(L.OP_A, _dev(x), m=m))
        assert relerr(got, Ls.A(e, x)) < 1e-12
    for kind, ref in ((L.PHAT_INV, Ls.P_hat_inv(ebar, x)), (L.PALPHA_INV, Ls.P_alpha_inv(ebar, x))):
        assert relerr(_host(T.precond(kind, _dev(x))), ref) < 1e-12


@pytest.mark.parametrize("shape,P", [((31, 15, 63), 2), ((15, 15, 15), 4), ((63, 63, 31), 8), ((511, 15, 31), 2)])
def test_sharded_march_matches_oracle_and_single_gpu(shape, P):
    from paper_2404_10221_b200.solver import RsfdeSolver, RsfdeTeam
    prob = I.config_c5(M=3, nn=shape)
    S = RsfdeSolver.from_problem(prob)
    F = S.compact_source(_dev(prob.f_closed(prob.t_half(0))))
    cfg = S.cfg(restart=prob.restart, tol=prob.tol)
    u1 = torch.zeros(prob.n, dtype=torch.float64, device="cuda")
    r1 = S.solve_steps(u1, F=F, F_static=True, cfg=cfg)
    T = RsfdeTeam(prob, nranks=P)
    u2 = torch.zeros(prob.n, dtype=torch.float64, device="cuda")
    r2 = T.solve_steps(u2, F=F, F_static=True, cfg=cfg)
    assert r2["iters"] == r1["iters"] and all(r2["converged"])
    assert relerr(_host(u2), _host(u1)) < 1e-12
    uo, ro, _ = scheme.solve(prob, F_static=scheme.source_F(prob, 0))
    assert max(abs(a - b) for a, b in zip(r2["iters"], ro.iters)) <= 1
    if r2["iters"] != ro.iters:
        uo, ro, _ = scheme.solve(prob, F_static=scheme.source_F(prob, 0), fixed_iters=r2["iters"])
    assert relerr(_host(u2), uo) < 1e-9


def test_single_rank_nccl_transport():
    # a one-rank NCCL communicator drives the NCCL code path (grouped send/recv, allreduce) on one GPU
    from paper_2404_10221_b200 import _lib as L
    from paper_2404_10221_b200.solver import RsfdeTeam
    prob = I.config_c5(M=2, nn=(15, 7, 31))
    uid = RsfdeTeam.nccl_unique_id()
    assert len(uid) == 128
    T = RsfdeTeam(prob, nranks=1, rank=0, nlocal=1, nccl_id=uid)
    Ls = LineSystem(prob.d, prob.n, prob.alpha, prob.kappa, prob.tau)
    x = I.seeded_vector(5, prob.n)
    got = _host(T.matvec(L.OP_K, _dev(x), m=1))
    ebar = scheme.e_bar(prob)[0]
    assert relerr(got, Ls.P_alpha_inv(ebar, Ls.A_tilde(prob.e_grid(prob.t_half(1)), x))) < 1e-12
    from paper_2404_10221_b200.solver import RsfdeSolver
    S = RsfdeSolver.from_problem(prob)
    F = S.compact_source(_dev(prob.f_closed(prob.t_half(0))))
    u1 = torch.zeros(prob.n, dtype=torch.float64, device="cuda")
    u2 = torch.zeros(prob.n, dtype=torch.float64, device="cuda")
    r1 = S.solve_steps(u1, F=F, cfg=S.cfg(restart=20, tol=1e-8))
    r2 = T.solve_steps(u2, F=F, cfg=S.cfg(restart=20, tol=1e-8))
    assert r1["iters"] == r2["iters"] and relerr(_host(u2), _host(u1)) < 1e-12


def test_slab_compact_source():
    from paper_2404_10221_b200.solver import RsfdeTeam
    prob = I.config_c5(M=2, nn=(31, 7, 15))
    T = RsfdeTeam(prob, nranks=4)
    f = np.random.default_rng(4).uniform(-1, 1, [v + 2 for v in prob.n])
    ref = scheme.compact_source(prob.alpha, f)
    for l in range(4):
        lo, cnt = T.slab(l)
        assert lo == 8 * l and cnt == min(8, 31 - lo)
        got = _host(T.compact_source(_dev(f[lo:lo + cnt + 2]), local=l))
        assert relerr(got, ref[lo:lo + cnt]) < 1e-14


@pytest.mark.parametrize("shape,P", [((511, 15, 31), 2), ((255, 31, 63), 4), ((255, 15, 31), 8), ((31, 15, 63), 2)])
def test_fused_exchanges_equal_explicit_transposes(shape, P, monkeypatch):
    # fused exchanges (the x1 passes read the receive blocks and write the send blocks directly:
    # segmented contiguous axis) against the explicit layout-T transposes (RSFDE_TEAM_UNFUSED=1):
    # the same arithmetic, so the K chain, the preconditioner and a march agree bit for bit
    from paper_2404_10221_b200 import _lib as L
    from paper_2404_10221_b200.solver import RsfdeSolver, RsfdeTeam
    prob = I.config_c5(M=2, nn=shape)
    x = _dev(I.seeded_vector(77, prob.n))
    S = RsfdeSolver.from_problem(prob)
    F = S.compact_source(_dev(prob.f_closed(prob.t_half(0))))
    cfg = S.cfg(restart=prob.restart, tol=prob.tol)
    outs = []
    for unfused in (False, True):
        if unfused:
            monkeypatch.setenv("RSFDE_TEAM_UNFUSED", "1")
        T = RsfdeTeam(prob, nranks=P)
        k = _host(T.matvec(L.OP_K, x, m=1))
        a = _host(T.matvec(L.OP_A, x, m=1))
        pr = _host(T.precond(L.PHAT_INV, x))
        u = torch.zeros(prob.n, dtype=torch.float64, device="cuda")
        r = T.solve_steps(u, F=F, F_static=True, cfg=cfg)
        outs.append((k, a, pr, _host(u), r["iters"]))
        del T
    monkeypatch.delenv("RSFDE_TEAM_UNFUSED")
    for name, v0, v1 in zip(("K", "A", "P_hat^-1", "march"), outs[0][:4], outs[1][:4]):
        assert np.array_equal(v0, v1), (name, float(np.abs(v0 - v1).max() / np.abs(v1).max()))
    assert outs[0][4] == outs[1][4]


@pytest.mark.parametrize("shape,P,chunks", [((511, 15, 31), 2, 4), ((255, 31, 63), 4, 2), ((255, 15, 31), 8, 4),
                                            ((63, 31, 15), 2, 8)])
def test_chunked_exchanges_equal_whole_slab_exchanges(shape, P, chunks, monkeypatch):
    # chunked exchanges (sub-slabs of the x1 slab; piece c travels on the exchange stream while the
    # passes of sub-slab c+1 / the unpack and inverse DSTs of sub-slab c-1 run on the caller's stream)
    # against whole-slab exchanges (RSFDE_TEAM_CHUNKS=1): the same arithmetic per pencil, so K, A,
    # P_hat^-1 and a march agree bit for bit -- and the chunked march agrees with the oracle-checked
    # single-GPU path
    from paper_2404_10221_b200 import _lib as L
    from paper_2404_10221_b200.solver import RsfdeSolver, RsfdeTeam
    prob = I.config_c5(M=2, nn=shape)
    x = _dev(I.seeded_vector(78, prob.n))
    S = RsfdeSolver.from_problem(prob)
    F = S.compact_source(_dev(prob.f_closed(prob.t_half(0))))
    cfg = S.cfg(restart=prob.restart, tol=prob.tol)
    outs = []
    for nc in (chunks, 1):
        monkeypatch.setenv("RSFDE_TEAM_CHUNKS", str(nc))
        T = RsfdeTeam(prob, nranks=P)
        k = _host(T.matvec(L.OP_K, x, m=1))
        a = _host(T.matvec(L.OP_A, x, m=1))
        pr = _host(T.precond(L.PHAT_INV, x))
        u = torch.zeros(prob.n, dtype=torch.float64, device="cuda")
        r = T.solve_steps(u, F=F, F_static=True, cfg=cfg)
        outs.append((k, a, pr, _host(u), r["iters"]))
        del T
    monkeypatch.delenv("RSFDE_TEAM_CHUNKS")
    for name, v0, v1 in zip(("K", "A", "P_hat^-1", "march"), outs[0][:4], outs[1][:4]):
        assert np.array_equal(v0, v1), (name, float(np.abs(v0 - v1).max() / np.abs(v1).max()))
    assert outs[0][4] == outs[1][4]
    ks = _host(S.matvec(L.OP_K, x, m=1))
    assert np.abs(outs[0][0] - ks).max() / np.abs(ks).max() < 1e-12
