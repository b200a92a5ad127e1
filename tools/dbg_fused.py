import os, numpy as np, torch, sys
sys.path.insert(0, '.')
from paper_2404_10221_b200 import _lib as L
from paper_2404_10221_b200 import inputs as I
from paper_2404_10221_b200.solver import RsfdeSolver, RsfdeTeam
from oracle.lines import LineSystem
from oracle import scheme
prob = I.config_c5(M=2, nn=(511, 15, 31))
x = torch.from_numpy(I.seeded_vector(77, prob.n)).cuda()
Ls = LineSystem(prob.d, prob.n, prob.alpha, prob.kappa, prob.tau)
ebar = scheme.e_bar(prob)[0]
xh = x.cpu().numpy()
refK = Ls.P_alpha_inv(ebar, Ls.A_tilde(prob.e_grid(prob.t_half(1)), xh))
refA = Ls.A(prob.e_grid(prob.t_half(1)), xh)
refP = Ls.P_hat_inv(ebar, xh)
S = RsfdeSolver.from_problem(prob)
res = {}
for uf in ("0", "1"):
    os.environ["RSFDE_TEAM_UNFUSED"] = uf
    T = RsfdeTeam(prob, nranks=2)
    k = T.matvec(L.OP_K, x, m=1).cpu().numpy(); a = T.matvec(L.OP_A, x, m=1).cpu().numpy(); p = T.precond(L.PHAT_INV, x).cpu().numpy()
    res[uf] = (k, a, p)
    for nm, v, r in (("K", k, refK), ("A", a, refA), ("P", p, refP)):
        print(uf, nm, "relerr vs oracle", np.abs(v - r).max() / np.abs(r).max())
    del T
for i, nm in enumerate("KAP"):
    d = np.abs(res["0"][i] - res["1"][i]); print(nm, "fused-unfused max", d.max(), "rel", d.max() / np.abs(res["1"][i]).max(), "argmax", np.unravel_index(d.argmax(), d.shape))
k1 = S.matvec(L.OP_K, x, m=1).cpu().numpy()
print("single-GPU vs unfused", np.abs(k1 - res["1"][0]).max() / np.abs(k1).max(), "vs fused", np.abs(k1 - res["0"][0]).max() / np.abs(k1).max())
F = S.compact_source(torch.from_numpy(prob.f_closed(prob.t_half(0))).cuda())
cfg = S.cfg(restart=prob.restart, tol=prob.tol)
us = {}
for uf in ("0", "1", "0", "1"):
    os.environ["RSFDE_TEAM_UNFUSED"] = uf
    T = RsfdeTeam(prob, nranks=2)
    u = torch.zeros(prob.n, dtype=torch.float64, device="cuda")
    r = T.solve_steps(u, F=F, F_static=True, cfg=cfg)
    un = u.cpu().numpy()
    if uf in us: print(uf, "repeat diff", np.abs(un - us[uf]).max())
    us[uf] = un
    print(uf, r["iters"], r["relres"])
    del T
print("march fused-unfused", np.abs(us["0"] - us["1"]).max() / np.abs(us["1"]).max())
