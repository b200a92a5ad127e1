import os, numpy as np, torch, sys
sys.path.insert(0, '.')
from paper_2404_10221_b200 import _lib as L
from paper_2404_10221_b200 import inputs as I
from paper_2404_10221_b200.solver import RsfdeSolver, RsfdeTeam
prob = I.config_c5(M=2, nn=(511, 15, 31))
x = torch.from_numpy(I.seeded_vector(77, prob.n)).cuda()
S = RsfdeSolver.from_problem(prob)
F = S.compact_source(torch.from_numpy(prob.f_closed(prob.t_half(0))).cuda())
cfg = S.cfg(restart=prob.restart, tol=prob.tol)
def march(uf, pre):
    os.environ["RSFDE_TEAM_UNFUSED"] = uf
    T = RsfdeTeam(prob, nranks=2)
    if pre:
        T.matvec(L.OP_K, x, m=1); T.matvec(L.OP_A, x, m=1); T.precond(L.PHAT_INV, x)
    u = torch.zeros(prob.n, dtype=torch.float64, device="cuda")
    r = T.solve_steps(u, F=F, F_static=True, cfg=cfg)
    torch.cuda.synchronize()
    return u.cpu().numpy()
res = {(uf, pre): march(uf, pre) for uf in ("0", "1") for pre in (False, True)}
for k, v in res.items():
    print(k, [float(np.abs(v - w).max()) for w in res.values()])
