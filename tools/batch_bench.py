"""Batched vs sequential marches (NEXT-4): an alpha sweep of the paper's Example 1 / Example 2 (as in
Tables 1-2) marched one system after another and all at once with rsfde_solve_steps_batch.
    python tools/batch_bench.py [d] [N+1] [M] [B]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2404_10221_b200 import inputs as I
from paper_2404_10221_b200 import solver as SV
from paper_2404_10221_b200.solver import RsfdeSolver

d = int(sys.argv[1]) if len(sys.argv) > 1 else 1
N1 = int(sys.argv[2]) if len(sys.argv) > 2 else 64
M = int(sys.argv[3]) if len(sys.argv) > 3 else 1024
B = int(sys.argv[4]) if len(sys.argv) > 4 else 8
alphas = np.linspace(1.1, 1.9, B)
probs = [I.example(d, N1 - 1, M, (a,) * d, tol=1e-9) for a in alphas]
sols = [RsfdeSolver.from_problem(p) for p in probs]
Fs = []
for S, p in zip(sols, probs):
    F = torch.stack([S.compact_source(torch.from_numpy(np.ascontiguousarray(p.f_closed(p.t_half(m)))).cuda())
                     for m in range(M)])
    Fs.append(F)
cfgs = [S.cfg(restart=50, tol=1e-9) for S in sols]


def run(batched):
    us = [torch.from_numpy(np.ascontiguousarray(p.psi_interior())).cuda() for p in probs]
    torch.cuda.synchronize()
    t = time.perf_counter()
    if batched:
        reps = SV.solve_steps_batch(sols, us, Fs=Fs, F_static=[False] * B, cfgs=cfgs)
    else:
        reps = [S.solve_steps(u, F=F, F_static=False, cfg=c) for S, u, F, c in zip(sols, us, Fs, cfgs)]
    torch.cuda.synchronize()
    return time.perf_counter() - t, sum(sum(r["iters"]) for r in reps), us


run(True)
ts, its, us_s = run(False)
tb, itb, us_b = run(True)
same = all(torch.equal(a, b) for a, b in zip(us_s, us_b))
N = (N1 - 1) ** d
print(f"d={d} N+1={N1} M={M} B={B}: sequential {ts:.3f} s, batched {tb:.3f} s, speed-up {ts / tb:.2f}x; "
      f"{its} iterations each way; {N * its / tb:.3e} unknown-iterations/s batched; bit-identical: {same}")
