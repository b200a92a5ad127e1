"""Run the hot operator chain in isolation for ncu: warm-up K = P_hat^{-1} A (3 spectral operator
passes + 2 inverse DST passes) once, then the same chain again (the profiled launches).

    python tools/prof_kernels.py [n] [reps] [--cfg C3]
ncu: -k regex:"oper_pass|dst_pass" -s 5 -c 5  captures the second chain (3D; a 2D chain is 3 launches).
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2404_10221_b200 import _lib as L
from paper_2404_10221_b200 import inputs as I
from paper_2404_10221_b200.solver import RsfdeSolver

if "--lib" in sys.argv:  # experiment variant of the library (tools/tile_variants.sh)
    i = sys.argv.index("--lib")
    L.load(sys.argv[i + 1])
    del sys.argv[i:i + 2]
cfg = "C5"
if "--cfg" in sys.argv:  # another BASELINE config at its full size (C2, C3, C4)
    i = sys.argv.index("--cfg")
    cfg = sys.argv[i + 1]
    del sys.argv[i:i + 2]
n = int(sys.argv[1]) if len(sys.argv) > 1 else 511
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
prob = I.config_c5(n=n) if cfg == "C5" else {"C2": I.config_c2, "C3": I.config_c3, "C4": I.config_c4}[cfg]()
S = RsfdeSolver.from_problem(prob)
x = torch.from_numpy(I.seeded_vector(1, prob.n)).cuda()
y = torch.empty_like(x)
S.profile(True)
for r in range(reps):
    torch.cuda.synchronize()
    t = time.perf_counter()
    S.matvec(L.OP_K, x, m=0, out=y)
    torch.cuda.synchronize()
    print(f"K chain {r}: {1e3*(time.perf_counter()-t):.2f} ms", flush=True)
for k, v in S.profile_read().items():
    if v["launches"]:
        print(f"{k:22s} launches {v['launches']:4d}  ms {v['ms']:9.3f}  GB/s {v['bytes']/(v['ms']*1e-3)/1e9 if v['ms'] else 0:8.1f}")
