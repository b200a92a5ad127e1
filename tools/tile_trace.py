"""Per-tile phase timing of the L = 1024 tile pipeline (experiment build, tools/tile_variants.sh):
run the K chain at 511^3 and summarise the clock64 stamps of the last launch (the axis-0 inverse DST).
    python tools/tile_trace.py"""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2404_10221_b200 import _lib as L
from paper_2404_10221_b200 import inputs as I
from paper_2404_10221_b200.solver import RsfdeSolver

lib = L.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "micro/var/librsfde_trace.so"))
prob = I.config_c5(n=511)
S = RsfdeSolver.from_problem(prob)
x = torch.from_numpy(I.seeded_vector(1, prob.n)).cuda()
y = torch.empty_like(x)
# which tile launch of the K chain to record: 0 oper axis 0, 1 oper axis 1, 2 oper axis 2 (last),
# 3 DST axis 1, 4 DST axis 0
which = int(sys.argv[1]) if len(sys.argv) > 1 else 4
S.matvec(L.OP_K, x, m=0, out=y)
torch.cuda.synchronize()
lib.rsfde_debug_tile_trace_select.argtypes = [ctypes.c_int]
lib.rsfde_debug_tile_trace_select(which)
S.matvec(L.OP_K, x, m=0, out=y)
torch.cuda.synchronize()
print("launch", which)
tr = np.zeros((512, 32, 12), dtype=np.uint64)
lib.rsfde_debug_tile_trace.restype = ctypes.c_int
lib.rsfde_debug_tile_trace.argtypes = [ctypes.c_void_p]
assert lib.rsfde_debug_tile_trace(tr.ctypes.data) == 0
tr = tr.astype(np.int64)
ncta = int((tr[:, 0, 0] > 0).sum())
print("CTAs traced", ncta)
last_ph = {0: 4, 1: 4, 2: 5, 3: 4, 4: 4}[which]
t0, t1, tf, te = tr[:ncta, :, 0], tr[:ncta, :, 1], tr[:ncta, :, last_ph], tr[:ncta, :, 6]
if which <= 2:
    for k, nm in [(2, "->fft conv fwd"), (3, "->fft conv inv (+C out)"), (4, "->fft dst1 (+X in)"),
                  (5, "->fft dst2")]:
        a = (tr[:ncta, 1:, k] - tr[:ncta, 1:, k - 1 if k > 2 else 1])
        a = a[tr[:ncta, 1:, k] > 0]
        if a.size:
            print(f"{nm:24s} median {np.median(a):8.0f} clk")
ok = (t0[:, 1:] > 0)
per_tile = (t0[:, 1:] - t0[:, :-1])[ok]
wait = (t1 - t0)[:, 1:][ok]
fft_ = (tf - t1)[:, 1:][ok]
rest = (te - tf)[:, 1:][ok]
nxt = (t0[:, 1:] - te[:, :-1])[ok]
def seg(a_slot, b_slot):
    a = tr[:ncta, 1:, b_slot] - tr[:ncta, 1:, a_slot]
    return a[(tr[:ncta, 1:, b_slot] > 0) & (tr[:ncta, 1:, a_slot] > 0)]
for nm, a_, b_ in [("fft0 -> C out done", 2, 9), ("C out -> fft1", 9, 3), ("fft1 -> X ready", 3, 11), ("X ready -> stencil", 11, 10),
                   ("stencil -> fft2", 10, 4), ("fft2 -> Lambda done", 4, 8), ("Lambda -> fft3", 8, 5)]:
    a = seg(a_, b_)
    if a.size:
        print(f"{nm:24s} median {np.median(a):8.0f} clk")
for name, a in [("tile period", per_tile), ("wait full", wait), ("data->last fft", fft_), ("output+store", rest),
                ("loop overhead", nxt)]:
    print(f"{name:18s} median {np.median(a):8.0f} clk  mean {a.mean():8.0f}  p90 {np.percentile(a, 90):8.0f}")
# do the two CTAs on one SM overlap their phases?  (clock64 is per SM: comparable within an SM)
sm = tr[:ncta, 0, 7]
pairs = {}
for c in range(ncta):
    pairs.setdefault(int(sm[c]), []).append(c)
both = [v for v in pairs.values() if len(v) == 2]
if both:
    a, b = both[0]
    print("SM", int(sm[a]), "CTA", a, "vs", b)
    for k in range(8):
        print("  tile", k, "A: start %d fft %d..%d end %d" % (t0[a, k] - t0[a, 0], t1[a, k] - t0[a, 0], tf[a, k] - t0[a, 0],
                                                            te[a, k] - t0[a, 0]),
              "| B: start %d fft %d..%d end %d" % (t0[b, k] - t0[a, 0], t1[b, k] - t0[a, 0], tf[b, k] - t0[a, 0],
                                                   te[b, k] - t0[a, 0]))
