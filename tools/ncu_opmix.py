"""Executed-instruction mix per opcode (and the most executed SASS lines) from an ncu report.
    python tools/ncu_opmix.py report.ncu-rep "<kernel substring>" [top]"""
import collections
import csv
import subprocess
import sys

path, sub = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
lines = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                       capture_output=True, text=True).stdout.splitlines()
cur, hdr, rows = None, None, {}
for line in lines:
    if line.startswith('"Kernel Name"'):
        cur = line.split(",", 1)[1]
        rows.setdefault(cur, [])
        continue
    if line.startswith('"Address"'):
        hdr = next(csv.reader([line]))
        continue
    r = next(csv.reader([line]))
    if cur is not None and hdr and len(r) == len(hdr):
        rows[cur].append(r)
for k, rs in rows.items():
    if sub not in k:
        continue
    ie = hdr.index("Instructions Executed")
    tot = sum(int(r[ie] or 0) for r in rs)
    ops = collections.Counter()
    for r in rs:
        txt = r[1].strip()
        toks = txt.split()
        op = toks[1] if toks and toks[0].startswith("@") and len(toks) > 1 else (toks[0] if toks else "?")
        ops[op.split(".")[0]] += int(r[ie] or 0)
    print(k, "total warp instructions", tot)
    print("  " + "  ".join(f"{o}={100*c/tot:.1f}%" for o, c in ops.most_common(25)))
    for r in sorted(rs, key=lambda r: -int(r[ie] or 0))[:top]:
        print(f"  {int(r[ie]):>12d}  {r[0]}  {r[1].strip()[:70]}")
    break
