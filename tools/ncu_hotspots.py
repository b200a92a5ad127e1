"""Per-opcode and per-instruction stall breakdown from an ncu report's source page.
    python tools/ncu_hotspots.py report.ncu-rep "<kernel substring>" [top]"""
import csv
import subprocess
import sys

path, sub = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
data = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                      capture_output=True, text=True).stdout.splitlines()
cur = None
hdr = None
out = {}
for line in data:
    if line.startswith('"Kernel Name"'):
        cur = line.split(",", 1)[1]
        out.setdefault(cur, [])
        continue
    if line.startswith('"Address"'):
        hdr = next(csv.reader([line]))
        continue
    r = next(csv.reader([line]))
    if cur is None or len(r) < 5:
        continue
    out[cur].append(r)
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
for k, rows in out.items():
    if sub not in k:
        continue
    print(k)
    tot = sum(int(r[2]) for r in rows)
    agg = {rs: 0 for rs in reasons}
    for r in rows:
        for rs in reasons:
            agg[rs] += int(r[hdr.index(rs)] or 0)
    print("  reasons: " + "  ".join(f"{rs[6:]}={100*v/tot:.1f}%" for rs, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
    ranked = sorted(rows, key=lambda r: -int(r[2]))[:top]
    for r in ranked:
        det = sorted(((int(r[hdr.index(rs)] or 0), rs[6:]) for rs in reasons), reverse=True)[:3]
        print(f"  {100*int(r[2])/tot:5.2f}%  {r[1].strip()[:60]:60s} " + " ".join(f"{n}:{v}" for v, n in det))
    break
