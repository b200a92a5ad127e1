"""Per-source-line stall samples of one kernel from an ncu report (needs -lineinfo and --import-source on).
    python tools/ncu_lines.py report.ncu-rep "<kernel substring>" [top]"""
import csv
import subprocess
import sys

path, sub = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
data = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                      capture_output=True, text=True).stdout.splitlines()
fname, func, hdr = None, None, None
seen = set()
rows = []
for line in data:
    r = next(csv.reader([line]))
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r[0] == "Function Name":
        func = r[1]
    elif r[0] == "Line No":
        hdr = r
    elif hdr and len(r) == len(hdr) and func and sub in func and r[2] == "-":
        key = (func, fname, r[0])
        if key in seen:
            continue
        seen.add(key)
        rows.append((fname, r, hdr))
if not rows:
    sys.exit("no rows")
def samp(x):
    return int(x[1][x[2].index("# Samples")])
tot = sum(samp(x) for x in rows)
print(rows[0][1] and sub, "samples", tot)
agg = {}
for f, r, h in rows:
    for i, name in enumerate(h):
        if name.startswith("stall_") and "Not Issued" not in name:
            agg[name[6:]] = agg.get(name[6:], 0) + int(r[i] or 0)
print("  reasons: " + "  ".join(f"{k}={100*v/tot:.1f}%" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:9]))
for x in sorted(rows, key=lambda x: -samp(x))[:top]:
    f, r, h = x
    det = sorted(((int(r[i] or 0), name[6:]) for i, name in enumerate(h)
                  if name.startswith("stall_") and "Not Issued" not in name), reverse=True)[:3]
    print(f"{100*samp(x)/tot:5.1f}%  {f}:{r[0]:>4s}  {r[1].strip()[:90]:90s} " + " ".join(f"{n}:{v}" for v, n in det))
