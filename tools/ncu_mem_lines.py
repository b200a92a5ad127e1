"""Per-source-line memory traffic of one kernel from an ncu report (-lineinfo, --import-source on):
global L1 tag requests, L2 theoretical sectors (and the ideal count), shared wavefronts (and ideal).
    python tools/ncu_mem_lines.py report.ncu-rep "<kernel substring>" [top]"""
import csv
import subprocess
import sys

path, sub = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
data = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                      capture_output=True, text=True).stdout.splitlines()
fname = func = hdr = None
seen, rows = set(), []
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
        if key not in seen:
            seen.add(key)
            rows.append((fname, r))
if not rows:
    sys.exit("no rows")
col = {n: i for i, n in reversed(list(enumerate(hdr)))}
def val(r, n):
    try:
        return int(float(r[col[n]] or 0))
    except ValueError:
        return 0
names = ["L1 Tag Requests Global", "L2 Theoretical Sectors Global", "L2 Theoretical Sectors Global Ideal",
         "L1 Wavefronts Shared", "L1 Wavefronts Shared Ideal"]
tot = {n: sum(val(r, n) for _, r in rows) for n in names}
print(sub, {n: tot[n] for n in names})
rows.sort(key=lambda x: -(val(x[1], names[1]) + val(x[1], names[3])))
print("  tagreq  l2sect  l2ideal  shwave  shideal  file:line  source")
for f, r in rows[:top]:
    print("  " + " ".join(f"{val(r, n):8d}" for n in names) + f"  {f}:{r[0]}  {r[1].strip()[:90]}")
