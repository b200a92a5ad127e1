#!/bin/bash
# same-box A/B of an environment switch on the in-tree library: A = default, B = the given VAR=VALUE
cd "$(dirname "$0")/.."
run() {
  local name=$1; shift
  env "$@" ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tile_kernel -s 5 -c 5 --csv \
    python tools/prof_kernels.py 511 2 > gpurun_out/abe_${name}.csv 2>/dev/null
}
rm -f gpurun_out/abe_*.csv
for r in 1 2; do
  run A_$r X=1
  run B_$r "$@"
done
python - <<'PY'
import csv, glob
for f in sorted(glob.glob("gpurun_out/abe_*.csv")):
    rows = [r for r in csv.reader(open(f)) if len(r) > 10 and r[0] != "ID"]
    t = [float(r[-1].replace(",", "")) / 1000 for r in rows if r[-3] == "gpu__time_duration.sum"]
    print(f.split("/")[-1], [round(x) for x in t], round(sum(t)))
PY
