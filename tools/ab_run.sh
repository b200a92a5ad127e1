#!/bin/bash
# same-box A/B of the C5 (and C4) K chain: A = tools/micro/var/librsfde_A.so, B = in-tree library
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py -q -x > gpurun_out/ab_tests.log 2>&1; echo "rc $?" >> gpurun_out/ab_tests.log
run() {
  local name=$1 lib=$2 cfg=$3
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tile_kernel -s 5 -c 5 --csv \
    python tools/prof_kernels.py $cfg $lib > gpurun_out/ab_${name}.csv 2>/dev/null
}
rm -f gpurun_out/ab_*.csv
for r in 1 2; do
  run A5_$r "--lib tools/micro/var/librsfde_A.so" "511 2"
  run B5_$r "" "511 2"
  run A4_$r "--lib tools/micro/var/librsfde_A.so" "--cfg C4 255 2"
  run B4_$r "" "--cfg C4 255 2"
done
python - <<'PY'
import csv, glob
for f in sorted(glob.glob("gpurun_out/ab_*.csv")):
    rows = [r for r in csv.reader(open(f)) if len(r) > 10 and r[0] != "ID"]
    t = [float(r[-1].replace(",", "")) / 1000 for r in rows if r[-3] == "gpu__time_duration.sum"]
    print(f.split("/")[-1], [round(x) for x in t], round(sum(t)))
PY
