#!/bin/bash
# A/B of the FP64 ping-pong tile variant: A = tools/micro/var/librsfde_A.so (base), B = in-tree library
cd "$(dirname "$0")/.."
run() {  # name, lib args, env...
  local name=$1 lib=$2; shift 2
  env "$@" ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tile_kernel -s 5 -c 5 --csv \
    python tools/prof_kernels.py 511 2 $lib > gpurun_out/pp_${name}.csv 2>/dev/null
}
RSFDE_TILE128=1 RSFDE_TILE_CT8=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "matvec or precond or tile128 or solve_steps" > gpurun_out/pp_tests.log 2>&1
for r in 1 2; do
  run A_$r "--lib tools/micro/var/librsfde_A.so" X=1
  run A128_$r "--lib tools/micro/var/librsfde_A.so" RSFDE_TILE128=1
  run B0_$r "" X=1
  run B1_$r "" RSFDE_TILE128=1 RSFDE_TILE_CT8=1
done
python - <<'PY'
import csv, glob
for f in sorted(glob.glob("gpurun_out/pp_*.csv")):
    rows = [r for r in csv.reader(open(f)) if len(r) > 10 and r[0] != "ID"]
    t = [float(r[-1].replace(",", "")) / 1000 for r in rows if r[-3] == "gpu__time_duration.sum"]
    print(f.split("/")[-1], [round(x) for x in t], round(sum(t)))
PY
