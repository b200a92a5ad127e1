cd "$(dirname "$0")/.."
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"tile_kernel" -s 5 -c 5 -o gpurun_out/r2c_tile python tools/prof_kernels.py 511 2 > gpurun_out/r2c_tile_ncu.log 2>&1
run() {
  local name=$1 lib=$2; shift 2
  env "$@" ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tile_kernel -s 5 -c 5 --csv \
    python tools/prof_kernels.py 511 2 $lib > gpurun_out/pp_${name}.csv 2>/dev/null
}
rm -f gpurun_out/pp_*.csv
for r in 1 2; do
  run B0_$r "" X=1
  run Bct8_$r "" RSFDE_TILE_CT8=1
done
python - <<'PY'
import csv, glob
for f in sorted(glob.glob("gpurun_out/pp_*.csv")):
    rows = [r for r in csv.reader(open(f)) if len(r) > 10 and r[0] != "ID"]
    t = [float(r[-1].replace(",", "")) / 1000 for r in rows if r[-3] == "gpu__time_duration.sum"]
    print(f.split("/")[-1], [round(x) for x in t], round(sum(t)))
PY
