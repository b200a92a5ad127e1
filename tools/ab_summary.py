"""Summarise tools/ab_kernels.sh output: per-launch microseconds of the A and B libraries."""
import csv
import glob
for v in "AB":
    runs = []
    for f in sorted(glob.glob(f"gpurun_out/ab_{v}_*.csv")):
        rows = [r for r in csv.reader(open(f)) if len(r) > 10 and r[0] != "ID"]
        runs.append([float(r[-1].replace(",", "")) / 1000 for r in rows if r[-3] == "gpu__time_duration.sum"])
    for r in runs:
        print(v, [round(x) for x in r], round(sum(r)))
