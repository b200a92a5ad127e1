"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into per-kernel shares.

    python tools/summarize_launches.py gpurun_out/launches_r01.csv > profiles/r01_launches_summary.txt
"""
import csv
import re
import sys
from collections import defaultdict


def main(path):
    lines = [ln for ln in open(path) if ln.startswith('"')]
    rows = list(csv.DictReader(lines))
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        name = re.sub(r"\(.*", "", name)
        name = name.replace("void ", "").replace("rsfde::", "")
        ns = float(r["Metric Value"].replace(",", ""))
        tot[name] += ns
        cnt[name] += 1
    grand = sum(tot.values())
    print(f"# {path}: {sum(cnt.values())} launches, {grand/1e6:.3f} ms total (cold-cache, serialised ncu times)")
    print(f"{'kernel':48s} {'launches':>8s} {'ms':>10s} {'share':>7s} {'mean_ms':>9s}")
    for k in sorted(tot, key=lambda k: -tot[k]):
        print(f"{k:48s} {cnt[k]:8d} {tot[k]/1e6:10.3f} {100*tot[k]/grand:6.2f}% {tot[k]/cnt[k]/1e6:9.4f}")


if __name__ == "__main__":
    main(sys.argv[1])
