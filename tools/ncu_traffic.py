"""DRAM traffic per launch of the pass kernels from an ncu --set full report (dram__bytes_read.sum +
dram__bytes_write.sum), grouped into bench.py's kernel classes; writes the JSON bench.py reports as
roofline.traffic.
    python tools/ncu_traffic.py gpurun_out/prof_tile_final.ncu-rep > profiles/r01_ncu_traffic.json"""
import csv
import json
import re
import subprocess
import sys
from collections import defaultdict

path = sys.argv[1]
out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
k_name = hdr.index("Kernel Name")
k_rd, k_wr = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
units = rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
cls = defaultdict(list)
for r in rows[2:]:
    name = r[k_name]
    m = re.search(r"tile_kernel<(\d)", name)
    if not m:
        continue
    mode = int(m.group(1))
    c = "oper_pass_spectral" if mode in (2, 3) else "dst_pass"
    b = float(r[k_rd].replace(",", "")) * scale[units[k_rd]] + float(r[k_wr].replace(",", "")) * scale[units[k_wr]]
    cls[c].append(b)
res = {c: {"bytes_per_launch": sum(v) / len(v), "launches": len(v)} for c, v in cls.items()}
res["source"] = f"ncu --set full of tools/prof_kernels.py 511 1 (one K chain at C5), {path.split('/')[-1]}"
print(json.dumps(res, indent=1))
