"""Summarise an ncu --set full report (per kernel: time, DRAM bytes, issue/FP64/warps, stalls).

    python tools/summarize_ncu.py gpurun_out/prof_r01_v2.ncu-rep > profiles/r01_ncu_v2_summary.txt
"""
import csv
import subprocess
import sys

KEYS = [("gpu__time_duration.sum", "time_ms"), ("dram__bytes_read.sum", "dram_read_GB"),
        ("dram__bytes_write.sum", "dram_write_GB"), ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%"),
        ("smsp__inst_executed.sum", "warp_inst"), ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_%"),
        ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64_pipe_%"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_%"),
        ("launch__registers_per_thread", "regs"), ("launch__grid_size", "grid"),
        ("launch__shared_mem_per_block_dynamic", "smem_KB"), ("lts__t_sector_hit_rate.pct", "L2_hit_%")]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    print(f"# {path}")
    for r in rows[2:]:
        print(r[hdr.index("Kernel Name")])
        vals = []
        for k, short in KEYS:
            if k in hdr:
                vals.append(f"{short}={r[hdr.index(k)]}")
        print("   " + "  ".join(vals))
        st = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled_"):
                try:
                    st.append((float(r[i]), h.replace("smsp__average_warps_issue_stalled_", "").replace(
                        "_per_issue_active.ratio", "")))
                except ValueError:
                    pass
        print("   stalls: " + "  ".join(f"{n}={v:.2f}" for v, n in sorted(st, reverse=True)[:8]))


if __name__ == "__main__":
    main(sys.argv[1])
