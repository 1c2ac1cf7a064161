#!/usr/bin/env python3
"""Summarise an `ncu --set full` report into the per-kernel JSON kept under
profiles/: duration, DRAM bytes, grid/cluster/block, registers, tensor-pipe
activity, L2 hit rate, dynamic shared memory.

usage: ncu_summary.py REPORT.ncu-rep CAPTION > profiles/rNN_ncu_full_summary.json
"""
import csv
import io
import json
import subprocess
import sys

KEEP = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "launch__grid_size", "launch__cluster_dim_x", "launch__block_size", "launch__registers_per_thread",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
        "launch__shared_mem_per_block_dynamic", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed"]


def main():
    rep, caption = sys.argv[1], sys.argv[2]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units = rows[0], rows[1]
    kernels = []
    for r in rows[2:]:
        d = dict(zip(head, r))
        u = dict(zip(head, units))
        kernels.append({k: (f"{d[k]} {u[k]}".strip() if k != "Kernel Name" else d[k]) for k in KEEP if k in d})
    json.dump({"capture": caption, "kernels": kernels}, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
