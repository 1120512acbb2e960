"""Summarise an ncu --set full capture into the numbers DESIGN.md / bench.py cite.

    python profiles/summarize.py gpurun_out/full_<tag>.ncu-rep > profiles/<round>/full_<tag>.txt
"""
from __future__ import annotations

import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "lts__t_bytes.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "launch__shared_mem_per_block_dynamic",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__cycles_elapsed.avg.per_second",
]


def main(path: str) -> None:
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    header, units = rows[0], rows[1]
    for r in rows[2:]:
        rec = dict(zip(header, r))
        print(f"kernel: {rec.get('Kernel Name', '?')[:160]}")
        for k in KEYS:
            if k in rec:
                i = header.index(k)
                print(f"  {k} = {r[i]} {units[i]}")
        for i, name in enumerate(header):
            if ("pipe_tensor" in name or "pipe_uma" in name or "tmem" in name) and name not in KEYS and r[i]:
                if name.endswith("pct_of_peak_sustained_active") and ".avg." in name:
                    print(f"  {name} = {r[i]} {units[i]}")


if __name__ == "__main__":
    main(sys.argv[1])
