"""Summarise an ncu --set full report into profiles/: per-kernel duration,
DRAM bytes, DRAM / L2 / tensor-pipe utilisation, registers, occupancy.

    python tools/ncu_summary.py gpurun_out/prof_r1.ncu-rep profiles/r1/ncu_full_summary
      -> <out>.md and <out>.json
"""
from __future__ import annotations

import csv
import io
import json
import subprocess
import sys

METRICS = {
    "duration_ms": "gpu__time_duration.sum",
    "dram_read_GB": "dram__bytes_read.sum",
    "dram_write_GB": "dram__bytes_write.sum",
    "dram_pct_peak": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_pct_peak": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "l2_sectors_pct": "lts__t_sectors.avg.pct_of_peak_sustained_elapsed",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "tensor_active_pct": "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "smem_tc_wavefronts_pct": "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread",
    "sm_clock_GHz": "sm__cycles_elapsed.avg.per_second",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
}


def main():
    rep, out = sys.argv[1], sys.argv[2]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    scale = {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3, "byte": 1e-9, "Kbyte": 1e-6,
             "Mbyte": 1e-3, "Gbyte": 1.0, "Tbyte": 1e3}
    kernels = []
    for r in rows[2:]:
        k = {"kernel": r[hdr.index("Kernel Name")].split("(")[0]}
        for key, m in METRICS.items():
            if m in hdr:
                i = hdr.index(m)
                v = r[i]
                try:
                    x = float(v.replace(",", ""))
                    if key.endswith("_ms") or key.endswith("_GB"):
                        x *= scale.get(units[i], 1.0)
                    k[key] = round(x, 4)
                except ValueError:
                    k[key] = v
        kernels.append(k)
    json.dump({"report": rep, "kernels": kernels}, open(out + ".json", "w"), indent=1)
    cols = ["kernel"] + list(METRICS)
    with open(out + ".md", "w") as f:
        f.write(f"# ncu --set full summary of `{rep}`\n\n")
        f.write("| " + " | ".join(cols) + " |\n|" + "---|" * len(cols) + "\n")
        for k in kernels:
            f.write("| " + " | ".join(str(k.get(c, "")) for c in cols) + " |\n")
    print(open(out + ".md").read())


if __name__ == "__main__":
    main()
