"""Per-kernel roofline table of one training step from an `ncu --set full`
capture of every launch (tools/gpu_prof.sh "." NAME with NCU_COUNT >= one
step): duration, achieved DRAM GB/s and its fraction of the measured HBM peak,
FP32 (FMA) / ALU / XU pipe utilisation, issue-active and warps per SM.

    python tools/ncu_step_table.py gpurun_out/allk.ncu-rep > profiles/rXX/step_kernels.md
"""

import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0}


def main():
    rep = sys.argv[1]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]

    def val(r, k):
        v = r[h.index(k)].replace(",", "")
        return float(v) * UNITS.get(u[h.index(k)], 1.0)

    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            hbm = float(json.load(fh)["hbm_gbs"])
        src = "MEASURED_PEAKS.json"
    except (OSError, KeyError, ValueError):
        hbm, src = 6650.0, "fallback"
    print(f"## One training step, every kernel (ncu --set full --clock-control none, config3)\n")
    print(f"HBM peak {hbm:.0f} GB/s ({src}); pipe columns are % of peak sustained while "
          "the SM is active (ncu `sm__pipe_*_cycles_active`, `sm__inst_executed_pipe_xu`).\n")
    print("| # | kernel | µs | DRAM GB | DRAM GB/s | % HBM peak | FMA pipe % | ALU pipe % "
          "| XU % | issue % | warps/SM |")
    print("|---|---|---|---|---|---|---|---|---|---|---|")
    tot = 0.0
    for i, r in enumerate(rows[2:]):
        name = r[h.index("Kernel Name")]
        short = name.split("(")[0].replace("void ", "")
        if len(short) > 60:
            short = short[:57] + "..."
        t = val(r, "gpu__time_duration.sum")
        b = val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum")
        gbs = b / t / 1e9
        tot += t
        print(f"| {i} | `{short}` | {t * 1e6:.1f} | {b / 1e9:.3f} | {gbs:.0f} | {100 * gbs / hbm:.1f} | "
              f"{float(r[h.index('sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active')]):.1f} | "
              f"{float(r[h.index('sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active')]):.1f} | "
              f"{float(r[h.index('sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active')]):.1f} | "
              f"{float(r[h.index('smsp__issue_active.avg.pct_of_peak_sustained_active')]):.1f} | "
              f"{float(r[h.index('sm__warps_active.avg.per_cycle_active')]):.1f} |")
    print(f"\nSum of captured kernel durations: {tot * 1e3:.3f} ms (serialised, cold caches "
          "per replay; shares, not absolutes, compare with the bench).")


if __name__ == "__main__":
    main()
