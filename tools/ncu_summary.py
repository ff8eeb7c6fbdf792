"""Summarise ncu output for profiles/: the launch list of the timed steps
(share per kernel) and the key counters of a `--set full` capture.

    python tools/ncu_summary.py --launches gpurun_out/launches.csv --steps 2 \
        --rep gpurun_out/prof.ncu-rep > profiles/rXX/ncu_summary.md
"""

import argparse
import csv
import io
import subprocess
from collections import defaultdict

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
    ("sm__warps_active.avg.per_cycle_active", "warps active / SM"),
    ("launch__registers_per_thread", "registers"),
    ("launch__shared_mem_per_block_static", "static smem / CTA"),
    ("launch__occupancy_limit_registers", "CTA limit (regs)"),
    ("launch__occupancy_limit_shared_mem", "CTA limit (smem)"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "threads / warp-inst"),
    ("smsp__inst_executed.sum", "warp instructions"),
]


def launches(path, steps):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    t, c = defaultdict(float), defaultdict(int)
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        t[name] += v
        c[name] += 1
    tot = sum(t.values())
    out = ["| kernel | us / step | share | launches / step |", "|---|---|---|---|"]
    for n, v in sorted(t.items(), key=lambda x: -x[1]):
        out.append(f"| `{n}` | {v / 1e3 / steps:.1f} | {100 * v / tot:.1f} % | {c[n] / steps:g} |")
    out.append(f"| **total** | {tot / 1e3 / steps:.1f} | | {sum(c.values()) / steps:g} |")
    return "\n".join(out)


def full(rep, raw=None):
    if raw:  # `ncu -i REP --page raw --csv` output written on the GPU box
        txt = open(raw).read()
    else:
        txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, units = rows[0], rows[1]
    data = rows[2:]
    names = [r[h.index("Kernel Name")].split("(")[0].replace("void ", "") for r in data]
    out = ["| counter | " + " | ".join(f"`{n}`" for n in names) + " |",
           "|---|" + "---|" * len(names)]
    for key, label in KEYS:
        if key not in h:
            continue
        i = h.index(key)
        out.append(f"| {label} ({units[i]}) | " + " | ".join(r[i] for r in data) + " |")
    return "\n".join(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--rep")
    ap.add_argument("--raw", help="the --page raw --csv dump instead of a report")
    a = ap.parse_args()
    if a.launches:
        print("## Launch list (ncu gpu__time_duration, --clock-control none, timed steps only)\n")
        print(launches(a.launches, a.steps))
        print()
    if a.rep or a.raw:
        print("## Full capture (ncu --set full)\n")
        print(full(a.rep, a.raw))


if __name__ == "__main__":
    main()
