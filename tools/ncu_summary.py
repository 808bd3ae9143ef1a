"""Summarise an ncu report (or a launch-list CSV) into the text committed under
profiles/.  Usage:
  python tools/ncu_summary.py report.ncu-rep  > profiles/rNN_<name>.md
  python tools/ncu_summary.py launches.csv    > profiles/rNN_launches.md
"""
import collections
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration (us)", 1e-3),
    ("dram__bytes_read.sum", "DRAM read (MB)", 1.0),
    ("dram__bytes_write.sum", "DRAM write (MB)", 1.0),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM thru %", 1.0),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM thru %", 1.0),
    ("smsp__issue_active.avg.per_cycle_active", "issue/cycle/SMSP", 1.0),
    ("smsp__warps_active.avg.per_cycle_active", "warps active/SMSP", 1.0),
    ("smsp__warps_eligible.avg.per_cycle_active", "warps eligible/SMSP", 1.0),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "threads/inst", 1.0),
    ("smsp__inst_executed.sum", "warp instructions (M)", 1e-6),
    ("launch__registers_per_thread", "registers", 1.0),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/CTA (KB)", 1.0),
    ("launch__occupancy_limit_shared_mem", "CTA/SM (smem limit)", 1.0),
]


def _unit_scale(unit: str, name: str) -> float:
    if name.startswith("dram__bytes"):
        return {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(unit, 1.0)
    if name == "gpu__time_duration.sum":
        return {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1.0)
    return 1.0


def report(path: str) -> None:
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    print(f"# ncu summary: {path.split('/')[-1]}\n")
    stall_cols = [i for i, h in enumerate(hdr) if h.startswith("smsp__average_warps_issue_stalled")
                  and h.endswith("per_issue_active.ratio")]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        print(f"## {name.split('(')[0]}\n")
        print("| metric | value |\n|---|---|")
        for m, label, _ in METRICS:
            if m in hdr:
                i = hdr.index(m)
                try:
                    v = float(r[i].replace(",", "")) * _unit_scale(units[i], m)
                    if m == "smsp__inst_executed.sum":
                        v *= 1e-6
                    print(f"| {label} (`{m}`) | {v:,.3f} |")
                except ValueError:
                    print(f"| {label} (`{m}`) | {r[i]} |")
        st = sorted(((float(r[i] or 0), hdr[i].replace("smsp__average_warps_issue_stalled_", "")
                      .replace("_per_issue_active.ratio", "")) for i in stall_cols), reverse=True)[:6]
        print("\nTop stall reasons (warps per issue): " + ", ".join(f"{n} {v:.2f}" for v, n in st) + "\n")


def launches(path: str) -> None:
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hi]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    ui = hdr.index("Metric Unit") if "Metric Unit" in hdr else None
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        scale = _unit_scale(r[ui], "gpu__time_duration.sum") if ui is not None else 1e-3
        agg.setdefault(r[ki].split("(")[0], []).append(float(r[vi].replace(",", "")) * scale)
    tot = sum(sum(v) for v in agg.values())
    print(f"# launch list: {path.split('/')[-1]} (ncu gpu__time_duration.sum, cold-cache, serialised)\n")
    print("| kernel | launches | mean us | total us | share |\n|---|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"| {k} | {len(v)} | {sum(v)/len(v):.1f} | {sum(v):.1f} | {100*sum(v)/tot:.1f}% |")


if __name__ == "__main__":
    p = sys.argv[1]
    (report if p.endswith(".ncu-rep") else launches)(p)
