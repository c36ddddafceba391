"""Summarise ncu reports / launch lists into profiles/ (markdown tables).

    python tools/ncu_summary.py report <file.ncu-rep> [...]
    python tools/ncu_summary.py launches <launches.csv>
"""
import collections
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration_us"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", "dmma_pipe_%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_throughput_%"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem_throughput_%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
]


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    print(f"### {path}\n")
    print("| kernel | " + " | ".join(n for _, n in METRICS) + " |")
    print("|---|" + "---|" * len(METRICS))
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0]
        vals = []
        for m, _ in METRICS:
            if m not in hdr:
                vals.append("-")
                continue
            v, u = r[hdr.index(m)], units[hdr.index(m)]
            if m.startswith("dram__bytes") and v:
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
                v = f"{float(v.replace(',', '')) * scale / 1e6:.2f} MB"
            vals.append(v)
        print(f"| {name} | " + " | ".join(vals) + " |")
    print()


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[hi]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        v *= {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(r[ui], 1.0)
        name = r[ki].split("(")[0]
        tot[name] += v
        cnt[name] += 1
    T = sum(tot.values())
    print(f"### launch list {path} (ncu, serialised, cold caches: compare shares)\n")
    print("| kernel | launches | total us | share |\n|---|---|---|---|")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"| {k} | {cnt[k]} | {v:.1f} | {100 * v / T:.1f}% |")
    print(f"| **total** | {sum(cnt.values())} | {T:.1f} | |\n")


if __name__ == "__main__":
    mode = sys.argv[1]
    for p in sys.argv[2:]:
        report(p) if mode == "report" else launches(p)
