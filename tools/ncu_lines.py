"""Attribute ncu per-instruction stall samples to CUDA source lines.

    python tools/ncu_lines.py <report.ncu-rep> <object.o> <kernel-substring> [mangled-name]

The SASS page of the report is matched instruction-by-instruction with the
line table nvdisasm -g prints for the same cubin (build with -lineinfo).
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile


def main():
    rep, obj, ksub = sys.argv[1:4]
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    secs = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"]
    data = hdr = None
    for si, s in enumerate(secs):
        if ksub in rows[s][1]:
            hdr = rows[s + 1]
            end = secs[si + 1] if si + 1 < len(secs) else len(rows)
            data = [r for r in rows[s + 2:end] if len(r) == len(hdr)]
            break
    if data is None:
        sys.exit("kernel not found")
    S = hdr.index("Warp Stall Sampling (All Samples)")
    I = hdr.index("Instructions Executed")
    addrs = [int(r[0], 16) for r in data]
    base = min(addrs)
    samples = {a - base: float(r[S] or 0) for a, r in zip(addrs, data)}
    insts = {a - base: float(r[I] or 0) for a, r in zip(addrs, data)}
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, capture_output=True)
    cub = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
    dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cub)], capture_output=True, text=True).stdout
    # locate the function: explicit mangled name, else the report's kernel name must be unique
    fn = sys.argv[4] if len(sys.argv) > 4 else None
    if fn is None:
        names = set(re.findall(r"\.text\.(\S+):", dis))
        cands = [nm for nm in names if ksub in nm]
        if len(cands) == 1:
            fn = cands[0]
        elif cands:
            sys.exit("ambiguous kernel; pass the mangled name: " + " ".join(sorted(cands)))
    lines_by_off = {}
    cur_line = None
    in_fn = fn is None
    for ln in dis.splitlines():
        m = re.match(r"\s*\.text\.(\S+):", ln)
        if m:
            in_fn = fn is None or m.group(1) == fn
            continue
        m = re.search(r'//## File "(.*?)", line (\d+)', ln)
        if m:
            cur_line = f"{os.path.basename(m.group(1))}:{m.group(2)}"
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m and in_fn:
            lines_by_off[int(m.group(1), 16)] = cur_line
    per_line = collections.Counter()
    per_line_i = collections.Counter()
    tot = sum(samples.values())
    for off, v in samples.items():
        per_line[lines_by_off.get(off)] += v
        per_line_i[lines_by_off.get(off)] += insts.get(off, 0)
    src = None
    for ln, v in sorted(per_line.items(), key=lambda x: -x[1])[:40]:
        print(f"{100 * v / tot:5.1f}%  inst {per_line_i[ln]:>12.0f}  {ln}")


if __name__ == "__main__":
    main()
