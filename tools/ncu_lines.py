"""Map ncu SASS-level stall samples to CUDA source lines.

usage: python tools/ncu_lines.py <report.ncu-rep> <kernel-substring> [cubin-name] [n]
Uses nvdisasm -g on the cubin extracted from lib/libabsp.so (cuobjdump -xelf) to map
instruction offsets to lines (needs -lineinfo, which build.py passes)."""
import csv
import io
import os
import re
import subprocess
import sys
import tempfile
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def sass_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    h = rows[hi]
    col = os.environ.get("NCU_REASON", "Warp Stall Sampling (All Samples)")
    si = h.index(col)
    ii = h.index("Instructions Executed")
    res = []
    for r in rows[hi + 1:]:
        if len(r) > ii and r[0].startswith("0x"):
            res.append((int(r[0], 16), r[1].strip(), float(r[si] or 0), float(r[ii] or 0)))
    return res


def line_map(cubin, func_sub):
    out = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
    cur_func, line, mapping = None, None, defaultdict(dict)
    for ln in out.splitlines():
        m = re.match(r"\s*\.text\.(\S+):", ln)
        if m:
            cur_func = m.group(1)
            continue
        m = re.search(r'//## File ".*?/([^/"]+)", line (\d+)', ln)
        if m:
            line = f"{m.group(1)}:{m.group(2)}"
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m and cur_func and func_sub in cur_func:
            mapping[cur_func][int(m.group(1), 16)] = line
    return mapping


def main():
    rep, func_sub = sys.argv[1], sys.argv[2]
    cubin_name = sys.argv[3] if len(sys.argv) > 3 else None
    n = int(sys.argv[4]) if len(sys.argv) > 4 else 25
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.join(ROOT, "paper_2605_12110_b200/lib/libabsp.so")],
                   cwd=d, capture_output=True)
    cubins = [os.path.join(d, f) for f in os.listdir(d) if f.endswith(".cubin") and (not cubin_name or cubin_name in f)]
    rows = sass_rows(rep)
    base = rows[0][0]
    best = None
    for cb in cubins:
        for fn, mp in line_map(cb, func_sub).items():
            # pick the function whose instruction count matches the report
            if best is None or abs(len(mp) - len(rows)) < abs(len(best[1]) - len(rows)):
                best = (fn, mp)
    fn, mp = best
    agg = defaultdict(lambda: [0.0, 0.0, set()])
    tot = sum(r[2] for r in rows) or 1
    for addr, ins, st, ex in rows:
        ln = mp.get(addr - base, "?")
        a = agg[ln]
        a[0] += st
        a[1] += ex
        a[2].add(ins.split()[0] if ins else "")
    print(f"{fn}  ({len(rows)} instrs, {tot:.0f} stall samples)")
    for ln, (st, ex, ops) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
        print(f"  {100 * st / tot:5.1f}%  exec={ex:9.0f}  {ln:18s} {' '.join(sorted(ops))[:70]}")


if __name__ == "__main__":
    main()
