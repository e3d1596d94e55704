"""Summarise an ncu report: headline metrics, top stall reasons, hottest source lines."""
import csv
import io
import subprocess
import sys


def page(rep, name):
    out = subprocess.run(["ncu", "-i", rep, "--page", name, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main(rep, nlines=25):
    raw = page(rep, "raw")
    h, v = raw[0], raw[2]
    d = dict(zip(h, v))
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
            "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
            "lts__t_sector_hit_rate.pct"]
    for k in keys:
        if k in d:
            print(f"  {k:60s} {d[k]} {raw[1][h.index(k)]}")
    st = [(float(d[k]), k) for k in h if k.startswith("smsp__average_warps_issue_stalled") and
          k.endswith("_per_issue_active.ratio") and d[k] not in ("", "n/a")]
    print("  stalls:", ", ".join(f"{k.split('stalled_')[1].split('_per')[0]}={x:.2f}" for x, k in sorted(st, reverse=True)[:8]))
    src = page(rep, "source")
    if not src:
        return
    hdr = src[0]
    try:
        li = hdr.index("Source")
        si = next(i for i, x in enumerate(hdr) if x.startswith("Warp Stall Sampling (All"))
        ii = hdr.index("Instructions Executed") if "Instructions Executed" in hdr else None
    except (ValueError, StopIteration):
        print("  (no source page)")
        return
    rows = []
    for r in src[1:]:
        try:
            rows.append((float(r[si] or 0), float(r[ii] or 0) if ii is not None else 0, r[0], r[li][:110]))
        except (ValueError, IndexError):
            pass
    tot = sum(x[0] for x in rows) or 1
    print("  hottest lines (stall samples %, inst executed):")
    for s, n, ln, code in sorted(rows, reverse=True)[:nlines]:
        print(f"   {100 * s / tot:5.1f}% {n:10.0f}  L{ln}: {code.strip()}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
