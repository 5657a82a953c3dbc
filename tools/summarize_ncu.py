"""Summarise a gpurun session's ncu outputs into profiles/ (tracked).

python tools/summarize_ncu.py gpurun_out/<tag> profiles/<round>_<tag>
Writes <out>_launches.txt (per-kernel share of the ncu launch list) and
<out>_<report>.txt (key metrics of every .ncu-rep in the session dir).
"""
import collections
import csv
import glob
import io
import os
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__cycles_elapsed.avg.per_second",
    "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
]
STALLS = "smsp__average_warps_issue_stalled_"


def launches(path):
    rows = list(csv.reader(open(path)))
    i = [k for k, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[i]
    ki, mi, vi, ui = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    agg = collections.OrderedDict()
    for r in rows[i + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        v *= {"ms": 1e3, "ns": 1e-3, "s": 1e6}.get(r[ui], 1.0)
        name = r[ki].split("(")[0][:80]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(a[1] for a in agg.values())
    out = io.StringIO()
    out.write(f"# ncu launch list ({path}); cold-cache serialised times, compare SHARES\n")
    out.write(f"{'launches':>8} {'total_us':>12} {'share':>7} {'us/launch':>10}  kernel\n")
    for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.write(f"{c:8d} {t:12.1f} {100 * t / tot:6.1f}% {t / c:10.1f}  {n}\n")
    out.write(f"total_us {tot:.1f}\n")
    return out.getvalue()


def report(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) < 3:
        return f"(no data in {path})\n"
    hdr, units = rows[0], rows[1]
    out = io.StringIO()
    for li, vals in enumerate(rows[2:]):
        d = dict(zip(hdr, vals))
        u = dict(zip(hdr, units))
        out.write(f"# {os.path.basename(path)} launch {li}: {d.get('Kernel Name', '')[:100]}\n")
        for k in KEYS:
            if k in d:
                out.write(f"{k} = {d[k]} {u.get(k, '')}\n")
        st = sorted(((k, d[k]) for k in d if k.startswith(STALLS) and k.endswith("per_issue_active.ratio")),
                    key=lambda x: -float(x[1] or 0))
        out.write("stalls (warps per issue): " + ", ".join(
            f"{k[len(STALLS):].replace('_per_issue_active.ratio', '')}={float(v):.3f}" for k, v in st[:8]) + "\n")
    return out.getvalue()


def main():
    src, dst = sys.argv[1], sys.argv[2]
    os.makedirs(os.path.dirname(dst) or ".", exist_ok=True)
    lc = os.path.join(src, "launches.csv")
    if os.path.exists(lc):
        open(dst + "_launches.txt", "w").write(launches(lc))
    for rep in sorted(glob.glob(os.path.join(src, "*.ncu-rep"))):
        name = os.path.basename(rep)[:-8]
        open(f"{dst}_{name}.txt", "w").write(report(rep))


if __name__ == "__main__":
    main()
