"""Top SASS instructions by warp-stall samples from an .ncu-rep, with the stall
reason columns that dominate.  usage: python tools/ncu_hot_lines.py report.ncu-rep [N]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rd = list(csv.reader(io.StringIO(out)))
k = next(i for i, r in enumerate(rd) if r and r[0] == "Address")
hdr, body = rd[k], rd[k + 1:]
i_s = hdr.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") or "Stall" in h and i != i_s]
rows = []
for idx, r in enumerate(body):
    if len(r) > i_s and r[i_s].isdigit() and int(r[i_s]) > 0:
        rows.append((int(r[i_s]), idx, r[1].strip()))
tot = sum(x[0] for x in rows) or 1
print(f"total samples {tot}")
for s, idx, src in sorted(rows, reverse=True)[:n]:
    print(f"{100 * s / tot:5.1f}%  #{idx:5d}  {src[:90]}")
