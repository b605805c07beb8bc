"""Summarise an ncu source page per CUDA source line: instructions executed and stall samples.
usage: python tools/ncu_lines.py REPORT.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, data, fname = None, [], ""
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    if len(r) > 3 and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) >= 8 and r[0] not in ("",):
        data.append((fname, r[0], r[1], r))
def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0
ii, si = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
tot_i = sum(num(r[ii]) for *_, r in data)
tot_s = sum(num(r[si]) for *_, r in data)
print(f"total inst {tot_i:.4g}  samples {tot_s:.4g}")
data.sort(key=lambda d: -num(d[3][si]))
for f, ln, src, r in data[:top]:
    print(f"{f[:10]}:{ln:>4} inst {100*num(r[ii])/tot_i:5.1f}% stall {100*num(r[si])/tot_s:5.1f}%  {src.strip()[:80]}")
