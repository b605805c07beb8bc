"""SASS instructions attributed to given CUDA source lines of an ncu capture, with their execution
counts (ncu --page source --print-source cuda,sass).
usage: python tools/ncu_sass_lines.py REPORT.ncu-rep LINE [LINE ...]"""
import csv
import io
import subprocess
import sys

rep, lines = sys.argv[1], set(sys.argv[2:])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur = None
for r in csv.reader(io.StringIO(out)):
    if len(r) < 8 or r[0] == "Line No":
        continue
    if r[0]:
        cur = r[0]
        if cur in lines:
            print(f"== {cur}: {r[1].strip()[:100]}  inst {r[7]}")
        continue
    if cur in lines and r[2] != "...":
        print(f"   {r[2][-5:]} {r[3].strip():60s} inst {r[7]:>12} stall {r[4]}")
