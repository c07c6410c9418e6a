#!/usr/bin/env python
"""Per-source-line instruction and stall totals of one ncu capture (run here):

  python tools/ncu_lines.py REP [top]

Aggregates the interleaved CUDA/SASS source page (--print-source cuda,sass)
by (file, CUDA line): warp-instructions executed and stall samples."""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
inst, stall, text = defaultdict(int), defaultdict(int), {}
fname = "?"
cur = None
hdr = None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    if r[0]:   # a CUDA line row
        cur = (fname, int(r[0]))
        text[cur] = r[1].strip()[:90]
        continue
    d = dict(zip(hdr[2:], r[2:]))
    try:
        inst[cur] += int(d.get("Instructions Executed", "0") or 0)
        stall[cur] += int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
    except ValueError:
        pass
tot_i, tot_s = sum(inst.values()) or 1, sum(stall.values()) or 1
print(f"total warp-instructions {tot_i}, stall samples {tot_s}")
for k in sorted(inst, key=lambda k: -inst[k])[:top]:
    print(f"{inst[k]:>11} {100*inst[k]/tot_i:5.1f}%  stall {100*stall[k]/tot_s:5.1f}%  {k[0]}:{k[1]}  {text.get(k,'')}")
