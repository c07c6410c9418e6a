#!/usr/bin/env python
"""Stall / instruction breakdown of the TC tick kernel by code region, from an
ncu --set full report (SASS source page).  Regions: prologue+producer+MMA+spike
stage (before the epilogue's LDTM), epilogue head (LDTM .. LIF), LIF (.. last
I2IP), epilogue tail (routing, outputs, waits).

  python tools/ncu_regions.py gpurun_out/prof.ncu-rep [tiles]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
tiles = float(sys.argv[2]) if len(sys.argv) > 2 else 512 * 157
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
data = rows[2:]
si = h.index("Warp Stall Sampling (All Samples)")
ii = h.index("Instructions Executed")
cols = {c: k for k, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c}
tot = sum(float(r[si] or 0) for r in data)
ldtm = [k for k, r in enumerate(data) if "LDTM" in r[1]]
i2ip = [k for k, r in enumerate(data) if "I2IP" in r[1]]
cuts = [0, ldtm[0] - 40, ldtm[0] + 60, (i2ip[-1] + 1) if i2ip else ldtm[0] + 400, len(data)]
names = ["before epilogue", "epilogue head", "LIF", "epilogue tail + waits"]


def agg(a, b):
    s = {c: 0.0 for c in cols}
    for r in data[a:b]:
        for c, k in cols.items():
            s[c] += float(r[k] or 0)
    t = sum(s.values()) or 1.0
    ins = sum(float(r[ii] or 0) for r in data[a:b])
    top = {c[6:]: round(v / t * 100, 1) for c, v in sorted(s.items(), key=lambda x: -x[1]) if v / t > 0.03}
    return t, ins, top


for nm, a, b in zip(names, cuts[:-1], cuts[1:]):
    t, ins, top = agg(a, b)
    print(f"{nm:24s} stall samples {t / tot * 100:5.1f}%  warp-instr/tile {ins / tiles:7.0f}  {top}")
hot = sorted(range(len(data)), key=lambda k: -float(data[k][si] or 0))[:12]
print("hottest instructions:")
for k in hot:
    print(f"  {k:5d} {float(data[k][si]) / tot * 100:5.1f}%  {data[k][1].strip()[:80]}")
