#!/usr/bin/env python3
"""Hottest CUDA source lines of one kernel in an ncu report (warp-stall samples, top stall reasons).
usage: src_hot.py report.ncu-rep [kernel_regex] [top]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
kre = sys.argv[2] if len(sys.argv) > 2 else "."
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
by_inst = len(sys.argv) > 4 and sys.argv[4] == "inst"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", f"regex:{kre}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, fname, recs = None, "", []
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r and r[0] == "Line No":
        hdr = r
    elif hdr and len(r) == len(hdr) and r[2] == "-":
        d = dict(zip(hdr[4:], r[4:]))
        try:
            s = float(d["Warp Stall Sampling (All Samples)"])
        except (KeyError, ValueError):
            continue
        if s <= 0 and not by_inst:
            continue
        stalls = sorted(((float(v), k[6:]) for k, v in d.items() if k.startswith("stall_") and v not in ("", "-")),
                        reverse=True)[:3]
        recs.append((s, f"{fname}:{r[0]}", r[1].strip()[:70], float(d.get("Instructions Executed", 0) or 0), stalls))
tot = sum(x[0] for x in recs) or 1.0
itot = sum(x[3] for x in recs) or 1.0
key = (lambda x: x[3]) if by_inst else (lambda x: x[0])
for s, loc, src, ins, st in sorted(recs, key=key, reverse=True)[:top]:
    if by_inst:
        print(f"{100 * ins / itot:5.1f}% inst ", end="")
    print(f"{100 * s / tot:5.1f}% {loc:22s} inst={ins:10.0f} {' '.join(f'{k}:{v:.0f}' for v, k in st):40s} | {src}")
