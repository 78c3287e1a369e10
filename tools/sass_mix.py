#!/usr/bin/env python3
"""Opcode mix (executed warp instructions) of one kernel from an ncu report's source page.
usage: sass_mix.py report.ncu-rep kernel_regex"""
import collections, csv, io, subprocess, sys

rep, kre = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", f"regex:{kre}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = [i for i, r in enumerate(rows) if "Source" in r and "Address" in r][0]
h = rows[hi]
si, ei = h.index("Source"), h.index("Instructions Executed")
cnt = collections.Counter()
for r in rows[hi + 1:]:
    if len(r) <= ei:
        continue
    try:
        v = float(r[ei])
    except ValueError:
        continue
    toks = r[si].strip().split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") else toks[0]
    cnt[op.split(".")[0]] += v
tot = sum(cnt.values())
for k, v in cnt.most_common(int(sys.argv[3]) if len(sys.argv) > 3 else 25):
    print(f"{k:10s} {v:14.0f} {100 * v / tot:5.1f}%")
print("total", tot)
