#!/usr/bin/env python3
"""Summarise an ncu --set full capture of one K1 apply (the three launches) into
profiles/<name>.md and profiles/k1_traffic.json (read by bench.py for roofline.traffic).

usage: k1_summary.py report.ncu-rep name "command line" [kernel_regex]
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
METRICS = [
    ("gpu__time_duration.sum", "us"),
    ("dram__bytes_read.sum", "byte"),
    ("dram__bytes_write.sum", "byte"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "%"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "%"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "%"),
    ("smsp__inst_executed.sum", "inst"),
    ("launch__registers_per_thread", ""),
    ("launch__block_size", ""),
    ("launch__grid_size", ""),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", ""),
    ("lts__t_sector_hit_rate.pct", "%"),
]
SCALE = {"us": {"usecond": 1, "msecond": 1e3, "nsecond": 1e-3},
         "byte": {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}}


def main():
    rep, name, cmd = sys.argv[1], sys.argv[2], sys.argv[3]
    kre = sys.argv[4] if len(sys.argv) > 4 else "k_(rowfwd|colpass|colnormal|rowinv)"
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "-k", f"regex:{kre}"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    kernels = []
    for r in rows[2:]:
        d = {"name": r[hdr.index("Kernel Name")].split("(")[0].replace("void <unnamed>::", "")}
        for m, kind in METRICS:
            if m not in hdr:
                continue
            i = hdr.index(m)
            v = float(r[i].replace(",", ""))
            v *= SCALE.get(kind, {}).get(units[i], 1.0)
            d[m] = v
        kernels.append(d)
    lines = [f"# K1 three-pass schedule, one config-1 apply -- ncu --set full ({name})", "",
             f"Command: `{cmd}`", f"Report: gpurun_out/{Path(rep).name} (cold-cache, serialised launches: compare shares).", "",
             "| metric | " + " | ".join(k["name"] for k in kernels) + " |",
             "|---|" + "---|" * len(kernels)]
    for m, kind in METRICS:
        if m in kernels[0]:
            lines.append(f"| {m} ({kind}) | " + " | ".join(f"{k[m]:.6g}" for k in kernels) + " |")
    rd = sum(k["dram__bytes_read.sum"] for k in kernels)
    wr = sum(k["dram__bytes_write.sum"] for k in kernels)
    t = sum(k["gpu__time_duration.sum"] for k in kernels)
    inst = sum(k["smsp__inst_executed.sum"] for k in kernels)
    lines += ["", f"Per apply: DRAM read {rd / 1e9:.3f} GB + write {wr / 1e9:.3f} GB = {(rd + wr) / 1e9:.3f} GB "
              f"(algorithmic 0.735 GB); {inst / 1e6:.1f} M warp instructions; sum of launch times {t:.1f} us."]
    (ROOT / "profiles" / f"{name}.md").write_text("\n".join(lines) + "\n")
    (ROOT / "profiles" / "k1_traffic.json").write_text(json.dumps({
        "kernel": "K1 three-pass (" + " + ".join(k["name"] for k in kernels) + "), one config-1 apply",
        "dram_read_bytes": rd, "dram_write_bytes": wr, "traffic_bytes": rd + wr,
        "warp_instructions": inst, "sum_launch_us": t,
        "per_kernel": kernels, "source": f"profiles/{name}.md"}, indent=1) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
