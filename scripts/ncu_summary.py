"""Summarise an ncu capture of the propose-scan and phase-loop launches of one solve
(gpurun_out/prof_loop.ncu-rep from scripts/gpu_round.sh) into
profiles/ncu_summary.json and profiles/<tag>_ncu_phase_loop.txt."""
import csv
import io
import json
import os
import subprocess
import sys

tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
rep = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/prof_loop.ncu-rep"
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "lts__t_sector_hit_rate.pct", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size"]
out, lines = {}, []
for r in rows[2:]:
    name = "propose" if "propose_stream" in r[hdr.index("Kernel Name")] else "loop"

    def g(k):
        return float(r[hdr.index(k)].replace(",", ""))
    rd = g("dram__bytes_read.sum") * scale[units[hdr.index("dram__bytes_read.sum")]]
    wr = g("dram__bytes_write.sum") * scale[units[hdr.index("dram__bytes_write.sum")]]
    out[f"{name}_dram_bytes_per_launch"] = int(rd + wr)
    out[f"{name}_duration_ms"] = g("gpu__time_duration.sum") * (1e-3 if units[hdr.index("gpu__time_duration.sum")] == "us" else 1.0)
    lines.append(f"--- {name}: {r[hdr.index('Kernel Name')][:80]}")
    for k in want:
        if k in hdr:
            lines.append(f"  {k} = {r[hdr.index(k)]} {units[hdr.index(k)]}")
out["source"] = f"ncu --set full of scripts/profile_solve.py (config 2 seed 1), {rep}"
os.makedirs("profiles", exist_ok=True)
with open("profiles/ncu_summary.json", "w") as f:
    json.dump(out, f, indent=1)
with open(f"profiles/{tag}_ncu_phase_loop.txt", "w") as f:
    f.write("\n".join(lines) + "\n")
print("\n".join(lines))
print(out)
