"""Refresh profiles/k1_profile.json (the per-evaluation instruction and DRAM
counts bench.py's roofline uses) from an ncu --set full capture of K1:
    python scripts/update_k1_profile.py REPORT.ncu-rep CANDIDATES "source text"
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

rep, cand, source = sys.argv[1], int(sys.argv[2]), sys.argv[3]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                     check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]


def metric(name, scale_to=None):
    i = hdr.index(name)
    x = float(vals[i].replace(",", ""))
    u = units[i]
    if scale_to == "B":
        x *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]
    if scale_to == "ms":
        x *= {"ms": 1.0, "us": 1e-3, "usecond": 1e-3, "msecond": 1.0, "ns": 1e-6}[u]
    return x


inst = metric("smsp__inst_executed.sum")
rd = metric("dram__bytes_read.sum", "B")
wr = metric("dram__bytes_write.sum", "B")
out = {
    "source": source,
    "warp_inst_per_eval": round(inst / cand),
    "dram_bytes_per_eval": round((rd + wr) / cand, 1),
    "dram_bytes_read": int(rd),
    "dram_bytes_write": int(wr),
    "candidates": cand,
    "gpu_time_ms_cold": round(metric("gpu__time_duration.sum", "ms"), 3),
    "ipc": round(metric("sm__inst_executed.avg.per_cycle_active"), 3),
    "issue_active_pct": round(metric("smsp__issue_active.avg.pct_of_peak_sustained_active"), 1),
    "warps_active_per_sm": round(metric("sm__warps_active.avg.per_cycle_active"), 2),
    "registers": int(metric("launch__registers_per_thread")),
}
Path("profiles/k1_profile.json").write_text(json.dumps(out, indent=1) + "\n")
print(json.dumps(out, indent=1))
