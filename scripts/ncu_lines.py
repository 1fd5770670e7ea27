"""Attribute an ncu --set full capture's per-instruction counts and stall
samples to source lines (nvdisasm -g line table of the in-tree library).
    python scripts/ncu_lines.py REPORT.ncu-rep KERNEL_SUBSTRING CUBIN_STEM [top]
KERNEL_SUBSTRING must pick the profiled instantiation out of the cubin (a
piece of its mangled name, e.g. makespan_kernelIsLb1ELi0ELb0ELb1ELb1ELi6ELi0E):
another instantiation of the same template has another address map."""
import collections
import csv
import io
import re
import subprocess
import sys
import tempfile
from pathlib import Path

rep, kname, stem = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                      capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(sass)))
hdr = rows[1]
data = rows[2:]
ii, ist, ia = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Address")
tmp = Path(tempfile.mkdtemp())
subprocess.run(["cuobjdump", "-xelf", "all", str(Path("paper_2602_23685_b200/lib/libvrprpd.so").resolve())],
               cwd=tmp, capture_output=True)
cub = next(tmp.glob(f"{stem}.sm_100a.cubin"))
dis = subprocess.run(["nvdisasm", "-g", "-c", str(cub)], capture_output=True, text=True).stdout.splitlines()
start = next(i for i, l in enumerate(dis) if kname in l and l.startswith(".text."))
cur, a2l = None, {}
for l in dis[start + 1:]:
    if l.startswith(".text.") or l.strip().startswith(".section"):
        if a2l:
            break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
    m2 = re.match(r'\s*/\*([0-9a-f]{4,})\*/', l)
    if m2 and cur:
        a2l[int(m2.group(1), 16)] = cur
base = int(data[0][ia], 16)
inst, st = collections.Counter(), collections.Counter()
for r in data:
    k = a2l.get(int(r[ia], 16) - base, ("?", 0))
    inst[k] += int(r[ii])
    st[k] += int(r[ist])
ti, ts = sum(inst.values()), sum(st.values())
print(f"total warp instructions {ti:.3e}, stall samples {ts}")
for k, c in st.most_common(top):
    print(f"{k[0]}:{k[1]:<5d} stall {100 * c / ts:5.1f}%  inst {100 * inst[k] / ti:5.1f}%")
