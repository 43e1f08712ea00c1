"""Summarise `nvcc -Xptxas -v` output: registers / spills per kernel.
usage: python tools/ptxas_report.py csrc/file.cu [filter]"""
import re
import subprocess
import sys

src = sys.argv[1]
flt = sys.argv[2] if len(sys.argv) > 2 else ""
cmd = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "--expt-relaxed-constexpr",
       "-Xptxas", "-v", "-c", src, "-o", "/tmp/_ptxas.o"]
out = subprocess.run(cmd, capture_output=True, text=True).stderr
cur = None
rows = {}
for line in out.splitlines():
    m = re.search(r"Compiling entry function '(\w+)'", line)
    if m:
        cur = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
        rows[cur] = {}
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        rows[cur]["spill"] = int(m.group(1))
    m = re.search(r"Used (\d+) registers", line)
    if m:
        rows[cur]["regs"] = int(m.group(1))
for k, v in sorted(rows.items()):
    if flt in k:
        short = re.sub(r"nttb200::|fastk::", "", k)[:110]
        print(f"regs={v.get('regs', '?'):>4} spill={v.get('spill', '?'):>4}  {short}")
