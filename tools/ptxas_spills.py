"""Summarise ptxas -v output (paper_2601_22585_b200/ptxas_info.txt): registers and spills per function."""
import re
import subprocess
import sys

path = sys.argv[1] if len(sys.argv) > 1 else "paper_2601_22585_b200/ptxas_info.txt"
cur = None
rows = {}
for line in open(path):
    m = re.search(r"Function properties for (\S+)", line)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        rows.setdefault(cur, {}).update(stack=int(m.group(1)), st=int(m.group(2)), ld=int(m.group(3)))
        continue
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1)
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        rows.setdefault(cur, {})["regs"] = int(m.group(1))
names = list(rows)
dem = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.split("\n")
for n, d in zip(names, dem):
    r = rows[n]
    if r.get("st", 0) or r.get("ld", 0) or "-a" in sys.argv:
        print(f"{r.get('regs', '-'):>4} regs  spill st {r.get('st', 0):5d} ld {r.get('ld', 0):5d}  {d[:150]}")
