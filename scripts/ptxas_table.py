"""Summarise an nvcc -Xptxas -v log: kernel -> registers, spill bytes."""
import re
import sys

cur = None
rows = {}
for line in open(sys.argv[1]):
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        rows.setdefault(cur, {})["spill"] = (int(m.group(1)), int(m.group(2)))
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        rows.setdefault(cur, {})["regs"] = int(m.group(1))
pat = sys.argv[2] if len(sys.argv) > 2 else ""
for k, v in sorted(rows.items()):
    if pat in k:
        dm = __import__("subprocess").run(["c++filt", k], capture_output=True, text=True).stdout.strip()
        print(f"{v.get('regs', '?'):>4} {str(v.get('spill')):>12}  {dm[:110]}")
