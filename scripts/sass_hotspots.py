"""Summarise an ncu source page (--page source --csv --print-source sass):
stall samples and executed instructions per opcode and per address window.
    ncu -i X.ncu-rep --page source --csv --print-source sass > x.csv
    python scripts/sass_hotspots.py x.csv
"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hdr_i]
ci = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows[hdr_i + 1:] if len(r) == len(hdr) and r[0].startswith("0x") or (len(r) == len(hdr) and r[0].isdigit())]
def num(r, k):
    try:
        return float(r[ci[k]].replace(",", ""))
    except Exception:
        return 0.0
S = "Warp Stall Sampling (All Samples)"
I = "Instructions Executed"
tot_s = sum(num(r, S) for r in data)
tot_i = sum(num(r, I) for r in data)
op = defaultdict(lambda: [0.0, 0.0])
for r in data:
    o = r[ci["Source"]].split()
    o = [x for x in o if not x.startswith("@")]
    name = o[0].split(".")[0] if o else "?"
    op[name][0] += num(r, S)
    op[name][1] += num(r, I)
print(f"total samples {tot_s:.0f}  instructions {tot_i:.3e}")
for k, v in sorted(op.items(), key=lambda kv: -kv[1][1])[:25]:
    print(f"  {k:10s} samples {100*v[0]/tot_s:5.1f}%  inst {100*v[1]/tot_i:5.1f}%")
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
print("stall reasons:", ", ".join(f"{h[6:]}={100*sum(num(r,h) for r in data)/tot_s:.1f}%" for h in sorted(stalls, key=lambda h: -sum(num(r, h) for r in data))[:8]))
# windows of 64 instructions
W = int(sys.argv[2]) if len(sys.argv) > 2 else 64
print(f"hot windows ({W} instr):")
win = []
for i in range(0, len(data), W):
    ch = data[i:i + W]
    win.append((sum(num(r, S) for r in ch), sum(num(r, I) for r in ch), i, ch[0][0]))
for s, n, i, a in sorted(win, reverse=True)[:12]:
    print(f"  idx {i:5d} addr {a}: samples {100*s/tot_s:5.1f}%  inst {100*n/tot_i:5.1f}%")
