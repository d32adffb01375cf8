"""Summarise ncu reports / launch lists into profiles/*.txt.

    python scripts/ncu_summary.py launches gpurun_out/launches.csv > profiles/rX_launch_summary.txt
    python scripts/ncu_summary.py full gpurun_out/prof.ncu-rep > profiles/rX_full_summary.txt
"""
import collections
import csv
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6,
             "ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6}
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in data:
        name = r[ki].split("(")[0].split("<")[0].replace("void ", "").strip()
        tot[name] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        cnt[name] += 1
    T = sum(tot.values())
    print(f"{'kernel':32s} {'launches':>8s} {'total us':>12s} {'share':>7s}")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{k:32s} {cnt[k]:8d} {v:12.1f} {100 * v / T:6.1f}%")


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    want = [
        "gpu__time_duration.sum", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__inst_executed.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    ]
    stall = [h for h in hdr if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        print("==", name[:90])
        for w in want:
            if w in hdr:
                print(f"   {w:64s} {r[hdr.index(w)]}")
        st = sorted(((float(r[hdr.index(h)] or 0), h) for h in stall), reverse=True)[:6]
        print("   top stalls: " + ", ".join(f"{h.split('stalled_')[1].split('_per')[0]}={v:.2f}" for v, h in st))


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
