"""Summarise an ncu report: key SOL metrics + top SASS stall sites.
usage: python scripts/ncu_summary.py report.ncu-rep [n_top]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 25
def run(args):
    return subprocess.run(["ncu", "-i", rep] + args, capture_output=True, text=True).stdout
want = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput",
        "Compute (SM) Throughput", "Executed Ipc Active", "Issued Instructions", "Registers Per Thread",
        "Achieved Occupancy", "Theoretical Occupancy", "Eligible Warps Per Scheduler", "No Eligible",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp",
        "Dynamic Shared Memory Per Block", "Grid Size", "Block Size"]
r = csv.reader(io.StringIO(run(["--page", "details", "--csv"])))
hdr = next(r)
cur = None
for row in r:
    d = dict(zip(hdr, row))
    k = (d.get("ID"), d.get("Kernel Name"))
    if k != cur and d.get("Kernel Name"):
        cur = k
        print(f"== [{d.get('ID')}] {d.get('Kernel Name')[:100]}")
    if d.get("Metric Name") in want:
        print(f"  {d['Metric Name']:40s} {d['Metric Value']:>16s} {d['Metric Unit']}")
raw = run(["--page", "raw", "--csv"])
rr = list(csv.reader(io.StringIO(raw)))
if len(rr) >= 3:
    h, units, vals = rr[0], rr[1], rr[2]
    for key in ["dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum", "gpu__time_duration.sum"]:
        if key in h:
            i = h.index(key)
            print(f"  {key:40s} {vals[i]:>16s} {units[i]}")
src = run(["--page", "source", "--csv", "--print-source=sass"])
r = csv.reader(io.StringIO(src))
next(r); hdr = next(r)
rows = [dict(zip(hdr, x)) for x in r]
tot = sum(int(x["Warp Stall Sampling (All Samples)"] or 0) for x in rows) or 1
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
print(f"  samples {tot}  executed {sum(int(x['Instructions Executed'] or 0) for x in rows)}")
for x in sorted(rows, key=lambda x: -int(x["Warp Stall Sampling (All Samples)"] or 0))[:ntop]:
    s = int(x["Warp Stall Sampling (All Samples)"] or 0)
    top = sorted(((int(x[c] or 0), c[6:]) for c in stall_cols), reverse=True)[:2]
    print(f"  {x['Address'][-5:]} {100*s/tot:5.2f}% {x['Instructions Executed']:>10s}  {x['Source'].strip()[:58]:58s} {top}")
