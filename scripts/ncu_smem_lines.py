"""Shared-memory wavefronts (actual vs ideal) per CUDA source line.
usage: python scripts/ncu_smem_lines.py report.ncu-rep <mangled kernel> <lib.so> [n_top]"""
import collections, csv, io, sys
sys.argv += [] 
rep, kern, so = sys.argv[1:4]
ntop = int(sys.argv[4]) if len(sys.argv) > 4 else 25
g = {}
src = open(__file__.replace("ncu_smem_lines.py", "ncu_lines.py")).read()
src = src.split("src = subprocess.run")[0]
exec(compile(src, "ncu_lines", "exec"), g)
lines = g["lines"]
import subprocess
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
r = csv.reader(io.StringIO(out)); next(r); hdr = next(r)
rows = [dict(zip(hdr, x)) for x in r]
base = int(rows[0]["Address"], 16)
agg = collections.defaultdict(lambda: [0, 0, 0])
for x in rows:
    k = lines.get(int(x["Address"], 16) - base, "?")
    f = lambda c: int(x[c]) if x[c] not in ("", "-") else 0
    agg[k][0] += f("L1 Wavefronts Shared"); agg[k][1] += f("L1 Wavefronts Shared Ideal"); agg[k][2] += f("Instructions Executed")
tot = sum(a[0] for a in agg.values()) or 1
print(f"shared wavefronts {tot}")
for k, a in sorted(agg.items(), key=lambda kv: -kv[1][0])[:ntop]:
    print(f"  {k:28s} wf {100*a[0]/tot:5.1f}%  {a[0]:>11d}  ideal {a[1]:>11d}  instr {a[2]:>11d}")
