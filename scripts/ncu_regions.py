"""Instruction/stall share per source-line range of a kernel.
usage: python scripts/ncu_regions.py rep kernel so file:lo-hi=name ..."""
import collections, sys
rep, kern, so = sys.argv[1:4]
ranges = []
for a in sys.argv[4:]:
    loc, name = a.split("=")
    f, rng = loc.split(":")
    lo, hi = (int(x) for x in rng.split("-"))
    ranges.append((f, lo, hi, name))
sys.argv = ["x", rep, kern, so, "100000"]
import io, contextlib
g = {}
src = open(__file__.replace("ncu_regions.py", "ncu_lines.py")).read().replace('print(f"total', 'AGG=agg\nprint(f"total')
with contextlib.redirect_stdout(io.StringIO()):
    exec(compile(src, "ncu_lines", "exec"), g)
agg = g["AGG"]
ti = sum(a[1] for a in agg.values()) or 1
ts = sum(a[0] for a in agg.values()) or 1
reg = collections.defaultdict(lambda: [0, 0])
for k, a in agg.items():
    f, _, l = k.partition(":")
    l = int(l) if l.isdigit() else -1
    name = next((n for (ff, lo, hi, n) in ranges if ff == f and lo <= l <= hi), f)
    reg[name][0] += a[1]
    reg[name][1] += a[0]
print(f"warp-instructions {ti}")
for n, (c, s_) in sorted(reg.items(), key=lambda kv: -kv[1][0]):
    print(f"  {n:32s} instr {100*c/ti:5.1f}%   stall-samples {100*s_/ts:5.1f}%")
