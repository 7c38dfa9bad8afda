"""Per-source-line warp instructions per unit (e.g. per root) and stall share.
usage: python scripts/ncu_perroot.py rep kernel so file units [n_top]"""
import contextlib, io, sys
rep, kern, so, fname, units = sys.argv[1:6]
ntop = int(sys.argv[6]) if len(sys.argv) > 6 else 40
units = float(units)
sys.argv = ["x", rep, kern, so, "100000"]
src = open(__file__.replace("ncu_perroot.py", "ncu_lines.py")).read().replace('print(f"total', 'AGG=agg\nprint(f"total')
g = {}
with contextlib.redirect_stdout(io.StringIO()):
    exec(compile(src, "ncu_lines", "exec"), g)
agg = g["AGG"]
code = {}
try:
    code = dict(enumerate(open(fname).read().split("\n"), 1))
except OSError:
    pass
ts = sum(a[0] for a in agg.values()) or 1
rows = []
for k, a in agg.items():
    f, _, l = k.partition(":")
    txt = code.get(int(l), "").strip()[:80] if l.isdigit() and fname.endswith(f) else ""
    rows.append((a[1] / units, 100 * a[0] / ts, k, txt))
print(f"warp-instructions per unit: {sum(r[0] for r in rows):.0f}")
for r in sorted(rows, reverse=True)[:ntop]:
    print(f"{r[0]:8.0f} {r[1]:5.1f}% {r[2]:30s} {r[3]}")
