"""Aggregate an ncu report's per-SASS metrics by CUDA source line.
usage: python scripts/ncu_lines.py report.ncu-rep <mangled kernel> <lib.so> [n_top]
Line info comes from nvdisasm -g on the cubin extracted from the .so (the
kernel must be built with -lineinfo)."""
import collections, csv, io, os, re, subprocess, sys, tempfile
rep, kern, so = sys.argv[1], sys.argv[2], sys.argv[3]
ntop = int(sys.argv[4]) if len(sys.argv) > 4 else 30
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=tmp, capture_output=True)
lines = {}
for cub in os.listdir(tmp):
    out = subprocess.run(["nvdisasm", "-g", os.path.join(tmp, cub)], capture_output=True, text=True).stdout
    sec = f".text.{kern}:"
    if sec not in out:
        continue
    body = out.split(sec, 1)[1].split("\n.L_x_")[0] if False else out.split(sec, 1)[1]
    cur = None
    for ln in body.splitlines():
        if ln.startswith("//---------------------") and ".text." in ln:
            break
        m = re.search(r'## File "([^"]+)", line (\d+)', ln)
        if m:
            cur = f"{os.path.basename(m.group(1))}:{m.group(2)}"
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", ln)
        if m:
            lines[int(m.group(1), 16)] = cur
    break
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass", "--kernel-name-base", "mangled", "-k", kern],
                     capture_output=True, text=True).stdout
if not src.strip():
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True).stdout
r = csv.reader(io.StringIO(src))
next(r); hdr = next(r)
rows = []
for x in r:  # first launch only (a report may hold several blocks)
    if x and x[0] == "Kernel Name":
        break
    rows.append(dict(zip(hdr, x)))
base = int(rows[0]["Address"], 16)
agg = collections.defaultdict(lambda: [0, 0, collections.Counter()])
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
for x in rows:
    off = int(x["Address"], 16) - base
    key = lines.get(off, "?")
    a = agg[key]
    a[0] += int(x["Warp Stall Sampling (All Samples)"] or 0)
    a[1] += int(x["Instructions Executed"] or 0)
    for c in stall_cols:
        a[2][c[6:]] += int(x[c] or 0)
ts = sum(a[0] for a in agg.values()) or 1
ti = sum(a[1] for a in agg.values()) or 1
print(f"total samples {ts}, warp-instructions {ti}")
print("by stall samples:")
for k, a in sorted(agg.items(), key=lambda kv: -kv[1][0])[:ntop]:
    top = ", ".join(f"{n}:{c}" for n, c in a[2].most_common(2))
    print(f"  {k:24s} samp {100*a[0]/ts:5.1f}%  instr {100*a[1]/ti:5.1f}%  {top}")
print("by instructions:")
for k, a in sorted(agg.items(), key=lambda kv: -kv[1][1])[:15]:
    print(f"  {k:24s} instr {100*a[1]/ti:5.1f}%  samp {100*a[0]/ts:5.1f}%")
