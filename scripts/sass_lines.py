"""Print SASS of a kernel with source-line tags for an address range or around a source line.
usage: python scripts/sass_lines.py lib.so mangled [file:line] [before] [after]"""
import os, re, subprocess, sys, tempfile
so, kern = sys.argv[1], sys.argv[2]
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=tmp, capture_output=True)
out = []
for cub in sorted(os.listdir(tmp)):
    txt = subprocess.run(["nvdisasm", "-g", os.path.join(tmp, cub)], capture_output=True, text=True).stdout
    sec = f".text.{kern}:"
    if sec not in txt: continue
    body = txt.split(sec, 1)[1].split(".section", 1)[0]
    cur = None
    for ln in body.splitlines():
        m = re.search(r'## File "([^"]+)", line (\d+)', ln)
        if m: cur = f"{os.path.basename(m.group(1))}:{m.group(2)}"; continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
        if m: out.append((m.group(1), cur, m.group(2).strip()))
    break
if len(sys.argv) > 3:
    tag = sys.argv[3]; b = int(sys.argv[4]) if len(sys.argv) > 4 else 20; a = int(sys.argv[5]) if len(sys.argv) > 5 else 40
    idx = [i for i, x in enumerate(out) if x[1] == tag]
    i0 = idx[len(idx)//2] if idx else 0
    for x in out[max(0, i0-b):i0+a]: print(*x)
else:
    for x in out: print(*x)
