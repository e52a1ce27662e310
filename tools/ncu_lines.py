"""Per-source-line executed instructions and stall samples of one kernel in an ncu report.
usage: python tools/ncu_lines.py REPORT.ncu-rep OBJ.o KERNEL_SUBSTR SOURCE.cu [N]"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

rep, obj, kname, srcf = sys.argv[1:5]
top = int(sys.argv[5]) if len(sys.argv) > 5 else 25
sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                      capture_output=True, text=True).stdout
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, capture_output=True)
cub = [os.path.join(tmp, f) for f in os.listdir(tmp) if f.endswith(".cubin")][0]
lines = subprocess.run(["nvdisasm", "--print-line-info", cub], capture_output=True, text=True).stdout
addr2, cur, fn = {}, None, None
for line in lines.split("\n"):
    m = re.match(r"\s*\.section\s+\.text\.(\S+),", line)
    if m:
        fn, cur = m.group(1), None
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', line)
    if m:
        cur = int(m.group(2))
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m and fn and kname in fn:
        addr2[int(m.group(1), 16)] = cur
rows = list(csv.reader(io.StringIO(sass)))
hdr = next(r for r in rows if r and r[0] == "Address")
ia, ie = hdr.index("Address"), hdr.index("Instructions Executed")
iss = hdr.index("Warp Stall Sampling (All Samples)")
base, byline, st, tot, stot = None, collections.Counter(), collections.Counter(), 0.0, 0.0
for r in rows:
    if len(r) != len(hdr):
        continue
    try:
        a = int(r[ia], 16)
    except ValueError:
        continue
    base = a if base is None else base
    ex, s = float(r[ie] or 0), float(r[iss] or 0)
    ln = addr2.get(a - base)
    byline[ln] += ex
    st[ln] += s
    tot += ex
    stot += s
src = open(srcf).read().split("\n")
print(f"total executed warp instructions {tot:.0f}, stall samples {stot:.0f}")
for ln, c in byline.most_common(top):
    txt = src[ln - 1].strip()[:80] if ln else ""
    print(f"{c / tot * 100:5.1f}% instr {st[ln] / max(1, stot) * 100:5.1f}% stall  L{ln}: {txt}")
