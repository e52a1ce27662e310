"""Attribute ncu warp-stall samples of k_search (ncu --page source --csv --print-source sass)
to source lines / functions using the cubin's line table (nvdisasm --print-line-info)."""
import collections
import csv
import re
import sys

sass_csv, line_dump = sys.argv[1], sys.argv[2]
KNAME = sys.argv[3] if len(sys.argv) > 3 else 'k_search'
src = {}
for f in ['search_core.cuh', 'search_warp.cuh', 'engine.cu', 'search_kernel.cuh']:
    lines = open('paper_2605_18710_b200/csrc/' + f).read().split('\n')
    cur, m = '?', []
    for l in lines:
        if re.match(r'^(__device__|MG_HD|MG_COLD|__global__|MG_HX|inline|static|double|bool|int|void)', l) and '(' in l:
            n = [x for x in re.findall(r'(\w+)\s*\(', l) if x not in ('__launch_bounds__', 'alignas')]
            if n:
                cur = n[0]
        m.append(cur)
    src[f] = m
addr2, ops, cur, fnm = {}, {}, None, None
for line in open(line_dump):
    m = re.match(r'\s*\.section\s+\.text\.(\S+),', line)
    if m:
        fnm, cur = m.group(1), None
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', line)
    if m:
        cur = (m.group(1).split('/')[-1], int(m.group(2)))
        continue
    m = re.match(r'\s+/\*([0-9a-f]{4,})\*/\s+(.*?);', line)
    if m and fnm and KNAME in fnm:
        addr2[int(m.group(1), 16)] = cur
        ops[int(m.group(1), 16)] = m.group(2).split()[0] if m.group(2).split() else ''
rows = list(csv.reader(open(sass_csv)))
hdr = next(r for r in rows if r and r[0] == 'Address')
ia, iss, isrc = hdr.index('Address'), hdr.index('Warp Stall Sampling (All Samples)'), hdr.index('Source')
base = int(next(r for r in rows if r and r[0].startswith('0x'))[ia], 16)
byline, byfn, tot, bad = collections.Counter(), collections.Counter(), 0.0, 0
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    a = int(r[ia], 16) - base
    s = float(r[iss] or 0)
    tot += s
    k = addr2.get(a)
    if k is None:
        continue
    if ops.get(a, '') != (r[isrc].split() or [''])[0].rstrip(';'):
        bad += 1
    f, l = k
    byline[(f, l)] += s
    byfn[f + ':' + (src[f][l - 1] if f in src else '')] += s
print(f'samples {tot:.0f}, opcode mismatches {bad}')
for k, n in byfn.most_common(20):
    print(f'{100 * n / tot:5.1f}% {k}')
print()
for (f, l), n in byline.most_common(30):
    print(f'{100 * n / tot:5.1f}% {f}:{l}')
