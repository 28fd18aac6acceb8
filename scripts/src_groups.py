"""Instruction / stall share per source-line group of one kernel from an ncu source
export (--page source --csv) and the matching SASS with line info (nvdisasm -g -c).
usage: src_groups.py SASS CSV SYM NAMEPAT name:lo-hi[,lo-hi] ..."""
import collections
import csv
import re
import sys

sass_file, ncu_csv, sym, pat = sys.argv[1:5]
groups = []
for a in sys.argv[5:]:
    nm, spec = a.split(':')
    s = set()
    for part in spec.split(','):
        lo, hi = map(int, part.split('-'))
        s |= set(range(lo, hi + 1))
    groups.append((nm, s))
sass = open(sass_file).read().split('\n')
st = next(i for i, l in enumerate(sass) if l.startswith('.text.' + sym + ':'))
cur, seq = None, []
for l in sass[st + 1:]:
    if l.startswith('.text.'):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split('/')[-1], int(m.group(2)))
        continue
    if re.search(r'/\*[0-9a-f]{4,}\*/\s+\S', l):
        seq.append(cur)
rows = list(csv.reader(open(ncu_csv)))
blocks, curb, hdr = [], None, None
for r in rows:
    if r and r[0] == 'Kernel Name':
        curb = {'name': r[1], 'rows': []}
        blocks.append(curb)
        continue
    if r and r[0] == 'Address':
        hdr = r
        continue
    if curb is not None and len(r) > 5:
        curb['rows'].append(r)
b = next(b for b in blocks if pat in b['name'])
assert len(b['rows']) == len(seq), (len(b['rows']), len(seq))
ie, te = hdr.index('Instructions Executed'), hdr.index('Predicated-On Thread Instructions Executed')
ss = hdr.index('Warp Stall Sampling (All Samples)')
agg, th, stl = collections.Counter(), collections.Counter(), collections.Counter()
for k, src in enumerate(seq):
    g = 'other'
    if src and src[0].endswith('.cu'):
        for nm, s in groups:
            if src[1] in s:
                g = nm
                break
    r = b['rows'][k]
    agg[g] += int(r[ie] or 0)
    th[g] += int(r[te] or 0)
    stl[g] += int(r[ss] or 0)
tot, ts = sum(agg.values()), max(sum(stl.values()), 1)
for g, v in agg.most_common():
    print(f"{g:14s} {v / 1e6:8.0f}M inst {100 * v / tot:5.1f}%  active lanes/inst "
          f"{th[g] / max(v, 1):5.1f}  stall samples {100 * stl[g] / ts:5.1f}%")
print(f"total {tot / 1e6:.0f}M warp instructions")
