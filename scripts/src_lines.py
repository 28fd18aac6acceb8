"""Warp instructions executed (and stall samples) per source line of one kernel: an ncu
source export (--page source --csv --print-source sass) joined with `nvdisasm -g -c`
of the object that ran.  usage: src_lines.py OBJ CSV SYM KERNEL_SUBSTR [TOP]"""
import collections
import csv
import re
import subprocess
import sys

obj, ncu_csv, sym, pat = sys.argv[1:5]
top = int(sys.argv[5]) if len(sys.argv) > 5 else 40
dis = subprocess.run(["cuobjdump", "-xelf", "all", __import__("os").path.abspath(obj)], capture_output=True, text=True, cwd="/tmp")
cubins = [l.split()[-1] for l in (dis.stdout + dis.stderr).split("\n") if l.strip().endswith(".cubin")]
sass = subprocess.run(["nvdisasm", "-g", "-c", "/tmp/" + cubins[0]], capture_output=True,
                      text=True).stdout.split('\n')
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
blocks, curb = [], None
for r in rows:
    if r and r[0] == 'Kernel Name':
        curb = [r[1], []]
        blocks.append(curb)
    elif curb is not None and r and r[0].startswith('0x'):
        curb[1].append(r)
hdr = next(r for r in rows if r and r[0] == 'Address')
iE, iS = hdr.index('Instructions Executed'), hdr.index('Warp Stall Sampling (All Samples)')
name, ins = next(b for b in blocks if pat in b[0])
assert len(ins) == len(seq), (len(ins), len(seq))
agg = collections.Counter()
stl = collections.Counter()
for r, ln in zip(ins, seq):
    agg[ln] += int(r[iE] or 0)
    stl[ln] += int(r[iS] or 0)
tot, tst = sum(agg.values()), sum(stl.values())
print(name, f"total warp inst {tot:.3e}")
for ln, v in agg.most_common(top):
    print(f"{ln[0]}:{ln[1]:5d}  inst {v / tot * 100:5.1f}%  stall {stl[ln] / max(tst, 1) * 100:5.1f}%")
if len(sys.argv) > 6:  # dump instructions of source lines lo-hi with their counts
    lo, hi = map(int, sys.argv[6].split('-'))
    iA = hdr.index('Avg. Threads Executed')
    for r, ln in zip(ins, seq):
        if ln and lo <= ln[1] <= hi and ln[0] == 'k_query.cu':
            print(f"{ln[1]:5d} {int(r[iE] or 0):>11d} thr {r[iA]:>6s}  {r[1].strip()[:70]}")
