"""Instructions executed per source-line range of one kernel (ncu source page + nvdisasm -g).
usage: sass_ranges.py SASS CSV SYM PAT name:lo-hi [name:lo-hi ...]   (other lines -> 'other')"""
import csv, re, sys, collections
sass_file, ncu_csv, sym, pat = sys.argv[1:5]
ranges = []
for a in sys.argv[5:]:
    nm, r = a.split(':'); lo, hi = map(int, r.split('-')); ranges.append((nm, lo, hi))
sass = open(sass_file).read().split('\n')
st = next(i for i, l in enumerate(sass) if l.startswith('.text.' + sym + ':'))
cur = None; seq = []
for l in sass[st + 1:]:
    if l.startswith('.text.'): break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m: cur = (m.group(1).split('/')[-1], int(m.group(2))); continue
    if re.search(r'/\*[0-9a-f]{4,}\*/', l): seq.append(cur)
rows = list(csv.reader(open(ncu_csv)))
blocks = []; curb = None
for r in rows:
    if r and r[0] == 'Kernel Name': curb = {'name': r[1], 'rows': []}; blocks.append(curb); continue
    if r and r[0] == 'Address': hdr = r; continue
    if curb is not None and len(r) > 5: curb['rows'].append(r)
b = next(b for b in blocks if re.search(pat, b['name']))
ie = hdr.index('Instructions Executed')
agg = collections.Counter()
for k, src in enumerate(seq[:len(b['rows'])]):
    n = int(b['rows'][k][ie] or 0)
    nm = 'other'
    if src and src[0] == 'k_query.cu':
        for (r_, lo, hi) in ranges:
            if lo <= src[1] <= hi: nm = r_; break
    agg[nm] += n
tot = sum(agg.values())
for nm, v in agg.most_common(): print(f'{nm:12s} {v/1e6:9.1f}M {100*v/tot:5.1f}%')
print(f'total {tot/1e6:.1f}M')
