"""Join an ncu SASS-level source page (csv) with nvdisasm -g line info:
per-source-line instruction executions and stall samples for one kernel."""
import csv, re, sys, collections
sass_file, ncu_csv, kernel_sym, kernel_pat = sys.argv[1:5]  # [top-N]
lines = open(sass_file).read().split('\n')
start = next(i for i, l in enumerate(lines) if l.startswith('.text.' + kernel_sym + ':'))
cur = None; seq = []
for l in lines[start + 1:]:
    if l.startswith('.text.'): break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m: cur = (m.group(1).split('/')[-1], int(m.group(2))); continue
    if re.search(r'/\*[0-9a-f]{4,}\*/', l): seq.append((cur, l.strip()))
rows = list(csv.reader(open(ncu_csv)))
blocks = []; curb = None
for r in rows:
    if r and r[0] == 'Kernel Name': curb = {'name': r[1], 'rows': []}; blocks.append(curb); continue
    if r and r[0] == 'Address': hdr = r; continue
    if curb is not None and len(r) > 5: curb['rows'].append(r)
b = next(b for b in blocks if re.search(kernel_pat, b['name']))
ie = hdr.index('Instructions Executed'); ss = hdr.index('Warp Stall Sampling (All Samples)')
n = min(len(seq), len(b['rows']))
print('sass instrs', len(seq), 'ncu instrs', len(b['rows']))
agg = collections.Counter(); st = collections.Counter()
for k in range(n):
    src = seq[k][0]
    agg[src] += int(b['rows'][k][ie] or 0); st[src] += int(b['rows'][k][ss] or 0)
tot = sum(agg.values()); tst = sum(st.values())
for src, v in sorted(agg.items(), key=lambda x: -x[1])[:int(sys.argv[5]) if len(sys.argv) > 5 else 40]:
    print(f'{src}  exec {100*v/tot:5.1f}%  stall {100*st[src]/tst:5.1f}%')
