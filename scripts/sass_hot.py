"""Per-instruction execution counts of one kernel: joins `nvdisasm -g` SASS with an
ncu source-page csv (--print-source sass).  Prints instructions executed at least
MIN times (default 1e7), with their source line and stall share."""
import csv, re, sys
sass_file, ncu_csv, sym, pat = sys.argv[1:5]
mn = float(sys.argv[5]) if len(sys.argv) > 5 else 1e7
sass = open(sass_file).read().split('\n')
st = next(i for i, l in enumerate(sass) if l.startswith('.text.' + sym + ':'))
cur = None; seq = []
for l in sass[st + 1:]:
    if l.startswith('.text.'): break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m: cur = int(m.group(2)); continue
    if re.search(r'/\*[0-9a-f]{4,}\*/', l): seq.append((cur, l.strip()))
rows = list(csv.reader(open(ncu_csv)))
blocks = []; curb = None
for r in rows:
    if r and r[0] == 'Kernel Name': curb = {'name': r[1], 'rows': []}; blocks.append(curb); continue
    if r and r[0] == 'Address': hdr = r; continue
    if curb is not None and len(r) > 5: curb['rows'].append(r)
b = next(b for b in blocks if re.search(pat, b['name']))
ie = hdr.index('Instructions Executed'); ss = hdr.index('Warp Stall Sampling (All Samples)')
assert len(seq) == len(b['rows']), (len(seq), len(b['rows']))
tot = sum(int(r[ie] or 0) for r in b['rows']); tst = sum(int(r[ss] or 0) for r in b['rows'])
print(f"total {tot/1e6:.1f}M instructions")
for k, (ln, ins) in enumerate(seq):
    n = int(b['rows'][k][ie] or 0); s_ = int(b['rows'][k][ss] or 0)
    if n >= mn:
        ins = re.sub(r'/\*[0-9a-f]+\*/', '', ins).strip()
        print(f"{n/1e6:7.1f}M st{100*s_/tst:5.1f}% L{ln} {ins[:84]}")
