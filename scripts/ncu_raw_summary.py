"""One line per kernel from an `ncu --page raw --csv` export: duration, instructions,
IPC, DRAM bytes, occupancy and the top warp-stall reasons."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = rows[0]
for r in rows[2:]:
    d = {h[i]: r[i] for i in range(len(h))}
    g = lambda k: d.get(k, '?')
    st = [(k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''), float(v))
          for k, v in d.items() if k.startswith('smsp__average_warps_issue_stalled_')
          and k.endswith('_per_issue_active.ratio') and v]
    st = sorted(st, key=lambda x: -x[1])[:6]
    print(f"{d['Kernel Name'][:40]} dur_us {g('gpu__time_duration.sum')} inst {g('smsp__inst_executed.sum')} "
          f"ipc {g('sm__inst_executed.avg.per_cycle_active')} dramR {g('dram__bytes_read.sum')} "
          f"dramW {g('dram__bytes_write.sum')} occ% {g('sm__warps_active.avg.pct_of_peak_sustained_active')}")
    print('    stalls/issue', [(a, round(b, 2)) for a, b in st])
