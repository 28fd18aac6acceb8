"""One line per kernel from an `ncu --page raw --csv` export: duration, instructions,
IPC, DRAM bytes, occupancy and the top warp-stall reasons.  Values are printed with
the unit ncu reports for them (second row of the export)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h, units = rows[0], rows[1]
U = {h[i]: units[i] for i in range(len(h))}
for r in rows[2:]:
    d = {h[i]: r[i] for i in range(len(h))}

    def g(k):
        return f"{d.get(k, '?')} {U.get(k, '')}".strip()

    st = [(k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''),
           float(v)) for k, v in d.items() if k.startswith('smsp__average_warps_issue_stalled_')
          and k.endswith('_per_issue_active.ratio') and v]
    st = sorted(st, key=lambda x: -x[1])[:6]
    print(f"{d['Kernel Name'][:48]} | time {g('gpu__time_duration.sum')} | warp inst "
          f"{g('smsp__inst_executed.sum')} | IPC {g('sm__inst_executed.avg.per_cycle_active')} | "
          f"DRAM read {g('dram__bytes_read.sum')} write {g('dram__bytes_write.sum')} | L2 hit "
          f"{g('lts__t_sector_hit_rate.pct')} | occupancy {g('sm__warps_active.avg.pct_of_peak_sustained_active')}"
          f" | threads/inst {g('smsp__thread_inst_executed_per_inst_executed.ratio')}")
    print('    stalls per issue:', [(a, round(b, 2)) for a, b in st])
