#!/bin/bash
# ncu --set full of the light query kernels (count + emit, one call) at CFG (default 3),
# ORDER (default 0); exports raw + source CSVs for scripts/src_groups.py.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out; T=${TAG:-kq}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_(query|heavy)$" -c 4 \
  -o $O/$T -f python scripts/prof_step.py --cfg ${CFG:-3} --reps 1 --order ${ORDER:-0} > $O/$T.log 2>&1
ncu -i $O/$T.ncu-rep --page raw --csv > $O/${T}_raw.csv 2>/dev/null
ncu -i $O/$T.ncu-rep --page source --csv --print-source sass > $O/${T}_src.csv 2>/dev/null
rm -f $O/$T.ncu-rep
python scripts/ncu_raw_summary.py $O/${T}_raw.csv 2>/dev/null | head -20
