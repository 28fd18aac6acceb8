#!/bin/bash
# ncu --set full of the non-query kernels (sort, index) and the query kernels at config 3, order $ORDER.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"^k_(rs_onesweep|rs_hist_all|gather|query|sample)$" -c 12 \
  -o $O/misc_cfg3 -f python scripts/prof_step.py --cfg 3 --reps 1 --order ${ORDER:-1} > $O/misc.log 2>&1
ncu -i $O/misc_cfg3.ncu-rep --page raw --csv > $O/misc_raw.csv 2>/dev/null
ncu -i $O/misc_cfg3.ncu-rep --page source --csv --print-source sass > $O/misc_src.csv 2>/dev/null
echo done
