#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_rs_onesweep$" -c 2 \
  -o $O/rs -f python scripts/prof_step.py --cfg 3 --reps 1 > $O/rs.log 2>&1
ncu -i $O/rs.ncu-rep --page raw --csv > $O/rs_raw.csv 2>/dev/null
ncu -i $O/rs.ncu-rep --page source --csv --print-source sass > $O/rs_src.csv 2>/dev/null
