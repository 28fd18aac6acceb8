#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"^k_(query|heavy)$" -c 4 \
  -o $O/kq5 -f python scripts/prof_step.py --cfg 5 --reps 1 --order 0 > $O/kq5.log 2>&1
ncu -i $O/kq5.ncu-rep --page raw --csv > $O/kq5_raw.csv 2>/dev/null
