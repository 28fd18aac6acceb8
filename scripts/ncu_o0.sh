#!/bin/bash
# ncu --set full of the query kernels at config 3, vertex_order 0.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_(query|heavy)$" -c 4 \
  -o $O/kq_o0 -f python scripts/prof_step.py --cfg 3 --reps 1 --order 0 > $O/kq_o0.log 2>&1
ncu -i $O/kq_o0.ncu-rep --page raw --csv > $O/kq_o0_raw.csv 2>/dev/null
ncu -i $O/kq_o0.ncu-rep --page source --csv --print-source sass > $O/kq_o0_src.csv 2>/dev/null
