#!/bin/bash
# vertex_order experiment: GPU tests, phases for both orders, launch list + ncu of the emit.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
rm -f $O/phases.log
for c in 2 3 4 5; do for o in 0 1; do timeout 300 python scripts/prof_step.py --cfg $c --reps 3 --order $o >> $O/phases.log 2>&1; done; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^k_query$" -c 3 \
  -o $O/kq1_cfg3 -f python scripts/prof_step.py --cfg 3 --reps 1 --order 1 > $O/kq1.log 2>&1
ncu -i $O/kq1_cfg3.ncu-rep --page raw --csv > $O/kq1_raw.csv 2>/dev/null
ncu -i $O/kq1_cfg3.ncu-rep --page source --csv --print-source sass > $O/kq1_src.csv 2>/dev/null
echo done
