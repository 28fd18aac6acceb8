#!/bin/bash
# Quick GPU iteration: GPU tests + per-config phase timings + launch list of one config-3 step.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
rm -f $O/phases.log
for c in 1 2 3 4 5; do timeout 300 python scripts/prof_step.py --cfg $c --reps 3 >> $O/phases.log 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_q.csv python scripts/prof_step.py --cfg 3 --reps 1 > $O/ncu_q.log 2>&1
echo done
if [ "${NCU_FULL:-1}" = "1" ]; then
  bash scripts/ncu_query.sh 3 kq "^k_(query|heavy)$" 4
  ncu -i gpurun_out/kq_cfg3.ncu-rep --page raw --csv > gpurun_out/kq_raw.csv 2>/dev/null
  ncu -i gpurun_out/kq_cfg3.ncu-rep --page source --csv --print-source sass > gpurun_out/kq_src.csv 2>/dev/null
fi
