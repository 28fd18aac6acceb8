#!/bin/bash
# ncu --set full of the light query kernels (count, emit) at a BASELINE config.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
CFG=${1:-3}; TAG=${2:-kq}; KREGEX=${3:-k_query}; CNT=${4:-2}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$KREGEX -c $CNT \
  -o gpurun_out/${TAG}_cfg${CFG} -f python scripts/prof_step.py --cfg $CFG --reps 1 > gpurun_out/${TAG}_cfg${CFG}.log 2>&1
echo "ncu exit $?" >> gpurun_out/${TAG}_cfg${CFG}.log
