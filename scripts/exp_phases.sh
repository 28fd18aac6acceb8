#!/bin/bash
# Phase timings of alternative builds in exp/ (experiments) vs the in-tree library.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out; rm -f $O/exp.log
for cfg in ${CFGS:-3}; do
  echo "== base cfg $cfg" >> $O/exp.log; timeout 300 python scripts/prof_step.py --cfg $cfg --reps 3 >> $O/exp.log 2>&1
  for so in exp/*.so; do
    echo "== $so cfg $cfg" >> $O/exp.log
    RHG_LIB_PATH=$PWD/$so timeout 300 python scripts/prof_step.py --cfg $cfg --reps 3 >> $O/exp.log 2>&1
  done
done
