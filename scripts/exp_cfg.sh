#!/bin/bash
# run prof_step for config $CFG (order $ORDER) with the in-tree library and every exp/*.so
cd "${GRAFT_REPO_ROOT:-/root/repo}"
A="--cfg ${CFG:-2} --reps 2 --order ${ORDER:-0}"
echo "== base" >> gpurun_out/exp1.log; timeout 120 python scripts/prof_step.py $A 2>&1 | tail -1 >> gpurun_out/exp1.log
for so in exp/*.so; do echo "== $so" >> gpurun_out/exp1.log; RHG_LIB_PATH=$PWD/$so timeout 120 python scripts/prof_step.py $A 2>&1 | tail -1 >> gpurun_out/exp1.log; done
