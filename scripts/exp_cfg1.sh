cd $GRAFT_REPO_ROOT
for so in exp/*.so; do echo "== $so" >> gpurun_out/exp1.log; RHG_LIB_PATH=$PWD/$so timeout 120 python scripts/prof_step.py --cfg 1 --reps 1 2>&1 | tail -1 >> gpurun_out/exp1.log; done
