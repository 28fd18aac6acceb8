#!/bin/bash
# Round-end style evidence: GPU tests, bench (default args), ncu launch list of a bench
# run, ncu --set full of the query kernels at config 3, phase timings for all configs.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out
nvidia-smi > $O/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench exit $?" >> $O/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-configs > $O/ncu_launch.log 2>&1
bash scripts/ncu_query.sh 3 kq "^k_(query|heavy)$" 4
ncu -i $O/kq_cfg3.ncu-rep --page raw --csv > $O/kq_raw.csv 2>/dev/null
ncu -i $O/kq_cfg3.ncu-rep --page source --csv --print-source sass > $O/kq_src.csv 2>/dev/null
rm -f $O/phases.log
for c in 1 2 3 4 5; do timeout 300 python scripts/prof_step.py --cfg $c --reps 3 >> $O/phases.log 2>&1; done
echo done
