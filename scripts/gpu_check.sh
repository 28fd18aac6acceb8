#!/bin/bash
# One gpurun call: GPU tests, per-config phase timings, bench, ncu launch list.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out
nvidia-smi > $O/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
for c in 1 2 3 4 5; do timeout 300 python scripts/prof_step.py --cfg $c --reps 3 >> $O/phases.log 2>&1; done
timeout 600 python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err; echo "bench exit $?" >> $O/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-configs > $O/ncu_launch.log 2>&1
echo done
