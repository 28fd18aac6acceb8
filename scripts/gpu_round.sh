#!/bin/bash
# Round evidence in one gpurun call: GPU tests, default bench, ncu launch list of a
# bench run, ncu --set full of the query kernels (both vertex orders) -> json,
# per-config phases.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out
nvidia-smi > $O/smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench exit $?" >> $O/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-configs > $O/ncu_launch.log 2>&1
for o in 1 0; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_(query|heavy)$" -c 4 \
    -o $O/kq_o${o} -f python scripts/prof_step.py --cfg 3 --reps 1 --order $o > $O/kq_o${o}.log 2>&1
  ncu -i $O/kq_o${o}.ncu-rep --page raw --csv > $O/kq_o${o}_raw.csv 2>/dev/null
  ncu -i $O/kq_o${o}.ncu-rep --page source --csv --print-source sass > $O/kq_o${o}_src.csv 2>/dev/null
done
python scripts/ncu_json.py $O/ncu_query_cfg3.json $O/kq_o1_raw.csv $O/kq_o0_raw.csv > $O/ncu_json.log 2>&1
# config 5 (list output): the light count and emit kernels
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_query$" -c 2 \
  -o $O/kq_cfg5 -f python scripts/prof_step.py --cfg 5 --reps 1 --order 0 > $O/kq_cfg5.log 2>&1
ncu -i $O/kq_cfg5.ncu-rep --page raw --csv > $O/kq_cfg5_raw.csv 2>/dev/null
python scripts/ncu_raw_summary.py $O/kq_cfg5_raw.csv > $O/kq_cfg5_summary.txt 2>&1
rm -f $O/kq_cfg5.ncu-rep
rm -f $O/phases.log
for c in 1 2 3 4 5; do for o in 1 0; do timeout 300 python scripts/prof_step.py --cfg $c --reps 3 --order $o >> $O/phases.log 2>&1; done; done
echo done
