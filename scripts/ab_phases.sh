#!/bin/bash
# A/B phases: the in-tree library against every exp/*.so on the same box, configs in
# $CFGS (default "5 3"), vertex orders in $ORDERS (default "0"), then the GPU tests
# selected by $TESTK (pytest -k expression; empty = none).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out; rm -f $O/ab.log
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks_throttle_reasons.active --format=csv >> $O/ab.log 2>&1
for cfg in ${CFGS:-5 3}; do for o in ${ORDERS:-0}; do
  echo "== in-tree cfg $cfg order $o" >> $O/ab.log
  timeout 300 python scripts/prof_step.py --cfg $cfg --reps 3 --order $o >> $O/ab.log 2>&1
  for so in exp/*.so; do
    echo "== $so cfg $cfg order $o" >> $O/ab.log
    RHG_LIB_PATH=$PWD/$so timeout 300 python scripts/prof_step.py --cfg $cfg --reps 3 --order $o >> $O/ab.log 2>&1
  done
done; done
if [ -n "$TESTK" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q -k "$TESTK" > $O/ab_pytest.log 2>&1; echo "pytest exit $?" >> $O/ab_pytest.log
fi
echo done >> $O/ab.log
