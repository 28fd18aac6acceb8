#!/bin/bash
# A/B of a runtime knob: phases of $CFGS x $ORDERS with the environment assignments in
# $VARIANTS (space-separated NAME=VALUE, the first is the baseline), then the GPU tests
# selected by $TESTK under $TESTENV (one NAME=VALUE).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out; rm -f $O/ab_env.log
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks_throttle_reasons.active --format=csv >> $O/ab_env.log 2>&1
for cfg in ${CFGS:-3}; do for o in ${ORDERS:-0}; do for v in $VARIANTS; do
  echo "== $v cfg $cfg order $o" >> $O/ab_env.log
  env $v timeout 300 python scripts/prof_step.py --cfg $cfg --reps 4 --order $o >> $O/ab_env.log 2>&1
done; done; done
if [ -n "$TESTK" ]; then
  env $TESTENV timeout 1500 python -m pytest tests -m gpu -x -q -k "$TESTK" > $O/ab_env_pytest.log 2>&1
  echo "pytest exit $?" >> $O/ab_env_pytest.log
fi
python - > $O/ab_env_summary.txt <<'PY'
import json
for l in open('gpurun_out/ab_env.log'):
    if l.startswith('{'):
        d = json.loads(l)
        print(d['cfg'], d['order'], 'count %.3f scan %.3f emit %.3f total %.3f' % (d['ms_count'], d['ms_scan'], d['ms_emit'], d['ms_total']))
    elif l.startswith('=='):
        print(l.rstrip())
PY
echo done >> $O/ab_env.log
