#!/bin/bash
# Development loop on the GPU box: build, a subset of the GPU tests (TESTS = pytest -k
# expression, empty = all), phases of CFGS in ORDERS, and exp/*.so variants if present.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
if [ "${TESTS-x}" != "none" ]; then
  timeout ${TTIME:-1200} python -m pytest tests -m gpu -q -x ${TESTS:+-k "$TESTS"} > $O/pytest_gpu.log 2>&1
  echo "pytest exit $?" >> $O/pytest_gpu.log; tail -3 $O/pytest_gpu.log
fi
rm -f $O/phases.log
for c in ${CFGS:-3}; do for o in ${ORDERS:-0}; do
  timeout 300 python scripts/prof_step.py --cfg $c --reps 3 --order $o >> $O/phases.log 2>&1
  for so in exp/*.so; do [ -f "$so" ] || continue
    echo "== $so" >> $O/phases.log
    RHG_LIB_PATH=$PWD/$so timeout 300 python scripts/prof_step.py --cfg $c --reps 3 --order $o >> $O/phases.log 2>&1
  done
done; done
cat $O/phases.log | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); print(d['cfg'], d['order'], d['fmt'], 'count %.3f scan %.3f emit %.3f total %.3f' % (d['ms_count'], d['ms_scan'], d['ms_emit'], d['ms_total']), 'retest', d['emit_retested'])
    else: print(l.rstrip())
"
