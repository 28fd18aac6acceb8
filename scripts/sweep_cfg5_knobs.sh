#!/bin/bash
# Config-5 knob sweep: directory granularity (exp/d*.so builds) x hub threshold.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for lib in paper_1606_09481_b200/librhg.so exp/d1.so exp/d2.so; do for h in ${HS:-0}; do
  echo "== $lib heavy $h"
  RHG_LIB_PATH=$PWD/$lib python scripts/prof_step.py --cfg ${CFG:-5} --reps 2 --heavy $h | tail -1
done; done
