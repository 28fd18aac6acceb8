#!/bin/bash
# Layout / hub-threshold sweep at config 3 (the edge set does not depend on them).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/sweep.log
rm -f $O
for h in 512 2048 4096; do echo "heavy $h" >> $O; timeout 120 python scripts/prof_step.py --cfg 3 --reps 2 --heavy $h 2>&1 | tail -1 >> $O; done
for L in 12 14 16 18 20 24; do for p in 0.8 0.85 0.9; do
  echo "L $L p $p" >> $O; timeout 120 python scripts/prof_step.py --cfg 3 --reps 2 --bands $L --ratio $p 2>&1 | tail -1 >> $O
done; done
