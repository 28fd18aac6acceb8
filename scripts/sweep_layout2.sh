#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/sweep2.log
rm -f $O
for L in 10 11 12 13; do for p in 0.7 0.75 0.8; do for h in 1024 2048; do
  echo "L $L p $p h $h" >> $O; timeout 120 python scripts/prof_step.py --cfg 3 --reps 3 --bands $L --ratio $p --heavy $h 2>&1 | tail -1 >> $O
done; done; done
for c in 2 4 5; do for L in 0 12; do p=0.8; [ $L = 0 ] && p=0
  echo "cfg $c L $L p $p" >> $O; timeout 200 python scripts/prof_step.py --cfg $c --reps 3 --bands $L --ratio $p 2>&1 | tail -1 >> $O
done; done
