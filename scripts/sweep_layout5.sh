#!/bin/bash
# Slab-layout sweep (num_bands L, band_ratio p) of the generation phases at configs
# 5, 2 and 4 (profiles/r02_layout_sweep.log); the edge set does not depend on (L, p).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for L in 12 13 14 15 16; do for p in 0.9 0.93 0.95; do
  python scripts/prof_step.py --cfg 5 --reps 2 --bands $L --ratio $p | tail -1
done; done
for c in 2 4; do for L in 12 14 16; do for p in 0.8 0.85 0.9 0.93; do
  python scripts/prof_step.py --cfg $c --reps 3 --bands $L --ratio $p | tail -1
done; done; done
