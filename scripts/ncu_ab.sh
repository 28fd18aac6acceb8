#!/bin/bash
# ncu --set full of the light query kernels (count + emit) at CFG, ORDER for the in-tree
# library and every exp/*.so (A/B of kernel variants on the same box).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
run() {  # tag, lib
  RHG_LIB_PATH=$2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_query$" --launch-skip ${SKIP:-0} -c ${NK:-2} \
    -o $O/$1 -f python scripts/prof_step.py --cfg ${CFG:-3} --reps 1 --order ${ORDER:-0} > $O/$1.log 2>&1
  ncu -i $O/$1.ncu-rep --page raw --csv > $O/${1}_raw.csv 2>/dev/null
  [ -n "$SRC" ] && ncu -i $O/$1.ncu-rep --page source --csv --print-source sass > $O/${1}_src.csv 2>/dev/null
  rm -f $O/$1.ncu-rep
  echo "== $1"; python scripts/ncu_raw_summary.py $O/${1}_raw.csv 2>/dev/null
}
run ab_main $PWD/paper_1606_09481_b200/librhg.so
for so in exp/*.so; do [ -f "$so" ] || continue; t=$(basename $so .so); run ab_$t $PWD/$so; done
