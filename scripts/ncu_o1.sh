cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_(query|heavy|gather_philox|directory|rs_scatter)$" -c 10 \
  -o $O/kq_o1 -f python scripts/prof_step.py --cfg 3 --reps 1 --order 1 > $O/kq_o1.log 2>&1
ncu -i $O/kq_o1.ncu-rep --page raw --csv > $O/kq_o1_raw.csv 2>/dev/null
ncu -i $O/kq_o1.ncu-rep --page source --csv --print-source sass > $O/kq_o1_src.csv 2>/dev/null
