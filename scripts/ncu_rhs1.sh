#!/bin/bash
# ncu --set full of the ONE-column rhs pass (EpiRhs1, r0's column from the
# carried w) at each BASELINE config: the rhs launches of ADMM steps 2-4 of an
# eager solve (step 1 forms both columns; steps 2-4 follow carried steps).
#   bash scripts/ncu_rhs1.sh "2 3 4 5a 5b"  ->  gpurun_out/ncu_r02_cfg*_rhs1_raw.csv
set -u
mkdir -p gpurun_out
for c in ${1:-"2 3 4 5a 5b"}; do
  rep=/tmp/ncu_rhs1_$c
  timeout 900 ncu --set full --clock-control none --kernel-name-base mangled \
    -k regex:EpiRhs1 --launch-skip 1 --launch-count 3 -f -o $rep \
    python scripts/ncu_capture.py $c f64 5 > gpurun_out/ncu_r02_cfg${c}_rhs1.log 2>&1
  echo "cfg $c rc=$?"
  ncu -i $rep.ncu-rep --page raw --csv > gpurun_out/ncu_r02_cfg${c}_rhs1_raw.csv 2>/dev/null
  rm -f $rep.ncu-rep
done
