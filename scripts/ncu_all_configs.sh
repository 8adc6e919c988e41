#!/bin/bash
# ncu --set full captures of the loop kernels of every BASELINE config
# (one GPU; the ADMM loop capped so svm's 50000-iteration run stays bounded).
#   bash scripts/ncu_all_configs.sh "3 4 5a 5b 2:f32" [ROUND]
# -> gpurun_out/ncu_<round>_cfg<c>[_f32].ncu-rep (+ .log)
set -u
CFGS=${1:-"2 3 4 5a 5b 2:f32"}
R=${2:-r02}
mkdir -p gpurun_out
for spec in $CFGS; do
  c=${spec%%:*}; dt=f64; [[ "$spec" == *:f32 ]] && dt=f32
  tag=cfg${c}; [[ $dt == f32 ]] && tag=${tag}_f32
  timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:'spmv_kernel|spmv_select_kernel|k_pcg' --launch-skip 60 --launch-count 30 \
    -f -o gpurun_out/ncu_${R}_${tag} python scripts/ncu_capture.py $c $dt 12 \
    > gpurun_out/ncu_${R}_${tag}.log 2>&1
  echo "$tag rc=$?"
done
