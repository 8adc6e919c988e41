#!/bin/bash
# ncu --set full captures of the loop kernels of every BASELINE config
# (one GPU; the ADMM loop capped so svm's 50000-iteration run stays bounded).
#   bash scripts/ncu_all_configs.sh "3 4 5a 5b 2:f32" [ROUND] [COUNT]
# Each report is exported on the box (raw page CSV + a details page of the
# first launch of each kernel), summarised into profiles/ncu_summary.json by
# scripts/ncu_summarize.py and then deleted (gpurun copies back <= 64 MiB).
set -u
CFGS=${1:-"2 3 4 5a 5b 2:f32"}
R=${2:-r02}
COUNT=${3:-20}
mkdir -p gpurun_out
for spec in $CFGS; do
  c=${spec%%:*}; dt=f64; [[ "$spec" == *:f32 ]] && dt=f32
  tag=cfg${c}; key=$c; [[ $dt == f32 ]] && { tag=${tag}_f32; key=${c}_f32; }
  rep=/tmp/ncu_${R}_${tag}
  # (1) the PCG-iteration kernels, past setup; (2) the two ADMM-step passes
  timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:'spmv_kernel|spmv_select_kernel|k_pcg' --launch-skip 60 --launch-count $COUNT \
    -f -o ${rep} python scripts/ncu_capture.py $c $dt 12 > gpurun_out/ncu_${R}_${tag}.log 2>&1
  echo "$tag pcg rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
    -k regex:'EpiRhs|EpiAdmm' --launch-count 4 \
    -f -o ${rep}_admm python scripts/ncu_capture.py $c $dt 3 >> gpurun_out/ncu_${R}_${tag}.log 2>&1
  echo "$tag admm rc=$?"
  ncu -i $rep.ncu-rep --page raw --csv > gpurun_out/ncu_${R}_${tag}_raw.csv 2>/dev/null
  ncu -i ${rep}_admm.ncu-rep --page raw --csv > gpurun_out/ncu_${R}_${tag}_admm_raw.csv 2>/dev/null
  ncu -i $rep.ncu-rep --page details --print-kernel-base function > gpurun_out/ncu_${R}_${tag}_details.txt 2>/dev/null
  ncu -i ${rep}_admm.ncu-rep --page details --print-kernel-base function > gpurun_out/ncu_${R}_${tag}_admm_details.txt 2>/dev/null
  python scripts/ncu_summarize.py gpurun_out/ncu_${R}_${tag}_raw.csv,gpurun_out/ncu_${R}_${tag}_admm_raw.csv $key \
    "ncu --set full, $R, config $c $dt (scripts/ncu_all_configs.sh)" > /dev/null
  cp profiles/ncu_summary.json gpurun_out/ncu_summary.json
  rm -f $rep.ncu-rep ${rep}_admm.ncu-rep
done
du -sh gpurun_out
