#!/bin/bash
# compute-sanitizer racecheck on scripts/repro/synccheck_cond.cu: the trivial
# shuffle kernel in a plain graph vs inside a WHILE conditional-node body, at
# several grid sizes, 3 runs each -> gpurun_out/r02_racecheck_repro.txt
cd "$(dirname "$0")"
nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/synccheck_cond synccheck_cond.cu || exit 1
mkdir -p ../../gpurun_out
for b in 3 1000 20000; do
  for m in plain graph while; do
    for r in 1 2 3; do
      echo "== compute-sanitizer --tool racecheck synccheck_cond $m $b (run $r)"
      timeout 300 compute-sanitizer --tool racecheck /tmp/synccheck_cond $m $b 2>&1 | grep -v "^=========     "
      echo "rc=${PIPESTATUS[0]}"
    done
  done
done > ../../gpurun_out/r02_racecheck_repro.txt 2>&1
grep -c "Target application returned an error" ../../gpurun_out/r02_racecheck_repro.txt
