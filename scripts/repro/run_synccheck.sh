#!/bin/bash
# Builds scripts/repro/synccheck_cond.cu and runs it under compute-sanitizer
# synccheck in its three launch modes; -> gpurun_out/r02_synccheck_repro.txt
cd "$(dirname "$0")"
nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/synccheck_cond synccheck_cond.cu || exit 1
mkdir -p ../../gpurun_out
for m in plain graph while; do
  echo "== compute-sanitizer --tool synccheck synccheck_cond $m"
  compute-sanitizer --tool synccheck --print-limit 4 /tmp/synccheck_cond $m 2>&1
  echo "== compute-sanitizer --tool memcheck synccheck_cond $m"
  compute-sanitizer --tool memcheck /tmp/synccheck_cond $m 2>&1 | tail -2
done > ../../gpurun_out/r02_synccheck_repro.txt
tail -5 ../../gpurun_out/r02_synccheck_repro.txt
