#!/bin/bash
# -> gpurun_out/r02_gpu_gen_counterexample.txt
cd "$(dirname "$0")"
nvcc -gencode arch=compute_100a,code=sm_100a --fmad=false -Xcompiler -ffp-contract=off -O3 \
  -o /tmp/gen_normals_device gen_normals_device.cu || exit 1
mkdir -p ../../gpurun_out
{ ldd /tmp/gen_normals_device | grep libm; /lib/x86_64-linux-gnu/libc.so.6 | head -1;
  /tmp/gen_normals_device ${1:-100000000}; } > ../../gpurun_out/r02_gpu_gen_counterexample.txt 2>&1
tail -3 ../../gpurun_out/r02_gpu_gen_counterexample.txt
