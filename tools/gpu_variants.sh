#!/bin/bash
# Experiment helper (through gpurun): short bench of every build/var/libsbdt_gpu_*.so
mkdir -p gpurun_out
for so in build/var/libsbdt_gpu_*.so; do
  name=$(basename $so .so); name=${name#libsbdt_gpu_}
  SBDT_GPU_LIB_EXPERIMENT=$PWD/$so python bench.py --no-parity --no-e2e --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/var_$name.log 2>&1
done
