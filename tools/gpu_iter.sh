#!/bin/bash
# Quick GPU iteration (through gpurun): short bench without the CPU legs, then
# the parity tests; optional ncu --set full capture of the kernels in $NCU_K.
mkdir -p gpurun_out
python bench.py --no-parity --no-e2e --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/iter_bench.log 2>&1; echo "EXIT $?" >> gpurun_out/iter_bench.log
if [ -n "$NCU_K" ]; then
  ncu --set full --clock-control none --import-source on -k "regex:$NCU_K" -s ${NCU_SKIP:-6} -c ${NCU_COUNT:-2} \
      -o gpurun_out/${NCU_OUT:-full} -f python bench.py --profile --steps 1 --warmup 3 > gpurun_out/ncu_full.log 2>&1
fi
if [ -z "$NO_TESTS" ]; then
  python -m pytest tests -m gpu -q -x -p no:cacheprovider ${TEST_ARGS:-tests/test_gpu_parity.py tests/test_gpu_edge_cases.py} > gpurun_out/iter_tests.log 2>&1
  echo "EXIT $?" >> gpurun_out/iter_tests.log
fi
