#!/bin/bash
# One GPU-box pass (run through gpurun): bench line, launch list, targeted ncu
# metrics, then the GPU test suite. Logs under gpurun_out/.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.log 2>&1; echo "EXIT $?" >> gpurun_out/bench.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --profile --steps 1 --warmup 3 > gpurun_out/ncu_launches.log 2>&1
bash tools/ncu_quick.sh gpurun_out/quick.csv --steps 1 --warmup 3 > gpurun_out/ncu_quick.log 2>&1
if [ -z "$NO_TESTS" ]; then
  python -m pytest tests -m gpu -q -p no:cacheprovider ${TEST_ARGS:-} > gpurun_out/gputests.log 2>&1
  echo "EXIT $?" >> gpurun_out/gputests.log
fi
