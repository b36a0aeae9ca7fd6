#!/bin/bash
# All BASELINE configs (short bench lines, no CPU legs), the exact policy and
# the slot-order leg of config 2 (through gpurun). Logs: gpurun_out/cfg_*.log
mkdir -p gpurun_out
for c in 1 3 4 5; do
  python bench.py --config $c --no-parity --no-e2e --no-cpu-baseline --steps 5 > gpurun_out/cfg_$c.log 2>&1
done
python bench.py --config 2 --policy exact --no-parity --no-e2e --no-cpu-baseline --steps 3 > gpurun_out/cfg_2_exact.log 2>&1
SBDT_HOST_ROW_ORDER=slot python bench.py --config 2 --no-parity --no-e2e --no-cpu-baseline --steps 10 > gpurun_out/cfg_2_slot.log 2>&1
