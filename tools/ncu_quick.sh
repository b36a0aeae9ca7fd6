#!/bin/bash
# Targeted ncu metrics for the hot kernels of one bench step (run ON the GPU box
# via gpurun, after the same bench command exited 0 without ncu):
#   tools/ncu_quick.sh <out.csv> [bench args...]
# Reads back here with: python tools/ncu_summary.py quick <out.csv>
out=$1; shift
METRICS=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,\
l1tex__t_sector_hit_rate.pct,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,\
sm__warps_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,\
sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,smsp__inst_executed_pipe_fp64.sum,\
gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sectors_srcunit_tex.sum,launch__registers_per_thread
KERN='regex:k_border_(prefilter|scan32|exact|wide|infinite)|k_assign_vlt|k_assign_overflow|k_vlt_build|k_owner_mark|k_field_tiles|k_bucket|k_reach'
ncu --metrics $METRICS --clock-control none -k "$KERN" --csv --log-file "$out" python bench.py --profile "$@"
