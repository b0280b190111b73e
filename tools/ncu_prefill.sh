#!/bin/bash
# ncu evidence for the config-3 prefill (run under gpurun from the repo root): launch list of one
# forward, then --set full of the steady-state backbone GEMMs (qkv/o LoRA-fold, gate/up, down).
set -u
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file gpurun_out/prefill_launches.csv \
  python tools/bench_prefill.py --steps 1 --warmup 0 --no-bare > gpurun_out/ncu_prefill_list.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 8 -c 8 \
  -o gpurun_out/prof_prefill_gemm_r02 -f python tools/bench_prefill.py --steps 1 --warmup 0 --no-bare \
  > gpurun_out/ncu_prefill_full.log 2>&1
echo done
