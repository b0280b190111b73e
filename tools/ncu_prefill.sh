#!/bin/bash
# ncu evidence for the config-3 prefill (run under gpurun from the repo root): launch list of one
# forward (our kernels only: tensor-pipe share, DRAM bytes), then --set full of the steady-state
# backbone GEMMs and of the tcgen05 flash attention.
set -u
mkdir -p gpurun_out
K='regex:gemm_tc|flash_tc|rope_kv|rmsnorm|lora|embedding|argmax'
timeout 900 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum \
  -k "$K" --clock-control none --csv --log-file gpurun_out/prefill_launches.csv \
  python tools/bench_prefill.py --steps 1 --warmup 0 --no-bare > gpurun_out/ncu_prefill_list.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:flash_tc -s 2 -c 1 \
  -o gpurun_out/prof_flash_r02 -f python tools/bench_prefill.py --steps 1 --warmup 0 --no-bare \
  > gpurun_out/ncu_flash_full.log 2>&1
echo done
