#!/bin/bash
# ncu evidence for the decode step (run under gpurun from the repo root).
#   1) launch list of one bench run (our kernels only; per-launch device time)
#   2) --set full capture of the top kernels inside the captured decode step
set -u
mkdir -p gpurun_out
K='regex:gemm_tc|lora|attn|rmsnorm|argmax|embedding'
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
  > gpurun_out/ncu_bench.log 2>&1
# full sets: skip the warm-up launches of each kernel family, capture a few in steady state
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 400 -c 5 \
  -o gpurun_out/prof_gemm -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_gemm.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'rope_attn|lora' -s 100 -c 4 \
  -o gpurun_out/prof_other -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_other.log 2>&1
echo done
