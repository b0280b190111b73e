#!/bin/bash
# Launch list of one decode bench run (our kernels only): per-launch device time (serialised).
mkdir -p gpurun_out
K='regex:gemm|lora|attn|rmsnorm|argmax|embedding'
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-prefill \
  > gpurun_out/ncu_bench.log 2>&1
python tools/launches_summary.py gpurun_out/launches.csv
