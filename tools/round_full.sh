#!/bin/bash
# Full round evidence on one B200 (run under gpurun from the repo root): bench lines (both arms),
# per-launch DRAM traffic and launch list of the decode step, and --set full captures of the
# top kernels (gate/up stream-K GEMM, decode attention) for profiles/.
set -u
bash tools/round_evidence.sh > gpurun_out/round_evidence.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_sk_kernel -s 3 -c 1 \
  -o gpurun_out/prof_sk_gu -f python tools/gemm_one.py 22016 4096 2 > gpurun_out/ncu_sk.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_decode_pipe -s 3 -c 1 \
  -o gpurun_out/prof_attn -f python tools/attn_one.py > gpurun_out/ncu_attn.log 2>&1
echo done
