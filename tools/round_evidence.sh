#!/bin/bash
# Round evidence on one B200: bench line, launch list (serialised per-launch times) and the
# per-launch DRAM traffic of the step's kernels (profiles/traffic.json).
set -u
mkdir -p gpurun_out
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
  --clock-control none -k 'regex:gemm_sk|attn_decode' --csv --log-file gpurun_out/traffic.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_traffic.log 2>&1
python tools/ncu_traffic.py gpurun_out/traffic.csv > gpurun_out/traffic_summary.json
bash tools/ncu_launches.sh > gpurun_out/launches_summary.txt
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
cp profiles/traffic.json gpurun_out/traffic.json
cat gpurun_out/launches_summary.txt
tail -c 2500 gpurun_out/bench.json
