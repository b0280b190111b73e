#!/bin/bash
# Round-2 evidence: decode timeline, decode launch list + traffic, prefill ncu (launch list with
# tensor-pipe + DRAM bytes, full sets of prefill GEMMs and the tcgen05 flash attention).
set -u
mkdir -p gpurun_out
O=gpurun_out
timeout 300 python tools/step_timeline.py > $O/ev2_timeline.txt 2>&1
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
  --clock-control none -k 'regex:gemm_sk|attn_decode|rmsnorm' --csv --log-file $O/traffic.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-prefill > $O/ncu_traffic.log 2>&1
python tools/ncu_traffic.py $O/traffic.csv > $O/traffic_summary.json 2>&1
bash tools/ncu_launches.sh > $O/launches_summary.txt 2>&1
bash tools/ncu_prefill.sh > $O/ncu_prefill.out 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:flash_prefill -s 2 -c 1 \
  -o $O/prof_flash_r02 -f python tools/bench_prefill.py --steps 1 --warmup 0 --no-bare \
  > $O/ncu_flash_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_sk_kernel -s 300 -c 4 \
  -o $O/prof_gemm_sk_r02 -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-prefill \
  > $O/ncu_sk_full.log 2>&1
echo done
