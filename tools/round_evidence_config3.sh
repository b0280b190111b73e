#!/bin/bash
# Round evidence, config 3: config-3 bench line, prefill launch list
# (tensor pipe, DRAM bytes per launch), decode against the config-3 adapter pool.
set -u
mkdir -p gpurun_out
O=gpurun_out
timeout 400 python bench.py --workload config3 --steps 5 --warmup 3 > $O/e3_bench3.json 2> $O/e3_bench3.err
K='regex:gemm_tc|flash_tc|rope_kv|rmsnorm|lora|embedding|argmax'
timeout 900 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum \
  -k "$K" --clock-control none --csv --log-file $O/prefill_launches.csv \
  python tools/bench_prefill.py --steps 1 --warmup 0 --no-bare > $O/ncu_prefill_list.log 2>&1
timeout 600 python tools/bench_decode_pool.py 20 > $O/e3_decode_pool.log 2>&1; echo rc=$? >> $O/e3_decode_pool.log
echo done
