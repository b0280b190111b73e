#!/bin/bash
# Round evidence on one B200 (run under gpurun from the repo root): GPU tests, the bench lines
# (config 2 both arms, config 3), decode launch list + per-launch DRAM traffic, prefill launch
# list (tensor-pipe share, DRAM bytes), full ncu sets of the flash prefill and a prefill GEMM,
# decode against config 3's adapter pool (+ ncu DRAM bytes of its gathered LoRA launches),
# compute-sanitizer on the kernels changed this round.
set -u
mkdir -p gpurun_out
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/fe_gputests.log 2>&1; echo rc=$? >> $O/fe_gputests.log
timeout 400 python bench.py > $O/fe_bench.json 2> $O/fe_bench.err
timeout 300 python bench.py --impl reference > $O/fe_bench_ref.json 2> $O/fe_bench_ref.err
timeout 400 python bench.py --workload config3 --steps 5 --warmup 3 > $O/fe_bench3.json 2> $O/fe_bench3.err
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
  --clock-control none -k 'regex:gemm_sk|attn_decode' --csv --log-file $O/traffic.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-prefill > $O/ncu_traffic.log 2>&1
python tools/ncu_traffic.py $O/traffic.csv > $O/traffic_summary.json 2>&1
bash tools/ncu_launches.sh > $O/launches_summary.txt 2>&1
K='regex:gemm_tc|flash_tc|rope_kv|rmsnorm|lora|embedding|argmax'
timeout 900 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum \
  -k "$K" --clock-control none --csv --log-file $O/prefill_launches.csv \
  python tools/bench_prefill.py --steps 1 --warmup 0 --no-bare > $O/ncu_prefill_list.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:flash_tc -s 2 -c 1 \
  -o $O/prof_flash_final -f python tools/bench_prefill.py --steps 1 --warmup 0 --no-bare > $O/ncu_flash_full.log 2>&1
timeout 600 python tools/bench_decode_pool.py 20 > $O/fe_pool.json 2> $O/fe_pool.err
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
  --clock-control none -k 'regex:lora_shrink_v|lora_expand_v' -c 320 --csv --log-file $O/pool_lora.csv \
  python tools/bench_decode_pool.py 2 > $O/ncu_pool.log 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -m pytest -x -q -p no:cacheprovider \
    "tests/test_gpu_kernels.py::test_flash_prefill_matches_oracle" \
    "tests/test_gpu_kernels.py::test_attention_decode_pipe_lora" \
    tests/test_gpu_lora_gather.py \
    > $O/sanitize_$tool.log 2>&1
  echo rc=$? >> $O/sanitize_$tool.log
done
echo done
