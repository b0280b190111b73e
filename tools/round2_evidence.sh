#!/bin/bash
# Round-2 evidence pass (run under gpurun from the repo root, one GPU): serving-runtime tests,
# the config-3 bench line, decode against the config-3 adapter pool, a real-time trace replay
# (p50 TTFT), ncu of the prefill GEMMs + tcgen05 flash attention, compute-sanitizer.
set -u
mkdir -p gpurun_out
O=gpurun_out
timeout 300 python -m pytest tests/test_gpu_runtime.py -x -q -p no:cacheprovider > $O/ev_runtime.log 2>&1; echo rc=$? >> $O/ev_runtime.log
timeout 400 python bench.py --workload config3 --steps 5 --warmup 3 > $O/ev_bench3.log 2>&1; echo rc=$? >> $O/ev_bench3.log
timeout 300 python tools/bench_decode_pool.py 20 > $O/ev_decode_pool.log 2>&1; echo rc=$? >> $O/ev_decode_pool.log
timeout 300 python tools/serve_trace.py profiles/r02_trace_7b_32fn_r2.csv $O/serve_r2 24 > $O/ev_serve_r2.log 2>&1; echo rc=$? >> $O/ev_serve_r2.log
# prefill: launch list with tensor-pipe + DRAM bytes, then full sets of the backbone GEMMs
timeout 900 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file $O/prefill_launches.csv \
  python tools/bench_prefill.py --steps 1 --warmup 0 --no-bare > $O/ncu_prefill_list.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 8 -c 4 \
  -o $O/prof_prefill_gemm_r02 -f python tools/bench_prefill.py --steps 1 --warmup 0 --no-bare \
  > $O/ncu_prefill_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:flash_prefill -s 2 -c 1 \
  -o $O/prof_flash_r02 -f python tools/bench_prefill.py --steps 1 --warmup 0 --no-bare \
  > $O/ncu_flash_full.log 2>&1
# sanitizer on the racy-by-construction kernels: pipelined decode attention ring, stream-K
# counters, split-K consumers, flash prefill
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -m pytest -x -q -p no:cacheprovider \
    "tests/test_gpu_kernels.py::test_attention_decode_pipe_lora" \
    "tests/test_gpu_kernels.py::test_gemm_stream_k" \
    "tests/test_gpu_kernels.py::test_gemm_splitk_pieces_and_consumer" \
    "tests/test_gpu_kernels.py::test_flash_prefill_matches_oracle" \
    > $O/sanitize_$tool.log 2>&1
  echo rc=$? >> $O/sanitize_$tool.log
done
echo done
