timeout 900 ncu --set full --clock-control none --import-source on -k regex:flash_tc -s 2 -c 1 \
  -o gpurun_out/prof_flash_v2 -f python tools/bench_prefill.py --steps 1 --warmup 0 --no-bare > gpurun_out/ncu_flash_v2.log 2>&1
echo rc=$?
