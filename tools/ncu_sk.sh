ncu --set full --clock-control none --import-source on -k regex:gemm_sk_kernel -s 3 -c 1 -o gpurun_out/prof_sk_gu -f python tools/gemm_one.py 22016 4096 2 > gpurun_out/ncu_sk.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_sk_kernel -s 3 -c 1 -o gpurun_out/prof_sk_lm -f python tools/gemm_one.py 32000 4096 0 >> gpurun_out/ncu_sk.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_sk_kernel -s 3 -c 1 -o gpurun_out/prof_sk_o -f python tools/gemm_one.py 4096 4096 1 >> gpurun_out/ncu_sk.log 2>&1
