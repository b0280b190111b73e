set -u
O=gpurun_out
python -m pytest tests/test_gpu_lora_gather.py tests/test_gpu_model.py -x -q -m gpu > $O/t3.log 2>&1; echo PYTEST_RC=$? >> $O/t3.log
python exp/lora_time.py exp/lora_head.so paper_2505_14468_b200/libslora_b200.so > $O/lt3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"lora_expand_v|lora_shrink_v" -s 80 -c 2 -o $O/lora_new -f python exp/lora_time.py paper_2505_14468_b200/libslora_b200.so > $O/ncu_new.log 2>&1
grep -E "passed|failed|RC" $O/t3.log | tail -3; cat $O/lt3.log
