set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_chain.py -x -q -p no:cacheprovider > gpurun_out/chain_tests.log 2>&1; echo rc=$? >> gpurun_out/chain_tests.log
tail -30 gpurun_out/chain_tests.log
if grep -q "rc=0" gpurun_out/chain_tests.log; then
  timeout 300 python bench.py --no-cpu-baseline --no-prefill --steps 30 > gpurun_out/chain_bench.json 2> gpurun_out/chain_bench.err
  python -c "
import json; b=json.load(open('gpurun_out/chain_bench.json'))
print(b['value'], b['ms_per_step'], b['e2e']['value'], b['run'], b['lora_kernels']['ms_per_step'])"
  tail -5 gpurun_out/chain_bench.err
fi
