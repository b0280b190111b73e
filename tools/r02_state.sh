#!/bin/bash
# Round-2 state check on one B200: GPU tests, smoke, decode bench (both arms), config-3 line.
set -u
mkdir -p gpurun_out
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/st_gputests.log 2>&1; echo rc=$? >> $O/st_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/st_smoke.log 2>&1; echo rc=$? >> $O/st_smoke.log
timeout 300 python bench.py > $O/st_bench.json 2> $O/st_bench.err; echo rc=$? >> $O/st_bench.err
timeout 300 python bench.py --impl reference > $O/st_bench_ref.json 2> $O/st_bench_ref.err
timeout 400 python bench.py --workload config3 --steps 5 --warmup 3 > $O/st_bench3.json 2> $O/st_bench3.err
tail -3 $O/st_gputests.log; tail -2 $O/st_smoke.log; tail -c 600 $O/st_bench.json
