"""Generate the serving-replay trace with the REFERENCE's own generator (CPU, this container:
imports /root/reference/pkg/src): ``n_fn`` 7B LoRA functions, ``generate_trace(NORMAL, ...)``
per function (MMPP arrivals, log-normal prompt/output lengths, median 60 / 64 tokens,
``workload.py:103-209``), merged, written with the reference's trace CSV writer.
python tools/make_trace.py OUT.csv [n_fn] [rate_per_fn] [duration_s] [seed] [fn_prefix]"""
import sys

sys.path.insert(0, "/root/reference/pkg/src")
from slorasim import workload  # noqa: E402
from slorasim.workload import CovClass  # noqa: E402

out = sys.argv[1]
n_fn = int(sys.argv[2]) if len(sys.argv) > 2 else 32
rate = float(sys.argv[3]) if len(sys.argv) > 3 else 2.0
dur = float(sys.argv[4]) if len(sys.argv) > 4 else 60.0
seed = int(sys.argv[5]) if len(sys.argv) > 5 else 0
prefix = sys.argv[6] if len(sys.argv) > 6 else "7b"
traces = []
for i in range(n_fn):
    for s in range(seed, seed + 20):   # retry-next-seed
        try:
            traces.append(workload.generate_trace(CovClass.NORMAL, dur, rate, s, function_id=f"{prefix}-fn{i:02d}"))
            break
        except workload.ClassUnreachable:
            continue
tr = workload.merge_traces(traces)
workload.write_trace_csv(tr, out)
print(f"{out}: {len(tr.records) if hasattr(tr, 'records') else len(list(tr))} requests, {n_fn} functions, "
      f"{rate} req/s/fn requested, {dur} s")
