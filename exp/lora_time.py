"""Experiment harness (not product): time the gathered decode shrink and expand at the config-3
pool (13B widths, 128 slots r{8,16,64}, batch 64, per-token adapters uniform, 53 distinct) from
a given build.  Each rep uses the next layer's adapter rows (40 layers, 5 GB), so the rows come
from HBM, not L2.  Reports us per launch and the bytes the launch must move (distinct adapters'
rows) as GB/s.
python exp/lora_time.py [lib.so ...]"""
import os
import subprocess
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if len(sys.argv) > 2:   # one process per library
    for so in sys.argv[1:]:
        subprocess.run([sys.executable, __file__, so], check=True)
    sys.exit(0)
from paper_2505_14468_b200 import _lib  # noqa: E402

if len(sys.argv) > 1:
    _lib.LIB_PATH = os.path.abspath(sys.argv[1])
from paper_2505_14468_b200 import ops  # noqa: E402
from paper_2505_14468_b200.config import LLAMA2_13B, LoraConfig  # noqa: E402
from paper_2505_14468_b200.model import AdapterPool  # noqa: E402

torch.cuda.set_device(0)
cfg, B, NS = LLAMA2_13B, 64, 128
dev = torch.device("cuda")
pool = AdapterPool(cfg, ("q", "k", "v", "o"), NS, 64, dev)
ranks = np.random.default_rng(0).choice([8, 16, 64], size=NS)
for a in range(NS):
    pool.load_random(a, LoraConfig(int(ranks[a]), 2.0 * ranks[a]), seed=100 + a)
sl = np.random.default_rng(0).integers(0, NS, size=B).astype(np.int32)
slots = torch.from_numpy(sl).to(dev)
ws = torch.zeros(ops.lora_workspace_bytes(B, NS, 64, 4) + 256, dtype=torch.uint8, device=dev)
ops.lora_plan_tokens(slots, NS, ws)
d = cfg.hidden
x = torch.randn(B, d, device=dev).to(torch.bfloat16)
qkv = torch.randn(B, 3 * d, device=dev).to(torch.bfloat16)
res = torch.randn(B, d, device=dev).to(torch.bfloat16)
v = torch.zeros(B, 3 * 64, device=dev)
vo = torch.zeros(B, 64, device=dev)
L = cfg.layers
tq = [ops.make_targets([(pool.a_ptr[l, i], pool.b_ptr[l, i], d, i * d, d, d) for i in range(3)])
      for l in range(L)]
to = [ops.make_targets([(pool.a_ptr[l, 3], pool.b_ptr[l, 3], d, 0, d, d)]) for l in range(L)]
offs = [0, 64, 128]
rows = sum(int(ranks[a]) for a in sorted(set(sl.tolist())))
mb_t = rows * d * 2 / 1e6   # one target's distinct A (or B) rows


def t(fn, n=80):
    for i in range(L):
        fn(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(n):
        fn(i % L)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1000 / n


r = {
    "shrink_qkv": (t(lambda l: ops.lora_shrink(v, x, pool.rank, 64, tq[l], offs, ws)), 3 * mb_t),
    "expand_qkv": (t(lambda l: ops.lora_expand(qkv, v, pool.rank, pool.scale, 64, tq[l], offs, ws,
                                               v_slot_stride=0)), 3 * mb_t),
    "shrink_o": (t(lambda l: ops.lora_shrink(vo, x, pool.rank, 64, to[l], [0], ws)), mb_t),
    "expand_o": (t(lambda l: ops.lora_expand(res, vo, pool.rank, pool.scale, 64, to[l], [0], ws,
                                             v_slot_stride=0)), mb_t),
}
name = os.path.basename(_lib.LIB_PATH)
tot = sum(u for u, _ in r.values())
print(name, " ".join(f"{k} {u:.1f}us ({m / u:.2f} TB/s)" for k, (u, m) in r.items()),
      f"| per layer {tot:.1f} us", flush=True)
