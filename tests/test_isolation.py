"""Isolation mode (§8 f3): function processes over one CUDA-IPC-exported backbone produce the
same outputs as the owner process, without a copy of the backbone."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_function_processes_share_the_backbone(golden):
    from paper_2505_14468_b200.config import TINY, TINY_LORA, init_adapter, init_backbone
    from paper_2505_14468_b200.isolation import IsolatedFunctions
    from paper_2505_14468_b200.model import MultiLoraModel

    seed = int(golden["seed"])
    m = MultiLoraModel(TINY, dtype=torch.bfloat16, max_seqs=8, max_ctx=128, n_slots=4, max_rank=16,
                       max_tokens=1024)
    m.load_backbone(init_backbone(TINY, seed))
    ads = {f"f{a}": init_adapter(TINY, TINY_LORA, seed, a) for a in (1, 2)}
    for a in (1, 2):
        m.pool.load(a, ads[f"f{a}"], TINY_LORA)
    m.use_stacked_decode = False   # the function processes run the unstacked LoRA kernels
    prompts = [[5, 9, 200, 31], [7, 7, 7, 1, 2]]
    ref = {}
    for a in (1, 2):
        seqs, logits = m.prefill(prompts, [a, a])
        toks = [m.argmax(logits).cpu().tolist()]
        for _ in range(3):
            toks.append(m.argmax(m.decode(seqs, toks[-1], [a, a])).cpu().tolist())
        for s in seqs:
            m.free_seq(s)
        ref[f"f{a}"] = (logits.float().cpu().numpy(), toks)
    iso = IsolatedFunctions(m, ads, TINY_LORA)
    try:
        for fid in ads:
            logits, toks = iso.run(fid, prompts, 4)
            np.testing.assert_array_equal(logits.numpy(), ref[fid][0])
            assert toks == ref[fid][1]
            info = iso.info[fid]
            # the function process holds its adapter, KV and workspaces, not the backbone
            assert info["own_bytes"] < info["shared_backbone_bytes"]
            assert info["context_bytes"] != 0
    finally:
        iso.close()
