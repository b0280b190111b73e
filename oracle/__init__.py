"""TEST INFRASTRUCTURE ONLY — CPU oracle for the shared-backbone multi-LoRA forward.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import this package, and only as the checker or
the timed CPU baseline.  The product (``paper_2505_14468_b200``) never imports
it and has no CPU fallback.

Parity status: the reference (``/root/reference/pkg``, ``slorasim``) has no
forward arithmetic — it models the forward as ``T0 + alpha*(b-1)``
(``pkg/src/slorasim/batching.py:17-21``).  The oracle restates the paper's
algorithm (unmerged LoRA atop a Llama backbone, ``PAPER.md:614-621,645-646``)
and is PINNED against Hugging Face transformers 5.5.0 ``LlamaForCausalLM``
(torch 2.11 fp32, CPU) with the LoRA term injected by forward hooks — see
``tests/golden/make_golden.py`` and the committed fixtures.  The reference's own
tests pin only boundary semantics (batcher KATs), which ``tests/test_batching.py``
checks against the mirror in the product package.
"""
