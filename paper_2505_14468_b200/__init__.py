"""B200-native shared-backbone multi-LoRA hot path of ServerlessLoRA (arxiv 2505.14468).

Host side mirrors the reference's Python interface for this path (``slorasim``:
``batching.predict_ttft`` / ``schedule_round`` / ``FlushDecision``, ``FunctionSpec``);
the compute runs in hand-written sm_100a CUDA behind the C ABI ``include/slora_b200.h``
(``libslora_b200.so``, loaded by ``_lib``).  There is no CPU fallback.
"""

__version__ = "0.1.0"
