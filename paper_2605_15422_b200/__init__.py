"""B200-native (sm_100a) DualKV shared-prompt attention.

Drop-in for the attention path of the reference CPU package `dualkv`
(arxiv 2605.15422): the same public names and signatures, executed by
hand-written tcgen05/TMEM/TMA kernels behind the C ABI of `libdkv.so`.
"""

from .api import (  # noqa: F401
    ContextGradScratch,
    DualKVInput,
    VarlenBatch,
    bf16_naive_accumulate,
    context_grad_contributions,
    convert_dkv_context,
    dualkv_attention_varlen,
    dualkv_bwd,
    dualkv_fwd,
    dualkv_two_call_attention,
    dualkv_two_call_bwd,
    dualkv_two_call_fwd,
    fa2_varlen_bwd,
    fa2_varlen_fwd,
    uses_tensor_cores,
)
from .costmodel import attention_flops, visible_pairs  # noqa: F401
from .rope import RoPE, repack_rope_to_dualkv, rope_logical  # noqa: F401
from .layer import DualKVBatch, DualKVSelfAttention  # noqa: F401
from . import library  # noqa: F401  (torch.library ops: dualkv::fwd/bwd/two_call_fwd/two_call_bwd/rope)

__version__ = "0.2.0"
