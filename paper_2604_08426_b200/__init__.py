"""kvb -- B200-native (sm_100a) decode hot path of arXiv 2604.08426's KV-cache
offloading study, a drop-in for the reference ``kvlab`` decode API.

``paper_2604_08426_b200.compat``  kvlab-signature functions (numpy in/out)
``paper_2604_08426_b200.store``   batched device stores (torch in/out)
``paper_2604_08426_b200.decode``  multi-layer decode step (CUDA graphs)
``include/kvb.h``                 the C-ABI of libkvb.so underneath

Importing the package does not touch the GPU; the first store creation loads
libkvb.so and fails loudly if it was not built (no CPU fallback).
"""

from .schemes import (SchemeDescriptor, bits_per_key, scheme_from_string, scheme_fp8,
                      scheme_higgs, scheme_none, scheme_nvfp4, scheme_svd, scheme_to_string)

__all__ = [
    "SchemeDescriptor", "bits_per_key", "scheme_from_string", "scheme_fp8", "scheme_higgs",
    "scheme_none", "scheme_nvfp4", "scheme_svd", "scheme_to_string",
    "BudgetConfig", "SelectionResult", "AttentionOutput", "ChunkedKVStore", "build_store",
    "select_by_landmarks", "approx_topk_residual", "residual_scores", "sparse_attention",
    "oracle_select", "full_attention_heads", "recall", "normalize_queries",
]


def __getattr__(name):
    # the compat layer imports torch; load it lazily
    if name in __all__:
        from . import compat
        return getattr(compat, name)
    raise AttributeError(name)
