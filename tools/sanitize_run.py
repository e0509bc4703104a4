"""Small-shape driver of every decode-path kernel family, for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck).

usage: compute-sanitizer --tool racecheck python tools/sanitize_run.py [N]
(N = context length, default 4096; racecheck runs use a shorter one)

Runs, on tiny stores (n = 4096, batch 2): the C2-style decode step
(k5_prep + k1_dense_sum + k5_attend_bulk with the prologue top-K +
k5_merge_rows), kvb_select + kvb_attend (K2a/K2b, token attention), the
tcgen05 reconstruction path (k3_recon_logits, k_path 2), the HIGGS
tensor-core scan + Appendix-E residual stages, the FP8 slow tier (token
kernel decode), the tier gather, prefill builds and one batch-1 append.
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2604_08426_b200 import schemes as S  # noqa: E402
from paper_2604_08426_b200.store import DeviceStore  # noqa: E402


def main():
    torch.cuda.set_device(0)
    g = torch.Generator(device="cuda").manual_seed(0)
    B, n, H, G, D = 2, int(sys.argv[1]) if len(sys.argv) > 1 else 4096, 8, 4, 128
    k = torch.randn((B, n, H, D), generator=g, device="cuda").bfloat16()
    v = torch.randn((B, n, H, D), generator=g, device="cuda").bfloat16()
    q = torch.randn((B, H, G, D), generator=g, device="cuda")
    # ShadowKV decode step (bulk attention, prologue top-K) + K3 reconstruction
    st = DeviceStore(batch=B, n_tokens=n, kv_heads=H, head_dim=D, chunk_size=8, dtype=torch.bfloat16,
                     landmark=S.scheme_none(), slow=S.scheme_svd(160, H * D), svd_groups=1,
                     outlier_tokens=64, local_window=32)
    st.build(k, v)
    K = st.n_select(min(256, n // 16) / n)
    for kp in (0, 2):
        plan = st.decode_plan(G, K, k_path=kp)
        plan.run(q)
    cid, sc, tok, ntok = st.select(q, K)
    st.attend(q, tok, ntok)
    st.gather_kv(0, tok[0, :16].contiguous())
    st.close()
    # HIGGS 2-bit @ chunk 1 tensor-core scan + K2a/K2b + attention
    st = DeviceStore(batch=B, n_tokens=n, kv_heads=H, head_dim=D, chunk_size=1, dtype=torch.bfloat16,
                     landmark=S.scheme_higgs(2), outlier_tokens=0, local_window=32)
    st.build(k, v)
    plan = st.decode_plan(G, st.n_select(min(256, n // 16) / n))
    plan.run(q)
    st.close()
    # Appendix E: 4-bit @ 8 landmarks + 1-bit residuals, both stages
    st = DeviceStore(batch=B, n_tokens=n, kv_heads=H, head_dim=D, chunk_size=8, dtype=torch.bfloat16,
                     landmark=S.scheme_higgs(4), residual=S.scheme_higgs(1), outlier_tokens=0,
                     local_window=32)
    st.build(k, v)
    for exact in (True, False):
        st.select_residual(q, min(256, n // 16), 4, exact=exact)
    st.close()
    # FP8 slow tier (token kernel decode path)
    st = DeviceStore(batch=B, n_tokens=n, kv_heads=H, head_dim=D, chunk_size=8, dtype=torch.bfloat16,
                     landmark=S.scheme_none(), slow=S.scheme_fp8(), outlier_tokens=64, local_window=32)
    st.build(k, v)
    st.decode_plan(G, K).run(q)
    st.close()
    # batch-1 append (capacity store)
    st = DeviceStore(batch=1, n_tokens=n - 8, kv_heads=H, head_dim=D, chunk_size=8, dtype=torch.bfloat16,
                     landmark=S.scheme_higgs(4), residual=S.scheme_higgs(1), outlier_tokens=64,
                     local_window=32, capacity=n)
    st.build(k[:1, : n - 8].contiguous(), v[:1, : n - 8].contiguous())
    for i in range(3):
        m = n - 8 + i + 1
        st.append(k[:1, :m].contiguous(), v[:1, :m].contiguous())
    st.close()
    torch.cuda.synchronize()
    print("sanitize driver done")


if __name__ == "__main__":
    main()
