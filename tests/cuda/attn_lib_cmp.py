"""Developer comparison: dense attention libraries at the cfg2 attention shape
(B=32, M=512, H=12, head_dim 64, bf16) on the same B200 -- the materialised
baseline the rank-space kernel replaces."""
import torch
import torch.nn.functional as F


def t(f, reps=50):
    for _ in range(5):
        f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        f()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


B, M, H, D = 32, 512, 12, 64
q, k, v = (torch.randn(B, H, M, D, device="cuda", dtype=torch.bfloat16) for _ in range(3))
for name, be in (("cudnn", torch.nn.attention.SDPBackend.CUDNN_ATTENTION),
                 ("flash", torch.nn.attention.SDPBackend.FLASH_ATTENTION),
                 ("efficient", torch.nn.attention.SDPBackend.EFFICIENT_ATTENTION)):
    try:
        with torch.nn.attention.sdpa_kernel(be):
            us = t(lambda: F.scaled_dot_product_attention(q, k, v))
        print(f"torch sdpa[{name}] B={B} M={M} H={H} d={D}: {us:7.1f} us")
    except Exception as e:
        print(f"torch sdpa[{name}]: unavailable ({str(e).splitlines()[0][:80]})")
try:
    from flash_attn import flash_attn_func
    qq, kk, vv = (x.transpose(1, 2).contiguous() for x in (q, k, v))
    us = t(lambda: flash_attn_func(qq, kk, vv))
    print(f"flash_attn {B}x{M}x{H}x{D}: {us:7.1f} us")
except Exception as e:
    print(f"flash_attn: unavailable ({str(e).splitlines()[0][:80]})")
