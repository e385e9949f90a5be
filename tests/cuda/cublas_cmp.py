import torch, time
torch.backends.cuda.matmul.allow_bf16_reduced_precision_reduction = True
def t(f, reps=50):
    for _ in range(5): f()
    torch.cuda.synchronize()
    a=torch.cuda.Event(enable_timing=True); b=torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): f()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b)/reps*1e3
for (M,N,K) in [(16384,1152,768),(16384,768,384),(16384,384,768),(16384,3072,384),(16384,384,3072),(8192,8192,8192)]:
    A=torch.randn(M,K,device='cuda').bfloat16(); B=torch.randn(N,K,device='cuda').bfloat16()
    us=t(lambda: torch.matmul(A,B.t()))
    print(f"cublas M={M} N={N} K={K}: {us:7.1f} us {2*M*N*K/us/1e6:7.0f} TF/s", flush=True)
