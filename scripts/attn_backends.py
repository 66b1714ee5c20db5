import torch, time
from torch.nn.attention import sdpa_kernel, SDPBackend
B,H,S,D=8,32,2048,64
q=torch.randn(B,H,S,D,device='cuda',dtype=torch.bfloat16)
k=torch.randn_like(q); v=torch.randn_like(q)
fl = 4*B*H*S*S*D/2
for name,be in [("cudnn",SDPBackend.CUDNN_ATTENTION),("flash",SDPBackend.FLASH_ATTENTION),("eff",SDPBackend.EFFICIENT_ATTENTION)]:
    try:
        with sdpa_kernel(be):
            for _ in range(3): torch.nn.functional.scaled_dot_product_attention(q,k,v,is_causal=True)
            torch.cuda.synchronize()
            e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20): torch.nn.functional.scaled_dot_product_attention(q,k,v,is_causal=True)
            e1.record(); torch.cuda.synchronize()
            ms=e0.elapsed_time(e1)/20
            print(name, f"{ms*1e3:.1f} us {fl/ms/1e9:.0f} TF/s")
    except Exception as ex: print(name, "fail", str(ex)[:100])
try:
    import flashinfer
    print("flashinfer", flashinfer.__version__)
    from flashinfer import prefill
    print([n for n in dir(flashinfer) if 'prefill' in n.lower()][:20])
except Exception as ex: print("flashinfer import fail", ex)
try:
    import flash_attn
    from flash_attn import flash_attn_func
    qq=q.transpose(1,2).contiguous(); kk=k.transpose(1,2).contiguous(); vv=v.transpose(1,2).contiguous()
    for _ in range(3): flash_attn_func(qq,kk,vv,causal=True)
    torch.cuda.synchronize()
    e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): flash_attn_func(qq,kk,vv,causal=True)
    e1.record(); torch.cuda.synchronize()
    ms=e0.elapsed_time(e1)/20
    print("flash_attn pkg", flash_attn.__version__, f"{ms*1e3:.1f} us {fl/ms/1e9:.0f} TF/s")
except Exception as ex: print("flash_attn fail", str(ex)[:200])
