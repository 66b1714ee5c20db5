import torch, time, os
import flashinfer
B,H,S,D=8,32,2048,64
q=torch.randn(B*S,H,D,device='cuda',dtype=torch.bfloat16)
k=torch.randn_like(q); v=torch.randn_like(q)
fl = 4*B*H*S*S*D/2
qo=torch.arange(0,B*S+1,S,device='cuda',dtype=torch.int32)
ws=torch.empty(256<<20,dtype=torch.uint8,device='cuda')
for backend in ["cutlass","trtllm-gen","fa2"]:
    try:
        t0=time.time()
        w=flashinfer.BatchPrefillWithRaggedKVCacheWrapper(ws,"NHD",backend=backend)
        w.plan(qo,qo,H,H,D,causal=True,q_data_type=torch.bfloat16)
        o=w.run(q,k,v); torch.cuda.synchronize()
        print(backend,"first call",time.time()-t0,"s")
        e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20): w.run(q,k,v)
        e1.record(); torch.cuda.synchronize()
        ms=e0.elapsed_time(e1)/20
        print(backend, f"{ms*1e3:.1f} us {fl/ms/1e9:.0f} TF/s", flush=True)
    except Exception as ex: print(backend,"fail", str(ex)[:300], flush=True)
