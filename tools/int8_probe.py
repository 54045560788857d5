import torch, time
def bench(fn, reps=5):
    fn(); torch.cuda.synchronize()
    best=1e9
    for _ in range(reps):
        e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); e1.synchronize(); best=min(best,e0.elapsed_time(e1))
    return best
for (M,N,K) in [(2048,2048,131072),(2048,2048,65536),(8192,8192,8192),(4194304//4,1024,1024),(1048576,2048,2048)]:
    a=torch.randint(-128,127,(M,K),dtype=torch.int8,device='cuda')
    b=torch.randint(-128,127,(N,K),dtype=torch.int8,device='cuda').t()   # K x N column-major
    try:
        ms=bench(lambda: torch._int_mm(a,b))
        print(M,N,K,'int_mm ms',round(ms,3),'TOPS',round(2*M*N*K/ms/1e9,1), flush=True)
    except Exception as e: print('fail',M,N,K,e)
    del a,b
a=torch.randn(8192,8192,dtype=torch.float64,device='cuda'); 
ms=bench(lambda: a@a); print('dgemm 8192 TF', 2*8192**3/ms/1e9)
h=torch.randn(8192,8192,dtype=torch.bfloat16,device='cuda'); ms=bench(lambda: h@h); print('bf16 8192 TF', 2*8192**3/ms/1e9)
