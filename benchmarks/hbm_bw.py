import torch
def t(fn, reps=10):
    for _ in range(3): fn()
    a,b=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); b.synchronize(); return a.elapsed_time(b)/reps
n=1<<30
x=torch.empty(n,dtype=torch.uint8,device='cuda'); y=torch.empty_like(x)
ms=t(lambda: x.fill_(1)); print('write-only 1GiB: %.1f us  %.0f GB/s'%(ms*1e3, n/ms/1e6))
ms=t(lambda: y.copy_(x)); print('copy 1GiB: %.1f us  %.0f GB/s (r+w)'%(ms*1e3, 2*n/ms/1e6))
ms=t(lambda: x.sum(dtype=torch.int64)); print('read-only 1GiB: %.1f us  %.0f GB/s'%(ms*1e3, n/ms/1e6))
