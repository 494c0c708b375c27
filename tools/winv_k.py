import sys, torch, time
sys.path.insert(0,'.')
from paper_2310_20285_b200 import kernels as K
for n,k in ((100000,800),(1000000,320),(100000,1),(1000000,8)):
    C=10
    pi=torch.softmax(torch.randn(n,C,device='cuda'),1).reshape(-1).contiguous()
    V=torch.randn(k,n*C,device='cuda')
    for _ in range(2): K.softmax_winv(pi,n,C,V)
    torch.cuda.synchronize()
    a,b=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    a.record(); K.softmax_winv(pi,n,C,V); b.record(); torch.cuda.synchronize()
    ms=a.elapsed_time(b); print(n,k,f"{ms:.3f} ms", f"{(2*k+1)*n*C*4/ms/1e6:.0f} GB/s")
