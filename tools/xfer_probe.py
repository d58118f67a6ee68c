import torch, time
dev=torch.device('cuda',0)
n=1<<20
h=[torch.randn(n,dtype=torch.float64).pin_memory() for _ in range(4)]
d=[torch.empty(n,dtype=torch.float64,device=dev) for _ in range(4)]
o=torch.empty((2,n),dtype=torch.float64,device=dev); ho=torch.empty((2,n),dtype=torch.float64).pin_memory()
s=torch.cuda.current_stream()
for rep in range(3):
    a=torch.cuda.Event(enable_timing=True); b=torch.cuda.Event(enable_timing=True); c=torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(4): d[i].copy_(h[i],non_blocking=True)
    b.record()
    ho.copy_(o,non_blocking=True)
    c.record(); c.synchronize()
    print('h2d 32MB %.3f ms  d2h 16MB %.3f ms'%(a.elapsed_time(b), b.elapsed_time(c)))
# two streams concurrently h2d
s2=torch.cuda.Stream()
a=torch.cuda.Event(enable_timing=True); b=torch.cuda.Event(enable_timing=True)
a.record()
d[0].copy_(h[0],non_blocking=True); d[1].copy_(h[1],non_blocking=True)
with torch.cuda.stream(s2):
    d[2].copy_(h[2],non_blocking=True); d[3].copy_(h[3],non_blocking=True)
s.wait_stream(s2); b.record(); b.synchronize()
print('h2d 2 streams %.3f'%a.elapsed_time(b))
