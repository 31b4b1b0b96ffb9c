import torch, time
N=65536
d=torch.empty((4096,N),dtype=torch.float32,device='cuda')
h=torch.empty((4096,N),dtype=torch.float32).pin_memory()
s=torch.cuda.Stream()
for rows in (4096,64,8,1):
    torch.cuda.synchronize(); t0=time.perf_counter()
    with torch.cuda.stream(s):
        for r in range(0,4096,rows):
            h[r:r+rows].copy_(d[r:r+rows],non_blocking=True)
    s.synchronize(); t=time.perf_counter()-t0
    print(f"rows per copy {rows}: {4096*N*4/t/1e9:.1f} GB/s ({t*1e3:.1f} ms for 1 GiB)")
