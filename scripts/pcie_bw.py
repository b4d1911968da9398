import torch, time
x = torch.empty(462_000_000 // 8, dtype=torch.int64).pin_memory()
y = torch.empty_like(x, device='cuda')
for _ in range(3):
    torch.cuda.synchronize(); t=time.perf_counter(); y.copy_(x, non_blocking=True); torch.cuda.synchronize(); dt=time.perf_counter()-t
print("H2D DMA GB/s", x.numel()*8/dt/1e9)
z = torch.empty_like(x)
z = z.pin_memory()
for _ in range(3):
    torch.cuda.synchronize(); t=time.perf_counter(); z.copy_(y, non_blocking=True); torch.cuda.synchronize(); dt=time.perf_counter()-t
print("D2H DMA GB/s", x.numel()*8/dt/1e9)
# concurrent H2D + D2H on two streams
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
y2 = torch.empty_like(y)
for _ in range(3):
    torch.cuda.synchronize(); t=time.perf_counter()
    with torch.cuda.stream(s1): y2.copy_(x, non_blocking=True)
    with torch.cuda.stream(s2): z.copy_(y, non_blocking=True)
    torch.cuda.synchronize(); dt=time.perf_counter()-t
print("H2D+D2H concurrent GB/s each", x.numel()*8/dt/1e9)
