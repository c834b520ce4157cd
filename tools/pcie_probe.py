import torch, time
d = torch.empty(56 << 20, dtype=torch.uint8, device="cuda")
h = torch.empty(56 << 20, dtype=torch.uint8).pin_memory()
hi = torch.empty(9 << 20, dtype=torch.uint8).pin_memory()
di = torch.empty(9 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3): h.copy_(d, non_blocking=True); torch.cuda.synchronize()
t=time.perf_counter()
for _ in range(20): h.copy_(d, non_blocking=True)
torch.cuda.synchronize(); dt=(time.perf_counter()-t)/20
print("D2H 56MB GB/s", 56*2**20/dt/1e9)
s2 = torch.cuda.Stream()
t=time.perf_counter()
for _ in range(20):
    h.copy_(d, non_blocking=True)
    with torch.cuda.stream(s2): di.copy_(hi, non_blocking=True)
torch.cuda.synchronize(); dt=(time.perf_counter()-t)/20
print("D2H 56MB + concurrent H2D 9MB per iter: ms", dt*1e3, "D2H GB/s", 56*2**20/dt/1e9)
