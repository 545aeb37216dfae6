import torch, time
n_in, n_out = 240_000_000, 440_000_000
hi = torch.empty(n_in, dtype=torch.uint8).pin_memory(); ho = torch.empty(n_out, dtype=torch.uint8).pin_memory()
di = torch.empty(n_in, dtype=torch.uint8, device="cuda"); do = torch.empty(n_out, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(2):
    di.copy_(hi, non_blocking=True); ho.copy_(do, non_blocking=True)
torch.cuda.synchronize()
def t(f, k=5):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(k): f()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / k
h2d = t(lambda: di.copy_(hi, non_blocking=True)); d2h = t(lambda: ho.copy_(do, non_blocking=True))
def both():
    with torch.cuda.stream(s1): di.copy_(hi, non_blocking=True)
    with torch.cuda.stream(s2): ho.copy_(do, non_blocking=True)
bo = t(both)
print(f"H2D {n_in/h2d/1e9:.1f} GB/s ({h2d*1e3:.2f} ms)  D2H {n_out/d2h/1e9:.1f} GB/s ({d2h*1e3:.2f} ms)  both concurrently {bo*1e3:.2f} ms")
