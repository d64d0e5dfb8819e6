import torch, time
N = 4 << 30  # bytes
a = torch.empty(N // 8, dtype=torch.float64, pin_memory=True)
b = torch.empty(N // 8, dtype=torch.float64, pin_memory=True)
da = torch.empty(N // 8, dtype=torch.float64, device='cuda')
db = torch.empty(N // 8, dtype=torch.float64, device='cuda')
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for rep in range(2):
    torch.cuda.synchronize(); t = time.perf_counter()
    with torch.cuda.stream(s1): da.copy_(a, non_blocking=True)
    torch.cuda.synchronize(); t1 = time.perf_counter() - t
    t = time.perf_counter()
    with torch.cuda.stream(s2): b.copy_(db, non_blocking=True)
    torch.cuda.synchronize(); t2 = time.perf_counter() - t
    t = time.perf_counter()
    with torch.cuda.stream(s1): da.copy_(a, non_blocking=True)
    with torch.cuda.stream(s2): b.copy_(db, non_blocking=True)
    torch.cuda.synchronize(); t3 = time.perf_counter() - t
    print(f"H2D {N/t1/1e9:.1f} GB/s  D2H {N/t2/1e9:.1f} GB/s  both {2*N/t3/1e9:.1f} GB/s aggregate ({t3*1e3:.0f} ms vs {1e3*(t1+t2):.0f} serial)")
