import torch, time
for mb in (16, 75, 256):
    n = mb * 1024 * 1024 // 4
    d = torch.empty(n, device='cuda'); h = torch.empty(n).pin_memory()
    for direction in ('d2h', 'h2d'):
        for _ in range(3):
            (h.copy_(d, non_blocking=True) if direction == 'd2h' else d.copy_(h, non_blocking=True))
        torch.cuda.synchronize()
        t = time.perf_counter(); reps = 10
        for _ in range(reps):
            (h.copy_(d, non_blocking=True) if direction == 'd2h' else d.copy_(h, non_blocking=True))
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t) / reps
        print(f"{direction} {mb} MB: {mb/1024/dt:.1f} GB/s")
# both directions at once on two streams
n = 75 * 1024 * 1024 // 4
d1 = torch.empty(n, device='cuda'); h1 = torch.empty(n).pin_memory(); d2 = torch.empty(n, device='cuda'); h2 = torch.empty(n).pin_memory()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(10):
    with torch.cuda.stream(s1): h1.copy_(d1, non_blocking=True)
    with torch.cuda.stream(s2): d2.copy_(h2, non_blocking=True)
torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 10
print(f"duplex 75 MB each way: {75/1024/dt:.1f} GB/s per direction")
