import torch, time
n = 800_000_000
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for chunk in [n, 64 << 20, 16 << 20]:
    s = torch.cuda.Stream()
    torch.cuda.synchronize()
    for rep in range(2):
        t0 = time.perf_counter()
        with torch.cuda.stream(s):
            for o in range(0, n, chunk):
                d[o:o + chunk].copy_(h[o:o + chunk], non_blocking=True)
        s.synchronize()
        dt = time.perf_counter() - t0
    print(f"chunk {chunk>>20} MB: {n/dt/1e9:.1f} GB/s")
# two streams concurrently
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize()
t0 = time.perf_counter()
with torch.cuda.stream(s1):
    d[:n//2].copy_(h[:n//2], non_blocking=True)
with torch.cuda.stream(s2):
    d[n//2:].copy_(h[n//2:], non_blocking=True)
torch.cuda.synchronize()
print(f"two streams: {n/(time.perf_counter()-t0)/1e9:.1f} GB/s")
