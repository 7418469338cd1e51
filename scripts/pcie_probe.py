"""Raw pinned host -> device copy bandwidth (the e2e bound), one and two streams."""
import torch, time
dev = torch.device("cuda", 0)
n = 1677721600 // 16
h = torch.empty(n, dtype=torch.complex128).pin_memory()
d = torch.empty(n, dtype=torch.complex128, device=dev)
for chunks, nstreams in ((1, 1), (4, 1), (8, 2), (16, 4)):
    ss = [torch.cuda.Stream(dev) for _ in range(nstreams)]
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        cs = n // chunks
        for i in range(chunks):
            with torch.cuda.stream(ss[i % nstreams]):
                d[i * cs:(i + 1) * cs].copy_(h[i * cs:(i + 1) * cs], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(f"chunks {chunks:2d} streams {nstreams}: {n * 16 / dt / 1e9:.1f} GB/s")
