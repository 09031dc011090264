import torch, time
d = torch.empty(44_000_000, dtype=torch.uint8, device="cuda")
h = torch.empty(44_000_000, dtype=torch.uint8).pin_memory()
s = torch.cuda.Stream()
for chunks in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(chunks)]
    n = d.numel() // chunks
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(20):
        for i, st in enumerate(streams):
            with torch.cuda.stream(st):
                h[i*n:(i+1)*n].copy_(d[i*n:(i+1)*n], non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 20
    print(f"D2H 44 MB in {chunks} streams: {dt*1e3:.3f} ms, {44e6/dt/1e9:.1f} GB/s")
