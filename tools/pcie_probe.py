import torch, time
for mb in (2, 16, 144, 288):
    h = torch.empty(mb * 1024 * 1024 // 8, dtype=torch.float64).pin_memory()
    d = torch.empty_like(h, device="cuda")
    for _ in range(3): d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10): d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    t = (time.perf_counter() - t0) / 10
    print(f"H2D {mb} MB: {t*1e3:.3f} ms  {mb/1024/t:.1f} GiB/s")
    t0 = time.perf_counter()
    for _ in range(10): h.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    t = (time.perf_counter() - t0) / 10
    print(f"D2H {mb} MB: {t*1e3:.3f} ms  {mb/1024/t:.1f} GiB/s")
