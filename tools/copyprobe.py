import torch, time
for mb in (22, 88, 128):
    n = mb * 1024 * 1024 // 4
    h = torch.empty(n, dtype=torch.int32).pin_memory()
    d = torch.empty(n, dtype=torch.int32, device="cuda")
    for _ in range(3):
        d.copy_(h, non_blocking=True); torch.cuda.synchronize()
    t0 = time.perf_counter(); d.copy_(h, non_blocking=True); torch.cuda.synchronize(); t1 = time.perf_counter()
    h.copy_(d, non_blocking=True); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"{mb} MB: H2D {mb/1024/(t1-t0):.1f} GB/s, D2H {mb/1024/(t2-t1):.1f} GB/s")
