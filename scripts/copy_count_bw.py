import torch, time
m = 613
for name, nbytes in (("lat 785KB", 5 * m * 64 * 4), ("S 4.9KB", 8 * m)):
    hs = [torch.empty(nbytes, dtype=torch.uint8, pin_memory=True) for _ in range(1000)]
    d = torch.empty(nbytes * 1000, dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    for it in range(2):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        with torch.cuda.stream(s):
            e0.record(s)
            for i, h in enumerate(hs):
                d[i * nbytes:(i + 1) * nbytes].copy_(h, non_blocking=True)
            e1.record(s)
        t1 = time.perf_counter(); s.synchronize()
        print(f"{name} x1000: host issue {1e3*(t1-t0):.1f} ms, device {e0.elapsed_time(e1):.2f} ms, {nbytes*1000/e0.elapsed_time(e1)/1e6:.1f} GB/s")
