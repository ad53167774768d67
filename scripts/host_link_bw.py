import torch, time
n = 256 << 20
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for pinned in (True,):
    h = torch.empty(n, dtype=torch.uint8, pin_memory=pinned)
    for name, fn in (("H2D", lambda: d.copy_(h, non_blocking=True)), ("D2H", lambda: h.copy_(d, non_blocking=True))):
        fn(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5): fn()
        e1.record(); torch.cuda.synchronize()
        print(name, "pinned" if pinned else "pageable", f"{5 * n / e0.elapsed_time(e1) / 1e6:.1f} GB/s")
# two streams D2H halves
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(5):
    with torch.cuda.stream(s1): h[: n // 2].copy_(d[: n // 2], non_blocking=True)
    with torch.cuda.stream(s2): h[n // 2 :].copy_(d[n // 2 :], non_blocking=True)
torch.cuda.synchronize(); print("D2H 2 streams", f"{5 * n / (time.perf_counter() - t) / 1e9:.1f} GB/s")
# bidirectional
h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True); d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(5):
    with torch.cuda.stream(s1): d2.copy_(h2, non_blocking=True)
    with torch.cuda.stream(s2): h.copy_(d, non_blocking=True)
torch.cuda.synchronize(); print("bidir each", f"{5 * n / (time.perf_counter() - t) / 1e9:.1f} GB/s")
import subprocess; print(subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout[:600])
print(subprocess.run(["bash", "-c", "nproc; numactl -H 2>/dev/null | head -3; lscpu | grep -i numa"], capture_output=True, text=True).stdout)
