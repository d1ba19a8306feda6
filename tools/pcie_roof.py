"""PCIe copy roof for bench.py's e2e: the step's D2H (368 MB) and H2D (249 MB) as bare pinned
cudaMemcpyAsync, alone and concurrently on two streams."""
import torch, time
n = 368 * 1024 * 1024 // 4
d = torch.empty(n, device="cuda"); h = torch.empty(n).pin_memory()
n2 = 249 * 1024 * 1024 // 4
d2 = torch.empty(n2, device="cuda"); h2 = torch.empty(n2).pin_memory()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3
d2h = t(lambda: h.copy_(d, non_blocking=True))
h2d = t(lambda: d2.copy_(h2, non_blocking=True))
def both():
    with torch.cuda.stream(s1): h.copy_(d, non_blocking=True)
    with torch.cuda.stream(s2): d2.copy_(h2, non_blocking=True)
bo = t(both)
print(f"D2H 368MB {d2h:.2f} ms {368*1.048576/d2h:.1f} GB/s; H2D 249MB {h2d:.2f} ms {249*1.048576/h2d:.1f} GB/s; both {bo:.2f} ms")
# chunked D2H (8 chunks)
ch = n // 8
def chunked():
    for i in range(8): h[i*ch:(i+1)*ch].copy_(d[i*ch:(i+1)*ch], non_blocking=True)
print(f"D2H 8 chunks {t(chunked):.2f} ms")
