"""Pinned H2D bandwidth of the C5 COO (2 x 8.6 GB): one stream vs the two
arrays on two streams vs 4/8 chunks round-robin over streams."""
import time
import torch

n = 1 << 31
a = torch.empty(n, dtype=torch.int32).pin_memory()
b = torch.empty(n, dtype=torch.int32).pin_memory()
da = torch.empty(n, dtype=torch.int32, device="cuda")
db = torch.empty(n, dtype=torch.int32, device="cuda")


def run(nstreams, chunks):
    ss = [torch.cuda.Stream() for _ in range(nstreams)]
    torch.cuda.synchronize()
    t = time.perf_counter()
    k = 0
    for src, dst in ((a, da), (b, db)):
        step = n // chunks
        for c in range(chunks):
            with torch.cuda.stream(ss[k % nstreams]):
                dst[c * step:(c + 1) * step].copy_(src[c * step:(c + 1) * step], non_blocking=True)
            k += 1
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    return 8 * n / dt / 1e9


for cfg in [(1, 1), (2, 1), (2, 4), (4, 8), (1, 1), (2, 1)]:
    print("streams %d chunks/array %d: %.1f GB/s" % (cfg[0], cfg[1], run(*cfg)))
