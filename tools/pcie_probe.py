"""PCIe copy rates on the box (pinned host memory): D2H / H2D alone, D2H split over two
streams, D2H concurrent with H2D — the ceiling of bench.py's e2e (3.07 GB D2H per c2 step)."""
import torch
G = 1 << 30
dev = torch.empty(3 * G, dtype=torch.uint8, device="cuda")
host = torch.empty(3 * G, dtype=torch.uint8).pin_memory()
din = torch.empty(int(0.69 * G), dtype=torch.uint8, device="cuda")
hin = torch.empty(int(0.69 * G), dtype=torch.uint8).pin_memory()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

def timed(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        torch.cuda.synchronize()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best

def d2h1():
    with torch.cuda.stream(s1):
        host.copy_(dev, non_blocking=True)
def d2h2():
    h = dev.numel() // 2
    with torch.cuda.stream(s1):
        host[:h].copy_(dev[:h], non_blocking=True)
    with torch.cuda.stream(s2):
        host[h:].copy_(dev[h:], non_blocking=True)
def h2d():
    with torch.cuda.stream(s1):
        din.copy_(hin, non_blocking=True)
def both():
    with torch.cuda.stream(s1):
        host.copy_(dev, non_blocking=True)
    with torch.cuda.stream(s2):
        din.copy_(hin, non_blocking=True)
for name, fn, nb in [("D2H 3 GB, 1 stream", d2h1, 3 * G), ("D2H 3 GB, 2 streams", d2h2, 3 * G),
                     ("H2D 0.69 GB", h2d, int(0.69 * G)), ("D2H 3 GB + H2D 0.69 GB", both, 3 * G)]:
    ms = timed(fn)
    print("%-26s %8.2f ms  %6.1f GB/s (of the D2H / H2D bytes)" % (name, ms, nb / ms / 1e6), flush=True)
