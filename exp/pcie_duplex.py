"""PCIe copy rates on the box: H2D alone, D2H alone, both at once (two streams), pinned host memory."""
import time, torch
n = 256 << 20  # bytes
h1 = torch.empty(n, dtype=torch.uint8).pin_memory(); h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d1 = torch.empty(n, dtype=torch.uint8, device="cuda"); d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def run(h2d, d2h, reps=8):
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(reps):
        if h2d:
            with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize(); dt = time.perf_counter() - t
    return reps * n * (int(h2d) + int(d2h)) / dt / 1e9
for _ in range(2): run(True, True, 2)
print(f"H2D {run(True, False):.1f} GB/s  D2H {run(False, True):.1f} GB/s  both {run(True, True):.1f} GB/s aggregate")
