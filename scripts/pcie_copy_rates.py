import torch, time
n = 64 << 20
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
streams = [torch.cuda.Stream() for _ in range(4)]
def run(k, direction):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for it in range(10):
        for i in range(k):
            s = streams[i]
            sl = slice(i * n // k, (i + 1) * n // k)
            with torch.cuda.stream(s):
                if direction == "h2d": d[sl].copy_(h[sl], non_blocking=True)
                else: h[sl].copy_(d[sl], non_blocking=True)
    torch.cuda.synchronize()
    return 10 * n / (time.perf_counter() - t0) / 1e9
for direction in ("h2d", "d2h"):
    for k in (1, 2, 4):
        print(direction, k, f"{run(k, direction):.1f} GB/s")
# both directions at once
torch.cuda.synchronize(); t0 = time.perf_counter()
for it in range(10):
    with torch.cuda.stream(streams[0]): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(streams[1]): h.copy_(d, non_blocking=True)
torch.cuda.synchronize(); print("duplex each", f"{10 * n / (time.perf_counter() - t0) / 1e9:.1f} GB/s")
