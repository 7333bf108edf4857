"""D2H bandwidth of the L=8 solution (134 MB) into pinned host memory: one copy vs chunks on
several streams (developer tool; the e2e leg of bench.py copies this much every step)."""
import time
import torch

nbytes = 65536 * 256 * 8
src = torch.empty(nbytes // 8, dtype=torch.float64, device="cuda").normal_()
dst = torch.empty(nbytes // 8, dtype=torch.float64).pin_memory()
print("pinned:", dst.is_pinned())


def run(nchunks, reps=6):
    streams = [torch.cuda.Stream() for _ in range(nchunks)]
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        n = src.numel()
        for i, s in enumerate(streams):
            a, b = i * n // nchunks, (i + 1) * n // nchunks
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                dst[a:b].copy_(src[a:b], non_blocking=True)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    best = min(ts[1:])
    print(f"chunks {nchunks}: best {best * 1e3:.2f} ms = {nbytes / best / 1e9:.1f} GB/s; all "
          + " ".join(f"{t * 1e3:.1f}" for t in ts))


for c in (1, 2, 4, 8):
    run(c)
