"""Pinned D2H bandwidth of a 64 MiB result-sized copy: one stream vs chunks over several streams."""
import time
import torch

n = 64 << 20
src = torch.empty(n, dtype=torch.uint8, device="cuda").random_()
dst = torch.empty(n, dtype=torch.uint8, pin_memory=True)
streams = [torch.cuda.Stream() for _ in range(4)]
for ns in (1, 2, 4):
    for chunks in (1, 4, 8):
        ts = []
        for _ in range(6):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            cs = n // chunks
            for c in range(chunks):
                s = streams[c % ns]
                s.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(s):
                    dst[c * cs:(c + 1) * cs].copy_(src[c * cs:(c + 1) * cs], non_blocking=True)
            for s in streams[:ns]:
                s.synchronize()
            ts.append(time.perf_counter() - t0)
        t = sorted(ts)[len(ts) // 2]
        print(f"streams {ns} chunks {chunks}: {t * 1e3:.2f} ms  {n / t / 1e9:.1f} GB/s")
