"""Host->device bandwidth of pinned buffers on this box (design check for the
host entry points): one stream vs two streams, 18 MB (the C2 step's inputs)."""
import time

import torch

n = 18_257_024
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for name, split in (("1 stream", 1), ("2 streams", 2), ("4 chunks 2 streams", 4)):
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(50):
            k = n // split
            for i in range(split):
                st = s1 if i % 2 == 0 else s2
                with torch.cuda.stream(st):
                    d[i * k:(i + 1) * k if i < split - 1 else n].copy_(h[i * k:(i + 1) * k if i < split - 1 else n], non_blocking=True)
            torch.cuda.synchronize()
        t = (time.perf_counter() - t0) / 50
    print(f"{name}: {t * 1e6:.1f} us per 18.26 MB = {n / t / 1e9:.1f} GB/s")
