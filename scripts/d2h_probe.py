"""D2H bandwidth probe for the e2e path (8.59 GB packed EDM to pinned host memory)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
n = 8590065664 // 4
g = torch.empty(n, dtype=torch.float32, device="cuda").fill_(1.0)
h = torch.empty(n, dtype=torch.float32, pin_memory=True)


def run(chunk_mb, nstreams):
    streams = [torch.cuda.Stream() for _ in range(nstreams)]
    torch.cuda.synchronize()
    t = time.perf_counter()
    if chunk_mb == 0:
        h.copy_(g, non_blocking=True)
    else:
        c = chunk_mb * 1024 * 1024 // 4
        for k, s0 in enumerate(range(0, n, c)):
            with torch.cuda.stream(streams[k % nstreams]):
                h[s0:s0 + c].copy_(g[s0:s0 + c], non_blocking=True)
    torch.cuda.synchronize()
    return time.perf_counter() - t


for rep in range(2):
    for cm, ns in [(0, 1), (256, 1), (256, 2), (512, 2), (128, 4), (1024, 2)]:
        dt = run(cm, ns)
        print(f"rep{rep} D2H chunk={cm}MB streams={ns}: {dt * 1e3:.1f} ms, {4 * n / dt / 1e9:.1f} GB/s", flush=True)
if "--e2e" in sys.argv:
    import numpy as np

    from paper_1308_1419_b200 import trigrid as tg
    del g
    pts = tg.gen_values(65536 * 3, 42).view(65536, 3).cpu().numpy()
    hp = torch.from_numpy(pts).pin_memory().numpy()
    ho = h.numpy()
    for rep in range(3):
        t = time.perf_counter()
        tg.edm_strategy("ltm-r", hp, 16, out=ho)
        dt = time.perf_counter() - t
        print(f"e2e edm_strategy: {dt * 1e3:.1f} ms ({4 * n / dt / 1e9:.1f} GB/s)", flush=True)
