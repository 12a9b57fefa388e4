"""Small-N span launches for a kernel-time launch list (ncu --metrics gpu__time_duration.sum)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1308_1419_b200 import trigrid as tg  # noqa: E402

strats = sys.argv[1].split(",") if len(sys.argv) > 1 else ["bb", "ltm-r", "rec"]
sizes = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1024, 4096]
kernel = sys.argv[3] if len(sys.argv) > 3 else "write"
for n in sizes:
    wb = torch.empty(n * (n + 1) // 2, dtype=torch.int32 if kernel == "write" else torch.float32, device="cuda")
    pts = tg.gen_values(n * 3, 42).view(n, 3) if kernel == "edm" else None
    for s in strats:
        for _ in range(2):
            tg.launch(kernel, s, n, points=pts, out=wb, rho=16, mode="span")
torch.cuda.synchronize()
