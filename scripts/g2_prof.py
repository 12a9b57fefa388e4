"""Gram-kernel wait-time breakdown (needs the TG_G2_PROF=1 variant build:
python -m paper_1308_1419_b200.build --variant prof TG_G2_PROF=1; run with
TG_LIB_PATH=paper_1308_1419_b200/libtrigrid_b200_prof.so)."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1308_1419_b200 import _lib, trigrid as tg  # noqa: E402

n, d = int(sys.argv[1]) if len(sys.argv) > 1 else 65536, int(sys.argv[2]) if len(sys.argv) > 2 else 64
pts = tg.gen_values(n * d, 42).view(n, d)
out = torch.empty(n * (n + 1) // 2, dtype=torch.float32, device="cuda")
L = _lib.load()
buf = (ctypes.c_ulonglong * 16)()
tg.launch("edm", "ltm-r", n, points=pts, out=out, d=d, mode="gram")
L.tg_debug_g2_prof(buf, 1)
tg.launch("edm", "ltm-r", n, points=pts, out=out, d=d, mode="gram")
torch.cuda.synchronize()
L.tg_debug_g2_prof(buf, 0)
names = ["prod:norm_empty", "prod:a_empty", "prod:b_empty", "mma:a_full", "mma:acc_empty", "mma:b_full",
         "epi:norm_full", "epi:acc_full", "epi:total(warp2 lane0)", "mma:total", "prod:total"]
tot = {"prod": buf[10], "mma": buf[9], "epi": buf[8]}
for k, nm in enumerate(names):
    role = nm.split(":")[0]
    print(f"{nm:24s} {buf[k] / 148:14.0f} cyc/CTA  {100 * buf[k] / max(tot[role], 1):6.1f}% of {role}")
