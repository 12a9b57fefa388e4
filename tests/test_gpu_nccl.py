"""The N > 1 collective path over NCCL (the backend bench.py uses on real
multi-GPU boxes), on the one GPU of the test box: a single-rank NCCL group
runs multi.max_over_ranks / multi.reduce_hits on CUDA tensors next to a
sharded collision launch, so the NCCL code path of the product is initialised
and exercised (the 2-rank tests share one GPU and therefore use gloo)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import json, os, sys
sys.path.insert(0, os.environ["TG_ROOT"])
import torch, torch.distributed as dist
from paper_1308_1419_b200 import multi, trigrid as tg
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
dist.init_process_group("nccl", device_id=dev)
assert dist.get_backend() == "nccl"
n, r_max, G = 4096, 0.0625, 4
sph = tg.gen_values(n * 4, 42, dev).view(n, 4)
_, whole = tg.collide(sph, r_max, strategy="ltm-r")
parts = []
for g in range(G):
    _, h = tg.collide(sph, r_max, strategy="ltm-r", shard=(g, G))
    parts.append(h)
hits = torch.cat(parts)                       # int64 on the GPU
total = torch.tensor([int(hits.sum().item())], dtype=torch.int64, device=dev)
dist.all_reduce(total, op=dist.ReduceOp.SUM)  # one-rank NCCL all-reduce of a device tensor
t = multi.max_over_ranks(1.25, device=dev)
s = multi.reduce_hits(total.clone(), device=dev)
dist.barrier()
dist.destroy_process_group()
print(json.dumps({"whole": int(whole.item()), "total": int(total.item()), "max": t, "reduced": s}))
"""


def test_nccl_single_rank_collectives():
    env = dict(os.environ, TG_ROOT=ROOT, MASTER_ADDR="127.0.0.1", MASTER_PORT="29547", RANK="0",
               WORLD_SIZE="1", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, "-c", SCRIPT], cwd=ROOT, capture_output=True, text=True, timeout=600,
                       env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    import json
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert d["total"] == d["whole"] == d["reduced"] and d["whole"] > 0
    assert d["max"] == 1.25
