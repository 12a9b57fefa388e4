"""Run one td-kernel configuration a few times (for ncu -k regex:... captures).

    python scripts/prof_driver.py edm   --n 65536 --d 3  --strategy ltm-r [--mode span|grid|gram]
    python scripts/prof_driver.py write --n 65536 --strategy ltm-r
    python scripts/prof_driver.py collide --n 32768
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("kernel", choices=["edm", "write", "collide", "dummy"])
    ap.add_argument("--n", type=int, default=65536)
    ap.add_argument("--d", type=int, default=3)
    ap.add_argument("--strategy", default="ltm-r")
    ap.add_argument("--mode", default="auto")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--time", action="store_true", help="print the median launch time (CUDA events)")
    a = ap.parse_args()
    import torch

    from paper_1308_1419_b200 import trigrid as tg
    n = a.n
    if a.kernel == "collide":
        sph = tg.gen_values(n * 4, 42).view(n, 4)
        ts = []
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            tg.collide(sph, 0.0625, strategy=a.strategy, mode=a.mode)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        if a.time:
            ts.sort()
            ms = ts[len(ts) // 2]
            print(f"collide n={n} {a.strategy} mode={a.mode}: median {ms:.4f} ms "
                  f"({n * (n - 1) / 2 / ms / 1e9:.1f} G pairs/s) over {a.reps}")
    elif a.kernel == "dummy":
        ts = []
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            tg.launch("dummy", a.strategy, n, mode=a.mode)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        if a.time:
            ts.sort()
            print(f"dummy n={n} {a.strategy} mode={a.mode}: median {ts[len(ts) // 2]:.4f} ms over {a.reps}")
    else:
        out = torch.empty(n * (n + 1) // 2, dtype=torch.float32 if a.kernel == "edm" else torch.int32, device="cuda")
        pts = tg.gen_values(n * a.d, 42).view(n, a.d) if a.kernel == "edm" else None
        ts = []
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            tg.launch(a.kernel, a.strategy, n, points=pts, out=out, d=a.d if pts is not None else 0, mode=a.mode)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        if a.time:
            ts.sort()
            ms = ts[len(ts) // 2]
            print(f"{a.kernel} n={n} d={a.d} {a.strategy} mode={a.mode}: median {ms:.4f} ms "
                  f"({4 * n * (n + 1) / 2 / ms / 1e6:.1f} GB/s of packed output) over {a.reps}")
    torch.cuda.synchronize()
    print("done")


if __name__ == "__main__":
    main()
