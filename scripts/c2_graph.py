"""C2 write/dummy sweep timed as CUDA-graph replays of back-to-back launches
(no host launch gaps): per-launch GPU time for small N.

    python scripts/c2_graph.py [--ns 1024,4096,16384] [--strats ltm-r,bb,rec,rb,utm]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ns", default="1024,2048,4096,8192,16384")
    ap.add_argument("--strats", default="ltm-r,bb,rec,rb,utm")
    ap.add_argument("--modes", default="span")
    ap.add_argument("--kernels", default="write,dummy")
    ap.add_argument("--k", type=int, default=20)
    a = ap.parse_args()
    import torch

    from paper_1308_1419_b200 import trigrid as tg
    dev = torch.device("cuda", 0)
    for n in [int(x) for x in a.ns.split(",")]:
        buf = torch.empty(n * (n + 1) // 2, dtype=torch.int32, device=dev)
        for mode in a.modes.split(","):
            for kern in a.kernels.split(","):
                for s in a.strats.split(","):
                    st = torch.cuda.Stream(dev)
                    kw = dict(rho=16, mode=mode, stream=st, sync=False)
                    if kern == "write":
                        kw["out"] = buf
                    with torch.cuda.stream(st):
                        for _ in range(3):
                            tg.launch(kern, s, n, **kw)
                    torch.cuda.synchronize()
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g, stream=st):
                        for _ in range(a.k):
                            tg.launch(kern, s, n, **kw)
                    with torch.cuda.stream(st):
                        g.replay()
                    torch.cuda.synchronize()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    ts = []
                    with torch.cuda.stream(st):  # replay runs on the current stream
                        for _ in range(5):
                            e0.record(st)
                            g.replay()
                            e1.record(st)
                            e1.synchronize()
                            ts.append(e0.elapsed_time(e1) / a.k)
                    ts.sort()
                    print(f"n={n} {mode} {kern} {s}: {ts[2] * 1e3:.2f} us/launch", flush=True)


if __name__ == "__main__":
    main()
