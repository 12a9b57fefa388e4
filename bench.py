#!/usr/bin/env python
"""bench.py -- headline benchmark (BASELINE.json metric) on 1..8 B200.

    python bench.py --gpus N --steps K --warmup W [--impl reference]
    torchrun --nproc-per-node N bench.py --gpus N ...   (driver, N > 1)

Workload (BASELINE.json metric "packed tri elements/s & HBM GB/s per mapping
(g(lambda) vs BB) at n=65536, 1/2/4/8 GPU"): the packed lower-triangular EDM
of gen_points(65536, 3, 42), rho=16, through the g(lambda) LTM-R mapping on
the sm_100a span kernel.  With N GPUs the lambda-range is split into N
contiguous block-row shards (one per rank, its own packed slice, no data-path
collective); total work is fixed, so scaling is "strong".

One JSON line on rank 0.  `value` = whole-job packed elements/s, device-timed
(CUDA events, max over ranks).  `e2e` = the same metric through the public
drop-in trigrid.edm_strategy with pinned host buffers (H2D of the points and
D2H of the packed result inside the timed region).  `per_mapping` = every
strategy (span and paper-faithful grid mode) for the EDM and write kernels,
with I = t_BB / t_strategy as in the reference's run_suite (bench.cpp:124-133).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "packed tri elements/s & HBM GB/s per mapping (g(λ) vs BB) at n=65536, 1/2/4/8 GPU"
UNIT = "packed tri elements/s"
N_DEFAULT, D_DEFAULT, RHO, SEED = 65536, 3, 16, 42


def tri(n: int) -> int:
    return n * (n + 1) // 2


def peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return {"hbm_gbs": d["hbm_gbs"], "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


def config(n: int, d: int, world: int, strategy: str) -> dict:
    return {
        "workload": f"packed lower-triangular EDM n={n} d={d} fp32, rho={RHO}, g(lambda) {strategy.upper()} "
                    f"span kernel, lambda-range sharded over {world} GPU(s)",
        "n": n, "d": d, "rho": RHO, "strategy": strategy, "seed": SEED,
        "parallelism": f"lambda-shard x{world}",
        "l2": f"no flush: each step writes {4 * tri(n) / 1e9:.2f} GB of packed output (> 126 MB L2); "
              f"the {4 * n * d / 1e6:.2f} MB point set stays L2-resident by design",
    }


# ------------------------------------------------------------------ clocks

class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the GPU-busy region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[str] = []
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, smax, reasons, power = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                smax = float(f[1])
                power.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        sm.sort()
        busy = [s for s in sm if s > 0]
        return {"sm_mhz": busy[len(busy) // 2] if busy else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w_max": max(power) if power else None}


# ------------------------------------------------------------------ verify

def golden_sha(n: int, d: int, rank: int, world: int):
    """The reference's sha256 of this rank's packed slice (tests/golden/
    golden_large.json, generated from oracle/_ref = the unmodified reference
    build; the GPU box has no /root/reference), or None if not recorded."""
    p = os.path.join(ROOT, "tests", "golden", "golden_large.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        g = json.load(f)
    if world == 1:
        return g.get("edm", {}).get(f"{n}|{d}", {}).get("sha256")
    sh = g.get("edm_shards", {}).get(f"{n}|{d}", {}).get(str(world))
    return sh["sha256"][rank] if sh else None


def golden_collide(n: int, r_max: float, rank: int, world: int):
    """(sha256, hits) of this rank's collision bit table (tests/golden/
    golden_large.json, from the oracle), or None."""
    p = os.path.join(ROOT, "tests", "golden", "golden_large.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        ref = json.load(f).get("collide", {}).get(f"{n}|{r_max}")
    if not ref:
        return None
    if world == 1:
        return ref["sha256"], ref["hits"]
    sh = ref.get("shards", {}).get(str(world))
    return (sh["sha256"][rank], sh["hits"][rank]) if sh else None


def sha256_device(t, chunk_bytes: int = 1 << 28) -> str:
    """sha256 of a CUDA tensor's bytes through a pinned staging buffer
    (outside every timed region)."""
    import hashlib

    import torch
    flat = t.reshape(-1).view(torch.uint8)
    h = hashlib.sha256()
    stage = torch.empty(min(chunk_bytes, flat.numel()), dtype=torch.uint8).pin_memory()
    for a in range(0, flat.numel(), chunk_bytes):
        m = min(chunk_bytes, flat.numel() - a)
        stage[:m].copy_(flat[a:a + m])
        h.update(memoryview(stage[:m].numpy()))
    return h.hexdigest()


def sha256_host(a) -> str:
    import hashlib
    h = hashlib.sha256()
    mv = memoryview(a.reshape(-1).view("u1"))
    step = 1 << 28
    for i in range(0, len(mv), step):
        h.update(mv[i:i + step])
    return h.hexdigest()


# ------------------------------------------------------------ reference arm

def cpu_reference_run(n: int, d: int, strategy: str, steps: int, warmup: int, budget_s: float | None):
    """The reference's own CPU launch_edm (oracle/_ref, compiled from
    /root/reference sources) with all host threads, into a buffer allocated
    once (as run_suite times it, bench.cpp:71-74,113-122)."""
    import ctypes as C

    import numpy as np

    import oracle
    if oracle.ref_available():
        R = oracle.ref()
        pts = oracle.gen_points(n, d, SEED)
        sess = R.ref_edm_session_create(strategy.encode(), pts.ctypes.data_as(C.POINTER(C.c_float)), n, d, RHO)
        if not sess:
            raise RuntimeError(R.ref_last_error().decode())
        cores = int(R.ref_hardware_concurrency())
        st = np.zeros(4, np.uint64)
        times = []
        try:
            for _ in range(warmup):
                R.ref_edm_session_run(sess, 0, st.ctypes.data_as(C.POINTER(C.c_uint64)))
            t_start = time.perf_counter()
            for k in range(steps):
                t0 = time.perf_counter()
                R.ref_edm_session_run(sess, 0, st.ctypes.data_as(C.POINTER(C.c_uint64)))
                times.append(time.perf_counter() - t0)
                if budget_s is not None and time.perf_counter() - t_start > budget_s and k >= 0:
                    break
        finally:
            R.ref_edm_session_destroy(sess)
        sec = sum(times) / len(times)
        return {"value": tri(n) / sec, "unit": UNIT, "cores": cores, "kind": "reference",
                "sample": f"full workload (T({n}) = {tri(n)} cells) x {len(times)} launch_edm calls, "
                          f"workers=0 (hardware_concurrency={cores}), {strategy}",
                "ms_per_step": sec * 1e3}
    # fallback: the oracle port, single thread, bounded row sample
    pts = oracle.gen_points(n, d, SEED)
    r1 = min(n, 4096)
    t0 = time.perf_counter()
    oracle.edm_rows(pts, 0, r1)
    sec = time.perf_counter() - t0
    return {"value": tri(r1) / sec, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"oracle restatement rows [0, {r1}) of n={n}, 1 thread", "ms_per_step": sec * 1e3}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    r = cpu_reference_run(args.n, args.d, args.strategy, args.steps, args.warmup, None)
    line = {
        "impl": "reference", "metric": METRIC, "value": r["value"], "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": r["ms_per_step"],
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "fp32",
        "data": f"synthetic: gen_points({args.n}, {args.d}, seed={SEED}) (splitmix64 U[0,1))",
        "config": config(args.n, args.d, args.gpus, args.strategy),
        "cpu_baseline": {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": r["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ our arm

def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1308_1419_b200 import _lib, multi
    from paper_1308_1419_b200 import trigrid as tg

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # NCCL for the (tiny) timing collectives; TG_DIST_BACKEND=gloo lets the
    # multi-rank path be exercised with several ranks on one GPU.
    backend = os.environ.get("TG_DIST_BACKEND", "nccl")
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    cdev = dev if backend == "nccl" else torch.device("cpu")

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        return multi.max_over_ranks(x, device=cdev)

    n, d, strategy = args.n, args.d, args.strategy
    shard = (rank, world) if world > 1 else None
    e0, e1 = tg.shard_elems(n, RHO, rank, world)
    cells_local = e1 - e0
    pk = peaks()

    clocks = ClockSampler(local)
    clocks.start()

    pts = tg.gen_values(n * d, SEED, dev).view(n, d)
    out = torch.empty(cells_local, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step(strat=strategy, kernel="edm", mode="span", persistent=False, o=out, sh=shard):
        if kernel == "edm":
            tg.launch("edm", strat, n, points=pts, out=o, d=d, rho=RHO, mode=mode, shard=sh,
                      persistent=persistent, stream=stream, sync=False)
        else:
            tg.launch("write", strat, n, out=o, rho=RHO, mode=mode, shard=sh, persistent=persistent,
                      stream=stream, sync=False)

    def cool_down(seconds: float = 0.5):
        """Idle pause (all ranks) before a comparison block, see per_mapping."""
        torch.cuda.synchronize(dev)
        barrier()
        time.sleep(seconds)

    def time_steps(fn, steps, warmup):
        for _ in range(warmup):
            fn()
        barrier()
        torch.cuda.synchronize(dev)
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(steps):
            fn()
        b.record(stream)
        torch.cuda.synchronize(dev)
        barrier()
        return max_over_ranks(a.elapsed_time(b) / steps)

    # ---- headline: device-timed K steps
    step()
    launches_per_step = int(_lib.load().tg_last_launch_count())
    ms = time_steps(step, args.steps, args.warmup)
    value = tri(n) / (ms / 1e3)

    # ---- dominant kernel: per-launch events on the launching stream
    per_launch = []
    for _ in range(max(3, min(args.steps, 20))):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        step()
        b.record(stream)
        per_launch.append((a, b))
    torch.cuda.synchronize(dev)
    k_med = max_over_ranks(sorted(x.elapsed_time(y) for x, y in per_launch)[len(per_launch) // 2])
    # achieved over the timed region itself: one step = one launch of the span
    # kernel (+ the point classifier and its 4-byte memset, charged to it)
    k_ms = ms
    alg_bytes = 4 * cells_local + 4 * n * d
    achieved = alg_bytes / (k_ms / 1e3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            traffic = json.load(f).get(f"edm_{strategy}_n{n}_d{d}_g{world}")
    roofline = {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / pk["hbm_gbs"], "traffic": traffic,
                "kernel": "tg::span_edm_kernel<3,2,1> (+ classify_points_kernel)",
                "algorithmic_bytes_per_launch": alg_bytes, "launch_ms": k_ms,
                "launch_ms_median_isolated": k_med,
                "timing": "CUDA events over the timed region (launch_ms = its average per step); "
                          "launch_ms_median_isolated = median of individually bracketed launches",
                "peak_source": pk["source"] + " copy bandwidth, burst"}

    # ---- store-only reference: cudaMemset of the same packed buffer
    fill_ms = time_steps(lambda: out.view(torch.int32).fill_(0), 5, 2)
    roofline["write_kernel_ms"] = time_steps(lambda: step(kernel="write", o=out.view(torch.int32)), 5, 2)
    roofline["store_only_peak_gbs"] = 4 * cells_local / (fill_ms / 1e3) / 1e9
    roofline["frac_of_store_peak"] = achieved / roofline["store_only_peak_gbs"]
    roofline["peak_note"] = ("peak = MEASURED_PEAKS.json copy bandwidth (read + write); this kernel is a pure "
                             "store stream, which can exceed it -- frac_of_store_peak compares with a fill_ of "
                             "the same buffer timed in this run")

    # ---- per mapping (I = t_BB / t_strategy, bench.cpp:124-133)
    per_mapping = {}
    if not args.quick:
        wbuf = out.view(torch.int32)
        pm_steps, pm_warm = 5, 2
        rows = {}
        span_strats = ["bb", "ltm-r", "ltm-n", "ltm-x", "ltm-exact", "rec", "rb", "utm"]
        for s in span_strats:
            # every mapping starts from the same power state: under a sustained
            # sweep the B200 power-caps progressively and the mappings measured
            # last lose up to 10 % (same-session test: RB 1.506 -> 1.366 ms, UTM
            # 1.631 -> 1.514 with the pause); sustained throughput is the headline
            cool_down()
            e_ms = time_steps(lambda: step(strat=s), pm_steps, pm_warm)
            w_ms = time_steps(lambda: step(strat=s, kernel="write", o=wbuf), pm_steps, pm_warm)
            p_ms = time_steps(lambda: step(strat=s, persistent=True), pm_steps, pm_warm)
            st = tg.dispatch_stats(s, n, RHO, shard)
            rows[f"span/{s}"] = {"edm_ms": e_ms, "edm_persistent_ms": p_ms, "write_ms": w_ms,
                                 "blocks_launched": st["blocks_launched"], "blocks_discarded": st["blocks_discarded"]}
        if world == 1:
            gbuf = torch.empty(tri(n), dtype=torch.float32, device=dev)
            for s in ["bb", "ltm-r", "ltm-n", "ltm-x", "rec", "rb", "utm"]:
                cool_down()
                steps_g = 3 if s in ("utm", "rb") else pm_steps
                e_ms = time_steps(lambda: step(strat=s, mode="grid", o=gbuf, sh=None), steps_g, 1)
                w_ms = time_steps(lambda: step(strat=s, kernel="write", mode="grid", o=gbuf.view(torch.int32), sh=None), steps_g, 1)
                st = tg.dispatch_stats(s, n, RHO)
                rows[f"grid/{s}"] = {"edm_ms": e_ms, "write_ms": w_ms, "blocks_launched": st["blocks_launched"],
                                     "blocks_discarded": st["blocks_discarded"]}
            del gbuf
        for key, r in rows.items():
            mode = key.split("/")[0]
            bb = rows.get(f"{mode}/bb")
            r["edm_elems_per_s"] = cells_local * world / (r["edm_ms"] / 1e3) if mode == "span" else tri(n) / (r["edm_ms"] / 1e3)
            r["edm_gbs"] = (4 * (cells_local if mode == "span" else tri(n))) / (r["edm_ms"] / 1e3) / 1e9
            r["write_gbs"] = (4 * (cells_local if mode == "span" else tri(n))) / (r["write_ms"] / 1e3) / 1e9
            r["edm_frac_hbm"] = r["edm_gbs"] / pk["hbm_gbs"]
            r["wasted_block_frac"] = r["blocks_discarded"] / max(1, r["blocks_launched"])
            if bb:
                r["I_edm_vs_bb"] = bb["edm_ms"] / r["edm_ms"]
                r["I_write_vs_bb"] = bb["write_ms"] / r["write_ms"]
        per_mapping = rows

    # ---- the other BASELINE.json configs (parity cases; timed for reference)
    other = {}

    def run_guarded(name, fn):
        """A secondary config must not cost the headline line: at N = 1 an
        exception is recorded under other[name]; at N > 1 it propagates (a rank
        that skipped a collective would hang the others)."""
        if world > 1:
            fn()
            return
        try:
            fn()
        except Exception as exc:  # noqa: BLE001
            other[name] = {"error": f"{type(exc).__name__}: {exc}"}
            torch.cuda.synchronize(dev)

    def _c2():
        # C2: write / dummy td-kernel sweep over N, every mapping (I = t_BB / t_strategy)
        # Each entry is the device time per launch of a CUDA graph of k
        # back-to-back launches (no host launch gaps: at N <= 4096 a launch is
        # ~10 us, below the Python + ctypes launch cost).
        def graph_ms(fn, k):
            side = torch.cuda.Stream(dev)
            side.wait_stream(stream)
            with torch.cuda.stream(side):
                for _ in range(2):
                    fn(side)
            torch.cuda.synchronize(dev)
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=side):
                for _ in range(k):
                    fn(side)
            ts = []
            with torch.cuda.stream(side):
                gr.replay()
                for _ in range(3):
                    a = torch.cuda.Event(enable_timing=True)
                    b = torch.cuda.Event(enable_timing=True)
                    a.record(side)
                    gr.replay()
                    b.record(side)
                    b.synchronize()
                    ts.append(a.elapsed_time(b) / k)
            del gr
            return sorted(ts)[1]

        sweep = {}
        for ns in (1024, 2048, 4096, 8192, 16384, 65536):
            cool_down()
            wb = torch.empty(tri(ns), dtype=torch.int32, device=dev)
            row = {}
            c2_strats = ("bb", "ltm-r", "ltm-x", "ltm-n", "utm", "rb", "rec")
            for mode, strats in (("grid", c2_strats), ("span", c2_strats)):
                for s in strats:
                    k = 2 if (ns == 65536 and mode == "grid") else (5 if ns == 65536 else 20)
                    w_ms = graph_ms(lambda st_: tg.launch("write", s, ns, out=wb, rho=RHO, mode=mode, stream=st_,
                                                          sync=False), k)
                    r = {"write_ms": w_ms, "write_gbs": 4 * tri(ns) / (w_ms / 1e3) / 1e9}
                    r["dummy_ms"] = graph_ms(lambda st_: tg.launch("dummy", s, ns, rho=RHO, mode=mode, stream=st_,
                                                                   sync=False), k)
                    # cells/s of the write and dummy kernels, grid blocks/s and
                    # the wasted-block fraction of the strategy's grid (closed form, reference tallies)
                    ds = tg.dispatch_stats(s, ns, RHO)
                    r["write_cells_per_s"] = tri(ns) / (w_ms / 1e3)
                    r["dummy_cells_per_s"] = tri(ns) / (r["dummy_ms"] / 1e3)
                    r["grid_blocks_per_s"] = ds["blocks_launched"] / (r["dummy_ms"] / 1e3)
                    r["wasted_block_frac"] = ds["blocks_discarded"] / max(1, ds["blocks_launched"])
                    row[f"{mode}/{s}"] = r
            for key, r in row.items():
                bbr = row[key.split("/")[0] + "/bb"]
                r["I_write_vs_bb"] = bbr["write_ms"] / r["write_ms"]
                if "dummy_ms" in r:
                    r["I_dummy_vs_bb"] = bbr["dummy_ms"] / r["dummy_ms"]
            sweep[str(ns)] = row
            del wb
        other["C2_write_dummy_sweep"] = sweep
        other["C2_timing"] = ("device ms per launch: median of 3 replays of a CUDA graph of k back-to-back launches "
                              "(k = 20; 5 at N=65536 span, 2 grid); I = t_BB / t_strategy in the same mode")

    def _c3():
        # C3: collision table N=32768 (bit-packed no-diagonal table + count)
        nc, r_max = 32768, 0.0625
        sph = tg.gen_values(nc * 4, SEED, dev).view(nc, 4)
        c_ms = time_steps(lambda: tg.collide(sph, r_max, strategy="ltm-r", shard=(rank, world) if world > 1 else None,
                                             stream=stream, sync=False), 5, 2)
        bits, hits = tg.collide(sph, r_max, strategy="ltm-r", shard=(rank, world) if world > 1 else None)
        p0, p1 = tg.shard_elems(nc, RHO, rank, world, with_diag=False)
        hits_shard = int(hits.item())
        c3_ref = golden_collide(nc, r_max, rank, world)
        c3_sha = sha256_device(bits)
        del bits
        other["C3_collide_n32768"] = {"ms": c_ms, "pairs_per_s": tri(nc - 1) / (c_ms / 1e3),
                                      "hits_shard": hits_shard,
                                      "hits_total": multi.reduce_hits(hits.to(cdev) if world > 1 else hits),
                                      "r_max": r_max,
                                      "verify": {"ok": bool(c3_ref) and c3_sha == c3_ref[0] and hits_shard == c3_ref[1],
                                                 "sha256": c3_sha, "want_sha256": c3_ref[0] if c3_ref else None,
                                                 "want_hits": c3_ref[1] if c3_ref else None,
                                                 "golden": "tests/golden/golden_large.json collide (oracle)"
                                                 + ("" if c3_ref else f" -- no entry for {world} shards")},
                                      "out_bytes_shard": 4 * ((p1 - p0 + 31) // 32)}

    def _c4():
        # C4: EDM N=65536, d=64, direct (bit-exact) wide span kernel
        p64 = tg.gen_values(n * 64, SEED, dev).view(n, 64)
        w_ms = time_steps(lambda: tg.launch("edm", strategy, n, points=p64, out=out, d=64, rho=RHO,
                                            shard=shard, stream=stream, sync=False), 3, 1)
        other["C4_edm_n65536_d64_direct"] = {"ms": w_ms, "elems_per_s": tri(n) / (w_ms / 1e3),
                                             "fp32_ops_per_cell": 3 * 64, "bit_exact": True}
        try:
            gm_ms = time_steps(lambda: tg.launch("edm", strategy, n, points=p64, out=out, d=64, rho=RHO,
                                                 shard=shard, mode="gram", stream=stream, sync=False), 3, 1)
            other["C4_edm_n65536_d64_gram_tcgen05"] = {
                "ms": gm_ms, "elems_per_s": tri(n) / (gm_ms / 1e3),
                "hbm_gbs": 4 * cells_local / (gm_ms / 1e3) / 1e9,
                "frac_hbm": 4 * cells_local / (gm_ms / 1e3) / 1e9 / pk["hbm_gbs"],
                # tcgen05 kind::f16, 3 products (hi*hi, hi*lo, lo*hi) of M=128 x N=136 x K=64 per tile
                "tensor_tflops": 3 * 2 * 64 * 128 * 136 * ((n // 128) * (n // 128 + 1) // 2) / (gm_ms / 1e3) / 1e12,
                "kernel": "gram2_edm_kernel (warp-specialised: bulk-copy producer, tcgen05 MMA, 16 epilogue warps)",
                "bit_exact": False, "tolerance": "|d^2 - d_exact^2| <= 2^-17 (|x_i|^2 + |x_j|^2)"}
        except RuntimeError as exc:
            other["C4_edm_n65536_d64_gram_tcgen05"] = {"error": str(exc)}
        del p64

    def _c5():
        # C5: EDM N=131072, d=3 -- this rank's lambda shard of the 34.4 GB output
        n5 = 131072
        b5, e5 = tg.shard_elems(n5, RHO, rank, world)
        if 4 * (e5 - b5) < 40e9:
            p5 = tg.gen_values(n5 * 3, SEED, dev).view(n5, 3)
            o5 = torch.empty(e5 - b5, dtype=torch.float32, device=dev)
            f_ms = time_steps(lambda: tg.launch("edm", strategy, n5, points=p5, out=o5, d=3, rho=RHO,
                                                shard=(rank, world) if world > 1 else None, stream=stream,
                                                sync=False), 3, 1)
            other["C5_edm_n131072_d3"] = {"ms": f_ms, "elems_per_s_total": tri(n5) / (f_ms / 1e3),
                                          "shard_gb": 4 * (e5 - b5) / 1e9,
                                          "hbm_gbs_per_gpu": 4 * (e5 - b5) / (f_ms / 1e3) / 1e9}
            del p5, o5

    if not args.quick and world == 1:
        run_guarded("C2_write_dummy_sweep", _c2)
    if not args.quick:
        run_guarded("C3_collide_n32768", _c3)
        run_guarded("C4_edm_n65536_d64_direct", _c4)
        run_guarded("C5_edm_n131072_d3", _c5)
        torch.cuda.empty_cache()

    # ---- e2e through the public drop-in with pinned host buffers
    host_pts = torch.from_numpy(pts.cpu().numpy()).pin_memory().numpy()
    host_out = torch.empty(cells_local, dtype=torch.float32).pin_memory().numpy()
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    for _ in range(min(args.warmup, 2)):
        tg.edm_strategy(strategy, host_pts, RHO, out=host_out, device=local, shard=shard)
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        tg.edm_strategy(strategy, host_pts, RHO, out=host_out, device=local, shard=shard)
    sec = max_over_ranks((time.perf_counter() - t0) / e2e_steps)
    e2e = {"value": tri(n) / sec, "unit": UNIT, "h2d_bytes_per_step": 4 * n * d,
           "d2h_bytes_per_step": 4 * cells_local, "ms_per_step": sec * 1e3,
           "path": "trigrid.edm_strategy(host pinned) -> tg_edm_strategy_host (C-ABI): H2D points, "
                   "kernel in block-row pieces, D2H pipelined per piece",
           "d2h_gbs_per_rank": 4 * cells_local / sec / 1e9}
    clk = clocks.stop()

    # ---- verify what was timed (outside every timed region): the headline
    # buffer and the e2e host buffer against the reference's sha256
    want = golden_sha(n, d, rank, world)
    step()
    torch.cuda.synchronize(dev)
    got_dev = sha256_device(out)
    got_host = sha256_host(host_out)
    verify = {"golden": "tests/golden/golden_large.json (reference launch_edm, oracle/_ref)",
              "want_sha256": want, "device_sha256": got_dev, "e2e_host_sha256": got_host,
              "ok": bool(want) and got_dev == want and got_host == want,
              "bytes": 4 * cells_local, "shard": [rank, world]}
    if not want:
        verify["note"] = f"no golden sha recorded for n={n} d={d} shards={world}"

    # ---- CPU baseline (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            r = cpu_reference_run(n, d, strategy, 3, 1, args.cpu_budget)
            cpu = {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")}
            if not args.quick:
                # the reference's own launch_edm per mapping (bench.cpp:86-96), one timed call each
                pm = {}
                for s in ("bb", "ltm-r", "rb", "rec", "utm"):
                    rs = cpu_reference_run(n, d, s, 1, 0, None)
                    pm[s] = {"value": rs["value"], "ms_per_step": rs["ms_per_step"], "kind": rs["kind"],
                             "cores": rs["cores"]}
                for s, r_ in pm.items():
                    r_["I_vs_bb"] = pm["bb"]["ms_per_step"] / r_["ms_per_step"]
                cpu["per_mapping"] = pm
        except Exception as exc:  # noqa: BLE001
            cpu = {"value": None, "unit": UNIT, "cores": None, "kind": "reference", "sample": f"failed: {exc}"}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "fp32",
        "data": f"synthetic: gen_points({n}, {d}, seed={SEED}) splitmix64 U[0,1), generated on device",
        "config": config(n, d, world, strategy),
        "hbm_gbs": 4 * tri(n) / (ms / 1e3) / 1e9 / world,
        "roofline": roofline, "e2e": e2e, "cpu_baseline": cpu, "clocks": clk,
        "gpu_launches": launches_per_step * args.steps,
        "per_mapping": per_mapping,
        "per_mapping_timing": ("CUDA events over 5 back-to-back launches after 2 warm-up, each mapping after a "
                               "0.5 s idle so all start from the same power state (sustained: the headline)"),
        "other_configs": other,
        "verify": verify,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--n", type=int, default=N_DEFAULT)
    ap.add_argument("--d", type=int, default=D_DEFAULT)
    ap.add_argument("--strategy", default="ltm-r")
    ap.add_argument("--quick", action="store_true", help="skip the per-mapping sweep")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--e2e-steps", type=int, default=5)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
