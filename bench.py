#!/usr/bin/env python
"""bench.py -- weighted-minhash signatures/sec (row x hash) on 1..8 B200s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--algo auto]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...
    python bench.py --impl reference ...      # the CPU oracle, timed on the host cores

The default workload is BASELINE.json configs[4] (c5: 16,000,000 dense rows x
4096, k = 1024, uint16 signatures), the largest configuration that fits one
B200 -- the metric names no config, so the line is quoted on it.  A step is
one wmh_hash launch over this rank's resident rows (all of §8(a)'s hot-path
rows a5-a9; a1-a4 -- column max, the NCCL max exchange, prefix sums,
IntToComp -- run once before timing, as the paper's "one time
pre-processing").  Scaling is strong: the N rows of ONE
dataset are split into contiguous shards shard(N, r, G) (the same rows for
every G, generated on the device for the counter-based configs c1/c5), so
the total work is fixed as G grows; the only collective is the max exchange
in prepare.  Timing: CUDA events on the launching stream around each step, an
L2 flush (256 MiB write) between steps outside the events (the c5 rows, 65 GB,
exceed L2 anyway), barrier + synchronize around the K steps, max over ranks.
Rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "weighted-minhash signatures/sec (row x hash)"
UNIT = "hashes/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", default="c5",
                   help="c1..c5, c2r (default c5 = configs[4], the largest single-GPU configuration)")
    p.add_argument("--rows", type=int, default=None,
                   help="total rows N over all GPUs (default: the config's N); rank r hashes shard(N, r, G)")
    p.add_argument("--algo", default="auto", choices=["auto", "simple", "tiled", "index"])
    p.add_argument("--tile", default="auto", choices=["auto", "bytes", "bitplanes", "bitslice"],
                   help="tiled, dense rows: which tile (performance only)")
    p.add_argument("--chunk", type=int, default=0, help="tiled: draws per re-queue (0 = auto)")
    p.add_argument("--horizon", type=int, default=0, help="index: draws filed per hash (0 = auto)")
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--graph", action="store_true",
                   help="replay the step as a captured CUDA graph (launch-bound c1), and report the library's "
                        "empty-launch floor measured the same way")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=15.0, help="target CPU work of the oracle sample")
    p.add_argument("--gpu-gen", action="store_true",
                   help="(kept for old command lines: c1/c5 rows are always generated on the device)")
    p.add_argument("--collide-pairs", type=int, default=-1,
                   help="also time wmh_collide (a10) on this many random pairs of the step's signatures "
                        "(-1 = the config's own: 10^7 for c5, else none)")
    p.add_argument("--gather", action="store_true",
                   help="under torchrun: all-gather the signatures (NCCL) before colliding pairs over all rows")
    return p.parse_args()


# ----------------------------------------------------------------- workload
def shard(n_rows: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous row block of rank r (the binding's shard(); restated here so the
    reference arm does not import the CUDA package)."""
    base, rem = divmod(n_rows, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def workload(cfg_name: str, rank: int, n_rows: int | None, world: int = 1):
    """This rank's shard of the config's N rows (host-generated configs)."""
    import datagen
    cfg = datagen.CONFIGS[cfg_name]
    N = cfg.n_rows if n_rows is None else n_rows
    lo, hi = shard(N, rank, world)
    n = hi - lo
    cache = os.environ.get("BENCH_CACHE_DIR")      # optional: reuse generated rows within one session
    if cache and cfg.kind == "dense":
        path = os.path.join(cache, f"{cfg_name}_{lo}_{hi}.npy")
        if os.path.exists(path):
            return cfg, n, datagen.Dense(np.load(path))
    data = _generate(cfg_name, cfg, lo, hi)
    if cache and cfg.kind == "dense":
        os.makedirs(cache, exist_ok=True)
        np.save(path, data.x)
    return cfg, n, data


def _generate(cfg_name, cfg, lo, hi):
    import datagen
    if cfg_name == "c2":
        data = datagen.Dense(datagen.gen_c2_rows(cfg.data_seed, lo, hi, cfg.dim))
    elif cfg_name == "c2r":
        data = datagen.Dense(datagen.gen_c2_real_rows(cfg.data_seed, lo, hi, cfg.dim))
    elif cfg_name == "c1":
        data = datagen.Dense(datagen.gen_counter_c1_rows(cfg.data_seed, np.arange(lo, hi), cfg.dim))
    elif cfg_name == "c5":
        data = datagen.Dense(datagen.gen_counter_c5_rows(cfg.data_seed, np.arange(lo, hi), cfg.dim))
    else:
        _, full = datagen.make(cfg_name, n_rows=hi)
        data = full.take(np.arange(lo, hi))
    return data


def desc(cfg, N):
    w = "real -> uint16 fixed point" if cfg.name == "c2r" else "uint8"
    return (f"{cfg.name}: N={N} rows, D={cfg.dim}, {cfg.kind} {w}, k={cfg.k}, cap={cfg.cap}, "
            f"uint{8 * cfg.sig_bytes} signatures, seed={cfg.seed}")


def host_cores():
    """(logical CPUs this process may use, physical cores) of the host."""
    logical = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    try:
        import psutil
        phys = psutil.cpu_count(logical=False)
    except Exception:                                  # noqa: BLE001
        phys = None
    return logical, phys


def expected_draws(x_sum: np.ndarray, M: int, k: int, cap: int) -> float:
    """sum_n k * E_n with E_n = (1 - (1 - s_n)^cap) / s_n (Theorem 2 capped, reading R9)."""
    s = x_sum.astype(np.float64) / M
    with np.errstate(divide="ignore"):                       # s = 1: log(0); that row needs one draw
        e = np.where(s > 0, -np.expm1(cap * np.log1p(-np.minimum(s, 1 - 1e-300))) / np.maximum(s, 1e-300), cap)
    e = np.where(s >= 1, 1.0, e)
    return float(k * e.sum())


def row_sums(data):
    import datagen
    if isinstance(data, datagen.Dense):
        return data.x.sum(axis=1, dtype=np.int64)
    return np.add.reduceat(data.val.astype(np.int64), data.row_ptr[:-1]) * (np.diff(data.row_ptr) > 0) \
        if len(data.val) else np.zeros(data.n_rows, np.int64)


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """NVML clock / throttle-reason sampling in a thread (every ~5 ms)."""
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, dev_index: int):
        self.samples = []
        self.ok = False
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(dev_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:                      # noqa: BLE001
            self.err = repr(e)
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                mhz = self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)
                rs = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((mhz, rs))
            except Exception:                       # noqa: BLE001
                pass
            time.sleep(0.005)

    def start(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()

    def stop(self):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0,
                    "note": getattr(self, "err", "no samples")}
        mhz = [m for m, _ in self.samples]
        bits = 0
        for _, r in self.samples:
            bits |= r
        reasons = [n for b, n in self.REASONS.items() if bits & b and n != "gpu_idle"]
        return {"sm_mhz": statistics.median(mhz), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(mhz), "sm_mhz_min": min(mhz)}


# ------------------------------------------------------------- CPU oracle leg
def oracle_rate(cfg, data, M_bounds, seconds: float):
    """Time the oracle (as it stands) on a bounded, seeded row sample of the same
    workload, on all host cores; returns (hashes/s, threads, sample description).
    Counter-based rows (c1/c5) are regenerated on the host for the sampled rows
    only, so the full 65 GB array never exists in host memory."""
    import datagen
    import oracle
    L = oracle.Layout(M_bounds)
    cores, _ = host_cores()
    n = data.n_rows

    def run(rows):
        if isinstance(data, (datagen.Dense, datagen.CounterRows)):
            x = np.ascontiguousarray(data.rows(rows) if isinstance(data, datagen.CounterRows) else data.x[rows])
            t0 = time.perf_counter()
            L.hash_dense(x, cfg.seed, cfg.k, cfg.cap, threads=cores)
        else:
            sub = data.take(rows)
            t0 = time.perf_counter()
            L.hash_csr(sub.row_ptr, sub.col, sub.val, cfg.seed, cfg.k, cfg.cap, threads=cores)
        return time.perf_counter() - t0

    rng = np.random.default_rng(2024)
    probe = np.sort(rng.choice(n, size=min(n, max(cores, 16)), replace=False))
    dt = run(probe)
    per_row = dt / len(probe) * cores / max(1, min(cores, len(probe)))
    want = int(min(n, max(len(probe), seconds / max(per_row, 1e-9))))
    rows = np.sort(rng.choice(n, size=want, replace=False))
    dt = run(rows)
    rate = len(rows) * cfg.k / dt
    return rate, cores, f"{len(rows)} of {n} rows (seeded uniform sample), all k={cfg.k} hashes, {dt:.1f} s"


def layout_bounds(cfg, data, N=None):
    """The oracle-side column maxima m_c of the whole N-row dataset:
    the fixed bound (c4), the host data's maxima, or -- for the counter-based
    full-size c5 -- tests/golden/c5_colmax.txt (written by
    scripts/make_golden_colmax.py through oracle.colmax_dense)."""
    import datagen
    if cfg.fixed_bound is not None:
        return np.full(data.dim, cfg.fixed_bound, np.uint32)
    if isinstance(data, datagen.CounterRows):
        N = data.n_rows if N is None else N
        gold = os.path.join(ROOT, "tests", "golden", f"{cfg.name}_colmax.txt")
        if N == cfg.n_rows and os.path.exists(gold):
            return np.loadtxt(gold, dtype=np.int64, comments="#").reshape(-1).astype(np.uint32)
        import oracle
        m = np.zeros(data.dim, np.uint32)
        for a0 in range(0, N, 65536):
            m = np.maximum(m, oracle.colmax_dense(data.rows(np.arange(a0, min(N, a0 + 65536)))))
        return m
    if isinstance(data, datagen.Dense):
        return data.x.max(axis=0).astype(np.uint32)
    m = np.zeros(data.dim, np.uint32)
    np.maximum.at(m, data.col, data.val.astype(np.uint32))
    return m


def reference_data(cfg_name, N):
    """The whole N-row dataset as the oracle sees it: lazy for c1/c5."""
    import datagen
    cfg = datagen.CONFIGS[cfg_name]
    if cfg_name in ("c1", "c5"):
        return cfg, datagen.CounterRows(cfg_name, cfg.data_seed, 0, N, cfg.dim)
    cfg, _, data = workload(cfg_name, 0, N, 1)
    return cfg, data


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import datagen
    cfg = datagen.CONFIGS[args.config]
    N = cfg.n_rows if args.rows is None else args.rows
    cfg, data = reference_data(args.config, N)
    bounds = layout_bounds(cfg, data)
    per_step = max(2.0, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
    rates = []
    for i in range(args.warmup + args.steps):
        r, cores, sample = oracle_rate(cfg, data, bounds, per_step)
        if i >= args.warmup:
            rates.append(r)
    value = statistics.mean(rates)
    _, phys = host_cores()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": N * cfg.k / value * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": desc(cfg, N), "parallelism": "host threads (rank 0 only)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "physical_cores": phys, "kind": "oracle",
                         "sample": sample + f"; each of the {args.steps} timed steps a fresh ~{per_step:.0f} s sample"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------- our arm
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)

    from paper_1602_08393_b200 import build
    build.build()
    import paper_1602_08393_b200 as wmh

    import datagen
    N = datagen.CONFIGS[args.config].n_rows if args.rows is None else args.rows   # total rows, all ranks
    lo, hi = shard(N, rank, world)
    assert (lo, hi) == wmh.shard(N, rank, world)
    xd = None
    if args.config in ("c1", "c5"):   # counter-based: this rank's shard generated on the device (bit-identical to the host recipe)
        cfg = datagen.CONFIGS[args.config]
        n = hi - lo
        xd = torch.empty((n, cfg.dim), dtype=torch.uint8, device=dev)
        for a0 in range(0, n, 1 << 20):
            b0 = min(n, a0 + (1 << 20))
            xd[a0:b0] = datagen.gpu_counter_rows(args.config, cfg.data_seed, lo + a0, b0 - a0, cfg.dim, dev)
        data = datagen.CounterRows(args.config, cfg.data_seed, lo, n, cfg.dim)
    else:
        cfg, n, data = workload(args.config, rank, N, world)
    # f1 (c2r): real-valued rows -> Sec. 4 scale choice -> uint16 fixed point, on the
    # device and before the timed region (the paper's "one time pre-processing")
    quant = None
    if cfg.name == "c2r":
        xf = torch.from_numpy(data.x).to(dev)
        grid = [1.0, 2.0, 4.0, 8.0, 16.0]           # M (and the index) grow linearly with the scale
        scale = wmh.choose_scale(wmh.Rows.from_dense(xf), grid)
        xd = wmh.quantize(xf, scale)
        del xf
        data = datagen.Dense(xd.cpu().numpy())
        quant = {"scale": scale, "grid": grid, "weights": "uint16 fixed point floor(x*scale)"}
    # inputs resident in HBM before the timed region
    if xd is not None:
        rows = wmh.Rows.from_dense(xd)
        in_bytes = xd.numel() * xd.element_size()
    elif isinstance(data, datagen.Dense):
        rows = wmh.Rows.from_dense(torch.from_numpy(data.x).to(dev))
        in_bytes = data.x.nbytes
    else:
        rows = wmh.Rows.from_csr(torch.from_numpy(data.row_ptr).to(dev), torch.from_numpy(data.col).to(dev),
                                 torch.from_numpy(data.val).to(dev), data.dim)
        in_bytes = data.row_ptr.nbytes + data.col.nbytes + data.val.nbytes
    if cfg.fixed_bound is not None:
        layout = wmh.prepare(rows, bounds=torch.full((data.dim,), cfg.fixed_bound, dtype=torch.uint32, device=dev))
    else:
        layout = wmh.prepare(rows)          # colmax + NCCL all-reduce(MAX) when world > 1
    M = layout.M
    sig = torch.empty((n, cfg.k), dtype=torch.uint8 if cfg.sig_bytes == 1 else torch.uint16, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream()

    def step(timed=False):
        wmh.hash(layout, rows, cfg.seed, cfg.k, cfg.cap, cfg.sig_bytes, algo=args.algo, out=sig, chunk=args.chunk,
                 horizon=args.horizon, time_kernel=timed and not args.graph, tile=args.tile)

    graph = None
    floor = None
    if args.graph:                      # capture the step (kernels only: no allocation, no sync on this path)
        step()
        torch.cuda.synchronize()
        l0 = wmh.kernel_launches()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step()
        graph_launches = wmh.kernel_launches() - l0
        eg = torch.cuda.CUDAGraph()
        with torch.cuda.graph(eg):
            wmh.empty_launch()
        torch.cuda.synchronize()
        fl = []
        for _ in range(max(3, args.warmup)):
            eg.replay()
        for _ in range(max(5, args.steps)):
            fa, fb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            flush.zero_()
            fa.record(stream)
            eg.replay()
            fb.record(stream)
            torch.cuda.synchronize()
            fl.append(fa.elapsed_time(fb))
        floor = {"empty_launch_graph_ms": statistics.median(fl), "kernels_per_step": graph_launches}

        def step(timed=False):         # noqa: F811  (the graph replaces the eager call)
            graph.replay()

    clocks = ClockSampler(dev.index if world == 1 else local)
    clocks.start()
    for _ in range(max(3, args.warmup)):
        step()
        flush.zero_()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches = 0
    kern_ms = []
    for a, b in evs:
        flush.zero_()                        # L2 flush outside the timed events
        a.record(stream)
        l0 = wmh.kernel_launches()
        step(timed=True)                     # + CUDA events around the dominant kernel, on its stream
        launches += (wmh.kernel_launches() - l0) if graph is None else floor["kernels_per_step"]
        b.record(stream)
        if graph is None:
            kern_ms.append(wmh.last_kernel_ms())  # waits for the kernel (after b is queued)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.stop()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    t_ms = sum(step_ms)
    t = torch.tensor([t_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_max_ms = float(t.item())
    hashes_per_step_total = N * cfg.k                      # every rank's shard: the whole dataset
    value = hashes_per_step_total * args.steps / (t_max_ms / 1e3)
    ms_per_step = t_max_ms / args.steps

    # ---- roofline of the dominant (only) kernel of the step
    if xd is not None:                  # row sums on the device, in chunks (no full int64 copy)
        x_sum = torch.cat([xd[a0:a0 + 65536].to(torch.int32).sum(1, dtype=torch.int64)
                           for a0 in range(0, n, 65536)]).cpu().numpy()
    else:
        x_sum = row_sums(data)
    draws = expected_draws(x_sum, M, cfg.k, cfg.cap)      # this rank's algorithmic draw-tests per launch
    dt_ = torch.tensor([draws], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(dt_)
    draws_total = float(dt_.item())
    if not kern_ms:                                       # graph replay: the step is the kernel
        kern_ms = step_ms
    kern_s = statistics.mean(kern_ms) / 1e3               # the dominant kernel's average launch (events)
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:                                      # noqa: BLE001
        pass
    sm_mhz = peaks.get("sm_max_mhz", 1965.0)
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    algo_used = wmh.last_algo or args.algo
    roof = roofline(algo_used, draws, kern_s, n_sm, sm_mhz, in_bytes, sig.numel() * sig.element_size(), peaks)
    if algo_used == "tiled" and wmh.last_tile == "bitslice":
        roof = roofline_bitslice(x_sum, M, cfg, kern_s, n_sm, sm_mhz, in_bytes, sig.numel() * sig.element_size(),
                                 peaks, draws, lambda R: tile_need_rate(xd, data, n, R, M))
    if algo_used == "index":
        if xd is not None:
            nnz = sum(int((xd[a0:a0 + 65536].to(torch.int32) != 0).sum().item()) for a0 in range(0, n, 65536))
        elif isinstance(data, datagen.Dense):
            nnz = int(np.count_nonzero(data.x))
        else:
            nnz = int(len(data.col))
        roof = roofline_index(x_sum, nnz, M, cfg, wmh.last_horizon, kern_s, in_bytes,
                              sig.numel() * sig.element_size(), peaks, draws, n_sm, sm_mhz,
                              dense=isinstance(data, datagen.Dense) or xd is not None)
    roof["step_share"] = kern_s * 1e3 / (t_ms / args.steps)
    try:                                 # DRAM bytes per launch of this kernel from the committed ncu capture
        tr = json.load(open(os.path.join(ROOT, "profiles", "traffic.json"))).get(f"{cfg.name}/{n}/{algo_used}")
        if tr:
            roof["traffic"] = tr["dram_bytes_read"] + tr["dram_bytes_write"]
            roof["traffic_source"] = tr["source"]
    except (OSError, ValueError):
        pass

    # ---- e2e: the public host-buffer API, H2D rows + hash + D2H signatures every step
    e2e = None
    if not args.no_e2e:
        e2e = measure_e2e(wmh, layout, data, cfg, n, args, dev, world, dist, xd)

    coll = None
    n_pairs = cfg.n_pairs if args.collide_pairs < 0 else args.collide_pairs
    if n_pairs > 0:
        gather_ms = None
        sig_c = sig
        if world > 1 and args.gather:   # the optional NCCL signature exchange, then pairs over all rows
            torch.cuda.synchronize()
            g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            g0.record()
            sig_c = wmh.gather_signatures(sig)
            g1.record()
            torch.cuda.synchronize()
            gather_ms = g0.elapsed_time(g1)
        coll = measure_collide(wmh, sig_c, n_pairs, cfg, dev, peaks)
        coll["gather_ms"] = gather_ms
        coll["pairs_over"] = "all ranks' rows (gathered)" if sig_c is not sig else \
            ("this rank's shard" if world > 1 else "all rows")

    # the oracle on a sample of the same N-row dataset (rank 0, host cores; the
    # other ranks wait at the barrier): bounds from the oracle side, never the GPU
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        rcfg, rdata = reference_data(args.config, N) if xd is not None or world > 1 else (cfg, data)
        if cfg.name == "c2r":
            rdata = data
        bnds = layout_bounds(rcfg, rdata)
        r, cores, sample = oracle_rate(rcfg, rdata, bnds, args.cpu_seconds)
        _, phys = host_cores()
        cpu = {"value": r, "unit": UNIT, "cores": cores, "physical_cores": phys, "kind": "oracle", "sample": sample}
    if world > 1:
        dist.barrier()

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": {"workload": desc(cfg, N), "global_rows": N, "rows_per_gpu_max": -(-N // world),
                       "k": cfg.k, "M": M, "algo": args.algo, "tile": args.tile,
                       "parallelism": f"rows sharded x{world} (contiguous shard(N, r, G)), no collective in the step",
                       "l2": "flushed between steps (256 MiB write outside the timed events); "
                             f"inputs {in_bytes / 2**20:.0f} MiB + signatures "
                             f"{sig.numel() * sig.element_size() / 2**20:.0f} MiB per step",
                       "expected_draws_per_step": draws_total,
                       "step_ms_min_med_max": [min(step_ms), statistics.median(step_ms), max(step_ms)]},
            "roofline": roof,
            "collide": coll,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": clocks.summary(),
            "quantization": quant,
            "graph": floor,
            "gpu_launches": launches,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


# Lane-instructions per draw-test of the dominant kernel's minimal sequence,
# counted from SASS.  SIMPLE: the paper's per-(row, draw) loop:
# SplitMix64 + 64x32 multiply-high + packed lookup + row lookup + compare +
# loop.  TILED: the draw is shared by the tile, so a draw-test of one row is
# IMAD (address) + LDS.U8 + ISETP + SEL.
I_DRAW = {"simple": 30.0, "tiled": 4.0}


def roofline(algo, draws, kern_s, n_sm, sm_mhz, in_bytes, out_bytes, peaks):
    issue = n_sm * 4 * 32 * sm_mhz * 1e6            # lane-instructions / s at the max SM clock
    i_draw = I_DRAW.get(algo, I_DRAW["simple"])
    peak = issue / i_draw / 1e9                     # Gdraw-tests / s
    achieved = draws / kern_s / 1e9
    hbm = peaks.get("hbm_gbs", 6650.0)
    return {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "Gdraws/s", "frac": achieved / peak,
            "traffic": None, "kernel": algo,
            "peak_source": f"{n_sm} SMs x 128 lanes x {sm_mhz:.0f} MHz (MEASURED_PEAKS sm_max_mhz) "
                           f"/ {i_draw:.0f} lane-instr per draw-test ({algo})",
            "frac_vs_paper_loop": achieved / (issue / I_DRAW["simple"] / 1e9),
            "t_hbm_ms": (in_bytes + out_bytes) / (hbm * 1e9) * 1e3, "t_kernel_ms": kern_s * 1e3}


def group_expected_max(x_sum: np.ndarray, M: int, cap: int, sample: int = 4096, seed: int = 3,
                       rows: int = 32) -> tuple[float, int]:
    """E[max over the live rows r of a `rows`-row group of min(G_r, cap)], G_r ~ Geom(s_r)
    (Theorem 2), summed over the groups of consecutive rows the
    bit-sliced tile tests together: sum_t P(max > t) = sum_t 1 - prod_r (1 - (1 - s_r)^t).
    Exact per group; computed on a seeded sample of groups and scaled when there
    are more than `sample` groups.  Returns (sum over groups, groups sampled)."""
    s = x_sum.astype(np.float64) / M
    n_groups = (len(s) + rows - 1) // rows
    pad = np.zeros(n_groups * rows)
    pad[:len(s)] = s
    g = pad.reshape(n_groups, rows)
    idx = np.arange(n_groups)
    if n_groups > sample:
        idx = np.sort(np.random.default_rng(seed).choice(n_groups, size=sample, replace=False))
    g = g[idx]
    live = g > 0
    lq = np.where(live, np.log1p(-np.minimum(g, 1 - 1e-15)), 0.0)          # log(1 - s_r)
    total = np.zeros(len(g))
    done = ~live.any(axis=1)
    t = 0
    step = 64
    while t < cap and not done.all():
        ts = np.arange(t, min(cap, t + step), dtype=np.float64)
        # P(max > t) = 1 - prod_r (1 - q_r^t) over live rows (dead rows contribute 1)
        qt = np.exp(lq[:, :, None] * ts[None, None, :])                   # [G, rows, T]
        with np.errstate(divide="ignore"):                                # t = 0: log(1 - 1) = -inf, P = 1
            logp = np.where(live[:, :, None], np.log1p(-qt), 0.0).sum(axis=1)
        tail = -np.expm1(logp)                                            # P(max > t)
        tail[done] = 0.0
        total += tail.sum(axis=1)
        done |= tail[:, -1] < 1e-12
        t += step
    return float(total.sum() * n_groups / len(g)), len(g)


def tile_need_rate(xd, data, n: int, R: int, M: int, sample: int = 512, seed: int = 5) -> float:
    """The fraction of draws the bit-sliced tile must test: a draw (c, off) is
    needed when off < the column maximum over the tile's R rows, so per tile
    q = sum_c colmax_tile(c) / M (Alg. 5's green test can only pass there).  Mean
    over a seeded sample of tiles."""
    n_tiles = (n + R - 1) // R
    if xd is not None:
        import torch  # noqa: F401  (xd is a device tensor)
    tiles = np.sort(np.random.default_rng(seed).choice(n_tiles, size=min(sample, n_tiles), replace=False))
    qs = []
    for t in tiles:
        r0, r1 = int(t) * R, min(n, int(t) * R + R)
        if xd is not None:
            cm = xd[r0:r1].amax(dim=0).to(torch.int64).sum().item()
        elif hasattr(data, "x"):
            cm = int(np.asarray(data.x[r0:r1]).max(axis=0).astype(np.int64).sum())
        elif hasattr(data, "rows"):
            cm = int(data.rows(np.arange(r0, r1)).max(axis=0).astype(np.int64).sum())
        else:
            return float("nan")
        qs.append(cm / M)
    return float(np.mean(qs))


def roofline_bitslice(x_sum, M, cfg, kern_s, n_sm, sm_mhz, in_bytes, out_bytes, peaks, draws, need_rate):
    """The bit-sliced tile (hash_bitslice.cu): integer-issue bound.  Its work per
    R-row tile and hash: screen every draw up to the tile's last row's first
    green -- E[max_r min(G_r, cap)] over the tile's rows (Theorem 2 per row) --
    against the tile's column maxima, and test the needed fraction q of them
    (need_rate(R), tile_need_rate) on the bit planes.  Floor = (screened draws x lane-instr per
    screened draw + tested draws x lane-instr per tested draw) / the SMs' lane
    issue rate, both per-unit costs counted statically from the kernel's own SASS
    (profiles/r2_sass_bitslice.json, scripts/sass_budget.py).  Waste the floor
    does not pay for: rounds of 96 draws past the max, passes with fewer than 32
    listed draws, staging the tile, flushing signatures, issue stalls."""
    try:
        sass = json.load(open(os.path.join(ROOT, "profiles", "r2_sass_bitslice.json")))
        a_scr, b_test = sass["lane_instr_per_screened_draw"], sass["lane_instr_per_tested_entry"]
    except (OSError, ValueError, KeyError) as e:  # the committed SASS budget is missing: say so, no fraction
        return {"bound": "alu", "achieved": None, "peak": None, "unit": "Gdraws/s", "frac": None,
                "traffic": None, "kernel": "tiled/bitslice", "error": f"profiles/r2_sass_bitslice.json: {e}",
                "t_kernel_ms": kern_s * 1e3}
    R = 32 * sass.get("groups", 2)                                  # rows per tile of the profiled variant
    q = need_rate(R)
    emax, sampled = group_expected_max(x_sum, M, cfg.cap, rows=R)
    screened = cfg.k * emax                                         # tile-draws screened
    tested = q * screened                                           # tile-draws tested on the planes
    per_draw = a_scr + q * b_test                                   # lane-instructions per screened draw
    issue = n_sm * 4 * 32 * sm_mhz * 1e6                            # lane-instructions / s
    t_floor = screened * per_draw / issue
    hbm = peaks.get("hbm_gbs", 6650.0)
    return {"bound": "alu", "achieved": screened / kern_s / 1e9, "peak": issue / per_draw / 1e9,
            "unit": "Gdraws/s", "frac": t_floor / kern_s, "traffic": None, "kernel": "tiled/bitslice",
            "peak_source": f"{n_sm} SMs x 128 lanes x {sm_mhz:.0f} MHz (MEASURED_PEAKS sm_max_mhz) / "
                           f"({a_scr:.1f} lane-instr per screened draw + q = {q:.3f} x {b_test:.1f} per tested draw; "
                           f"SASS of the round and pass loops, profiles/r2_sass_bitslice.json)",
            "tile_rows": R, "draws_screened_required": screened, "draws_tested_required": tested,
            "need_rate_q": q, "tiles_sampled": sampled,
            "t_floor_ms": t_floor * 1e3, "t_kernel_ms": kern_s * 1e3,
            "t_hbm_ms": (in_bytes + out_bytes) / (hbm * 1e9) * 1e3,
            "frac_vs_paper_loop": draws / kern_s / 1e9 / (issue / I_DRAW["simple"] / 1e9)}


def index_epochs(T: int):
    """The index kernel's nested epoch boundaries for horizon T (hash_index.cu index_epochs)."""
    B, b = [], 32
    x2max = int(os.environ.get("WMH_INDEX_X2MAX", "512"))
    while b < T and len(B) < 13:
        B.append(b)
        b *= 2 if b < x2max else 4
    if B and 2 * T < 3 * B[-1]:
        B.pop()
    return B + [T]


def index_cf(k: int, dense: bool, dim: int = 1 << 30) -> float:
    """The plan's fallback-draw cost the kernel uses (hash_index.cu index_rows):
    2 for dense rows; CSR rows with 8 warps per row 6 when the row's column bitmap
    fits the range buffers (ceil(dim/32) + its uint16 first-column index + the
    uint16 hash list within 2*2048 + 33 words: dim <= ~66,000), else 24; with
    fewer warps 64 (warps per row: 2, doubled while 64/nw rows' h[k] would exceed
    128 KiB)."""
    if dense:
        return 2.0
    nw = 2
    while nw < 8 and (64 // nw) * k * 4 > (128 << 10):
        nw *= 2
    if nw < 8:
        return 64.0
    bmw = (dim + 31) // 32
    return 6.0 if bmw + (bmw + 1) // 2 + 1024 <= 2 * 2048 + 33 else 24.0


def index_plan(s: np.ndarray, k: int, cap: int, B, cf: float) -> np.ndarray:
    """Per row the horizon T_x the index kernel picks (hash_index.cu ix_plan): the
    epoch minimising k*T*s + k*(1-s)^T * max(32, min(1/s, cap-T)) * cf."""
    s = np.clip(s.astype(np.float64), 1e-30, 1 - 1e-12)
    costs = []
    for T in B:
        rest = 0.0 if T >= cap else np.maximum(32.0, np.minimum(1.0 / s, cap - T))
        costs.append(T * s + np.exp(T * np.log1p(-s)) * rest * cf)
    return np.asarray(B, np.float64)[np.argmin(np.stack(costs), axis=0)]


def roofline_index(x_sum, nnz, M, cfg, T, kern_s, in_bytes, out_bytes, peaks, draws, n_sm, sm_mhz, dense):
    """INDEX kernel: memory-bound.  Algorithmic bytes per launch = rows in +
    signatures out + the filed draws the rows must visit (4 B each: k*T_x*s per
    row, T_x the kernel's own per-row horizon) + two 4 B range bounds per nonzero."""
    s = x_sum.astype(np.float64) / M
    live = s > 0
    Tx = index_plan(s[live], cfg.k, cfg.cap, index_epochs(int(T)), index_cf(cfg.k, dense, cfg.dim))
    entries = float(cfg.k * (Tx * s[live]).sum())
    algo_bytes = in_bytes + out_bytes + 4.0 * entries + 8.0 * nnz
    hbm = peaks.get("hbm_gbs", 6650.0)
    gbs = algo_bytes / kern_s / 1e9
    issue = n_sm * 4 * 32 * sm_mhz * 1e6
    # the issue floor of the entry walk: lane-instructions per visited entry from SASS
    try:
        per_entry = json.load(open(os.path.join(ROOT, "profiles", "r2_sass_index.json")))["lane_instr_per_unit"]
    except (OSError, ValueError, KeyError):
        per_entry = None
    t_hbm = algo_bytes / (hbm * 1e9)
    t_issue = entries * per_entry / issue if per_entry else 0.0
    out = {"bound": "hbm", "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm, "traffic": None,
           "kernel": "index", "peak_source": "MEASURED_PEAKS hbm_gbs (copy)",
           "algo_bytes": algo_bytes, "entries_visited": entries, "horizon": int(T),
           "t_hbm_floor_ms": t_hbm * 1e3, "t_issue_floor_ms": t_issue * 1e3,
           "issue_floor_source": f"{per_entry} lane-instr per visited entry (profiles/r2_sass_index.json)",
           "frac_vs_paper_loop": draws / kern_s / 1e9 / (issue / I_DRAW["simple"] / 1e9),
           "t_kernel_ms": kern_s * 1e3}
    if t_issue > t_hbm:              # the walk's instructions bind, not the bytes
        out.update({"bound": "alu", "achieved": entries / kern_s / 1e9, "peak": issue / per_entry / 1e9,
                    "unit": "Gentries/s", "frac": t_issue / kern_s,
                    "peak_source": f"{n_sm} SMs x 128 lanes x {sm_mhz:.0f} MHz / {per_entry:.2f} lane-instr per "
                                   "visited entry (SASS, profiles/r2_sass_index.json)"})
    return out


def measure_e2e(wmh, layout, data, cfg, n, args, dev, world, dist, xd=None):
    import datagen
    import torch
    if xd is not None:                  # device-generated rows: e2e over the first <= 2^20 rows
        n = min(n, 1 << 20)
        hx = xd[:n].cpu().pin_memory()
        hrows = wmh.Rows.from_dense(hx)
        h2d = hx.numel() * hx.element_size()
    elif isinstance(data, datagen.Dense):
        hx = torch.from_numpy(data.x).pin_memory()
        hrows = wmh.Rows.from_dense(hx)
        h2d = hx.numel()
    else:
        rp = torch.from_numpy(data.row_ptr).pin_memory()
        col = torch.from_numpy(data.col).pin_memory()
        val = torch.from_numpy(data.val).pin_memory()
        hrows = wmh.Rows.from_csr(rp, col, val, data.dim)
        h2d = rp.numel() * 8 + col.numel() * 4 + val.numel()
    out = torch.empty((n, cfg.k), dtype=torch.uint8 if cfg.sig_bytes == 1 else torch.uint16).pin_memory()
    for _ in range(2):
        wmh.hash_host(layout, hrows, cfg.seed, cfg.k, cfg.cap, cfg.sig_bytes, out=out)
    steps = max(1, min(args.steps, 5))
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        wmh.hash_host(layout, hrows, cfg.seed, cfg.k, cfg.cap, cfg.sig_bytes, out=out)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    t = torch.tensor([dt], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dt = float(t.item())
    d2h = int(out.numel() * out.element_size())
    bound_s = pcie_bound(h2d, d2h, dev)
    value = n * cfg.k * world * steps / dt
    return {"value": value, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": d2h, "steps": steps, "rows": n,
            "api": "wmh_hash_host (pinned host rows -> H2D -> hash -> D2H signatures, synchronised)",
            "pcie_bound_ms": bound_s * 1e3, "ms_per_call": dt / steps * 1e3,
            "frac_of_pcie_bound": bound_s / (dt / steps),
            "pcie_bound_how": "the same byte counts copied pinned H2D and D2H at once on two streams (torch), "
                              "best of 3; the call cannot beat it"}


def pcie_bound(h2d: int, d2h: int, dev) -> float:
    """Seconds to move h2d bytes in and d2h bytes out at once over this box's link
    (pinned buffers, two streams, best of 3) -- the e2e call's copy floor."""
    import torch
    hi = torch.empty(h2d, dtype=torch.uint8).pin_memory()
    di = torch.empty(h2d, dtype=torch.uint8, device=dev)
    ho = torch.empty(d2h, dtype=torch.uint8).pin_memory()
    do = torch.empty(d2h, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    best = float("inf")
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        with torch.cuda.stream(s1):
            di.copy_(hi, non_blocking=True)
        with torch.cuda.stream(s2):
            ho.copy_(do, non_blocking=True)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    del hi, di, ho, do
    return best



def measure_collide(wmh, sig, n_pairs, cfg, dev, peaks):
    """a10: wmh_collide on random row pairs of the step's signatures; HBM roofline
    (2 * k * sig_bytes read per pair + 4 B match + 4 B J-hat written)."""
    import datagen
    import torch
    pairs = torch.from_numpy(datagen.random_pairs(cfg.data_seed, sig.shape[0], n_pairs)).to(dev)
    for _ in range(2):
        wmh.collide(sig, pairs, check_pairs=False)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    a.record()
    for _ in range(reps):
        wmh.collide(sig, pairs, check_pairs=False)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    sig_bytes = sig.shape[1] * sig.element_size()
    # algorithmic bytes: every DISTINCT signature row the pairs touch once (a row
    # named by several pairs is read from L2 after the first), the pairs, the outputs
    distinct = int(torch.unique(pairs).numel())
    algo_bytes = distinct * sig_bytes + n_pairs * (16 + 8)
    hbm = peaks.get("hbm_gbs", 6650.0)
    gbs = algo_bytes / (ms / 1e3) / 1e9
    return {"pairs": n_pairs, "distinct_rows": distinct, "ms": ms, "bound": "hbm", "achieved": gbs, "peak": hbm,
            "unit": "GB/s",
            "frac": gbs / hbm, "note": f"signatures {sig.numel() * sig.element_size() / 2**30:.2f} GiB "
                                        f"({'fits' if sig.numel() * sig.element_size() < 100 * 2**20 else 'exceeds'} L2)"}


if __name__ == "__main__":
    sys.exit(main())
