#!/usr/bin/env python
"""Benchmark of the piecy hot path on B200: stream -> BICO coreset -> k-means.

One "step" = one full pass of the hot path over the configured synthetic
stream: ``run_piecy`` (piece projection when active, BICO insertion) ->
extract the coreset -> ``kmeans_repetitions`` (5 reps of weighted k-means++
and Lloyd).  Metric: stream points per second (BASELINE.json).

Default workload: cfg2 (BASELINE.json configs[1], the config the metric is
quoted on; fits one GPU).  piecy is a single sequential engine, so with
``--gpus N`` every rank runs an independent replica on its own GPU
("replicas only") and ``value`` is the aggregate.

Arms:
  (default)         this framework on the GPU(s).
  --impl reference  the reference algorithm's CPU path on the host cores:
                    the CPU restatement in oracle/ (C BICO engine + numpy
                    clustering); rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "stream points/sec (BICO+piecy, 1-8 GPU)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--rows", type=int, default=None, help="override stream length (smaller same-family stream)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-full-eval", action="store_true", help="skip the full-data evaluation pass (SURVEY 8f row 1)")
    ap.add_argument("--ncu", action="store_true", help="one short step for profiler capture, no JSON")
    return ap.parse_args()


def config_json(cfg, n, N):
    return {
        "workload": (f"{cfg.name}: {cfg.entry} n={n} d={cfg.d} {cfg.dtype} k={cfg.k} m={cfg.m} "
                     f"svd_dim={cfg.svd_dim} piece={cfg.piece_size}"
                     + (f" num_pieces={cfg.num_pieces}" if cfg.num_pieces else "")
                     + f" + kmeans_repetitions(reps={cfg.reps}, max_iters={cfg.max_iters}, tol=1e-4)"),
        "n": int(n), "d": cfg.d, "k": cfg.k, "coreset_size": cfg.m, "svd_dim": cfg.svd_dim,
        "piece_size": cfg.piece_size, "reps": cfg.reps, "seed": cfg.seed,
        "parallelism": (("replicas" if N > 1 else "single-engine") if cfg.entry == "piecy"
                        else f"level-0 groups sharded over {N} GPU(s), NCCL gather to rank 0"),
        "l2": "256 MiB buffer written between timed steps (input is ~L2-sized)",
    }


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []
        self.first = 0

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def wait_first(self, timeout: float = 3.0):
        """Block until nvidia-smi printed its first sample (its start-up is over)."""
        t0 = time.perf_counter()
        while self.proc is not None and not self.lines and time.perf_counter() - t0 < timeout:
            time.sleep(0.01)

    def mark(self):
        """Start of the timed region: earlier samples are dropped (unless no later one arrives)."""
        self.first = len(self.lines)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        timed = self.lines[self.first:] or self.lines
        for ln in timed:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------- reference
REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def reference_module():
    """The unmodified reference package installed (pip --target, no deps) into
    baseline/_ref, or None.  It is the reference's own CPU implementation of
    the path: pure Python BICO on one thread, numpy/OpenBLAS elsewhere."""
    if not os.path.isdir(os.path.join(REF_DIR, "piecy")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        import piecy
    except Exception:
        return None
    return piecy if os.path.dirname(os.path.abspath(piecy.__file__)).startswith(REF_DIR) else None


def cpu_run(cfg, X, kind):
    """One pass of the CPU path over X: the unmodified reference (kind
    "reference") or the oracle's C/numpy restatement ("port"); returns seconds."""
    t0 = time.perf_counter()
    if kind == "reference":
        from piecy.evaluation import kmeans_repetitions as ref_km
        from piecy.mergereduce import MrConfig as RefMr, run_piecy_mr as ref_mr
        from piecy.pipeline import PiecyConfig as RefPc, run_piecy as ref_piecy
        if cfg.entry == "piecy":
            cs = ref_piecy(iter(X), cfg.d, RefPc(k=cfg.k, piece_size=cfg.piece_size, svd_dim=cfg.svd_dim,
                                                 coreset_size=cfg.m, seed=cfg.seed))
        else:
            cs = ref_mr(iter(X), cfg.d, RefMr(k=cfg.k, piece_size=cfg.piece_size, num_pieces=cfg.num_pieces,
                                              svd_dim=cfg.svd_dim, coreset_size=cfg.m, seed=cfg.seed))
        ref_km(cs.points, cs.weights.astype(np.float64), cfg.k, reps=cfg.reps, seed=cfg.seed,
               max_iters=cfg.max_iters, tol=1e-4)
        return time.perf_counter() - t0
    from oracle import piecy_oracle as O
    if cfg.entry == "piecy":
        P, w = O.piecy(X, cfg.k, cfg.piece_size, cfg.svd_dim, cfg.m, seed=cfg.seed)
    else:
        P, w = O.piecy_mr(X, cfg.k, cfg.piece_size, cfg.num_pieces, cfg.svd_dim, cfg.m, seed=cfg.seed)
    O.kmeans_reps(P, w.astype(np.float64), cfg.k, reps=cfg.reps, seed=cfg.seed, max_iters=cfg.max_iters)
    return time.perf_counter() - t0


def stream_prefix(cfg, rows, n_total=None):
    from paper_1502_04265_b200 import workloads as W
    if cfg.entry == "piecy":
        return W.generate(cfg.name, n_total)[:rows]
    return W.generate_rows(cfg.name, 0, rows, n=n_total)


def cpu_sample(cfg, n_total, kind, budget_s=20.0):
    """Bounded CPU sample: the whole stream when it fits ~budget, else a prefix
    (a shorter stream of the same workload).  Returns (rows, seconds, prefix)."""
    probe = min(n_total, (50_000 if cfg.d <= 256 else 10_000) // (10 if kind == "reference" else 1))
    Xp = stream_prefix(cfg, probe, n_total)
    t = cpu_run(cfg, Xp, kind)
    rows = n_total if t * n_total / probe <= budget_s else max(probe, int(n_total * budget_s / (t * n_total / probe)))
    if rows != probe:
        Xp = stream_prefix(cfg, rows, n_total)
        t = cpu_run(cfg, Xp, kind)
    return rows, t, Xp


def cpu_env(kind):
    model = ""
    try:
        with open("/proc/cpuinfo") as f:
            model = next((ln.split(":", 1)[1].strip() for ln in f if ln.startswith("model name")), "")
    except OSError:
        pass
    blas = None
    try:
        cfgd = np.show_config(mode="dicts")
        blas = cfgd.get("Build Dependencies", {}).get("blas", {})
        blas = {k: blas.get(k) for k in ("name", "version", "openblas configuration") if k in blas}
    except Exception:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count(), "OPENBLAS_NUM_THREADS": os.environ.get("OPENBLAS_NUM_THREADS"),
            "numpy": np.__version__, "blas": blas,
            "threads": ("BICO insertion 1 Python thread (the reference is sequential); projection and clustering "
                        f"numpy/OpenBLAS on {os.cpu_count()} threads") if kind == "reference" else
                       (f"BICO engine in C (1 thread); projection and clustering numpy/OpenBLAS on {os.cpu_count()} threads")}


def baseline_kind():
    return "reference" if reference_module() is not None else "port"


def run_reference(args, rank):
    if rank != 0:
        return
    from paper_1502_04265_b200 import workloads as W
    cfg = W.CONFIGS[args.config]
    n_total = args.rows or cfg.n
    kind = baseline_kind()
    # every step is the same bounded sample; warm-up equals the GPU arm's
    per = max(3.0, 150.0 / max(1, args.steps + args.warmup))
    rows, t, Xs = cpu_sample(cfg, n_total, kind, budget_s=per)
    for _ in range(max(0, args.warmup - 1)):   # the sizing pass above is the first warm-up step
        cpu_run(cfg, Xs, kind)
    times = [cpu_run(cfg, Xs, kind) for _ in range(args.steps)]
    ms = 1000.0 * float(np.mean(times))
    val = rows / (ms / 1000.0)
    cores = os.cpu_count() or 1
    what = ("unmodified reference (baseline/_ref piecy " + reference_module().__version__ + ")"
            if kind == "reference" else "oracle port (C BICO + numpy)")
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "points/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": config_json(cfg, n_total, 1),
        "cpu_baseline": {"value": val, "unit": "points/s", "cores": cores, "kind": kind,
                         "sample": f"first {rows} of {n_total} rows of {cfg.name} through the {what}: "
                                   f"{'run_piecy' if cfg.entry == 'piecy' else 'run_piecy_mr'} + "
                                   f"kmeans_repetitions(reps={cfg.reps}) per step",
                         **cpu_env(kind)},
        "e2e": {"value": val, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------- ours
class PiecyWork:
    """cfg1-3: run_piecy on one engine; replicas across ranks (weak scaling)."""

    scaling = "weak"

    def __init__(self, cfg, args, dev):
        import torch
        from paper_1502_04265_b200 import workloads as W
        from paper_1502_04265_b200.pipeline import PiecyConfig
        self.cfg = cfg
        self.X = W.generate(cfg.name, args.rows)
        self.X_host_sample = self.X
        self.Xd = torch.from_numpy(self.X).to(dev)
        self.pcfg = PiecyConfig(k=cfg.k, piece_size=cfg.piece_size, svd_dim=cfg.svd_dim, coreset_size=cfg.m,
                                seed=cfg.seed)
        self.units = int(os.environ.get("WORLD_SIZE", "1"))
        self.h2d_bytes = self.X.nbytes

    def coreset_device(self):
        from paper_1502_04265_b200.pipeline import run_piecy_device
        eng = run_piecy_device(self.Xd, self.cfg.d, self.pcfg)
        P, w = eng.extract_device()
        return P, w, eng

    def coreset_public(self):
        from paper_1502_04265_b200.pipeline import run_piecy
        return run_piecy(self.X, self.cfg.d, self.pcfg)

    def cpu_rows(self):
        return self.X


class MrWork:
    """cfg4-5: piecy-mr, level-0 groups sharded over the ranks (strong scaling);
    each rank generates and uploads only its own groups' rows."""

    scaling = "strong"

    def __init__(self, cfg, args, dev, n_total, rank, world):
        import torch
        from paper_1502_04265_b200 import workloads as W
        from paper_1502_04265_b200.distributed import level0_groups, owner
        from paper_1502_04265_b200.mergereduce import MrConfig
        self.cfg, self.dev, self.n, self.rank, self.world = cfg, dev, n_total, rank, world
        self.mcfg = MrConfig(k=cfg.k, piece_size=cfg.piece_size, num_pieces=cfg.num_pieces, svd_dim=cfg.svd_dim,
                             coreset_size=cfg.m, seed=cfg.seed)
        self.groups = level0_groups(n_total, cfg.piece_size, cfg.num_pieces)
        self.host = {}
        self.dev_rows = {}
        for g in self.groups:
            if owner(g.index, world) == rank:
                self.host[g.index] = W.generate_rows(cfg.name, g.row_start, g.row_end, n=n_total)
                self.dev_rows[g.index] = torch.from_numpy(self.host[g.index]).to(dev)
        self.X_host_sample = next(iter(self.host.values())) if self.host else np.zeros((0, cfg.d), np.float32)
        self.units = 1
        self.h2d_bytes = sum(a.nbytes for a in self.host.values())

    def _src(self, table):
        gs = self.groups

        def source(a, b):
            for g in gs:
                if g.row_start <= a < g.row_end:
                    return table[g.index][a - g.row_start:b - g.row_start]
            raise IndexError(a)
        return source

    def _run(self, table):
        from paper_1502_04265_b200.distributed import DeviceOps, run_piecy_mr_sharded
        ops = DeviceOps(self.mcfg, self.dev)
        dev = self.dev
        import torch
        src = self._src(table)

        def source(a, b):
            blk = src(a, b)
            return blk if isinstance(blk, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(blk)).to(dev)
        return run_piecy_mr_sharded(source, self.n, self.cfg.d, self.mcfg, rank=self.rank, world=self.world, ops=ops)

    def coreset_device(self):
        import torch
        cs = self._run(self.dev_rows)
        if cs is None:
            return None, None, None
        P = torch.from_numpy(cs.points).to(self.dev)
        w = torch.from_numpy(cs.weights).to(self.dev)
        return P, w, None

    def coreset_public(self):
        return self._run(self.host)

    def cpu_rows(self):
        return self.X_host_sample


def measure_gemm_peaks(dev):
    """cuBLAS TF32 and FP64 GEMM throughput on this GPU (best of a few 8192^3 /
    4096^3 runs): the denominators of the tensor-core and DMMA distance kernels,
    which MEASURED_PEAKS.json does not carry (it has bf16 and HBM only)."""
    import torch
    out = {}
    prev = torch.backends.cuda.matmul.allow_tf32
    try:
        for name, dt, nn, reps in (("tf32_tflops", torch.float32, 8192, 5), ("fp64_tflops", torch.float64, 4096, 3)):
            torch.backends.cuda.matmul.allow_tf32 = name == "tf32_tflops"
            a = torch.randn(nn, nn, dtype=dt, device=dev)
            b = torch.randn(nn, nn, dtype=dt, device=dev)
            torch.matmul(a, b)
            best = 1e30
            for _ in range(reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                torch.matmul(a, b)
                e1.record()
                e1.synchronize()
                best = min(best, e0.elapsed_time(e1))
            out[name] = 2.0 * nn ** 3 / (best / 1e3) / 1e12
            del a, b
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    return out


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return 0

    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    from paper_1502_04265_b200 import _native as nat
    from paper_1502_04265_b200 import workloads as W
    from paper_1502_04265_b200.evaluation import kmeans_repetitions, kmeans_repetitions_device

    cfg = W.CONFIGS[args.config]
    n_total = args.rows or cfg.n
    d = cfg.d
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    if cfg.entry == "piecy":
        work = PiecyWork(cfg, args, dev)
    else:
        work = MrWork(cfg, args, dev, n_total, rank, world)
    X = work.X_host_sample
    n = n_total
    gemm_peaks = measure_gemm_peaks(dev) if rank == 0 and not args.ncu else {}

    def step_device():
        st0 = torch.cuda.current_stream()
        a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        a.record(st0)
        P, w, eng = work.coreset_device()
        b.record(st0)
        F, costs = 0, None
        if P is not None:
            F = int(P.shape[0])
            C, costs = kmeans_repetitions_device(P, w, cfg.k, cfg.reps, cfg.seed, cfg.max_iters, 1e-4)
            step_device.C = C
        c.record(st0)
        c.synchronize()
        step_device.phases.append((a.elapsed_time(b), b.elapsed_time(c)))
        step_device.engine = eng
        return F, costs
    step_device.phases = []
    step_device.engine = None
    step_device.C = None

    if args.ncu:
        step_device()
        torch.cuda.synchronize()
        return 0

    # nvidia-smi is started before the warm-up: its start-up (NVML initialisation
    # holds driver locks for several hundred ms and stalled the launches of whatever
    # steps it overlapped: 97 / 99 / 97 / 112 / 125 ms) then lands in untimed
    # steps.  Only the samples taken inside the timed region are reported.
    clocks = ClockSampler(local)
    clocks.start()
    clocks.wait_first()
    for _ in range(args.warmup):
        step_device()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks.mark()
    l0 = nat.launch_count()
    st = torch.cuda.current_stream()
    evs = []
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    for _ in range(args.steps):
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        F, costs = step_device()
        e1.record(st)
        evs.append((e0, e1))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = nat.launch_count() - l0
    clk = clocks.stop()
    ms_steps = [a.elapsed_time(b) for a, b in evs]
    ms_timed = float(np.sum(ms_steps))

    # per-kernel breakdown: a second pass of the same steps with the engine's
    # per-launch event timing on (its host-side event reads sit between
    # launches, so it is kept out of the timed steps above)
    nat.prof_reset()
    nat.prof_enable(True)
    torch.cuda.synchronize()
    evp = []
    for _ in range(args.steps):
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        step_device()
        e1.record(st)
        evp.append((e0, e1))
    torch.cuda.synchronize()
    nat.prof_enable(False)
    ms = float(np.sum([a.elapsed_time(b) for a, b in evp]))   # profiled pass: denominators of the shares
    prof = {k: nat.prof_read(k) for k in ("resolve", "chain", "reattach")}
    # K1 useful-work fraction: the last step's engine counters
    work_k1 = None
    if step_device.engine is not None and hasattr(step_device.engine, "work"):
        work_k1 = step_device.engine.work()
    prof_x = {k: nat.prof_read(k) for k in ("gemm", "seed", "lloyd")}

    # e2e: public API with host buffers (H2D of the stream, D2H of coreset + centers + costs)
    e2e_times = []
    h2d = d2h = 0
    # untimed passes of the public path, as many as the device arm's warm-up (at most 3): the
    # first passes pay for the pinned staging buffers and for the caching allocator's copy-stream
    # blocks (cudaMalloc), e.g. 131 / 127 / 102 / 102 / 102 ms on cfg2 with a single warm pass
    e2e_warm = max(1, min(args.warmup, 3))
    for it in range(e2e_warm + max(1, min(args.steps, 5))):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        cs = work.coreset_public()
        if cs is not None:
            runs = kmeans_repetitions(cs.points, cs.weights.astype(np.float64), cfg.k, reps=cfg.reps,
                                      seed=cfg.seed, max_iters=cfg.max_iters, tol=1e-4)
        torch.cuda.synchronize()
        if it >= e2e_warm:
            e2e_times.append(time.perf_counter() - t0)
        h2d = work.h2d_bytes + (cs.points.nbytes + cs.weights.size * 8 + cfg.reps * cfg.k * 8 if cs is not None else 0)
        d2h = (cs.points.nbytes + cs.weights.nbytes + sum(c.nbytes + 8 for c, _ in runs)) if cs is not None else 0

    # parity of this run's public-API result against the unmodified reference's
    # output on the same bytes (tests/golden/full_<cfg>.npz, written by
    # tests/golden/make_fullsize.py); full-size streams only
    parity = None
    if rank == 0 and cs is not None and args.rows in (None, cfg.n):
        sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
        try:
            import fullsize as FS
            fx = FS.load(cfg.name)
            if fx is None:
                parity = {"checked": False, "why": f"no fixture tests/golden/full_{cfg.name}.npz"}
            else:
                Cr = np.stack([c for c, _ in runs])
                cr = np.array([v for _, v in runs])
                parity = FS.compare(fx, cs.points, cs.weights, Cr, cr, exact_points=cfg.svd_dim >= cfg.d)
                parity.update({"checked": True, "against": f"tests/golden/full_{cfg.name}.npz (unmodified reference "
                                                          f"run_{'piecy' if cfg.entry == 'piecy' else 'piecy_mr'} + "
                                                          "kmeans_repetitions on the same stream bytes)",
                               "tolerance": "weights/order exact; points bit-exact without projection, else 1e-9 "
                                            "of row scale; costs and centres 1e-9 relative"})
        except Exception as exc:   # a checker failure must not hide the measurement
            parity = {"checked": False, "why": f"checker error: {exc!r}"}

    # full-data second pass, unweighted SSE of the whole
    # stream against every repetition's centres (evaluate_cost_multi), stream
    # resident in HBM; one GPU (it is a separate pass, not part of the step)
    full_eval = None
    if world == 1 and step_device.C is not None and not args.no_full_eval:
        from paper_1502_04265_b200.evaluation import evaluate_cost_multi
        Cs = [step_device.C[r].cpu().numpy() for r in range(step_device.C.shape[0])]
        stream = work.Xd if hasattr(work, "Xd") else torch.cat([work.dev_rows[g] for g in sorted(work.dev_rows)])
        evaluate_cost_multi(Cs, stream[: min(int(stream.shape[0]), 65536)])   # warm-up
        flush.fill_(1.0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fcost = evaluate_cost_multi(Cs, stream)
        torch.cuda.synchronize()
        tf = time.perf_counter() - t0
        flops = 2.0 * int(stream.shape[0]) * sum(c.shape[0] for c in Cs) * d
        full_eval = {"value": int(stream.shape[0]) / tf, "unit": "points/s", "center_sets": len(Cs), "k": cfg.k,
                     "seconds": tf, "achieved_tflops": flops / tf / 1e12,
                     "frac_of_fp64_peak": (flops / tf / 1e12) / max(gemm_peaks.get("fp64_tflops", 40.0), 1e-9)
                     if rank == 0 else None,
                     "costs": fcost, "chunk": 8192,
                     "note": "evaluate_cost_multi over the resident stream (chunks of 8192 rows, fp64 DMMA "
                             "distance + first-min per set, chunk costs summed in order)"}

    t_local = torch.tensor([ms_timed / args.steps, float(np.mean(e2e_times))], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
    ms_step, e2e_s = float(t_local[0]), float(t_local[1])

    if rank == 0:
        peaks = {}
        try:
            with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
                peaks = json.load(f)
        except Exception:
            pass
        hbm = float(peaks.get("hbm_gbs", 6650.0))
        peak_src = ("MEASURED_PEAKS.json hbm_gbs (driver-measured copy bandwidth)" if "hbm_gbs" in peaks
                    else "fallback: B200_PROFILING.md HBM figure")
        # per-launch DRAM traffic from the committed ncu --set full captures
        # (profiles/ncu_traffic.json, tools/ncu_traffic.py); None when the
        # config has no capture
        ncu_tr = {}
        try:
            with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
                ncu_tr = json.load(f).get(cfg.name, {})
        except Exception:
            pass

        def traffic(pred):
            ks = [v["bytes_per_launch"] for k, v in ncu_tr.get("kernels", {}).items() if pred(k)]
            return max(ks) if ks else None

        # Per-kernel rooflines from the engine's live event pairs (profiled pass).
        # Peaks: HBM from MEASURED_PEAKS.json; TF32 and FP64 are not in that
        # file, so cuBLAS GEMMs measured at start-up by this run stand in.
        K = args.steps
        tf32 = gemm_peaks.get("tf32_tflops")
        fp64 = gemm_peaks.get("fp64_tflops")
        tf32_src = "measured in this run: cuBLAS TF32 GEMM 8192^3 (MEASURED_PEAKS.json has bf16/HBM only)"
        fp64_src = "measured in this run: cuBLAS FP64 GEMM 4096^3 (MEASURED_PEAKS.json has bf16/HBM only)"
        if tf32 is None:
            tf32, tf32_src = 1100.0, "fallback: TF32 ~ half the bf16 dense peak"
        if fp64 is None:
            fp64, fp64_src = 37.0, "fallback: B200 FP64 datasheet"
        rooflines = []

        def share(ms_):
            return ms_ / ms if ms > 0 else None

        g_ms, g_cnt, g_flops = prof_x["gemm"]
        c_ms, c_cnt, c_units = prof["chain"]
        r_ms, r_cnt, r_units = prof["resolve"]
        a_ms, a_cnt, a_units = prof["reattach"]
        if g_ms > 0:
            ach = g_flops / (g_ms / 1e3) / 1e12
            pk = tf32 / 3.0
            rooflines.append({"kernel": "k_tc_dots (K1 panel contraction: split-TF32 on tcgen05, big groups only)"
                              if d <= 256 else "k_tc_dots (K1 full-set contraction, split-TF32 on tcgen05)",
                              "bound": "tensor", "achieved": ach, "peak": pk, "unit": "TFLOP/s", "frac": ach / pk,
                              "launches_per_step": g_cnt / K, "traffic": traffic(lambda k: k.startswith("k_tc_dots")),
                              "ms_per_step": g_ms / K, "share_of_step": share(g_ms),
                              "peak_source": tf32_src + " / 3 (three TF32 products per fp32-faithful product); "
                                             "achieved = 2*M*N*d per launch (M batch rows x N panel columns)"})
        walk_ms = max(0.0, c_ms - g_ms)
        if c_cnt:
            # chain walk: per item the visited members' reference rows (8d B
            # each, from L2/HBM) -- latency-bound pointer chasing down the tree
            vis = (work_k1 or {}).get("member_visits")
            bytes_ = (vis * 8.0 * d) if vis else None
            rooflines.append({"kernel": "k_chain2 (K1 chain walk: direct fp64 scans + panel reads, per-level argmin)",
                              "bound": "latency", "achieved": (c_units / (walk_ms / 1e3)) if walk_ms else None,
                              "unit": "items/s", "peak": None, "frac": None,
                              "traffic": traffic(lambda k: k.startswith("k_chain2")),
                              "ms_per_step": walk_ms / K, "share_of_step": share(walk_ms),
                              "ns_per_item": walk_ms * 1e6 / c_units if c_units else None,
                              "l2_gbs": (bytes_ / (walk_ms / 1e3) / 1e9) if bytes_ and walk_ms else None,
                              "note": "latency-bound: ~3 dependent L2 round trips per tree level; the visited "
                                      "reference rows (member visits x 8d bytes, l2_gbs) are L2-resident"})
        # K3 algorithmic bytes per point: x row read, s row read+write (fp64),
        # node scalars (w, q, sn) read+write, chain entry (id + part)
        bytes_per_pt = 8 * d * 3 + 48 + 12
        achieved = (r_units * bytes_per_pt) / (r_ms / 1e3) / 1e9 if r_ms > 0 else 0.0
        rooflines.append({"kernel": "k_plan + k_resolve2/3 (K3 subtree-parallel resolve + CF update)", "bound": "hbm",
                          "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                          "traffic": traffic(lambda k: k.startswith("k_resolve") and ("x<" in k or k.endswith("1>"))),
                          "traffic_unit": "bytes per launch (ncu dram read+write of the window's resolve launch; ncu replays start cold, in the bench the tree is L2-resident)",
                          "bytes_per_launch": (r_units * bytes_per_pt / r_cnt) if r_cnt else None,
                          "peak_source": peak_src,
                          "note": "latency-bound: one CTA per k_plan domain walks its items in stream order; "
                                  "algorithmic bytes = 24*d+60 per point",
                          "ns_per_point": (r_ms * 1e6 / r_units) if r_units else None,
                          "ms_per_step": r_ms / K, "share_of_step": share(r_ms)})
        if a_ms > 0:
            ab = a_units * (8.0 * d * 3 + 48)
            rooflines.append({"kernel": "k_rchain + k_reattach2/3 (K4 rebuild reattach)", "bound": "hbm",
                              "achieved": ab / (a_ms / 1e3) / 1e9, "peak": hbm, "unit": "GB/s",
                              "frac": ab / (a_ms / 1e3) / 1e9 / hbm, "traffic": None,
                              "ms_per_step": a_ms / K, "share_of_step": share(a_ms),
                              "ns_per_node": a_ms * 1e6 / a_units if a_units else None, "peak_source": peak_src,
                              "note": "latency-bound in-order reattach; algorithmic bytes = 24*d+48 per node"})
        s_ms, s_cnt, s_bytes = prof_x["seed"]
        if s_ms > 0:
            ach = s_bytes / (s_ms / 1e3) / 1e9
            rooflines.append({"kernel": "k_seed_coop (weighted k-means++, all repetitions)", "bound": "hbm",
                              "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                              "launches_per_step": s_cnt / K, "traffic": None,
                              "ms_per_step": s_ms / K, "share_of_step": share(s_ms),
                              "peak_source": peak_src + " HBM; algorithmic bytes = (k-1)(8nd + 24n*reps + 8n)"})
        l_ms, l_cnt, l_flops = prof_x["lloyd"]
        if l_ms > 0:
            ach = l_flops / (l_ms / 1e3) / 1e12
            rooflines.append({"kernel": "k_dist_tile<3> (Lloyd assignment, fp64 DMMA + argmin)", "bound": "tensor",
                              "achieved": ach, "peak": fp64, "unit": "TFLOP/s", "frac": ach / fp64,
                              "launches_per_step": l_cnt / K, "traffic": None,
                              "ms_per_step": l_ms / K, "share_of_step": share(l_ms),
                              "peak_source": fp64_src + "; achieved = 2*n*k*d per repetition"})
        kernel_ms = {k: {"ms": v[0] / K, "launches": v[1] / K, "units": v[2] / K} for k, v in prof.items()}
        # the headline roofline is the single kernel (set) with the largest
        # measured share of the step; dominant_kernel names the same entry
        roof = max(rooflines, key=lambda r: r.get("ms_per_step") or 0.0)
        dom = roof["kernel"]
        rooflines = [r for r in rooflines if r is not roof]
        cpu = None
        if not args.no_cpu_baseline:
            kind = baseline_kind()
            rows, t, _ = cpu_sample(cfg, n, kind)
            cpu = {"value": rows / t, "unit": "points/s", "cores": os.cpu_count() or 1, "kind": kind,
                   "sample": f"first {rows} of {n} rows of {cfg.name}, one pass of "
                             f"{'the unmodified reference (baseline/_ref)' if kind == 'reference' else 'the oracle port'}"
                             f" incl. kmeans_repetitions", **cpu_env(kind)}
            if kind == "reference":   # the C port beside it, same sample rule
                rows2, t2, _ = cpu_sample(cfg, n, "port")
                cpu["port"] = {"value": rows2 / t2, "unit": "points/s", "cores": os.cpu_count() or 1,
                               "sample": f"first {rows2} of {n} rows, oracle/ C BICO + numpy"}
        line = {
            "metric": METRIC, "value": work.units * n / (ms_step / 1e3), "unit": "points/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": work.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_json(cfg, n, world),
            "e2e": {"value": work.units * n / e2e_s, "unit": "points/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "steps": len(e2e_times), "warmup": e2e_warm,
                    "ms_steps": [round(1e3 * t, 2) for t in e2e_times],
                    "timing": "host wall clock around the public call (H2D, kernels, D2H), synchronize on both sides; mean"},
            "gpu_launches": int(launches),
            "roofline": roof,
            "rooflines": rooflines,
            "full_data_eval": full_eval,
            "parity": parity,
            "gemm_peaks": gemm_peaks,
            "cpu_baseline": cpu,
            "clocks": clk,
            "kernel_ms_per_step": kernel_ms,
            "dominant_kernel": dom,
            "k1_work": work_k1,
            "coreset_size": int(F),
            "engine_counters": step_device.engine.counters() if step_device.engine is not None else None,
            "step_ms": ms_steps,
            "phase_ms": [{"coreset": round(p[0], 2), "kmeans": round(p[1], 2)} for p in step_device.phases[-2 * args.steps:-args.steps]],
            "profiled_ms_per_step": ms / args.steps,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
