#!/usr/bin/env python
"""bench.py — FP64 arrowhead tile Cholesky on B200.

Default workload (``--workload auto``): N=1 -> C4, the largest single-GPU
BASELINE configuration (n=1,000,000, b=2000, t=500, HBM-resident); N>1 -> C5,
the 64-problem INLA batch sharded over the ranks (the only workload that
shards).

One *step* (single factorisations) = device scatter of the HBM-resident CSC
values into tile storage + one persistent-kernel factorisation with fused
log-determinant.  ``value`` = factorizations/s over all ranks.  ``e2e`` = the
same through the public API ``api.factorize`` from HOST CSC values (H2D,
scatter, factorisation, D2H of logdet/fail word inside the timed region).
The N=1 line carries ``batch_c5``: the C5 batch on one GPU (first point of
the 1->8 curve).

    python bench.py [--workload auto|c1..c5] [--tile NT] [--gpus N --steps K --warmup W]
    python bench.py --impl reference ...     # reference CPU arm (oracle port, all host cores)
    python bench.py --measure-peaks           # FP64 DMMA / DGEMM peaks -> profiles/

``--gpus N`` with N>1 re-executes itself under torch.distributed.run (one rank
per GPU, NCCL) unless already launched that way.  The reference arm never
imports the product package: matrices and op streams come from oracle/ only.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# default tile per workload: 128 (128x64 update blocks; the tile sweep in
# profiles/ compares 120-480); swept with --tile
DEFAULT_NT = {"c1": 128, "c2": 128, "c3": 128, "c4": 128, "c5": 128}
N_OF = {"c1": 10_000, "c2": 100_000, "c3": 200_010, "c4": 1_000_000, "c5": 200_010}
PEAKS_FILE = os.path.join(ROOT, "profiles", "fp64_peaks.json")
FP64_FALLBACK_TFLOPS = 37.0  # NVIDIA B200 FP64 (tensor) nominal, used only if unmeasured
CPU_SAMPLE_FLOPS_OURS = 4.0e11   # ~15 s of one core (cpu_baseline leg)
CPU_SAMPLE_FLOPS_REF = 1.0e11    # ~4 s per process per step (reference arm)


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="auto", choices=["auto", "c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--tile", type=int, default=0)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--no-batch", action="store_true", help="N=1: skip the batch_c5 sub-measurement")
    ap.add_argument("--no-profile", action="store_true")
    ap.add_argument("--measure-peaks", action="store_true")
    ap.add_argument("--ref-procs", type=int, default=0)
    ap.add_argument("--executor", default="persistent", choices=["persistent", "graph", "direct"])
    ap.add_argument("--lookahead", type=int, default=None, help="bulk-update lookahead depth (default: api default)")
    ap.add_argument("--lanes", type=int, default=4, help="c5: factorisations in flight per GPU")
    ap.add_argument("--share", type=int, default=4,
                    help="c5: persistent kernels sharing the GPU (each takes 1/share of the SMs; "
                         "C5 on one B200: 12.7 / 15.4 / 16.0 fact/s at 1 / 2 / 4)")
    ap.add_argument("--occupancy", type=int, default=0, help="persistent CTAs per SM (0 = plan default)")
    ap.add_argument("--ordering", default="auto",
                    help="auto (SPEC policy) | identity (C4: auto provably picks identity, zero fill)")
    return ap.parse_args(argv)


def workload_of(a) -> str:
    if a.workload != "auto":
        return a.workload
    return "c4" if a.gpus <= 1 else "c5"


def maybe_spawn(a) -> bool:
    """--gpus N>1 outside torchrun: re-exec under torch.distributed.run."""
    if a.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return False
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def common_config(name, nt, world, a):
    """The workload description both arms print (identical by construction)."""
    from oracle.workloads import WORKLOAD_DESC
    cfg = {"workload": WORKLOAD_DESC[name], "tile": nt, "n": N_OF[name], "ordering": a.ordering,
           "l2": "inputs larger than L2 (tile storage >= 0.9 GB per factorisation; 126 MB L2)"}
    if name == "c5":
        cfg["problems"] = 64
        cfg["parallelism"] = f"batch sharded over {world} GPU(s), contiguous blocks, NCCL all-gather of results"
    else:
        cfg["parallelism"] = f"replicas x{world} (one factorisation per GPU per step)"
    return cfg


# ------------------------------------------------------------------ clocks --
class Clocks:
    """nvidia-smi sampler (200 ms) running during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", str(self.idx)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.3)  # sampler running before the timed region starts
        except OSError:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------ peaks --
def measure_peaks():
    import torch
    from paper_2501_02483_b200._lib import check, lib, f64p
    out = {"how": "DMMA m8n8k4 register microbenchmark (all SMs) and torch.matmul float64 "
                  "8192^3 (cuBLAS DGEMM), best of 5, CUDA events", "gpu": torch.cuda.get_device_name()}
    best = 0.0
    cfgs = {}
    for bps, wpb in ((1, 4), (2, 4), (1, 8), (2, 8), (4, 8)):
        v = np.zeros(1)
        vals = []
        for _ in range(3):
            check("dmma", lib.tc_bench_dmma_peak(200000, bps, wpb, v.ctypes.data_as(f64p)))
            vals.append(float(v[0]))
        cfgs[f"{bps}x{wpb}warps"] = max(vals)
        best = max(best, max(vals))
    out["dmma_tflops"] = best
    out["dmma_configs"] = cfgs
    a = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
    b = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
    for _ in range(2):
        a @ b
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        a @ b
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    out["dgemm_tflops"] = 2 * 8192 ** 3 / (min(ts) * 1e-3) / 1e12
    out["fp64_peak_tflops"] = max(out["dmma_tflops"], out["dgemm_tflops"])
    os.makedirs(os.path.dirname(PEAKS_FILE), exist_ok=True)
    with open(PEAKS_FILE, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out))


def fp64_peak():
    try:
        with open(PEAKS_FILE) as f:
            d = json.load(f)
        return float(d["fp64_peak_tflops"]), "measured (profiles/fp64_peaks.json: max of DMMA microbenchmark and cuBLAS DGEMM)"
    except (OSError, KeyError, ValueError):
        return FP64_FALLBACK_TFLOPS, "fallback nominal B200 FP64 (unmeasured)"


def traffic_of(name, nt):
    """dram__bytes_read.sum + dram__bytes_write.sum of the dominant kernel per
    launch, from the committed ncu --set full capture (profiles/traffic.json),
    or None when this workload/tile was not captured."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            d = json.load(f).get(f"{name}@{nt}")
        return (float(d["bytes_per_launch"]), d.get("source", "")) if d else (None, "")
    except (OSError, ValueError, KeyError):
        return None, ""


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md)"


# ----------------------------------------------- CPU arms (oracle only) --
def oracle_sample(name, nt, target_flops, with_storage=True):
    """Bounded sample of one factorisation of workload `name` for the CPU
    arms: the reference op stream of the first K tile columns (oracle/
    workloads.prefix_problem), K chosen for ~target_flops tile flops; plus the
    tile flops of the WHOLE factorisation, so sample time scales to
    factorizations/s exactly by flop fraction."""
    import oracle.workloads as OW
    if name == "c4":
        n, b, t = OW.C4_SPEC
        F, _ = OW.arrowhead_tile_flops(n, b, t, nt)
        T = -(-n // nt)
        K = max(1, min(T, int(np.ceil(target_flops / (F / T)))))
        nn, cp, ri, v = OW.c4_columns(min(K * nt, n - t))
        pr = OW.prefix_problem(nn, cp, ri, v, nt, K, with_storage=with_storage)
        pr["F_total"] = F
        return pr
    gen = {"c1": OW.c1, "c2": OW.c2, "c3": OW.c3, "c5": OW.c3}[name]
    n, cp, ri, v = gen()
    full = OW.prefix_problem(n, cp, ri, v, nt, 1 << 30, with_storage=False)
    T = full["columns"]
    F = full["flops"]
    if F <= target_flops * 1.2:
        pr = OW.prefix_problem(n, cp, ri, v, nt, T, with_storage=with_storage)
    else:
        # prefix flops are not uniform per column: grow K geometrically
        K = max(1, int(T * target_flops / F))
        while True:
            pr = OW.prefix_problem(n, cp, ri, v, nt, K, with_storage=False)
            if pr["flops"] >= target_flops or K >= T:
                break
            K = min(T, int(K * 1.25) + 1)
        pr = OW.prefix_problem(n, cp, ri, v, nt, K, with_storage=with_storage)
    pr["F_total"] = F
    return pr


def time_sample(pr):
    """Oracle run_ops (numba loops + OpenBLAS via np.dot, 1 thread) over the
    sample; returns (seconds, factor storage)."""
    import oracle as O
    nt = pr["storage"].shape[1]
    sc = np.zeros((0, nt, nt))
    O.run_ops(pr["storage"][:1].copy(), sc, pr["op"][:0], pr["dst"][:0], pr["src1"][:0], pr["src2"][:0], 0, 0)
    st = pr["storage"].copy()
    t0 = time.perf_counter()
    p, info = O.run_ops(st, sc, pr["op"], pr["dst"], pr["src1"], pr["src2"], 0, pr["ops"])
    dt = time.perf_counter() - t0
    if info != -1:
        raise RuntimeError(f"oracle sample failed at op {p} (info {info})")
    return dt, st


def _ref_worker(args):
    path, q_in, q_out = args
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    import oracle as O
    z = np.load(path)
    tpl = z["storage"]
    op, dst, s1, s2 = z["op"], z["dst"], z["src1"], z["src2"]
    nt = tpl.shape[1]
    sc = np.zeros((0, nt, nt))
    st = np.empty_like(tpl)
    O.run_ops(tpl[:1].copy(), sc, op[:0], dst[:0], s1[:0], s2[:0], 0, 0)  # JIT
    q_out.put("ready")
    while True:
        cmd = q_in.get()
        if cmd is None:
            break
        np.copyto(st, tpl)
        t0 = time.perf_counter()
        p, info = O.run_ops(st, sc, op, dst, s1, s2, 0, op.size)
        q_out.put((time.perf_counter() - t0, int(info)))


def run_reference(a, name, nt, world):
    """Reference CPU implementation of the path (oracle port of
    _backend_numba.run_ops over the reference op stream) on
    the box's host cores: one process per core, each running the same
    bounded sample (the first K tile columns of one factorisation) per step;
    value = processes x (sample tile flops / factorisation tile flops) / wall."""
    import multiprocessing as mp
    import tempfile
    cores = len(os.sched_getaffinity(0))
    t0 = time.perf_counter()
    pr = oracle_sample(name, nt, CPU_SAMPLE_FLOPS_REF)
    setup_s = time.perf_counter() - t0
    per_proc = 2.5 * pr["storage"].nbytes / 1e9 + 0.5
    try:
        import psutil
        mem = psutil.virtual_memory().available / 1e9
    except ImportError:
        mem = 32.0
    procs = a.ref_procs or max(1, min(cores, int(mem * 0.6 / per_proc)))
    tmpd = tempfile.mkdtemp(prefix="tc_ref_")
    path = os.path.join(tmpd, "sample.npz")
    np.savez(path, storage=pr["storage"], op=pr["op"], dst=pr["dst"], src1=pr["src1"], src2=pr["src2"])
    ctx = mp.get_context("spawn")
    qin = [ctx.Queue() for _ in range(procs)]
    qout = ctx.Queue()
    ps = [ctx.Process(target=_ref_worker, args=((path, qin[i], qout),)) for i in range(procs)]
    for p in ps:
        p.start()
    for _ in ps:
        assert qout.get() == "ready"

    def step():
        t0 = time.perf_counter()
        for q in qin:
            q.put(1)
        res = [qout.get() for _ in ps]
        assert all(r[1] == -1 for r in res), "reference sample failed"
        return time.perf_counter() - t0

    for _ in range(a.warmup):
        step()
    walls = [step() for _ in range(a.steps)]
    for q in qin:
        q.put(None)
    for p in ps:
        p.join()
    try:
        os.remove(path)
        os.rmdir(tmpd)
    except OSError:
        pass
    wall = float(np.mean(walls))
    frac = pr["flops"] / pr["F_total"]
    value = procs * frac / wall
    metric, unit = ("batched factorizations/s (FP64, C5)" if name == "c5" else
                    "factorizations/s (FP64 time-to-factor)"), "factorizations/s"
    sample = (f"{procs} processes x the first {pr['columns']} tile columns of one {name} factorisation "
              f"({pr['ops']} reference ops, {pr['flops']:.3e} of {pr['F_total']:.3e} tile flops = "
              f"{100 * frac:.2f}%) per step; oracle run_ops = numba loops + OpenBLAS dgemm, 1 thread each")
    line = {"impl": "reference", "metric": metric, "value": value, "unit": unit, "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": wall * 1e3,
            "higher_is_better": True, "scaling": "strong" if name == "c5" else "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "config": common_config(name, nt, world, a),
            "cpu_baseline": {"value": value, "unit": unit, "cores": procs, "kind": "port", "sample": sample,
                             "wall_s_per_step": wall, "sample_fraction": frac, "setup_s": setup_s},
            "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------- GPU arm, batch --
def run_batch(a, nt, rank, world, sub=False):
    """C5: 64 INLA factorisations Q(theta) sharing the C3 pattern, sharded in
    contiguous blocks over the ranks (strong scaling), `lanes` in flight per
    GPU.  Device step: values assembled on the GPU from the 13 basis vectors
    of the family (tc_plan_pack_lincomb), factorised, log-determinants handed
    off device-side, one NCCL all-gather of the 64 log-determinants (N>1).
    e2e: api.logdet_many_sharded from host CSC values (H2D per problem) + the
    all-gather."""
    import torch
    import torch.distributed as dist
    from paper_2501_02483_b200 import api, matcore, workloads as W
    from paper_2501_02483_b200.batch import shard_range
    fam = W.InlaFamily()
    thetas = W.c5_thetas()
    P = len(thetas)
    lo, hi = shard_range(P, world, rank)
    L = max(1, a.lanes)
    opts = api.FactorOptions(tile_size=nt, ordering=a.ordering, executor=a.executor, occupancy=a.occupancy,
                             concurrent=max(1, a.share))
    m0 = fam.matrix(*thetas[0])
    t0 = time.perf_counter()
    pat = api._pattern_for(m0, opts)
    setup_s = time.perf_counter() - t0
    plan = pat.plan
    F = plan.info()["tile_flops"]
    coefs = [fam.lincomb(*t)[0] for t in thetas]
    basis = fam.lincomb(*thetas[0])[1]
    bd = torch.from_numpy(np.stack([pat.permuted_values(matcore.SymmetricCsc(m0.n, m0.col_ptr, m0.row_idx, b))
                                    for b in basis])).cuda()
    offs = pat.offsets()
    streams = [torch.cuda.Stream() for _ in range(L)]
    stor = [plan.new_storage() for _ in range(L)]
    nloc = hi - lo
    fail = torch.zeros(max(1, nloc), dtype=torch.int64, device="cuda")
    ld = torch.zeros(max(1, nloc), dtype=torch.float64, device="cuda")
    cap = -(-P // world)
    gbuf = torch.zeros(cap, dtype=torch.float64, device="cuda")
    gout = [torch.zeros(cap, dtype=torch.float64, device="cuda") for _ in range(world)]
    main = torch.cuda.current_stream()

    def step():
        start = torch.cuda.Event(enable_timing=True)
        start.record(main)
        for s in streams:
            s.wait_stream(main)
        for j in range(nloc):
            lane = j % L
            s = streams[lane]
            sh = s.cuda_stream
            plan.pack_lincomb(bd, coefs[lo + j], offs, stor[lane], sh)
            plan.factorize_async(stor[lane], lane, sh)
            plan.copy_result(lane, sh, fail[j:j + 1], ld[j:j + 1])
        for s in streams:
            main.wait_stream(s)
        gbuf[:nloc].copy_(ld[:nloc])
        if world > 1:
            dist.all_gather(gout, gbuf)
        end = torch.cuda.Event(enable_timing=True)
        end.record(main)
        return start, end

    t0 = time.perf_counter()
    for _ in range(max(a.warmup if not sub else 1, 1)):
        step()
    torch.cuda.synchronize()
    print(f"[c5] warm-up {time.perf_counter() - t0:.1f} s", file=sys.stderr, flush=True)
    ok = bool((fail[:nloc] == np.iinfo(np.int64).max).all().item()) if nloc else True
    if not ok:
        raise RuntimeError("a batch factorisation failed")
    ld_ref = ld[:nloc].clone()
    steps = 1 if sub else a.steps
    if world > 1:
        dist.barrier()
    clk = Clocks(int(os.environ.get("LOCAL_RANK", "0")))
    clk.start()
    torch.cuda.synchronize()
    evs = [step() for _ in range(steps)]
    torch.cuda.synchronize()
    clocks = clk.stop()
    ms = evs[0][0].elapsed_time(evs[-1][1]) / steps
    repro_dev = bool(torch.equal(ld[:nloc], ld_ref))
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    # ---- end to end: host values of this rank's problems -> logdet_many_sharded
    probs = [None] * P
    for i in range(lo, hi):
        probs[i] = fam.matrix(*thetas[i])
    h2d = sum(probs[i].nnz * 8 for i in range(lo, hi))
    e2e_ms = []
    for i in range((1 if sub else a.e2e_steps) + 1):
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        lds = api.logdet_many_sharded(probs, opts, lanes=L)
        dt = (time.perf_counter() - t0) * 1e3
        if i > 0:
            e2e_ms.append(dt)
    e2e = float(np.mean(e2e_ms)) if e2e_ms else float("nan")
    if world > 1:
        t = torch.tensor([e2e], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e = float(t.item())
    ldr = ld_ref.cpu().numpy()[:nloc]
    repro_api = bool(np.array_equal(lds[lo:hi], ldr))
    peak, peak_src = fp64_peak()
    value = P * 1000.0 / ms
    line = {"metric": "batched factorizations/s (FP64, C5)", "value": value, "unit": "factorizations/s",
            "n_gpus": world, "steps": steps, "warmup": a.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": common_config("c5", nt, world, a),
            "lanes_per_gpu": L, "grid_share": max(1, a.share), "nnz": m0.nnz,
            "roofline": {"bound": "tensor", "kernel": "k_persist x lanes", "achieved": P * F / (ms * 1e-3) / 1e12,
                         "peak": peak, "unit": "TFLOP/s", "frac": P * F / (ms * 1e-3) / 1e12 / peak,
                         "traffic": None, "peak_source": peak_src},
            "gpu_launches": 5 * max(1, nloc) * steps, "setup_s": setup_s,
            "bitwise_reproducible": repro_dev and repro_api,
            "e2e": {"value": P * 1000.0 / e2e, "unit": "factorizations/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(16 * nloc + 8 * P), "ms_per_step": e2e,
                    "path": "api.logdet_many_sharded(host CSC values)" + (" + NCCL all_gather" if world > 1 else "")},
            "clocks": clocks}
    if sub:
        return {k: line[k] for k in ("metric", "value", "unit", "ms_per_step", "steps", "roofline", "e2e",
                                     "bitwise_reproducible", "lanes_per_gpu", "clocks")}
    if rank == 0:
        print(json.dumps(line), flush=True)


# --------------------------------------------------------------- GPU arm --
def build_matrix(name):
    from paper_2501_02483_b200 import workloads as W
    return {"c1": W.c1, "c2": W.c2_variable_band, "c3": W.c3, "c4": W.c4}[name]()


def prefix_parity(pat, storage, pr, nt):
    """Compare the device factor with the oracle's factor of the first K tile
    columns (the CPU sample): relative Frobenius difference over those tiles
    and the partial log-determinant (2 sum log diag over columns < K)."""
    fg = pat.symbolic.factor_grid
    K = pr["columns"]
    sel = np.nonzero(pr["gcol"] < K)[0]
    slots = fg.slots_of(pr["grow"][sel], pr["gcol"][sel])
    assert (slots >= 0).all()
    import torch
    got = storage[torch.from_numpy(slots).to(storage.device)].cpu().numpy()
    ref = pr["factor"][sel]
    rel = float(np.linalg.norm(got - ref) / np.linalg.norm(ref))
    dg = np.nonzero(pr["grow"][sel] == pr["gcol"][sel])[0]
    ld_g = 2.0 * sum(float(np.sum(np.log(np.diagonal(got[i].T)))) for i in dg)
    ld_r = 2.0 * sum(float(np.sum(np.log(np.diagonal(ref[i].T)))) for i in dg)
    return {"prefix_columns": int(K), "prefix_tiles": int(sel.size), "factor_rel_diff": rel,
            "partial_logdet_rel_diff": abs(ld_g - ld_r) / abs(ld_r)}


def run_ours(a, name, nt, rank, world):
    if name == "c5":
        return run_batch(a, nt, rank, world)
    import torch
    import torch.distributed as dist
    from paper_2501_02483_b200 import api
    from paper_2501_02483_b200._lib import check, lib, f64p, i64p

    t0 = time.perf_counter()
    m = build_matrix(name)
    gen_s = time.perf_counter() - t0
    opts = api.FactorOptions(tile_size=nt, executor=a.executor, ordering=a.ordering, occupancy=a.occupancy,
                             **({} if a.lookahead is None else {"lookahead": a.lookahead}))
    t0 = time.perf_counter()
    pat = api._pattern_for(m, opts)
    setup_s = time.perf_counter() - t0
    plan = pat.plan
    info = plan.info()
    F = info["tile_flops"]
    vals_dev = torch.from_numpy(np.ascontiguousarray(pat.permuted_values(m))).cuda()
    offs = pat.offsets()
    storage = plan.new_storage()
    stream = torch.cuda.current_stream()
    sh = stream.cuda_stream

    def step():
        plan.pack(vals_dev, offs, storage, sh)
        plan.factorize_async(storage, 0, sh)

    for _ in range(max(a.warmup, 1)):
        step()
    fail, ld = plan.collect(0, sh)
    if fail >= 0:
        raise RuntimeError(f"factorisation failed at {fail}")
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = Clocks(int(os.environ.get("LOCAL_RANK", "0")))
    clk.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(a.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    clocks = clk.stop()
    ms = e0.elapsed_time(e1) / a.steps
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    fail, ld2 = plan.collect(0, sh)
    if fail >= 0:
        raise RuntimeError(f"timed factorisation failed at {fail}")
    reproducible = bool(ld2 == ld)
    if not reproducible:
        print(f"[bench] timed logdet differs from warm-up: {ld2!r} vs {ld!r}", file=sys.stderr, flush=True)

    # ---- dominant kernel: k_persist alone, CUDA events on its stream
    peak, peak_src = fp64_peak()
    hbm, hbm_src = hbm_peak()
    kms = []
    for _ in range(max(2, min(a.steps, 5))):
        plan.pack(vals_dev, offs, storage, sh)
        k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        k0.record(stream)
        plan.factorize_async(storage, 0, sh)
        k1.record(stream)
        torch.cuda.synchronize()
        kms.append(k0.elapsed_time(k1))
    kernel_ms = float(np.mean(kms))

    # ---- parity at full size: device backward error + oracle prefix factor
    parity = None
    pr = None
    if rank == 0 and world == 1 and not (a.no_parity and a.no_cpu_baseline):
        pr = oracle_sample(name, nt, CPU_SAMPLE_FLOPS_OURS)
        cpu_dt, pr["factor"] = time_sample(pr)
    if rank == 0 and not a.no_parity:
        parity = {}
        if pr is not None:
            parity.update(prefix_parity(pat, storage, pr, nt))
        parity.update(device_backward_error(pat, m, storage, vals_dev, offs, sh))
        parity["tolerances"] = {"backward_error": 1e-12, "factor_rel_diff": 1e-12, "logdet_rel_diff": 1e-10}

    # ---- triangular solves with the factor just computed:
    # device sweep (plan.solve, one persistent launch per direction) for 1 and
    # 8 right-hand sides, bytes = the factor's tiles read once per direction
    solve_info = None
    if not a.no_parity:
        fbytes = storage.numel() * 8
        solve_info = {"factor_bytes": int(fbytes), "hbm_peak_gbs": hbm_peak()[0]}
        for nrhs in (1, 8):
            rdev = torch.ones((nrhs, plan.T * nt), dtype=torch.float64, device="cuda")
            plan.solve(storage, rdev, sh)
            ts = []
            for _ in range(5):
                rdev.fill_(1.0)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                plan.solve(storage, rdev, sh)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            ms_s = float(np.median(ts))
            solve_info[f"nrhs{nrhs}"] = {"ms": ms_s, "gbs": 2 * fbytes / (ms_s * 1e-3) / 1e9,
                                         "frac_hbm": 2 * fbytes / (ms_s * 1e-3) / 1e9 / solve_info["hbm_peak_gbs"]}
            del rdev

    # ---- end to end through the public API (host values, H2D/D2H inside)
    e2e_ms = []
    del_vals = vals_dev
    for i in range(a.e2e_steps + 1):
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        ctx = api.factorize(m, opts)
        ldv = api.logdet(ctx)
        if world > 1:
            buf = torch.tensor([ldv], dtype=torch.float64, device="cuda")
            outl = [torch.empty_like(buf) for _ in range(world)]
            dist.all_gather(outl, buf)
            torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) * 1e3
        if i > 0:
            e2e_ms.append(dt)
        del ctx
    e2e = float(np.mean(e2e_ms))
    if world > 1:
        t = torch.tensor([e2e], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e = float(t.item())

    prof = None
    if not a.no_profile and rank == 0 and name != "c4":
        nc = 7
        pms = np.zeros(nc)
        pcnt = np.zeros(nc, dtype=np.int64)
        pfl = np.zeros(nc)
        plan.pack(del_vals, offs, storage, sh)
        check("tc_plan_profile", lib.tc_plan_profile(plan.h, storage.data_ptr(), sh, nc,
                                                     pms.ctypes.data_as(f64p), pcnt.ctypes.data_as(i64p),
                                                     pfl.ctypes.data_as(f64p)))
        names = ["update_bulk", "update_last", "potrf", "trsm", "combine", "logdet", "update_splitk"]
        prof = {names[i]: {"ms": float(pms[i]), "launches": int(pcnt[i]), "gflop": float(pfl[i] / 1e9)}
                for i in range(nc) if pcnt[i]}
    S, T = plan.S, plan.T
    B = 16.0 * nt * nt * S
    t_roof = max(F / (peak * 1e12), B / (hbm * 1e9))
    useful = _useful_flops(pat)
    value = world * 1000.0 / ms
    kname = {"persistent": "k_persist (persistent dataflow executor)", "graph": "CUDA graph of k_update/k_potrf/k_trsm",
             "direct": "direct k_update/k_potrf/k_trsm launches"}[a.executor]
    per_step = 4 if a.executor == "persistent" else int(info["launches"]) + 3
    line = {"metric": "factorizations/s (FP64 time-to-factor)", "value": value, "unit": "factorizations/s",
            "n_gpus": world, "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": common_config(name, nt, world, a),
            "structure": {"nnz": m.nnz, "tiles_per_side": T, "slots": S, "tile_storage_gb": B / 2 / 1e9,
                          "executor": a.executor,
                          "lookahead": opts.lookahead if opts.lookahead >= 0 else (3 if plan.S >= 20 * plan.T else 4)},
            "time_to_factor_ms": ms, "gflops_tile": F / (ms * 1e-3) / 1e9,
            "gflops_useful": useful / (ms * 1e-3) / 1e9 if useful else None,
            "fp64_roofline": {"time_ms": t_roof * 1e3, "frac": t_roof * 1e3 / ms, "tile_flops": F,
                              "compulsory_bytes": B, "peak_tflops": peak, "peak_source": peak_src,
                              "hbm_gbs": hbm, "hbm_source": hbm_src},
            "roofline": {"bound": "tensor", "kernel": kname, "achieved": F / (kernel_ms * 1e-3) / 1e12,
                         "peak": peak, "unit": "TFLOP/s", "frac": F / (kernel_ms * 1e-3) / 1e12 / peak,
                         "traffic": traffic_of(name, nt)[0], "traffic_source": traffic_of(name, nt)[1],
                         "kernel_ms": kernel_ms, "peak_source": peak_src,
                         "note": "algorithmic tile flops (SYRK = nt^3, GEMM = 2 nt^3, POTRF = nt^3/3, TRSM = nt^3) "
                                 "per launch / CUDA-event launch time; traffic: see profiles/"},
            "gpu_launches": per_step * a.steps, "gpu_launches_per_step": per_step,
            "setup_s": setup_s, "generate_s": gen_s, "pattern_times_s": pat.times,
            "logdet": ld, "bitwise_reproducible": reproducible}
    if parity is not None:
        line["parity"] = parity
    if solve_info is not None:
        line["solve"] = solve_info
    if prof:
        line["profile_direct"] = prof
    line["e2e"] = {"value": world * 1000.0 / e2e, "unit": "factorizations/s",
                   "h2d_bytes_per_step": int(m.nnz * 8), "d2h_bytes_per_step": 16,
                   "ms_per_step": e2e, "path": "api.factorize(SymmetricCsc host values) + logdet"
                   + (" + NCCL all_gather of logdets" if world > 1 else "")}
    line["clocks"] = clocks
    if rank == 0 and world == 1 and not a.no_cpu_baseline and pr is not None:
        frac = pr["flops"] / pr["F_total"]
        line["cpu_baseline"] = {"value": frac / cpu_dt, "unit": "factorizations/s", "cores": 1, "kind": "port",
                                "sample": f"first {pr['columns']} tile columns of one {name} factorisation "
                                          f"({pr['ops']} reference ops, {pr['flops']:.3e} of {pr['F_total']:.3e} "
                                          f"tile flops = {100 * frac:.2f}%) in {cpu_dt:.2f} s; oracle run_ops "
                                          f"(numba + OpenBLAS dgemm, OPENBLAS_NUM_THREADS=1), scaled by flop fraction"}
    del m, vals_dev, del_vals, storage
    if world == 1 and not a.no_batch and name == "c4":
        import gc
        gc.collect()
        api.clear_plan_cache()
        torch.cuda.empty_cache()
        line["batch_c5"] = run_batch(a, DEFAULT_NT["c5"], rank, world, sub=True)
    if rank == 0:
        print(json.dumps(line), flush=True)


def device_backward_error(pat, m, storage, vals_dev, offs, sh):
    """||PAP^T - LL^T||_F / ||A||_F by the device replay of the reference op
    stream (tc_replay_residual, reference _backend_numba.py:136-185) against
    the packed original."""
    from paper_2501_02483_b200 import symbolic
    from paper_2501_02483_b200.backend import impl
    import torch
    op, dst, s1, s2, _ = symbolic.compile_ops(pat.symbolic)
    tpl = pat.plan.new_storage()
    pat.plan.pack(vals_dev, offs, tpl, sh)
    fg = pat.symbolic.factor_grid
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e2 = impl.replay_residual(storage, tpl, op, dst, s1, s2, fg.tile_rows == fg.tile_cols)
    dt = time.perf_counter() - t0
    del tpl
    v = m.values
    d = v[m.col_ptr[:-1]]
    anorm = float(np.sqrt(2.0 * np.dot(v, v) - np.dot(d, d)))
    return {"backward_error": float(np.sqrt(e2)) / anorm, "replay_s": dt}


def _useful_flops(pat):
    """sum_j c_j^2 over the scalar factor's column counts (tile-size
    independent flop figure of survey 8(d))."""
    from paper_2501_02483_b200.ordering import factor_column_counts
    c = factor_column_counts(pat.pm_pattern).astype(np.float64)
    return float(np.sum(c * c))


def main():
    a = parse()
    if os.environ.get("TC_BENCH_TRACEBACK"):  # debugging hangs: dump the Python stack after N s
        import faulthandler
        faulthandler.dump_traceback_later(float(os.environ["TC_BENCH_TRACEBACK"]), exit=True)
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    name = workload_of(a)
    nt = a.tile or DEFAULT_NT[name]
    if a.impl == "reference":
        if rank != 0:
            return
        run_reference(a, name, nt, max(world, a.gpus))
        return
    maybe_spawn(a)
    import torch
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
        dist.init_process_group("nccl")
    if a.measure_peaks:
        if rank == 0:
            measure_peaks()
        return
    try:
        run_ours(a, name, nt, rank, world)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
