#!/usr/bin/env python
"""Benchmark of the B200 frPCA / frPCAt hot path (BASELINE.json metric:
"frPCA seconds to top-k PCs; SpMM HBM GB/s (% of peak) at 1/2/4/8 B200").

One step = one full frpcat / frpca run (randsvd.hpp:224-328) on the config's
synthetic CSR (SURVEY §8d generators, seeded), Omega from PcaConfig::seed = 0.
  value : device time of the run with A (CSR + transposed CSR) resident in HBM
          and U/S/V left in HBM (CUDA events on the library's stream, max over
          ranks), seconds per run (lower is better).
  e2e   : the same run through the C ABI with HOST buffers: pinned host CSR ->
          frpca_dmat_upload (H2D + validation + device transpose + work lists)
          -> frpca_run -> U/S/V copied back to host, per step.
  roofline: the SpMM kernels (K1/K2), algorithmic bytes per launch / measured
          average launch time, against MEASURED_PEAKS.json hbm_gbs.
  cpu_baseline: the CPU oracle (a faithful port of the reference, oracle/)
          on the box's host cores, rank 0 only.

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3]
       python bench.py --impl reference ...   (CPU reference arm)
Multi-GPU (N > 1): launched by torchrun, one rank per GPU; frpcat row-block /
frpca column-block shards with NCCL allreduce inside the library.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

L2_BYTES = 126 * 1024 * 1024
# L2 gather ceiling of this B200: a warp per 1600-byte row from an L2-resident
# table (tools/probe/l2_bw.cu, profiles/r1_l2_probe.txt; 8.8 TB/s from a
# uniform 160 MB table, 16.9 TB/s from 32 MB)
L2_GATHER_PEAK_GBS = 16933.7


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


class Dist:
    """Host-side plumbing for N > 1 (torch.distributed over gloo): barrier,
    broadcast of the NCCL unique id, max over ranks. The data path uses the
    library's own NCCL communicator."""

    def __init__(self, rank, world):
        self.rank, self.world = rank, world
        self.pg = None
        if world > 1:
            import torch.distributed as tdist
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            tdist.init_process_group("gloo", rank=rank, world_size=world)
            self.tdist = tdist

    def barrier(self):
        if self.world > 1:
            self.tdist.barrier()

    def bcast_bytes(self, b: bytes | None) -> bytes:
        if self.world == 1:
            return b
        obj = [b]
        self.tdist.broadcast_object_list(obj, src=0)
        return obj[0]

    def max(self, x: float) -> float:
        if self.world == 1:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.float64)
        self.tdist.all_reduce(t, op=self.tdist.ReduceOp.MAX)
        return float(t.item())

    def sum(self, x: float) -> float:
        if self.world == 1:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.float64)
        self.tdist.all_reduce(t, op=self.tdist.ReduceOp.SUM)
        return float(t.item())

    def close(self):
        if self.world > 1:
            self.tdist.destroy_process_group()


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        sm, smax, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = max(smax, float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


def ncu_traffic(config: str):
    """Per-launch DRAM bytes of the SpMM kernels from the committed ncu capture."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p))
    e = d.get(config, {}).get("spmm")
    return None if e is None else e.get("dram_bytes_per_launch")


# --------------------------------------------------------------------------- arms

def config_dict(cfg, m, n, nnz):
    """The workload, identical in both arms (the driver compares them)."""
    return {"workload": cfg.name, "algorithm": cfg.algorithm, "rows": int(m), "cols": int(n), "nnz": int(nnz),
            "k": cfg.k, "s": cfg.s, "q": cfg.q, "seed": 0, "matrix_seed": cfg.seed}


REF_NOTE = ("oracle/ (C++ restatement of the reference path, bitwise equal for any thread count); the "
            "reference's own kernels are single-threaded (proj/README.md:145-146), so a multi-core run of "
            "the port makes the GPU/CPU ratio conservative")


def cpu_reference_seconds(cfg, A_arrays, threads: int):
    """Times the oracle (CPU port of the reference path) on the config's matrix:
    one full run. Returns (seconds, sample description)."""
    import oracle
    oracle.build()
    oracle.set_threads(threads)
    m, n, rp, ci, va = A_arrays
    A = oracle.Csr.create(m, n, rp, ci, va)
    algo = oracle.FRPCA if cfg.algorithm == "frpca" else oracle.FRPCAT
    t0 = time.perf_counter()
    oracle.pca(A, algo, cfg.k, cfg.s, cfg.q, seed=0)
    dt = time.perf_counter() - t0
    return dt, (f"one full {cfg.name} {cfg.algorithm} run (k={cfg.k}, s={cfg.s}, q={cfg.q}) on the oracle, "
                f"{threads} threads")


def run_reference_arm(args, cfg):
    """The reference's CPU path (the oracle port: the reference itself cannot
    be built, Eigen is absent) on the same matrix and config.
    Each step is one full run; the steps stop early when the next one would
    exceed --ref-budget seconds (at least one step always runs), and the line
    says how many ran."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from paper_1810_06825_b200 import synth
    threads = os.cpu_count() or 1
    A = synth.generate(cfg.name)
    m, n, rp = A[0], A[1], A[2]
    times = []
    t_start = time.perf_counter()
    warm_done = 0
    for it in range(args.warmup + args.steps):
        elapsed = time.perf_counter() - t_start
        est = statistics.mean(times) if times else 0.0
        if times and elapsed + est > args.ref_budget:
            break
        dt, sample = cpu_reference_seconds(cfg, A, threads)
        if it < args.warmup and elapsed + 2 * dt < args.ref_budget / 2:
            warm_done += 1
            continue
        times.append(dt)
    v = statistics.mean(times)
    line = {
        "impl": "reference", "metric": "frPCA seconds to top-k PCs", "value": round(v, 6), "unit": "s",
        "n_gpus": world, "steps": len(times), "warmup": warm_done, "steps_requested": args.steps,
        "warmup_requested": args.warmup, "ms_per_step": round(v * 1e3, 3),
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generator, SURVEY §8d)",
        "config": config_dict(cfg, m, n, rp[-1]),
        "cpu_baseline": {"value": round(v, 6), "unit": "s", "cores": threads, "kind": "port",
                         "sample": sample, "note": REF_NOTE},
        "e2e": {"value": round(v, 6), "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "statistic": "mean of steps",
    }
    if len(times) < args.steps:
        line["steps_note"] = (f"{len(times)} of {args.steps} steps: each is a full {cfg.name} run; the arm stops "
                              f"before exceeding {args.ref_budget:.0f} s")
    print(json.dumps(line), flush=True)
    return 0


def run_gpu_arm(args, cfg):
    import ctypes as C
    import paper_1810_06825_b200 as fb
    from paper_1810_06825_b200 import _lib, shard, synth

    rank, world, local = dist_env()
    dist = Dist(rank, world)
    L = _lib.load()
    nccl_id = fb.Context.nccl_unique_id() if (world > 1 and rank == 0) else None
    nccl_id = dist.bcast_bytes(nccl_id) if world > 1 else None
    ctx = fb.Context(local, rank, world, nccl_id)

    # ---- inputs (pinned host memory; generated once, outside every timed region)
    pinned = []

    def alloc(n, dt):
        nbytes = max(1, int(n) * np.dtype(dt).itemsize)
        p = C.c_void_p()
        _lib.check(L.frpca_host_alloc(nbytes, C.byref(p)))
        pinned.append(p)
        return np.frombuffer((C.c_char * nbytes).from_address(p.value), dtype=dt, count=int(n))

    t0 = time.perf_counter()
    m, n, rp, ci, va = synth.generate(cfg.name, alloc=alloc)
    log(f"[rank {rank}] generated {cfg.name}: {m}x{n}, nnz={int(rp[-1])} in {time.perf_counter() - t0:.1f}s")
    algo = _lib.ALGO_FRPCA if cfg.algorithm == "frpca" else _lib.ALGO_FRPCAT
    if world == 1:
        shard_ = dict(grows=m, gcols=n, col_shard=0, off=0, rows=m, cols=n, rp=rp, ci=ci, va=va)
    elif algo == _lib.ALGO_FRPCAT:
        r0, r1, lrp, lci, lva = shard.shard_rows(rp, ci, va, world, rank)
        shard_ = dict(grows=m, gcols=n, col_shard=0, off=r0, rows=r1 - r0, cols=n, rp=lrp, ci=lci, va=lva)
    else:
        c0, c1, lrp, lci, lva = shard.shard_cols(rp, ci, va, n, world, rank)
        shard_ = dict(grows=m, gcols=n, col_shard=1, off=c0, rows=m, cols=c1 - c0, rp=lrp, ci=lci, va=lva)
    nnz_loc = int(shard_["rp"][-1])

    def upload():
        h = C.c_void_p()
        _lib.check(L.frpca_dmat_upload_shard(
            ctx._h, shard_["grows"], shard_["gcols"], shard_["col_shard"], shard_["off"], shard_["rows"],
            shard_["cols"], nnz_loc, shard_["rp"].ctypes.data, shard_["ci"].ctypes.data,
            shard_["va"].ctypes.data, C.byref(h)))
        return h

    k, l = cfg.k, cfg.k + cfg.s
    m_loc = shard_["rows"]
    n_loc = shard_["cols"]
    import torch  # device buffers for the device-resident outputs (plumbing only)
    dU = torch.empty(max(1, m_loc * k), dtype=torch.float64, device=f"cuda:{local}")
    dS = torch.empty(k, dtype=torch.float64, device=f"cuda:{local}")
    dV = torch.empty(max(1, n_loc * k), dtype=torch.float64, device=f"cuda:{local}")
    flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device=f"cuda:{local}")

    cfg_dev = fb.PcaConfig(k=cfg.k, oversample=cfg.s, passes=cfg.q, seed=0,
                           host_omega=args.host_omega).to_c(device_io=True)
    cfg_host = fb.PcaConfig(k=cfg.k, oversample=cfg.s, passes=cfg.q, seed=0,
                            host_omega=args.host_omega).to_c(device_io=False)
    st = _lib.FrpcaStats()

    def run_device(hmat):
        _lib.check(L.frpca_run(ctx._h, hmat, algo, C.byref(cfg_dev), None, 0, 0,
                               C.c_void_p(dU.data_ptr()), C.c_void_p(dS.data_ptr()),
                               C.c_void_p(dV.data_ptr()), None, C.byref(st), None))

    # ---- value: device-resident A, device outputs
    hmat = upload()
    for _ in range(args.warmup):
        run_device(hmat)
    ctx.sync()
    torch.cuda.synchronize(local)
    clocks = ClockSampler(local)
    clocks.start()
    ctx.profile(True)
    ctx.profile_reset()
    lc0 = C.c_uint64()
    _lib.check(L.frpca_launch_count(C.byref(lc0)))
    step_ms = []
    for _ in range(args.steps):
        flush.zero_()                      # L2 flush between timed iterations (outside events)
        torch.cuda.synchronize(local)
        dist.barrier()
        _lib.check(L.frpca_timer_begin(ctx._h))
        run_device(hmat)
        ms = C.c_double()
        _lib.check(L.frpca_timer_end(ctx._h, C.byref(ms)))
        dist.barrier()
        step_ms.append(dist.max(ms.value))
    lc1 = C.c_uint64()
    _lib.check(L.frpca_launch_count(C.byref(lc1)))
    prof = ctx.profile_report()
    ctx.profile(False)
    clk = clocks.stop()
    passes = st.passes_over_matrix
    L.frpca_dmat_destroy(hmat)

    # ---- e2e: host CSR -> upload -> run -> host U/S/V, per step
    hU = alloc(m_loc * k, np.float64)
    hS = alloc(k, np.float64)
    hV = alloc(n_loc * k, np.float64)

    def run_e2e():
        if world == 1:
            # the one-shot host-CSR call (frpca_run_csr): upload, run, outputs
            # back to pinned host memory; the sketch overlaps the upload
            _lib.check(L.frpca_run_csr(ctx._h, shard_["rows"], shard_["cols"], nnz_loc,
                                       shard_["rp"].ctypes.data, shard_["ci"].ctypes.data,
                                       shard_["va"].ctypes.data, algo, C.byref(cfg_host), None, 0, 0,
                                       C.c_void_p(hU.ctypes.data), C.c_void_p(hS.ctypes.data),
                                       C.c_void_p(hV.ctypes.data), None, None, None))
            return
        h = upload()
        try:
            _lib.check(L.frpca_run(ctx._h, h, algo, C.byref(cfg_host), None, 0, 0,
                                   C.c_void_p(hU.ctypes.data), C.c_void_p(hS.ctypes.data),
                                   C.c_void_p(hV.ctypes.data), None, None, None))
        finally:
            L.frpca_dmat_destroy(h)

    for _ in range(max(1, args.warmup // 2)):
        run_e2e()
    e2e_ms = []
    for _ in range(args.e2e_steps or args.steps):
        flush.zero_()
        torch.cuda.synchronize(local)
        dist.barrier()
        _lib.check(L.frpca_timer_begin(ctx._h))
        run_e2e()
        ms = C.c_double()
        _lib.check(L.frpca_timer_end(ctx._h, C.byref(ms)))
        dist.barrier()
        e2e_ms.append(dist.max(ms.value))
    h2d = (shard_["rp"].nbytes + shard_["ci"].nbytes + shard_["va"].nbytes)
    d2h = 8 * (m_loc * k + k + n_loc * k)

    # ---- roofline of the SpMM kernels (algorithmic bytes / measured launch time)
    hbm_peak, peak_kind = measured_peaks()
    sp = [v for kname, v in prof.items() if kname in ("spmm_AX", "spmm_AtY")]  # sub-tags are nested
    sp_bytes = sum(v["bytes"] for v in sp)
    sp_ms = sum(v["ms"] for v in sp)
    sp_launches = sum(v["launches"] for v in sp)
    achieved = (sp_bytes / (sp_ms / 1e3)) / 1e9 if sp_ms > 0 else 0.0
    achieved = dist.sum(achieved) if world > 1 else achieved
    # the binding unit at l = 200: every nonzero gathers one l-double row of the
    # dense operand through L2 (nnz * l * 8 bytes per launch)
    l_cols = cfg.k + cfg.s
    l2_gathers = {}
    for kname in ("spmm_AX", "spmm_AtY"):
        v = prof.get(kname)
        if v and v["ms"] > 0:
            l2_gathers[kname] = round(nnz_loc * l_cols * 8.0 * v["launches"] / (v["ms"] / 1e3) / 1e9, 1)
    l2_ms = sum(prof[kn]["ms"] for kn in l2_gathers)
    l2_launch = sum(prof[kn]["launches"] for kn in l2_gathers)
    l2_achieved = nnz_loc * l_cols * 8.0 * l2_launch / (l2_ms / 1e3) / 1e9 if l2_ms > 0 else 0.0
    l2_achieved = dist.sum(l2_achieved) if world > 1 else l2_achieved
    total_ms = sum(v["ms"] for kname, v in prof.items() if kname not in ("lu_basis",)) or 1.0
    kernels = {kname: {"launches": v["launches"] // max(1, args.steps) if v["launches"] >= args.steps else v["launches"],
                       "ms_per_step": round(v["ms"] / args.steps, 4),
                       "GBps": round(v["bytes"] / (v["ms"] / 1e3) / 1e9, 1) if v["ms"] > 0 else None,
                       "TFLOPps": round(v["flops"] / (v["ms"] / 1e3) / 1e12, 2) if v["ms"] > 0 else None}
               for kname, v in sorted(prof.items())}

    value_s = statistics.mean(step_ms) / 1e3
    # median over the e2e steps: host-side hiccups (page/PCIe, thread wake-up)
    # occasionally stretch one step 2-3x (tools/e2e_probe.py); the mean is
    # reported next to it
    e2e_s = statistics.median(e2e_ms) / 1e3
    e2e_mean_s = statistics.mean(e2e_ms) / 1e3
    line = {
        "metric": "frPCA seconds to top-k PCs", "value": round(value_s, 6), "unit": "s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(value_s * 1e3, 3), "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generator, SURVEY §8d)",
        "config": config_dict(cfg, m, n, rp[-1]),
        "parallelism": f"{'row' if algo == _lib.ALGO_FRPCAT else 'col'}-block x{world}",
        "l2": "flushed between timed steps (256 MB write)",
        "omega": "host libstdc++" if args.host_omega else "device (bit-compatible)",
        "roofline": {"bound": "hbm", "kernel": "spmm (K1 A*X + K2 A^T*Y)",
                     "achieved": round(achieved, 1), "peak": hbm_peak, "unit": "GB/s",
                     "frac": round(achieved / hbm_peak, 4), "peak_kind": peak_kind,
                     "traffic": ncu_traffic(cfg.name),
                     "launches_per_step": sp_launches // max(1, args.steps),
                     "share_of_step": round(sp_ms / max(1e-9, sum(step_ms)), 4)},
        "roofline_l2": {"bound": "l2", "kernel": "spmm row gathers (nnz * l * 8 B per launch)",
                        "achieved": round(l2_achieved, 1), "peak": L2_GATHER_PEAK_GBS, "unit": "GB/s",
                        "frac": round(l2_achieved / L2_GATHER_PEAK_GBS, 4),
                        "peak_kind": "measured L2-resident row gather (profiles/r1_l2_probe.txt)",
                        "per_kernel": l2_gathers},
        "e2e": {"value": round(e2e_s, 6), "unit": "s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h), "statistic": "median of steps",
                "mean": round(e2e_mean_s, 6), "steps_ms": [round(x, 2) for x in e2e_ms],
                "call": "frpca_run_csr" if world == 1 else "frpca_dmat_upload_shard + frpca_run"},
        "gpu_launches": int((lc1.value - lc0.value) // max(1, args.steps)),
        "passes_over_matrix": int(passes),
        "kernels": kernels,
    }
    if clk:
        line["clocks"] = clk
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        A_arrays = (m, n, rp, ci, va)
        threads = os.cpu_count() or 1
        cpu_s, sample = cpu_reference_seconds(cfg, A_arrays, threads)
        line["cpu_baseline"] = {"value": round(cpu_s, 3), "unit": "s", "cores": threads,
                                "kind": "port", "sample": sample, "note": REF_NOTE}
    if rank == 0:
        print(json.dumps(line), flush=True)
    for p in pinned:
        L.frpca_host_free(p)
    ctx.close()
    dist.close()
    return 0


def self_launch(n: int) -> int:
    """`bench.py --gpus N` without a launcher: start N ranks with torchrun on
    this node (127.0.0.1 rendezvous) and pass the same arguments through."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--e2e-steps", type=int, default=0)
    # C3 (the AMiner shape) is the largest config frpcat serves
    # on one GPU: the north_star's "largest config"; C4 is the frpca one
    ap.add_argument("--config", default="C3", choices=["C0", "C1", "C2", "C3", "C4"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--host-omega", action="store_true")
    ap.add_argument("--ref-budget", type=float, default=900.0,
                    help="seconds the reference arm may spend on its steps")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(args.gpus)
    from paper_1810_06825_b200.synth import CONFIGS
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference_arm(args, cfg)
    return run_gpu_arm(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
