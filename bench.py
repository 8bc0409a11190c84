#!/usr/bin/env python
"""Benchmark: randomized PSD projections/s at BASELINE config 3
(n=32768, k=256, p=16, q=1, fp64) on B200, with the tensor-core roofline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one projection (``ran_proj``, Alg. 2) of a seeded C3 matrix that is
already resident in HBM; the K timed steps cycle through a pool of distinct
matrices (8.6 GB each ≫ 126 MB L2, so no L2 flush is needed).  Ω is drawn on
the device each step (Philox).  The FP64 n×n sketch products run by default on
the INT8 tensor cores as an exact FP64 emulation (Ozaki scheme II, csrc/ozaki.cu;
same ≤1e-10 parity as the DMMA path); ``--fp64-engine dmma`` keeps them on the
FP64 DMMA kernel.

Multi-GPU: ``--gpus N`` without a torchrun environment relaunches itself under
``torch.distributed.run`` with N ranks (one per GPU).  The C3 projections are
independent: one replica per rank, value = all ranks' projections /
max-over-ranks device time (``scaling: weak``).  The same line carries
``c4_sharded``: BASELINE config 4 (n=131072, k=512, p=32, q=2) row-sharded over
all N ranks (NCCL all-gather / all-reduce), so a scaling run measures the
sharded path at every N.

``--impl reference`` times the UNMODIFIED reference ``psdcone.ran_proj``
(oracle/_ref, installed offline by oracle/make_ref.sh) on this box's host
cores at the full C3 size, for as many of the K steps as fit a time budget
(the count actually timed is reported as ``steps``); the oracle port
(oracle/psd_oracle.py) stands in only if the reference package is absent.
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

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "rand-PSD projections/s at n=32768,k=256 fp64; % of FP64 tensor-core roofline"
UNIT = "projections/s"
CPU_SAMPLE_N = 8192

# BASELINE.json configs; c3 is the headline (metric) workload.
CONFIGS = {
    "c1": dict(n=1000, k=40, p=10, q=2, desc="config 1: Haar basis, 30 geometric + uniform[-1,0] spectrum"),
    "c2": dict(n=8192, k=128, p=16, q=2, desc="config 2: Wigner (G+Gᵀ)/(2√n)"),
    "c3": dict(n=32768, k=256, p=16, q=1, desc="config 3: U diag(s)Uᵀ − W diag(t)Wᵀ + 1e-3 E"),
    "c4": dict(n=131072, k=512, p=32, q=2, desc="config 4: config-3 form, row-sharded over ranks"),
    "c5": dict(n=4096, k=64, p=10, q=1, m=20000, desc="config 5: SDLS dual ascent, sparse constraints"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=16)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c3")
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--k", type=int, default=None)
    ap.add_argument("--p", type=int, default=None)
    ap.add_argument("--q", type=int, default=None)
    ap.add_argument("--pool", type=int, default=4, help="distinct X matrices cycled per rank")
    ap.add_argument("--e2e-steps", type=int, default=16)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-fp32", action="store_true", help="skip the config-3 FP32 (3xTF32) leg")
    ap.add_argument("--no-scaled", action="store_true", help="skip the scaled (Alg. 3 + Alg. 5) leg")
    ap.add_argument("--no-c4", action="store_true", help="skip the config-4 row-sharded leg")
    ap.add_argument("--no-prefetch", action="store_true",
                    help="do not pipeline consecutive projections (psd_plan_prefetch)")
    ap.add_argument("--no-peaks", action="store_true",
                    help="skip the in-run cuBLAS peak measurement (profiling runs; roofline then uses "
                         "MEASURED_PEAKS.json)")
    ap.add_argument("--c4-steps", type=int, default=3)
    ap.add_argument("--ref-budget-s", type=float, default=float(os.environ.get("PSD_REF_BUDGET_S", 300)),
                    help="reference arm: wall-clock budget for the timed full-size projections")
    ap.add_argument("--fp64-engine", choices=["auto", "int8", "dmma"], default="auto",
                    help="FP64 n×n products: exact emulation on the INT8 tensor cores (auto: n >= 3072), or DMMA")
    a = ap.parse_args()
    cfg = CONFIGS[a.config]
    for key in ("n", "k", "p", "q"):
        if getattr(a, key) is None:
            setattr(a, key, cfg[key])
    return a


def workload_config(a, n_gpus):
    return {
        "workload": f"BASELINE {CONFIGS[a.config]['desc']}: ran_proj (Alg. 2) n={a.n}, k={a.k}, "
                    f"p={a.p}, q={a.q}, fp64, {a.steps} sequential projections per rank",
        "n": a.n, "k": a.k, "p": a.p, "q": a.q, "width": a.k + a.p,
        "x_pool": a.pool,
        "l2": "inputs larger than L2 (each X is 8·n² bytes ≫ 126 MB)",
        "omega": "device Philox N(0,1) per projection",
        "parallelism": f"replicas x{n_gpus}" if n_gpus > 1 else "single GPU",
        "pipelining": ("none" if getattr(a, "no_prefetch", False) or a.config == "c1" else
                       "ran_proj(..., prefetch=next X): projection i+1's symmetry pass and INT8 "
                       "residue planes run on a low-priority side stream under projection i's "
                       "CholeskyQR / eigensolver; the first timed step prepares its own X and the "
                       "last one prefetches nothing, so the K steps do exactly K projections' work"),
    }


# --------------------------------------------------------------------- CPU ---

def cpu_cores():
    try:
        from threadpoolctl import threadpool_info
        nt = max((d.get("num_threads") or 0) for d in threadpool_info() if d.get("user_api") == "blas")
        return int(nt) if nt else os.cpu_count()
    except Exception:
        return os.cpu_count()


def _reference_module():
    """The unmodified reference package (oracle/_ref or /root/reference), or None."""
    try:
        from oracle import refpkg
        return refpkg.import_psdcone()
    except Exception:
        return None


def _host_matrix(config, n, seed):
    from oracle import psd_oracle as orc
    return {"c1": lambda: orc.c1_matrix(seed=seed, n=n), "c2": lambda: orc.wigner(n, seed=seed),
            "c3": lambda: orc.c3_matrix(n, seed=seed)}[config]()


def _cpu_project(ref, x, a, seed):
    """One CPU projection: the real psdcone.ran_proj (its own validation, Ω draw,
    QR, eigh and reconstruction — projection.py:92-119) or the oracle port."""
    import numpy as np
    if ref is not None:
        return ref.ran_proj(x, ref.RangeParams(k=a.k, l=a.p, q=a.q), np.random.default_rng(seed))
    from oracle import psd_oracle as orc
    return orc.ran_proj(x, a.k, a.p, a.q, rng=np.random.default_rng(seed))


def cpu_sample(a, ns=CPU_SAMPLE_N):
    """Bounded CPU sample for the ``cpu_baseline`` key of our line: one projection
    at n=ns (C3's k, p, q) by the reference (or the port), scaled to the metric's
    unit by (ns/n)² (every stage of the path is O(n²) at fixed width)."""
    ref = _reference_module()
    ns = min(ns, a.n)
    x = _host_matrix(a.config, ns, 11)
    t0 = time.perf_counter()
    _cpu_project(ref, x, a, 100)
    sec = time.perf_counter() - t0
    return (ns / a.n) ** 2 / sec, sec, ns, ("reference" if ref is not None else "port")


def run_reference(a):
    """The reference arm: psdcone.ran_proj on this box's host cores at the FULL
    workload size (n = a.n), timed with time.perf_counter around the public call.
    Warm-up runs at n=2048 (BLAS thread pool, page cache); then full-size
    projections until ``--steps`` are done or the next one would overrun
    ``--ref-budget-s``; ``steps`` reports how many were timed."""
    rank = int(os.environ.get("RANK", "0"))
    n_gpus = int(os.environ.get("WORLD_SIZE", str(a.gpus)))
    if rank != 0:
        return
    ref = _reference_module()
    kind = "reference" if ref is not None else "port"
    xw = _host_matrix(a.config, min(2048, a.n), 3)
    for i in range(max(a.warmup, 0)):
        _cpu_project(ref, xw, a, 200 + i)
    del xw
    t0 = time.perf_counter()
    x = _host_matrix(a.config, a.n, 11)
    gen_s = time.perf_counter() - t0
    secs = []
    budget_start = time.perf_counter()
    for i in range(a.steps):
        if secs and (time.perf_counter() - budget_start) + max(secs) > a.ref_budget_s:
            break
        t0 = time.perf_counter()
        rep = _cpu_project(ref, x, a, 1000 + i)
        secs.append(time.perf_counter() - t0)
    value = len(secs) / sum(secs)
    cores = cpu_cores()
    who = ("psdcone.ran_proj (the unmodified reference, oracle/_ref)" if ref is not None else
           "the oracle port of psdcone.ran_proj (reference package absent)")
    sample = (f"{who}, numpy/OpenBLAS with {cores} threads, on a {a.config} matrix at the full n={a.n} "
              f"(k={a.k}, p={a.p}, q={a.q}); {len(secs)} of {a.steps} requested projections timed "
              f"(budget {a.ref_budget_s:.0f} s), {min(secs):.1f}-{max(secs):.1f} s each; X generated "
              f"on the host in {gen_s:.1f} s (untimed)")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": n_gpus,
        "steps": len(secs), "steps_requested": a.steps, "warmup": a.warmup,
        "ms_per_step": 1000.0 * sum(secs) / len(secs),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded C3 matrix, host numpy)",
        "config": workload_config(a, 1),
        "effective_rank": int(rep.effective_rank),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ clocks ---

class ClockSampler:
    """SM clocks, power and clock-event (throttle) reasons sampled during the
    timed region — in-process NVML polling every 20 ms (no child process: forking
    a process that maps tens of GB of pinned memory stalls the timed steps);
    nvidia-smi only if NVML is unavailable."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []
        self.samples = []
        self.nvml = None
        self.stop_flag = threading.Event()

    def _handle(self, nv):
        count = nv.nvmlDeviceGetCount()
        if count == 1:
            return nv.nvmlDeviceGetHandleByIndex(0)
        try:   # match the CUDA device to its NVML handle by UUID
            import torch
            want = str(torch.cuda.get_device_properties(self.index).uuid).lower()
            for i in range(count):
                h = nv.nvmlDeviceGetHandleByIndex(i)
                u = nv.nvmlDeviceGetUUID(h)
                u = (u.decode() if isinstance(u, bytes) else u).lower()
                if want in u:
                    return h
        except Exception:
            pass
        return nv.nvmlDeviceGetHandleByIndex(self.index)

    def start(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.h = self._handle(nv)
            self.nvml = nv
            self.bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                         "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                         "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                         "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
            self.smax = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
            return
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _poll(self):
        nv = self.nvml
        while not self.stop_flag.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                pw = nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                util = nv.nvmlDeviceGetUtilizationRates(self.h).gpu
                self.samples.append((sm, pw, rs, util))
            except Exception:
                pass
            self.stop_flag.wait(0.02)

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self):
        if self.nvml is not None:
            self.stop_flag.set()
            self.thread.join(timeout=5)
            busy = [s for s in self.samples if s[3] > 0] or self.samples
            sm = [s[0] for s in busy]
            reasons = sorted({nm for s in busy for nm, bit in self.bits.items() if s[2] & bit})
            return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.smax,
                    "power_w_max": max(s[1] for s in busy) if busy else None,
                    "samples": len(sm), "source": "NVML, 20 ms polling", "reasons": reasons}
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons, power = [], [], set(), []
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
                power.append(float(parts[2]))
            except ValueError:
                continue
            for nm, val in zip(self.NAMES, parts[4:8]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "power_w_max": max(power) if power else None,
                "samples": len(sm), "source": "nvidia-smi -lms 200", "reasons": sorted(reasons)}


# ------------------------------------------------------------------- ours ---

def _gemm_rate(torch, fn, flops, sustained_s=1.5):
    """(burst, sustained) rate of ``fn`` in TFLOP/s (or TOP/s): best single launch of 5
    (CUDA events), then back-to-back launches for ``sustained_s`` seconds."""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    reps = max(4, int(sustained_s * 1000.0 / best))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return flops / best / 1e9, flops * reps / e0.elapsed_time(e1) / 1e9


def measure_peaks(torch, dev):
    """Tensor-core denominators measured in this run with cuBLAS at 8192³ (the
    MEASURED_PEAKS.json file carries HBM and bf16 only): FP64 (DGEMM), INT8
    (torch._int_mm → cuBLASLt IMMA) and TF32 (fp32 matmul with TF32 allowed).
    Each as burst (best single launch) and sustained (back to back ≈1.5 s, the
    clock a kernel inside a long step runs at)."""
    n = 8192
    flops = 2.0 * n ** 3
    out = {"how": "cuBLAS 8192^3 in this process: burst = best of 5 launches, sustained = "
                  "back-to-back launches for ~1.5 s (CUDA events)"}
    a = torch.randn(n, n, dtype=torch.float64, device=dev)
    b = torch.randn(n, n, dtype=torch.float64, device=dev)
    out["fp64_tflops"], out["fp64_tflops_sustained"] = _gemm_rate(torch, lambda: a @ b, flops, 0.5)
    del a, b
    try:
        a8 = torch.randint(-128, 127, (n, n), dtype=torch.int8, device=dev)
        b8 = torch.randint(-128, 127, (n, n), dtype=torch.int8, device=dev)
        out["int8_tops"], out["int8_tops_sustained"] = _gemm_rate(torch, lambda: torch._int_mm(a8, b8), flops)
        del a8, b8
    except Exception as exc:  # pragma: no cover - cuBLASLt without IMMA
        out["int8_error"] = str(exc)[:200]
    prev = torch.backends.cuda.matmul.allow_tf32
    try:
        torch.backends.cuda.matmul.allow_tf32 = True
        a32 = torch.randn(n, n, dtype=torch.float32, device=dev)
        b32 = torch.randn(n, n, dtype=torch.float32, device=dev)
        out["tf32_tflops"], out["tf32_tflops_sustained"] = _gemm_rate(torch, lambda: a32 @ b32, flops)
        del a32, b32
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    torch.cuda.empty_cache()
    return out


def measured_peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except Exception:
        return {}


def int8_roofline(n, w, i8_ms, i8_cnt, traffic, peaks):
    """Roofline of i8_gemm2_kernel (the 16 residue products of one emulated FP64
    sketch product), bound by the INT8 tensor pipe: ``achieved`` = algorithmic int8
    ops per launch (16 · 2n²w) over its average CUDA-event time in the timed
    region; ``peak`` = cuBLASLt INT8 8192³ best single launch (burst) measured in
    this run (the sustained figure is reported beside it).  Fallback: 2 ×
    MEASURED_PEAKS bf16 sustained.  The HBM view is kept beside it."""
    L = 16
    ldk = (n + 127) // 128 * 128
    wpad = (w + 15) // 16 * 16
    algo_bytes = L * n * ldk + L * wpad * ldk + L * n * wpad   # A planes + panel planes + outputs
    pk = measured_peaks()
    hbm = pk.get("hbm_gbs") or 7700.0
    gbs = algo_bytes / (i8_ms / 1000.0) / 1e9
    int8_ops = 2.0 * L * n * n * w
    tops = int8_ops / (i8_ms / 1000.0) / 1e12
    if peaks.get("int8_tops"):
        # burst, not sustained: back-to-back cuBLAS INT8 GEMMs hold the GPU at its power
        # cap and clock lower than this kernel does inside the projection step (where it
        # alternates with HBM-bound kernels), so the sustained figure would put frac > 1
        peak, src = peaks["int8_tops"], ("cuBLASLt INT8 (torch._int_mm) 8192^3 burst, measured in "
                                         "this run (nominal dense INT8: 4500 TOP/s)")
    else:
        peak = 2.0 * (pk.get("bf16_tflops_sustained") or pk.get("bf16_tflops") or 1125.0)
        src = "2 x MEASURED_PEAKS.json bf16_tflops_sustained (no in-run INT8 measurement)"
    return {
        "bound": "tensor", "achieved": tops, "peak": peak, "unit": "TFLOP/s", "frac": tops / peak,
        "traffic": traffic.get("bytes_per_launch") if traffic else None,
        "algorithmic_ops_per_launch": int8_ops,
        "kernel": f"i8_gemm2_kernel<tcgen05.mma.cta_group::2.kind::i8, TMEM, TMA> — the 16 residue "
                  f"products of X·P mod m_l for one FP64 sketch product; {int8_ops / 1e15:.2f} int8 POP "
                  f"algorithmic per launch, {i8_ms:.3f} ms avg over {i8_cnt} launches (CUDA events "
                  f"on the launching stream, timed region); unit: int8 TOP/s",
        "peak_source": src,
        "peak_sustained": peaks.get("int8_tops_sustained"),
        "frac_of_nominal": tops / 4500.0,
        "hbm_view": {"achieved_gbs": gbs, "peak_gbs": hbm, "frac": gbs / hbm,
                     "algorithmic_bytes_per_launch": algo_bytes},
        "traffic_source": traffic.get("source") if traffic else None,
    }


def load_traffic(name="gemm_traffic.json"):
    path = os.path.join(REPO, "profiles", name)  # from the committed ncu --set full capture
    try:
        with open(path) as fh:
            return json.load(fh)
    except Exception:
        return None


def _dist_setup(torch, dist):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    if world > 1 and not dist.is_initialized():
        dist.init_process_group("nccl", device_id=dev)
    return world, rank, local, dev


def _max_over_ranks(torch, dist, world, ms, dev):
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return ms


def run_ours(a):
    import torch
    import torch.distributed as dist

    import paper_2410_19208_b200 as psd
    from paper_2410_19208_b200 import workloads

    world, rank, local, dev = _dist_setup(torch, dist)
    n, params = a.n, psd.RangeParams(k=a.k, l=a.p, q=a.q)
    psd.set_fp64_engine(a.fp64_engine)

    peaks = measure_peaks(torch, dev) if rank == 0 and not a.no_peaks else {}
    peak = peaks.get("fp64_tflops")
    nominal = 148 * 128 * 1.965  # GFLOP/s: 148 SMs × 64 DMMA FMA/clk × 2 × 1965 MHz

    gen = {"c1": lambda sd: workloads.c1_device(n, seed=sd, device=dev),
           "c2": lambda sd: workloads.wigner_device(n, seed=sd, device=dev),
           "c3": lambda sd: workloads.c3_device(n, seed=sd, device=dev)}[a.config]
    pool = [gen(1000 * rank + i) for i in range(a.pool)]
    # inputs smaller than L2 (config 1: 8 MB) → flush L2 between steps with a 256 MB write
    flush = torch.empty(32 << 20, dtype=torch.float64, device=dev) if 8 * n * n < (256 << 20) else None
    rng = psd.DeviceRng(seed=4242 + rank)
    plan = psd._native.get_plan(n, params.width, dev)

    out64 = torch.empty((n, n), dtype=torch.float64, device=dev)   # no allocation in the timed loop
    # pipelined batch: each call names the next X (none across the warm-up/timed boundary
    # and after the last timed step, so the timed region holds exactly its own work)
    nxt = (lambda i, last: None if a.no_prefetch or i == last else pool[(i + 1) % a.pool])
    nwarm = max(a.warmup, 3 if a.warmup >= 3 else a.warmup)
    for i in range(nwarm):
        psd.ran_proj(pool[i % a.pool], params, rng, out=out64, prefetch=nxt(i, nwarm - 1))
    torch.cuda.synchronize(dev)
    plan.profile(enable=True, reset=True)
    clocks = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clocks.start()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    launches = 0
    ranks = []
    engine = 0
    marks = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps + 1)]
    e0.record()
    for i in range(a.steps):
        marks[i].record()
        if flush is not None:
            flush.zero_()
        rep = psd.ran_proj(pool[i % a.pool], params, rng, out=out64, prefetch=nxt(i, a.steps - 1))
        launches += rep.device_info["gpu_launches"]
        ranks.append(rep.effective_rank)
        engine = rep.device_info["sketch_engine"]
    marks[a.steps].record()
    e1.record()
    torch.cuda.synchronize(dev)
    per_step = sorted(marks[i].elapsed_time(marks[i + 1]) for i in range(a.steps))
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    ms = _max_over_ranks(torch, dist, world, e0.elapsed_time(e1), dev)
    prof = plan.profile(enable=False, reset=True)
    value = world * a.steps / (ms / 1000.0)

    # roofline of the dominant kernel.  DMMA engine: the op(X)·P FP64 GEMM (2n²w flops
    # per launch).  INT8 engine: the residue GEMM i8_gemm2_kernel (16 · 2n²w int8 ops).
    g_ms, g_cnt = prof["sketch_gemm"]
    gemm_ms = g_ms / max(g_cnt, 1)
    gemm_tf = 2.0 * n * n * params.width / (gemm_ms / 1000.0) / 1e12
    i8_ms, i8_cnt = prof.get("int8_gemm", (0.0, 0))
    r_plus = statistics.median(ranks) if ranks else 0
    flops = psd.flops(n, params, r_plus)
    traffic = load_traffic("oz_traffic.json" if engine == 1 else "gemm_traffic.json")
    stages = {k: round(v[0] / a.steps, 3) for k, v in prof.items() if v[1]}

    # the same K steps with no prefetch hints (every projection validates and prepares its
    # own X on the caller's stream): reported beside the pipelined headline value
    unpipelined = None
    if a.config != "c1" and not a.no_prefetch:
        for i in range(min(nwarm, 2)):
            psd.ran_proj(pool[i % a.pool], params, rng, out=out64)
        torch.cuda.synchronize(dev)
        u0 = torch.cuda.Event(enable_timing=True)
        u1 = torch.cuda.Event(enable_timing=True)
        u0.record()
        for i in range(a.steps):
            psd.ran_proj(pool[i % a.pool], params, rng, out=out64)
        u1.record()
        torch.cuda.synchronize(dev)
        ums = _max_over_ranks(torch, dist, world, u0.elapsed_time(u1), dev)
        unpipelined = {"value": world * a.steps / (ums / 1000.0), "unit": UNIT, "ms_per_step": ums / a.steps,
                       "steps": a.steps, "note": "same pool and steps, ran_proj without prefetch= hints"}

    fp32 = None
    if a.config == "c3" and not a.no_fp32:
        fp32 = run_fp32_leg(a, torch, psd, pool, params, rng, dev, world, peaks)
    scaled = None
    if a.config == "c3" and not a.no_scaled:
        scaled = run_scaled_leg(a, torch, psd, pool, params, dev, world, out64)

    e2e = None
    if rank == 0 and not a.no_e2e:
        e2e = run_e2e(a, torch, psd, pool[0], params, dev)
    del pool, out64
    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        v, sec, ns, kind = cpu_sample(a)
        cpu = {"value": v, "unit": UNIT, "cores": cpu_cores(), "kind": kind,
               "sample": f"1 projection of a {a.config} matrix at n={ns} (k={a.k}, p={a.p}, q={a.q}) by "
                         + ("the unmodified reference psdcone.ran_proj (oracle/_ref)" if kind == "reference"
                            else "the oracle port of psdcone.ran_proj")
                         + f" on host cores in {sec:.2f} s, scaled by ({ns}/{a.n})²; the full-size "
                           "reference is timed by `bench.py --impl reference`"}
    c4 = None
    if a.config == "c3" and not a.no_c4:
        psd._native.free_plans()
        torch.cuda.empty_cache()
        try:
            c4 = c4_leg(a, torch, dist, psd, world, rank, dev)
        except Exception as exc:   # never lose the headline line to the secondary leg
            c4 = {"error": f"{type(exc).__name__}: {str(exc)[:300]}"}
    if world > 1:
        dist.destroy_process_group()
    if rank != 0:
        return
    peak_tf = peak if peak else nominal / 1000.0
    metric = METRIC if a.config == "c3" else (
        f"rand-PSD projections/s at n={n},k={a.k} fp64 ({a.config})")
    line = {
        "metric": metric, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": ms / a.steps, "higher_is_better": True,
        "step_ms_min_median_max": [per_step[0], per_step[len(per_step) // 2], per_step[-1]],
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic (seeded BASELINE {a.config} matrices generated in HBM)",
        "config": workload_config(a, world),
        "roofline": (int8_roofline(n, params.width, i8_ms / max(i8_cnt, 1), i8_cnt, traffic, peaks)
                     if engine == 1 and i8_cnt else {
            "bound": "tensor", "achieved": gemm_tf, "peak": peak_tf, "unit": "TFLOP/s",
            "frac": gemm_tf / peak_tf, "traffic": traffic.get("bytes_per_launch") if traffic else None,
            "kernel": "gemm_tma_kernel<TMA-fed, warp-specialised DMMA, 64x272 tiles> — op(X)·P "
                      f"(n×n·n×w), {2 * n * n * params.width / 1e9:.0f} GFLOP per launch, "
                      f"{gemm_ms:.2f} ms avg over {g_cnt} launches (CUDA events, timed region)",
            "peak_source": "cuBLAS DGEMM 8192³ burst measured in this run (MEASURED_PEAKS.json has "
                           f"no FP64 entry); nominal DMMA peak at 1965 MHz = {nominal / 1000:.1f}",
            "traffic_source": traffic.get("source") if traffic else None,
        }),
        "peaks_in_run": peaks,
        "sketch_engine": {0: "fp64-dmma", 1: "int8-ozaki2 (exact FP64 emulation)", 2: "3xtf32"}[engine],
        "sketch_product_fp64_equiv_tflops": gemm_tf,
        "sketch_product_ms": gemm_ms,
        "fp64_dmma_peak_tflops": peak_tf,
        "projection_tflops": flops * value / world / 1e12,
        "projection_roofline_frac": flops * value / world / 1e12 / peak_tf,
        "flops_per_projection": flops,
        "effective_rank": r_plus,
        "stages_ms_per_projection": stages,
        "gpu_launches": launches,
        "clocks": clk,
    }
    if cpu:
        line["cpu_baseline"] = cpu
    if e2e:
        line["e2e"] = e2e
    if unpipelined:
        line["unpipelined"] = unpipelined
    if fp32:
        line["fp32"] = fp32
    if scaled:
        line["scaled"] = scaled
    if c4:
        line["c4_sharded"] = c4
    print(json.dumps(line), flush=True)


def run_scaled_leg(a, torch, psd, pool, params, dev, world, out64):
    """Alg. 3 with α estimated by Alg. 5 (``project(method="scaled_randomized")``,
    projection.py:200-223): 2(N+1) HBM-bound GEMV passes over X (sketch.py:106-114,
    :126-129) then the shifted projection.  Timed like the main line; the α
    estimate is bracketed separately so its GEMV bandwidth can be read against HBM."""
    import torch.distributed as dist
    from paper_2410_19208_b200._tensors import Operand
    from paper_2410_19208_b200.sketch import min_eig_magnitude_device
    n = a.n
    power_n = 10
    cfg = psd.ProjectorConfig(method="scaled_randomized", params=params, power_N=power_n)
    rng = psd.DeviceRng(seed=977)
    steps = max(2, min(a.steps, 8))
    for i in range(2):
        psd.project(pool[i % len(pool)], cfg, rng)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    falls = 0
    for i in range(steps):
        rep = psd.project(pool[i % len(pool)], cfg, rng)
        falls += int(rep.fallback)
    e1.record()
    torch.cuda.synchronize(dev)
    ms = _max_over_ranks(torch, dist, world, e0.elapsed_time(e1), dev)
    # the α estimate alone (two power iterations of N+1 products each), as project() runs it on
    # these bitwise-symmetric matrices: every product reads X's lower 64×64 tiles only
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 4
    torch.cuda.synchronize(dev)
    a0.record()
    for i in range(reps):
        min_eig_magnitude_device(Operand(pool[i % len(pool)], "torch_cuda", dev), power_n, rng,
                                 bitwise_symmetric=True)
    a1.record()
    torch.cuda.synchronize(dev)
    alpha_ms = a0.elapsed_time(a1) / reps
    passes = 2 * (power_n + 1)
    nt = n // 64
    gemv_bytes = passes * 8.0 * (nt * (nt + 1) // 2) * 64 * 64   # lower tiles incl. the diagonal ones
    gbs = gemv_bytes / (alpha_ms / 1000.0) / 1e9
    hbm = measured_peaks().get("hbm_gbs") or 7700.0
    return {"value": world * steps / (ms / 1000.0), "unit": UNIT, "ms_per_step": ms / steps,
            "steps": steps, "fallbacks": falls,
            "workload": f"project(method='scaled_randomized', power_N={power_n}) on the C3 matrices: "
                        "α = min_eig_magnitude (Alg. 5) then ran_proj_scal (Alg. 3)",
            "alpha_estimate": {"ms": alpha_ms, "gemv_passes": passes,
                               "algorithmic_bytes": gemv_bytes, "achieved_gbs": gbs, "peak_gbs": hbm,
                               "frac": gbs / hbm,
                               "peak_source": "MEASURED_PEAKS.json hbm_gbs",
                               "note": "CUDA events around 4 min_eig_magnitude calls on the lower "
                                       "triangle (symv tile + reduce + normalise kernels, one host read "
                                       "per power iteration); algorithmic bytes = the lower 64×64 tiles "
                                       "read once per product (half of the row GEMV's 8n²)"}}


def c4_leg(a, torch, dist, psd, world, rank, dev):
    """BASELINE config 4: one projection of n=131072 (k=512, p=32, q=2) row-sharded
    over all ranks per step (sharded.py), X rows generated in place (bitwise
    symmetric by construction → symmetric="assume"; the sharded check is
    measured separately as ``symcheck_ms``).  Factored result below 4 ranks (X_g and
    the dense X̂₊_g together would exceed a GPU's 180 GB), dense row blocks from 4 up."""
    from paper_2410_19208_b200 import sharded, workloads
    cfg = CONFIGS["c4"]
    n, params = cfg["n"], psd.RangeParams(k=cfg["k"], l=cfg["p"], q=cfg["q"])
    starts = sharded.row_split(n, world)
    r0, r1 = starts[rank], starts[rank + 1]
    x = workloads.c4_rows(n, r0, r1, seed=11, device=dev, chunk_rows=4096)
    om = psd.DeviceRng(99).normal((n, params.width), dev)      # identical on every rank
    # dense X̂₊ row blocks from 4 ranks up (X_g + X̂₊_g = 2·137/N GB); factored (W, d) below
    want = world >= 4
    ops = sharded.KernelOps(dev)
    comm = sharded.Comm()
    sharded.sharded_ran_proj(x, r0, n, om, params, comm=comm, ops=ops, want_result=want,
                             symmetric="assume")
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    steps = max(1, a.c4_steps)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        rep = sharded.sharded_ran_proj(x, r0, n, om, params, comm=comm, ops=ops, want_result=want,
                                       symmetric="assume")
    e1.record()
    torch.cuda.synchronize(dev)
    ms = _max_over_ranks(torch, dist, world, e0.elapsed_time(e1), dev)
    # the sharded require_symmetric pass (block-pair exchange), timed once
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    s0.record()
    mx, defect, bitwise, _ = sharded.sharded_symmetry_stats(x, r0, n, comm, ops)
    s1.record()
    torch.cuda.synchronize(dev)
    sym_ms = _max_over_ranks(torch, dist, world, s0.elapsed_time(s1), dev)
    del x, om
    torch.cuda.empty_cache()
    value = steps / (ms / 1000.0)
    flops = 2.0 * n * n * params.width * (2 * params.q + 2) + (float(n) * n * rep.effective_rank if want else 0)
    return {"metric": f"rand-PSD projections/s at n={n},k={cfg['k']} fp64 (config 4, row-sharded)",
            "value": value, "unit": UNIT, "n_gpus": world, "steps": steps, "ms_per_step": ms / steps,
            "scaling": "strong", "effective_rank": rep.effective_rank,
            "tflops_fp64_equiv": flops * value / 1e12,
            "result": "dense row blocks" if want else "factored (W, d): X_g and the dense X̂₊_g together exceed 180 GB below 4 ranks",
            "symcheck_ms": sym_ms, "symcheck_bitwise": bitwise,
            "sketch_engine": "int8-ozaki2 (exact FP64 emulation, X_g streamed in 8192-row chunks)"
                             if ops.int8_products else "fp64-dmma",
            "exchanges": "NCCL all_gather_into_tensor of the n×w panel before each product, all_reduce "
                         "of the w×w Grams and T"}


def run_solver(a):
    """Config 5: `--steps` iterations of the dual gradient ascent (Alg. 6) with a
    randomized projection each; value = solver iterations/s."""
    import numpy as np

    from paper_2410_19208_b200 import workloads
    cfg = CONFIGS["c5"]
    n, m = a.n, cfg["m"]
    sp = workloads.c5_problem(n, m, nnz_per=4, seed=5)
    beta = workloads.c5_step_size(sp)

    def cpu_solve(its):
        """The CPU arm of this line (reference arm / cpu_baseline leg only): the
        oracle's sparse-COO restatement of psdcone.solve on the same instance."""
        from oracle import sdls_oracle as so
        prob = so.SparseProblem(sp.c, sp.rho, sp.con, sp.rows, sp.cols, sp.vals, sp.b)
        t0 = time.perf_counter()
        so.solve(prob, "randomized", a.k, a.p, a.q, beta=beta, epsilon=1e-300, max_iter=its, rng=1)
        return its / (time.perf_counter() - t0)
    metric = "SDLS solver iterations/s at n=4096, m=20000, k=64, q=1 (config 5)"
    conf = {"workload": f"BASELINE config 5: sdls.solve, n={n}, m={m}, k={a.k}, p={a.p}, q={a.q}, "
                        f"randomized projector, beta=1/L={beta:.4g}, {a.steps} iterations",
            "n": n, "m": m, "k": a.k, "p": a.p, "q": a.q, "beta": beta}
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    if a.impl == "reference":
        its = max(1, min(a.steps, 3))
        value = cpu_solve(its)
        cores = cpu_cores()
        print(json.dumps({"metric": metric, "value": value, "unit": "iterations/s", "impl": "reference",
                          "n_gpus": 1, "steps": its, "warmup": 0, "ms_per_step": 1000 / value,
                          "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                          "dtype": "f64", "data": "synthetic (seeded config-5 instance)", "config": conf,
                          "cpu_baseline": {"value": value, "unit": "iterations/s", "cores": cores,
                                           "kind": "port", "sample": f"{its} iterations of the oracle "
                                           "sparse-COO restatement of psdcone.solve"},
                          "e2e": {"value": value, "unit": "iterations/s", "h2d_bytes_per_step": 0,
                                  "d2h_bytes_per_step": 0}}), flush=True)
        return
    import torch

    import paper_2410_19208_b200 as psd
    dev = torch.device("cuda", 0)
    pcfg = psd.ProjectorConfig(method="randomized", params=psd.RangeParams(k=a.k, l=a.p, q=a.q))
    # y0 / Ω from the device Philox stream (perf mode, as the C3 line); the numpy
    # stream (reference draw order) costs ~3 ms of host RNG per iteration
    psd.solve(sp, pcfg, beta=beta, epsilon=1e-300, max_iter=max(a.warmup, 1), rng=psd.DeviceRng(1))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep = psd.solve(sp, pcfg, beta=beta, epsilon=1e-300, max_iter=a.steps, rng=psd.DeviceRng(2))
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    value = rep.iterations / dt
    line = {"metric": metric, "value": value, "unit": "iterations/s", "n_gpus": 1, "steps": rep.iterations,
            "warmup": a.warmup, "ms_per_step": 1000 * dt / rep.iterations, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded config-5 instance)", "config": conf,
            "final_grad_norm": rep.grad_norm_final,
            "timing": "wall clock around solve() incl. per-iteration host syncs, problem upload "
                      "and the final dense reconstruction; y0 and Ω from the device Philox stream"}
    if not a.no_cpu_baseline:
        v = cpu_solve(2)
        line["cpu_baseline"] = {"value": v, "unit": "iterations/s", "cores": cpu_cores(), "kind": "port",
                                "sample": "2 iterations of the oracle sparse-COO restatement of psdcone.solve"}
    print(json.dumps(line), flush=True)


def run_sharded(a):
    """``--config c4``: only the config-4 row-sharded line (see c4_leg)."""
    import torch
    import torch.distributed as dist

    import paper_2410_19208_b200 as psd
    world, rank, local, dev = _dist_setup(torch, dist)
    psd.set_fp64_engine(a.fp64_engine)
    c4 = c4_leg(a, torch, dist, psd, world, rank, dev)
    if world > 1:
        dist.destroy_process_group()
    if rank != 0:
        return
    line = dict(c4)
    line.update({"warmup": 1, "higher_is_better": True, "vs_baseline": None, "dtype": "f64",
                 "data": "synthetic (config-4 rows generated per rank, bitwise symmetric)",
                 "config": {"workload": f"BASELINE config 4: n={CONFIGS['c4']['n']}, k={CONFIGS['c4']['k']}, "
                                        f"p={CONFIGS['c4']['p']}, q={CONFIGS['c4']['q']}, row-sharded x{world}"}})
    print(json.dumps(line), flush=True)


def run_fp32_leg(a, torch, psd, pool, params, rng, dev, world, peaks):
    """BASELINE config 3 "fp32": the same projections on the fp32-rounded matrices
    through the FP32 path (3xTF32 tcgen05 GEMMs, FP64 QR/eigh), timed like the
    FP64 line (CUDA events, max over ranks)."""
    import torch.distributed as dist
    n = a.n
    pool32 = [x.float() for x in pool]
    plan = psd._native.get_plan(n, params.width, dev)
    out32 = torch.empty((n, n), dtype=torch.float32, device=dev)   # no allocation in the timed loop
    # pipelined like the FP64 line (psd_plan_prefetch_f32): none across the warm-up/timed
    # boundary and after the last timed step
    nxt = (lambda i, last: None if a.no_prefetch or i == last else pool32[(i + 1) % len(pool32)])
    nwarm = max(a.warmup, 2)
    for i in range(nwarm):
        psd.ran_proj(pool32[i % len(pool32)], params, rng, dtype="fp32", out=out32, prefetch=nxt(i, nwarm - 1))
    torch.cuda.synchronize(dev)
    plan.profile(enable=True, reset=True)
    if world > 1:
        dist.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    launches = 0
    marks = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps + 1)]
    e0.record()
    for i in range(a.steps):
        marks[i].record()
        rep = psd.ran_proj(pool32[i % len(pool32)], params, rng, dtype="fp32", out=out32,
                           prefetch=nxt(i, a.steps - 1))
        launches += rep.device_info["gpu_launches"]
    marks[a.steps].record()
    e1.record()
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1)
    per_step = sorted(marks[i].elapsed_time(marks[i + 1]) for i in range(a.steps))
    prof = plan.profile(enable=False, reset=True)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    g_ms, g_cnt = prof["sketch_gemm"]
    gemm_ms = g_ms / max(g_cnt, 1)
    eff_tf = 2.0 * n * n * params.width / (gemm_ms / 1000.0) / 1e12
    del pool32, out32
    return {
        "value": world * a.steps / (ms / 1000.0), "unit": UNIT, "ms_per_step": ms / a.steps,
        "step_ms_min_median_max": [per_step[0], per_step[len(per_step) // 2], per_step[-1]],
        "dtype": "f32 (3xTF32 tcgen05, FP32 TMEM accumulation in ≤4096-K chunks, FP64 QR/eigh)",
        "gpu_launches": launches,
        "stages_ms_per_projection": {k: round(v[0] / a.steps, 3) for k, v in prof.items() if v[1]},
        "sketch_gemm": {
            "ms_per_launch": gemm_ms,
            "effective_tflops": eff_tf,
            "tf32_tensor_tflops": 3.0 * eff_tf,
            "note": "3 tf32 MMAs (lo·hi, hi·lo, hi·hi) per FP32 product; effective = 2n²w/t",
        },
        "roofline": fp32_roofline(3.0 * eff_tf, peaks),
        "parity": "≤1e-4 rel. Frobenius vs the FP64 path on the same fp32-rounded X (tests/test_gpu_fp32.py)",
    }


def fp32_roofline(tf32_tflops, peaks):
    """tf32 issue rate of the 3xTF32 sketch GEMM against the TF32 tensor peak: cuBLAS
    fp32 8192³ with TF32 allowed, best single launch (burst), measured in this run —
    the same policy as the INT8 line.  Fallback: MEASURED_PEAKS bf16 sustained / 2."""
    if peaks.get("tf32_tflops"):
        peak, src = peaks["tf32_tflops"], ("cuBLAS TF32 8192^3 burst, measured in this run (nominal "
                                           "dense TF32: 1100 TFLOP/s)")
    else:
        try:
            with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as fh:
                pk = json.load(fh)
            peak = float(pk.get("bf16_tflops_sustained") or pk["bf16_tflops"]) / 2.0
            src = "MEASURED_PEAKS.json bf16 sustained / 2"
        except Exception:
            peak, src = 1100.0, "B200_PROFILING.md nominal tf32 dense 1.1 PFLOP/s"
    return {"bound": "tensor", "achieved": tf32_tflops, "peak": peak, "unit": "TFLOP/s",
            "frac": tf32_tflops / peak, "traffic": load_traffic32(),
            "peak_sustained": peaks.get("tf32_tflops_sustained"),
            "frac_of_nominal": tf32_tflops / 1100.0,
            "kernel": "tc32_gemm2_kernel (tcgen05.mma.cta_group::2.kind::tf32, TMA SW128, TMEM accumulators)",
            "peak_source": src}


def load_traffic32():
    try:
        with open(os.path.join(REPO, "profiles", "tc32_traffic.json")) as fh:
            return json.load(fh).get("bytes_per_launch")
    except Exception:
        return None


def run_e2e(a, torch, psd, x_dev, params, dev):
    """Same metric through the public API with HOST buffers: every step uploads
    its X from pinned host memory and downloads its X̂₊ into pinned host memory,
    all inside the timed region.  ``psd.ran_proj_many`` overlaps the upload of
    X_{i+1} and the download of X̂₊_{i−1} with the projection of X_i (two copy
    streams, double-buffered device X / result)."""
    n = a.n
    try:
        hx = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
        hr = [torch.empty((n, n), dtype=torch.float64, pin_memory=True) for _ in range(2)]
    except Exception as exc:  # pragma: no cover - host RAM
        return {"value": None, "unit": UNIT, "error": f"pinned alloc failed: {exc}"}
    hx.copy_(x_dev.cpu())
    rng = psd.DeviceRng(seed=777)
    steps = max(1, a.e2e_steps)
    psd.ran_proj_many([hx], params, rng, out=[hr[0]])      # warm-up (buffers, plan)
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    reps = psd.ran_proj_many([hx] * steps, params, rng, out=[hr[i % 2] for i in range(steps)])
    e1.record()
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1)
    wall = time.perf_counter() - t0
    ok = all(r.effective_rank > 0 for r in reps)
    return {"value": steps / (ms / 1000.0), "unit": UNIT, "h2d_bytes_per_step": 8 * n * n,
            "d2h_bytes_per_step": 8 * n * n, "steps": steps, "wall_s": wall, "results_ok": ok,
            "path": "pinned host X → paper_2410_19208_b200.ran_proj_many (H2D / projection / D2H "
                    "overlapped on three streams) → pinned host X̂₊"}


def relaunch(a):
    """``--gpus N`` (N > 1) outside torchrun: re-run this script under
    torch.distributed.run with N ranks (one per GPU, NCCL); never quietly
    measure one GPU."""
    import socket
    import torch
    have = torch.cuda.device_count()
    if have < a.gpus:
        print(json.dumps({"metric": METRIC, "error": f"--gpus {a.gpus} requested, {have} CUDA devices "
                                                     "visible"}), flush=True)
        sys.exit(2)
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__),
           *sys.argv[1:]]
    sys.exit(subprocess.run(cmd).returncode)


def main():
    a = parse()
    world_env = os.environ.get("WORLD_SIZE")
    if a.impl == "ours" and a.config != "c5":
        if world_env is None and a.gpus > 1:
            relaunch(a)
        if world_env is not None and int(world_env) != a.gpus:
            raise SystemExit(f"bench.py: --gpus {a.gpus} but WORLD_SIZE={world_env}; launch with "
                             f"--nproc-per-node equal to --gpus")
    if a.config == "c5":
        run_solver(a)
    elif a.config == "c4":
        run_sharded(a)
    elif a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
