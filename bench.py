#!/usr/bin/env python
"""Benchmark: randomized PSD projections/s at BASELINE config 3
(n=32768, k=256, p=16, q=1, fp64) on B200, with FP64 tensor-core roofline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one projection (``ran_proj``, Alg. 2) of a seeded C3 matrix that is
already resident in HBM; the K timed steps cycle through a pool of distinct
matrices (8.6 GB each ≫ 126 MB L2, so no L2 flush is needed).  Ω is drawn on
the device each step (Philox).  The FP64 n×n sketch products run by default on
the INT8 tensor cores as an exact FP64 emulation (Ozaki scheme II, csrc/ozaki.cu;
same ≤1e-10 parity as the DMMA path); ``--fp64-engine dmma`` keeps them on the
FP64 DMMA kernel.  Multi-GPU: independent replicas, one process
per GPU (the C3 projections are independent), value
= all ranks' projections / max-over-ranks device time.

``--impl reference`` times the reference algorithm's CPU implementation (the
oracle port in oracle/psd_oracle.py — same numpy/OpenBLAS calls as
psdcone.ran_proj) on this box's host cores, on a bounded sample (n=8192 with
C3's k, p, q), scaled by (8192/32768)² to the metric's unit.
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
    }


# --------------------------------------------------------------------- CPU ---

def cpu_cores():
    try:
        from threadpoolctl import threadpool_info
        nt = max((d.get("num_threads") or 0) for d in threadpool_info() if d.get("user_api") == "blas")
        return int(nt) if nt else os.cpu_count()
    except Exception:
        return os.cpu_count()


def cpu_sample(a, reps=1):
    """Oracle port (same numpy calls as psdcone.ran_proj) at n=CPU_SAMPLE_N; returns
    (projections/s scaled to n=a.n, seconds per sample)."""
    import numpy as np

    from oracle import psd_oracle as orc
    ns = min(CPU_SAMPLE_N, a.n)
    x = {"c1": lambda: orc.c1_matrix(seed=11, n=ns), "c2": lambda: orc.wigner(ns, seed=11),
         "c3": lambda: orc.c3_matrix(ns, seed=11)}[a.config]()
    best = 1e300
    for r in range(reps):
        om = np.random.default_rng(100 + r).standard_normal((ns, a.k + a.p))
        t0 = time.perf_counter()
        orc.ran_proj(x, a.k, a.p, a.q, omega=om)
        best = min(best, time.perf_counter() - t0)
    scale = (ns / a.n) ** 2  # every stage of the path is O(n²) at fixed width
    return scale / best, best, ns


def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    n_gpus = int(os.environ.get("WORLD_SIZE", str(a.gpus)))
    if rank != 0:
        return
    for _ in range(max(a.warmup, 0)):
        cpu_sample(a)
    vals, secs = [], []
    for _ in range(a.steps):
        v, s, ns = cpu_sample(a)
        vals.append(v)
        secs.append(s)
    value = a.steps / sum(s / ((ns / a.n) ** 2) for s in secs)
    cores = cpu_cores()
    ns = min(CPU_SAMPLE_N, a.n)
    sample = (f"oracle port of psdcone.ran_proj (numpy/OpenBLAS, {cores} threads) on a {a.config} matrix at "
              f"n={ns}, k={a.k}, p={a.p}, q={a.q}; time × (n/{ns})² per step")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": n_gpus,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1000.0 / value,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded C3 matrix, host numpy)",
        "config": workload_config(a, 1),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": sample},
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

def fp64_peak(torch, dev):
    """cuBLAS DGEMM 8192³ burst rate (MEASURED_PEAKS.json carries no FP64 entry)."""
    a = torch.randn(8192, 8192, dtype=torch.float64, device=dev)
    b = torch.randn(8192, 8192, dtype=torch.float64, device=dev)
    for _ in range(2):
        a @ b
    torch.cuda.synchronize(dev)
    best = 1e9
    for _ in range(5):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        a @ b
        e1.record()
        torch.cuda.synchronize(dev)
        best = min(best, e0.elapsed_time(e1))
    del a, b
    torch.cuda.empty_cache()
    return 2 * 8192 ** 3 / best / 1e9


def measured_peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except Exception:
        return {}


def int8_roofline(n, w, i8_ms, i8_cnt, traffic):
    """Roofline of i8_gemm2_kernel (one emulated FP64 sketch product): bound by the
    INT8 tensor pipe (ncu: tensor pipe ≈89% busy, DRAM ≈59%), so `achieved` is the
    algorithmic int8 ops per launch over its CUDA-event time, against the dense int8
    peak = 2 × the MEASURED_PEAKS bf16 rate (B200: 4.5 POPS int8 vs 2.25 PF bf16) —
    the sustained figure, the kernel runs inside a long step.  The HBM view is kept
    beside it."""
    L = 16
    ldk = (n + 127) // 128 * 128
    wpad = (w + 15) // 16 * 16
    algo_bytes = L * n * ldk + L * wpad * ldk + L * n * wpad   # A planes + panel planes + outputs
    pk = measured_peaks()
    hbm = pk.get("hbm_gbs") or 7700.0
    gbs = algo_bytes / (i8_ms / 1000.0) / 1e9
    int8_ops = 2.0 * L * n * n * w
    tops = int8_ops / (i8_ms / 1000.0) / 1e12
    sustained = pk.get("bf16_tflops_sustained")
    peak = 2.0 * (sustained or pk.get("bf16_tflops") or 2250.0)
    return {
        "bound": "tensor", "achieved": tops, "peak": peak, "unit": "TFLOP/s", "frac": tops / peak,
        "traffic": traffic.get("bytes_per_launch") if traffic else None,
        "algorithmic_ops_per_launch": int8_ops,
        "kernel": f"i8_gemm2_kernel<tcgen05.mma.cta_group::2.kind::i8, TMEM, TMA> — the 16 residue "
                  f"products of X·P mod m_l for one FP64 sketch product; {int8_ops / 1e15:.2f} int8 POP "
                  f"algorithmic per launch, {i8_ms:.3f} ms avg over {i8_cnt} launches (CUDA events "
                  f"on the launching stream, timed region); unit: int8 TOP/s",
        "peak_source": ("2 x MEASURED_PEAKS.json bf16_tflops_sustained" if sustained else
                        "2 x MEASURED_PEAKS.json bf16_tflops (burst)" if pk.get("bf16_tflops") else
                        "nominal dense int8 4.5 POPS / 2"),
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


def run_ours(a):
    import torch
    import torch.distributed as dist

    import paper_2410_19208_b200 as psd
    from paper_2410_19208_b200 import workloads

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    n, params = a.n, psd.RangeParams(k=a.k, l=a.p, q=a.q)
    psd.set_fp64_engine(a.fp64_engine)

    peak = fp64_peak(torch, dev) if rank == 0 else None
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
    for i in range(max(a.warmup, 3 if a.warmup >= 3 else a.warmup)):
        psd.ran_proj(pool[i % a.pool], params, rng, out=out64)
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
        rep = psd.ran_proj(pool[i % a.pool], params, rng, out=out64)
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
    ms = e0.elapsed_time(e1)
    prof = plan.profile(enable=False, reset=True)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = world * a.steps / (ms / 1000.0)

    # roofline of the dominant kernel.  DMMA engine: the op(X)·P FP64 GEMM (2n²w flops
    # per launch).  INT8 engine: the residue GEMM i8_gemm2_kernel, HBM-bound — per
    # launch it streams the 16 int8 residue planes of X (16·n·ld_k bytes) plus the
    # panel residues and the per-modulus outputs.
    g_ms, g_cnt = prof["sketch_gemm"]
    gemm_ms = g_ms / max(g_cnt, 1)
    gemm_tf = 2.0 * n * n * params.width / (gemm_ms / 1000.0) / 1e12
    i8_ms, i8_cnt = prof.get("int8_gemm", (0.0, 0))
    r_plus = statistics.median(ranks) if ranks else 0
    flops = psd.flops(n, params, r_plus)
    traffic = load_traffic("oz_traffic.json" if engine == 1 else "gemm_traffic.json")
    stages = {k: round(v[0] / a.steps, 3) for k, v in prof.items() if v[1]}

    fp32 = None
    if a.config == "c3" and not a.no_fp32:
        fp32 = run_fp32_leg(a, torch, psd, pool, params, rng, dev, world)

    e2e = None
    if rank == 0 and not a.no_e2e:
        e2e = run_e2e(a, torch, psd, pool[0], params, dev)
    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        v, s, ns = cpu_sample(a, reps=1)
        cpu = {"value": v, "unit": UNIT, "cores": cpu_cores(), "kind": "port",
               "sample": f"1 projection of a {a.config} matrix at n={ns} (k={a.k}, p={a.p}, q={a.q}) "
                         f"by the oracle port of psdcone.ran_proj on host cores in {s:.2f} s, "
                         f"scaled by ({ns}/{a.n})²"}
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
        "roofline": (int8_roofline(n, params.width, i8_ms / max(i8_cnt, 1), i8_cnt, traffic)
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
    if fp32:
        line["fp32"] = fp32
    print(json.dumps(line), flush=True)


def run_solver(a):
    """Config 5: `--steps` iterations of the dual gradient ascent (Alg. 6) with a
    randomized projection each; value = solver iterations/s."""
    import numpy as np

    from oracle import sdls_oracle as so
    cfg = CONFIGS["c5"]
    n, m = a.n, cfg["m"]
    prob = so.config5_instance(n, m, nnz_per=4, seed=5)
    beta = so.lipschitz_beta(prob)
    metric = "SDLS solver iterations/s at n=4096, m=20000, k=64, q=1 (config 5)"
    conf = {"workload": f"BASELINE config 5: sdls.solve, n={n}, m={m}, k={a.k}, p={a.p}, q={a.q}, "
                        f"randomized projector, beta=1/L={beta:.4g}, {a.steps} iterations",
            "n": n, "m": m, "k": a.k, "p": a.p, "q": a.q, "beta": beta}
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    if a.impl == "reference":
        its = max(1, min(a.steps, 3))
        t0 = time.perf_counter()
        so.solve(prob, "randomized", a.k, a.p, a.q, beta=beta, epsilon=1e-300, max_iter=its, rng=1)
        value = its / (time.perf_counter() - t0)
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
    sp = psd.SparseSdlsProblem(prob.c, 1.0, prob.con, prob.rows, prob.cols, prob.vals, prob.b)
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
        t0 = time.perf_counter()
        so.solve(prob, "randomized", a.k, a.p, a.q, beta=beta, epsilon=1e-300, max_iter=2, rng=1)
        v = 2 / (time.perf_counter() - t0)
        line["cpu_baseline"] = {"value": v, "unit": "iterations/s", "cores": cpu_cores(), "kind": "port",
                                "sample": "2 iterations of the oracle sparse-COO restatement of psdcone.solve"}
    print(json.dumps(line), flush=True)


def run_sharded(a):
    """Config 4: one row-sharded projection per step over all ranks (NCCL)."""
    import torch
    import torch.distributed as dist

    import paper_2410_19208_b200 as psd
    from paper_2410_19208_b200 import sharded, workloads
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    n = a.n
    params = psd.RangeParams(k=a.k, l=a.p, q=a.q)
    psd.set_fp64_engine(a.fp64_engine)
    starts = sharded.row_split(n, world)
    r0, r1 = starts[rank], starts[rank + 1]
    x = workloads.c4_rows(n, r0, r1, seed=11, device=dev, chunk_rows=4096)
    om = psd.DeviceRng(99).normal((n, params.width), dev)      # identical on every rank
    want = world > 1   # one GPU cannot hold X (137 GB) and the dense result together
    ops = sharded.KernelOps(dev)
    comm = sharded.Comm()
    for _ in range(max(1, a.warmup)):
        sharded.sharded_ran_proj(x, r0, n, om, params, comm=comm, ops=ops, want_result=want)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.steps):
        rep = sharded.sharded_ran_proj(x, r0, n, om, params, comm=comm, ops=ops, want_result=want)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.destroy_process_group()
    if rank != 0:
        return
    value = a.steps / (ms / 1000.0)
    flops = 2.0 * n * n * params.width * (2 * params.q + 2) + (float(n) * n * rep.effective_rank if want else 0)
    print(json.dumps({
        "metric": f"rand-PSD projections/s at n={n},k={a.k} fp64 (config 4, row-sharded)", "value": value,
        "unit": UNIT, "n_gpus": world, "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms / a.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (config-4 rows generated per rank, bitwise symmetric)",
        "config": {"workload": f"BASELINE config 4: n={n}, k={a.k}, p={a.p}, q={a.q}, row-sharded x{world}",
                   "result": "dense row blocks" if want else "factored (W, d): X and X₊ do not fit one GPU"},
        "effective_rank": rep.effective_rank, "tflops": flops * value / 1e12,
        "sketch_engine": "int8-ozaki2 (exact FP64 emulation, X_g streamed in 8192-row chunks)"
                         if ops.int8_products else "fp64-dmma"}), flush=True)


def run_fp32_leg(a, torch, psd, pool, params, rng, dev, world):
    """BASELINE config 3 "fp32": the same projections on the fp32-rounded matrices
    through the FP32 path (3xTF32 tcgen05 GEMMs, FP64 QR/eigh), timed like the
    FP64 line (CUDA events, max over ranks)."""
    import torch.distributed as dist
    n = a.n
    pool32 = [x.float() for x in pool]
    plan = psd._native.get_plan(n, params.width, dev)
    out32 = torch.empty((n, n), dtype=torch.float32, device=dev)   # no allocation in the timed loop
    for i in range(max(a.warmup, 2)):
        psd.ran_proj(pool32[i % len(pool32)], params, rng, dtype="fp32", out=out32)
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
        rep = psd.ran_proj(pool32[i % len(pool32)], params, rng, dtype="fp32", out=out32)
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
        "roofline": fp32_roofline(3.0 * eff_tf),
        "parity": "≤1e-4 rel. Frobenius vs the FP64 path on the same fp32-rounded X (tests/test_gpu_fp32.py)",
    }


def fp32_roofline(tf32_tflops):
    """tf32 issue rate of the 3xTF32 sketch GEMM against the tf32 tensor peak:
    MEASURED_PEAKS.json's bf16 burst / 2 (kind::tf32 runs the tcgen05 datapath
    at half the f16 rate — 1.1 vs 2.25 PFLOP/s nominal in B200_PROFILING.md)."""
    peak, src = None, None
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as fh:
            peak = float(json.load(fh)["bf16_tflops"]) / 2.0
            src = "MEASURED_PEAKS.json bf16_tflops (burst) / 2"
    except Exception:
        peak, src = 1100.0, "B200_PROFILING.md nominal tf32 dense 1.1 PFLOP/s (no MEASURED_PEAKS.json)"
    return {"bound": "tensor", "achieved": tf32_tflops, "peak": peak, "unit": "TFLOP/s",
            "frac": tf32_tflops / peak, "traffic": load_traffic32(),
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


def main():
    a = parse()
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
