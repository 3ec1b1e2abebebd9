"""Benchmark of the B200 implicit moment-tensor CP f+grad (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--config c2] [--mode fp64]

A step is one f+grad evaluation (f, grad_lam, grad_A at (lam, A)) over the whole observation
set of the workload.  Default workload: BASELINE.json configs[1] = c2 (n=100, p=1e6, d=4,
r=10, float64), the configuration the metric is quoted on.  For N > 1 (torchrun, one process
per GPU) the p rows are sharded across ranks (strong scaling: total work fixed) and the
[Y | w] partials are combined by one NCCL all-reduce per step.

Printed (rank 0, one JSON line):
  value      evals/s with lam, A already in HBM (mcp_fg_device / partial+all-reduce+finish),
             K steps between barriers + device syncs, CUDA events, max over ranks.
  e2e        the same metric through the public API (packed_fg_implicit(obs, d, r)(x) with a
             host numpy x): H2D of x and D2H of [f; g] inside every step.
  roofline   dominant kernel K1: algorithmic bytes (n*p*sizeof(V)) per launch / its
             event-timed duration vs measured HBM peak (MEASURED_PEAKS.json), with the
             FP64 view (4 n p r flops) vs the measured DMMA peak (profiles/peaks_*.json).
  cpu_baseline  the reference algorithm (CPU oracle port, numpy/OpenBLAS, all host threads)
             on the same workload, rank 0 at N=1.
--impl reference runs only that CPU arm, on the same config/metric.
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

DEFAULT_CONFIG = "c2"
SEED = 2024


def _env_rank():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def _read_json(path):
    try:
        with open(path) as fh:
            return json.load(fh)
    except (OSError, ValueError):
        return None


def _peaks():
    hbm = _read_json(os.path.join(ROOT, "MEASURED_PEAKS.json"))
    if hbm and "hbm_gbs" in hbm:
        hbm_gbs, hbm_src = float(hbm["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    else:
        hbm_gbs, hbm_src = 6650.0, "fallback (B200_PROFILING.md)"
    fp = _read_json(os.path.join(ROOT, "profiles", "peaks_fp64_tf32_r01.json")) or {}
    return hbm_gbs, hbm_src, float(fp.get("dmma_884_tflops", 37.09)), float(
        fp.get("cublas_tf32_8192_tflops", 741.9))


def _sustained_tensor_peak(mode):
    """Sustained (back-to-back, power-capped) library peak for kernels timed inside long steps."""
    fp = _read_json(os.path.join(ROOT, "profiles", "peaks_fp64_tf32_r01.json")) or {}
    key = "cublas_tf32_8192_sustained_tflops" if mode == "tf32x3" else "cublas_dgemm_8192_sustained_tflops"
    return fp.get(key)


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 100 ms while the GPU is under load."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_id: str):
        self.gpu = gpu_id
        self.proc = None
        self.lines = []
        self._t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self._t = threading.Thread(target=self._drain, daemon=True)
        self._t.start()

    def _drain(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self._t.join(timeout=5)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_arm(cfg, V_nxp, lam, A, budget_s=12.0, min_evals=2, max_evals=None):
    """Reference algorithm (oracle port of pkg/src/momentcp/objective.py:77-94) on the host."""
    from oracle import momentcp_oracle as om

    nu = np.full(V_nxp.shape[1], 1.0 / V_nxp.shape[1])
    times = []
    t_start = time.perf_counter()
    while True:
        t0 = time.perf_counter()
        om.fg_implicit(V_nxp, nu, lam, A, cfg.d, 0.0)
        times.append(time.perf_counter() - t0)
        if len(times) >= min_evals and time.perf_counter() - t_start > budget_s:
            break
        if max_evals and len(times) >= max_evals:
            break
    return times


def _blas_threads():
    try:
        from threadpoolctl import threadpool_info

        return max((d.get("num_threads", 1) for d in threadpool_info()), default=os.cpu_count())
    except Exception:  # noqa: BLE001
        return os.cpu_count()


def run_reference(args, cfg, rank, world):
    """--impl reference: the CPU reference arm alone (rank 0; other ranks exit 0)."""
    if rank != 0:
        return
    from paper_1911_03813_b200 import synth

    # torchrun exports OMP_NUM_THREADS=1; the reference arm uses every host core
    try:
        from threadpoolctl import threadpool_limits

        threadpool_limits(limits=os.cpu_count())
    except Exception:  # noqa: BLE001
        pass
    p_sample = cfg.p if cfg.name in ("c1", "c2") else min(cfg.p, 200_000)
    V = synth.host_observations(cfg, SEED, p=p_sample)
    V = np.asarray(V, dtype=float)
    lam, A = synth.initial_point(cfg, SEED)
    for _ in range(args.warmup):
        cpu_arm(cfg, V, lam, A, budget_s=0.0, min_evals=1, max_evals=1)
    times = cpu_arm(cfg, V, lam, A, budget_s=0.0, min_evals=args.steps, max_evals=args.steps)
    scale = cfg.p / p_sample
    evals = 1.0 / (sum(times) / len(times) * scale)
    threads = _blas_threads()
    line = {
        "metric": "f+grad evals/s", "value": evals, "unit": "evals/s", "n_gpus": world,
        "devices": "host cores only (the reference is CPU-only; n_gpus = the N it was launched at)",
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 / evals, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "impl": "reference",
        "data": f"synthetic seeded Gaussian mixture ({cfg.name})",
        "config": _config_dict(cfg, args, world),
        "cpu_baseline": {"value": evals, "unit": "evals/s", "cores": threads, "kind": "port",
                         "sample": (f"full {cfg.name} workload, p={p_sample}" if scale == 1 else
                                    f"{cfg.name} row sample p={p_sample}, scaled x{scale:g} "
                                    "(f+grad is linear in p)")
                                   + f"; numpy/OpenBLAS {threads} threads, fp64"},
        "e2e": {"value": evals, "unit": "evals/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_data_norm(args, cfg, rank, world, local):
    """Config 4: ||X||^2 = nu^T (V^T V)^d nu (one step = one full Gram-power reduction).

    Every rank holds the full V (generated identically on each GPU) and computes its slice
    of the upper-triangular tile-pair list; the W partial sums are all-gathered and added in
    rank order (paper_1911_03813_b200.distributed.data_norm_sq_split)."""
    import torch
    import torch.distributed as dist

    import paper_1911_03813_b200 as mcp
    from paper_1911_03813_b200 import distributed as D
    from paper_1911_03813_b200 import synth

    same_dev = os.environ.get("MCP_BENCH_SAME_DEVICE") == "1"   # test only, see main()
    if same_dev:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if same_dev:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    if args.impl == "reference":
        return
    V = synth.device_observations(cfg, SEED, device=dev)
    obs = mcp.ObservationSet.from_device(V)
    ctx = obs.device_context()
    for _ in range(args.warmup):
        D.data_norm_sq_split(obs, cfg.d)
    torch.cuda.synchronize()
    ctx.set_kernel_timing(True)
    ctx.kernel_time_ms(reset=True)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        val = D.data_norm_sq_split(obs, cfg.d)
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([el], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        el = float(t.item())
    k_ms, k_n = ctx.kernel_time_ms(reset=True)
    _, _, fp64_peak, _ = _peaks()
    flops = cfg.n * cfg.p * (cfg.p + 1.0)       # 2n per pair l <= l'
    if rank == 0:
        line = {"metric": "||X||^2 evals/s", "value": args.steps / el, "unit": "evals/s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": 1e3 * el / args.steps, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic seeded V ~ N(0,1)/sqrt(n), generated on GPU",
                "config": _config_dict(cfg, args, world), "value_check": val,
                "roofline": {"bound": "tensor", "kernel": ctx.last_variant,
                             "kernel_avg_ms": k_ms / max(k_n, 1),
                             "achieved": flops / world / (k_ms / max(k_n, 1) * 1e-3) / 1e12,
                             "peak": fp64_peak, "unit": "TFLOP/s",
                             "frac": flops / world / (k_ms / max(k_n, 1) * 1e-3) / 1e12 / fp64_peak}}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def _config_dict(cfg, args, world):
    return {"workload": f"{cfg.name}: n={cfg.n} p={cfg.p} d={cfg.d} r={cfg.r} V {cfg.dtype}, "
                        f"{'Gaussian' if cfg.k == 0 else str(cfg.k) + '-component mixture'} "
                        f"sigma={cfg.sigma}",
            "n": cfg.n, "p": cfg.p, "d": cfg.d, "r": cfg.r, "v_dtype": cfg.dtype,
            "mode": args.mode, "parallelism": f"row-shard dp{world}",
            "l2": _l2_note(cfg)}


L2_BYTES = 126 * 2**20


def _v_bytes(cfg) -> int:
    return cfg.n * cfg.p * (4 if cfg.dtype == "f32" else 8)


def _l2_note(cfg) -> str:
    vb = _v_bytes(cfg)
    if vb > L2_BYTES:
        return "inputs larger than L2 (V = %.0f MB > 126 MB), no flush needed" % (vb / 1e6)
    return ("V = %.1f MB fits L2: L2 flushed (256 MB write) before every timed step; steps "
            "timed individually with CUDA events, flush excluded" % (vb / 1e6))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default=DEFAULT_CONFIG)
    ap.add_argument("--mode", default="fp64", choices=["fp64", "tf32x3"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    from paper_1911_03813_b200 import synth

    cfg = synth.CONFIGS[args.config]
    rank, world, local = _env_rank()
    if cfg.r == 0:
        return run_data_norm(args, cfg, rank, world, local)
    if args.impl == "reference":
        return run_reference(args, cfg, rank, world)

    import torch
    import torch.distributed as dist

    import paper_1911_03813_b200 as mcp
    from paper_1911_03813_b200 import _native
    from paper_1911_03813_b200 import distributed as D

    # MCP_BENCH_SAME_DEVICE=1 (test only): every rank on cuda:0 over gloo, to exercise the
    # multi-rank flow on a one-GPU box (NCCL refuses two ranks on one device).
    same_dev = os.environ.get("MCP_BENCH_SAME_DEVICE") == "1"
    if same_dev:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if same_dev:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    group = None

    # ---- data: this rank's rows, generated on its GPU ----
    lo, hi = D.shard_bounds(cfg.p, world, rank)
    Vrows = synth.device_observations(cfg, SEED, device=dev, row_offset=lo, rows=hi - lo)
    obs = mcp.ObservationSet.from_device(Vrows, p_total=cfg.p, release=True)
    t_up = time.perf_counter()
    ctx = obs.device_context()
    torch.cuda.synchronize()
    t_up = time.perf_counter() - t_up
    # the CPU leg's bounded sample (host copy), then free the generator's copy: the context
    # holds the rows (and the fast mode's V_lo needs the room at c5)
    p_sample = cfg.p if cfg.name in ("c1", "c2") else min(cfg.p, 100_000)
    Vh_sample = (Vrows[:p_sample].double().cpu().numpy().T
                 if world == 1 and not args.no_cpu else None)
    del Vrows
    torch.cuda.empty_cache()
    lam, A = synth.initial_point(cfg, SEED)
    n, r, d = cfg.n, cfg.r, cfg.d
    x_host = mcp.pack(lam, A)
    x_dev = torch.as_tensor(x_host, device=dev)
    Yw = torch.empty(n * r + r, dtype=torch.float64, device=dev)
    out = torch.empty(1 + r + n * r, dtype=torch.float64, device=dev)
    stream = _native.stream_handle(torch.cuda.current_stream(dev))

    def step_nccl():
        ctx.fg_partial_device(d, r, x_dev.data_ptr(), args.mode, Yw.data_ptr(), stream)
        dist.all_reduce(Yw, op=dist.ReduceOp.SUM)
        ctx.fg_finish_device(d, r, x_dev.data_ptr(), Yw.data_ptr(), 0.0, out.data_ptr(), stream)

    # multi-GPU exchange: NVLink peer memory fused with the finish (csrc/peer.cu), verified
    # against the NCCL all-reduce path once; NCCL stays the fallback
    pex, exchange = None, "none"
    if world > 1:
        exchange = "nccl-allreduce"
        if not same_dev and os.environ.get("MCP_PEER", "1") != "0":
            try:
                pex = D.PeerExchange(ctx, n, r, rank, world, group)
            except Exception as exc:  # noqa: BLE001 - NCCL path stays
                print(f"peer exchange unavailable: {exc}", file=sys.stderr)
                pex = None
            ok_t = torch.tensor([1.0 if pex is not None else 0.0], device=dev)
            dist.all_reduce(ok_t, op=dist.ReduceOp.MIN)
            if float(ok_t.item()) == 0.0:
                pex = None
            else:
                step_nccl()
                torch.cuda.synchronize()
                ref_out = out.clone()
                pex.step(d, x_dev.data_ptr(), args.mode, 0.0, out.data_ptr(), stream)
                torch.cuda.synchronize()
                bad = pex.failed() or not torch.allclose(out, ref_out, rtol=1e-12, atol=1e-300)
                bad_t = torch.tensor([1.0 if bad else 0.0], device=dev)
                dist.all_reduce(bad_t, op=dist.ReduceOp.MAX)
                if float(bad_t.item()) == 0.0:
                    exchange = "nvlink-peer (fused reduce+finish, csrc/peer.cu)"
                else:
                    print("peer exchange self-test failed; using the NCCL all-reduce",
                          file=sys.stderr)
                    pex = None

    def step_device():
        if world == 1:
            ctx.fg_device(d, r, x_dev.data_ptr(), 0.0, args.mode, out.data_ptr(), stream)
        elif pex is not None:
            pex.step(d, x_dev.data_ptr(), args.mode, 0.0, out.data_ptr(), stream)
        else:
            step_nccl()

    def barrier_sync():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- warm-up, then a clock soak under the same load (nvidia-smi needs >= ~1 s) ----
    for _ in range(args.warmup):
        step_device()
    barrier_sync()
    try:
        gpu_id = "GPU-" + str(torch.cuda.get_device_properties(dev).uuid)
    except Exception:  # noqa: BLE001
        gpu_id = str(local)
    clocks = ClockSampler(gpu_id)
    if rank == 0:
        clocks.start()
    t_soak = time.perf_counter()
    while time.perf_counter() - t_soak < 1.5:
        for _ in range(20):
            step_device()
        torch.cuda.synchronize()
    barrier_sync()

    # ---- timed region: exactly K device-resident steps ----
    # K1 is event-timed on every 8th step (each event pair costs ~5 us of a ~0.19 ms c2 step)
    ctx.set_kernel_timing(True, every=8 if args.steps >= 64 else (4 if args.steps >= 8 else 1))
    ctx.kernel_time_ms(reset=True)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    barrier_sync()
    if _v_bytes(cfg) // max(world, 1) > L2_BYTES:
        e0.record()
        for _ in range(args.steps):
            step_device()
        e1.record()
        barrier_sync()
        ms_total = max_over_ranks(e0.elapsed_time(e1))
    else:
        # V fits in L2: flush it before every step and time the steps one by one
        scrub = torch.empty(256 * 2**20 // 4, dtype=torch.float32, device=dev)
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
        for a, b in evs:
            scrub.fill_(1.0)
            a.record()
            step_device()
            b.record()
        barrier_sync()
        ms_total = max_over_ranks(sum(a.elapsed_time(b) for a, b in evs))
    k1_ms, k1_launches = ctx.kernel_time_ms(reset=True)
    ctx.set_kernel_timing(False)
    launches_per_step = ctx.last_launch_count if world == 1 else (3 if pex is not None else 6)
    scaling_breakdown = None
    if world > 1:
        # the same K steps without the exchange (this rank's partial only): what the exchange and
        # finish add per step, for the scaling analysis (max over ranks)
        p0 = torch.cuda.Event(enable_timing=True)
        p1 = torch.cuda.Event(enable_timing=True)
        barrier_sync()
        p0.record()
        for _ in range(args.steps):
            ctx.fg_partial_device(d, r, x_dev.data_ptr(), args.mode, Yw.data_ptr(), stream)
        p1.record()
        barrier_sync()
        partial_ms = max_over_ranks(p0.elapsed_time(p1)) / args.steps
        scaling_breakdown = {"partial_ms_per_step": partial_ms,
                             "step_ms": ms_total / args.steps,
                             "exchange_and_finish_ms": ms_total / args.steps - partial_ms,
                             "rows_per_rank": hi - lo}
    variant = ctx.last_variant
    clk = clocks.stop() if rank == 0 else None

    # ---- e2e through the public API (host x in, host f, g out every step) ----
    if world == 1:
        fg = mcp.packed_fg_implicit(obs, d, r, mode=args.mode)
    else:
        sobs = D.ShardedObservationSet(obs, cfg.p, lo, group)
        fg = D.packed_fg_sharded(sobs, d, r)
    for _ in range(3):
        fg(x_host)
    barrier_sync()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        f_val, g_val = fg(x_host)
    barrier_sync()
    e2e_s = max_over_ranks(time.perf_counter() - t0)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    hbm_gbs, hbm_src, fp64_peak, tf32_peak = _peaks()
    vbytes = 4 if cfg.dtype == "f32" else 8
    rows_here = hi - lo
    k1_avg_ms = k1_ms / max(k1_launches, 1)
    alg_bytes = n * rows_here * vbytes
    alg_flops = 4.0 * n * rows_here * r
    achieved_gbs = alg_bytes / (k1_avg_ms * 1e-3) / 1e9
    achieved_tf = alg_flops / (k1_avg_ms * 1e-3) / 1e12
    if args.mode == "tf32x3":
        # 3xTF32: the tensor pipe executes 3 TF32 products per algorithmic flop
        tensor_peak, tensor_kind = tf32_peak, "measured cuBLAS TF32 8192^3 (profiles/peaks_fp64_tf32_r01.json)"
        exec_factor = 3.0
    else:
        tensor_peak, tensor_kind = fp64_peak, "measured DMMA.8x8x4 FP64"
        exec_factor = 1.0
    ridge = tensor_peak * 1e12 / exec_factor / (hbm_gbs * 1e9)
    ai = alg_flops / alg_bytes
    bound = "hbm" if ai < ridge else "tensor"
    traffic = None
    prof = _read_json(os.path.join(ROOT, "profiles", f"ncu_k1_{cfg.name}_r01.json"))
    if prof and prof.get("variant") == variant and world == 1:
        traffic = prof.get("dram_bytes_per_launch")   # captured at N = 1 (the full row range)
    value = args.steps / (ms_total * 1e-3)
    step_flops = 4.0 * n * cfg.p * r
    line = {
        "metric": "f+grad evals/s", "value": value, "unit": "evals/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_total / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64" if args.mode == "fp64" else "tf32x3 (fp32 data, fp64 epilogue/tail)",
        "data": f"synthetic seeded Gaussian mixture ({cfg.name}), generated on GPU",
        "config": dict(_config_dict(cfg, args, world), kernel=variant,
                       upload_s=round(t_up, 4), exchange=exchange),
        "tflops": {"achieved": step_flops * value / 1e12, "peak": fp64_peak,
                   "peak_kind": "measured DMMA.8x8x4 FP64 (profiles/peaks_fp64_tf32_r01.json)",
                   "frac": step_flops * value / 1e12 / fp64_peak,
                   "flops_per_step": step_flops},
        "roofline": {"bound": bound,
                     "achieved": achieved_gbs if bound == "hbm" else achieved_tf * exec_factor,
                     "peak": hbm_gbs if bound == "hbm" else tensor_peak,
                     "unit": "GB/s" if bound == "hbm" else "TFLOP/s",
                     "frac": (achieved_gbs / hbm_gbs) if bound == "hbm"
                     else achieved_tf * exec_factor / tensor_peak,
                     "executed_flops_per_alg_flop": exec_factor,
                     "traffic": traffic,
                     "kernel": variant, "kernel_avg_ms": k1_avg_ms,
                     "kernel_share_of_step": k1_avg_ms / (ms_total / args.steps),
                     "alg_bytes_per_launch": alg_bytes, "alg_flops_per_launch": alg_flops,
                     "fp64_tflops": achieved_tf, "fp64_frac": achieved_tf / fp64_peak,
                     "peak_source": hbm_src if bound == "hbm" else tensor_kind},
        "e2e": {"value": args.steps / e2e_s, "unit": "evals/s",
                "h2d_bytes_per_step": 8 * (r + n * r + 1),
                "d2h_bytes_per_step": 8 * (1 + r + n * r)},
        "clocks": clk,
        "gpu_launches": launches_per_step * args.steps,
    }
    if scaling_breakdown is not None:
        line["scaling_breakdown"] = scaling_breakdown
    sus = _sustained_tensor_peak(args.mode)
    if bound == "tensor" and sus:
        # the burst peak stays the headline denominator; the sustained one (library GEMM back to
        # back, profiles/peaks_fp64_tf32_r01.json) is what a long power-capped step can hold
        line["roofline"]["peak_sustained"] = sus
        line["roofline"]["frac_sustained"] = line["roofline"]["achieved"] / sus
    if world == 1 and not args.no_cpu:
        try:
            from threadpoolctl import threadpool_limits

            threadpool_limits(limits=os.cpu_count())
        except Exception:  # noqa: BLE001
            pass
        # bounded CPU sample on this host: the full workload when it fits (c1, c2), else rows
        times = cpu_arm(cfg, Vh_sample, lam, A, budget_s=12.0)
        scale = cfg.p / p_sample
        med = statistics.median(times) * scale
        threads = _blas_threads()
        line["cpu_baseline"] = {
            "value": 1.0 / med, "unit": "evals/s", "cores": threads, "kind": "port",
            "sample": (f"{len(times)} evals of the full {cfg.name} workload" if scale == 1 else
                       f"{len(times)} evals of a {p_sample}-row sample scaled x{scale:g}")
                      + f", median; oracle port of objective.py:77-94 on numpy/OpenBLAS "
                        f"({threads} threads, fp64)"}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
