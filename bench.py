"""Benchmark of the B200 implicit moment-tensor CP f+grad (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--config c3] [--mode fp64|tf32x3]

A step is one f+grad evaluation (f, grad_lam, grad_A at (lam, A)) over the whole observation
set of the workload (c4: one ||X||^2 reduction).  Default workload: c3 (n=512, p=4e6, d=6, r=64,
float32 observations, FP64 arithmetic) -- the largest BASELINE configuration run on one GPU and
the FP64-compute-bound case the north star's ">= 70% of FP64 peak" target is quoted on.  c2
(the HBM-bound n=100 case), c5 and c4 are selectable with --config.

Multi-GPU: `--gpus N` under torchrun (WORLD_SIZE = N) runs one rank per GPU; without torchrun
and N > 1 the script relaunches itself under `python -m torch.distributed.run` with N local
ranks (127.0.0.1).  The p rows are sharded across ranks (strong scaling: total work fixed); the
[Y | w] partials are exchanged over NVLink peer memory fused with the finish (csrc/peer.cu),
self-tested against the NCCL all-reduce path, which stays the fallback.

Printed (rank 0, one JSON line):
  value      evals/s with lam, A already in HBM, K steps between barriers + device syncs, CUDA
             events, max over ranks.
  e2e        the same metric through the public API (packed_fg_implicit(obs, d, r)(x) with a
             host numpy x): H2D of x and D2H of [f; g] inside every step.
  roofline   dominant kernel (K1 / K5), event-timed inside the timed region: algorithmic
             bytes (n p sizeof(V)) or flops (4 n p r; 3x that executed in tf32x3) per launch /
             its duration vs the measured peak of its bound.
  cpu_baseline  the reference algorithm (CPU oracle port, numpy/OpenBLAS, all host threads) on
             a bounded sample of the same workload (rows scaled by p / p_sample, or p^2 for
             ||X||^2), rank 0 at N=1; median and best of the sample evaluations.
--impl reference runs only that CPU arm, on the same config/metric.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DEFAULT_CONFIG = "c3"
SEED = 2024
# bounded CPU sample per config (rows of V); None = the whole workload
CPU_SAMPLE_ROWS = {"c1": None, "c2": None, "c3": 200_000, "c4": 16_000, "c5": 40_000,
                   "t2": None}
L2_BYTES = 126 * 2**20


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
    """(hbm GB/s, source, fp64 TF/s, tf32 TF/s, source note)."""
    hbm = _read_json(os.path.join(ROOT, "MEASURED_PEAKS.json"))
    if hbm and "hbm_gbs" in hbm:
        hbm_gbs, hbm_src = float(hbm["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    else:
        hbm_gbs, hbm_src = 6650.0, "fallback (B200_PROFILING.md)"
    fp = _read_json(os.path.join(ROOT, "profiles", "peaks_fp64_tf32_r01.json")) or {}
    return (hbm_gbs, hbm_src, float(fp.get("dmma_884_tflops", 37.09)),
            float(fp.get("cublas_tf32_8192_tflops", 741.9)))


def _sustained_tensor_peak(mode):
    """Sustained (back-to-back, power-capped) library peak for kernels timed inside long steps."""
    fp = _read_json(os.path.join(ROOT, "profiles", "peaks_fp64_tf32_r01.json")) or {}
    key = "cublas_tf32_8192_sustained_tflops" if mode == "tf32x3" else "cublas_dgemm_8192_sustained_tflops"
    return fp.get(key)


PEAK_NOTE = ("FP64 = DMMA.8x8x4 throughput and TF32 = cuBLAS 8192^3 TF32 GEMM, both measured by "
             "this build on the pool's B200 (tools/probe_fp64.cu, tools/probe_peaks.py -> "
             "profiles/peaks_fp64_tf32_r01.json; MEASURED_PEAKS.json carries only HBM and bf16)")


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
        sm, smax, power, reasons = [], None, [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
                power.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w_median": statistics.median(power) if power else None}


# ------------------------------------------------------------------------------------------
# CPU reference arm (oracle port of the reference's numpy path; test/bench infrastructure)
# ------------------------------------------------------------------------------------------

def _use_all_host_threads():
    # torchrun exports OMP_NUM_THREADS=1; the reference arm uses every host core
    try:
        from threadpoolctl import threadpool_limits

        threadpool_limits(limits=os.cpu_count())
    except Exception:  # noqa: BLE001
        pass


def _blas_threads():
    try:
        from threadpoolctl import threadpool_info

        return max((d.get("num_threads", 1) for d in threadpool_info()), default=os.cpu_count())
    except Exception:  # noqa: BLE001
        return os.cpu_count()


def _cpu_sample_rows(cfg):
    s = CPU_SAMPLE_ROWS.get(cfg.name)
    return cfg.p if s is None else min(cfg.p, s)


def _cpu_scale(cfg, p_sample):
    # f+grad is linear in p; ||X||^2 is O(p^2) (implicit.py:116-121: a p x p Gram)
    ratio = cfg.p / p_sample
    return ratio * ratio if cfg.r == 0 else ratio


def cpu_eval_times(cfg, V_nxp, lam, A, *, budget_s=12.0, min_evals=3, max_evals=None):
    """Wall times of the reference algorithm on the host sample (seconds per evaluation).

    f+grad: oracle fg_implicit (objective.py:77-94); ||X||^2: the blocked restatement of
    implicit.py:116-121 (the reference's own p x p Gram does not fit the host at c4)."""
    from oracle import momentcp_oracle as om

    nu = np.full(V_nxp.shape[1], 1.0 / V_nxp.shape[1])
    times = []
    t_start = time.perf_counter()
    while True:
        t0 = time.perf_counter()
        if cfg.r == 0:
            om.data_norm_sq_blocked(V_nxp, nu, cfg.d, block=4000)
        else:
            om.fg_implicit(V_nxp, nu, lam, A, cfg.d, 0.0)
        times.append(time.perf_counter() - t0)
        if max_evals and len(times) >= max_evals:
            break
        if len(times) >= min_evals and time.perf_counter() - t_start > budget_s:
            break
    return times


def _cpu_baseline_block(cfg, times, p_sample, what):
    scale = _cpu_scale(cfg, p_sample)
    med = statistics.median(times) * scale
    best = min(times) * scale
    threads = _blas_threads()
    if scale == 1:
        sample = f"{len(times)} evaluations of the full {cfg.name} workload"
    elif cfg.r == 0:
        sample = (f"{len(times)} blocked ||X||^2 reductions at p={p_sample}, EXTRAPOLATED "
                  f"x{scale:g} = (p/p_sample)^2 (the reduction is O(n p^2))")
    else:
        sample = (f"{len(times)} evaluations on a {p_sample}-row sample, EXTRAPOLATED "
                  f"x{scale:g} = p/p_sample (f+grad is linear in p)")
    return {"value": 1.0 / med, "unit": "evals/s", "cores": threads, "kind": "port",
            "best": 1.0 / best, "statistic": "value = median, best = fastest evaluation",
            "extrapolated": scale != 1,
            "sample": sample + f"; {what} on numpy/OpenBLAS ({threads} threads, fp64)"}


def _cpu_what(cfg):
    return ("oracle data_norm_sq_blocked (restates implicit.py:116-121)" if cfg.r == 0 else
            "oracle fg_implicit (restates objective.py:77-94)")


def run_reference(args, cfg, rank, world):
    """--impl reference: the CPU reference arm alone (rank 0; other ranks exit 0)."""
    if rank != 0:
        return
    from paper_1911_03813_b200 import synth

    _use_all_host_threads()
    p_sample = _cpu_sample_rows(cfg)
    V = np.asarray(synth.host_observations(cfg, SEED, p=p_sample), dtype=float)
    lam, A = synth.initial_point(cfg, SEED) if cfg.r else (None, None)
    cpu_eval_times(cfg, V, lam, A, max_evals=args.warmup, min_evals=args.warmup)
    times = cpu_eval_times(cfg, V, lam, A, max_evals=args.steps, min_evals=args.steps)
    cb = _cpu_baseline_block(cfg, times, p_sample, _cpu_what(cfg))
    evals = cb["value"]
    line = {
        "metric": _metric(cfg), "value": evals, "unit": "evals/s", "n_gpus": world,
        "devices": "host cores only (the reference is CPU-only; n_gpus = the N it was launched at)",
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 / evals, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "impl": "reference",
        "data": f"synthetic seeded {'Gaussian' if cfg.k == 0 else 'Gaussian mixture'} ({cfg.name})",
        "config": _config_dict(cfg, args.mode, world),
        "cpu_baseline": cb,
        "e2e": {"value": evals, "unit": "evals/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------
# helpers shared by the GPU arms
# ------------------------------------------------------------------------------------------

def _metric(cfg):
    return "||X||^2 evals/s" if cfg.r == 0 else "f+grad evals/s"


def _config_dict(cfg, mode, world):
    """The workload only (no implementation keys: the reference arm prints the same dict)."""
    return {"workload": f"{cfg.name}: n={cfg.n} p={cfg.p} d={cfg.d} r={cfg.r} V {cfg.dtype}, "
                        f"{'Gaussian' if cfg.k == 0 else str(cfg.k) + '-component mixture'} "
                        f"sigma={cfg.sigma}",
            "n": cfg.n, "p": cfg.p, "d": cfg.d, "r": cfg.r, "v_dtype": cfg.dtype,
            "mode": mode if cfg.r else "fp64", "parallelism": f"row-shard dp{world}",
            "l2": _l2_note(cfg)}


def _v_bytes(cfg) -> int:
    return cfg.n * cfg.p * (4 if cfg.dtype == "f32" else 8)


def _l2_note(cfg) -> str:
    vb = _v_bytes(cfg)
    if vb > L2_BYTES:
        return "inputs larger than L2 (V = %.0f MB > 126 MB), no flush needed" % (vb / 1e6)
    return ("V = %.1f MB fits L2: L2 flushed (256 MB write) before every timed step; steps "
            "timed individually with CUDA events, flush excluded" % (vb / 1e6))


def _free_port() -> int:
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _relaunch_under_torchrun(n: int) -> int:
    """`--gpus N` without torchrun: run this script as N local ranks (one per GPU)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.abspath(__file__), *sys.argv[1:]]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    return subprocess.call(cmd, env=env)


def _init_dist(world, dev, same_dev):
    import torch.distributed as dist

    if world > 1:
        if same_dev:
            dist.init_process_group("gloo")
        else:
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=dev)


def _clock_sampler(torch, dev, local):
    try:
        gpu_id = "GPU-" + str(torch.cuda.get_device_properties(dev).uuid)
    except Exception:  # noqa: BLE001
        gpu_id = str(local)
    return ClockSampler(gpu_id)


def _nvtx(torch, name):
    class _R:
        def __enter__(self):
            torch.cuda.nvtx.range_push(name)

        def __exit__(self, *a):
            torch.cuda.nvtx.range_pop()
    return _R()


# ------------------------------------------------------------------------------------------
# ||X||^2 (config 4)
# ------------------------------------------------------------------------------------------

def run_data_norm(args, cfg, rank, world, local):
    """Config 4: ||X||^2 = nu^T (V^T V)^d nu (one step = one full Gram-power reduction).

    Rank k holds row shard k of V; the tile pairs are split over the ranks with the shards
    passed around a ring over NVLink (paper_1911_03813_b200.distributed.data_norm_sq_sharded),
    the W partial sums are added in rank order."""
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
    _init_dist(world, dev, same_dev)
    lo, hi = D.shard_bounds(cfg.p, world, rank)
    Vrows = synth.device_observations(cfg, SEED, device=dev, row_offset=lo, rows=hi - lo)
    sobs = D.ShardedObservationSet.from_device_rows(Vrows, cfg.p, lo)
    ctx = sobs.local.device_context()

    def step():
        return D.data_norm_sq_sharded(sobs, cfg.d)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    clocks = _clock_sampler(torch, dev, local)
    if rank == 0:
        clocks.start()
    ctx.set_kernel_timing(True)
    ctx.kernel_time_ms(reset=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with _nvtx(torch, "timed"):
        e0.record()
        for _ in range(args.steps):
            val = step()
        e1.record()
    torch.cuda.synchronize()
    el = e0.elapsed_time(e1) * 1e-3
    if world > 1:
        t = torch.tensor([el], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        el = float(t.item())
    k_ms, k_n = ctx.kernel_time_ms(reset=True)
    ctx.set_kernel_timing(False)
    variant = ctx.last_variant
    clk = clocks.stop() if rank == 0 else None

    # e2e: the public API from a host array each step (upload of V + reduction + scalar D2H)
    e2e = None
    if world == 1:
        Vh = Vrows.t().contiguous().cpu().numpy()   # (n, p) host, the reference layout
        del Vrows
        torch.cuda.empty_cache()
        for _ in range(1):
            mcp.data_norm_sq(mcp.ObservationSet(Vh), cfg.d)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ne = max(1, min(args.steps, 5))
        for _ in range(ne):
            mcp.data_norm_sq(mcp.ObservationSet(Vh), cfg.d)
        e2e_s = (time.perf_counter() - t0) / ne
        e2e = {"value": 1.0 / e2e_s, "unit": "evals/s", "h2d_bytes_per_step": int(Vh.nbytes),
               "d2h_bytes_per_step": 8,
               "what": "mcp.data_norm_sq(mcp.ObservationSet(V_host), d): upload + reduction"}
    _, _, fp64_peak, _ = _peaks()
    flops = cfg.n * cfg.p * (cfg.p + 1.0)       # 2n per pair l <= l'
    if rank == 0:
        kavg = k_ms / max(k_n, 1) / max(1, (world + 1) // 2 if world > 1 else 1)
        achieved = flops / world / (el / args.steps) / 1e12
        line = {"metric": _metric(cfg), "value": args.steps / el, "unit": "evals/s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": 1e3 * el / args.steps, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic seeded V ~ N(0,1)/sqrt(n), generated on GPU",
                "config": _config_dict(cfg, "fp64", world), "kernel": variant,
                "value_check": val,
                "roofline": {"bound": "tensor", "kernel": variant,
                             "kernel_launches_per_step": k_n / max(args.steps, 1),
                             "achieved": achieved, "peak": fp64_peak, "unit": "TFLOP/s",
                             "frac": achieved / fp64_peak, "traffic": None,
                             "alg_flops_per_step": flops, "peak_source": PEAK_NOTE,
                             "note": "achieved = n p (p+1) flops / world / device step time "
                                     "(the K5 launches are the whole step)"},
                "e2e": e2e, "clocks": clk, "gpu_launches": None}
        line["gpu_launches"] = int(round(k_n + args.steps * (1 + max(world - 1, 0))))
        if world == 1 and not args.no_cpu:
            _use_all_host_threads()
            p_s = _cpu_sample_rows(cfg)
            Vs = np.asarray(synth.host_observations(cfg, SEED, p=p_s), dtype=float)
            times = cpu_eval_times(cfg, Vs, None, None, budget_s=12.0, min_evals=3)
            line["cpu_baseline"] = _cpu_baseline_block(cfg, times, p_s, _cpu_what(cfg))
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ------------------------------------------------------------------------------------------
# f+grad (configs 1, 2, 3, 5)
# ------------------------------------------------------------------------------------------

def run_fg(args, cfg, rank, world, local):
    import torch
    import torch.distributed as dist

    import paper_1911_03813_b200 as mcp
    from paper_1911_03813_b200 import _native
    from paper_1911_03813_b200 import distributed as D
    from paper_1911_03813_b200 import synth

    # MCP_BENCH_SAME_DEVICE=1 (test only): every rank on cuda:0 over gloo, to exercise the
    # multi-rank flow on a one-GPU box (NCCL refuses two ranks on one device).
    same_dev = os.environ.get("MCP_BENCH_SAME_DEVICE") == "1"
    if same_dev:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    _init_dist(world, dev, same_dev)
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
    p_sample = _cpu_sample_rows(cfg)
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
                try:
                    pex.step(d, x_dev.data_ptr(), args.mode, 0.0, out.data_ptr(), stream)
                    torch.cuda.synchronize()
                    bad = not torch.allclose(out, ref_out, rtol=1e-12, atol=1e-300)
                except D.PeerExchangeError:
                    bad = True
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
            pex.step(d, x_dev.data_ptr(), args.mode, 0.0, out.data_ptr(), stream, check=False)
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
    with _nvtx(torch, "warmup"):
        for _ in range(args.warmup):
            step_device()
        barrier_sync()
    clocks = _clock_sampler(torch, dev, local)
    if rank == 0:
        clocks.start()
    t_soak = time.perf_counter()
    while time.perf_counter() - t_soak < 1.5:
        for _ in range(4):
            step_device()
        torch.cuda.synchronize()
    barrier_sync()

    # ---- timed region: exactly K device-resident steps ----
    # K1 is event-timed on every 8th step for short steps (an event pair costs ~5 us)
    every = 1 if cfg.p * cfg.n * cfg.r >= 10**10 else (8 if args.steps >= 64 else
                                                      (4 if args.steps >= 8 else 1))
    ctx.set_kernel_timing(True, every=every)
    ctx.kernel_time_ms(reset=True)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    barrier_sync()
    with _nvtx(torch, "timed"):
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
    if pex is not None:
        # a timed step whose peer partial never arrived produced NaN: reject the run
        pex.raise_if_failed()
    if not bool(torch.isfinite(out).all()):
        raise RuntimeError("non-finite f+grad in the timed region")
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
        fg = D.packed_fg_sharded(sobs, d, r, mode=args.mode)
    for _ in range(3):
        fg(x_host)
    barrier_sync()
    t0 = time.perf_counter()
    with _nvtx(torch, "e2e"):
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
        tensor_peak, tensor_kind = tf32_peak, "measured cuBLAS TF32 8192^3 (burst)"
        exec_factor = 3.0
    else:
        tensor_peak, tensor_kind = fp64_peak, "measured DMMA.8x8x4 FP64"
        exec_factor = 1.0
    ridge = tensor_peak * 1e12 / exec_factor / (hbm_gbs * 1e9)
    ai = alg_flops / alg_bytes
    bound = "hbm" if ai < ridge else "tensor"
    traffic = None
    prof = _read_json(os.path.join(ROOT, "profiles", f"ncu_k1_{cfg.name}_{args.mode}_r02.json"))
    if prof and prof.get("variant") == variant and world == 1:
        traffic = prof.get("dram_bytes_per_launch")   # captured at N = 1 (the full row range)
    value = args.steps / (ms_total * 1e-3)
    step_flops = 4.0 * n * cfg.p * r
    line = {
        "metric": _metric(cfg), "value": value, "unit": "evals/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_total / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64" if args.mode == "fp64" else "tf32x3 (fp32 data, fp64 epilogue/tail)",
        "data": f"synthetic seeded Gaussian mixture ({cfg.name}), generated on GPU",
        "config": _config_dict(cfg, args.mode, world),
        "kernel": variant, "upload_s": round(t_up, 4), "exchange": exchange,
        "tflops": {"achieved": step_flops * value / 1e12,
                   "executed": step_flops * value * exec_factor / 1e12,
                   "peak": tensor_peak, "peak_kind": tensor_kind,
                   "frac": step_flops * value * exec_factor / 1e12 / tensor_peak,
                   "flops_per_step": step_flops, "executed_flops_per_alg_flop": exec_factor,
                   "note": "whole-step rate (all launches) over the peak of the mode's pipe"},
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
                     "fp64_tflops": achieved_tf if args.mode == "fp64" else None,
                     "hbm_gbs": achieved_gbs,
                     "peak_source": hbm_src if bound == "hbm" else PEAK_NOTE},
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
        _use_all_host_threads()
        # bounded CPU sample on this host: the full workload when it fits (c1, c2), else rows
        times = cpu_eval_times(cfg, Vh_sample, lam, A, budget_s=12.0, min_evals=3)
        line["cpu_baseline"] = _cpu_baseline_block(cfg, times, p_sample, _cpu_what(cfg))
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps (default: 20 for c3/c4/c5, 200 otherwise)")
    ap.add_argument("--warmup", type=int, default=None)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default=DEFAULT_CONFIG)
    ap.add_argument("--mode", default="fp64", choices=["fp64", "tf32x3"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    args = ap.parse_args()

    from paper_1911_03813_b200 import synth

    cfg = synth.CONFIGS[args.config]
    big = cfg.name in ("c3", "c4", "c5")
    if args.steps is None:
        args.steps = 20 if big else 200
    if args.warmup is None:
        args.warmup = 5 if big else 10
    args.warmup = max(args.warmup, 3)
    rank, world, local = _env_rank()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(_relaunch_under_torchrun(args.gpus))
    if world != args.gpus and os.environ.get("MCP_BENCH_SAME_DEVICE") != "1":
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU")
    if args.impl == "reference":
        return run_reference(args, cfg, rank, world)
    if cfg.r == 0:
        return run_data_norm(args, cfg, rank, world, local)
    return run_fg(args, cfg, rank, world, local)


if __name__ == "__main__":
    main()
