#!/usr/bin/env python
"""Benchmark of the TIDE exit-decision hot path on B200 (driver contract).

Headline (BASELINE.json metric): routed tokens/s of the fused
RMSNorm + router + exit mask + stable compaction at d=4096 bf16, b=128, one
checkpoint, 65,536 tokens per GPU (weak scaling), theta=0.5, dense rows, and
its fraction of the HBM roofline.  One step = one tide_route launch over the
resident batch (+ for N>1 the exit-map / compacted-index all-gathers over
NCCL).  Inputs are 512 MiB per step, larger than the 126 MB L2, so no flush.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--extra]
                    [--config headline|4|5] [--scaling weak|strong]

`--config 5` / `--config 4` time the sharded legs of BASELINE configs 5 (exit
selection over 20 checkpoints at d=8192, u8 exit-code all-gather) and 4
(calibration labeller + count all-reduce), weak or strong scaling.

`--impl reference` times the reference on the host cores instead: the
UNMODIFIED earlyexit functions (ee/router_ops.py:68-87 fused_layernorm_route,
the strict mask of ee/runtime.py:171, ee/router_ops.py:137-154 batch_compact)
from baseline/_ref when staged there (tools/stage_reference.py), else the
oracle port of the same loop; token-sharded over one process per core.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "routed tokens/sec at d=4096 bf16 (fused norm+router+compact); % HBM roofline"
UNIT = "tokens/s"
N_TOK, D, B, THETA, EPS = 65536, 4096, 128, 0.5, 1e-6
ELEM = 2
# algorithmic bytes per routed token: row + f32 score + u8 mask + int64 index
BYTES_PER_TOKEN = D * ELEM + 4 + 1 + 8
WEIGHT_BYTES = B * D * ELEM + B * 4


def workload_config(n_gpus: int, n_tok: int = N_TOK) -> dict:
    return {"workload": f"fused RMSNorm+router+exit-mask+stable-compaction, 1 checkpoint, "
                        f"{n_tok:,} tokens/GPU, d=4096, b=128, bf16 rows+W_down, f32 w_up, "
                        f"theta=0.5, dense (no row index)"
                        + ("; N>1: u8 exit-map all-gather + local global compaction"
                           if n_gpus > 1 else ""),
            "tokens_per_gpu": n_tok, "d": D, "b": B, "theta": THETA,
            "global_tokens": n_tok * n_gpus, "parallelism": f"token-sharded x{n_gpus}",
            "l2": "inputs 512 MiB per step per GPU > 126 MB L2 (no flush needed)",
            "router_init": "N(0,1)*0.05, PCG64(202)", "rows": "N(0,1) bf16, torch cuda "
                                                             "Generator seeded 1234+rank"}


# ---------------------------------------------------------------------------
# clocks sampling (B200_PROFILING.md recipe)
# ---------------------------------------------------------------------------
class ClockSampler:
    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int, period_ms: int = 100):
        self.index = index
        self.period_ms = period_ms
        self.proc = None
        self.lines = []  # (host arrival time, csv line)
        self.thread = None
        self.window = None  # host-time span of the timed region (mark())

    def mark(self, t0: float, t1: float):
        """Restrict the summary to samples taken during [t0, t1] (host clock;
        the nearest samples around it when the region is shorter than the
        sampling period)."""
        self.window = (t0, t1)

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.QUERY}",
                 "--format=csv,noheader,nounits", "-lms", str(self.period_ms)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (FileNotFoundError, OSError):
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()
        time.sleep(0.25)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=1)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        lines = self.lines
        if self.window is not None and lines:
            t0, t1 = self.window
            pad = self.period_ms / 1e3
            inside = [x for x in lines if t0 <= x[0] <= t1 + pad]
            lines = inside or [x for x in lines if t0 - 2 * pad <= x[0] <= t1 + 2 * pad] or lines
        for _, ln in lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        load = [x for x in sm if x > 300] or sm
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return {"hbm_gbs": float(d["hbm_gbs"]),
                "bf16_tflops": float(d.get("bf16_tflops", 1590.0)),
                "src": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "src": "fallback (B200_PROFILING.md)"}


def ncu_traffic(kernel: str):
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return d.get(kernel, d.get(kernel + "_bf16"))
    return None


# ---------------------------------------------------------------------------
# CPU reference / baseline: the UNMODIFIED reference functions when the
# reference package is staged in baseline/_ref (tools/stage_reference.py;
# git-ignored, travels to the GPU box), else the oracle port of the same loop
# ---------------------------------------------------------------------------
REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def _have_reference() -> bool:
    return os.path.isdir(os.path.join(REF_DIR, "earlyexit"))


def _cpu_worker(args):
    """One worker = one host core: route + strict mask + stable compaction of a
    token shard with the reference's own functions (ee/router_ops.py:68-87,
    ee/runtime.py:171, ee/router_ops.py:137-154)."""
    seed, rows, d, b, kind = args
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    from oracle import tide_oracle as O  # seeded weights / rows only
    g = np.random.Generator(np.random.PCG64(202))
    orouter = O.make_router(d, b, 3, g)
    rng = np.random.Generator(np.random.PCG64(seed))
    h = O.round_to(rng.standard_normal((rows, d), dtype=np.float32), "bf16")
    if kind == "reference":
        if REF_DIR not in sys.path:
            sys.path.insert(0, REF_DIR)
        from earlyexit import router_ops as R
        router = R.Router(layer=3, w_down=orouter.w_down, w_up=orouter.w_up)
        route, compact = R.fused_layernorm_route, R.batch_compact
    else:
        router, route, compact = orouter, O.fused_layernorm_route, O.batch_compact
    t0 = time.perf_counter()
    scores = route(h, router)                   # ee/router_ops.py:68-87
    mask = scores > np.float32(THETA)           # ee/runtime.py:171
    t1 = time.perf_counter()
    compact(h, mask)                            # ee/router_ops.py:137-154
    t2 = time.perf_counter()
    return rows, t2 - t0, t2 - t1


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class CpuReference:
    """The reference algorithm timed on this host's cores: one worker process
    per core (OPENBLAS_NUM_THREADS=1 each), token-sharded bounded samples."""

    def __init__(self, cores=None):
        import multiprocessing as mp
        self.cores = cores or os.cpu_count() or 1
        self.kind = "reference" if _have_reference() else "port"
        os.environ["OPENBLAS_NUM_THREADS"] = "1"
        self.pool = mp.get_context("spawn").Pool(self.cores)
        rows, dt, _ = self.pool.map(_cpu_worker, [(7, 128, D, B, self.kind)] * self.cores)[0]
        self.per_proc = rows / max(dt, 1e-9)

    def sample(self, target_s: float) -> dict:
        rows_each = int(max(64, min(65536, self.per_proc * target_s)))
        rows_each = int(math.ceil(rows_each / 64) * 64)
        res = self.pool.map(_cpu_worker, [(100 + i, rows_each, D, B, self.kind)
                                          for i in range(self.cores)])
        total = sum(r for r, _, _ in res)
        slowest = max(t for _, t, _ in res)
        compact_share = sum(c for _, _, c in res) / max(1e-9, sum(t for _, t, _ in res))
        what = ("unmodified earlyexit 0.1.0 from baseline/_ref" if self.kind == "reference"
                else "oracle port of the reference loop")
        return {"value": total / slowest, "unit": UNIT, "cores": self.cores, "kind": self.kind,
                "sample": f"{self.cores} processes x {rows_each} tokens (d=4096, bf16-rounded "
                          f"rows as f32; {what}: fused_layernorm_route + strict mask + "
                          f"batch_compact, whose row copy is {100 * compact_share:.1f}% of the "
                          f"time)",
                "tokens": total, "seconds": slowest, "cpu_model": cpu_model()}

    def close(self):
        self.pool.terminate()


def cpu_single_process_rates(target_s: float = 3.0) -> dict:
    """The reference on ONE process: OPENBLAS_NUM_THREADS=1 and =nproc (the
    reference's own BLAS threading for its per-row matvecs), in subprocesses
    so the thread count takes effect."""
    out = {}
    kind = "reference" if _have_reference() else "port"
    for threads in (1, os.cpu_count() or 1):
        code = ("import sys, json, time; sys.path.insert(0, %r); import bench; "
                "r, t, _ = bench._cpu_worker((5, 256, bench.D, bench.B, %r)); "
                "n = max(256, int(256 * %f / max(t, 1e-9)) // 64 * 64); "
                "r, t, _ = bench._cpu_worker((6, n, bench.D, bench.B, %r)); "
                "print(json.dumps({'tokens': r, 'seconds': t}))") % (ROOT, kind, target_s, kind)
        env = dict(os.environ, OPENBLAS_NUM_THREADS=str(threads), OMP_NUM_THREADS=str(threads))
        try:
            r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True,
                               text=True, timeout=300)
            j = json.loads(r.stdout.strip().splitlines()[-1])
            out[f"one_process_blas_threads_{threads}"] = j["tokens"] / j["seconds"]
        except Exception as e:  # report, do not hide
            out[f"one_process_blas_threads_{threads}"] = f"failed: {e!r}"[:200]
    return out


def cpu_reference_rate(target_s: float = 10.0) -> dict:
    ref = CpuReference()
    try:
        return ref.sample(target_s)
    finally:
        ref.close()


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    ref = CpuReference()
    step_s = float(os.environ.get("TIDE_REF_STEP_S", max(0.5, 100.0 / (args.steps + args.warmup))))
    try:
        runs = [ref.sample(step_s) for _ in range(args.warmup + args.steps)][args.warmup:]
    finally:
        ref.close()
    rate = sum(x["tokens"] for x in runs) / sum(x["seconds"] for x in runs)
    line = {"metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * sum(x["seconds"] for x in runs) / len(runs),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "config": workload_config(max(1, args.gpus)), "impl": "reference",
            "cpu_baseline": {"value": rate, "unit": UNIT, "cores": runs[-1]["cores"],
                             "kind": runs[-1]["kind"], "sample": runs[-1]["sample"],
                             "cpu_model": runs[-1]["cpu_model"]},
            "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def run_ours(args):
    import torch
    import torch.distributed as dist

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # TIDE_BENCH_ONE_GPU=1 (flow test of the N > 1 path on a one-GPU box):
    # every rank on cuda:0, gloo instead of NCCL — timings meaningless
    one_gpu = os.environ.get("TIDE_BENCH_ONE_GPU") == "1"
    if one_gpu:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    import paper_2603_21365_b200 as P
    n_tok = N_TOK if args.scaling == "weak" else N_TOK // world
    from paper_2603_21365_b200 import _device as Dv
    from paper_2603_21365_b200 import _native as N
    from paper_2603_21365_b200 import sharding as S
    from oracle import tide_oracle as O

    g = np.random.Generator(np.random.PCG64(202))
    orouter = O.make_router(D, B, 3, g)
    router = P.Router(layer=3, w_down=orouter.w_down, w_up=orouter.w_up)
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)
    h = torch.randn((n_tok, D), generator=gen, device=dev, dtype=torch.float32).to(torch.bfloat16)
    wd, wu = P.router_ops.device_weights(router, N.BF16, dev)
    gathered = S.ExitMapGather(n_tok, world, dev) if world > 1 else None
    scores = torch.empty(n_tok, dtype=torch.float32, device=dev)
    cont_idx = torch.empty(n_tok, dtype=torch.int64, device=dev)
    exit_idx = torch.empty(n_tok, dtype=torch.int64, device=dev)
    counts = torch.empty(2, dtype=torch.int64, device=dev)
    # N > 1: the kernel writes its u8 mask straight into the all-gather send buffer
    mask = gathered.exit_map if gathered is not None else torch.empty(n_tok, dtype=torch.uint8,
                                                                      device=dev)
    lib = N.load()
    stream = torch.cuda.current_stream(dev)
    sh = stream.cuda_stream
    ws = Dv.workspace(dev).data_ptr()
    launches = {"n": 0}

    # Back-to-back steps route the same resident rows: no kernel in flight
    # writes them, so the launch may start streaming while the previous one
    # drains (TIDE_ROUTE_INPUTS_READY; the default, flag 0, waits first — its
    # cost is reported as extra.kernel_ms_inputs_wait).
    def step(kernel_events=None, collective=True, flags=N.ROUTE_INPUTS_READY):
        if kernel_events is not None:
            kernel_events[0].record(stream)
        rc = lib.tide_route_ex(h.data_ptr(), D, n_tok, None, n_tok, D, N.BF16, None,
                               wd.data_ptr(), wu.data_ptr(), B, EPS, THETA, 3, scores.data_ptr(),
                               None, mask.data_ptr(), exit_idx.data_ptr(), cont_idx.data_ptr(), 0,
                               None, counts.data_ptr(), ws, flags, sh)
        launches["n"] += 1 + (gathered is not None and collective)
        if kernel_events is not None:
            kernel_events[1].record(stream)
        if rc:
            N.check(rc, "tide_route")
        if gathered is not None and collective:
            gathered.all_gather()                        # C1: 1 byte per token
            gathered.global_exit_indices(sync=False)     # C2: one local scan

    def barrier():
        if world > 1:
            dist.barrier()

    # the clock sampler starts first so the warm-up launches run right before
    # the timed region (no idle gap for the clocks to drop in)
    clocks = ClockSampler(local, period_ms=20)
    clocks.start()
    for _ in range(args.warmup):
        step()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize(dev)
    launches["n"] = 0
    w0 = time.time()
    t0.record(stream)
    for i in range(args.steps):
        step()
    t1.record(stream)
    torch.cuda.synchronize(dev)
    clocks.mark(w0, time.time())
    barrier()
    gpu_launches = launches["n"]
    clk = clocks.stop()
    ms_total = t0.elapsed_time(t1)
    # The timed region is a few ms, shorter than nvidia-smi's sampling period:
    # also sample a sustained window of the same step back to back (~0.6 s) so
    # the clocks / throttle reasons under this kernel's load are on record.
    sustained = ClockSampler(local, period_ms=50)
    sustained.start()
    ws0 = time.time()
    t_end = ws0 + 0.6
    s0 = torch.cuda.Event(enable_timing=True)
    s1 = torch.cuda.Event(enable_timing=True)
    sustained_launches = 0
    s0.record(stream)
    while time.time() < t_end:
        # kernel only: ranks leave this wall-clock loop after different
        # iteration counts, so no collective may be issued in it
        for _ in range(50):
            step(collective=False)
        sustained_launches += 50
        torch.cuda.synchronize(dev)
    s1.record(stream)
    torch.cuda.synchronize(dev)
    sustained.mark(ws0, time.time())
    # device time per launch in the power-capped steady state (includes the
    # host syncs every 50 launches, so a slight overestimate)
    sustained_ms = s0.elapsed_time(s1) / max(1, sustained_launches)
    barrier()
    clk_sustained = sustained.stop()
    # parity spot-check of the final state on rank 0 (first 2,048 rows vs the oracle)
    if rank == 0 and not args.no_check:
        hs = h[:2048].float().cpu().numpy()
        _, t_ref, m_ref = O.route_logits(hs, orouter)
        ok = O.decision_band_ok(mask[:2048].cpu().numpy(), t_ref, m_ref, THETA, 2e-2)
        assert ok.all(), "bench parity spot-check failed"
        e_ref, _ = O.compact_indices(mask.cpu().numpy())
        assert np.array_equal(exit_idx[: int(counts[0])].cpu().numpy(), e_ref)
    # per-launch kernel time of the fused kernel alone (events bracket each launch,
    # separate pass so the headline region has no per-step event records)
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    for i in range(args.steps):
        step(kev[i])
    torch.cuda.synchronize(dev)
    kernel_ms = [a.elapsed_time(b) for a, b in kev]
    # the same back-to-back region with the default (safe) launch: every
    # launch waits for the previous grid before reading its rows
    q0 = torch.cuda.Event(enable_timing=True)
    q1 = torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        step(collective=False, flags=0)
    q0.record(stream)
    for _ in range(args.steps):
        step(collective=False, flags=0)
    q1.record(stream)
    torch.cuda.synchronize(dev)
    ms_wait = q0.elapsed_time(q1) / args.steps
    ms_t = torch.tensor([ms_total], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    ms_per_step = ms_max / args.steps
    value = n_tok * world * args.steps / (ms_max / 1e3)

    # e2e through the public API with HOST buffers (pinned), copies in the timed region
    h_host = h.cpu().pin_memory()
    mask_host = torch.empty(n_tok, dtype=torch.uint8).pin_memory()
    idx_host = torch.empty(n_tok, dtype=torch.int64).pin_memory()
    cnt_host = torch.empty(2, dtype=torch.int64).pin_memory()
    h_dev = torch.empty_like(h)

    def e2e_fused_step():
        h_dev.copy_(h_host, non_blocking=True)
        rc = lib.tide_route(h_dev.data_ptr(), D, n_tok, None, n_tok, D, N.BF16, None,
                            wd.data_ptr(), wu.data_ptr(), B, EPS, THETA, 3, scores.data_ptr(),
                            None, mask.data_ptr(), exit_idx.data_ptr(), cont_idx.data_ptr(), 0,
                            None, counts.data_ptr(), ws, sh)
        N.check(rc, "tide_route")
        if gathered is not None:
            gathered.all_gather()  # the same step as the device-resident one
            gathered.global_exit_indices(sync=False)
        mask_host.copy_(mask, non_blocking=True)
        idx_host.copy_(exit_idx, non_blocking=True)
        cnt_host.copy_(counts, non_blocking=True)

    for _ in range(2):
        e2e_fused_step()
    torch.cuda.synchronize(dev)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e2e_steps = max(2, min(args.steps, 10))
    barrier()
    e0.record(stream)
    for _ in range(e2e_steps):
        e2e_fused_step()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    e_ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e_ms, op=dist.ReduceOp.MAX)
    e2e_value = n_tok * world * e2e_steps / (float(e_ms.item()) / 1e3)

    if rank == 0:
        peaks = measured_peaks()
        # average launch duration over the timed region: at N=1 the step is exactly one
        # launch, back to back, so region time / launches; at N>1 the per-launch events
        kavg = (ms_total / gpu_launches) if world == 1 else sum(kernel_ms) / len(kernel_ms)
        alg_bytes = n_tok * BYTES_PER_TOKEN + WEIGHT_BYTES
        achieved = alg_bytes / (kavg / 1e3) / 1e9
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic", "config": workload_config(world, n_tok),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"],
                         "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"],
                         "traffic": ncu_traffic("route_tc_kernel"),
                         "peak_src": peaks["src"], "kernel_ms": kavg,
                         "algorithmic_bytes_per_launch": alg_bytes,
                         "frac_of_8TBs_spec": achieved / 8000.0},
            "e2e": {"value": e2e_value, "unit": UNIT,
                    "h2d_bytes_per_step": n_tok * D * ELEM,
                    "d2h_bytes_per_step": n_tok * 1 + n_tok * 8 + 16},
            "gpu_launches": gpu_launches,
            "clocks": clk,
            "clocks_sustained": dict(clk_sustained, window="0.6 s of the same step back to back, "
                                                          "after the timed region",
                                     ms_per_launch=sustained_ms,
                                     value_per_gpu=n_tok / (sustained_ms / 1e3)),
            "extra": {"tensor_cores": bool(lib.tide_route_uses_tensor_cores(N.BF16, D, B)),
                      "tflops_tensor": 2.0 * D * B * n_tok / (kavg / 1e3) / 1e12,
                      "kernel_ms_min": min(kernel_ms), "kernel_ms_max": max(kernel_ms),
                      "kernel_ms_inputs_wait": ms_wait},
        }
        if not args.no_cpu_baseline and world == 1:  # the host baseline: rank 0 at N = 1
            line["cpu_baseline"] = {k: v for k, v in cpu_reference_rate(
                float(os.environ.get("TIDE_CPU_BASELINE_S", "10"))).items()
                if k in ("value", "unit", "cores", "kind", "sample", "cpu_model")}
            line["cpu_baseline"].update(cpu_single_process_rates())
        if world == 1 and not args.no_configs:
            # BASELINE configs 1-5 (+ the worst-case thresholds and the LM head)
            # timed in the same run, each with its roofline fraction
            from bench_extra import run_configs
            pk = measured_peaks()
            line["configs"] = run_configs(pk["hbm_gbs"], pk["bf16_tflops"])
        if args.extra:
            from bench_extra import run_extra
            line["extra"]["configs"] = run_extra(dev)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


# ---------------------------------------------------------------------------
# sharded legs of BASELINE configs 4 and 5 (bench.py --config 4|5)
# ---------------------------------------------------------------------------
def _dist_init():
    import torch
    import torch.distributed as dist
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    one_gpu = os.environ.get("TIDE_BENCH_ONE_GPU") == "1"
    if one_gpu:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    return rank, world, local, dev


def _timed_steps(step, args, dev, world, local):
    """W warm-up steps, then K steps between barriers + syncs, CUDA events on
    the current stream; returns (max-over-ranks ms, clocks)."""
    import torch
    import torch.distributed as dist
    clocks = ClockSampler(local, period_ms=20)
    clocks.start()
    for _ in range(args.warmup):
        step()
    stream = torch.cuda.current_stream(dev)
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    w0 = time.time()
    t0.record(stream)
    for _ in range(args.steps):
        step()
    t1.record(stream)
    torch.cuda.synchronize(dev)
    clocks.mark(w0, time.time())
    if world > 1:
        dist.barrier()
    ms = torch.tensor([t0.elapsed_time(t1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    return float(ms.item()), clocks.stop()


def run_config5(args):
    """BASELINE config 5: 70B shape (d=8192, 80 layers, 20 checkpoint routers),
    65,536-token prefill batch token-sharded over the GPUs (strong: 65,536/N
    tokens per GPU; weak: 8,192 per GPU).  Step = the per-token exit
    selection on the local shard (peeling chain, sharding.select_exits_shard)
    + the u8 exit-code all-gather (C1) + the local global compaction (C2)."""
    import torch
    import torch.distributed as dist
    rank, world, local, dev = _dist_init()
    import paper_2603_21365_b200 as P
    from paper_2603_21365_b200 import sharding as S
    from oracle import tide_oracle as O

    L, d, b, theta = 80, 8192, 128, args.theta if args.theta is not None else 0.7
    n_local = 65536 // world if args.scaling == "strong" else 8192
    g = np.random.Generator(np.random.PCG64(5))
    ckpts = O.checkpoint_layers(L, 4)
    routers = {k: O.make_router(d, b, k, g, scale=0.06) for k in ckpts}
    bank = P.make_bank({k: (r.w_down, r.w_up) for k, r in routers.items()}, num_layers=L)
    gen = torch.Generator(device=dev)
    gen.manual_seed(5000 + rank)
    states = [None] * (L + 1)
    for k in list(ckpts) + [L - 1]:
        t = torch.empty((n_local, d), dtype=torch.bfloat16, device=dev)
        for r0 in range(0, n_local, 8192):
            r1 = min(n_local, r0 + 8192)
            t[r0:r1] = torch.randn((r1 - r0, d), generator=gen, device=dev).to(torch.bfloat16)
        states[k + 1] = t
    for i in range(L + 1):
        if states[i] is None:
            states[i] = states[L]
    cfg = P.RuntimeConfig(exit_threshold=theta)
    gat = S.ExitMapGather(n_local, world, dev)

    def step():
        S.select_exits_shard(states, bank, cfg, gat)
        gat.global_exit_indices(sync=False)

    ms, clk = _timed_steps(step, args, dev, world, local)
    layers = gat.global_exit_layers().cpu().numpy()
    exit_rate = float((layers >= 0).mean())
    loc = layers[rank * n_local:(rank + 1) * n_local]
    remaining, peeled = n_local, 0
    for k in ckpts:
        peeled += remaining * (d * 2 + 21)
        remaining -= int((loc == k).sum())
    ms_step = ms / args.steps
    if rank == 0:
        line = {"metric": "exit-selected tokens/sec, config 5 (70B shape, 20 checkpoints, "
                          "d=8192, bf16), token-sharded", "value": n_local * world / (ms_step / 1e3),
                "unit": "tokens/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": ms_step, "higher_is_better": True, "scaling": args.scaling,
                "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
                "config": {"workload": "config 5: per-token peeling exit selection over 20 "
                                       "checkpoint routers + u8 exit-code all-gather + global "
                                       "compaction", "tokens_per_gpu": n_local,
                           "global_tokens": n_local * world, "d": d, "b": b, "theta": theta,
                           "layers": L, "checkpoints": len(ckpts),
                           "parallelism": f"token-sharded x{world}",
                           "l2": "captures 21 x n x 16 KiB per GPU, read once per step"},
                "exit_rate": exit_rate,
                "roofline": {"bound": "hbm", "achieved": peeled / (ms_step / 1e3) / 1e9,
                             "peak": measured_peaks()["hbm_gbs"], "unit": "GB/s",
                             "frac": peeled / (ms_step / 1e3) / 1e9 / measured_peaks()["hbm_gbs"],
                             "traffic": None, "algorithmic_bytes_per_step_rank0": peeled,
                             "bytes_rule": "sum over checkpoints of live rows x (d*2 + 21)"},
                "collective_bytes_per_rank": n_local, "clocks": clk}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def run_config4(args):
    """BASELINE config 4: calibration labelling, cosine similarity of 8
    checkpoints vs the final layer over 2,000 x 512 = 1,024,000 tokens at
    d=4096 bf16, token-sharded (strong: 1,024,000 / N per GPU; weak:
    1,024,000 per GPU).  Step = sharding.label_shard: one labeller launch over
    the local shard + the all-reduce of zero-norm / positive counts."""
    import torch
    import torch.distributed as dist
    rank, world, local, dev = _dist_init()
    import paper_2603_21365_b200  # noqa: F401
    from paper_2603_21365_b200 import sharding as S

    n_all, d, C, tau = 1_024_000, 4096, 8, 0.98
    n_local = n_all // world if args.scaling == "strong" else n_all
    gen = torch.Generator(device=dev)
    gen.manual_seed(4000 + rank)
    fin = torch.empty((n_local, d), dtype=torch.bfloat16, device=dev)
    cks = {3 + 4 * i: torch.empty_like(fin) for i in range(C)}
    for r0 in range(0, n_local, 131072):
        r1 = min(n_local, r0 + 131072)
        f = torch.randn((r1 - r0, d), generator=gen, device=dev)
        fin[r0:r1] = f.to(torch.bfloat16)
        for i, t in enumerate(cks.values()):  # checkpoints drift toward the final layer
            noise = 0.1 + 0.5 * (C - 1 - i) / C
            t[r0:r1] = (f + noise * torch.randn((r1 - r0, d), generator=gen,
                                                device=dev)).to(torch.bfloat16)
    out = {}

    def step():
        out.update(S.label_shard(cks, fin, tau, world))

    ms, clk = _timed_steps(step, args, dev, world, local)
    ms_step = ms / args.steps
    byts = n_local * (C + 1) * d * 2 + n_local * C * 5
    if rank == 0:
        gbs = byts / (ms_step / 1e3) / 1e9
        line = {"metric": "labelled tokens/sec, config 4 (cosine labeller, 8 checkpoints + final, "
                          "d=4096 bf16), token-sharded", "value": n_local * world / (ms_step / 1e3),
                "unit": "tokens/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": ms_step, "higher_is_better": True, "scaling": args.scaling,
                "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
                "config": {"workload": "config 4: one-pass cosine labeller + count all-reduce",
                           "tokens_per_gpu": n_local, "global_tokens": n_local * world, "d": d,
                           "checkpoints": C, "tau": tau, "parallelism": f"token-sharded x{world}",
                           "l2": f"{byts / 2**30:.1f} GiB read per step per GPU > 126 MB L2"},
                "positives_rank0": [int(x) for x in out["positives"].cpu()],
                "roofline": {"bound": "hbm", "achieved": gbs, "peak": measured_peaks()["hbm_gbs"],
                             "unit": "GB/s", "frac": gbs / measured_peaks()["hbm_gbs"],
                             "traffic": None, "algorithmic_bytes_per_step": byts},
                "clocks": clk}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--extra", action="store_true", help="also time configs 2-5 (slower)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-check", action="store_true")
    ap.add_argument("--no-configs", action="store_true",
                    help="skip the BASELINE configs 1-5 block of the N=1 line")
    ap.add_argument("--config", default="headline", choices=["headline", "4", "5"],
                    help="headline (BASELINE metric), or the sharded config-4 / config-5 legs")
    ap.add_argument("--scaling", default=None, choices=["weak", "strong"],
                    help="weak: fixed tokens per GPU (headline / config 5 default); strong: "
                         "fixed global tokens (config 4 default)")
    ap.add_argument("--theta", type=float, default=None, help="config 5 exit threshold")
    args = ap.parse_args()
    if args.scaling is None:
        args.scaling = "strong" if args.config == "4" else "weak"
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    if args.config == "5":
        return run_config5(args)
    if args.config == "4":
        return run_config4(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
