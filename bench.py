#!/usr/bin/env python3
"""Benchmark of the stick-breaking attention hot path (fwd + two-phase bwd) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[1], "C2"): B=8, H=16, L=4096, d=128 bf16, strictly
causal stick-breaking fwd+bwd, skip off (algorithmic FLOPs == executed tiles), per GPU.
(batch, head) units are independent: every rank runs its own C2
batch with no collective on the data path -> weak scaling; the only NCCL use is the
max-over-ranks of the timings.  One step = sb_fwd + sb_bwd (phase 1 + phase 2).

value   = whole-job tokens/s with inputs resident in HBM (CUDA events, max over ranks).
e2e     = the same metric through the public autograd op stickbreaking_attention()
          with q, k, v, dO copied host->device from pinned memory every step and the
          step's results (o, dq, dk, dv) read back device->host every step.
roofline = the dominant kernel's algorithmic tensor FLOPs per launch / its CUDA-event
          duration, against MEASURED_PEAKS.json bf16: the burst peak when the run held
          its SM clock at max without a power cap, else the sustained one (both
          fractions are reported).
cpu_baseline = the reference's own CPU path (baseline/_ref: its NumPy blocked_forward +
          blocked_backward_twophase, float32, one unit per host core) on a bounded sample
          of the same workload (rank 0, N=1 only); the C port in oracle/ when the
          reference is not installed.
--impl reference times that CPU path as the reference arm (no GPU work).
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

B, H, L, D = 8, 16, 4096, 128
METRIC = "stick-breaking attn fwd+bwd TFLOP/s & tokens/s at L=4096 d=128 bf16, 1/2/4/8 B200"
UNIT = "tokens/s"
WORKLOAD = "C2: B=8 H=16 L=4096 d=128 bf16 causal stick-breaking fwd+bwd per GPU, skip off"


def gemm_flops(b, h, l, d):
    """One causal GEMM over the triangle, FA convention: 2*d*(L^2/2) per unit."""
    return b * h * d * l * l


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["bf16_tflops"], p.get("bf16_tflops_sustained", p["bf16_tflops"]), "measured"
    except Exception:
        return 1590.0, 1400.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.thread is not None:
            self.thread.join(timeout=2)
        sm = [float(r[1]) for r in self.rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            if len(r) >= 9:
                for n, v in zip(names, r[5:9]):
                    if v.lower() == "active":
                        reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_sample(n_units=None, threads=None):
    """Time the C oracle (float32, all host threads) on n_units (b,h) units of C2."""
    import oracle
    threads = threads or oracle.n_threads_default()
    rng = np.random.default_rng(0)
    # one unit per host thread (units are independent), capped at the batch
    n_units = max(1, min(n_units or threads, B * H))
    q, k, v, d_o = (rng.standard_normal((n_units, L, D), dtype=np.float32) for _ in range(4))
    t0 = time.perf_counter()
    fwd = oracle.tiled_forward(q, k, v, block=64, dtype=np.float32, n_threads=threads)
    oracle.tiled_backward(q, k, v, d_o, fwd, block=64, dtype=np.float32, n_threads=threads)
    dt = time.perf_counter() - t0
    # tokens/s for the whole C2 batch (B*H units), units are independent and equal-cost
    t_full = dt * (B * H) / n_units
    return {"value": B * L / t_full, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{n_units} of {B * H} (b,h) units of C2 (L=4096, d=128), fp32 C port "
                      f"of blocked_forward+blocked_backward_twophase, {dt:.1f}s; scaled "
                      f"linearly to the full batch",
            "seconds_per_unit": dt / n_units}


REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def _ref_unit(seed):
    """One C2 (b, h) unit through the UNMODIFIED reference (baseline/_ref, installed from
    /root/reference/pkg): blocked_forward(two_phase=True) + blocked_backward_twophase in
    float32, its own NumPy code (blocked.py:129-206, :299-392).  Returns seconds."""
    from sbattn import blocked as bl
    rng = np.random.default_rng(seed)
    q, k, v, w = (rng.standard_normal((L, D)).astype(np.float32) for _ in range(4))
    lay = bl.plan_blocks(L)
    t0 = time.perf_counter()
    _, acc, st = bl.blocked_forward(q, k, v, lay, two_phase=True, dtype=np.float32)
    bl.blocked_backward_twophase(bl.make_cache(q, k, v, lay, acc, st), w, lay)
    return time.perf_counter() - t0


def _ref_unit_fused(seed):
    """The same unit through blocked_forward(two_phase=False) + blocked_backward_fused, the
    variant the reference's own `sb bench` times (cli.py:433-438).  Returns seconds."""
    from sbattn import blocked as bl
    rng = np.random.default_rng(seed)
    q, k, v, w = (rng.standard_normal((L, D)).astype(np.float32) for _ in range(4))
    lay = bl.plan_blocks(L)
    t0 = time.perf_counter()
    _, acc, st = bl.blocked_forward(q, k, v, lay, dtype=np.float32)
    bl.blocked_backward_fused(bl.make_cache(q, k, v, lay, acc, st), w, lay)
    return time.perf_counter() - t0


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _ref_init():
    sys.path.insert(0, REF_DIR)


class RefSampler:
    """The reference's own CPU path on all host cores: one unit per worker process
    (spawned, one BLAS thread each: the reference's own threading is slower than serial,
    SURVEY.md §8(a) `_map_ordered`).  None when baseline/_ref is not installed."""

    def __init__(self):
        self.pool = None
        if not os.path.isdir(os.path.join(REF_DIR, "sbattn")):
            return
        import multiprocessing as mp
        self.procs = os.cpu_count() or 1
        old = {k: os.environ.get(k) for k in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS")}
        os.environ["OPENBLAS_NUM_THREADS"] = os.environ["OMP_NUM_THREADS"] = "1"
        try:
            self.pool = mp.get_context("spawn").Pool(self.procs, initializer=_ref_init)
            self.pool.map(_ref_init_probe, range(self.procs))  # workers up, sbattn imported
        except Exception:
            self.pool = None
        for k_, v_ in old.items():
            if v_ is None:
                os.environ.pop(k_, None)
            else:
                os.environ[k_] = v_

    def sample(self, n_units=None, fused=False):
        n_units = max(1, min(n_units or self.procs, B * H))
        t0 = time.perf_counter()
        per = self.pool.map(_ref_unit_fused if fused else _ref_unit, range(n_units))
        dt = time.perf_counter() - t0
        t_full = dt * (B * H) / n_units
        if fused:
            return {"value": B * L / t_full, "seconds": dt}
        return {"value": B * L / t_full, "unit": UNIT, "cores": self.procs, "kind": "reference",
                "cpu": _cpu_model(),
                "sample": f"{n_units} of {B * H} (b,h) units of C2 (L=4096, d=128) through the "
                          f"reference's own blocked_forward(two_phase=True) + "
                          f"blocked_backward_twophase (NumPy, float32; baseline/_ref), one unit "
                          f"per process on {self.procs} host cores, {dt:.1f}s wall "
                          f"({statistics.median(per):.2f}s per unit); scaled linearly to the "
                          f"full batch", "seconds": dt}

    def close(self):
        if self.pool is not None:
            self.pool.terminate()


def _ref_init_probe(_):
    from sbattn import blocked  # noqa: F401
    return 0


def run_reference(args, rank, world):
    """Reference arm: the reference's own CPU implementation of the path on the host cores
    (baseline/_ref: its NumPy blocked_forward + blocked_backward_twophase), or the C port of
    it in oracle/ when the reference is not installed.

    One step = one bounded sample of C2: as many (b, h) units as host cores, each unit a
    full L=4096 d=128 fwd + two-phase bwd in f32.  value = tokens/s of that sample (units are
    independent and equal-cost, so it is the whole-batch rate); ms_per_step is the sample's
    measured wall time (not extrapolated)."""
    if rank != 0:
        return
    ref = RefSampler()
    if ref.pool is not None:
        def one():
            r = ref.sample(args.cpu_units or None)
            return r, r["seconds"]
        threads = ref.procs
        units = max(1, min(args.cpu_units or threads, B * H))
    else:
        import oracle
        oracle.build()
        threads = oracle.n_threads_default()
        units = max(1, min(args.cpu_units or threads, B * H))

        def one():
            r = cpu_sample(units, threads)
            return r, r["seconds_per_unit"] * units
    t_all = time.perf_counter()
    for _ in range(max(1, args.warmup)):  # same-size samples, untimed
        one()
        if time.perf_counter() - t_all > 60:
            break
    n_warm = _ + 1
    vals, secs = [], []
    t_all = time.perf_counter()
    for _ in range(max(1, args.steps)):
        s, sec = one()
        vals.append(s["value"])
        secs.append(sec)
        if time.perf_counter() - t_all > 150:
            break
    ref.close()
    value = statistics.median(vals)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": len(vals), "warmup": n_warm, "ms_per_step": statistics.median(secs) * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": WORKLOAD + " (CPU)",
                       "step": f"one sample of {units} of the {B * H} (b,h) units, one per host "
                               f"thread; tokens/s = units/{B * H} x {B * L} tokens / sample time"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": s["kind"],
                             "sample": s["sample"]},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-sdpa", action="store_true")
    ap.add_argument("--cpu-units", type=int, default=0, help="0: one per host thread")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    # one process per GPU; SB_BENCH_BACKEND=gloo lets a plumbing check run several ranks
    # on one GPU (ranks then share device local % device_count)
    backend = os.environ.get("SB_BENCH_BACKEND", "nccl")
    local_dev = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local_dev)
    dev = torch.device("cuda", local_dev)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    import paper_2410_17980_b200 as sb
    from paper_2410_17980_b200 import build as sbbuild

    if local == 0:
        sbbuild.build()
    if world > 1:
        dist.barrier()  # the other ranks load the library local rank 0 made current
    W = max(3, args.warmup)
    K = max(1, args.steps)

    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    q, k, v, d_o = (torch.randn(B, H, L, D, device=dev, dtype=torch.bfloat16, generator=g)
                    for _ in range(4))
    stream = torch.cuda.current_stream()

    # preallocated outputs and workspace so the timed region holds only our kernels
    def step(ev=None):
        o, log_rem, _, cache = sb.blocked_forward(q, k, v, counters=False)
        if ev is not None:
            ev[1].record(stream)
        sb.blocked_backward_twophase(cache, d_o, out=step.out, phases=1, workspace=step.ws)
        if ev is not None:
            ev[2].record(stream)
        sb.blocked_backward_twophase(cache, d_o, out=step.out, phases=2, workspace=step.ws)
        return o

    # the backward's transient workspace: M snapshots (phase 1 -> phase 2) + dZ tiles
    _, _, _, cache0 = sb.blocked_forward(q, k, v, counters=False)
    ws_bytes = sb.ops.workspace_bytes(cache0, store=True)
    state_bytes = cache0.state.numel() * 4
    del cache0
    step.ws = torch.empty(ws_bytes, device=dev, dtype=torch.uint8)
    step.out = tuple(torch.empty_like(q) for _ in range(3))
    M_bytes = sb.ops._lib.load().sb_snapshot_elems(
        __import__("ctypes").byref(sb.ops._params(q, 1.0 / math.sqrt(D), False, 1e-6))) * 4
    intermediates = {
        "saved_state_bytes": state_bytes, "M_bytes": M_bytes, "N_bytes": 0,
        "dZ_workspace_bytes": ws_bytes - M_bytes, "workspace_bytes": ws_bytes,
        "note": "forward -> backward: only the O(L) state (final a per row, float64) plus "
                "first_kb; the M snapshots are rolled back by phase 1 and live in the "
                "backward's transient workspace with the store mode's dZ tiles (bf16, O(L^2), "
                "written by phase 1, read by phase 2); no N; an inference forward (no autograd) "
                "writes no state"}

    for _ in range(W):
        step()
    torch.cuda.synchronize()

    clocks = ClockSampler(local_dev)
    clocks.start()
    time.sleep(0.3)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(K)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record(stream)
    for i in range(K):
        evs[i][0].record(stream)
        step(evs[i])
        evs[i][3].record(stream)
    t_end.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    total_ms = t_start.elapsed_time(t_end)
    fwd_ms = sum(e[0].elapsed_time(e[1]) for e in evs) / K
    p1_ms = sum(e[1].elapsed_time(e[2]) for e in evs) / K
    p2_ms = sum(e[2].elapsed_time(e[3]) for e in evs) / K
    t = torch.tensor([total_ms, fwd_ms, p1_ms, p2_ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms, fwd_ms, p1_ms, p2_ms = t.tolist()
    ms_step = total_ms / K
    tokens = world * B * L * K
    value = tokens / (total_ms / 1e3)

    G = gemm_flops(B, H, L, D)
    alg_flops = 7 * G  # fwd 2G + bwd 5G (FA convention)
    # executed: fwd 2G (QK^T, AV) + phase 1 3G (QK^T, dO V^T, dZ K) + phase 2: store mode
    # 3G (QK^T, A^T dO, dZ^T Q; dZ read from phase 1's tiles), recompute mode 4G
    store = True
    p2_exec = 3 * G
    exec_flops = 5 * G + p2_exec
    tflops = world * alg_flops * K / (total_ms / 1e3) / 1e12
    burst, sustained, peak_kind = load_peaks()
    # Denominator: the burst peak applies when this run held its clock (median SM clock
    # within 5% of max and no power cap), the sustained one (measured at a power-capped
    # 1327 MHz median) otherwise.  Both fractions are reported.
    held = (clk.get("sm_mhz") and clk.get("sm_max_mhz")
            and clk["sm_mhz"] >= 0.95 * clk["sm_max_mhz"] and "sw_power_cap" not in clk["reasons"])
    peak = burst if held else sustained
    kernels = {"sb_fwd_pp_kernel": (fwd_ms, 2 * G, 2 * G), "sb_bwd_q_kernel": (p1_ms, 3 * G, 3 * G),
               "sb_bwd_kvs_kernel": (p2_ms, 2 * G, p2_exec)}
    dom = max(kernels, key=lambda n: kernels[n][0])
    d_ms, d_alg, d_exec = kernels[dom]
    achieved = d_alg / (d_ms / 1e3) / 1e12
    roofline = {"bound": "tensor", "kernel": dom, "achieved": achieved, "peak": peak,
                "unit": "TFLOP/s", "frac": achieved / peak,
                "peak_kind": (f"{peak_kind} bf16 dense {'burst' if held else 'sustained'} "
                              f"(clock {'held at max, no power cap' if held else 'below max or power-capped'})"),
                "frac_burst": achieved / burst, "frac_sustained": achieved / sustained,
                "executed_tflops": d_exec / (d_ms / 1e3) / 1e12, "traffic": None,
                "per_kernel_ms": {n: round(v[0], 4) for n, v in kernels.items()},
                "per_kernel_frac_burst": {n: round(v[1] / (v[0] / 1e3) / 1e12 / burst, 4)
                                          for n, v in kernels.items()},
                "step_frac_of_peak": tflops / world / peak,
                "step_frac_burst": tflops / world / burst,
                "step_frac_sustained": tflops / world / sustained}
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            traffic = json.load(f)
        roofline["traffic"] = traffic.get(dom)
        # achieved DRAM rate per kernel: ncu bytes per launch (profiles/traffic.json, the
        # M snapshot and dZ tile round trip included) over this run's kernel time
        roofline["hbm_gbs_per_kernel"] = {n: round(traffic[n] / (v[0] / 1e3) / 1e9, 1)
                                          for n, v in kernels.items() if n in traffic}
    except Exception:
        pass
    # Secondary bound: the special-function unit.  MUFU operations per
    # score element from the kernels' SASS (per 64-column row of a tile: forward 65 ex2 +
    # 4 rcp + 2 lg2; phase 1 65 ex2 + 4 rcp + 2 lg2; phase 2 65 ex2 + 4 rcp), elements per
    # pass = tiles x 64 x 64 (diagonal tiles whole), at 16 per clock per SM.
    elems = B * H * (L // 64) * (L // 64 + 1) // 2 * 4096
    mufu = {"sb_fwd_pp_kernel": 71 / 64, "sb_bwd_q_kernel": 71 / 64, "sb_bwd_kvs_kernel": 69 / 64}
    sm_count = torch.cuda.get_device_properties(dev).multi_processor_count
    mhz = clk.get("sm_mhz") or clk.get("sm_max_mhz") or 1965.0
    mufu_rate = 16 * sm_count * mhz * 1e6  # ops/s
    roofline["sfu"] = {
        "unit": "MUFU ops/s", "peak": mufu_rate,
        "per_kernel_frac": {n: round(mufu[n] * elems / (kernels[n][0] / 1e3) / mufu_rate, 3)
                            for n in kernels if n in mufu},
        "step_floor_ms": sum(mufu.values()) * elems / mufu_rate * 1e3,
        "note": "16 MUFU ops/clk/SM at the run's median SM clock; ops per element from SASS"}

    # ---------------------------------------------------------------- e2e
    e2e = None
    if not args.no_e2e:
        # Inputs of every step come from pinned host memory; step i+1's H2D copy runs
        # on a copy stream while step i computes (double-buffered prefetch, as a data
        # loader would).  Each step's results (o, dq, dk, dv: 512 MiB) go back to
        # pinned host memory on a third stream, overlapped with the next step; the
        # timed region ends when the last step's results are on the host.
        hq, hk, hv, hdo = (x.cpu().pin_memory() for x in (q, k, v, d_o))
        hout = [[torch.empty(q.shape, dtype=q.dtype).pin_memory() for _ in range(4)]
                for _ in range(2)]
        h2d = sum(x.numel() * x.element_size() for x in (hq, hk, hv, hdo))
        d2h = sum(x.numel() * x.element_size() for x in hout[0])
        sets = [[torch.empty_like(q) for _ in range(4)] for _ in range(2)]
        copy_stream = torch.cuda.Stream(device=dev)
        back_stream = torch.cuda.Stream(device=dev)
        landed = [torch.cuda.Event() for _ in range(2)]      # q, k, v of set i on the device
        landed_do = [torch.cuda.Event() for _ in range(2)]   # dO of set i
        consumed = [torch.cuda.Event() for _ in range(2)]
        o_ready = [torch.cuda.Event() for _ in range(2)]
        computed = [torch.cuda.Event() for _ in range(2)]
        read_back = [torch.cuda.Event() for _ in range(2)]

        def prefetch(i):
            # q, k, v first (the forward needs only them), dO last (only the backward)
            with torch.cuda.stream(copy_stream):
                copy_stream.wait_event(consumed[i % 2])
                for buf, hx in zip(sets[i % 2][:3], (hq, hk, hv)):
                    buf.copy_(hx, non_blocking=True)
                landed[i % 2].record(copy_stream)
                sets[i % 2][3].copy_(hdo, non_blocking=True)
                landed_do[i % 2].record(copy_stream)

        def e2e_run(n):
            for c in consumed + read_back:
                c.record(stream)
            prefetch(0)
            for i in range(n):
                if i + 1 < n:
                    prefetch(i + 1)
                stream.wait_event(landed[i % 2])
                bq, bk, bv, bdo = sets[i % 2]
                qq, kk, vv = (x.requires_grad_(True) for x in (bq, bk, bv))
                o = sb.stickbreaking_attention(qq, kk, vv)
                o_ready[i % 2].record(stream)
                with torch.cuda.stream(back_stream):
                    # o leaves while the backward runs
                    back_stream.wait_event(o_ready[i % 2])
                    back_stream.wait_event(read_back[i % 2])  # host buffers of step i-2 free
                    hout[i % 2][0].copy_(o.detach(), non_blocking=True)
                    o.record_stream(back_stream)
                stream.wait_event(landed_do[i % 2])
                o.backward(bdo)
                res = (qq.grad, kk.grad, vv.grad)
                consumed[i % 2].record(stream)
                computed[i % 2].record(stream)
                with torch.cuda.stream(back_stream):
                    back_stream.wait_event(computed[i % 2])
                    for hx, x in zip(hout[i % 2][1:], res):
                        hx.copy_(x, non_blocking=True)
                        x.record_stream(back_stream)
                    read_back[i % 2].record(back_stream)
                for x in (qq, kk, vv):
                    x.grad = None
                    x.requires_grad_(False)
            stream.wait_stream(back_stream)

        e2e_run(2)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        Ke = max(3, min(2 * K, 20))  # steady state: the first H2D and last D2H are one step
        a, bev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        e2e_run(Ke)
        bev.record(stream)
        torch.cuda.synchronize()
        te = torch.tensor([a.elapsed_time(bev)], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": world * B * L * Ke / (te.item() / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": te.item() / Ke,
               "api": "stickbreaking_attention(q,k,v) + o.backward(dO); q,k,v,dO copied from "
                      "pinned host memory every step (next step's copy overlapped with this "
                      "step's compute on a copy stream, dO last); o (after the forward) and "
                      "dq,dk,dv copied back to pinned host memory every step on a third stream",
               "h2d_gbps": h2d * Ke / (te.item() / 1e3) / 1e9,
               "d2h_gbps": d2h * Ke / (te.item() / 1e3) / 1e9}

    # ---------------------------------------------------------------- comparators
    comparator = None
    if not args.no_sdpa and rank == 0:
        try:
            import torch.nn.functional as F
            qs, ks, vs = (x.detach().clone().requires_grad_(True) for x in (q, k, v))
            res = {}
            for name, ctx in (("cudnn", torch.nn.attention.SDPBackend.CUDNN_ATTENTION),
                              ("flash", torch.nn.attention.SDPBackend.FLASH_ATTENTION)):
                try:
                    with torch.nn.attention.sdpa_kernel([ctx]):
                        def sdpa_step():
                            o = F.scaled_dot_product_attention(qs, ks, vs, is_causal=True)
                            o.backward(d_o)
                        for _ in range(3):
                            sdpa_step()
                        torch.cuda.synchronize()
                        a2, b2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        a2.record()
                        for _ in range(5):
                            sdpa_step()
                        b2.record()
                        torch.cuda.synchronize()
                        res[name] = a2.elapsed_time(b2) / 5
                except Exception as ex:  # backend unavailable for this shape
                    res[name] = f"unavailable: {type(ex).__name__}"
            best = min((v for v in res.values() if isinstance(v, float)), default=None)
            comparator = {"softmax_sdpa_fwd_bwd_ms": res,
                          "ours_over_best_softmax": (ms_step / best) if best else None,
                          "note": "softmax attention keeps the inclusive diagonal; same shape"}
        except Exception as ex:
            comparator = {"error": repr(ex)}

    cpu = None
    if not args.no_cpu and rank == 0 and world == 1:
        try:
            ref = RefSampler()
            if ref.pool is not None:
                ref.sample(args.cpu_units or None)  # warm-up sample
                cpu = ref.sample(args.cpu_units or None)
                cpu.pop("seconds")
                # the fused-backward variant the reference's `sb bench` times, for scale
                cpu["fused_value"] = ref.sample(args.cpu_units or None, fused=True)["value"]
                ref.close()
                port = cpu_sample(args.cpu_units or None)
                cpu["port_value"] = port["value"]  # the C port of the same algorithm, for scale
            else:
                cpu = cpu_sample(args.cpu_units or None)
        except Exception as ex:
            cpu = {"error": repr(ex)}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
        "warmup": W, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": WORKLOAD, "batch_per_gpu": B, "heads": H, "seq_len": L,
                   "head_dim": D, "global_batch": B * world,
                   "parallelism": f"(b,h) units sharded, {world} independent ranks, no collective",
                   "l2": "inputs (4 x 128 MiB bf16 per rank) exceed the 126 MB L2; no flush",
                   "backward": "store mode (phase 1 writes dZ tiles, %.2f GB workspace)"
                            % (ws_bytes / 1e9)},
        "tflops": tflops, "tflops_note": "algorithmic 7*B*H*L^2*d per step (FA causal convention)",
        "executed_tflops": world * exec_flops * K / (total_ms / 1e3) / 1e12,
        "ms": {"fwd": fwd_ms, "bwd_phase1": p1_ms, "bwd_phase2": p2_ms},
        "roofline": roofline, "intermediates": intermediates, "cpu_baseline": cpu, "e2e": e2e,
        "gpu_launches": 3 * K,
        "clocks": clk, "comparator": comparator,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
