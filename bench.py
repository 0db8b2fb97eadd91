#!/usr/bin/env python
"""Benchmark of the GPipe hot path (BASELINE.json metric: training samples/sec, m = 32).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl tgp|reference]
    python -m torch.distributed.run --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 \
        --master-port P bench.py --gpus N --steps K --warmup W

Workload (BASELINE.json configs[1], "C2"): 32 pre-LN residual MLP blocks, width 4096 (GELU,
LayerNorm), global batch 512, m = 32 micro-batches of 16 rows, checkpoint = except_last (the
paper's default, P:108 / P:305 fn), bf16 operands with fp32 accumulation, plain SGD, MSE loss on
synthetic N(0,1) data.  N GPUs = N partitions of 32/N blocks (one process per GPU, partitions
connected through CUDA-IPC receive arenas); total work fixed -> "scaling": "strong".

A step = tgp_forward + tgp_mse_loss_grad + tgp_backward_step (all GPipe tasks: F, F', B, W with the
SGD update fused into it, copies; --unfused-sgd: tgp_backward + tgp_step).  `value` is timed with
CUDA events on the device with inputs resident in HBM;
`e2e` additionally copies x / target host->device (pinned) every step and reads the loss back.
The 2.15 GB of bf16 weights streamed per step exceed the 126 MB L2, so no explicit L2 flush.
`--impl reference` times the fp64 CPU oracle (oracle/) on a bounded sample of the same workload.
"""
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

BLOCKS, WIDTH, BATCH, M_CHUNKS = 32, 4096, 512, 32
METRIC = "training samples/sec (m=32)"
UNIT = "samples/s"


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return None


class ClockSampler:
    """Samples nvidia-smi clocks / throttle reasons during the timed region (the recipe's clocks line).
    Every line is stamped with its host arrival time; only samples inside [begin(), end()] (+ one
    sampling period of lag) are reported."""

    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.sw_power_cap", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown"]
    PERIOD_MS = 100

    def __init__(self, dev):
        self.dev = dev
        self.proc = None
        self.lines = []
        self.t0 = self.t1 = None

    def start(self):
        """Start sampling and wait (<= 3 s) for the first sample, so the timed region is covered."""
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", str(self.PERIOD_MS)], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            deadline = time.time() + 3.0
            while not self.lines and time.time() < deadline:
                time.sleep(0.02)
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def begin(self):
        self.t0 = time.time()

    def end(self):
        self.t1 = time.time()

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(self.PERIOD_MS / 1000.0)  # the sample covering the end of the window
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        lag = self.PERIOD_MS / 1000.0
        t0 = self.t0 if self.t0 is not None else 0.0
        t1 = (self.t1 if self.t1 is not None else time.time()) + lag
        sm, mx, reasons = [], [], set()
        names = ["sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"]
        for ts, ln in self.lines:
            if not (t0 <= ts <= t1):
                continue
            p = [q.strip() for q in ln.split(",")]
            if len(p) < 6:
                continue
            try:
                sm.append(float(p[0]))
                mx.append(float(p[1]))
            except ValueError:
                continue
            for nm, v in zip(names, p[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm), "period_ms": self.PERIOD_MS}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    lrank = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, lrank


def _host_info():
    """CPU model, BLAS implementation / version and its thread count (threadpoolctl)."""
    model = None
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    blas, threads = None, os.cpu_count()
    try:
        from threadpoolctl import threadpool_info
        info = [i for i in threadpool_info() if i.get("user_api") == "blas"]
        if info:
            blas = f"{info[0].get('internal_api')} {info[0].get('version')}"
            threads = max(int(i.get("num_threads", 0)) for i in info)
    except Exception:
        pass
    return model, blas, threads


def cpu_oracle_sample(steps=3, batch=64, width=WIDTH):
    """Time the fp64 oracle (as it stands) on a bounded sample of C2: the FULL 32-block model at full
    width on `batch` of the 512 rows (the oracle is full-batch: its cost is linear in the rows, so
    samples/s does not depend on the sample size).  Median of `steps` timed steps after one untimed.
    Returns (samples/s, threads, description, median step seconds)."""
    from oracle import model as OM
    from synth import configs as C
    from synth import gen as G

    layers = C.resmlp_stack(BLOCKS, width)
    x, t = G.inputs(layers, batch, seed=1234, dtype="bf16")
    params = G.params(layers, seed=1234, dtype="bf16")
    model, blas, threads = _host_info()
    OM.train_step(layers, params, x, t, lr=0.05, m=M_CHUNKS, want_dx=False)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        OM.train_step(layers, params, x, t, lr=0.05, m=M_CHUNKS, want_dx=False)
        times.append(time.perf_counter() - t0)
    per_step = statistics.median(times)
    desc = (f"oracle.model.train_step (numpy fp64), the full {BLOCKS}-block model at width {width} on {batch} of the "
            f"{BATCH} rows (m={M_CHUNKS}); median of {steps} steps ({per_step:.2f} s each) after one untimed; "
            f"CPU: {model}; BLAS: {blas}, {threads} threads")
    return batch / per_step, threads, desc, per_step


def run_reference(args):
    ws, rank, _ = _dist()
    if rank != 0:
        return
    # each step = the full 32-block model on a bounded sample of the batch (64 of 512 rows, ~2 s on 16
    # cores): ms_per_step is what was timed, so a --steps K run of this arm fits its wall time
    v, cores, desc, per_step = cpu_oracle_sample(steps=max(1, args.steps), batch=args.ref_rows)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * per_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": _config(args.gpus),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _config(n, m=M_CHUNKS, ckpt="except_last"):
    return {"workload": f"C2: {BLOCKS}-block pre-LN residual MLP (width {WIDTH}, GELU, LayerNorm), global batch "
                        f"{BATCH}, m={m}, checkpoint={ckpt}, plain SGD, MSE",
            "global_batch": BATCH, "micro_batch_rows": BATCH // m, "chunks": m, "checkpoint": ckpt, "partitions": n,
            "parallelism": f"pp{n}", "seq_len": None,
            "l2": "no flush: 2.15 GB of bf16 weights streamed per step exceed the 126 MB L2"}


def run_tgp(args):
    import torch
    import torch.distributed as dist

    from paper_2004_09910_b200 import Pipeline
    from synth import configs as C

    ws, rank, lrank = _dist()
    n = ws
    if args.gpus != n and ws > 1:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE {ws}")
    if ws > 1:
        dist.init_process_group("gloo")
    # one GPU per rank; on a box with fewer GPUs than ranks (code-path tests only) ranks share devices
    lrank = lrank % max(1, torch.cuda.device_count())
    torch.cuda.set_device(lrank)
    dev = torch.device("cuda", lrank)
    layers = C.resmlp_stack(BLOCKS, WIDTH)
    devices = [-1] * n
    devices[rank] = lrank
    free0 = torch.cuda.mem_get_info(dev)[0]
    bal = [BLOCKS // n + (1 if j < BLOCKS % n else 0) for j in range(n)]
    P = Pipeline(layers, chunks=args.chunks, devices=devices, balance=bal, checkpoint=args.checkpoint,
                 max_batch=BATCH, dtype="bf16", seed=1234)
    if ws > 1:
        from paper_2004_09910_b200.dist import connect_pipeline
        connect_pipeline(P, rank, ws)
    for kv in args.opt:
        k, v = kv.split("=")
        P.set_option(k, int(v))
    P.init_params(seed=1234)
    free1 = torch.cuda.mem_get_info(dev)[0]
    mem = P.memory(rank)
    first, last = rank == 0, rank == n - 1
    g = torch.Generator(device="cpu").manual_seed(1234)
    x_h = torch.randn(BATCH, WIDTH, generator=g).pin_memory()
    t_h = torch.randn(BATCH, WIDTH, generator=g).pin_memory()
    X = x_h.to(dev) if first else None
    T = t_h.to(dev) if last else None
    Y = torch.empty(BATCH, WIDTH, device=dev) if last else None
    DY = torch.empty(BATCH, WIDTH, device=dev) if last else None

    def step(e2e=False):
        if e2e:
            if first:
                X.copy_(x_h, non_blocking=True)
            if last:
                T.copy_(t_h, non_blocking=True)
            torch.cuda.current_stream().synchronize()
        P.forward(X, BATCH, Y)
        loss = P.mse_loss_grad(Y, T, BATCH, DY) if last else None  # loss is read back to the host
        if args.unfused_sgd:
            P.backward(DY, None)
            P.step(args.lr)
        else:
            P.backward_step(DY, args.lr)
        return loss

    def barrier():
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def timed(k, e2e, clk=None):
        barrier()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(k + 1)]
        k0 = P.kernel_count()
        if clk:
            clk.begin()
        ev[0].record()
        losses = []
        for q in range(k):
            losses.append(step(e2e))
            ev[q + 1].record()
        ev[k].synchronize()
        if clk:
            clk.end()
        ms = ev[0].elapsed_time(ev[k])
        per = [ev[q].elapsed_time(ev[q + 1]) for q in range(k)]
        nk = P.kernel_count() - k0
        barrier()
        if ws > 1:
            from paper_2004_09910_b200.dist import max_over_ranks
            ms = max_over_ranks(ms)
            per = [max_over_ranks(v) for v in per]
        return ms, nk, losses, per

    for _ in range(args.warmup):
        step()
    clk = ClockSampler(lrank)
    clk.start()
    free_t0 = torch.cuda.mem_get_info(dev)[0]
    ms, nk, losses, per_step = timed(args.steps, False, clk)
    free_t1 = torch.cuda.mem_get_info(dev)[0]
    clocks = clk.stop()
    e2e_ms, _, _, _ = timed(args.steps, True)

    # one traced step (after the timed ones): per-task device intervals -> busy / bubble fraction of
    # this partition's compute stream (busy_j against m / (m + n - 1)) and task times
    P.set_trace(True)
    barrier()
    P.forward(X, BATCH, Y)
    if last:
        P.mse_loss_grad(Y, T, BATCH, DY)
    if args.unfused_sgd:
        P.backward(DY, None)
    else:
        P.backward_step(DY, args.lr)
    tl = P.timeline()
    P.set_trace(False)
    if args.unfused_sgd:
        P.step(args.lr)
    # compute lanes: stream 0 (every task) and 3 (F' paired beside B on a second lane)
    comp = tl[(tl[:, 0] == rank) & ((tl[:, 1] == 0) | (tl[:, 1] == 3))]
    kinds = {0: "F", 1: "F'", 2: "B", 7: "W"}
    task_us = {}
    for kd, nm in kinds.items():
        d = (comp[comp[:, 2] == kd][:, 5] - comp[comp[:, 2] == kd][:, 4]) / 1e3
        if len(d):
            task_us[nm] = {"n": int(len(d)), "median_us": float(np.median(d)), "sum_ms": float(d.sum() / 1e3)}
    busy_ns, end = 0, None  # union of the compute intervals (paired tasks overlap)
    for a0, a1 in sorted((int(r[4]), int(r[5])) for r in comp):
        if end is None or a0 > end:
            busy_ns += a1 - a0
            end = a1
        elif a1 > end:
            busy_ns += a1 - end
            end = a1
    busy_ms = busy_ns / 1e6

    # dominant kernel: forward weight-streaming GEMM, timed live on its stream (cycling cold weights)
    # dominant kernel: the persistent weight-streaming task kernel (F task of micro-batch 1: 2 GEMMs
    # per block, weights streamed from HBM), timed live on the partition's compute stream
    stream = P.stream_enabled(rank)
    gemm_ms, gemm_bytes, gemm_n = P.bench_dominant_gemm(rank, BATCH, reps=10 if stream else 3)
    mrows = BATCH // args.chunks
    kname = (f"task_stream_kernel F task ({BLOCKS // n} blocks x 2 weight-streaming GEMMs, M={mrows} rows, d=H={WIDTH})"
             if stream else f"{'gemm_wide_kernel' if mrows >= 256 else 'gemm_tc_kernel'} forward W1 GEMM "
             f"(M={mrows} rows, K=N={WIDTH})")
    peaks = _peaks()
    if peaks and "hbm_gbs" in peaks:
        peak, peak_src = float(peaks["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    else:
        peak, peak_src = 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"
    achieved = gemm_bytes / (gemm_ms * 1e-3) / 1e9
    traffic = None  # DRAM bytes per launch of the same kernel from the committed ncu --set full capture
    if stream:
        try:
            # captured on the 32-block (n = 1) F task; per block the traffic is the same
            traffic = json.load(open(os.path.join(ROOT, "profiles", "stream_traffic.json")))["dram_bytes_per_launch"]
            traffic *= (BLOCKS // n) / BLOCKS
        except Exception:
            traffic = None
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        v, cores, desc, _ = cpu_oracle_sample(steps=3, batch=args.cpu_rows)
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc}
    # per GEMM class, three fractions: achieved TFLOP/s / bf16 peak, achieved DRAM GB/s /
    # HBM peak, and achieved / the class's own roofline min(TC peak, AI x HBM)
    tc_peak = float(peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops", 1385.9))) if peaks else 1385.9
    nb, d_, m_ = BLOCKS // n, WIDTH, BATCH // args.chunks

    def fractions(flop, dram_bytes, sec):
        tf, gbs = flop / sec / 1e12, dram_bytes / sec / 1e9
        roof = min(tc_peak, (flop / dram_bytes) * peak / 1e3)  # TFLOP/s
        return {"tflops": tf, "frac_tc": tf / tc_peak, "dram_gbs": gbs, "frac_hbm": gbs / peak,
                "frac_own_roofline": tf / roof}
    gemm_fr = {}
    if stream:
        gemm_fr["stream_F_task"] = fractions(nb * 2 * 2.0 * m_ * d_ * d_, gemm_bytes, gemm_ms * 1e-3)
    if "W" in task_us:
        # deferred dW: 2 GEMMs per block of 4096 x 4096 x B, bf16 operands; unfused: fp32 dW out;
        # fused with SGD: fp32 master read + write and bf16 shadow write (10 B/param), no dW out
        wflop = nb * 2 * 2.0 * d_ * d_ * BATCH
        wbytes = nb * 2 * (2.0 * BATCH * d_ * 2 + (4.0 if args.unfused_sgd else 10.0) * d_ * d_)
        gemm_fr["wgrad_task" if args.unfused_sgd else "wgrad_sgd_task"] = fractions(wflop, wbytes,
                                                                                   task_us["W"]["median_us"] * 1e-6)
    if rank == 0:
        sps = BATCH * args.steps / (ms * 1e-3)
        line = {
            "metric": METRIC, "value": sps, "unit": UNIT, "n_gpus": n, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "step_ms": {"p10": float(np.percentile(per_step, 10)), "p50": float(np.percentile(per_step, 50)),
                        "p90": float(np.percentile(per_step, 90))},
            "pipeline": {"busy": busy_ms / (ms / args.steps), "bubble": 1.0 - busy_ms / (ms / args.steps),
                         "ideal_busy": args.chunks / (args.chunks + n - 1), "tasks": task_us,
                         "note": "busy = union of this rank's compute-task intervals (both lanes) in one traced step / ms_per_step"},
            "gemm_fractions": gemm_fr,
            "dtype": "bf16", "data": "synthetic (N(0,1) inputs/targets, on-device U(+-1/sqrt(fan_in)) init)",
            "config": _config(n, args.chunks, args.checkpoint),
            "e2e": {"value": BATCH * args.steps / (e2e_ms * 1e-3), "unit": UNIT,
                    "h2d_bytes_per_step": 4 * BATCH * WIDTH * 2, "d2h_bytes_per_step": 8},
            "gpu_launches": int(nk),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic, "kernel": kname,
                         "algorithmic_bytes_per_launch": gemm_bytes, "avg_launch_us": gemm_ms * 1e3,
                         "launches_timed": gemm_n, "peak_source": peak_src},
            "clocks": clocks,
            "memory": {"plan_used_gb": mem["used"] / 1e9, "plan_reserved_gb": mem["reserved"] / 1e9,
                       "params_gb": mem["params"] / 1e9, "device_delta_gb": (free0 - free1) / 1e9,
                       "step_alloc_gb": (free_t0 - free_t1) / 1e9, "note": "per partition; all device memory is allocated in "
                       "tgp_create (device_delta = cudaMemGetInfo before/after create incl. CUDA context "
                       "growth), nothing on the step path"},
            "loss_first_last": [losses[0], losses[-1]] if losses and losses[0] is not None else None,
        }
        if cpu:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    P.close()
    if ws > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="tgp", choices=["tgp", "reference"])
    ap.add_argument("--checkpoint", default="except_last", choices=["always", "except_last", "never"])
    ap.add_argument("--chunks", type=int, default=M_CHUNKS, help="m (BASELINE metric: 32; other values = C3 sweep)")
    ap.add_argument("--lr", type=float, default=0.05)
    ap.add_argument("--ref-rows", type=int, default=64, help="reference arm: rows of the full-model oracle sample")
    ap.add_argument("--cpu-rows", type=int, default=128, help="cpu_baseline: rows of the full-model oracle sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--unfused-sgd", action="store_true", help="tgp_backward + tgp_step instead of tgp_backward_step")
    ap.add_argument("--opt", action="append", default=[], help="runtime option name=value (tgp_set_option)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_tgp(args)


if __name__ == "__main__":
    main()
