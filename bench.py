#!/usr/bin/env python3
"""Benchmark of the B200 mini-batch gradient oracle (bench contract, one JSON line).

A step = one pass of the hot path over one batch: forward sweep + reverse
sweep + batch reduction (+ NCCL all-reduce of the d-vector when N > 1) + GD
update, i.e. one reference `train_step` over the batch.

Default workload: BASELINE.json configs[1] (cfg2, scalar-node MLP 2-16-16-1,
fp64, hinge + 1e-4 L2, b = 65,536).  `--config cfgN` selects another.
Multi-GPU: one process per GPU (torchrun), each rank owns `batch` samples
(weak scaling), one all-reduce of the gradient per step.

`--impl reference` times the reference's own CPU path (the unmodified
tapegrad headers built into oracle/_ref) on the host cores, same config.
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

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

# BASELINE.json configs.  flop = algorithmic flops per ∇f_i,
# bytes = compulsory per-sample HBM bytes (inputs + loss).
CONFIGS = {
    "cfg1": dict(model="fig1", dims=None, dtype="f64", batch=1_000_000, gamma=0.0,
                 flop=25, bytes=40, bound="hbm", desc="Fig.1 tiny graph (10 nodes), fp64"),
    "cfg2": dict(model="moons", dims=None, dtype="f64", batch=65_536, gamma=0.05,
                 flop=1824, bytes=32, bound="fp64", desc="scalar MLP 2-16-16-1 tanh, hinge+1e-4 L2, fp64"),
    "cfg3": dict(model="char_mlp", dims=None, dtype="f32", batch=262_144, gamma=0.1,
                 flop=68_400, bytes=20, bound="fp32", desc="char MLP 27/3/10/200 tanh, CE, fp32"),
    "cfg4": dict(model="gpt", dims=None, dtype="f32", batch=8192, gamma=0.1,
                 flop=83_000_000, bytes=264, bound="tensor", desc="mini GPT 65/64/64/4H/4L, fp32"),
    "cfg5": dict(model="wide_mlp", dims=None, dtype="f32", batch=1_048_576, gamma=0.1,
                 flop=9_564_160, bytes=3144, bound="tensor", desc="wide MLP 784-1024-1024-10 relu, CE, fp32"),
}


def peaks():
    p = {"hbm_gbs": 6536.0, "bf16_tflops": 1639.9, "source": "fallback B200_PROFILING.md"}
    path = os.path.join(HERE, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            m = json.load(f)
        p.update({k: m[k] for k in ("hbm_gbs", "bf16_tflops", "bf16_tflops_sustained") if k in m})
        p["source"] = "MEASURED_PEAKS.json"
    return p


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled while the timed region runs."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [s.strip() for s in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def reference_cpu_step(cfg, desc, x, k, params, threads, samples):
    """The reference's own per-sample path on `samples` samples; returns seconds."""
    import oracle
    from paper_2503_13795_b200.tape import model_id
    xs = x[:, :samples] if x.size else x
    ks = k[:, :samples] if k.size else k
    t0 = time.perf_counter()
    if oracle.ref_available():
        r = oracle.ref_run(model_id(cfg["model"]), cfg["dims"], cfg["dtype"], params, xs, ks, threads=threads)
        kind = "reference"
    else:
        r = oracle.run(desc, xs, ks, params, threads=threads)
        kind = "port"
    g = r["grad_sum"]
    p2 = params.copy()
    oracle.sgd(cfg["dtype"], p2, g, cfg["gamma"], samples)
    return time.perf_counter() - t0, kind


def run_reference_arm(args, cfg):
    """--impl reference: the reference CPU path, rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import paper_2503_13795_b200 as tg
    desc = tg.build_model(cfg["model"], cfg["dims"], cfg["dtype"], seed=0).describe()
    threads = cpu_threads()
    # bounded sample per step: ~ a few seconds of CPU work per step at most
    per_sample_s = {"cfg1": 5e-7, "cfg2": 1.2e-5, "cfg3": 1.5e-4, "cfg4": 0.25, "cfg5": 0.035}[args.config]
    samples = int(min(cfg["batch"], max(threads, 2.0 * threads / per_sample_s)))
    x, k = tg.synth_batch(cfg["model"], cfg["dims"], cfg["dtype"], seed=1234, batch=samples,
                          n_inputs=desc.n_inputs, n_index=desc.n_index_inputs)
    params = desc.param_values()
    for _ in range(args.warmup):
        reference_cpu_step(cfg, desc, x, k, params, threads, samples)
    ts = []
    kind = "reference"
    for _ in range(args.steps):
        dt, kind = reference_cpu_step(cfg, desc, x, k, params, threads, samples)
        ts.append(dt)
    tot = sum(ts)
    value = samples * args.steps / tot
    line = {
        "metric": "per-sample gradient evals/sec (∇f_i/s)", "value": value, "unit": "grad/s",
        "impl": "reference", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": {"f64": "f64", "f32": "f32"}[cfg["dtype"]], "data": "synthetic",
        "config": {"workload": f"{args.config}: {cfg['desc']}", "batch_per_step": samples,
                   "full_batch": cfg["batch"]},
        "cpu_baseline": {"value": value, "unit": "grad/s", "cores": threads, "kind": kind,
                         "sample": f"{samples} samples of {args.config} per step (full batch {cfg['batch']})"},
        "e2e": {"value": value, "unit": "grad/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--batch", type=int, default=0, help="per-GPU batch (default: the config's)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfg = dict(CONFIGS[args.config])
    if args.batch:
        cfg["batch"] = args.batch
    if args.impl == "reference":
        run_reference_arm(args, cfg)
        return

    import torch
    import torch.distributed as dist
    import paper_2503_13795_b200 as tg

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    tdt = torch.float64 if cfg["dtype"] == "f64" else torch.float32
    b = cfg["batch"]

    desc = tg.build_model(cfg["model"], cfg["dims"], cfg["dtype"], seed=0).describe()
    prog = tg.Program(desc)
    x, k = tg.synth_batch(cfg["model"], cfg["dims"], cfg["dtype"], seed=1000 + rank, batch=b,
                          n_inputs=desc.n_inputs, n_index=desc.n_index_inputs)
    params0 = desc.param_values()
    X = torch.tensor(x, device=dev) if x.size else None
    K = torch.tensor(k, device=dev) if k.size else None
    P = torch.tensor(params0, device=dev, dtype=tdt)
    L = torch.zeros(b, device=dev, dtype=tdt)
    G = torch.zeros(max(desc.n_params, 1), device=dev, dtype=tdt)
    W = prog.alloc_workspace(b)
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)   # > 126 MB L2
    flush_rd = torch.ones(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MiB, read after the write
    flush_out = torch.empty((), dtype=torch.float32, device=dev)

    def flush_l2():
        # write 256 MiB (evicts the previous step's lines), then read another
        # 256 MiB so the write-back of those dirty lines happens here, outside
        # the timed region: the timed step starts on a cold, clean L2 (the
        # state ncu's cache control gives a profiled kernel)
        flush.zero_()
        torch.sum(flush_rd, dim=0, out=flush_out)

    from paper_2503_13795_b200.dp import DataParallelStep
    dp = DataParallelStep(prog)

    def step(Xs=X, Ks=K, st=None):
        st = st or stream
        if world == 1:   # fused: GD applied in the reduction epilogue
            prog.train_step(Xs, Ks, b, P, L, G, cfg["gamma"], W, st)
        else:            # local sum -> NCCL all-reduce of the d-vector -> GD with the global batch
            prog.forward_backward(Xs, Ks, b, P, L, None, G, W, st)
            dp.step(P, G, cfg["gamma"], b * world, stream=st)

    l0 = prog.launches
    step()
    launches_per_step = prog.launches - l0
    torch.cuda.synchronize()
    prog.check_device_error()

    graph = None
    if world == 1 and not args.no_graph:
        s2 = torch.cuda.Stream()
        s2.wait_stream(stream)
        with torch.cuda.stream(s2):
            for _ in range(2):
                step(st=s2)
        stream.wait_stream(s2)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=s2):
            step(st=s2)
        torch.cuda.synchronize()

    def run_step():
        if graph is not None:
            graph.replay()
        else:
            step()

    for _ in range(args.warmup):
        run_step()
    # clock soak (untimed, same work) so the sampler sees the load
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        t_soak = time.perf_counter()
        while time.perf_counter() - t_soak < 1.0:
            for _ in range(20):
                run_step()
            torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        for i in range(args.steps):
            flush_l2()                          # L2 flushed between timed steps
            ev[i][0].record(stream)
            run_step()
            ev[i][1].record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    step_ms = [a.elapsed_time(bb) for a, bb in ev]
    ms = sum(step_ms) / len(step_ms)
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = b * world / (ms * 1e-3)

    # ---- dominant kernel time (CUDA events around the tape kernel) ----
    # long steps (cfg4 / cfg5 at full batch): bounded extra passes (~5 s each)
    cap = max(3, int(5000.0 / max(ms, 1e-3)))
    prog.profile(True)
    for _ in range(min(max(args.steps // 4, 10), cap)):
        flush_l2()
        step()
    tape_ms, tape_n = prog.profile_read()
    prog.profile(False)
    tape_ms = tape_ms / max(tape_n, 1)
    if prog.info["storage"] == 3 and graph is not None:
        # staged tier: the "kernel" is the whole chain of the step; the eager
        # profiling pass would also count host launch gaps between its kernels,
        # so the chain is timed by the graph-replayed step itself
        tape_ms = ms

    # ---- end to end through the public API: pinned host in, loss out ----
    xh = torch.from_numpy(x).pin_memory() if x.size else None
    kh = torch.from_numpy(k).pin_memory() if k.size else None
    lh = torch.empty(b, dtype=tdt).pin_memory()
    Xd = torch.empty_like(X) if X is not None else None
    Kd = torch.empty_like(K) if K is not None else None
    h2d = (xh.numel() * xh.element_size() if xh is not None else 0) + (kh.numel() * 4 if kh is not None else 0)
    d2h = b * L.element_size()

    pipe = prog.pipeline(b, P, stream) if world == 1 else None

    def e2e_step():
        if pipe is not None:   # public host-buffer API: H2D / compute / D2H overlapped across steps
            pipe.step(xh, kh, lh, cfg["gamma"])
            return
        if Xd is not None:
            Xd.copy_(xh, non_blocking=True)
        if Kd is not None:
            Kd.copy_(kh, non_blocking=True)
        step(Xd, Kd)
        lh.copy_(L, non_blocking=True)

    # warm-up until steady state: the host-copy path ramps up over ~1 s of
    # traffic on this box (measured: 127 -> 37 us/step across 1,600 steps)
    t_w = time.perf_counter()
    n_w = 0
    while n_w < max(args.warmup, 10) or time.perf_counter() - t_w < float(os.environ.get("TG_E2E_SOAK", "1.5")):
        e2e_step()
        n_w += 1
        if pipe is not None and n_w % 64 == 0:
            pipe.sync()
    if pipe is not None:
        pipe.sync()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n_e2e = min(max(args.steps, 100), cap)
    windows = []
    for _ in range(int(os.environ.get("TG_E2E_WINDOWS", "1"))):
        e0.record(stream)
        for _ in range(n_e2e):
            e2e_step()
        if pipe is not None:
            pipe.join(stream)      # e1 after the last step's loss has reached host memory
        e1.record(stream)
        torch.cuda.synchronize()
        windows.append(e0.elapsed_time(e1) / n_e2e)
    if len(windows) > 1:
        print("e2e windows (ms/step):", [round(w, 4) for w in windows], file=sys.stderr)
    e2e_ms = windows[0]
    # the same step's host<->device copies alone (no compute): the link bound of e2e
    cs_in, cs_out = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c0.record(stream)
    cs_in.wait_stream(stream)
    cs_out.wait_stream(stream)
    for _ in range(n_e2e):
        with torch.cuda.stream(cs_in):
            if Xd is not None:
                Xd.copy_(xh, non_blocking=True)
            if Kd is not None:
                Kd.copy_(kh, non_blocking=True)
        with torch.cuda.stream(cs_out):
            lh.copy_(L, non_blocking=True)
    stream.wait_stream(cs_in)
    stream.wait_stream(cs_out)
    c1.record(stream)
    torch.cuda.synchronize()
    copy_ms = c0.elapsed_time(c1) / n_e2e
    if world > 1:
        t = torch.tensor([e2e_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    prog.check_device_error()

    # ---- on-device input pipeline: each step's batch is
    # generated on the GPU (tg_synth_ctr_device, fresh samples every step, the
    # bits of the host generator tg_synth_ctr), then the step, then the losses
    # back to pinned host memory: no input bytes cross PCIe ----
    def synth_into(i):
        tg.synth_ctr_device(cfg["model"], X, K, cfg["dims"], cfg["dtype"], seed=2000,
                            first=(i * world + rank) * b, batch=b, stream=stream)

    # losses leave through two device slots on a copy stream, so step i+1's
    # generation and compute overlap step i's device->host copy
    cps = torch.cuda.Stream(device=dev)
    Lslot = [torch.empty_like(L) for _ in range(2)]
    lhs = [lh, torch.empty_like(lh).pin_memory()]
    slot_free = [None, None]

    def dev_step(i):
        synth_into(i)
        run_step()
        j = i & 1
        if slot_free[j] is not None:
            stream.wait_event(slot_free[j])
        Lslot[j].copy_(L, non_blocking=True)
        cps.wait_stream(stream)
        with torch.cuda.stream(cps):
            lhs[j].copy_(Lslot[j], non_blocking=True)
            slot_free[j] = torch.cuda.Event()
            slot_free[j].record(cps)

    for i in range(args.warmup):
        dev_step(i)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    n_dev = min(max(args.steps, 20), cap)
    d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    d0.record(stream)
    for i in range(n_dev):
        dev_step(args.warmup + i)
    stream.wait_stream(cps)                # the last step's losses are in host memory
    d1.record(stream)
    torch.cuda.synchronize()
    dev_ms = d0.elapsed_time(d1) / n_dev
    g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g0.record(stream)
    for i in range(n_dev):
        synth_into(i)
    g1.record(stream)
    torch.cuda.synchronize()
    synth_ms = g0.elapsed_time(g1) / n_dev
    if world > 1:
        t = torch.tensor([dev_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_ms = float(t.item())
    prog.check_device_error()

    # ---- roofline of the dominant kernel ----
    pk = peaks()
    info = prog.info
    if cfg["bound"] == "hbm":
        alg = b * cfg["bytes"]
        achieved = alg / (tape_ms * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / pk["hbm_gbs"], "traffic": None,
                "algorithmic_bytes_per_launch": alg, "peak_source": pk["source"]}
    else:
        alg = b * cfg["flop"]
        achieved = alg / (tape_ms * 1e-3) / 1e12
        fp_peak = measured_simt_peak(cfg["dtype"])
        roof = {"bound": cfg["bound"], "achieved": achieved, "peak": fp_peak, "unit": "TFLOP/s",
                "frac": achieved / fp_peak if fp_peak else None, "traffic": None,
                "algorithmic_flops_per_launch": alg,
                "peak_source": "profiles/fp_peaks.json (FMA-throughput microbenchmark on this B200)",
                "hbm_achieved_gbs": b * cfg["bytes"] / (tape_ms * 1e-3) / 1e9}
        if cfg["bound"] == "tensor" and cfg["dtype"] == "f32":
            # dense products on tcgen05 as 3xTF32 (three kind::tf32 MMAs per fp32
            # product): the roof is the measured dense bf16 peak / 2 (TF32 rate) / 3
            t_peak = pk["bf16_tflops"] / 2 / 3
            roof.update({"peak": t_peak, "frac": achieved / t_peak,
                         "peak_source": f"{pk['source']} bf16 dense {pk['bf16_tflops']} TF/s / 2 (TF32) / 3 (3xTF32 passes)",
                         "frac_of_fp32_fma_peak": achieved / fp_peak if fp_peak else None})
    tier = ["smem-interpreter", "hbm-interpreter", "jit-register", "staged"][info["storage"]]
    roof["kernel"] = {"smem-interpreter": "tgk::k_tape<T,true>", "hbm-interpreter": "tgk::k_tape<T,false>",
                      "jit-register": "tg_jit_tape (NVRTC sm_100a)",
                      "staged": "staged chain: k_umma_tma (tcgen05 3xTF32, TMA-fed) / k_tape_range"}[tier]
    roof["kernel_ms"] = tape_ms
    roof["kernel_share_of_step"] = tape_ms / ms
    roof["traffic"] = measured_traffic(args.config, b)

    line = {
        "metric": "per-sample gradient evals/sec (∇f_i/s)", "value": value, "unit": "grad/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": cfg["dtype"], "data": "synthetic (seeded mt19937_64 generators, SURVEY.md §8d)",
        "config": {"workload": f"{args.config}: {cfg['desc']}", "batch_per_gpu": b, "global_batch": b * world,
                   "parallelism": f"dp{world}", "l2": "flushed between timed steps (256 MiB write, then 256 MiB read so no dirty lines remain)",
                   "cuda_graph": graph is not None, "tile_samples": info["tile_samples"],
                   "kernel_tier": tier},
        "node_evals_per_s": value * (info["n_sample_nodes"] + info["n_uniform_nodes"] / max(b, 1)),
        "roofline": roof,
        "gpu_launches": launches_per_step * args.steps,
        "e2e": {"value": b * world / (e2e_ms * 1e-3), "unit": "grad/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms,
                "copies_only_ms_per_step": copy_ms,
                "h2d_link_gbs": h2d / (copy_ms * 1e-3) / 1e9 if h2d else None,
                "api": ("tg_pipeline_step (pinned host inputs in, per-sample losses out, 4 steps in flight)"
                        if pipe is not None else "copies + tg_forward_backward + NCCL all-reduce + tg_gd_update")},
        "device_input_pipeline": {"value": b * world / (dev_ms * 1e-3), "unit": "grad/s", "ms_per_step": dev_ms,
                                  "synth_ms_per_step": synth_ms, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": d2h,
                                  "api": "tg_synth_ctr_device (fresh counter-based samples each step) + the step + "
                                         "losses to pinned host memory (copy stream, two slots)"},
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = cpu_threads()
        per = {"cfg1": 5e-7, "cfg2": 1.2e-5, "cfg3": 1.5e-4, "cfg4": 0.25, "cfg5": 0.035}[args.config]
        samples = int(min(b, max(threads, 10.0 * threads / per)))
        dt, kind = reference_cpu_step(cfg, desc, x, k, params0, threads, samples)
        line["cpu_baseline"] = {"value": samples / dt, "unit": "grad/s", "cores": threads, "kind": kind,
                                "sample": f"{samples} samples of {args.config}, one reference train_step"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def measured_traffic(config: str, batch: int):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant
    kernel from the committed ncu --set full capture (profiles/traffic.json),
    scaled to this batch; None when not captured for this config."""
    path = os.path.join(HERE, "profiles", "traffic.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        d = json.load(f).get(config)
    if not d:
        return None
    return d["dram_bytes_per_launch"] * batch / d["batch"]


def measured_simt_peak(dtype: str):
    """FMA-throughput peak measured on this GPU (profiles/fp_peaks.json, written
    by scripts/fp_peak.py); None when not measured yet."""
    path = os.path.join(HERE, "profiles", "fp_peaks.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return d.get({"f64": "fp64_tflops", "f32": "fp32_tflops"}[dtype])
    return None


if __name__ == "__main__":
    main()
