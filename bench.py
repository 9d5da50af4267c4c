#!/usr/bin/env python3
"""Benchmark of the B200 mini-batch gradient oracle (bench contract, one JSON line).

A step = one pass of the hot path over one batch: forward sweep + reverse
sweep + batch reduction (+ NCCL all-reduce of the d-vector when N > 1) + GD
update, i.e. one reference `train_step` over the batch.

Default workload: the headline, BASELINE.json configs[4] (cfg5: wide MLP
784-1024-1024-10, relu, softmax CE, fp32) at b = 1,048,576 — "b up to 1M,
sharded across 1/2/4/8 B200": the global batch is split across the ranks
(strong scaling), one all-reduce of the 1,863,690-parameter gradient per step.
`--config cfgN` selects another BASELINE config (weak scaling: each rank owns
`batch` samples); `--global-batch B` forces strong scaling with B samples.

Data: synthetic, the SURVEY.md §8d generators (mt19937_64 TestRng, seed 1234),
one global sample stream; rank r owns its contiguous shard of it.  Both arms
draw identical samples and parameters (the reference arm from oracle/_ref).

`--impl reference` times the reference's own CPU path (the unmodified
tapegrad headers built into oracle/_ref) on the host cores, same config and
samples; it never loads this package's library.
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

DATA_SEED = 1234      # both arms: the global sample stream
PARAM_SEED = 0        # both arms: make_params seed
METRIC = "per-sample gradient evals/sec (∇f_i/s)"

# tg_model ids (include/tg_abi.h), so the reference arm needs no product import
MODEL_IDS = {"fig1": 1, "listing1": 2, "moons": 3, "char_mlp": 4, "gpt": 5, "wide_mlp": 6}

# BASELINE.json configs.  flop = algorithmic flops per ∇f_i,
# bytes = compulsory per-sample HBM bytes (inputs + outputs the step writes),
# cpu_s = reference CPU seconds per sample on one core (bounds the CPU samples).
CONFIGS = {
    "cfg1": dict(model="fig1", dims=None, dtype="f64", batch=1_000_000, gamma=0.0, strong=False,
                 flop=25, bytes=40, bound="hbm", cpu_s=5e-7,
                 desc="Fig.1 tiny graph (10 nodes), fp64: f, df/da, df/db per sample"),
    "cfg2": dict(model="moons", dims=None, dtype="f64", batch=65_536, gamma=0.05, strong=False,
                 flop=1824, bytes=32, bound="fp64", cpu_s=1.2e-5,
                 desc="scalar MLP 2-16-16-1 tanh, hinge+1e-4 L2, fp64"),
    "cfg3": dict(model="char_mlp", dims=None, dtype="f32", batch=262_144, gamma=0.1, strong=False,
                 flop=68_400, bytes=20, bound="fp32", cpu_s=1.5e-4,
                 desc="char MLP 27/3/10/200 tanh, CE, fp32"),
    "cfg4": dict(model="gpt", dims=None, dtype="f32", batch=8192, gamma=0.1, strong=False,
                 flop=83_000_000, bytes=264, bound="tensor", cpu_s=0.25,
                 desc="mini GPT 65/64/64/4H/4L, fp32"),
    "cfg5": dict(model="wide_mlp", dims=None, dtype="f32", batch=1_048_576, gamma=0.1, strong=True,
                 flop=9_564_160, bytes=3144, bound="tensor", cpu_s=0.035,
                 desc="wide MLP 784-1024-1024-10 relu, CE, fp32"),
}


def shard(global_batch: int, rank: int, world: int):
    return global_batch * rank // world, global_batch * (rank + 1) // world


def plan(cfg, args, world: int, rank: int):
    """(local batch, global batch, first global sample of this rank, scaling)."""
    if args.global_batch or (cfg["strong"] and not args.batch):
        gb = args.global_batch or cfg["batch"]
        lo, hi = shard(gb, rank, world)
        return hi - lo, gb, lo, "strong"
    b = args.batch or cfg["batch"]
    return b, b * world, b * rank, "weak"


def config_dict(args, cfg, world: int, rank: int = 0):
    """The `config` object, identical in both arms."""
    b, gb, _, scaling = plan(cfg, args, world, rank)
    return {"workload": f"{args.config}: {cfg['desc']}", "global_batch": gb, "batch_per_gpu": b,
            "parallelism": f"dp{world}", "scaling": scaling, "data_seed": DATA_SEED, "param_seed": PARAM_SEED,
            "dtype": cfg["dtype"]}


def peaks():
    p = {"hbm_gbs": 6536.0, "bf16_tflops": 1639.9, "source": "fallback B200_PROFILING.md"}
    path = os.path.join(HERE, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            m = json.load(f)
        p.update({k: m[k] for k in ("hbm_gbs", "bf16_tflops", "bf16_tflops_sustained") if k in m})
        p["source"] = "MEASURED_PEAKS.json"
    return p


def _json(path):
    path = os.path.join(HERE, path)
    if os.path.exists(path):
        with open(path) as f:
            return json.load(f)
    return {}


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


# ---------------------------------------------------------------------------
# the reference's CPU path (oracle/_ref: the unmodified tapegrad headers)
# ---------------------------------------------------------------------------

def reference_inputs(cfg, samples: int):
    """Parameters and the first `samples` samples of the global stream, from
    oracle/_ref (never from the product library)."""
    import oracle
    m = MODEL_IDS[cfg["model"]]
    params = oracle.ref_params(m, cfg["dims"], cfg["dtype"], seed=PARAM_SEED)
    x, k = oracle.ref_synth(m, cfg["dims"], cfg["dtype"], DATA_SEED, samples)
    return params, x, k


def reference_cpu_step(cfg, params, x, k, threads: int, samples: int):
    """One reference train_step (per sample: rewind, re-record, zero_grads,
    backward_with_scratch, accumulate; then sgd_step) over `samples` samples;
    returns seconds."""
    import oracle
    xs = x[:, :samples] if x.size else x
    ks = k[:, :samples] if k.size else k
    t0 = time.perf_counter()
    r = oracle.ref_run(MODEL_IDS[cfg["model"]], cfg["dims"], cfg["dtype"], params, xs, ks, threads=threads)
    p2 = params.copy()
    oracle.sgd(cfg["dtype"], p2, r["grad_sum"], cfg["gamma"], samples)
    return time.perf_counter() - t0


def cpu_sample_size(cfg, threads: int, seconds: float, cap: int):
    return int(min(cap, max(threads, seconds * threads / cfg["cpu_s"])))


def run_reference_arm(args, cfg):
    """--impl reference: the reference CPU path, rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    if not oracle.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libtgref.so was not built"}), flush=True)
        return
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    threads = cpu_threads()
    b, gb, _, scaling = plan(cfg, args, world, 0)
    samples = cpu_sample_size(cfg, threads, 2.0, gb)          # ~2 s of wall time per step
    params, x, k = reference_inputs(cfg, samples)
    for _ in range(args.warmup):
        reference_cpu_step(cfg, params, x, k, threads, samples)
    ts = [reference_cpu_step(cfg, params, x, k, threads, samples) for _ in range(args.steps)]
    tot = sum(ts)
    value = samples * args.steps / tot
    line = {
        "metric": METRIC, "value": value, "unit": "grad/s", "impl": "reference", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
        "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": cfg["dtype"],
        "data": "synthetic (seeded mt19937_64 generators, SURVEY.md §8d; same samples as the GPU arm)",
        "config": config_dict(args, cfg, world),
        "cpu_baseline": {"value": value, "unit": "grad/s", "cores": threads, "kind": "reference",
                         "sample": f"each step: the first {samples} samples of the {gb}-sample global batch "
                                   f"(tapegrad::Tape per thread, oracle/_ref)"},
        "e2e": {"value": value, "unit": "grad/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# this implementation
# ---------------------------------------------------------------------------

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg5", choices=sorted(CONFIGS))
    ap.add_argument("--batch", type=int, default=0, help="per-GPU batch, weak scaling")
    ap.add_argument("--global-batch", type=int, default=0, help="global batch split across ranks, strong scaling")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "fused"],
                    help="N > 1: NCCL all-reduce + GD (tg_allreduce_gd_step) or the fused exchange + GD kernel over "
                         "NCCL symmetric memory (tg_window_allreduce_gd, NVLS multicast when available)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfg = dict(CONFIGS[args.config])
    if args.impl == "reference":
        run_reference_arm(args, cfg)
        return

    import torch
    import torch.distributed as dist
    import paper_2503_13795_b200 as tg
    from paper_2503_13795_b200.dp import NcclComm

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    comm = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        comm = NcclComm(rank, world)       # libtg's own communicator: tg_allreduce_gd_step
    dev = torch.device("cuda", local)
    tdt = torch.float64 if cfg["dtype"] == "f64" else torch.float32
    b, gb, first, scaling = plan(cfg, args, world, rank)

    desc = tg.build_model(cfg["model"], cfg["dims"], cfg["dtype"], seed=PARAM_SEED).describe()
    prog = tg.Program(desc)
    # this rank's shard of the global stream (mt19937: samples [0, first + b) drawn, the shard kept)
    xa, ka = tg.synth_batch(cfg["model"], cfg["dims"], cfg["dtype"], seed=DATA_SEED, batch=first + b,
                            n_inputs=desc.n_inputs, n_index=desc.n_index_inputs)
    x = np.ascontiguousarray(xa[:, first:]) if first else xa
    k = np.ascontiguousarray(ka[:, first:]) if first else ka
    del xa, ka
    params0 = desc.param_values()
    hbm_bound = cfg["bound"] == "hbm"
    # HBM-bound config: rotate over input/output sets whose total exceeds 2x L2,
    # back to back without a flush, so every step reads cold inputs and pays the
    # write-back of earlier steps' outputs (steady state); others: one set and
    # an L2 flush between timed steps
    set_bytes = b * cfg["bytes"]
    n_sets = max(1, min(16, -(-2 * 126 * 2**20 // max(set_bytes, 1)) + 1)) if hbm_bound else 1
    Xs = [torch.tensor(x, device=dev) if x.size else None for _ in range(n_sets)]
    Ks = [torch.tensor(k, device=dev) if k.size else None for _ in range(n_sets)]
    Ls = [torch.zeros(b, device=dev, dtype=tdt) for _ in range(n_sets)]
    IGs = [torch.zeros((desc.n_inputs, b), device=dev, dtype=tdt) if hbm_bound and desc.n_inputs else None
           for _ in range(n_sets)]
    X, K, L = Xs[0], Ks[0], Ls[0]
    P = torch.tensor(params0, device=dev, dtype=tdt)
    G = torch.zeros(max(desc.n_params, 1), device=dev, dtype=tdt)
    win = None
    if world > 1 and args.exchange == "fused" and desc.n_params:
        from paper_2503_13795_b200.dp import SymmetricWindow
        win = SymmetricWindow(comm, cfg["dtype"], desc.n_params)   # G is this rank's window buffer
        G = win.grad
    W = prog.alloc_workspace(b)
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)   # > 126 MB L2
    flush_rd = torch.ones(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MiB, read after the write
    flush_out = torch.empty((), dtype=torch.float32, device=dev)

    def flush_l2():
        # write 256 MiB (evicts the previous step's lines), then read another
        # 256 MiB so the write-back of those dirty lines happens here, outside
        # the timed region: the timed step starts on a cold, clean L2
        flush.zero_()
        torch.sum(flush_rd, dim=0, out=flush_out)

    def step(i=0, st=None, Xi=None, Ki=None):
        st = st or stream
        j = i % n_sets
        Xi = Xs[j] if Xi is None else Xi
        Ki = Ks[j] if Ki is None else Ki
        if hbm_bound:      # cfg1: no parameters; per-sample f and input gradients are the outputs
            prog.forward_backward(Xi, Ki, b, P, Ls[j], IGs[j], G, W, st)
        elif world == 1:   # fused: GD applied in the reduction epilogue
            prog.train_step(Xi, Ki, b, P, Ls[j], G, cfg["gamma"], W, st)
        else:              # local sum -> NCCL all-reduce of the d-vector -> GD with the global batch
            prog.forward_backward(Xi, Ki, b, P, Ls[j], None, G, W, st)
            if win is not None:
                win.allreduce_gd(P, cfg["gamma"], gb, st)
            else:
                prog.allreduce_gd_step(P, G, cfg["gamma"], gb, comm, st)

    l0 = prog.launches
    step()
    launches_per_step = prog.launches - l0
    torch.cuda.synchronize()
    prog.check_device_error()

    graphs = None
    chain = None
    if not args.no_graph:
        try:
            s2 = torch.cuda.Stream()
            s2.wait_stream(stream)
            with torch.cuda.stream(s2):
                for i in range(2):
                    step(i, st=s2)
            stream.wait_stream(s2)
            graphs = []
            for j in range(n_sets):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=s2):
                    step(j, st=s2)
                graphs.append(g)
            if hbm_bound:
                chain = torch.cuda.CUDAGraph()
                with torch.cuda.graph(chain, stream=s2):
                    for i in range(args.steps):
                        step(i, st=s2)
            torch.cuda.synchronize()
        except Exception as e:   # (capture unsupported: eager launches)
            print(f"cuda graph capture failed, eager launches: {e}", file=sys.stderr)
            graphs = None
            torch.cuda.synchronize()

    def run_step(i=0):
        if graphs is not None:
            graphs[i % n_sets].replay()
        else:
            step(i)

    for i in range(args.warmup):
        run_step(i)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        t_soak = time.perf_counter()        # clock soak (untimed, same work) so the sampler sees the load
        i = 0
        while time.perf_counter() - t_soak < 1.0:
            for _ in range(4):
                run_step(i)
                i += 1
            torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        for i in range(args.steps):
            if not hbm_bound:
                flush_l2()                      # L2 flushed between timed steps
            ev[i][0].record(stream)
            run_step(i)
            ev[i][1].record(stream)
        torch.cuda.synchronize()
        chain_ms = None
        if hbm_bound and chain is not None:
            # the K timed steps as ONE graph launch (K kernel nodes over the rotating
            # sets): the device runs them back to back, so the per-step time holds
            # no host launch / event gap.  This is the HBM-bound config's headline;
            # the launch-by-launch time above is reported beside it.
            chain.replay()
            torch.cuda.synchronize()
            c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            c0.record(stream)
            chain.replay()
            c1.record(stream)
            torch.cuda.synchronize()
            chain_ms = c0.elapsed_time(c1) / args.steps
        if world > 1:
            dist.barrier()
    step_ms = [a.elapsed_time(bb) for a, bb in ev]
    ms = sum(step_ms) / len(step_ms)
    ms_by_launch = ms
    if chain_ms is not None:
        ms = chain_ms
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = gb / (ms * 1e-3)

    # ---- dominant kernel time (CUDA events around the tape kernel, on the launch stream) ----
    cap = max(3, int(5000.0 / max(ms, 1e-3)))
    prog.profile(True)
    for i in range(min(max(args.steps // 4, 10), cap)):
        if not hbm_bound:
            flush_l2()
        step(i)
    tape_ms, tape_n = prog.profile_read()
    prog.profile(False)
    tape_ms = tape_ms / max(tape_n, 1)
    if graphs is not None and (prog.info["storage"] == 3 or launches_per_step == 1):
        # staged tier: the "kernel" is the whole chain of the step; a
        # one-launch step (cfg1) is the kernel itself.  The eager profiling
        # pass would also count host launch gaps (cfg1: 16.0 us profiled vs
        # 12.2 us per graph-replayed step), so they are timed by the step
        tape_ms = ms
    torch.cuda.synchronize()

    # ---- end to end through the public API: pinned host in, loss out ----
    e2e = None
    if not args.no_e2e:
        e2e = measure_e2e(args, cfg, prog, x, k, b, gb, P, L, stream, world, dev, tdt, cap, step)
    prog.check_device_error()

    # ---- on-device input pipeline ----
    dip = None
    if not args.no_e2e:
        dip = measure_device_pipeline(args, cfg, tg, prog, X, K, L, b, gb, first, rank, world, stream, dev, cap, run_step)
    prog.check_device_error()

    # ---- sequential-accumulation memory mode: the same step with a bounded workspace ----
    mem = None
    if prog.info["storage"] == 3 and not args.no_e2e:
        mem = measure_bounded_memory(prog, cfg, X, K, P, L, G, b, stream, world)
    prog.check_device_error()

    # ---- roofline of the dominant kernel ----
    pk = peaks()
    info = prog.info
    fp = _json("profiles/fp_peaks.json")
    mma = _json("profiles/mma_peaks.json")
    if hbm_bound:
        alg = b * cfg["bytes"]
        achieved = alg / (tape_ms * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / pk["hbm_gbs"], "algorithmic_bytes_per_launch": alg,
                "peak_source": f"{pk['source']} hbm_gbs (burst copy)",
                "timing": f"{n_sets} rotating input/output sets ({n_sets * set_bytes / 2**20:.0f} MiB > 2x L2), "
                          "back to back: each launch reads cold inputs and pays earlier launches' write-backs"}
    else:
        alg = b * cfg["flop"]
        achieved = alg / (tape_ms * 1e-3) / 1e12
        if cfg["bound"] == "tensor":
            # dense products on tcgen05 as 3xTF32 (three kind::tf32 MMAs per fp32
            # product): roof = measured kind::tf32 rate / 3.  The step is a long
            # chain timed inside back-to-back steps: the sustained rate applies.
            if mma.get("tf32_tcgen05_tflops_sustained"):
                t_peak = mma["tf32_tcgen05_tflops_sustained"] / 3
                src = (f"profiles/mma_peaks.json tcgen05 kind::tf32 sustained {mma['tf32_tcgen05_tflops_sustained']} "
                       f"TF/s (burst {mma.get('tf32_tcgen05_tflops')}) / 3 (3xTF32 passes)")
            else:
                t_peak = pk.get("bf16_tflops_sustained", pk["bf16_tflops"]) / 2 / 3
                src = f"{pk['source']} bf16 sustained / 2 (TF32 rate, not measured) / 3 (3xTF32 passes)"
            roof = {"bound": "tensor", "achieved": achieved, "peak": t_peak, "unit": "TFLOP/s",
                    "frac": achieved / t_peak, "algorithmic_flops_per_launch": alg, "peak_source": src,
                    "frac_of_burst_roof": (achieved / (mma["tf32_tcgen05_tflops"] / 3)) if mma.get("tf32_tcgen05_tflops") else None}
        else:
            fp_peak = fp.get({"f64": "fp64_tflops", "f32": "fp32_tflops"}[cfg["dtype"]])
            roof = {"bound": cfg["bound"], "achieved": achieved, "peak": fp_peak, "unit": "TFLOP/s",
                    "frac": achieved / fp_peak if fp_peak else None, "algorithmic_flops_per_launch": alg,
                    "peak_source": "profiles/fp_peaks.json (FMA-throughput microbenchmark on a B200, tools/fp_peak.cu)"}
        roof["hbm_achieved_gbs"] = b * cfg["bytes"] / (tape_ms * 1e-3) / 1e9
    tier = ["smem-interpreter", "hbm-interpreter", "jit-register", "staged"][info["storage"]]
    roof["kernel"] = {"smem-interpreter": "tgk::k_tape<T,true>", "hbm-interpreter": "tgk::k_tape<T,false>",
                      "jit-register": "tg_jit_tape (NVRTC sm_100a)",
                      "staged": "staged chain: k_umma_pair / k_umma_tma_p (tcgen05 3xTF32, TMA-fed) + level / attention kernels"}[tier]
    roof["kernel_ms"] = tape_ms
    roof["kernel_share_of_step"] = tape_ms / ms
    roof["traffic"], roof["traffic_source"] = measured_traffic(args.config, b)

    line = {
        "metric": METRIC, "value": value, "unit": "grad/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": scaling, "vs_baseline": None,
        "dtype": cfg["dtype"], "data": "synthetic (seeded mt19937_64 generators, SURVEY.md §8d; same samples as the reference arm)",
        "config": config_dict(args, cfg, world),
        "l2": ("rotating buffer sets > 2x L2, back to back" if hbm_bound else
               "flushed between timed steps (256 MiB write, then 256 MiB read so no dirty lines remain)"),
        "timed_as": ("one graph launch of the K steps (K kernel nodes back to back); launch by launch: %.4f ms per step"
                     % ms_by_launch) if chain_ms is not None else "one graph launch (or eager call) per step",
        "cuda_graph": graphs is not None, "kernel_tier": tier, "tile_samples": info["tile_samples"],
        "exchange": ("none (one rank: GD fused in the reduction epilogue)" if world == 1 else
                     "tg_allreduce_gd_step (NCCL all-reduce + GD)" if win is None else
                     "tg_window_allreduce_gd (fused, %s)" % ("NVLS multimem" if win.multimem else "NVLink peer loads")),
        "node_evals_per_s": value * (info["n_sample_nodes"] + info["n_uniform_nodes"] / max(b, 1)),
        "roofline": roof,
        "gpu_launches": launches_per_step * args.steps,
        "e2e": e2e,
        "device_input_pipeline": dip,
        "memory": mem,
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"], line["cpu_baseline_1core"] = cpu_baselines(cfg, b)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if win is not None:
        win.close()
    if comm is not None:
        comm.close()
    if world > 1:
        dist.destroy_process_group()


def measure_e2e(args, cfg, prog, x, k, b, gb, P, L, stream, world, dev, tdt, cap, step):
    """The same metric through the public host-buffer API: each step's inputs
    from pinned host memory, its per-sample losses back to host memory."""
    import torch
    import torch.distributed as dist
    xh = torch.from_numpy(x).pin_memory() if x.size else None
    kh = torch.from_numpy(k).pin_memory() if k.size else None
    lh = torch.empty(b, dtype=tdt).pin_memory()
    h2d = (xh.numel() * xh.element_size() if xh is not None else 0) + (kh.numel() * 4 if kh is not None else 0)
    d2h = b * lh.element_size()
    hbm_bound = cfg["bound"] == "hbm"
    pipe = prog.pipeline(b, P, stream) if world == 1 and not hbm_bound else None
    Xd = torch.empty(x.shape, dtype=tdt, device=dev) if pipe is None and x.size else None
    Kd = torch.empty(k.shape, dtype=torch.int32, device=dev) if pipe is None and k.size else None
    def e2e_step():
        if pipe is not None:   # tg_pipeline_step: H2D / compute / D2H overlapped across steps
            pipe.step(xh, kh, lh, cfg["gamma"])
            return
        if Xd is not None:
            Xd.copy_(xh, non_blocking=True)
        if Kd is not None:
            Kd.copy_(kh, non_blocking=True)
        step(0, Xi=Xd, Ki=Kd)
        lh.copy_(L, non_blocking=True)      # the step's per-sample losses (set 0)

    t_w = time.perf_counter()
    n_w = 0
    while n_w < max(args.warmup, 10) or time.perf_counter() - t_w < float(os.environ.get("TG_E2E_SOAK", "1.5")):
        e2e_step()
        n_w += 1
        if pipe is not None and n_w % 16 == 0:
            pipe.sync()
    if pipe is not None:
        pipe.sync()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n_e2e = min(max(args.steps, 100), cap)
    e0.record(stream)
    for _ in range(n_e2e):
        e2e_step()
    if pipe is not None:
        pipe.join(stream)      # e1 after the last step's loss has reached host memory
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / n_e2e
    # the same step's host<->device copies alone (no compute): the link bound of e2e
    Xc = torch.empty(x.shape, dtype=tdt, device=dev) if x.size else None
    Kc = torch.empty(k.shape, dtype=torch.int32, device=dev) if k.size else None
    cs_in, cs_out = torch.cuda.Stream(), torch.cuda.Stream()
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n_c = min(n_e2e, 50)
    torch.cuda.synchronize()
    c0.record(stream)
    cs_in.wait_stream(stream)
    cs_out.wait_stream(stream)
    for _ in range(n_c):
        with torch.cuda.stream(cs_in):
            if Xc is not None:
                Xc.copy_(xh, non_blocking=True)
            if Kc is not None:
                Kc.copy_(kh, non_blocking=True)
        with torch.cuda.stream(cs_out):
            lh.copy_(L, non_blocking=True)
    stream.wait_stream(cs_in)
    stream.wait_stream(cs_out)
    c1.record(stream)
    torch.cuda.synchronize()
    copy_ms = c0.elapsed_time(c1) / n_c
    if world > 1:
        t = torch.tensor([e2e_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    del pipe
    return {"value": gb / (e2e_ms * 1e-3), "unit": "grad/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "ms_per_step": e2e_ms, "copies_only_ms_per_step": copy_ms,
            "h2d_link_gbs": h2d / (copy_ms * 1e-3) / 1e9 if h2d else None,
            "api": ("tg_pipeline_step (pinned host inputs in, per-sample losses out, 4 steps in flight)"
                    if world == 1 and not hbm_bound else
                    "copies + tg_forward_backward (+ tg_allreduce_gd_step over NCCL at N > 1)")}


def measure_bounded_memory(prog, cfg, X, K, P, L, G, b, stream, world, budget=4 << 30, steps=3):
    """The staged tier with its rows bounded to `budget` bytes per chunk
    (tg_set_memory_budget): workspace and step time beside the default
    one-chunk run — peak device memory independent of b."""
    import torch
    full = prog.workspace_size(b)
    full_chunk = prog.chunk_samples(b)
    prog.set_memory_budget(budget)
    try:
        ws = prog.workspace_size(b)
        chunk = prog.chunk_samples(b)
        W2 = torch.empty(max(ws, 1), dtype=torch.uint8, device=P.device)
        P2 = P.clone()
        G2 = torch.empty_like(G)
        for _ in range(2):
            prog.train_step(X, K, b, P2, L, G2, cfg["gamma"], W2, stream)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            prog.train_step(X, K, b, P2, L, G2, cfg["gamma"], W2, stream)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        del W2, P2, G2
    finally:
        prog.set_memory_budget(0)
    return {"default": {"workspace_gb": full / 1e9, "chunk_samples": full_chunk},
            "bounded": {"budget_gb": budget / 2**30, "workspace_gb": ws / 1e9, "chunk_samples": chunk,
                        "chunks": -(-b // chunk), "ms_per_step": ms, "value": b / (ms * 1e-3),
                        "note": "same step, rows streamed chunk by chunk into one grad_sum (tg_set_memory_budget); "
                                "L2 not flushed between these steps"}}


def measure_device_pipeline(args, cfg, tg, prog, X, K, L, b, gb, first, rank, world, stream, dev, cap, run_step):
    """Each step's batch generated on the GPU (tg_synth_ctr_device, fresh
    counter-based samples every step), then the step, then the losses to
    pinned host memory through two device slots on a copy stream."""
    import torch
    import torch.distributed as dist

    def synth_into(i):
        tg.synth_ctr_device(cfg["model"], X, K, cfg["dims"], cfg["dtype"], seed=2000,
                            first=i * gb + first, batch=b, stream=stream)

    cps = torch.cuda.Stream(device=dev)
    Lslot = [torch.empty_like(L) for _ in range(2)]
    lhs = [torch.empty(L.shape, dtype=L.dtype).pin_memory() for _ in range(2)]
    slot_free = [None, None]

    def dev_step(i):
        synth_into(i)
        run_step(0)
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
    stream.wait_stream(cps)
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
    return {"value": gb / (dev_ms * 1e-3), "unit": "grad/s", "ms_per_step": dev_ms, "synth_ms_per_step": synth_ms,
            "h2d_bytes_per_step": 0, "d2h_bytes_per_step": b * L.element_size(),
            "api": "tg_synth_ctr_device (fresh counter-based samples each step) + the step + "
                   "losses to pinned host memory (copy stream, two slots)"}


def cpu_baselines(cfg, b):
    """The reference CPU path on this host: all cores, and one core (the
    paper's protocol), each on a bounded sample."""
    import oracle
    if not oracle.ref_available():
        return None, None
    threads = cpu_threads()
    out = []
    for th, secs in ((threads, 8.0), (1, 4.0)):
        samples = cpu_sample_size(cfg, th, secs, b)
        params, x, k = reference_inputs(cfg, samples)
        reference_cpu_step(cfg, params, x, k, th, min(samples, th * 2))   # warm-up
        dt = reference_cpu_step(cfg, params, x, k, th, samples)
        out.append({"value": samples / dt, "unit": "grad/s", "cores": th, "kind": "reference",
                    "sample": f"the first {samples} samples of the batch, one reference train_step "
                              f"(oracle/_ref: unmodified tapegrad headers, one Tape per thread)"})
    return out[0], out[1]


def measured_traffic(config: str, batch: int):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant
    kernel (the whole staged chain for the staged configs) from the committed
    ncu capture (profiles/traffic.json), scaled to this batch."""
    d = _json("profiles/traffic.json").get(config)
    if not d:
        return None, None
    return d["dram_bytes_per_launch"] * batch / d["batch"], d.get("source")


if __name__ == "__main__":
    main()
