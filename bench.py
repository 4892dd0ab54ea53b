"""Benchmark of the ISA attention layer (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[2], the config the metric is quoted on):
one ISA attention layer at 32K source + 32K context tokens, Wan-14B shape
(B=1, H=40, D=128), bf16, default knobs (alpha_s=0.125, alpha_ns=0.0625,
alpha_f=0.5, b=64), synthetic i.i.d. N(0,1) Q/K/V (seeded). Inputs are 2 GB,
larger than the 126 MB L2, so no explicit flush is needed between steps.

One step = one full isa_forward (all five stages, routing included) over the
heads this rank owns. N > 1: heads are sharded round-robin over ranks and the
outputs are reassembled with an NCCL all-gather (paper_2605_04569_b200.parallel);
value = max over ranks of the step time (strong scaling: the layer is fixed).

Prints ONE JSON line on rank 0. `--impl reference` times the reference
algorithm on the host CPU instead (the oracle port of the pure-Python
reference, run on a bounded sample and extrapolated).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ISA attn-layer latency (ms) & TFLOPS at 2x32K tokens vs dense attn; GPU scaling"
WORKLOAD = dict(workload="cfg3: ISA attention layer, Wan-14B shape, 32K source + 32K context",
                batch=1, heads=40, head_dim=128, l_src=32768, l_ctx=32768, block=64,
                alpha_s=0.125, alpha_ns=0.0625, alpha_f=0.5,
                inputs="iid N(0,1) bf16 drawn per head h on the GPU (torch.Generator seed 1000 + h; Q, K, V "
                       "in that order: bench.synth_qkv)")


# BASELINE.json configs: the metric is quoted on cfg3 (the default); the others
# run through the same harness with --config (cfg4-grid adds the knob sweep).
CONFIGS = {
    "cfg1": dict(workload="cfg1: the reference's CPU-runnable case (B=1, H=2, d=64, 1024 + 1024 tokens)",
                 heads=2, head_dim=64, l_src=1024, l_ctx=1024),
    "cfg2": dict(workload="cfg2: single ISA layer, Wan-14B shape, 8K source + 8K context",
                 heads=40, head_dim=128, l_src=8192, l_ctx=8192),
    "cfg3": dict(workload=WORKLOAD["workload"], heads=40, head_dim=128, l_src=32768, l_ctx=32768),
    "cfg4": dict(workload="cfg4: ISA layer at 16K source + 16K context (default knobs; cfg4-grid sweeps "
                          "alpha_s x alpha_f against dense)", heads=40, head_dim=128, l_src=16384, l_ctx=16384),
    "cfg5": dict(workload="cfg5: one LIVEditor-14B-shaped layer, 50,000 + 50,000 tokens (ragged segments)",
                 heads=40, head_dim=128, l_src=50000, l_ctx=50000),
}
CFG4_GRID = dict(alpha_s=(0.0625, 0.125, 0.25, 0.5, 1.0), alpha_f=(0.0, 0.25, 0.5, 0.75))


def synth_qkv(heads, S, D, dev):
    """The bench's synthetic inputs for the listed heads: per head h an
    independent torch.Generator(seed 1000 + h) on `dev` draws Q, K, V (S, D)
    fp32 N(0, 1), rounded to bf16. Returns (1, len(heads), S, D) bf16 tensors.
    Per-head seeding makes a rank's shard identical to slicing the full
    tensor, and lets tests/test_gpu_shipped.py regenerate any head."""
    import torch

    q = torch.empty((1, len(heads), S, D), dtype=torch.bfloat16, device=dev)
    k, v = torch.empty_like(q), torch.empty_like(q)
    for j, h in enumerate(heads):
        g = torch.Generator(device=dev).manual_seed(1000 + h)
        for t in (q, k, v):
            t[0, j].copy_(torch.randn((S, D), generator=g, device=dev, dtype=torch.float32).to(torch.bfloat16))
    return q, k, v


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS) + ["cfg4-grid"], default="cfg3")
    ap.add_argument("--heads", type=int, default=None)
    ap.add_argument("--l-src", type=int, default=None)
    ap.add_argument("--l-ctx", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-full", action="store_true", help="reference arm: every head, every query block")
    ap.add_argument("--no-extras", action="store_true", help="skip dense/SDPA/e2e side measurements")
    args = ap.parse_args()
    c = CONFIGS["cfg4" if args.config == "cfg4-grid" else args.config]
    args.heads = args.heads or c["heads"]
    args.l_src = args.l_src if args.l_src is not None else c["l_src"]
    args.l_ctx = args.l_ctx if args.l_ctx is not None else c["l_ctx"]
    args.head_dim = c["head_dim"]
    args.workload = dict(WORKLOAD, workload=c["workload"], heads=args.heads, head_dim=args.head_dim,
                         l_src=args.l_src, l_ctx=args.l_ctx)
    return args


# --------------------------------------------------------------------------- CPU (reference algorithm)
def cpu_sample(l_src, l_ctx, heads, D=128, fraction=1 / 16, seed=0, heads_run=1):
    """Time the reference algorithm (oracle port, numpy/BLAS on all host cores)
    on `heads_run` heads of the workload: routing (stages 1-3) in full,
    attention on a `fraction` of the query blocks; extrapolate to all heads
    (the reference runs heads serially: reference.py:159-160, taylor.py:176-177).
    heads_run = heads and fraction = 1 is the full workload, no extrapolation."""
    import numpy as np

    from oracle import isa_oracle as O

    rng = np.random.default_rng(seed)
    S = l_src + l_ctx
    route = attn = 0.0
    for _ in range(heads_run):
        q, k, v = (O.round_bf16(rng.standard_normal((1, 1, S, D), dtype=np.float32)) for _ in range(3))
        t0 = time.perf_counter()
        asm = O.OracleAssembly(q, k, v, l_src, l_ctx)
        t1 = time.perf_counter()
        asm.forward(block_fraction=fraction)
        t2 = time.perf_counter()
        route += t1 - t0
        attn += t2 - t1
    per_head = (route + attn / fraction) / heads_run
    return per_head * heads * 1e3, dict(route_s=route, attn_sample_s=attn, heads_run=heads_run, fraction=fraction)


def cpu_plan(args):
    """Bounded CPU sample per config: (heads_run, fraction). cfg1 runs in full;
    --cpu-full runs every head and every query block of any config."""
    if args.cpu_full or args.config == "cfg1":
        return args.heads, 1.0
    if args.config == "cfg2":
        return 2, 1.0
    return 1, 1 / 16


def cpu_cores():
    try:
        from threadpoolctl import threadpool_info

        info = threadpool_info()
        n = max((i.get("num_threads", 1) for i in info), default=os.cpu_count())
        return int(n), [i.get("internal_api") for i in info]
    except Exception:
        return os.cpu_count(), []


def run_reference(args, rank, world):
    if rank != 0:
        return
    heads_run, fraction = cpu_plan(args)
    vals = []
    for i in range(args.warmup + args.steps):
        ms, detail = cpu_sample(args.l_src, args.l_ctx, args.heads, D=args.head_dim, fraction=fraction,
                                heads_run=heads_run)
        if i >= args.warmup:
            vals.append(ms)
    value = statistics.median(vals)
    cores, apis = cpu_cores()
    sample = _sample_text(args, heads_run, fraction, apis)
    line = {
        "metric": METRIC, "value": value, "unit": "ms", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": value, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
        "config": dict(args.workload, parallelism="cpu",
                       inputs="iid N(0,1) rounded to bf16 values (numpy default_rng, fp32 -> fp64 arithmetic)"),
        "cpu_baseline": {"value": value, "unit": "ms", "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _sample_text(args, heads_run, fraction, apis):
    full = heads_run == args.heads and fraction == 1.0
    what = (f"{heads_run} of {args.heads} heads: routing (stages 1-3) in full + attention on "
            f"{'all' if fraction == 1.0 else f'1/{round(1 / fraction)} of the'} query blocks")
    return (what + ("" if full else f", extrapolated to {args.heads} heads")
            + f" (oracle port of the pure-Python reference; numpy fp64 over {apis})")


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_rank{index}.csv")

    def start(self):
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.fh.close()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for name, flag in zip(names, parts[4:8]):
                if flag.lower() == "active":
                    reasons.add(name)
        load = [s for s in sm if s > 0.5 * max(sm)] if sm else []
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------------------- GPU
def run_ours(args, rank, world, local_rank):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2605_04569_b200 as P
    from paper_2605_04569_b200 import _native as N
    from paper_2605_04569_b200.parallel import ShardedIsa, head_shard

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    H, D = args.heads, args.head_dim
    S = args.l_src + args.l_ctx
    icl = P.IclLayout(args.l_src, args.l_ctx)
    cfg = P.IsaConfig(strict=(args.l_src % 64 == 0 and args.l_ctx % 64 == 0))  # ragged segments (cfg5) allowed
    my_heads = head_shard(H, rank, world)
    Hl = len(my_heads)
    # Each rank synthesises only its own heads (round-robin): identical to
    # slicing the full (1,H,S,D) inputs because heads are drawn per head.
    q, k, v = synth_qkv(my_heads, S, D, dev)
    dims = P.IsaDims.derive((1, H, S, D), icl, cfg)
    flops = dims.flops()
    f_isa = flops.total()
    f_dense = flops.dense_equivalent_mas
    f_sharp = 4 * 64 * 64 * D * dims.n_sharp * dims.t_new * 1 * Hl
    f_taylor_alg = (4 * 64 * 64 * D * dims.n_flat * dims.k + 4 * 64 * D * dims.n_flat * (dims.t_new - dims.k)) * Hl

    out_full = torch.empty((1, H, S, D), dtype=torch.bfloat16, device=dev) if world > 1 else None
    prep = P.prepare(q, k, v, icl, cfg)
    # N > 1: one fused call over the local heads publishing per-head completion;
    # head c's NCCL all-gather waits on its counter and runs under the later heads
    shard_mode = os.environ.get("ISA_SHARD_MODE", "signal")
    sharded = ShardedIsa(q, k, v, icl, cfg, world, mode=shard_mode) if world > 1 else None

    # per-kernel CUDA events recorded by the C ABI inside every timed step
    # (N = 1): the stage / roofline durations come from the timed region itself
    step_evs = [[torch.cuda.Event(enable_timing=True) for _ in range(6)] for _ in range(args.steps)]
    step_structs = []
    for evl in step_evs:
        es = N.IsaEvents()
        for j_, e_ in enumerate(evl):
            e_.record()
            es.ev[j_] = e_.cuda_event
        step_structs.append(es)
    timed_step = [None]

    def step():
        if world > 1:
            return sharded(out_full)
        if timed_step[0] is not None:
            _call_with_events(prep, step_structs[timed_step[0]], 0)
            timed_step[0] += 1
            return prep.out
        return prep()

    # warmup
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches = N.load().isa_last_launch_count()
    if world > 1:
        dist.barrier()
    clk = ClockSampler(local_rank)
    clk.start()
    time.sleep(0.3)
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    timed_step[0] = 0
    e0.record(st)
    for _ in range(args.steps):
        step()
    e1.record(st)
    timed_step[0] = None
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = clk.stop()
    ms = e0.elapsed_time(e1) / args.steps
    compute_only_ms = gather_ok = None
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        # the same schedule without the all-gathers (scaling without the collective)
        dist.barrier()
        torch.cuda.synchronize()
        e0.record(st)
        for _ in range(args.steps):
            sharded(out_full, gather=False)
        e1.record(st)
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / args.steps], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        compute_only_ms = float(t.item())
        # placement check: every head slab of the gathered output equals its
        # owner's local result (per-head sums, exact: same bits, same reduction)
        sharded(out_full)
        torch.cuda.synchronize()
        mine_sums = torch.stack([o[0, 0].float().sum() for o in sharded.local_output()]).to(dev)
        all_sums = [torch.empty_like(mine_sums) for _ in range(world)]
        dist.all_gather(all_sums, mine_sums)
        full_sums = torch.stack([out_full[0, h].float().sum() for h in range(H)])
        gather_ok = all(bool(torch.equal(full_sums[c * world + r], all_sums[r][c]))
                        for r in range(world) for c in range(Hl))

    # ---- per-stage / per-kernel times (events recorded by the C ABI on the launching stream)
    def make_events():
        evl = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
        es = N.IsaEvents()
        for i_, e_ in enumerate(evl):
            e_.record()
            es.ev[i_] = e_.cuda_event
        return evl, es

    def stages(evl):
        return {"coarse": evl[0].elapsed_time(evl[1]), "select": evl[1].elapsed_time(evl[2]),
                "split": evl[2].elapsed_time(evl[3]), "attn": evl[3].elapsed_time(evl[5]),
                "exact": evl[3].elapsed_time(evl[4]), "taylor": evl[4].elapsed_time(evl[5])}

    def mean_stages(lst):
        return {k_: sum(d_[k_] for d_ in lst) / len(lst) for k_ in lst[0]}

    # shipped configuration (D = 128): one launch, K6 items over the sharp
    # blocks and K7T / K7 items over the flat ones. N = 1: stage times are the
    # timed steps' own events.
    step_stats = None
    if world == 1:
        per = sorted(evl[0].elapsed_time(evl[5]) for evl in step_evs)
        q_ = lambda f: per[min(len(per) - 1, int(round(f * (len(per) - 1))))]  # noqa: E731
        step_stats = {"median": statistics.median(per), "p10": q_(0.1), "p90": q_(0.9), "n": len(per),
                      "note": "per-step device time (first to last kernel event of the step)"}
        shipped = mean_stages([stages(evl) for evl in step_evs])
    # A/B in ONE loop alternating the shipped step (K6 launch + Taylor launch)
    # with the single fused grid (ISA_FLAG_FUSED_GRID), so both see the same clocks.
    ev_a = [make_events() for _ in range(args.steps)]
    ev_b = [make_events() for _ in range(args.steps)]
    ev_c = [make_events() for _ in range(args.steps)]
    torch.cuda.synchronize()
    for i_ in range(args.steps):
        _call_with_events(prep, ev_a[i_][1], 0)
        _call_with_events(prep, ev_b[i_][1], N.FLAG_FUSED_GRID)
        _call_with_events(prep, ev_c[i_][1], N.FLAG_SINGLE_CTA)
    torch.cuda.synchronize()
    shipped_alt = mean_stages([stages(e_[0]) for e_ in ev_a])
    fused_alt = mean_stages([stages(e_[0]) for e_ in ev_b])
    single_alt = mean_stages([stages(e_[0]) for e_ in ev_c])
    if world > 1:
        shipped = shipped_alt
    stage = {"coarse": shipped["coarse"], "select": shipped["select"], "split": shipped["split"],
             "attention": shipped["attn"], "exact_k6": shipped["exact"], "taylor": shipped["taylor"],
             "ab_loop": {"shipped_two_launches": shipped_alt["attn"], "fused_single_grid": fused_alt["attn"],
                         "shipped_exact_k6": shipped_alt["exact"], "shipped_taylor": shipped_alt["taylor"],
                         "single_cta_exact_k6": single_alt["exact"],
                         "steps": args.steps,
                         "note": "shipped, fused-grid and single-CTA-K6 steps alternated in one loop after the "
                                 "timed region (same clocks); per-launch CUDA events"}}
    peaks = _peaks()
    # K6 runs ~18 ms inside a ~23 ms step: a kernel timed on its own at burst
    # clocks, not a seconds-long sustained run -> the burst peak
    peak_tc = peaks.get("bf16_tflops") or 1666.4
    attn_tflops = (f_sharp + f_taylor_alg) / (shipped["attn"] * 1e-3) / 1e12
    exact_tflops = f_sharp / (shipped["exact"] * 1e-3) / 1e12
    taylor_tflops = f_taylor_alg / (shipped["taylor"] * 1e-3) / 1e12 if shipped["taylor"] > 0 else None
    prof = _profile_summary()

    result = {
        "metric": METRIC, "value": ms, "unit": "ms", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
        "dtype": "bf16", "data": "synthetic",
        "config": dict(args.workload, parallelism=f"head-sharded x{world}" if world > 1 else "single GPU",
                       l2="inputs larger than L2" if 3 * H * S * D * 2 > 126e6 else
                          "inputs fit in L2: steps back to back (no flush); routing reads are warm"),
        "tflops_isa_alg": f_isa / (ms * 1e-3) / 1e12,
        "tflops_dense_equiv": f_dense / (ms * 1e-3) / 1e12,
        "flops": {"isa": f_isa, "dense": f_dense, "sharp": f_sharp * world, "taylor_alg": f_taylor_alg * world},
        "stage_ms": stage,
        "step_ms_stats": step_stats,
        "sharded": None if world == 1 else {
            "compute_only_ms": compute_only_ms, "heads_per_rank": Hl, "schedule": shard_mode,
            "gather_check": gather_ok, "backend": os.environ.get("ISA_BENCH_BACKEND", "nccl"),
            "note": "value = max over ranks of the step (compute + per-head NCCL all-gathers overlapped with "
                    "it); compute_only_ms = the same schedule without the gathers (max over ranks)"},
        "gpu_launches": launches * args.steps,
        "roofline": {
            "kernel": "gba_attention_pair_kernel<128, MODE_EXACT> (K6 on CTA pairs, cta_group::2: the sharp "
                      "branch, the dominant launch)",
            "bound": "tensor", "achieved": exact_tflops, "peak": peak_tc, "unit": "TFLOP/s",
            "frac": exact_tflops / peak_tc, "traffic": prof.get("k6_dram_bytes"),
            "peak_source": "MEASURED_PEAKS.json bf16_tflops (burst: K6 runs ~18 ms per step, not a seconds-long "
                           "sustained run)",
            "algorithmic": "F_sharp = 4*b^2*D*n_sharp*t_new (pipeline.py:278) per launch / average CUDA-event "
                           "duration of the launch over the timed steps, on its stream",
        },
        "attention_kernels": {"achieved": attn_tflops, "frac": attn_tflops / peak_tc, "unit": "TFLOP/s",
                              "kernels": "K6 launch + Taylor launch (per-head K7T / K7)",
                              "algorithmic": "F_sharp + F_taylor (pipeline.py:269-289, taylor.py:299-316)",
                              "traffic": prof.get("attn_dram_bytes")},
        "taylor_kernel": {"achieved": taylor_tflops, "frac": (taylor_tflops / peak_tc) if taylor_tflops else None,
                          "unit": "TFLOP/s", "kernel": "gba_isa_hybrid_kernel<128> with 0 exact items "
                                                       "(per head K7T gba_taylor_t body or K7 union tiles)",
                          "algorithmic": "reference flop_count (taylor.py:299-316): F_taylor",
                          "timed": "its launch inside the timed steps",
                          "traffic": prof.get("k7t_dram_bytes"), "l2_bytes": prof.get("k7t_l2_bytes"),
                          "l2_roofline": _l2_roofline(prof.get("k7t_l2_bytes"), shipped["taylor"])},
        "clocks": clocks,
    }
    if rank == 0 and world == 1 and not args.no_extras:
        result.update(_extras(args, P, q, k, v, icl, cfg, ms, dev))
    if args.config == "cfg4-grid":
        result["grid"] = _cfg4_grid(P, q, k, v, icl, result.get("dense_ms"), result.get("cudnn_sdpa_ms"))
    if world > 1 and not args.no_extras:
        e = _e2e(args, P, q, k, v, icl, cfg, world)
        t = torch.tensor([e["value"]], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e["value"] = float(t.item())
        result["e2e"] = e
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        heads_run, fraction = cpu_plan(args)
        cms, detail = cpu_sample(args.l_src, args.l_ctx, H, D=D, fraction=fraction, heads_run=heads_run)
        cores, apis = cpu_cores()
        result["cpu_baseline"] = {
            "value": cms, "unit": "ms", "cores": cores, "kind": "port",
            "sample": _sample_text(args, heads_run, fraction, apis)
                      + f"; route {detail['route_s']:.2f}s, attention sample {detail['attn_sample_s']:.2f}s",
        }
    if rank == 0:
        print(json.dumps(result), flush=True)


def _call_with_events(prep, ev_struct, flags=0):
    import ctypes

    import torch

    from paper_2605_04569_b200 import _native as N
    from paper_2605_04569_b200.pipeline import _ptr

    inp = prep.inp
    kn = N.IsaKnobs(inp.knobs.scale, inp.knobs.k_ctx, inp.knobs.n_flat, inp.knobs.k_mask, inp.knobs.softmax_first,
                    flags, inp.knobs.gamma, inp.knobs.residual_softmax)
    N.check(N.load().isa_forward(ctypes.byref(inp.shape), ctypes.byref(kn), _ptr(inp.q), _ptr(inp.k),
                                 _ptr(inp.v), _ptr(prep.out), _ptr(prep.ws), prep.nbytes, None, None, _ptr(prep.err),
                                 ctypes.byref(ev_struct), torch.cuda.current_stream().cuda_stream))


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "hbm_gbs": 6650.0, "fallback": True}


def _l2_roofline(l2_bytes, ms):
    """K7T streams its K/V and centroid tiles from L2: achieved L2->SM GB/s
    against the measured L2->SM bandwidth (profiles/ ubench, TMA bulk copies
    with 2 CTAs x 64 KB in flight per SM)."""
    peak = _profile_summary().get("l2_to_sm_gbs")
    if not l2_bytes or not ms or not peak:
        return None
    ach = l2_bytes / (ms * 1e-3) / 1e9
    return {"achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
            "source": "profiles/r2_ubench_l2bw.txt (tools/ubench/l2bw.cu)"}


def _profile_summary():
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))
    except Exception:
        return {}


def _extras(args, P, q, k, v, icl, cfg, ms, dev):
    """Dense sm_100a baseline (K8), cuDNN SDPA cross-check and the e2e number."""
    import torch
    import torch.nn.functional as F

    res = {}
    st = torch.cuda.current_stream()

    def timeit(fn, reps=2):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(reps):
            fn()
        b.record(st)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps

    dense_ms = timeit(lambda: P.dense_attention(q, k, v))
    res["dense_ms"] = dense_ms
    res["speedup_vs_dense_sm100a"] = dense_ms / ms
    try:
        from torch.nn.attention import SDPBackend, sdpa_kernel

        with sdpa_kernel([SDPBackend.CUDNN_ATTENTION]):
            sdpa_ms = timeit(lambda: F.scaled_dot_product_attention(q, k, v))
        res["cudnn_sdpa_ms"] = sdpa_ms
        res["speedup_vs_cudnn_sdpa"] = sdpa_ms / ms
    except Exception as exc:  # pragma: no cover
        res["cudnn_sdpa_ms"] = None
        res["cudnn_sdpa_error"] = str(exc)[:200]
    d = P.IsaDims.derive(q.shape, icl, cfg)
    res["dense_tflops"] = d.flops().dense_equivalent_mas / (dense_ms * 1e-3) / 1e12

    # §8f rank 2: isa_backward (pipeline.py:373-466) on the same inputs: forward
    # recompute + tcgen05 dK/dV, dQ and centroid kernels; side measurement (not the metric)
    try:
        do = torch.randn(q.shape, device=q.device, dtype=torch.float32).to(q.dtype)
        bwd_ms = timeit(lambda: P.isa_backward(q, k, v, icl, cfg, do))
        f = d.flops()
        res["backward"] = {"ms": bwd_ms, "alg_tflops": 2.5 * (f.exact_mas + f.taylor_mas) / (bwd_ms * 1e-3) / 1e12,
                           "note": "CUDA events over 2 calls after one warm-up call, incl. the forward recompute; "
                                   "TFLOP/s at the 2.5x-forward convention"}
        del do
    except Exception as exc:  # pragma: no cover
        res["backward"] = {"error": str(exc)[:200]}

    res["e2e"] = _e2e(args, P, q, k, v, icl, cfg, 1)
    return res


def _cfg4_grid(P, q, k, v, icl, dense_ms, sdpa_ms, reps=3):
    """BASELINE configs[3]: the ISA layer over alpha_s x alpha_f (alpha_ns =
    0.0625; alpha_f is the sharpness threshold as a rank cut, coarse.py:197)
    against dense attention on the same tensors. CUDA events around `reps`
    calls after one warm-up, per point."""
    import torch

    st = torch.cuda.current_stream()
    rows = []
    for a_s in CFG4_GRID["alpha_s"]:
        for a_f in CFG4_GRID["alpha_f"]:
            cfg = P.IsaConfig(alpha_s=a_s, alpha_f=a_f, alpha_ns=0.0625)
            prep = P.prepare(q, k, v, icl, cfg)
            prep()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(reps):
                prep()
            e1.record(st)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            d = P.IsaDims.derive(q.shape, icl, cfg)
            f = d.flops()
            rows.append({"alpha_s": a_s, "alpha_f": a_f, "ms": ms, "isa_alg_tflops": f.total() / ms / 1e9,
                         "flop_ratio_dense_over_isa": f.dense_equivalent_mas / f.total(),
                         "speedup_vs_dense_sm100a": dense_ms / ms if dense_ms else None,
                         "speedup_vs_cudnn_sdpa": sdpa_ms / ms if sdpa_ms else None,
                         "k_ctx": d.k_ctx, "n_flat": d.n_flat, "k": d.k})
            del prep
    return rows


def _e2e(args, P, q, k, v, icl, cfg, world):
    """e2e through the public API with host buffers (pinned): H2D + D2H inside
    the timed region. At N > 1 every rank streams its own heads (max over
    ranks; the caller reduces)."""
    import torch

    st = torch.cuda.current_stream()
    qh, kh, vh = (t.cpu().pin_memory() for t in (q, k, v))
    outh = torch.empty(q.shape, dtype=q.dtype, pin_memory=True)

    def e2e():
        # host tensors in, host tensor out: the native head-chunk streaming
        # (isa_forward_host) overlaps H2D / pipeline / D2H; returns completed
        P.isa_forward(qh, kh, vh, icl, cfg, collect_trace=False, out=outh)

    e2e()
    torch.cuda.synchronize()
    steps = max(2, min(args.steps, 5))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(steps):
        e2e()
    b.record(st)
    torch.cuda.synchronize()
    e2e_ms = a.elapsed_time(b) / steps
    # copy floor: the same bytes as plain pinned copies, H2D and D2H concurrent on two streams
    dev_in = torch.empty((3,) + tuple(q.shape), dtype=q.dtype, device=q.device)
    dev_out = torch.empty_like(q)
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()

    def copies():
        with torch.cuda.stream(s_in):
            for i_, t_ in enumerate((qh, kh, vh)):
                dev_in[i_].copy_(t_, non_blocking=True)
        with torch.cuda.stream(s_out):
            outh.copy_(dev_out, non_blocking=True)
        st.wait_stream(s_in)
        st.wait_stream(s_out)

    copies()
    torch.cuda.synchronize()
    a.record(st)
    copies()
    b.record(st)
    torch.cuda.synchronize()
    floor_ms = a.elapsed_time(b)
    del dev_in, dev_out
    nb = q.numel() * q.element_size() * world
    return {"value": e2e_ms, "unit": "ms", "h2d_bytes_per_step": 3 * nb, "d2h_bytes_per_step": nb,
            "copy_floor_ms": floor_ms,
            "note": "public isa_forward API on pinned host Q/K/V/out: native head-chunk streaming "
                    "(H2D of chunk c+1 and D2H of chunk c-1 overlap the pipeline of chunk c)"
                    + ("; each rank streams its own heads, max over ranks" if world > 1 else "")}


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # self-launch: one process per GPU under torch.distributed.run (rank 0 prints)
        import socket

        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
        sys.stdout.flush()
        os.execv(sys.executable, cmd)
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        backend = os.environ.get("ISA_BENCH_BACKEND", "nccl")
        if backend == "gloo":  # functional check of the N > 1 schedule on fewer GPUs than ranks
            local_rank %= torch.cuda.device_count()
            torch.cuda.set_device(local_rank)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
