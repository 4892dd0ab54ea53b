"""BASELINE.json configs[4]: the LIVEditor-14B-shaped DiT attention stack
(H=40, D=128, E=5120) at 50,000 source + 50,000 context tokens (ragged
segments, cfg.strict=False), random-init weights, bf16, on 1..8 GPUs.

    python tools/bench_stack.py [--gpus N] [--layers 40] [--l-src 50000] [--l-ctx 50000] [--dense-layers 1]

N > 1 re-launches itself under torch.distributed.run (one process per GPU,
NCCL): heads are sharded round-robin, QKV column-parallel, O row-parallel with
a chunked all-reduce (paper_2605_04569_b200/stack.py). Times the whole stack
with CUDA events after one warm-up layer (max over ranks), the per-stage split
(QKV GEMM, RoPE + ISA attention, O GEMM [+ all-reduce]) from a second pass,
and one layer with dense attention (our sm_100a dense kernel, standalone RoPE)
for the speed-up. Rank 0 prints one JSON line.
"""
import argparse
import json
import os
import socket
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--layers", type=int, default=40)
    ap.add_argument("--l-src", type=int, default=50000)
    ap.add_argument("--l-ctx", type=int, default=50000)
    ap.add_argument("--heads", type=int, default=40)
    ap.add_argument("--dense-layers", type=int, default=1)
    a = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and a.gpus > 1:
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        os.execv(sys.executable, [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                                  f"--nproc-per-node={a.gpus}", "--master-addr", "127.0.0.1", "--master-port",
                                  str(port), os.path.abspath(__file__), *sys.argv[1:]])
    import torch
    import torch.distributed as dist

    import paper_2605_04569_b200 as P
    from paper_2605_04569_b200.stack import DiTAttentionStack

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    S = a.l_src + a.l_ctx
    icl = P.IclLayout(a.l_src, a.l_ctx)
    strict = a.l_src % 64 == 0 and a.l_ctx % 64 == 0
    cfg = P.IsaConfig(strict=strict)
    stack = DiTAttentionStack(a.layers, a.heads, world=world, rank=rank)
    g = torch.Generator(device="cuda").manual_seed(1)
    x0 = torch.randn(1, S, a.heads * 128, device="cuda", generator=g).to(torch.bfloat16)
    stack.layers[0](x0, icl, cfg)  # warm-up (workspaces, cuBLAS heuristics, NCCL communicators)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    y = stack(x0, icl, cfg)
    e1.record()
    torch.cuda.synchronize()
    total = max_over_ranks(e0.elapsed_time(e1))
    stages = {}
    stack(x0, icl, cfg, timings=stages)
    per_layer = {k: max_over_ranks(v / a.layers) for k, v in stages.items()}
    dense = {}
    if world == 1:
        for layer in stack.layers[: a.dense_layers]:
            layer(x0, icl, cfg, attention="dense", timings=dense)
        dense = {k: v / max(a.dense_layers, 1) for k, v in dense.items()}
    d = P.IsaDims.derive((1, a.heads, S, 128), icl, cfg)
    f = d.flops()
    att = per_layer["attention_with_rope"]
    line = {
        "workload": f"cfg5: {a.layers}-layer DiT attention stack, {a.l_src}+{a.l_ctx} tokens, H={a.heads}, D=128",
        "n_gpus": world, "parallelism": f"heads x{world} (QKV column-parallel, O row-parallel + all-reduce)"
        if world > 1 else "single GPU",
        "stack_ms": total, "layer_ms": total / a.layers, "stage_ms_per_layer": per_layer,
        "dense_attention_layer_stage_ms": dense or None,
        "attention_speedup_vs_dense_kernel": (dense["attention_with_rope"] / att) if dense else None,
        "isa_alg_tflops": f.total() / world / att / 1e9,
        "dense_equiv_tflops": f.dense_equivalent_mas / world / att / 1e9,
        "strict": strict, "finite": bool(torch.isfinite(y.float()).all()),
        "timing": "CUDA events around the whole stack after a warm-up layer, max over ranks",
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
