"""BASELINE.json configs[4] on one B200: the LIVEditor-14B-shaped DiT attention
stack (H=40, D=128, E=5120) at 50,000 source + 50,000 context tokens (ragged
segments, cfg.strict=False), random-init weights, bf16.

    python tools/bench_stack.py [--layers 40] [--l-src 50000] [--l-ctx 50000] [--dense-layers 1]

Times the whole stack with CUDA events (after one warm-up layer) and the
per-stage split (QKV GEMM, decoupled RoPE, attention, O GEMM) from a second
pass with per-stage events; also one layer with dense attention (our sm_100a
dense kernel) for the speed-up. Prints one JSON line.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_2605_04569_b200 as P
    from paper_2605_04569_b200.stack import DiTAttentionStack

    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=40)
    ap.add_argument("--l-src", type=int, default=50000)
    ap.add_argument("--l-ctx", type=int, default=50000)
    ap.add_argument("--heads", type=int, default=40)
    ap.add_argument("--dense-layers", type=int, default=1)
    a = ap.parse_args()
    S = a.l_src + a.l_ctx
    icl = P.IclLayout(a.l_src, a.l_ctx)
    strict = a.l_src % 64 == 0 and a.l_ctx % 64 == 0
    cfg = P.IsaConfig(strict=strict)
    stack = DiTAttentionStack(a.layers, a.heads)
    g = torch.Generator(device="cuda").manual_seed(1)
    x0 = torch.randn(1, S, a.heads * 128, device="cuda", generator=g).to(torch.bfloat16)
    stack.layers[0](x0, icl, cfg)  # warm-up (workspaces, cuBLAS heuristics)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    y = stack(x0, icl, cfg)
    e1.record()
    torch.cuda.synchronize()
    total = e0.elapsed_time(e1)
    stages = {}
    stack(x0, icl, cfg, timings=stages)
    per_layer = {k: v / a.layers for k, v in stages.items()}
    dense = {}
    for layer in stack.layers[: a.dense_layers]:
        layer(x0, icl, cfg, attention="dense", timings=dense)
    dense = {k: v / max(a.dense_layers, 1) for k, v in dense.items()}
    d = P.IsaDims.derive((1, a.heads, S, 128), icl, cfg)
    f = d.flops()
    line = {
        "workload": f"cfg5: {a.layers}-layer DiT attention stack, {a.l_src}+{a.l_ctx} tokens, H={a.heads}, D=128",
        "stack_ms": total, "layer_ms": total / a.layers, "stage_ms_per_layer": per_layer,
        "dense_attention_layer_stage_ms": dense,
        "attention_speedup_vs_dense_kernel": (dense.get("attention", 0) / per_layer["attention"]) if dense else None,
        "isa_alg_tflops": f.total() / per_layer["attention"] / 1e9,
        "dense_equiv_tflops": f.dense_equivalent_mas / per_layer["attention"] / 1e9,
        "strict": strict, "finite": bool(torch.isfinite(y.float()).all()),
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
