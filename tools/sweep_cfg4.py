"""BASELINE.json configs[3]: ISA sweep over the context keep-ratio (alpha_s) and
the sharpness split (alpha_f, the "sharpness threshold" as a rank cut) at
16K source + 16K context, Wan-14B shape (H=40, D=128), bf16, vs dense
attention on the same tensors (our sm_100a dense kernel and cuDNN SDPA).

    python tools/sweep_cfg4.py [--heads 40] [--reps 5] [--out profiles/r1_sweep_cfg4.md]

One JSON line per grid point on stdout, a markdown table in --out. Timing:
CUDA events around `reps` back-to-back calls after 2 warm-ups; Q/K/V are
(1,40,32768,128) bf16 = 1 GB (> 126 MB L2).
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

    ap = argparse.ArgumentParser()
    ap.add_argument("--heads", type=int, default=40)
    ap.add_argument("--l", type=int, default=16384)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r1_sweep_cfg4.md"))
    a = ap.parse_args()
    H, L, D = a.heads, a.l, 128
    g = torch.Generator(device="cuda").manual_seed(0)
    q, k, v = (torch.randn(1, H, 2 * L, D, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
    st = torch.cuda.current_stream()

    def timeit(fn):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(a.reps):
            fn()
        e1.record(st)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / a.reps

    dense_ms = timeit(lambda: P.dense_attention(q, k, v))
    try:
        from torch.nn.attention import SDPBackend, sdpa_kernel

        with sdpa_kernel([SDPBackend.CUDNN_ATTENTION]):
            sdpa_ms = timeit(lambda: torch.nn.functional.scaled_dot_product_attention(q, k, v))
    except Exception:
        sdpa_ms = None
    icl = P.IclLayout(L, L)
    rows = []
    for a_s in (0.0625, 0.125, 0.25, 0.5, 1.0):
        for a_f in (0.0, 0.25, 0.5, 0.75):
            cfg = P.IsaConfig(alpha_s=a_s, alpha_f=a_f, alpha_ns=0.0625)
            prep = P.prepare(q, k, v, icl, cfg)
            ms = timeit(prep)
            d = P.IsaDims.derive(q.shape, icl, cfg)
            f = d.flops()
            row = {"alpha_s": a_s, "alpha_f": a_f, "alpha_ns": 0.0625, "isa_ms": ms,
                   "isa_alg_tflops": f.total() / ms / 1e9, "dense_equiv_tflops": f.dense_equivalent_mas / ms / 1e9,
                   "flop_ratio_dense_over_isa": f.dense_equivalent_mas / f.total(),
                   "speedup_vs_dense_sm100a": dense_ms / ms,
                   "speedup_vs_cudnn_sdpa": (sdpa_ms / ms) if sdpa_ms else None,
                   "k_ctx": d.k_ctx, "n_flat": d.n_flat, "k": d.k}
            rows.append(row)
            print(json.dumps(row), flush=True)
            del prep
    hdr = (f"# cfg4 sweep (BASELINE configs[3]): {L}+{L} tokens, H={H}, D=128, bf16, one B200\n\n"
           f"dense sm_100a kernel: {dense_ms:.3f} ms; cuDNN SDPA: "
           f"{'%.3f ms' % sdpa_ms if sdpa_ms else 'n/a'}. CUDA events, {a.reps} reps after 2 warm-ups. "
           "alpha_ns = 0.0625. TFLOP/s use the reference accounting (pipeline.py:269-289).\n\n"
           "| alpha_s | alpha_f | k_ctx | n_flat | k | ISA ms | alg TFLOP/s | dense FLOP / ISA FLOP | "
           "speed-up vs dense kernel | vs cuDNN SDPA |\n|---|---|---|---|---|---|---|---|---|---|\n")
    body = "".join(
        f"| {r['alpha_s']} | {r['alpha_f']} | {r['k_ctx']} | {r['n_flat']} | {r['k']} | {r['isa_ms']:.3f} | "
        f"{r['isa_alg_tflops']:.0f} | {r['flop_ratio_dense_over_isa']:.2f} | {r['speedup_vs_dense_sm100a']:.2f} | "
        f"{(r['speedup_vs_cudnn_sdpa'] or float('nan')):.2f} |\n" for r in rows)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as fh:
        fh.write(hdr + body)
    print(hdr + body)


if __name__ == "__main__":
    main()
