"""Generate golden vectors from the REFERENCE implementation (`isattn`).

Run in the build container, where /root/reference exists:

    python tests/golden/make_golden.py

For each case it generates inputs with the reference's own workload
generator (`isattn.generate`, workload.py:127-144), rounds them to bf16
values (the B200 path computes on bf16), runs the unmodified reference
`isa_routing` / `isa_forward` (pipeline.py:302-316) and `full_attention`
(reference.py:79-123), and stores the routing decisions and outputs in
`tests/golden/<case>.npz`. Inputs are NOT stored: they are regenerated from
the spec by `oracle.isa_oracle.workload` (a restatement of workload.py) and
pinned by the stored checksums.

The GPU box never runs this script (it has no /root/reference); the tests
only read the committed .npz files.
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

import isattn  # noqa: E402  (the reference)

from oracle.isa_oracle import round_bf16  # noqa: E402

CASES = [
    # name, workload kind, B, H, S, D, l_src, l_ctx, seed, cfg overrides
    ("cfg1_iid_s0", "iid-gaussian", 1, 2, 2048, 64, 1024, 1024, 0, {}),
    ("cfg1_clustered_s1", "clustered", 1, 2, 2048, 64, 1024, 1024, 1, {}),
    ("cfg1_lowrank_s2", "lowrank", 1, 2, 2048, 64, 1024, 1024, 2, {}),
    ("ragged_iid_s3", "iid-gaussian", 1, 2, 2100, 64, 1000, 1100, 3, {"strict": False}),
    ("d128_clustered_s4", "clustered", 1, 1, 2048, 128, 1024, 1024, 4, {}),
    ("knobs_iid_s5", "iid-gaussian", 1, 2, 2048, 64, 1024, 1024, 5,
     {"alpha_s": 0.25, "alpha_f": 0.25, "alpha_ns": 0.125}),
    ("allsharp_iid_s6", "iid-gaussian", 1, 2, 2048, 64, 1024, 1024, 6, {"alpha_s": 1.0, "alpha_f": 0.0}),
    ("allflat_exact_s7", "iid-gaussian", 1, 2, 2048, 64, 1024, 1024, 7,
     {"alpha_s": 1.0, "alpha_f": 1.0, "alpha_ns": 1.0}),
    ("srconly_s8", "clustered", 1, 2, 1024, 64, 1024, 0, 8, {}),
    ("rawvar_clustered_s9", "clustered", 2, 1, 2048, 64, 1024, 1024, 9, {"softmax_first": False}),
    ("ragged_clustered_s10", "clustered", 1, 2, 1500, 128, 900, 600, 10,
     {"strict": False, "alpha_s": 0.5, "alpha_ns": 0.25}),
    # gamma coarse residual (pipeline.py:261-267, 354-356), softmax and raw-score variants
    ("gamma_clustered_s14", "clustered", 1, 2, 2048, 64, 1024, 1024, 14, {"gamma": 0.5}),
    ("gamma_raw_iid_s15", "iid-gaussian", 1, 2, 2100, 128, 1000, 1100, 15,
     {"gamma": 0.05, "residual_softmax": False, "strict": False}),
    # routing-only cases (no stored output): larger T so the block mask has k > 1
    ("mid_iid_s11", "iid-gaussian", 1, 2, 8192, 64, 4096, 4096, 11, {"_routing_only": True}),
    ("mid_clustered_s12", "clustered", 1, 2, 8192, 128, 4096, 4096, 12, {"_routing_only": True}),
    ("mid_lowrank_s13", "lowrank", 1, 1, 16384, 64, 8192, 8192, 13, {"_routing_only": True}),
]

IDENTITY = {"allsharp_iid_s6", "allflat_exact_s7"}


def make_case(name, kind, B, H, S, D, l_src, l_ctx, seed, over):
    spec = isattn.WorkloadSpec(batch=B, heads=H, seq_len=S, dim=D, l_src=l_src, l_ctx=l_ctx, kind=kind, seed=seed)
    q, k, v, icl = isattn.generate(spec)
    raw_sums = [float(x.astype(np.float64).sum()) for x in (q, k, v)]
    q, k, v = (round_bf16(x) for x in (q, k, v))
    over = dict(over)
    routing_only = over.pop("_routing_only", False)
    cfg = isattn.IsaConfig(**over)
    t0 = time.perf_counter()
    out, trace = isattn.isa_forward(q, k, v, icl, cfg)
    t_isa = time.perf_counter() - t0
    routing = isattn.isa_routing(q, k, v, icl, cfg)
    payload = {
        "selection": routing.selection.indices.astype(np.int64),
        "sharp": routing.split.sharp.astype(np.int64),
        "flat": routing.split.flat.astype(np.int64),
        "sharpness": routing.split.sharpness.astype(np.float64),
        "mask": (routing.mask.indices.astype(np.int64) if routing.mask is not None
                 else np.zeros((B, H, 0, 0), np.int64)),
        "input_sums": np.array([float(x.astype(np.float64).sum()) for x in (q, k, v)]),
        "raw_input_sums": np.array(raw_sums),
        "flops": np.array([trace.flops.exact_mas, trace.flops.taylor_mas, trace.flops.overhead_mas,
                           trace.flops.dense_equivalent_mas], dtype=np.int64),
    }
    if not routing_only:
        payload["out"] = out.astype(np.float32)
    if name in IDENTITY:
        payload["full"] = isattn.full_attention(q, k, v).astype(np.float32)
    meta = {"name": name, "kind": kind, "B": B, "H": H, "S": S, "D": D, "l_src": l_src, "l_ctx": l_ctx,
            "seed": seed, "cfg": over, "routing_only": routing_only, "ref_isa_seconds": t_isa,
            "generator": "isattn.generate(WorkloadSpec(...)) then round to bf16"}
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), meta=json.dumps(meta), **payload)
    print(f"{name}: isa_forward {t_isa:.2f}s  k_ctx={payload['selection'].shape[2]} "
          f"n_flat={payload['flat'].shape[2]} k={payload['mask'].shape[3]}")


ROPE_CASES = [
    # name, B, H, l_src, l_ctx, D, base, seed
    ("rope_small", 1, 2, 100, 60, 64, 10000.0, 0),
    ("rope_ragged_d128", 2, 1, 300, 257, 128, 500.0, 1),
    ("rope_long_positions", 1, 1, 50000, 64, 128, 10000.0, 2),
]


def make_rope(name, B, H, l_src, l_ctx, D, base, seed):
    """Golden vectors for the reference apply_decoupled_rope (pipeline.py:469-490)."""
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((B, H, l_src + l_ctx, D)).astype(np.float32)
    out = isattn.apply_decoupled_rope(x, isattn.IclLayout(l_src, l_ctx), base=base)
    # store a row sample (ends of both segments + strided interior); x is
    # regenerated from the seed and pinned by its checksum
    S = l_src + l_ctx
    rows = np.unique(np.concatenate([np.arange(min(S, 96)), np.arange(max(0, l_src - 96), min(S, l_src + 96)),
                                     np.arange(max(0, S - 96), S), np.arange(0, S, 997)]))
    meta = {"name": name, "B": B, "H": H, "D": D, "l_src": l_src, "l_ctx": l_ctx, "base": base, "seed": seed,
            "x_sum": float(x.astype(np.float64).sum())}
    np.savez_compressed(os.path.join(HERE, "rope", f"{name}.npz"), meta=json.dumps(meta), rows=rows,
                        out=out[:, :, rows])
    print(f"{name}: {x.shape}, {rows.size} rows stored")


BWD_CASES = [
    # name, kind, B, H, S, D, l_src, l_ctx, seed, cfg overrides
    ("bwd_cfg1_iid_s20", "iid-gaussian", 1, 2, 2048, 64, 1024, 1024, 20, {}),
    ("bwd_clustered_d128_s21", "clustered", 1, 1, 2048, 128, 1024, 1024, 21, {}),
    ("bwd_ragged_s22", "iid-gaussian", 1, 2, 1500, 64, 900, 600, 22, {"strict": False, "alpha_s": 0.5}),
    ("bwd_knobs_s23", "lowrank", 2, 1, 2048, 64, 1024, 1024, 23, {"alpha_f": 0.75, "alpha_ns": 0.25}),
    ("bwd_gamma_s24", "clustered", 1, 2, 2048, 64, 1024, 1024, 24, {"gamma": 0.5}),
    ("bwd_gamma_raw_s25", "iid-gaussian", 1, 1, 1500, 128, 900, 600, 25,
     {"gamma": 0.05, "residual_softmax": False, "strict": False}),
    # round 2: the D = 128 backward kernels one branch at a time (sharp dQ on CTA pairs, centroid
    # adjoint + flat dQ), and batch 2 with ragged segments
    ("bwd_allsharp_d128_s26", "iid-gaussian", 1, 2, 2048, 128, 1024, 1024, 26, {"alpha_s": 1.0, "alpha_f": 0.0}),
    ("bwd_allflat_d128_s27", "clustered", 1, 1, 2048, 128, 1024, 1024, 27, {"alpha_s": 0.0, "alpha_f": 1.0}),
    ("bwd_b2_ragged_d128_s28", "lowrank", 2, 1, 1700, 128, 1000, 700, 28, {"strict": False, "alpha_s": 0.25}),
    ("bwd_mid_d128_s29", "iid-gaussian", 1, 1, 4096, 128, 2048, 2048, 29, {}),  # longer K/V and query streams
]


def make_bwd(name, kind, B, H, S, D, l_src, l_ctx, seed, over):
    """Golden gradients of the reference isa_backward (pipeline.py:373-466). dO is
    regenerated from the seed (numpy default_rng) and pinned by its checksum."""
    spec = isattn.WorkloadSpec(batch=B, heads=H, seq_len=S, dim=D, l_src=l_src, l_ctx=l_ctx, kind=kind, seed=seed)
    q, k, v, icl = isattn.generate(spec)
    q, k, v = (round_bf16(x) for x in (q, k, v))
    do = round_bf16(np.random.default_rng(seed).standard_normal((B, H, S, D)).astype(np.float32))
    cfg = isattn.IsaConfig(**over)
    t0 = time.perf_counter()
    g = isattn.isa_backward(q, k, v, icl, cfg, do)
    t = time.perf_counter() - t0
    meta = {"name": name, "kind": kind, "B": B, "H": H, "S": S, "D": D, "l_src": l_src, "l_ctx": l_ctx,
            "seed": seed, "cfg": over, "ref_backward_seconds": t,
            "input_sums": [float(x.astype(np.float64).sum()) for x in (q, k, v, do)]}
    np.savez_compressed(os.path.join(HERE, "bwd", f"{name}.npz"), meta=json.dumps(meta),
                        dq=g.dq.astype(np.float32), dk=g.dk.astype(np.float32), dv=g.dv.astype(np.float32))
    print(f"{name}: isa_backward {t:.2f}s")


if __name__ == "__main__":
    only = set(sys.argv[1:])
    os.makedirs(os.path.join(HERE, "bwd"), exist_ok=True)
    for case in BWD_CASES:
        if not only or case[0] in only:
            make_bwd(*case)
    for case in CASES:
        if not only or case[0] in only:
            make_case(*case)
    os.makedirs(os.path.join(HERE, "rope"), exist_ok=True)
    for case in ROPE_CASES:
        if not only or case[0] in only:
            make_rope(*case)
