"""Parity of the SHIPPED configuration (D = 128, the hybrid K6 + per-head
K7/K7T grid) against the CPU oracle:

* each Taylor-branch kernel forced for every head (`taylor_kernel="k7"` /
  `"k7t"`) and the automatic per-head pick, on iid and clustered inputs at
  the cfg2 geometry and on the K7T corner shapes; the exported per-head
  choice (`IsaTrace.taylor_kernel`) proves which kernel ran;
* the benchmark's own inputs (bench.synth_qkv, seeds 1000 + h) at cfg3:
  routing bit-exact on all 40 heads, outputs on sampled rows of 4 heads.

Oracle: oracle/isa_oracle.py (taylor.py:124-160, coarse.py:139-201).
"""

from __future__ import annotations

import math

import numpy as np
import pytest
import torch

from oracle import isa_oracle as O

pytestmark = pytest.mark.gpu


def _P():
    import paper_2605_04569_b200 as P

    return P


def _bf16(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda().to(torch.bfloat16)


def _close(a, r, max_abs=2e-2, min_cos=0.999):
    a = np.asarray(a, dtype=np.float64).ravel()
    r = np.asarray(r, dtype=np.float64).ravel()
    err = float(np.max(np.abs(a - r)))
    cos = float(a @ r / (np.linalg.norm(a) * np.linalg.norm(r) + 1e-300))
    assert err <= max_abs and cos >= min_cos, f"max_abs={err:.3e} cos={cos:.6f}"


def _rows(asm, frac, l_src, l_ctx):
    """Token rows of head (0, h) the oracle computed with forward(block_fraction=frac)."""
    b = 64
    H = asm.sharp.shape[1]
    rows = np.zeros((1, H, l_src + l_ctx), dtype=bool)
    ns, nf = int(math.ceil(frac * asm.n_sharp)), int(math.ceil(frac * asm.n_flat))
    for hi in range(H):
        for u in list(asm.sharp[0, hi, :ns]) + list(asm.flat[0, hi, :nf]):
            lo = u * b if u < asm.t_src else l_src + (u - asm.t_src) * b
            hi_ = min(lo + b, l_src if u < asm.t_src else l_src + l_ctx)
            rows[0, hi, lo:hi_] = True
    return rows


def _check_routing(trace, asm):
    np.testing.assert_array_equal(trace.selection.numpy(), asm.sel)
    np.testing.assert_array_equal(trace.split.sharp.cpu().numpy(), asm.sharp)
    np.testing.assert_array_equal(trace.split.flat.cpu().numpy(), asm.flat)
    if asm.mask is not None:
        np.testing.assert_array_equal(trace.mask.numpy(), asm.mask)


EXPECT = {"k7": 0, "k7t": 1}


# ------------------------------------------------------------------ forced Taylor kernels at the cfg2 geometry
@pytest.mark.parametrize("kind", ["iid-gaussian", "clustered"])
def test_taylor_kernels_forced_and_auto_vs_oracle(kind):
    """8K + 8K, D = 128, 2 heads: K7 forced, K7T forced and the automatic pick
    each match the oracle (taylor.py:124-160); the auto output of every head is
    bit-identical to the forced run of the kernel it reports."""
    P = _P()
    q, k, v = (O.round_bf16(x) for x in O.workload(kind, 1, 2, 16384, 128, seed=31))
    asm = O.OracleAssembly(q, k, v, 8192, 8192)
    ref = asm.forward()
    args = (_bf16(q), _bf16(k), _bf16(v), P.IclLayout(8192, 8192), P.IsaConfig())
    outs = {}
    for mode in ("k7", "k7t", None):
        out, tr = P.isa_forward(*args, taylor_kernel=mode)
        _check_routing(tr, asm)
        ran = tr.taylor_kernel.cpu().numpy()
        if mode is not None:
            assert (ran == EXPECT[mode]).all(), (mode, ran)
        _close(out.float().cpu().numpy(), ref)
        outs[mode] = (out.float().cpu().numpy(), ran)
    auto, ran = outs[None]
    for h in range(2):
        forced = outs["k7" if ran[0, h] == 0 else "k7t"][0]
        np.testing.assert_array_equal(auto[:, h], forced[:, h])


@pytest.mark.parametrize("mode", ["k7", "k7t"])
@pytest.mark.parametrize("l_src,l_ctx,kw", [
    (64 * 11, 64 * 10, dict(alpha_f=0.5, alpha_ns=0.01)),                  # k = 1
    (64 * 12 + 7, 64 * 9 - 20, dict(strict=False, alpha_f=0.45)),          # ragged: short blocks, weights
    (64 * 9, 64 * 12, dict(alpha_f=0.55, alpha_s=0.5, alpha_ns=0.3)),      # odd n_flat
    (64 * 20, 64 * 20, dict(alpha_f=1.0, alpha_ns=1.0)),                   # all flat, all exact
])
def test_taylor_kernel_corners_forced_vs_oracle(mode, l_src, l_ctx, kw):
    P = _P()
    q, k, v = (O.round_bf16(x) for x in O.workload("clustered", 1, 2, l_src + l_ctx, 128, seed=l_src + l_ctx))
    okw = {kk: vv for kk, vv in kw.items() if kk != "strict"}
    asm = O.OracleAssembly(q, k, v, l_src, l_ctx, **okw)
    ref = asm.forward()
    out, tr = P.isa_forward(_bf16(q), _bf16(k), _bf16(v), P.IclLayout(l_src, l_ctx),
                            P.IsaConfig(strict=kw.get("strict", True), **okw), taylor_kernel=mode)
    _check_routing(tr, asm)
    assert (tr.taylor_kernel.cpu().numpy() == EXPECT[mode]).all()
    _close(out.float().cpu().numpy(), ref)


# ------------------------------------------------------------------ the benchmark's own inputs (cfg3)
@pytest.mark.slow
def test_bench_inputs_cfg3_all_heads():
    """bench.py's workload exactly (bench.synth_qkv, 40 heads, 32K + 32K):
    routing bit-exact against the oracle on every head; outputs of 4 heads on
    a 1/16 sample of their query blocks."""
    import bench

    P = _P()
    H, S, D, L = 40, 65536, 128, 32768
    dev = torch.device("cuda", 0)
    q, k, v = bench.synth_qkv(list(range(H)), S, D, dev)
    out, tr = P.isa_forward(q, k, v, P.IclLayout(L, L), P.IsaConfig())
    sel, sharp, flat, mask = (x.cpu().numpy() for x in (tr.selection.indices, tr.split.sharp, tr.split.flat,
                                                        tr.mask.indices))
    ctx = tr.ctx_scores.cpu().numpy()
    for h in range(H):
        qh, kh, vh = (t[:, h:h + 1].float().cpu().numpy() for t in (q, k, v))
        r = O.isa_routing(qh, kh, vh, L, L)
        # the saliency scores themselves: numpy's bits (coarse_dmma_kernel + ctx_mean_kernel)
        np.testing.assert_array_equal(ctx[:, h:h + 1], r.ctx_scores, err_msg=f"head {h}")
        np.testing.assert_array_equal(sel[:, h:h + 1], r.selection, err_msg=f"head {h}")
        np.testing.assert_array_equal(sharp[:, h:h + 1], r.sharp, err_msg=f"head {h}")
        np.testing.assert_array_equal(flat[:, h:h + 1], r.flat, err_msg=f"head {h}")
        np.testing.assert_array_equal(mask[:, h:h + 1], r.mask, err_msg=f"head {h}")
    frac = 1 / 16
    for h in (0, 13, 26, 39):
        qh, kh, vh = (t[:, h:h + 1].float().cpu().numpy() for t in (q, k, v))
        asm = O.OracleAssembly(qh, kh, vh, L, L)
        ref = asm.forward(block_fraction=frac)
        rows = _rows(asm, frac, L, L)
        _close(out[:, h:h + 1].float().cpu().numpy()[rows], ref[rows])
