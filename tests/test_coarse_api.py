"""Function-level routing drop-ins (`build_coarse`, `rank_context`,
`build_block_mask`, `sharpness_split`; reference coarse.py:110-201) against the
reference's own outputs (`tests/golden/coarse`, made by
`tests/golden/make_coarse_golden.py`): block means bit-exact, fp64 scores to
1e-12, every discrete decision bit-exact."""

from __future__ import annotations

import os

import numpy as np
import pytest

from oracle import isa_oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden", "coarse")
CASES = sorted(f[:-4] for f in os.listdir(GOLD) if f.endswith(".npz"))


def _segment_aligned(g) -> bool:
    """build_coarse's single BlockLayout over [src | ctx] equals the pipeline's
    per-segment blocks (pipeline.py:238-243) only when both segments are
    whole blocks."""
    ls, lc = int(g["params"][2]), int(g["params"][3])
    return ls % 64 == 0 and lc % 64 == 0


def make_inputs(B, H, S, D, seed):
    """Same draws as make_coarse_golden.make_inputs."""
    rng = np.random.default_rng(seed)
    return tuple(O.round_bf16(rng.standard_normal((B, H, S, D)).astype(np.float32)) for _ in range(3))


def case_inputs(g, name):
    """Inputs of a golden case: seeded draws, or the duplicated / near-tied
    context blocks of tests/golden/tie_inputs.py for the ties_* cases."""
    import sys

    B, H, ls, lc, D, seed = (int(x) for x in g["params"][:6])
    if name.startswith("ties"):
        sys.path.insert(0, GOLD.rsplit(os.sep, 1)[0])
        from tie_inputs import tie_inputs

        return tie_inputs(B, H, ls, lc, D, seed, float(g["params"][6]))
    return make_inputs(B, H, ls + lc, D, seed)


@pytest.mark.parametrize("name", CASES)
def test_oracle_reproduces_reference_saliency_bits(name):
    """The oracle (numpy, same operations as coarse.py:126,155) reproduces the
    reference's context saliency bit for bit, incl. the tie cases."""
    g = np.load(os.path.join(GOLD, f"{name}.npz"))
    if not _segment_aligned(g):
        pytest.skip("ragged segments: the pipeline blocks per segment, build_coarse does not")
    B, H, ls, lc, D, seed = (int(x) for x in g["params"][:6])
    q, k, v = case_inputs(g, name)
    asm = O.OracleAssembly(q, k, v, ls, lc, alpha_s=float(g["params"][6]))
    r = asm.routing()
    np.testing.assert_array_equal(r.ctx_scores, g["ctx"])
    np.testing.assert_array_equal(r.selection, g["sel"])


def test_errors_without_device():
    from paper_2605_04569_b200.coarse import CoarseSet, build_block_mask, rank_context, sharpness_split
    from paper_2605_04569_b200.errors import ConfigError
    from paper_2605_04569_b200.types import IclLayout

    import torch

    cs = CoarseSet(torch.zeros(1, 1, 4, 64), torch.zeros(1, 1, 4, 64), torch.zeros(1, 1, 4, 64),
                   torch.zeros(1, 1, 4, 4, dtype=torch.float64), 64)
    with pytest.raises(ConfigError):
        rank_context(cs, IclLayout(128, 128), 1.5)
    with pytest.raises(ConfigError):
        build_block_mask(cs, 0.0)
    with pytest.raises(ConfigError):
        sharpness_split(cs, IclLayout(128, 128), -0.1)
    assert cs.summary()["query_blocks"] == 4


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_matches_reference_golden(name):
    import paper_2605_04569_b200 as P
    from paper_2605_04569_b200.coarse import build_block_mask, build_coarse, rank_context, sharpness_split

    g = np.load(os.path.join(GOLD, f"{name}.npz"))
    B, H, ls, lc, D, seed = (int(x) for x in g["params"][:6])
    a_s, a_ns, a_f, sf = (float(x) for x in g["params"][6:])
    q, k, v = case_inputs(g, name)
    lay = P.BlockLayout(64, ls + lc)
    cs = build_coarse(q, k, v, lay, lay)  # numpy in -> numpy out, like the reference
    for key, t in (("qc", cs.qc), ("kc", cs.kc), ("vc", cs.vc)):
        assert isinstance(t, np.ndarray)
        np.testing.assert_array_equal(t, g[key], err_msg=key)
    # the fp64 scores are numpy einsum's own bits (coarse_dmma_kernel)
    np.testing.assert_array_equal(cs.s_coarse, g["s_coarse"])
    icl = P.IclLayout(ls, lc)
    sel = rank_context(cs, icl, a_s)
    assert isinstance(sel.indices, np.ndarray)
    np.testing.assert_array_equal(sel.numpy(), g["sel"])
    np.testing.assert_array_equal(build_block_mask(cs, a_ns).numpy(), g["mask"])
    split = sharpness_split(cs, icl, a_f, bool(sf))
    np.testing.assert_array_equal(split.sharp, g["sharp"])
    np.testing.assert_array_equal(split.flat, g["flat"])
    np.testing.assert_allclose(split.sharpness, g["sharpness"], rtol=1e-10, atol=1e-14)
    # torch in -> device tensors, same bits
    import torch

    cs_t = build_coarse(*(torch.from_numpy(x).cuda() for x in (q, k, v)), lay, lay)
    np.testing.assert_array_equal(cs_t.s_coarse.cpu().numpy(), g["s_coarse"])
    np.testing.assert_array_equal(rank_context(cs_t, icl, a_s).indices.cpu().numpy(), g["sel"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_pipeline_saliency_bits_and_selection(name):
    """The fused pipeline's context saliency (coarse_dmma_kernel over the source
    rows x context columns, then ctx_mean_kernel) equals the reference's
    s_coarse[:, :, :T_src, T_src:].mean(axis=2) bit for bit (coarse.py:155),
    so duplicated and near-tied context blocks at the top-k boundary select
    exactly what the reference selects."""
    import torch

    import paper_2605_04569_b200 as P

    g = np.load(os.path.join(GOLD, f"{name}.npz"))
    if not _segment_aligned(g):
        pytest.skip("ragged segments: the pipeline blocks per segment, build_coarse does not")
    B, H, ls, lc, D, seed = (int(x) for x in g["params"][:6])
    a_s, a_ns, a_f, sf = (float(x) for x in g["params"][6:])
    q, k, v = (torch.from_numpy(x).cuda().to(torch.bfloat16) for x in case_inputs(g, name))
    cfg = P.IsaConfig(alpha_s=a_s, alpha_ns=a_ns, alpha_f=a_f, softmax_first=bool(sf),
                      strict=ls % 64 == 0 and lc % 64 == 0)
    _, tr = P.isa_forward(q, k, v, P.IclLayout(ls, lc), cfg)
    np.testing.assert_array_equal(tr.ctx_scores.cpu().numpy(), g["ctx"])
    np.testing.assert_array_equal(tr.selection.numpy(), g["sel"])


@pytest.mark.gpu
def test_block_mean_seq_and_padded_inputs():
    """block_mean (tensor.py:96-119) on unpadded and pre-padded inputs (ragged last block)."""
    import torch

    import paper_2605_04569_b200 as P
    from paper_2605_04569_b200.coarse import block_mean

    g = np.load(os.path.join(GOLD, f"{CASES[0]}.npz"))
    B, H, ls, lc, D, seed = (int(x) for x in g["params"][:6])
    q, _, _ = make_inputs(B, H, ls + lc, D, seed)
    np.testing.assert_array_equal(block_mean(q, P.BlockLayout(64, ls + lc)), g["qc"])
    S = ls + lc - 37  # ragged: last block has 27 valid rows
    lay = P.BlockLayout(64, S)
    ref = O.block_mean(q[:, :, :S], 64)
    np.testing.assert_array_equal(block_mean(q[:, :, :S], lay), ref)
    padded = np.concatenate([q[:, :, :S], np.full((B, H, lay.padded_len - S, D), 7.0, np.float32)], axis=2)
    np.testing.assert_array_equal(block_mean(torch.from_numpy(padded).cuda(), lay).cpu().numpy(), ref)
