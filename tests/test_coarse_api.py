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


def make_inputs(B, H, S, D, seed):
    """Same draws as make_coarse_golden.make_inputs."""
    rng = np.random.default_rng(seed)
    return tuple(O.round_bf16(rng.standard_normal((B, H, S, D)).astype(np.float32)) for _ in range(3))


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
    q, k, v = make_inputs(B, H, ls + lc, D, seed)
    lay = P.BlockLayout(64, ls + lc)
    cs = build_coarse(q, k, v, lay, lay)
    for key, t in (("qc", cs.qc), ("kc", cs.kc), ("vc", cs.vc)):
        np.testing.assert_array_equal(t.cpu().numpy(), g[key], err_msg=key)
    np.testing.assert_allclose(cs.s_coarse.cpu().numpy(), g["s_coarse"], rtol=1e-12, atol=1e-12)
    icl = P.IclLayout(ls, lc)
    np.testing.assert_array_equal(rank_context(cs, icl, a_s).numpy(), g["sel"])
    np.testing.assert_array_equal(build_block_mask(cs, a_ns).numpy(), g["mask"])
    split = sharpness_split(cs, icl, a_f, bool(sf))
    np.testing.assert_array_equal(split.sharp.cpu().numpy(), g["sharp"])
    np.testing.assert_array_equal(split.flat.cpu().numpy(), g["flat"])
    np.testing.assert_allclose(split.sharpness.cpu().numpy(), g["sharpness"], rtol=1e-10, atol=1e-14)


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
