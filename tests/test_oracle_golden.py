"""Pin the CPU oracle (oracle/isa_oracle.py) against the reference's golden
vectors: routing bit-exact, outputs to fp32 rounding. CPU only."""

import numpy as np
import pytest

from golden_cases import GoldenCase, case_names
from oracle import isa_oracle as O


@pytest.mark.parametrize("name", case_names())
def test_oracle_routing_matches_reference(name):
    c = GoldenCase(name)
    q, k, v = c.inputs()
    r = O.isa_routing(q, k, v, c.meta["l_src"], c.meta["l_ctx"], **c.oracle_kwargs())
    np.testing.assert_array_equal(r.selection, c.data["selection"])
    np.testing.assert_array_equal(r.sharp, c.data["sharp"])
    np.testing.assert_array_equal(r.flat, c.data["flat"])
    np.testing.assert_allclose(r.sharpness, c.data["sharpness"], rtol=1e-12, atol=1e-300)
    if r.mask is None:
        assert c.data["mask"].size == 0
    else:
        np.testing.assert_array_equal(r.mask, c.data["mask"])


@pytest.mark.parametrize("name", [n for n in case_names() if not n.startswith("mid_")])
def test_oracle_output_matches_reference(name):
    c = GoldenCase(name)
    q, k, v = c.inputs()
    out, _ = O.isa_forward(q, k, v, c.meta["l_src"], c.meta["l_ctx"], **c.oracle_kwargs())
    ref = c.data["out"]
    assert out.shape == ref.shape
    assert np.max(np.abs(out.astype(np.float64) - ref)) <= 1e-5 * max(1.0, np.abs(ref).max())
    if "full" in c.data:  # reduction identities (test_pipeline.py:33-61)
        full = O.full_attention(q, k, v)
        assert np.max(np.abs(full.astype(np.float64) - c.data["full"])) <= 1e-5
        assert np.max(np.abs(out.astype(np.float64) - c.data["full"])) <= 1e-5


def test_flop_accounting_matches_reference():
    from paper_2605_04569_b200.types import IclLayout, IsaConfig, IsaDims

    for name in case_names():
        c = GoldenCase(name)
        m = c.meta
        cfg = IsaConfig(**{k: v for k, v in c.cfg.items()})
        dims = IsaDims.derive((m["B"], m["H"], m["S"], m["D"]), IclLayout(m["l_src"], m["l_ctx"]), cfg)
        f = dims.flops()
        np.testing.assert_array_equal(
            np.array([f.exact_mas, f.taylor_mas, f.overhead_mas, f.dense_equivalent_mas]), c.data["flops"], err_msg=name)
