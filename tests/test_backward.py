"""isa_backward (pipeline.py:373-466) vs golden gradients of the reference
(tests/golden/bwd/*.npz, made by tests/golden/make_golden.py from `isattn`).
bf16 tensor arithmetic with fp32 accumulation: per tensor cosine >= 0.999 and
max-abs error <= 3e-2 x max |reference gradient|."""

import glob
import json
import os

import numpy as np
import pytest

from oracle import isa_oracle as O

BWD_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "bwd")
BWD_CASES = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(BWD_DIR, "*.npz")))


def _case(name):
    z = np.load(os.path.join(BWD_DIR, name + ".npz"))
    m = json.loads(str(z["meta"]))
    q, k, v = (O.round_bf16(x) for x in O.workload(m["kind"], m["B"], m["H"], m["S"], m["D"], m["seed"]))
    do = O.round_bf16(np.random.default_rng(m["seed"]).standard_normal(q.shape).astype(np.float32))
    sums = [float(x.astype(np.float64).sum()) for x in (q, k, v, do)]
    assert np.allclose(sums, m["input_sums"], rtol=0, atol=1e-6 * max(1.0, max(abs(s) for s in sums)))
    return m, (q, k, v, do), {n: z[n] for n in ("dq", "dk", "dv")}


def test_backward_golden_inputs_regenerate():
    for name in BWD_CASES:
        _case(name)


@pytest.mark.gpu
@pytest.mark.parametrize("name", BWD_CASES)
def test_backward_vs_reference(name):
    import torch

    import paper_2605_04569_b200 as P

    m, (q, k, v, do), ref = _case(name)
    dev = [torch.from_numpy(x).cuda().to(torch.bfloat16) for x in (q, k, v, do)]
    g = P.isa_backward(*dev[:3], P.IclLayout(m["l_src"], m["l_ctx"]), P.IsaConfig(**m["cfg"]), dev[3])
    for n in ("dq", "dk", "dv"):
        a = getattr(g, n).float().cpu().numpy().astype(np.float64).ravel()
        b = ref[n].astype(np.float64).ravel()
        err = float(np.max(np.abs(a - b)))
        cos = float(a @ b / (np.linalg.norm(a) * np.linalg.norm(b) + 1e-300))
        assert cos >= 0.999 and err <= 3e-2 * np.abs(b).max(), f"{n}: max_abs={err:.3e} (|ref|max {np.abs(b).max():.3e}) cos={cos:.6f}"


@pytest.mark.gpu
def test_backward_numpy_io_and_pinned_routing():
    import torch

    import paper_2605_04569_b200 as P

    m, (q, k, v, do), ref = _case("bwd_cfg1_iid_s20")
    icl, cfg = P.IclLayout(m["l_src"], m["l_ctx"]), P.IsaConfig(**m["cfg"])
    g = P.isa_backward(q, k, v, icl, cfg, do)
    assert isinstance(g.dq, np.ndarray) and g.dq.dtype == np.float32
    dev = [torch.from_numpy(x).cuda().to(torch.bfloat16) for x in (q, k, v, do)]
    r = P.isa_routing(*dev[:3], icl, cfg)
    g2 = P.isa_backward(*dev[:3], icl, cfg, dev[3], routing=r)
    g3 = P.isa_backward(*dev[:3], icl, cfg, dev[3])
    for n in ("dq", "dk", "dv"):
        assert torch.equal(getattr(g2, n), getattr(g3, n))


@pytest.mark.gpu
def test_backward_strided_inputs_and_fp32():
    """(B,S,H,D)-strided bf16 inputs give the same gradients as contiguous ones;
    fp32 inputs are computed in bf16 and returned as fp32."""
    import torch

    import paper_2605_04569_b200 as P

    m, (q, k, v, do), ref = _case("bwd_cfg1_iid_s20")
    icl, cfg = P.IclLayout(m["l_src"], m["l_ctx"]), P.IsaConfig(**m["cfg"])
    dev = [torch.from_numpy(x).cuda().to(torch.bfloat16) for x in (q, k, v, do)]
    g = P.isa_backward(*dev[:3], icl, cfg, dev[3])
    strided = [t.permute(0, 2, 1, 3).contiguous().permute(0, 2, 1, 3) for t in dev]
    assert not strided[0].is_contiguous()
    gs = P.isa_backward(*strided[:3], icl, cfg, strided[3])
    for n in ("dq", "dk", "dv"):
        assert torch.equal(getattr(g, n), getattr(gs, n))
    g32 = P.isa_backward(*(t.float() for t in dev[:3]), icl, cfg, dev[3].float())
    assert g32.dq.dtype == torch.float32
    for n in ("dq", "dk", "dv"):  # same fp32 gradients; the bf16 call rounds them on return
        assert torch.equal(getattr(g32, n).to(torch.bfloat16), getattr(g, n))


@pytest.mark.gpu
def test_backward_cta_pair_matches_single_cta(tmp_path):
    """The sharp-block dQ on CTA pairs (bwd_dq_pair_kernel, the default at D = 128)
    against the single-CTA dQ kernel (ISA_PAIR=0 in a child process, which also
    runs the forward recompute's K6 on single CTAs): same routing, gradients
    equal up to accumulation rounding; odd sharp-pair counts included (a
    padding CTA completes the last cluster)."""
    import subprocess
    import sys

    import torch

    import paper_2605_04569_b200 as P

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for S, ls in ((4096, 2048), (2048 + 640, 2048)):
        out = tmp_path / f"single_{S}.npz"
        code = (
            "import sys, torch, numpy as np; sys.path.insert(0, %r)\n"
            "import paper_2605_04569_b200 as P\n"
            "g = torch.Generator(device='cuda').manual_seed(%d)\n"
            "q, k, v, do = (torch.randn((1, 3, %d, 128), generator=g, device='cuda').to(torch.bfloat16) for _ in range(4))\n"
            "r = P.isa_backward(q, k, v, P.IclLayout(%d, %d), P.IsaConfig(strict=False), do)\n"
            "np.savez(%r, dq=r.dq.float().cpu().numpy(), dk=r.dk.float().cpu().numpy(), dv=r.dv.float().cpu().numpy())\n"
        ) % (root, S, S, ls, S - ls, str(out))
        env = dict(os.environ, ISA_PAIR="0")
        subprocess.run([sys.executable, "-c", code], check=True, env=env, timeout=600)
        ref = np.load(out)
        g = torch.Generator(device="cuda").manual_seed(S)
        q, k, v, do = (torch.randn((1, 3, S, 128), generator=g, device="cuda").to(torch.bfloat16) for _ in range(4))
        r = P.isa_backward(q, k, v, P.IclLayout(ls, S - ls), P.IsaConfig(strict=False), do)
        for name in ("dq", "dk", "dv"):
            a = getattr(r, name).float().cpu().numpy().astype(np.float64)
            b = ref[name].astype(np.float64)
            scale = np.abs(b).max()
            assert np.abs(a - b).max() <= 1e-2 * scale, (S, name, float(np.abs(a - b).max()), float(scale))


@pytest.mark.gpu
def test_backward_deterministic():
    """The reference's determinism contract for the backward: two calls on the same inputs give
    bit-identical gradients (fixed-order epilogues, slab-reduced centroid partials, no atomics
    on the gradients), with sharp CTA pairs, flat blocks and the centroid adjoint all active."""
    import torch

    import paper_2605_04569_b200 as P

    g = torch.Generator(device="cuda").manual_seed(77)
    q, k, v, do = (torch.randn((1, 3, 4096, 128), generator=g, device="cuda").to(torch.bfloat16) for _ in range(4))
    icl, cfg = P.IclLayout(2048, 2048), P.IsaConfig()
    a = P.isa_backward(q, k, v, icl, cfg, do)
    b = P.isa_backward(q, k, v, icl, cfg, do)
    for n in ("dq", "dk", "dv"):
        assert torch.equal(getattr(a, n), getattr(b, n)), n
