"""GPU parity of the sm_100a path against the reference golden vectors and the
CPU oracle. Routing must match bit-exactly; outputs within the north-star
tolerance (bf16 compute): max-abs <= 2e-2 and cosine >= 0.999 versus the fp32
reference output."""

import ctypes
import math

import numpy as np
import pytest
import torch

from golden_cases import GoldenCase, case_names
from oracle import isa_oracle as O

pytestmark = pytest.mark.gpu

MAX_ABS = 2e-2
MIN_COS = 0.999


def _api():
    import paper_2605_04569_b200 as P

    return P


def _bf16(x: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda().to(torch.bfloat16)


def _close(out, ref, max_abs=MAX_ABS, min_cos=MIN_COS):
    a = out.detach().float().cpu().numpy().astype(np.float64).ravel() if isinstance(out, torch.Tensor) else \
        np.asarray(out, dtype=np.float64).ravel()
    b = np.asarray(ref, dtype=np.float64).ravel()
    err = float(np.max(np.abs(a - b)))
    cos = float(a @ b / (np.linalg.norm(a) * np.linalg.norm(b) + 1e-300))
    assert err <= max_abs and cos >= min_cos, f"max_abs={err:.3e} cos={cos:.6f}"
    return err, cos


def _cfg(case):
    P = _api()
    return P.IsaConfig(**case.cfg)


# ------------------------------------------------------------------ K1 pooling
@pytest.mark.parametrize("D,l_src,l_ctx", [(64, 1024, 1024), (128, 1000, 1100), (128, 960, 0)])
def test_pool_means_bit_exact(D, l_src, l_ctx):
    from paper_2605_04569_b200 import _native as N

    rng = np.random.default_rng(D + l_src)
    S = l_src + l_ctx
    q, k, v = (O.round_bf16(rng.standard_normal((1, 3, S, D)).astype(np.float32) * 3) for _ in range(3))
    T = -(-l_src // 64) + (-(-l_ctx // 64) if l_ctx else 0)
    means = torch.empty((3, 1, 3, T, D), dtype=torch.float32, device="cuda")
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    tq, tk, tv = _bf16(q), _bf16(k), _bf16(v)
    sh = N.IsaShape(1, 3, S, D, l_src, l_ctx, 64, 0, tq.stride(0), tq.stride(1), tq.stride(2))
    N.check(N.load().isa_pool_means(ctypes.byref(sh), tq.data_ptr(), tk.data_ptr(), tv.data_ptr(), means.data_ptr(),
                                    err.data_ptr(), torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    for i, x in enumerate((q, k, v)):
        ref = O.icl_means(x, l_src, l_ctx, 64)
        np.testing.assert_array_equal(means[i].cpu().numpy(), ref)
    assert int(err.item()) == 0


# ------------------------------------------------------------------ routing primitives (test_coarse.py KATs)
def _topk(scores, k, method):
    from paper_2605_04569_b200 import _native as N

    s = torch.as_tensor(np.atleast_2d(np.asarray(scores, dtype=np.float64))).cuda()
    out = torch.empty((s.shape[0], k), dtype=torch.int64, device="cuda")
    N.check(N.load().isa_topk_rows_f64(s.data_ptr(), s.shape[0], s.shape[1], k, out.data_ptr(), method,
                                       torch.cuda.current_stream().cuda_stream))
    return out.cpu().numpy()


@pytest.mark.parametrize("method", [0, 1, 2])
def test_topk_known_answers(method):
    # argmax / top-2 / ties to the lowest index (test_coarse.py:71-84)
    assert _topk([0.1, 0.9, 0.3], 1, method).tolist() == [[1]]
    assert _topk([0.1, 0.9, 0.3, 0.8], 2, method).tolist() == [[1, 3]]
    assert _topk([0.5, 0.5, 0.5, 0.1], 2, method).tolist() == [[0, 1]]
    # mask argmax [1,7,3,5] at alpha_ns = 0.25 -> {1} (test_coarse.py:141-144)
    assert _topk([1.0, 7.0, 3.0, 5.0], 1, method).tolist() == [[1]]
    # random rows vs the sort oracle (test_coarse.py:157-167), with injected ties
    rng = np.random.default_rng(7)
    x = np.round(rng.standard_normal((37, 300)), 1)
    for k in (1, 5, 37, 150, 300):
        np.testing.assert_array_equal(_topk(x, k, method), O.topk_rows(x, k))


def test_split_and_sharpness_known_answers():
    from paper_2605_04569_b200 import _native as N

    lib = N.load()
    st = torch.cuda.current_stream().cuda_stream

    def split(m, n_flat):
        t = torch.as_tensor(np.atleast_2d(np.asarray(m, dtype=np.float64))).cuda()
        r, n = t.shape
        sharp = torch.empty((r, n - n_flat), dtype=torch.int64, device="cuda")
        flat = torch.empty((r, n_flat), dtype=torch.int64, device="cuda")
        N.check(lib.isa_split_rows_f64(t.data_ptr(), r, n, n_flat, sharp.data_ptr(), flat.data_ptr(), st))
        return sharp.cpu().numpy(), flat.cpu().numpy()

    # sort oracle M = (0.3, 0.1, 0.4, 0.1) -> flat {1, 3} (test_coarse.py:194-203)
    s, f = split([0.3, 0.1, 0.4, 0.1], 2)
    assert f.tolist() == [[1, 3]] and s.tolist() == [[0, 2]]
    # boundary tie keeps the lower index sharp (test_coarse.py:205-212)
    s, f = split([0.2, 0.2, 0.2, 0.2], 1)
    assert f.tolist() == [[3]]
    rng = np.random.default_rng(3)
    m = np.round(rng.random((20, 257)), 2)
    for n_flat in (0, 1, 100, 257):
        s, f = split(m, n_flat)
        order = np.argsort(-m, axis=-1, kind="stable")
        np.testing.assert_array_equal(s, np.sort(order[:, : 257 - n_flat], axis=-1))
        np.testing.assert_array_equal(f, np.sort(order[:, 257 - n_flat:], axis=-1))

    def sharp(x, sf):
        t = torch.as_tensor(np.atleast_2d(np.asarray(x, dtype=np.float64))).cuda()
        out = torch.empty(t.shape[0], dtype=torch.float64, device="cuda")
        N.check(lib.isa_sharpness_rows_f64(t.data_ptr(), t.shape[0], t.shape[1], sf, out.data_ptr(), st))
        return out.cpu().numpy()

    # one-hot raw variance = 0.1875 (test_coarse.py:182-192)
    assert abs(sharp([1.0, 0.0, 0.0, 0.0], 0)[0] - 0.1875) < 1e-15
    assert sharp([2.0, 2.0, 2.0], 1)[0] == 0.0
    x = rng.standard_normal((50, 130)) * 3
    np.testing.assert_allclose(sharp(x, 1), O.softmax_rows(x).var(axis=-1), rtol=1e-12)
    np.testing.assert_allclose(sharp(x, 0), x.var(axis=-1), rtol=1e-12)


# ------------------------------------------------------------------ dense kernel (K8)
@pytest.mark.parametrize("D,S", [(64, 1024), (128, 2048), (128, 1000)])
def test_dense_attention_vs_torch_fp32(D, S):
    P = _api()
    torch.manual_seed(D + S)
    q, k, v = (torch.randn(1, 2, S, D, device="cuda").to(torch.bfloat16) for _ in range(3))
    out = P.dense_attention(q, k, v)
    ref = torch.softmax(q.float() @ k.float().transpose(-1, -2) / math.sqrt(D), dim=-1) @ v.float()
    _close(out, ref.cpu().numpy())


@pytest.mark.parametrize("growth", [0.5, 4.0, 40.0])
def test_dense_attention_rising_scores_vs_torch_fp32(growth):
    """Key norms grow along the sequence, so the running row max keeps jumping:
    exercises the speculative softmax path's fallback (tile max > m + 8 ->
    recompute with a forced rescale) on every few tiles, incl. jumps far
    beyond the exp2 range of a stale max (growth 40)."""
    P = _api()
    torch.manual_seed(7)
    S, D = 2048, 128
    q, k, v = (torch.randn(1, 2, S, D, device="cuda") for _ in range(3))
    ramp = torch.linspace(0.05, 1.0, S, device="cuda").pow(2) * growth
    k = k * ramp[None, None, :, None]
    q, k, v = (t.to(torch.bfloat16) for t in (q, k, v))
    out = P.dense_attention(q, k, v)
    ref = torch.softmax(q.float() @ k.float().transpose(-1, -2) / math.sqrt(D), dim=-1) @ v.float()
    assert torch.isfinite(out.float()).all()
    _close(out, ref.cpu().numpy())


# ------------------------------------------------------------------ routing vs reference golden vectors
@pytest.mark.parametrize("name", case_names())
def test_routing_bit_exact_vs_reference(name):
    P = _api()
    c = GoldenCase(name)
    q, k, v = c.inputs()
    m = c.meta
    r = P.isa_routing(_bf16(q), _bf16(k), _bf16(v), P.IclLayout(m["l_src"], m["l_ctx"]), _cfg(c))
    np.testing.assert_array_equal(r.selection.numpy(), c.data["selection"])
    np.testing.assert_array_equal(r.split.sharp.cpu().numpy(), c.data["sharp"])
    np.testing.assert_array_equal(r.split.flat.cpu().numpy(), c.data["flat"])
    np.testing.assert_allclose(r.split.sharpness.cpu().numpy(), c.data["sharpness"], rtol=1e-9, atol=1e-300)
    if c.data["mask"].size:
        np.testing.assert_array_equal(r.mask.numpy(), c.data["mask"])
    else:
        assert r.mask is None


@pytest.mark.parametrize("name", [n for n in case_names() if not n.startswith("mid_")])
def test_forward_vs_reference_output(name):
    P = _api()
    c = GoldenCase(name)
    q, k, v = c.inputs()
    m = c.meta
    out, trace = P.isa_forward(_bf16(q), _bf16(k), _bf16(v), P.IclLayout(m["l_src"], m["l_ctx"]), _cfg(c))
    _close(out, c.data["out"])
    np.testing.assert_array_equal(trace.selection.numpy(), c.data["selection"])
    f = trace.flops
    np.testing.assert_array_equal(np.array([f.exact_mas, f.taylor_mas, f.overhead_mas, f.dense_equivalent_mas]),
                                  c.data["flops"])


def test_numpy_io_drop_in():
    """numpy in -> numpy fp32 out, like the reference call sites (cli.py:123-126)."""
    P = _api()
    c = GoldenCase("cfg1_clustered_s1")
    q, k, v = c.inputs()
    out, _ = P.isa_forward(q, k, v, P.IclLayout(1024, 1024), P.IsaConfig())
    assert isinstance(out, np.ndarray) and out.dtype == np.float32
    _close(out, c.data["out"])


def test_forward_with_pinned_reference_routing():
    P = _api()
    c = GoldenCase("cfg1_iid_s0")
    q, k, v = c.inputs()
    icl = P.IclLayout(1024, 1024)
    r = P.isa_routing(_bf16(q), _bf16(k), _bf16(v), icl, P.IsaConfig())
    a = P.isa_forward_with_routing(_bf16(q), _bf16(k), _bf16(v), icl, P.IsaConfig(), r)
    b, _ = P.isa_forward(_bf16(q), _bf16(k), _bf16(v), icl, P.IsaConfig())
    assert torch.equal(a, b)


def test_value_ones_gives_ones():
    """Write-count / coverage (test_pipeline.py:74-81): V == 1 -> O == 1 everywhere."""
    P = _api()
    torch.manual_seed(0)
    q = torch.randn(1, 4, 4096, 128, device="cuda").to(torch.bfloat16)
    k = torch.randn_like(q)
    v = torch.ones_like(q)
    out, _ = P.isa_forward(q, k, v, P.IclLayout(2048, 2048), P.IsaConfig(), collect_trace=False)
    assert torch.all(out == 1)


def test_all_sharp_equals_dense():
    """ISA(alpha_s=1, alpha_f=0) == dense attention (test_pipeline.py:34-40)."""
    P = _api()
    torch.manual_seed(1)
    q, k, v = (torch.randn(1, 2, 4096, 128, device="cuda").to(torch.bfloat16) for _ in range(3))
    out, _ = P.isa_forward(q, k, v, P.IclLayout(2048, 2048), P.IsaConfig(alpha_s=1.0, alpha_f=0.0))
    dense = P.dense_attention(q, k, v)
    _close(out, dense.float().cpu().numpy(), max_abs=1e-2, min_cos=0.9999)


@pytest.mark.parametrize("kind", ["iid-gaussian", "clustered"])
def test_wan_shaped_head_subset_vs_oracle(kind):
    """cfg2 geometry (8K + 8K, D = 128) on 2 heads (heads are independent)."""
    P = _api()
    q, k, v = O.workload(kind, 1, 2, 16384, 128, seed=21)
    q, k, v = (O.round_bf16(x) for x in (q, k, v))
    out_ref, r_ref = O.isa_forward(q, k, v, 8192, 8192)
    out, trace = P.isa_forward(_bf16(q), _bf16(k), _bf16(v), P.IclLayout(8192, 8192), P.IsaConfig())
    np.testing.assert_array_equal(trace.selection.numpy(), r_ref.selection)
    np.testing.assert_array_equal(trace.split.flat.cpu().numpy(), r_ref.flat)
    np.testing.assert_array_equal(trace.mask.numpy(), r_ref.mask)
    _close(out, out_ref)


def test_fp32_inputs():
    P = _api()
    c = GoldenCase("d128_clustered_s4")
    q, k, v = c.inputs()
    out, _ = P.isa_forward(torch.from_numpy(q).cuda(), torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda(),
                           P.IclLayout(1024, 1024), P.IsaConfig())
    assert out.dtype == torch.float32
    _close(out, c.data["out"])


def test_nonfinite_input_raises():
    P = _api()
    q = torch.randn(1, 1, 256, 64, device="cuda").to(torch.bfloat16)
    k, v = torch.randn_like(q), torch.randn_like(q)
    q[0, 0, 5, 3] = float("nan")
    with pytest.raises(P.InputError):
        P.isa_forward(q, k, v, P.IclLayout(128, 128), P.IsaConfig())


# ------------------------------------------------------------------ host-streamed path (isa_forward_host)
@pytest.mark.parametrize("hpc", [0, 1, 4])
def test_host_streamed_matches_device_path(hpc):
    """CPU (pinned) bf16 tensors stream through the GPU in head chunks; the
    result and the routing equal the all-device call bit-for-bit (heads are
    independent, reference.py:159-160). hpc=4 leaves a ragged last chunk."""
    P = _api()
    rng = np.random.default_rng(11)
    H, S, D = 6, 2048, 128
    q, k, v = (torch.from_numpy(O.round_bf16(rng.standard_normal((1, H, S, D)).astype(np.float32)))
               .to(torch.bfloat16) for _ in range(3))
    icl, cfg = P.IclLayout(1024, 1024), P.IsaConfig()
    ref, rtr = P.isa_forward(q.cuda(), k.cuda(), v.cuda(), icl, cfg)
    qh, kh, vh = (t.pin_memory() for t in (q, k, v))
    out, tr = P.isa_forward(qh, kh, vh, icl, cfg, heads_per_chunk=hpc)
    assert not out.is_cuda and out.dtype == torch.bfloat16
    assert torch.equal(out, ref.cpu())
    assert torch.equal(tr.selection.indices, rtr.selection.indices)
    assert torch.equal(tr.split.sharp, rtr.split.sharp) and torch.equal(tr.split.flat, rtr.split.flat)
    assert torch.equal(tr.mask.indices, rtr.mask.indices)
    assert tr.stage_times_us["kernel"] > 0


def test_host_streamed_unpinned_and_pinned_routing():
    """Pageable host memory works too (no overlap); isa_forward_with_routing on
    host data takes the reference's numpy routing."""
    P = _api()
    c = GoldenCase("cfg1_iid_s0")
    q, k, v = c.inputs()
    icl, cfg = P.IclLayout(1024, 1024), P.IsaConfig()
    qt, kt, vt = (torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(torch.bfloat16) for x in (q, k, v))
    out, _ = P.isa_forward(qt, kt, vt, icl, cfg, heads_per_chunk=1)
    _close(out, c.data["out"])
    r = P.isa_routing(_bf16(q), _bf16(k), _bf16(v), icl, cfg)
    a = P.isa_forward_with_routing(qt, kt, vt, icl, cfg, r)
    assert torch.equal(a, out)


def test_mixed_host_and_device_inputs_rejected():
    P = _api()
    x = torch.zeros(1, 1, 128, 64, dtype=torch.bfloat16)
    with pytest.raises(P.LayoutError):
        P.isa_forward(x, x.cuda(), x, P.IclLayout(64, 64), P.IsaConfig())
