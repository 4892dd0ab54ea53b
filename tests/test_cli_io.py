"""Bench CLI, workload generator and ISA4 IO against fixtures made by the
reference (`tests/golden/make_cli_golden.py`): reference cli.py, workload.py,
tensor.py:192-219.

CPU: generator bit-equality, ISA4 byte-compatibility and error cases, CSV
format, FLOP columns, exit codes. GPU: the CLI's rows against the reference
CLI's rows for the same argv (knob/shape/FLOP columns exact, error columns close).
"""

from __future__ import annotations

import ast
import csv
import io
import math
import os
import struct

import numpy as np
import pytest

from paper_2605_04569_b200 import cli
from paper_2605_04569_b200.errors import FormatError, InputError, LayoutError
from paper_2605_04569_b200.tensorio import dump, load, load_tensor4, save_tensor4
from paper_2605_04569_b200.types import IclLayout, IsaConfig, IsaDims
from paper_2605_04569_b200.workload import WorkloadSpec, generate

GOLD = os.path.join(os.path.dirname(__file__), "golden")
WORKLOADS = sorted(f[:-4] for f in os.listdir(os.path.join(GOLD, "workload")) if f.endswith(".npz"))
CLI_RUNS = sorted(f[:-4] for f in os.listdir(os.path.join(GOLD, "cli")) if f.endswith(".csv"))
INT_COLS = ("schema_version", "S", "L_src", "L_ctx", "b", "seed", "mas_exact", "mas_taylor", "mas_dense_equiv")
KNOB_COLS = ("alpha_s", "alpha_ns", "alpha_f", "gamma")


def _read_csv(path_or_text):
    text = open(path_or_text).read() if os.path.exists(path_or_text) else path_or_text
    lines = text.splitlines()
    assert lines[0] == "# isa-bench schema_version=1"
    argv = [ln for ln in lines if ln.startswith("# argv:")]
    body = [ln for ln in lines[1:] if not ln.startswith("#")]
    rows = list(csv.DictReader(io.StringIO("\n".join(body))))
    return rows, (argv[0][len("# argv: "):].split("  exit=")[0].split() if argv else None)


@pytest.mark.parametrize("name", WORKLOADS)
def test_generator_bit_identical(name):
    g = np.load(os.path.join(GOLD, "workload", f"{name}.npz"))
    spec = WorkloadSpec(**dict(ast.literal_eval(str(g["spec"]))))
    q, k, v, icl = generate(spec)
    for ours, key in ((q, "q"), (k, "k"), (v, "v")):
        assert ours.dtype == g[key].dtype and np.array_equal(ours, g[key]), key
    assert (icl.l_src, icl.l_ctx) == (int(g["l_src"]), int(g["l_ctx"]))


def test_generator_spec_errors():
    from paper_2605_04569_b200.errors import ConfigError

    for kw in (dict(kind="nope"), dict(l_src=10, l_ctx=10, seq_len=30), dict(context_attenuation=1.5),
               dict(cluster_noise=-1.0), dict(precision="half"), dict(kind="loaded"), dict(heads=0)):
        with pytest.raises(ConfigError):
            WorkloadSpec(**kw).resolved()


@pytest.mark.parametrize("prefix,spec", [
    ("small", dict(kind="clustered", heads=1, seq_len=24, dim=4, l_src=16, seed=2)),
    ("small64", dict(kind="iid-gaussian", heads=2, seq_len=8, dim=2, precision="double")),
])
def test_isa4_reads_and_writes_reference_bytes(tmp_path, prefix, spec):
    ref = os.path.join(GOLD, "isa4", prefix)
    q, k, v, icl = load(ref)
    gq, gk, gv, gicl = generate(WorkloadSpec(**spec))
    assert icl == gicl
    for a, b in ((q, gq), (k, gk), (v, gv)):
        assert a.dtype == b.dtype and np.array_equal(a, b)
    ours = str(tmp_path / "x")
    dump(ours, q, k, v, icl, WorkloadSpec(**spec).resolved().precision)
    for suffix in (".q.isa4", ".k.isa4", ".v.isa4", ".meta"):
        assert open(ref + suffix, "rb").read() == open(ours + suffix, "rb").read(), suffix


def test_isa4_error_cases(tmp_path):
    good = tmp_path / "g.isa4"
    save_tensor4(good, np.ones((1, 2, 3, 4), np.float32))
    raw = good.read_bytes()
    assert raw[:4] == b"ISA4" and struct.unpack("<4I", raw[4:20]) == (1, 2, 3, 4) and len(raw) == 20 + 24 * 4
    cases = {
        "magic": (b"ISA5" + raw[4:], FormatError, "bad magic"),
        "header": (raw[:10], FormatError, "truncated header"),
        "zero": (raw[:4] + struct.pack("<4I", 1, 0, 3, 4) + raw[20:], FormatError, "zero dim"),
        "short": (raw[:-4], FormatError, "file ends at byte"),
        "long": (raw + b"\0\0\0\0", FormatError, "expected"),
        "nan": (raw[:20] + np.full(24, np.nan, np.float32).tobytes(), InputError, "non-finite"),
    }
    for name, (data, exc, msg) in cases.items():
        p = tmp_path / f"{name}.isa4"
        p.write_bytes(data)
        with pytest.raises(exc, match=msg):
            load_tensor4(p)
    with pytest.raises(LayoutError):
        save_tensor4(tmp_path / "bad.isa4", np.ones((2, 3), np.float32))
    # sidecar: unparsable, unknown precision, length mismatch
    pre = str(tmp_path / "w")
    x = np.zeros((1, 1, 8, 2), np.float32)
    dump(pre, x, x, x, IclLayout(5, 3))
    assert load(pre)[3] == IclLayout(5, 3)
    for text, exc in (("5\n", FormatError), ("5\n3\nquad\n", FormatError), ("5\n4\nsingle\n", LayoutError)):
        open(pre + ".meta", "w").write(text)
        with pytest.raises(exc):
            load(pre)


def test_cli_exit_codes(tmp_path, capsys):
    assert cli.main(["--alpha-s", "2"]) == 2
    assert cli.main(["--alpha-ns", "0"]) == 2
    assert cli.main(["--repeats", "0"]) == 2
    assert cli.main(["--block-size", "32"]) == 2  # only b = 64 on the sm_100a kernels
    assert cli.main(["--precision", "double"]) == 2  # bf16 tensor-core path only
    assert cli.main(["--load", str(tmp_path / "missing")]) == 4
    err = capsys.readouterr().err
    assert "config error" in err and "io error" in err


def test_csv_format_matches_reference(tmp_path):
    ref_rows, _ = _read_csv(os.path.join(GOLD, "cli", "isa_2048.csv"))
    out = tmp_path / "o.csv"
    cli.write_csv(ref_rows, str(out))
    ref_lines = open(os.path.join(GOLD, "cli", "isa_2048.csv")).read().splitlines()
    ours = out.read_text().splitlines()
    assert ours[:2] == ref_lines[:2]  # schema comment + header
    assert ours[2:] == ref_lines[2:2 + len(ours) - 2]


@pytest.mark.parametrize("name", CLI_RUNS)
def test_flop_columns_match_reference(name):
    """mas_* columns from our FLOP accounting equal the reference CLI's, row by row."""
    rows, argv = _read_csv(os.path.join(GOLD, "cli", f"{name}.csv"))
    args = cli.build_parser().parse_args(argv)
    for r in rows:
        if r["repeat"] == "failed":
            continue
        S, b, D, H = int(r["S"]), int(r["b"]), args.dim, args.heads
        if r["mode"] in ("full", "online"):
            fc = cli.dense_flops(1, H, S, b, D)
        elif r["mode"] == "taylor":
            fc = cli.taylor_flops(1, H, S, b, D, float(r["alpha_ns"]))
        else:
            cfg = IsaConfig(alpha_s=float(r["alpha_s"]), alpha_ns=float(r["alpha_ns"]), alpha_f=float(r["alpha_f"]),
                            gamma=float(r["gamma"]))
            fc = IsaDims.derive((1, H, S, D), IclLayout(int(r["L_src"]), int(r["L_ctx"])), cfg).flops()
        assert (fc.exact_mas, fc.taylor_mas, fc.dense_equivalent_mas) == (
            int(r["mas_exact"]), int(r["mas_taylor"]), int(r["mas_dense_equiv"]))


@pytest.mark.gpu
@pytest.mark.parametrize("name", CLI_RUNS)
def test_cli_rows_match_reference(tmp_path, name):
    ref_rows, argv = _read_csv(os.path.join(GOLD, "cli", f"{name}.csv"))
    out = tmp_path / "o.csv"
    assert cli.main(argv + ["--out", str(out)]) == 0
    rows, _ = _read_csv(str(out))
    assert len(rows) == len(ref_rows)
    for ours, ref in zip(rows, ref_rows):
        assert ours["mode"] == ref["mode"] and ours["repeat"] == ref["repeat"]
        for c in INT_COLS:
            assert int(ours[c]) == int(ref[c]), c
        for c in KNOB_COLS:
            assert float(ours[c]) == float(ref[c]), c
        for c in ("t_total_us", "t_kernel_us"):
            assert float(ours[c]) > 0
        if ref["mode"] == "full":
            assert math.isnan(float(ours["max_rel_err"]))
            continue
        # same routing (bit-exact from the fp32 inputs); the kernels compute on
        # bf16 operands: the error columns agree to ~1e-2
        for c in ("max_rel_err", "mean_rel_err"):
            a, r = float(ours[c]), float(ref[c])
            assert abs(a - r) <= 0.02 + 0.03 * r, (c, a, r)


@pytest.mark.gpu
def test_cli_dump_then_load_replays(tmp_path):
    pre = str(tmp_path / "w")
    a, b = tmp_path / "a.csv", tmp_path / "b.csv"
    base = ["--seq-len", "1024", "--heads", "2", "--dim", "64", "--seed", "3"]
    assert cli.main(base + ["--dump", pre, "--out", str(a)]) == 0
    assert cli.main(["--load", pre, "--out", str(b)]) == 0
    ra, _ = _read_csv(str(a))
    rb, _ = _read_csv(str(b))
    for x, y in zip(ra, rb):
        for c in INT_COLS + ("max_rel_err", "mean_rel_err"):
            if c != "seed":  # --load keeps the command line's seed (cli.py:137-141)
                assert x[c] == y[c], c
