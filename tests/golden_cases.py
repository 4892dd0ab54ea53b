"""Loader for the committed golden vectors (made by tests/golden/make_golden.py
from the reference `isattn`). Inputs are regenerated with the oracle's
restatement of the reference workload generator and pinned by checksums."""

from __future__ import annotations

import glob
import json
import os

import numpy as np

from oracle.isa_oracle import round_bf16, workload

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def case_names():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN_DIR, "*.npz")))


class GoldenCase:
    def __init__(self, name: str):
        z = np.load(os.path.join(GOLDEN_DIR, name + ".npz"))
        self.meta = json.loads(str(z["meta"]))
        self.data = {k: z[k] for k in z.files if k != "meta"}
        self.name = name

    @property
    def cfg(self) -> dict:
        return dict(self.meta["cfg"])

    def inputs(self):
        m = self.meta
        q, k, v = workload(m["kind"], m["B"], m["H"], m["S"], m["D"], m["seed"])
        q, k, v = (round_bf16(x) for x in (q, k, v))
        sums = np.array([float(x.astype(np.float64).sum()) for x in (q, k, v)])
        if not np.allclose(sums, self.data["input_sums"], rtol=0, atol=1e-6 * max(1.0, np.abs(sums).max())):
            raise AssertionError(f"{self.name}: regenerated inputs do not match the reference's checksums")
        return q, k, v

    def oracle_kwargs(self) -> dict:
        c = self.cfg
        kw = {}
        for key in ("alpha_s", "alpha_ns", "alpha_f", "softmax_first", "scale", "gamma", "residual_softmax"):
            if key in c:
                kw[key] = c[key]
        return kw
