"""Golden fixtures for the bench CLI, the workload generator and ISA4 IO, made
by the REFERENCE (`isattn`). Run in the build container (needs /root/reference):

    python tests/golden/make_cli_golden.py

Writes
  tests/golden/workload/<name>.npz  `isattn.generate(spec)` outputs (workload.py:127-144)
  tests/golden/isa4/<name>.*        `isattn.workload.dump` containers (tensor.py:192-199)
  tests/golden/cli/<name>.csv       `isa-bench` CSV from the reference CLI (cli.py:277-338)

The GPU box never runs this; tests read only the committed files.
"""

from __future__ import annotations

import contextlib
import io
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from isattn import cli as ref_cli  # noqa: E402
from isattn.workload import WorkloadSpec, dump, generate  # noqa: E402

WORKLOADS = [
    # name, WorkloadSpec kwargs
    ("iid_f32", dict(kind="iid-gaussian", batch=1, heads=2, seq_len=128, dim=16)),
    ("clustered_f32", dict(kind="clustered", batch=2, heads=2, seq_len=160, dim=16, l_src=96, seed=3)),
    ("lowrank_f64", dict(kind="lowrank", batch=1, heads=2, seq_len=128, dim=16, precision="double", seed=5)),
    ("atten_clustered", dict(kind="clustered", batch=1, heads=2, seq_len=192, dim=16, context_attenuation=0.25,
                             seed=9)),
]

CLI_RUNS = [
    # name, argv (small: the reference CLI finishes each in seconds)
    ("isa_2048", ["--mode", "isa", "--seq-len", "2048", "--heads", "2", "--dim", "64", "--repeats", "1"]),
    ("taylor_2048", ["--mode", "taylor", "--seq-len", "2048", "--heads", "2", "--dim", "64"]),
    ("online_1024", ["--mode", "online", "--seq-len", "1024", "--heads", "2", "--dim", "64"]),
    ("full_1024", ["--mode", "full", "--seq-len", "1024", "--heads", "2", "--dim", "128"]),
    ("isa_gamma_rope", ["--mode", "isa", "--seq-len", "2048", "--heads", "2", "--dim", "64", "--gamma", "0.5",
                        "--rope", "--alpha-f", "0.25", "--seed", "4"]),
    ("sweep", ["--mode", "isa", "--seq-len", "1024,1536", "--alpha-f", "0.5,1.0", "--heads", "1", "--dim", "64",
               "--ctx-len", "512"]),
]


def main():
    os.makedirs(os.path.join(HERE, "workload"), exist_ok=True)
    for name, kw in WORKLOADS:
        q, k, v, icl = generate(WorkloadSpec(**kw))
        np.savez_compressed(os.path.join(HERE, "workload", f"{name}.npz"), q=q, k=k, v=v,
                            l_src=icl.l_src, l_ctx=icl.l_ctx, spec=repr(sorted(kw.items())))
    os.makedirs(os.path.join(HERE, "isa4"), exist_ok=True)
    q, k, v, icl = generate(WorkloadSpec(kind="clustered", heads=1, seq_len=24, dim=4, l_src=16, seed=2))
    dump(os.path.join(HERE, "isa4", "small"), q, k, v, icl, "single")
    q, k, v, icl = generate(WorkloadSpec(kind="iid-gaussian", heads=2, seq_len=8, dim=2, precision="double"))
    dump(os.path.join(HERE, "isa4", "small64"), q, k, v, icl, "double")
    os.makedirs(os.path.join(HERE, "cli"), exist_ok=True)
    for name, argv in CLI_RUNS:
        path = os.path.join(HERE, "cli", f"{name}.csv")
        err = io.StringIO()
        with contextlib.redirect_stderr(err):
            rc = ref_cli.main(argv + ["--out", path])
        with open(path, "a") as f:  # provenance line, skipped by the test's reader
            f.write(f"# argv: {' '.join(argv)}  exit={rc}\n")
        print(name, "exit", rc)


if __name__ == "__main__":
    main()
