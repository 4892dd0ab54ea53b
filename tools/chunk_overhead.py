"""Cost of the chunked multi-GPU schedule on ONE GPU: the full 40-head layer as
one prepared call vs ShardedIsa(world=1) compute-only with chunks of 1/2/5
heads (two alternating compute streams). python tools/chunk_overhead.py"""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2605_04569_b200 as P  # noqa: E402
from paper_2605_04569_b200.parallel import ShardedIsa  # noqa: E402

H, S, D, L = 40, 65536, 128, 32768
dev = torch.device("cuda", 0)
q, k, v = bench.synth_qkv(list(range(H)), S, D, dev)
icl, cfg = P.IclLayout(L, L), P.IsaConfig()


def timeit(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


prep = P.prepare(q, k, v, icl, cfg)
print(f"one call, 40 heads: {timeit(prep):.2f} ms")
out = torch.empty_like(q)
for n_heads in (40, 5):
    one = P.prepare(q[:, :n_heads], k[:, :n_heads], v[:, :n_heads], icl, cfg)
    print(f"{n_heads:2d} heads, one call: {timeit(one):.2f} ms")
    for mode, ch in (("signal", 1), ("chunks", 1), ("chunks", 2), ("chunks", 5)):
        lay = ShardedIsa(q[:, :n_heads], k[:, :n_heads], v[:, :n_heads], icl, cfg, 1, chunk_heads=ch, mode=mode)
        t = timeit(lambda: lay(out[:, :n_heads], gather=False))
        t2 = timeit(lambda: lay(out[:, :n_heads]))
        print(f"{n_heads:2d} heads, {mode} (chunk {ch}): compute {t:.2f} ms, with per-head D2D copies {t2:.2f} ms")
        del lay
    del one
