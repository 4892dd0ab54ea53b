"""K6 / K8 A/B across library builds: per-launch CUDA-event time of the exact
(sharp) attention launch inside isa_forward at cfg3 (events 3 -> 4) and of the
dense kernel at 40 x 32768. python tools/ab_k6.py [reps]; ISA_B200_LIB picks the build."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2605_04569_b200 as P  # noqa: E402
from paper_2605_04569_b200 import _native as N  # noqa: E402
from paper_2605_04569_b200.pipeline import _ptr  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
q, k, v = bench.synth_qkv(list(range(40)), 65536, 128, torch.device("cuda", 0))
prep = P.prepare(q, k, v, P.IclLayout(32768, 32768), P.IsaConfig())
inp = prep.inp
k6, lay = [], []
for it in range(reps + 1):
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
    es = N.IsaEvents()
    for i, e in enumerate(evs):
        e.record()
        es.ev[i] = e.cuda_event
    N.check(N.load().isa_forward(ctypes.byref(inp.shape), ctypes.byref(inp.knobs), _ptr(inp.q), _ptr(inp.k),
                                 _ptr(inp.v), _ptr(prep.out), _ptr(prep.ws), prep.nbytes, None, None, _ptr(prep.err),
                                 ctypes.byref(es), torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    if it:
        k6.append(evs[3].elapsed_time(evs[4]))
        lay.append(evs[0].elapsed_time(evs[5]))
qd, kd, vd = (t[:, :, :32768].contiguous() for t in (q, k, v))
P.dense_attention(qd, kd, vd)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(reps):
    P.dense_attention(qd, kd, vd)
b.record()
torch.cuda.synchronize()
dense_ms = a.elapsed_time(b) / reps
f_sharp = 4 * 64 * 64 * 128 * 512 * 576 * 40
print(json.dumps({"lib": os.path.basename(os.environ.get("ISA_B200_LIB", "default")),
                  "k6_ms": sum(k6) / len(k6), "k6_tflops": f_sharp / (sum(k6) / len(k6)) / 1e9,
                  "layer_ms": sum(lay) / len(lay), "dense32k_ms": dense_ms,
                  "dense_tflops": 4 * 32768 ** 2 * 128 * 40 / dense_ms / 1e9}))
