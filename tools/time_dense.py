"""Time the dense sm_100a kernel: python tools/time_dense.py [H] [S] [libpath]"""
import sys, torch
sys.path.insert(0, ".")
from paper_2605_04569_b200 import _native as N
if len(sys.argv) > 3:
    N.load(sys.argv[3])
import paper_2605_04569_b200 as P
H = int(sys.argv[1]) if len(sys.argv) > 1 else 40
S = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
q, k, v = (torch.randn(1, H, S, 128, device="cuda").to(torch.bfloat16) for _ in range(3))
for _ in range(2):
    P.dense_attention(q, k, v)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(3):
    P.dense_attention(q, k, v)
b.record(); torch.cuda.synchronize()
ms = a.elapsed_time(b) / 3
fl = 4.0 * S * S * 128 * H
print(f"dense H={H} S={S}: {ms:.2f} ms  {fl/ms/1e9:.0f} TFLOP/s  lib={sys.argv[3] if len(sys.argv) > 3 else 'default'}")
