"""Timeline of one bwd_dkv_tc_kernel CTA (blockIdx (ISA_TRACE, 0)) from an
ISA_TRACE build: per query tile, SM clocks of S^T/dP^T ready (softmax), P
arrival (warp 0 / warp 4), and the MMA warp's qo_full / p_full / issue times."""
import ctypes, os, sys, subprocess
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
LIB = os.path.join(ROOT, "paper_2605_04569_b200", "libisa_b200_tracebwd.so")
if "--build" in sys.argv:
    from paper_2605_04569_b200 import build as B
    os.environ["ISA_EXTRA_DEFINES"] = "ISA_TRACE=7"
    r = subprocess.run(B.nvcc_command(out=LIB), capture_output=True, text=True)
    print("built" if r.returncode == 0 else r.stderr[-2000:])
    raise SystemExit
import torch
from paper_2605_04569_b200 import _native as N
N._lib = None
lib = N.load(LIB)
lib.isa_debug_trace_copy.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
import paper_2605_04569_b200 as P
H, L = 40, 32768
q, k, v, do = (torch.randn(1, H, 2 * L, 128, device="cuda").to(torch.bfloat16) for _ in range(4))
P.isa_backward(q, k, v, P.IclLayout(L, L), P.IsaConfig(), do)
torch.cuda.synchronize()
buf = np.zeros((96, 2, 8), dtype=np.int64)
N.check(lib.isa_debug_trace_copy(buf.ctypes.data, buf.nbytes))
t = buf - buf[1, 0, 0]
print("unit | S_rdy  P_arr q0 q1 q2 q3 (group warps) | mma: qo_full  p_seen  issued | unit_dt(same group)")
for i in range(2, 40):
    a = t[i]
    q = " ".join(f"{a[1, w] - a[0, 0]:5d}" for w in range(4))
    print(f"{i:4d} | {a[0,0]:8d} {q} | {a[0,5]-a[0,0]:6d} {a[0,6]-a[0,0]:6d} {a[0,7]-a[0,0]:6d} | {t[i+2,0,0]-a[0,0]:6d}")
