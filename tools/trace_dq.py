"""Per-CTA spans and one CTA's per-tile timeline of bwd_dq_tc_kernel from an
ISA_TRACE build (python tools/trace_dq.py --build [CTA], then run on the GPU):
CTA count, work-unit (64-key tile) histogram, busy fraction of the SMs over
the kernel span, and for CTA blockIdx (ISA_TRACE, 0) the SM-clock stamps of
softmax S-ready / dS-stored and the MMA warp's S/dP-issued / dS-seen."""
import ctypes, os, sys, subprocess
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
LIB = os.path.join(ROOT, "paper_2605_04569_b200", "libisa_b200_tracedq.so")
if "--build" in sys.argv:
    from paper_2605_04569_b200 import build as B
    cta = [a for a in sys.argv[1:] if not a.startswith("--")]
    os.environ["ISA_EXTRA_DEFINES"] = f"ISA_TRACE={cta[0] if cta else 7}," + (
        "ISA_TRACE_DQP" if "--pair" in sys.argv else "ISA_TRACE_DQ")
    r = subprocess.run(B.nvcc_command(out=LIB), capture_output=True, text=True)
    print("built" if r.returncode == 0 else r.stderr[-2000:])
    raise SystemExit
import torch
from paper_2605_04569_b200 import _native as N
N._lib = None
lib = N.load(LIB)
lib.isa_debug_trace_copy.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
lib.isa_debug_cta_copy.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
import paper_2605_04569_b200 as P
H, L = 40, 32768
q, k, v, do = (torch.randn(1, H, 2 * L, 128, device="cuda").to(torch.bfloat16) for _ in range(4))
P.isa_backward(q, k, v, P.IclLayout(L, L), P.IsaConfig(), do)
torch.cuda.synchronize()
cta = np.zeros((1 << 16, 4), dtype=np.int64)
N.check(lib.isa_debug_cta_copy(cta.ctypes.data, cta.nbytes))
cta = cta[cta[:, 1] > 0]
t0, t1 = cta[:, 0].min(), cta[:, 1].max()
dur = (cta[:, 1] - cta[:, 0]) / 1e3
span = (t1 - t0) / 1e3
print(f"CTAs {len(cta)}  kernel span {span:.0f} us  (first start -> last end)")
print(f"work units (64-key tiles): total {cta[:, 2].sum()}  max {cta[:, 2].max()}  "
      f"mean {cta[:, 2].mean():.1f}  per SM {cta[:, 2].sum() / 148:.0f}")
print(f"us per tile (CTA duration / tiles): median {np.median(dur / np.maximum(cta[:, 2], 1)):.3f}")
print(f"SM busy fraction over the span: {dur.sum() / (148 * span):.3f}")
hist = np.histogram(cta[:, 2], bins=[0, 1, 16, 64, 128, 256, 512, 768, 1024, 4096])
print("tiles histogram:", dict(zip([f"<{b}" for b in hist[1][1:]], hist[0].tolist())))
late = cta[np.argsort(cta[:, 1])[-5:]]
print("last CTAs to end (start us, end us, tiles):", [(round((a - t0) / 1e3), round((b - t0) / 1e3), int(n))
                                                       for a, b, n, _ in late])
buf = np.zeros((96, 2, 8), dtype=np.int64)
N.check(lib.isa_debug_trace_copy(buf.ctypes.data, buf.nbytes))
t = buf - buf[0, 1, 2]
print("tile | sdp_issued(i+1) dS_seen(i) | kv_seen(i) S_done(i) dS_stored(i) | prod_go(i) tma_issued(i) | clk")
for i in range(0, 40):
    a = t[i]
    print(f"{i:4d} | {a[1,2]:8d} {a[1,3]:8d} | {a[0,2]:8d} {a[0,1]:8d} {a[0,3]:8d} | {a[1,4]:8d} {a[1,5]:8d} | {t[i+1,1,3]-a[1,3]:6d}")
