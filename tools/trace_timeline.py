"""Per-step SM-clock timeline of one attention CTA (softmax / MMA events).

Build the instrumented library here (cross-compiles):
    python tools/trace_timeline.py --build
Run on the GPU box:
    python tools/trace_timeline.py [--heads 8 --seq 16384]
Stamps (isa_attn.cuh, ISA_TSTAMP): per step i and stage s
  0 S ready (softmax saw s_full)   1 S in registers    2 row max done
  3 exps + P stores issued         4 p_full arrived
  5 (MMA warp, s=0) K/V of step i resident   6 MMA warp saw p_full[s]
  7 PV_s(i-1) + QK_s(i) issued and committed
"""
import argparse
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
_LIB = os.path.join(ROOT, "paper_2605_04569_b200", "libisa_b200_trace{}.so")


class _Lib:
    @staticmethod
    def format(variant):  # file-name-safe variant tag (nvcc rejects ',' in output paths)
        return _LIB.format(variant.replace(",", "_").replace("=", "_"))


LIB = _Lib


def build(cta, variant):
    from paper_2605_04569_b200 import build as B

    os.environ["ISA_EXTRA_DEFINES"] = ",".join([f"ISA_TRACE={cta}"] + ([variant] if variant else []))
    cmd = B.nvcc_command(out=LIB.format(variant))
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        print(r.stderr[-3000:])
        raise SystemExit(1)
    print("built", LIB.format(variant))


def run(args):
    import numpy as np
    import torch

    from paper_2605_04569_b200 import _native as N

    N._lib = None
    lib = N.load(LIB.format(args.variant))
    lib.isa_debug_trace_copy.restype = ctypes.c_int
    lib.isa_debug_trace_copy.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
    import paper_2605_04569_b200 as P

    H, S, D = args.heads, args.seq, 128
    q, k, v = (torch.randn(1, H, S, D, device="cuda", dtype=torch.bfloat16) for _ in range(3))
    if args.isa:  # ISA forward, branches launched separately (trace CTA of the branch built for)
        prep = P.prepare(q, k, v, P.IclLayout(S // 2, S // 2), P.IsaConfig(), separate_branches=True)
        for _ in range(3):
            prep()
    else:
        for _ in range(3):
            P.dense_attention(q, k, v)
    torch.cuda.synchronize()
    buf = np.zeros((96, 2, 8), dtype=np.int64)
    N.check(lib.isa_debug_trace_copy(buf.ctypes.data, buf.nbytes))
    if args.k7t:  # one query block per CTA (isa_taylor_t.cuh): stage 0 only
        t = buf[:, 0] - buf[0, 0, 0]
        print("tile |  S_rdy  ld  chk  exp+st  arrive | mma_see(P_i) V_taken QK(i+2)_issued | tile_dt")
        n = int((buf[:, 0, 0] != 0).sum())
        for i in range(n):
            a = t[i]
            m = t[i + 1] if i + 1 < 96 else np.zeros(8, dtype=np.int64)
            dt = t[i + 1, 0] - a[0] if i + 1 < n else 0
            print(f"{i:4d} | {a[0]:7d} {a[1]-a[0]:4d} {a[2]-a[1]:4d} {a[3]-a[2]:6d} {a[4]-a[3]:6d} |"
                  f" {m[6]-a[4]:8d} {m[5]-m[6]:7d} {m[7]-m[5]:8d} | {dt:6d}")
        print(f"CTA span: {t[n - 1, 4]} clk for {n} tiles ({t[n - 1, 4] / max(n, 1):.0f} clk/tile)")
        u = buf[:, 1] - buf[0, 0, 0]
        print("tile | prodK_issue prodV_issue | PV_issued K_taken  (MMA warp, relative to V_taken of tile i)")
        for i in range(n):
            m = t[i + 1] if i + 1 < 96 else np.zeros(8, dtype=np.int64)
            w = u[i + 1] if i + 1 < 96 else np.zeros(8, dtype=np.int64)
            print(f"{i:4d} | {u[i, 4]:9d} {u[i, 5]:9d} | {w[0] - m[5]:8d} {w[1] - m[5]:8d}   Ktile(i+2) issued at {u[i + 2, 4] if i + 2 < 96 else 0}")
        return
    t = buf - buf[1, 0, 0]
    print("step st |  S_rdy   ld  exps st_wait  S->P(arrive) | mma_see issue | S_rdy(i+1)-issue | step_dt")
    for i in range(args.first, min(args.first + args.n, 95)):
        for s in range(2):
            a = t[i, s]
            nxt = t[i + 1, s, 0] - t[i + 1, s, 7] if i + 1 < 96 else 0
            dt = t[i + 1, s, 0] - a[0]
            print(f"{i:4d} {s}  | {a[0]:7d} {a[1]-a[0]:4d} {a[2]-a[1]:5d} {a[3]-a[2]:5d} {a[4]-a[0]:6d} |"
                  f" {t[i+1, s, 6]-a[4]:6d} {t[i+1, s, 7]-t[i+1, s, 6]:5d} | {nxt:6d} | {dt:6d}")
    steps = t[args.first + args.n, 0, 0] - t[args.first, 0, 0]
    print(f"avg clk/step over {args.n} steps: {steps / args.n:.0f} (ideal MMA 2048 at D=128)")
    cnt = np.zeros((3, 4), dtype=np.uint64)
    lib.isa_debug_count_copy.restype = ctypes.c_int
    lib.isa_debug_count_copy.argtypes = [ctypes.c_void_p, ctypes.c_int]
    N.check(lib.isa_debug_count_copy(cnt.ctypes.data, 0))
    for mode, name in enumerate(("dense", "exact", "taylor")):
        if cnt[mode].sum():
            print(f"softmax warp-tiles {name}: spec {cnt[mode][0]}  redo {cnt[mode][1]}  general {cnt[mode][2]}  skip {cnt[mode][3]}")
    if args.isa:
        return
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        P.dense_attention(q, k, v)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 5
    print(f"dense {H}x{S}: {ms:.3f} ms = {4 * S * S * D * H / ms / 1e9:.0f} TFLOP/s")


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--build", action="store_true")
    ap.add_argument("--variant", default="", help="extra define, e.g. ISA_EXP_NOSOFTMAX")
    ap.add_argument("--cta", type=int, default=5)
    ap.add_argument("--heads", type=int, default=8)
    ap.add_argument("--seq", type=int, default=16384)
    ap.add_argument("--first", type=int, default=20)
    ap.add_argument("--isa", action="store_true", help="trace an isa_forward (separate branches) instead of dense")
    ap.add_argument("--n", type=int, default=24)
    ap.add_argument("--k7t", action="store_true", help="print the one-block-per-CTA K7T layout (use with --isa)")
    a = ap.parse_args()
    if a.build:
        build(a.cta, a.variant)
    else:
        run(a)
