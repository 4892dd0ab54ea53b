import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2605_04569_b200 as P
from oracle import isa_oracle as O
q, k, v = O.workload("iid-gaussian", 1, 1, 2048, 128, seed=0)
q, k, v = (O.round_bf16(x) for x in (q, k, v))
asm = O.OracleAssembly(q, k, v, 1024, 1024)
ref = asm.forward()
dev = [torch.from_numpy(x).cuda().to(torch.bfloat16) for x in (q, k, v)]
out, tr = P.isa_forward(*dev, P.IclLayout(1024, 1024), P.IsaConfig())
o = out.float().cpu().numpy()
err = np.abs(o - ref).max(axis=-1)[0, 0]  # per row
blk = err.reshape(-1, 64).max(axis=1)
print("flat blocks", asm.flat[0, 0])
print("sharp blocks", asm.sharp[0, 0])
print("per-block max err", np.round(blk, 3))
ones = torch.ones_like(dev[2])
out1, _ = P.isa_forward(dev[0], dev[1], ones, P.IclLayout(1024, 1024), P.IsaConfig())
print("V=1 per-block mean", np.round(out1.float().cpu().numpy()[0, 0].reshape(-1, 64, 128).mean(axis=(1, 2)), 3))

# ---- dump the Taylor plan from the workspace (replicates isa_capi.cu carve)
prep = P.prepare(*dev, P.IclLayout(1024, 1024), P.IsaConfig())
prep()
torch.cuda.synchronize()
d = prep.inp.dims
BH, T, D, S = d.B * d.H, d.T, d.D, d.S
t_new, k_ctx, n_flat, n_sharp, k = d.t_new, d.k_ctx, d.n_flat, d.n_sharp, max(d.k, 1)
tn_pad = (t_new + 127) // 128 * 128
W = tn_pad // 32
items_f = (n_flat + 3) // 4
u = min(2 * k, t_new)
max_tiles = max((u + 1) // 2, 1)
al = lambda x: (max(x, 1) + 255) // 256 * 256
sizes = [("err", 16), ("means", 12 * BH * T * D), ("s_new", 8 * BH * T * t_new), ("qsum", 8 * BH * D),
         ("flags", BH * max(T, d.t_ctx)), ("ctx", 8 * BH * d.t_ctx), ("sel", 4 * BH * k_ctx), ("kv_blk", 4 * BH * t_new),
         ("sharpness", 8 * BH * T), ("sharp", 4 * BH * n_sharp), ("flat", 4 * BH * n_flat), ("mask", 4 * BH * n_flat * k),
         ("bits", 4 * BH * n_flat * W), ("kc", 2 * BH * tn_pad * D), ("vc", 2 * BH * tn_pad * D), ("ctx_short", 4 * BH),
         ("tiles", 16 * BH * items_f * 2 * max_tiles), ("n_tiles", 4 * BH * items_f)]
off = {}
o = 0
for n, sz in sizes:
    off[n] = o
    o += al(sz)
ws = prep.ws
def view(n, cnt):
    return ws[off[n]: off[n] + 4 * cnt].view(torch.int32).cpu().numpy()
print("kv_blk", view("kv_blk", t_new))
print("flat", view("flat", n_flat), "mask", asm.mask[0, 0].ravel())
print("n_tiles", view("n_tiles", items_f), "max_tiles", max_tiles)
print("tiles", view("tiles", items_f * 2 * max_tiles * 4).reshape(items_f, 2, max_tiles, 4))
