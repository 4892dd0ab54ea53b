// ISA backward with frozen routing (isa_backward, pipeline.py:373-466):
// gradients of the sharp branch (full_attention_backward, reference.py:173-225)
// and of the Taylor branch (taylor_sparse_backward, taylor.py:225-296), with
// the K_new gather adjoint (pipeline.py:423-433) fused into the key-major
// kernel's stores. gamma = 0.
//
// Softmax statistics come from the forward kernels (AttnParams::lse, log2
// domain: P = exp2(scale*log2e * q.k + log2(w) - lse)); rho = rowsum(dO * O).
// This file holds the mma.sync m16n8k16 bf16 -> fp32 centroid pass; the
// exact-pair dK/dV and the dQ kernels are tcgen05 (isa_bwd_tc.cuh):
//   bwd_dkv_kernel<CENTROID=1>: per tile of 64 K_new centroids, over all flat
//       query blocks: dkc, dvc (taylor.py:286-289), fp32 [BH][t_new][D]
#pragma once
#include "isa_ptx.cuh"

namespace isa {

struct BwdParams {
  int H, S, D;
  int l_src, l_ctx, t_src, t_ctx, t_new;
  int n_sharp, n_flat, k, W, tn_pad;
  float sl2;    // scale * log2(e)
  float scale;  // softmax scale (dS -> dQ/dK factor)
  const __nv_bfloat16 *q, *kx, *v, *dout;  // token-major with element strides below
  long long sb, sh, ss;                    // q/k/v strides
  long long db, dh, ds;                    // dout strides
  const float* lse;                        // [BH][S]
  const float* rho;                        // [BH][S]
  const int* sharp;                        // [BH][n_sharp]
  const int* flat;                         // [BH][n_flat]
  const int* mask;                         // [BH][n_flat][k] K_new indices
  const int* kv_blk;                       // [BH][t_new]
  const uint32_t* bits;                    // [BH][n_flat][W] member bits
  const __nv_bfloat16 *kc, *vc;            // [BH][tn_pad][D] K_new centroids
  float *dkc, *dvc;                        // [BH][t_new][D] (x c_splits partials before the reduce)
  float *dq, *dk, *dv;                     // [BH][S][D]
  int c_splits;                            // centroid kernel: flat query list split across gridDim.z
  long long c_part;                        // elements per partial dkc/dvc slab (BH * t_new * D)
};

__device__ __forceinline__ int bw_tok0(const BwdParams& p, int u) {
  return u < p.t_src ? u * 64 : p.l_src + (u - p.t_src) * 64;
}
__device__ __forceinline__ int bw_valid(const BwdParams& p, int u) {
  const int r = u < p.t_src ? p.l_src - u * 64 : p.l_ctx - (u - p.t_src) * 64;
  return r < 64 ? r : 64;
}

// ---------------------------------------------------------------- mma.sync helpers
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void ldsm4(uint32_t (&r)[4], uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void ldsm4t(uint32_t (&r)[4], uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}

// 64-row x D bf16 tile in shared memory, 16-byte chunks XOR-swizzled by row
// (conflict-free ldmatrix on 8 consecutive rows).
template <int D>
struct SmTile {
  static constexpr int kChunks = D / 8;
  __device__ __forceinline__ static uint32_t addr(uint32_t base, int row, int chunk) {
    return base + (uint32_t)(row * D * 2 + ((chunk ^ (row & 7)) << 4));
  }
};

// Cooperative load of `rows` valid rows (the rest zero) of a token-major bf16
// matrix (row stride `rs` elements) into a swizzled tile. 128 threads.
template <int D>
__device__ __forceinline__ void load_tile(uint8_t* sm, const __nv_bfloat16* src, long long rs, int rows) {
  constexpr int C = D / 8;
  const uint32_t base = smem_u32(sm);
  for (int e = threadIdx.x; e < 64 * C; e += 128) {
    const int r = e / C, c = e % C;
    uint4 val = make_uint4(0, 0, 0, 0);
    if (r < rows) val = *reinterpret_cast<const uint4*>(src + r * rs + c * 8);
    asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(SmTile<D>::addr(base, r, c)), "r"(val.x), "r"(val.y),
                 "r"(val.z), "r"(val.w));
  }
}

// Same tile load through cp.async (16-byte, zero-fill past `rows`); the
// caller commits / waits the group.
template <int D>
__device__ __forceinline__ void load_tile_async(uint8_t* sm, const __nv_bfloat16* src, long long rs, int rows) {
  constexpr int C = D / 8;
  const uint32_t base = smem_u32(sm);
  for (int e = threadIdx.x; e < 64 * C; e += 128) {
    const int r = e / C, c = e % C;
    const __nv_bfloat16* g = src + (r < rows ? r : 0) * rs + c * 8;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(SmTile<D>::addr(base, r, c)), "l"(g),
                 "r"(r < rows ? 16 : 0)
                 : "memory");
  }
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// A fragments (16 rows from row0, 16 columns from col0) of a swizzled tile.
template <int D>
__device__ __forceinline__ void frag_a(uint32_t (&a)[4], uint32_t base, int row0, int col0) {
  const int t = threadIdx.x & 31;
  ldsm4(a, SmTile<D>::addr(base, row0 + (t & 15), (col0 >> 3) + (t >> 4)));
}
// B fragments of two n8 tiles (n0, n0+8) x k16 from a [n][k] row-major tile.
template <int D>
__device__ __forceinline__ void frag_b(uint32_t (&b)[4], uint32_t base, int n0, int k0) {
  const int t = threadIdx.x & 31;
  ldsm4(b, SmTile<D>::addr(base, n0 + (t & 7) + ((t >> 4) << 3), (k0 >> 3) + ((t >> 3) & 1)));
}
// B fragments of two n8 tiles (n0, n0+8) x k16 from a [k][n] row-major tile.
template <int D>
__device__ __forceinline__ void frag_bt(uint32_t (&b)[4], uint32_t base, int k0, int n0) {
  const int t = threadIdx.x & 31;
  ldsm4t(b, SmTile<D>::addr(base, k0 + (t & 7) + (((t >> 3) & 1) << 3), (n0 >> 3) + (t >> 4)));
}

// ---------------------------------------------------------------- rho
// rho[bh][row] = sum_d dO * O (taylor.py:274; reference.py:218 in closed form).
__global__ void bwd_rho_kernel(const __nv_bfloat16* __restrict__ dout, long long db, long long dh, long long ds,
                               const __nv_bfloat16* __restrict__ o, int H, int S, int D, float* __restrict__ rho,
                               long long n_rows) {
  const long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= n_rows) return;
  const int bh = static_cast<int>(w / S), tok = static_cast<int>(w % S);
  const __nv_bfloat16* a = dout + (bh / H) * db + (bh % H) * dh + tok * ds;
  const __nv_bfloat16* b = o + w * D;
  float acc = 0.f;
  for (int d = lane * 2; d < D; d += 64) {
    const float2 x = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(a + d));
    const float2 y = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(b + d));
    acc = fmaf(x.x, y.x, fmaf(x.y, y.y, acc));
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (lane == 0) rho[w] = acc;
}

// ---------------------------------------------------------------- dK/dV (key-major)
// CTA = 64 keys (a K_new block, or a tile of 64 centroids), 4 warps x 16 keys;
// loops over the query blocks that see those keys, Q/dO tiles double-buffered
// with cp.async (plus per-buffer lse, rho and the centroid exclusion mask).
template <int D, int CENTROID>
__global__ void __launch_bounds__(128, 2) bwd_dkv_kernel(const BwdParams p) {
  extern __shared__ __align__(128) uint8_t smem_bw[];
  constexpr int TB = 64 * D * 2;
  uint8_t* sK = smem_bw;
  uint8_t* sV = smem_bw + TB;
  uint8_t* sQO = smem_bw + 2 * TB;  // [2 buffers][Q, dO]
  float* sLse = reinterpret_cast<float*>(smem_bw + 6 * TB);  // [2][64]
  float* sRho = sLse + 128;                                    // [2][64]
  uint32_t* sMem = reinterpret_cast<uint32_t*>(sRho + 128);  // [2][2] centroid member words
  int* sList = reinterpret_cast<int*>(sMem + 4);             // query-block list (positions)
  __shared__ int s_count;
  const int bh = blockIdx.y;
  const int hh = bh % p.H, bb = bh / p.H;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, tig = lane & 3;
  int vk = 64, uk = 0, j = 0, c0 = 0;
  if (!CENTROID) {
    j = blockIdx.x;
    uk = p.kv_blk[(long long)bh * p.t_new + j];
    vk = bw_valid(p, uk);
    const long long off = bb * p.sb + hh * p.sh + (long long)bw_tok0(p, uk) * p.ss;
    load_tile_async<D>(sK, p.kx + off, p.ss, vk);
    load_tile_async<D>(sV, p.v + off, p.ss, vk);
  } else {
    c0 = blockIdx.x * 64;
    const long long off = ((long long)bh * p.tn_pad + c0) * D;
    load_tile_async<D>(sK, p.kc + off, D, 64);
    load_tile_async<D>(sV, p.vc + off, D, 64);
  }
  cp_commit();
  // query blocks: [sharp ...] (exact only) then the flat ones (exact: listing j; centroid: all)
  if (threadIdx.x == 0) s_count = 0;
  __syncthreads();
  if (!CENTROID)
    for (int x = threadIdx.x; x < p.n_sharp; x += 128) sList[x] = x;
  const int base = CENTROID ? 0 : p.n_sharp;
  for (int f = threadIdx.x; f < p.n_flat; f += 128) {
    bool take = true;
    if (!CENTROID) take = (p.bits[((long long)bh * p.n_flat + f) * p.W + (j >> 5)] >> (j & 31)) & 1u;
    if (take) sList[base + atomicAdd(&s_count, 1)] = p.n_sharp + f;
  }
  __syncthreads();
  int li0 = 0, n_list = base + s_count;
  if (CENTROID && p.c_splits > 1) {  // this CTA's share of the flat list (gridDim.z-way split)
    const int per = (n_list + p.c_splits - 1) / p.c_splits;
    li0 = blockIdx.z * per;
    n_list = min(n_list, li0 + per);
  }
  auto prefetch = [&](int li, int buf) {
    const int x = sList[li];
    const bool is_flat = x >= p.n_sharp;
    const int f = x - p.n_sharp;
    const int u = is_flat ? p.flat[bh * p.n_flat + f] : p.sharp[bh * p.n_sharp + x];
    const int tok = bw_tok0(p, u), vq = bw_valid(p, u);
    uint8_t* sQ = sQO + buf * 2 * TB;
    load_tile_async<D>(sQ, p.q + bb * p.sb + hh * p.sh + tok * p.ss, p.ss, vq);
    load_tile_async<D>(sQ + TB, p.dout + bb * p.db + hh * p.dh + tok * p.ds, p.ds, vq);
    const long long rowbase = (long long)bh * p.S + tok;
    if (threadIdx.x < 64) {
      const int r = threadIdx.x;
      sLse[buf * 64 + r] = r < vq ? p.lse[rowbase + r] : -INFINITY;
      sRho[buf * 64 + r] = r < vq ? p.rho[rowbase + r] : 0.f;
    } else if (CENTROID && threadIdx.x < 66) {  // this query block's members among the 64 centroids
      const int w = threadIdx.x - 64;
      const uint32_t* mb = p.bits + ((long long)bh * p.n_flat + f) * p.W;
      sMem[buf * 2 + w] = mb[(c0 >> 5) + w];
    }
    cp_commit();
  };
  // per-key bias (log2 of the centroid weight; -inf = invalid key row)
  const int kr0 = warp * 16 + g, kr1 = kr0 + 8;
  float kb0 = kr0 < vk ? 0.f : -INFINITY, kb1 = kr1 < vk ? 0.f : -INFINITY;
  if (CENTROID) {
    kb0 = c0 + kr0 < p.t_new ? __log2f((float)bw_valid(p, p.kv_blk[(long long)bh * p.t_new + c0 + kr0])) : -INFINITY;
    kb1 = c0 + kr1 < p.t_new ? __log2f((float)bw_valid(p, p.kv_blk[(long long)bh * p.t_new + c0 + kr1])) : -INFINITY;
  }
  float dk[D / 8][4], dv[D / 8][4];
#pragma unroll
  for (int n = 0; n < D / 8; ++n)
#pragma unroll
    for (int e = 0; e < 4; ++e) dk[n][e] = dv[n][e] = 0.f;
  if (n_list > li0) prefetch(li0, 0);
  const uint32_t bk = smem_u32(sK), bvv = smem_u32(sV);
  for (int li = li0; li < n_list; ++li) {
    const int buf = (li - li0) & 1;
    if (li + 1 < n_list) {
      prefetch(li + 1, buf ^ 1);
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    const uint32_t bq = smem_u32(sQO + buf * 2 * TB), bo = bq + TB;
    const float* lse = sLse + buf * 64;
    const float* rho = sRho + buf * 64;
    // S^T = K Q^T, dP^T = V dO^T (16 keys x 64 queries per warp)
    float sc[8][4], dp[8][4];
#pragma unroll
    for (int n = 0; n < 8; ++n)
#pragma unroll
      for (int e = 0; e < 4; ++e) sc[n][e] = dp[n][e] = 0.f;
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
      uint32_t ak[4], av[4];
      frag_a<D>(ak, bk, warp * 16, kk * 16);
      frag_a<D>(av, bvv, warp * 16, kk * 16);
#pragma unroll
      for (int n = 0; n < 8; n += 2) {
        uint32_t b[4];
        frag_b<D>(b, bq, n * 8, kk * 16);
        mma16816(sc[n], ak, b[0], b[1]);
        mma16816(sc[n + 1], ak, b[2], b[3]);
        frag_b<D>(b, bo, n * 8, kk * 16);
        mma16816(dp[n], av, b[0], b[1]);
        mma16816(dp[n + 1], av, b[2], b[3]);
      }
    }
    float b0 = kb0, b1 = kb1;
    if (CENTROID) {  // the row block's own exact members are excluded (taylor.py:154)
      if ((sMem[buf * 2 + (kr0 >> 5)] >> (kr0 & 31)) & 1u) b0 = -INFINITY;
      if ((sMem[buf * 2 + (kr1 >> 5)] >> (kr1 & 31)) & 1u) b1 = -INFINITY;
    }
    uint32_t ap[4][4], ads[4][4];
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      float pv[4], dsv[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int q = n * 8 + tig * 2 + (e & 1);
        const float ls = lse[q];
        const float pr = ls > -INFINITY ? exp2f(fmaf(sc[n][e], p.sl2, (e >= 2 ? b1 : b0) - ls)) : 0.f;
        pv[e] = pr;
        dsv[e] = pr * (dp[n][e] - rho[q]);
      }
      const int kk = n >> 1;
      const int o = (n & 1) ? 2 : 0;
      ap[kk][o] = pack_bf16x2(pv[0], pv[1]);
      ap[kk][o + 1] = pack_bf16x2(pv[2], pv[3]);
      ads[kk][o] = pack_bf16x2(dsv[0], dsv[1]);
      ads[kk][o + 1] = pack_bf16x2(dsv[2], dsv[3]);
    }
    // dV += P^T dO, dK += dS^T Q (B operands as [k=query][n=d])
#pragma unroll
    for (int kk = 0; kk < 4; ++kk)
#pragma unroll
      for (int n = 0; n < D / 8; n += 2) {
        uint32_t b[4];
        frag_bt<D>(b, bo, kk * 16, n * 8);
        mma16816(dv[n], ap[kk], b[0], b[1]);
        mma16816(dv[n + 1], ap[kk], b[2], b[3]);
        frag_bt<D>(b, bq, kk * 16, n * 8);
        mma16816(dk[n], ads[kk], b[0], b[1]);
        mma16816(dk[n + 1], ads[kk], b[2], b[3]);
      }
    __syncthreads();  // buffer `buf` is refilled by the prefetch of block li + 2
  }
  const bool kv0 = CENTROID ? c0 + kr0 < p.t_new : kr0 < vk;
  const bool kv1 = CENTROID ? c0 + kr1 < p.t_new : kr1 < vk;
  // stores
  if (CENTROID) {
    const long long part = blockIdx.z * p.c_part;  // partial slab (reduced by bwd_centroid_reduce_kernel)
#pragma unroll
    for (int n = 0; n < D / 8; ++n) {
      const int col = n * 8 + tig * 2;
      if (kv0) {
        const long long o = part + ((long long)bh * p.t_new + c0 + kr0) * D + col;
        p.dkc[o] = p.scale * dk[n][0];
        p.dkc[o + 1] = p.scale * dk[n][1];
        p.dvc[o] = dv[n][0];
        p.dvc[o + 1] = dv[n][1];
      }
      if (kv1) {
        const long long o = part + ((long long)bh * p.t_new + c0 + kr1) * D + col;
        p.dkc[o] = p.scale * dk[n][2];
        p.dkc[o + 1] = p.scale * dk[n][3];
        p.dvc[o] = dv[n][2];
        p.dvc[o + 1] = dv[n][3];
      }
    }
  } else {
    // + block-mean adjoint of the centroid gradients (taylor.py:290-292), then
    // the K_new gather adjoint: rows go back to the block's original positions
    const float invw = 1.f / (float)vk;
    const long long cb = ((long long)bh * p.t_new + j) * D;
    const long long rowbase = (long long)bh * p.S + bw_tok0(p, uk);
#pragma unroll
    for (int n = 0; n < D / 8; ++n) {
      const int col = n * 8 + tig * 2;
      float ck0 = 0.f, ck1 = 0.f, cv0 = 0.f, cv1 = 0.f;
      if (p.n_flat) {
        ck0 = p.dkc[cb + col] * invw;
        ck1 = p.dkc[cb + col + 1] * invw;
        cv0 = p.dvc[cb + col] * invw;
        cv1 = p.dvc[cb + col + 1] * invw;
      }
      if (kv0) {
        const long long o = (rowbase + kr0) * D + col;
        p.dk[o] = p.scale * dk[n][0] + ck0;
        p.dk[o + 1] = p.scale * dk[n][1] + ck1;
        p.dv[o] = dv[n][0] + cv0;
        p.dv[o + 1] = dv[n][1] + cv1;
      }
      if (kv1) {
        const long long o = (rowbase + kr1) * D + col;
        p.dk[o] = p.scale * dk[n][2] + ck0;
        p.dk[o + 1] = p.scale * dk[n][3] + ck1;
        p.dv[o] = dv[n][2] + cv0;
        p.dv[o + 1] = dv[n][3] + cv1;
      }
    }
  }
}

}  // namespace isa

namespace isa {

// ---------------------------------------------------------------- gamma residual backward
// pipeline.py:435-452: do_c = gamma * (sum of dO over each block's rows);
// softmax variant: full_attention_backward(qc, kc, vc, scale, do_c)
// (reference.py:173-225) on the T x T coarse problem; raw variant: ds = do_c
// vc^T, dqc = ds kc, dkc = ds^T qc, dvc = (qc kc^T)^T do_c. The block-mean
// adjoint then spreads d{q,k,v}c[u] / valid(u) over block u's rows
// (_spread_mean_grad, pipeline.py:460-466). fp32.

struct GammaBwdParams {
  int H, S, D, T, t_src, l_src, l_ctx;
  float gamma, scale;
  int softmax;
  const __nv_bfloat16* dout;
  long long db, dh, ds;
  const float *qc, *kc, *vc;  // [BH][T][D] block means
  float* doc;                 // [BH][T][D]
  float *m, *l, *rho;         // [BH][T] coarse softmax stats (softmax variant)
  float *dqc, *dkc, *dvc;     // [BH][T][D]
  float *dq, *dk, *dv;        // [BH][S][D] (accumulated into)
};

__device__ __forceinline__ int gb_tok0(const GammaBwdParams& p, int u) {
  return u < p.t_src ? u * 64 : p.l_src + (u - p.t_src) * 64;
}
__device__ __forceinline__ int gb_valid(const GammaBwdParams& p, int u) {
  const int r = u < p.t_src ? p.l_src - u * 64 : p.l_ctx - (u - p.t_src) * 64;
  return r < 64 ? r : 64;
}

// do_c: grid (T, BH), D threads
__global__ void gamma_doc_kernel(const GammaBwdParams p) {
  const int u = blockIdx.x, bh = blockIdx.y, d = threadIdx.x;
  const __nv_bfloat16* src = p.dout + (bh / p.H) * p.db + (bh % p.H) * p.dh + (long long)gb_tok0(p, u) * p.ds + d;
  float acc = 0.f;
  const int vr = gb_valid(p, u);
  for (int r = 0; r < vr; ++r) acc += __bfloat162float(src[r * p.ds]);
  p.doc[((long long)bh * p.T + u) * p.D + d] = p.gamma * acc;
}

__device__ __forceinline__ float warp_dot(const float* a, const float* b, int D, int lane) {
  float s = 0.f;
  for (int d = lane; d < D; d += 32) s = fmaf(a[d], b[d], s);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}

// Row pass: one warp per query block u. Softmax stats, rho and dqc.
// grid (ceil(T/4), BH), 128 threads.
__global__ void gamma_row_kernel(const GammaBwdParams p) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int u = blockIdx.x * 4 + warp, bh = blockIdx.y;
  if (u >= p.T) return;
  const long long base = (long long)bh * p.T * p.D;
  const float* q = p.qc + base + (long long)u * p.D;
  const float* g = p.doc + base + (long long)u * p.D;
  float m = -INFINITY, l = 0.f, rho = 0.f;
  if (p.softmax) {
    for (int j = 0; j < p.T; ++j) {
      const float s = p.scale * warp_dot(q, p.kc + base + (long long)j * p.D, p.D, lane);
      const float mn = fmaxf(m, s);
      l = l * __expf(m - mn) + __expf(s - mn);
      m = mn;
    }
    for (int j = 0; j < p.T; ++j) {
      const float s = p.scale * warp_dot(q, p.kc + base + (long long)j * p.D, p.D, lane);
      const float gj = warp_dot(g, p.vc + base + (long long)j * p.D, p.D, lane);
      rho += __expf(s - m) / l * gj;
    }
  }
  float acc[4] = {0.f, 0.f, 0.f, 0.f};  // D <= 128: lane holds columns lane + 32c
  for (int j = 0; j < p.T; ++j) {
    const float* kj = p.kc + base + (long long)j * p.D;
    const float gj = warp_dot(g, p.vc + base + (long long)j * p.D, p.D, lane);
    float dsj;
    if (p.softmax) {
      const float s = p.scale * warp_dot(q, kj, p.D, lane);
      dsj = p.scale * __expf(s - m) / l * (gj - rho);
    } else {
      dsj = gj;
    }
    for (int c = 0; c < p.D / 32; ++c) acc[c] = fmaf(dsj, kj[lane + 32 * c], acc[c]);
  }
  for (int c = 0; c < p.D / 32; ++c) p.dqc[base + (long long)u * p.D + lane + 32 * c] = acc[c];
  if (lane == 0 && p.softmax) {
    p.m[(long long)bh * p.T + u] = m;
    p.l[(long long)bh * p.T + u] = l;
    p.rho[(long long)bh * p.T + u] = rho;
  }
}

// Column pass: one warp per key block j: dkc_j, dvc_j over all query blocks u.
__global__ void gamma_col_kernel(const GammaBwdParams p) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j = blockIdx.x * 4 + warp, bh = blockIdx.y;
  if (j >= p.T) return;
  const long long base = (long long)bh * p.T * p.D;
  const float* kj = p.kc + base + (long long)j * p.D;
  const float* vj = p.vc + base + (long long)j * p.D;
  float ak[4] = {0.f, 0.f, 0.f, 0.f}, av[4] = {0.f, 0.f, 0.f, 0.f};
  for (int u = 0; u < p.T; ++u) {
    const float* qu = p.qc + base + (long long)u * p.D;
    const float* gu = p.doc + base + (long long)u * p.D;
    const float s_raw = warp_dot(qu, kj, p.D, lane);
    const float gj = warp_dot(gu, vj, p.D, lane);
    float ds, pv;
    if (p.softmax) {
      const long long r = (long long)bh * p.T + u;
      const float pr = __expf(p.scale * s_raw - p.m[r]) / p.l[r];
      ds = p.scale * pr * (gj - p.rho[r]);
      pv = pr;
    } else {
      ds = gj;      // dkc = ds^T qc
      pv = s_raw;   // dvc = (qc kc^T)^T do_c
    }
    for (int c = 0; c < p.D / 32; ++c) {
      ak[c] = fmaf(ds, qu[lane + 32 * c], ak[c]);
      av[c] = fmaf(pv, gu[lane + 32 * c], av[c]);
    }
  }
  for (int c = 0; c < p.D / 32; ++c) {
    p.dkc[base + (long long)j * p.D + lane + 32 * c] = ak[c];
    p.dvc[base + (long long)j * p.D + lane + 32 * c] = av[c];
  }
}

// Spread: every valid row of block u += d{q,k,v}c[u] / valid(u). grid (T, BH), D threads.
__global__ void gamma_spread_kernel(const GammaBwdParams p) {
  const int u = blockIdx.x, bh = blockIdx.y, d = threadIdx.x;
  const int vr = gb_valid(p, u);
  const float inv = 1.f / (float)vr;
  const long long c = ((long long)bh * p.T + u) * p.D + d;
  const float a = p.dqc[c] * inv, b = p.dkc[c] * inv, e = p.dvc[c] * inv;
  const long long row0 = (long long)bh * p.S + gb_tok0(p, u);
  for (int r = 0; r < vr; ++r) {
    const long long o = (row0 + r) * p.D + d;
    p.dq[o] += a;
    p.dk[o] += b;
    p.dv[o] += e;
  }
}

// Sum of the c_splits partial centroid-gradient slabs into slab 0, in slab
// order (deterministic: no atomics).
__global__ void bwd_centroid_reduce_kernel(float* __restrict__ dkc, float* __restrict__ dvc, long long n,
                                           int splits) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    float a = dkc[i], b = dvc[i];
    for (int z = 1; z < splits; ++z) {
      a += dkc[z * n + i];
      b += dvc[z * n + i];
    }
    dkc[i] = a;
    dvc[i] = b;
  }
}

}  // namespace isa
