// ISA backward with frozen routing (isa_backward, pipeline.py:373-466):
// gradients of the sharp branch (full_attention_backward, reference.py:173-225)
// and of the Taylor branch (taylor_sparse_backward, taylor.py:225-296), with
// the K_new gather adjoint (pipeline.py:423-433) fused into the key-major
// kernel's stores. gamma = 0.
//
// Softmax statistics come from the forward kernels (AttnParams::lse, log2
// domain: P = exp2(scale*log2e * q.k + log2(w) - lse)); rho = rowsum(dO * O).
// This file holds the shared parameters and the small CUDA-core kernels (rho,
// gamma residual, centroid partial reduce); every contraction runs on the
// tcgen05 kernels in isa_bwd_tc.cuh (dK/dV of the exact pairs and of the
// Taylor centroids, dQ).
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

// ---------------------------------------------------------------- rho
// rho[bh][row] = sum_d dO * O (taylor.py:274; reference.py:218 in closed form).
__global__ void bwd_rho_kernel(const __nv_bfloat16* __restrict__ dout, long long db, long long dh, long long ds,
                               const __nv_bfloat16* __restrict__ o, int H, int S, int D, float* __restrict__ rho,
                               long long n_rows) {
  // D / 8 lanes per row, one 16-byte load of dO and of O per lane (D = 128: two rows per warp)
  const int lpr = D >> 3;
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long w = t / lpr;
  const int sub = static_cast<int>(t % lpr);
  float acc = 0.f;
  if (w < n_rows) {
    const int bh = static_cast<int>(w / S), tok = static_cast<int>(w % S);
    const uint4 x = *reinterpret_cast<const uint4*>(dout + (bh / H) * db + (bh % H) * dh + tok * ds + sub * 8);
    const uint4 y = *reinterpret_cast<const uint4*>(o + w * D + sub * 8);
    const uint32_t xs[4] = {x.x, x.y, x.z, x.w}, ys[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 a2 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&xs[e]));
      const float2 b2 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&ys[e]));
      acc = fmaf(a2.x, b2.x, fmaf(a2.y, b2.y, acc));
    }
  }
  for (int off = lpr >> 1; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (w < n_rows && sub == 0) rho[w] = acc;
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
