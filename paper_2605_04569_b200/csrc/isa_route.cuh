// ISA routing kernels (north-star stages 1-2) on sm_100a CUDA cores.
//
// All index decisions are bit-exact restatements of the reference's float64
// arithmetic: block sums in fp64 -> fp32 means (tensor.py:96-119), fp64 coarse
// scores (pipeline.py:180-182), fp64 softmax-variance (coarse.py:193-195,
// util.py:32-40) and stable (score desc, index asc) rank selection
// (coarse.py:130-136, 196-200). No float atomics: results are independent of
// thread count and scheduling.
#pragma once
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace isa {

struct SegInfo {
  int l_src, l_ctx, t_src, t_ctx;
  __device__ __forceinline__ int tok0(int u) const { return u < t_src ? u * 64 : l_src + (u - t_src) * 64; }
  __device__ __forceinline__ int valid(int u) const {
    int r = u < t_src ? l_src - u * 64 : l_ctx - (u - t_src) * 64;
    return r < 64 ? r : 64;
  }
};

// (score desc, index asc): true when (a, ia) ranks before (b, ib). NaN ranks
// after every number, so the order stays total and every selection emits
// exactly k indices even on non-finite input (which is then reported as
// InputError by the pooling kernel's flag).
__device__ __forceinline__ bool ranks_before(double a, int ia, double b, int ib) {
  const bool na = a != a, nb = b != b;
  if (na || nb) return na && nb ? ia < ib : nb;
  return a > b || (a == b && ia < ib);
}

// ----------------------------------------------------------------------------
// K1: block means of Q, K, V (fp64 sums over valid rows -> fp32), finiteness
// flag, and (fp32 inputs) the bf16 copy consumed by the TMA attention kernels.
// grid (T, BH, 3), block 256. One CTA = one 64-row block of one tensor.
// ----------------------------------------------------------------------------
template <typename Tin, int D>
__global__ void __launch_bounds__(256) pool_means_kernel(const Tin* __restrict__ q, const Tin* __restrict__ k,
                                                         const Tin* __restrict__ v, long long sb, long long sh,
                                                         long long ss, int H, SegInfo seg, int T,
                                                         float* __restrict__ means,  // [3][BH][T][D]
                                                         __nv_bfloat16* __restrict__ bf_copy,  // [3][BH][S][D] or null
                                                         int S, int* __restrict__ err) {
  constexpr int VEC = 8;                    // elements per thread-load
  constexpr int LPR = D / VEC;              // threads per row
  constexpr int RPAR = 256 / LPR;           // rows in flight
  __shared__ double part[RPAR][D + 1];
  const int u = blockIdx.x, bh = blockIdx.y, which = blockIdx.z;
  const Tin* x = which == 0 ? q : (which == 1 ? k : v);
  const int b = bh / H, h = bh % H;
  const int tok0 = seg.tok0(u), valid = seg.valid(u);
  const int col = (threadIdx.x % LPR) * VEC;
  const int r0 = threadIdx.x / LPR;
  double acc[VEC];
#pragma unroll
  for (int e = 0; e < VEC; ++e) acc[e] = 0.0;
  bool finite = true;
  const Tin* base = x + b * sb + h * sh;
  for (int r = r0; r < valid; r += RPAR) {
    const Tin* rowp = base + (long long)(tok0 + r) * ss + col;
    float f[VEC];
    if constexpr (sizeof(Tin) == 2) {
      const uint4 w = *reinterpret_cast<const uint4*>(rowp);
      const __nv_bfloat162* hw = reinterpret_cast<const __nv_bfloat162*>(&w);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 t = __bfloat1622float2(hw[e]);
        f[2 * e] = t.x;
        f[2 * e + 1] = t.y;
      }
    } else {
      const float4 a = *reinterpret_cast<const float4*>(rowp);
      const float4 c = *reinterpret_cast<const float4*>(rowp + 4);
      f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w;
      f[4] = c.x; f[5] = c.y; f[6] = c.z; f[7] = c.w;
      if (bf_copy) {
        uint4 w;
        __nv_bfloat162 t0 = __floats2bfloat162_rn(f[0], f[1]);
        __nv_bfloat162 t1 = __floats2bfloat162_rn(f[2], f[3]);
        __nv_bfloat162 t2 = __floats2bfloat162_rn(f[4], f[5]);
        __nv_bfloat162 t3 = __floats2bfloat162_rn(f[6], f[7]);
        w.x = *reinterpret_cast<uint32_t*>(&t0);
        w.y = *reinterpret_cast<uint32_t*>(&t1);
        w.z = *reinterpret_cast<uint32_t*>(&t2);
        w.w = *reinterpret_cast<uint32_t*>(&t3);
        *reinterpret_cast<uint4*>(bf_copy + (((long long)which * (gridDim.y) + bh) * S + tok0 + r) * D + col) = w;
      }
    }
#pragma unroll
    for (int e = 0; e < VEC; ++e) {
      finite &= isfinite(f[e]);
      acc[e] += static_cast<double>(f[e]);
    }
  }
#pragma unroll
  for (int e = 0; e < VEC; ++e) part[r0][col + e] = acc[e];
  if (!finite && err) atomicOr(err, 1);
  __syncthreads();
  float* out = means + (((long long)which * gridDim.y + bh) * T + u) * D;
  for (int c = threadIdx.x; c < D; c += 256) {
    double s = 0.0;
#pragma unroll 4
    for (int r = 0; r < RPAR; ++r) s += part[r][c];  // fixed order: deterministic
    out[c] = static_cast<float>(s / static_cast<double>(valid));
  }
}

// ----------------------------------------------------------------------------
// K2a: S_src[bh][u][j] = scale * <qc_u, kc_j>, u < T, j < t_src, float64.
// 64x64 tiles, 256 threads, 4x4 outputs per thread. grid (ceil(t_src/64),
// ceil(T/64), BH).
// ----------------------------------------------------------------------------
__global__ void __launch_bounds__(256) coarse_src_kernel(const float* __restrict__ qc, const float* __restrict__ kc,
                                                         int T, int t_src, int D, double scale,
                                                         double* __restrict__ s_src) {
  __shared__ double As[16][64 + 1];
  __shared__ double Bs[16][64 + 1];
  const int bh = blockIdx.z;
  const int i0 = blockIdx.y * 64, j0 = blockIdx.x * 64;
  const float* qb = qc + (long long)bh * T * D;
  const float* kb = kc + (long long)bh * T * D;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  double acc[4][4] = {};
  for (int d0 = 0; d0 < D; d0 += 16) {
    for (int e = threadIdx.x; e < 64 * 16; e += 256) {
      const int r = e / 16, dd = e % 16;
      const int gi = i0 + r, gj = j0 + r;
      As[dd][r] = gi < T ? static_cast<double>(qb[(long long)gi * D + d0 + dd]) : 0.0;
      Bs[dd][r] = gj < t_src ? static_cast<double>(kb[(long long)gj * D + d0 + dd]) : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int dd = 0; dd < 16; ++dd) {
      double a[4], bv[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        a[t] = As[dd][ty + 16 * t];
        bv[t] = Bs[dd][tx + 16 * t];
      }
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] = fma(a[r], bv[c], acc[r][c]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int gi = i0 + ty + 16 * r;
    if (gi >= T) continue;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int gj = j0 + tx + 16 * c;
      if (gj < t_src) s_src[((long long)bh * T + gi) * t_src + gj] = scale * acc[r][c];
    }
  }
}

// ----------------------------------------------------------------------------
// K2b: context saliency = mean over source query blocks of the scaled coarse
// score (coarse.py:155), computed through linearity:
//   ctx[c] = scale * <sum_{i<t_src} qc_i, kc_{t_src+c}> / t_src   (fp64).
// grid BH, block 256.
// ----------------------------------------------------------------------------
__global__ void __launch_bounds__(256) ctx_score_kernel(const float* __restrict__ qc, const float* __restrict__ kc,
                                                        int T, int t_src, int t_ctx, int D, double scale,
                                                        double* __restrict__ ctx) {
  extern __shared__ double qsum[];  // [D]
  const int bh = blockIdx.x;
  const float* qb = qc + (long long)bh * T * D;
  const float* kb = kc + (long long)bh * T * D;
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    double s = 0.0;
    for (int i = 0; i < t_src; ++i) s += static_cast<double>(qb[(long long)i * D + d]);
    qsum[d] = s;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int c = warp; c < t_ctx; c += blockDim.x / 32) {
    const float* kr = kb + (long long)(t_src + c) * D;
    double s = 0.0;
    for (int d = lane; d < D; d += 32) s = fma(qsum[d], static_cast<double>(kr[d]), s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) ctx[(long long)bh * t_ctx + c] = scale * s / static_cast<double>(t_src);
  }
}

// ----------------------------------------------------------------------------
// Block-wide helpers: stable rank selection and ascending compaction.
// ----------------------------------------------------------------------------
// Exclusive prefix sum of flags[0..n) into pos[0..n); returns the total.
__device__ int block_exclusive_scan(const uint8_t* flags, int* pos, int n, int* scratch /* >= 33 ints */) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  int base = 0;
  for (int c0 = 0; c0 < n; c0 += blockDim.x) {
    const int idx = c0 + threadIdx.x;
    const int f = idx < n ? flags[idx] : 0;
    const unsigned bal = __ballot_sync(0xffffffffu, f);
    const int within = __popc(bal & ((1u << lane) - 1u));
    if (lane == 0) scratch[warp] = __popc(bal);
    __syncthreads();
    if (warp == 0) {
      int v = lane < nw ? scratch[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
      }
      if (lane < nw) scratch[lane] = v;  // inclusive
    }
    __syncthreads();
    const int woff = warp ? scratch[warp - 1] : 0;
    if (idx < n) pos[idx] = base + woff + within;
    const int tot = scratch[nw - 1];
    __syncthreads();
    base += tot;
  }
  return base;
}

// ----------------------------------------------------------------------------
// K3: per row, keep the k best of n fp64 scores (desc, ties -> lower index),
// emitted ascending (coarse.py:130-136). One CTA per row; rank by counting.
// Used for context selection (coarse.py:139-157) and as the explicit-score
// test primitive. Optionally also writes the K_new block table.
// dyn smem: n doubles + n bytes + n ints.
// ----------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) topk_rank_kernel(const double* __restrict__ scores, int n, int k,
                                                         int* __restrict__ out_idx,    // [rows][k] (int32) or null
                                                         int64_t* __restrict__ out_idx64) {  // [rows][k] or null
  extern __shared__ __align__(16) uint8_t sm[];
  double* sv = reinterpret_cast<double*>(sm);
  int* pos = reinterpret_cast<int*>(sm + sizeof(double) * n);
  uint8_t* flag = reinterpret_cast<uint8_t*>(sm + sizeof(double) * n + sizeof(int) * n);
  __shared__ int scratch[40];
  const int row = blockIdx.x;
  const double* sr = scores + (long long)row * n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) sv[i] = sr[i];
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double a = sv[i];
    int rank = 0;
    for (int j = 0; j < n; ++j) rank += ranks_before(sv[j], j, a, i) ? 1 : 0;
    flag[i] = rank < k;
  }
  __syncthreads();
  block_exclusive_scan(flag, pos, n, scratch);
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    if (flag[i]) {
      if (out_idx) out_idx[(long long)row * k + pos[i]] = i;
      if (out_idx64) out_idx64[(long long)row * k + pos[i]] = i;
    }
  }
}

// ----------------------------------------------------------------------------
// K4a: sharpness of every query block: population variance over the source
// columns of the row-softmax (softmax_first) or of the raw scaled scores
// (coarse.py:193-195; softmax_rows util.py:32-40; numpy var = mean((x-mean)^2)).
// One warp per row. grid ceil(rows/8), block 256.
// ----------------------------------------------------------------------------
__global__ void __launch_bounds__(256) sharpness_kernel(const double* __restrict__ s, int rows, int n,
                                                        int softmax_first, double* __restrict__ out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = blockIdx.x * 8 + warp;
  if (row >= rows) return;
  const double* x = s + (long long)row * n;
  double mx = -INFINITY;
  for (int j = lane; j < n; j += 32) mx = fmax(mx, x[j]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  double z = 1.0;
  if (softmax_first) {
    double se = 0.0;
    for (int j = lane; j < n; j += 32) se += exp(x[j] - mx);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
    z = se;
  }
  auto val = [&](double xv) { return softmax_first ? exp(xv - mx) / z : xv; };
  double sum = 0.0;
  for (int j = lane; j < n; j += 32) sum += val(x[j]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  const double mean = sum / n;
  double sq = 0.0;
  for (int j = lane; j < n; j += 32) {
    const double d = val(x[j]) - mean;
    sq += d * d;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
  if (lane == 0) out[row] = sq / n;
}

// ----------------------------------------------------------------------------
// K4b: split (coarse.py:196-200): order = argsort(-M, stable); the first
// T - n_flat stay sharp. Both lists ascending. One CTA per row.
// dyn smem: n doubles + n ints + n bytes.
// ----------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) split_kernel(const double* __restrict__ m, int n, int n_flat,
                                                     int* __restrict__ sharp, int* __restrict__ flat,
                                                     int64_t* __restrict__ sharp64, int64_t* __restrict__ flat64) {
  extern __shared__ __align__(16) uint8_t sm[];
  double* sv = reinterpret_cast<double*>(sm);
  int* pos = reinterpret_cast<int*>(sm + sizeof(double) * n);
  uint8_t* flag = reinterpret_cast<uint8_t*>(sm + sizeof(double) * n + sizeof(int) * n);
  __shared__ int scratch[40];
  const int row = blockIdx.x;
  const int n_sharp = n - n_flat;
  for (int i = threadIdx.x; i < n; i += blockDim.x) sv[i] = m[(long long)row * n + i];
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double a = sv[i];
    int rank = 0;
    for (int j = 0; j < n; ++j) rank += ranks_before(sv[j], j, a, i) ? 1 : 0;
    flag[i] = rank < n_sharp;
  }
  __syncthreads();
  block_exclusive_scan(flag, pos, n, scratch);
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    if (flag[i]) {
      const int p = pos[i];
      if (sharp) sharp[(long long)row * n_sharp + p] = i;
      if (sharp64) sharp64[(long long)row * n_sharp + p] = i;
    } else {
      const int p = i - pos[i];
      if (flat) flat[(long long)row * n_flat + p] = i;
      if (flat64) flat64[(long long)row * n_flat + p] = i;
    }
  }
}

// ----------------------------------------------------------------------------
// K5: block mask for the flat query blocks (pipeline.py:219-225,
// coarse.py:160-170): fp64 scores of the flat block's mean query against the
// means of every K_new block (source columns read from S_src, selected
// context columns recomputed), top-k by k rounds of warp arg-max (desc, ties ->
// lower index), emitted ascending plus a membership bitmask (W words).
// One warp per flat row; 4 warps per CTA. When `explicit_scores` is given the
// scores are read from it instead ([rows][n]; test primitive).
// dyn smem: 4 * (n doubles + W words).
// ----------------------------------------------------------------------------
__global__ void __launch_bounds__(128) block_mask_kernel(
    const double* __restrict__ explicit_scores, int rows, const double* __restrict__ s_src,
    const float* __restrict__ qc, const float* __restrict__ kc, const int* __restrict__ flat,
    const int* __restrict__ kv_blk, int T, int t_src, int n_flat, int D, double scale, int n, int k, int W,
    int* __restrict__ mask_idx, int64_t* __restrict__ mask64, uint32_t* __restrict__ member_bits) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = blockIdx.x * 4 + warp;
  double* sv = reinterpret_cast<double*>(sm) + (long long)warp * n;
  uint32_t* bits = reinterpret_cast<uint32_t*>(sm + sizeof(double) * 4 * n) + warp * W;
  if (row >= rows) return;
  if (explicit_scores) {
    for (int j = lane; j < n; j += 32) sv[j] = explicit_scores[(long long)row * n + j];
  } else {
    const int bh = row / n_flat, f = row % n_flat;
    const int u = flat[(long long)bh * n_flat + f];
    const double* srow = s_src + ((long long)bh * T + u) * t_src;
    const float* qrow = qc + ((long long)bh * T + u) * D;
    const int* tab = kv_blk + (long long)bh * n;
    for (int j = lane; j < t_src; j += 32) sv[j] = srow[j];
    for (int j = t_src; j < n; ++j) {  // selected context columns: warp-cooperative fp64 dot
      const float* krow = kc + ((long long)bh * T + tab[j]) * D;
      double s = 0.0;
      for (int d = lane; d < D; d += 32) s = fma(static_cast<double>(qrow[d]), static_cast<double>(krow[d]), s);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) sv[j] = scale * s;
    }
  }
  for (int w = lane; w < W; w += 32) bits[w] = 0u;
  __syncwarp();
  for (int r = 0; r < k; ++r) {
    double best = -INFINITY;
    int bi = 0x7fffffff;
    for (int j = lane; j < n; j += 32) {
      const bool taken = (bits[j >> 5] >> (j & 31)) & 1u;
      if (!taken && (bi == 0x7fffffff || ranks_before(sv[j], j, best, bi))) {
        best = sv[j];
        bi = j;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (oi != 0x7fffffff && (bi == 0x7fffffff || ranks_before(ob, oi, best, bi))) {
        best = ob;
        bi = oi;
      }
    }
    if (lane == 0) bits[bi >> 5] |= 1u << (bi & 31);
    __syncwarp();
  }
  // ascending emission: lane-parallel over words with a warp prefix of popcounts
  int base = 0;
  for (int w0 = 0; w0 < W; w0 += 32) {
    const int w = w0 + lane;
    const uint32_t word = w < W ? bits[w] : 0u;
    int cnt = __popc(word), incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    int p = base + incl - cnt;
    uint32_t wb = word;
    while (wb) {
      const int bpos = __ffs(wb) - 1;
      wb &= wb - 1;
      const int j = w * 32 + bpos;
      if (mask_idx) mask_idx[(long long)row * k + p] = j;
      if (mask64) mask64[(long long)row * k + p] = j;
      ++p;
    }
    if (w < W && member_bits) member_bits[(long long)row * W + w] = word;
    base += __shfl_sync(0xffffffffu, incl, 31);
  }
}

// ----------------------------------------------------------------------------
// K_new centroids in bf16 for the Taylor kernel's centroid tiles (rows j <
// t_new copy kc/vc of original block kv_blk[j]; rows >= t_new are zero), and
// the K_new index of the selected short last context block (its centroid
// weight is its valid-row count, taylor.py:156). grid (tn_pad, BH), block D.
// ----------------------------------------------------------------------------
__global__ void centroid_kernel(const float* __restrict__ kc, const float* __restrict__ vc,
                                const int* __restrict__ kv_blk, int T, int t_new, int tn_pad, int D, SegInfo seg,
                                __nv_bfloat16* __restrict__ kc_bf, __nv_bfloat16* __restrict__ vc_bf,
                                int* __restrict__ ctx_short_j) {
  const int j = blockIdx.x, bh = blockIdx.y;
  const long long o = ((long long)bh * tn_pad + j) * D;
  if (j < t_new) {
    const int u = kv_blk[(long long)bh * t_new + j];
    const long long src = ((long long)bh * T + u) * D;
    for (int d = threadIdx.x; d < D; d += blockDim.x) {
      kc_bf[o + d] = __float2bfloat16_rn(kc[src + d]);
      vc_bf[o + d] = __float2bfloat16_rn(vc[src + d]);
    }
    if (threadIdx.x == 0 && j >= seg.t_src && u == seg.t_src + seg.t_ctx - 1) ctx_short_j[bh] = j;
  } else {
    for (int d = threadIdx.x; d < D; d += blockDim.x) {
      kc_bf[o + d] = __float2bfloat16_rn(0.f);
      vc_bf[o + d] = __float2bfloat16_rn(0.f);
    }
  }
}

// ----------------------------------------------------------------------------
// Taylor work plan: for each CTA item (4 flat query blocks) merge the 4 exact
// lists (bitmask OR) into an ascending union stream paired into 128-key tiles;
// each half carries a 4-bit visibility mask (which of the 4 query blocks has
// that K_new block on its exact list). One warp per item.
// ----------------------------------------------------------------------------
__global__ void taylor_plan_kernel(const uint32_t* __restrict__ member_bits, int n_flat, int W, int n_items,
                                   int max_tiles, int4* __restrict__ tiles, int* __restrict__ n_tiles) {
  const int item = blockIdx.x, bh = blockIdx.y, lane = threadIdx.x;
  const uint32_t* mb[4];
  int nq = 0;
  for (int q = 0; q < 4; ++q) {
    const int f = item * 4 + q;
    mb[q] = f < n_flat ? member_bits + ((long long)bh * n_flat + f) * W : nullptr;
    nq += f < n_flat;
  }
  int4* out = tiles + ((long long)bh * n_items + item) * max_tiles;
  int base = 0;
  for (int w0 = 0; w0 < W; w0 += 32) {
    const int w = w0 + lane;
    uint32_t wq[4] = {0u, 0u, 0u, 0u};
    uint32_t uni = 0u;
    if (w < W) {
      for (int q = 0; q < 4; ++q)
        if (mb[q]) {
          wq[q] = mb[q][w];
          uni |= wq[q];
        }
    }
    const int cnt = __popc(uni);
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    int p = base + incl - cnt;
    uint32_t wb = uni;
    while (wb) {
      const int bpos = __ffs(wb) - 1;
      wb &= wb - 1;
      const int j = w * 32 + bpos;
      int vis = 0;
      for (int q = 0; q < 4; ++q) vis |= ((wq[q] >> bpos) & 1u) << q;
      int* e = reinterpret_cast<int*>(out + (p >> 1));
      if (p & 1) {
        e[1] = j;
        e[3] = vis;
      } else {
        e[0] = j;
        e[2] = vis;
      }
      ++p;
    }
    base += __shfl_sync(0xffffffffu, incl, 31);
  }
  __syncwarp();
  if (lane == 0) {
    n_tiles[bh * n_items + item] = (base + 1) >> 1;
    if (base & 1) {  // odd union: the last tile's second half is absent (fully masked)
      int* e = reinterpret_cast<int*>(out + (base >> 1));
      e[1] = -1;
      e[3] = 0;
    }
  }
  (void)nq;
}

// int32 -> int64 export of routing lists (caller-facing int64 API, pipeline types).
__global__ void widen_kernel(const int* __restrict__ src, int64_t* __restrict__ dst, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    dst[i] = src[i];
}
// int64 -> int32 import of pinned routing.
__global__ void narrow_kernel(const int64_t* __restrict__ src, int* __restrict__ dst, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    dst[i] = static_cast<int>(src[i]);
}

// Pinned selection -> K_new block table.
__global__ void kvblk_from_sel_kernel(const int* __restrict__ sel, int t_src, int k_ctx, int* __restrict__ kv_blk,
                                      int* __restrict__ ctx_short_j) {
  const int bh = blockIdx.x;
  if (threadIdx.x == 0) ctx_short_j[bh] = -1;
  const int t_new = t_src + k_ctx;
  for (int j = threadIdx.x; j < t_new; j += blockDim.x)
    kv_blk[(long long)bh * t_new + j] = j < t_src ? j : t_src + sel[(long long)bh * k_ctx + j - t_src];
}

// Pinned mask -> membership bitmask.
__global__ void bits_from_mask_kernel(const int* __restrict__ mask, int k, int W, uint32_t* __restrict__ bits) {
  const long long row = blockIdx.x;
  for (int w = threadIdx.x; w < W; w += blockDim.x) bits[row * W + w] = 0u;
  __syncthreads();
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    const int j = mask[row * k + i];
    atomicOr(&bits[row * W + (j >> 5)], 1u << (j & 31));
  }
}

}  // namespace isa
