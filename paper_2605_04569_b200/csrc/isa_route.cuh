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

#include "../../include/isa_b200.h"
#include "isa_ptx.cuh"

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

// Decoupled RoPE rotation of one pair (pipeline.py:469-490): fp32 with the
// operation order pinned (no contraction differences between the standalone
// kernel and the one fused into the pooling pass: same bits either way).
__device__ __forceinline__ void rope_pair(float e, float o, float c, float s, float& r0, float& r1) {
  r0 = __fsub_rn(__fmul_rn(e, c), __fmul_rn(o, s));
  r1 = __fadd_rn(__fmul_rn(e, s), __fmul_rn(o, c));
}

// cos / sin of pos * base^(-2i/D) for every token and pair, computed in fp64
// and rounded to fp32 (the values decoupled_rope_kernel forms per token);
// positions restart at 0 for the context segment. tab[tok][i] = (cos, sin).
__global__ void rope_table_kernel(float2* __restrict__ tab, int S, int D, int l_src, double log2_base) {
  const int half = D / 2;
  const long long gid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (gid >= (long long)S * half) return;
  const int tok = static_cast<int>(gid / half), i = static_cast<int>(gid % half);
  const double pos = tok < l_src ? tok : tok - l_src;
  const double theta = pos * exp2(-log2_base * (2.0 * i) / D);  // pos * base^(-2i/D)
  double sd, cd;
  sincos(theta, &sd, &cd);
  tab[gid] = make_float2(static_cast<float>(cd), static_cast<float>(sd));
}

// ----------------------------------------------------------------------------
// K1: block means of Q, K, V (fp64 sums over valid rows -> fp32; bit-identical
// to tensor.py:115-119 whenever the 64-term fp64 sum is exact, always for bf16
// inputs), finiteness flag, and (fp32 inputs) the bf16 copy consumed by the TMA
// attention kernels. One warp per 64-row block: lanes own 8 consecutive
// columns (16-byte loads), D/8 lanes per row, 32/(D/8) rows per load wave,
// 8 waves unrolled for memory-level parallelism. grid (ceil(T/4), BH, 3).
// ----------------------------------------------------------------------------
template <typename Tin, int D>
__global__ void __launch_bounds__(128) pool_means_kernel(const Tin* __restrict__ q, const Tin* __restrict__ k,
                                                         const Tin* __restrict__ v, long long sb, long long sh,
                                                         long long ss, int H, SegInfo seg, int T,
                                                         float* __restrict__ means,  // [3][BH][T][D]
                                                         __nv_bfloat16* __restrict__ bf_copy,  // [3][BH][S][D] or null
                                                         int S, int* __restrict__ err,
                                                         const float2* __restrict__ rope_tab = nullptr) {
  constexpr int VEC = 8;
  constexpr int LPR = D / VEC;     // lanes per row
  constexpr int RPW = 32 / LPR;    // rows per warp wave
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int u = blockIdx.x * 4 + warp, bh = blockIdx.y, which = blockIdx.z;
  if (u >= T) return;
  const Tin* x = which == 0 ? q : (which == 1 ? k : v);
  const int b = bh / H, h = bh % H;
  const int tok0 = seg.tok0(u), valid = seg.valid(u);
  const int col = (lane % LPR) * VEC;
  const int r0 = lane / LPR;
  double acc[VEC];
#pragma unroll
  for (int e = 0; e < VEC; ++e) acc[e] = 0.0;
  bool finite = true;
  const Tin* base = x + b * sb + h * sh + (long long)tok0 * ss + col;
  constexpr int WAVES = 64 / RPW;
  // full blocks (every block in strict mode): no per-wave exit, so all loads
  // of a 16-wave group are in flight together
  const int nw = valid == 64 ? WAVES : (valid - r0 + RPW - 1) / RPW;
#pragma unroll 16
  for (int w = 0; w < nw; ++w) {
    const int r = r0 + w * RPW;
    const Tin* rowp = base + (long long)r * ss;
    float f[VEC];
    if constexpr (sizeof(Tin) == 2) {
      const uint4 wv = __ldg(reinterpret_cast<const uint4*>(rowp));
      const __nv_bfloat162* hw = reinterpret_cast<const __nv_bfloat162*>(&wv);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 t = __bfloat1622float2(hw[e]);
        f[2 * e] = t.x;
        f[2 * e + 1] = t.y;
      }
      if (rope_tab && which < 2) {
        // fused decoupled RoPE (bf16 inputs): rotate Q / K rows, round to bf16
        // like the standalone kernel, write the copy the attention kernels
        // load, and pool the rounded rotated values (== RoPE then isa_forward)
        const float4* tr = reinterpret_cast<const float4*>(rope_tab + (long long)(tok0 + r) * (D / 2) + col / 2);
        uint32_t pk[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float4 cs2 = __ldg(tr + e / 2);
          const float cc = (e & 1) ? cs2.z : cs2.x, sn = (e & 1) ? cs2.w : cs2.y;
          float r0, r1;
          rope_pair(f[2 * e], f[2 * e + 1], cc, sn, r0, r1);
          pk[e] = pack_bf16x2(r0, r1);
          f[2 * e] = __uint_as_float(pk[e] << 16);
          f[2 * e + 1] = __uint_as_float(pk[e] & 0xffff0000u);
        }
        *reinterpret_cast<uint4*>(bf_copy + (((long long)which * gridDim.y + bh) * S + tok0 + r) * D + col) =
            make_uint4(pk[0], pk[1], pk[2], pk[3]);
      }
    } else {
      const float4 a = __ldg(reinterpret_cast<const float4*>(rowp));
      const float4 c = __ldg(reinterpret_cast<const float4*>(rowp + 4));
      f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w;
      f[4] = c.x; f[5] = c.y; f[6] = c.z; f[7] = c.w;
      if (bf_copy) {
        uint4 wv;
        __nv_bfloat162 t0 = __floats2bfloat162_rn(f[0], f[1]);
        __nv_bfloat162 t1 = __floats2bfloat162_rn(f[2], f[3]);
        __nv_bfloat162 t2 = __floats2bfloat162_rn(f[4], f[5]);
        __nv_bfloat162 t3 = __floats2bfloat162_rn(f[6], f[7]);
        wv.x = *reinterpret_cast<uint32_t*>(&t0);
        wv.y = *reinterpret_cast<uint32_t*>(&t1);
        wv.z = *reinterpret_cast<uint32_t*>(&t2);
        wv.w = *reinterpret_cast<uint32_t*>(&t3);
        *reinterpret_cast<uint4*>(bf_copy + (((long long)which * gridDim.y + bh) * S + tok0 + r) * D + col) = wv;
      }
    }
#pragma unroll
    for (int e = 0; e < VEC; ++e) {
      finite &= isfinite(f[e]);
      acc[e] += static_cast<double>(f[e]);
    }
  }
  // combine the RPW row-groups of the warp (lanes with equal column): fixed tree order
#pragma unroll
  for (int o = LPR; o < 32; o <<= 1)
#pragma unroll
    for (int e = 0; e < VEC; ++e) acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], o);
  if (__any_sync(0xffffffffu, !finite) && lane == 0 && err) atomicOr(err, 1);
  if (lane < LPR) {
    float* out = means + (((long long)which * gridDim.y + bh) * T + u) * D + col;
    float4 o0, o1;
    const double inv = static_cast<double>(valid);
    o0.x = static_cast<float>(acc[0] / inv); o0.y = static_cast<float>(acc[1] / inv);
    o0.z = static_cast<float>(acc[2] / inv); o0.w = static_cast<float>(acc[3] / inv);
    o1.x = static_cast<float>(acc[4] / inv); o1.y = static_cast<float>(acc[5] / inv);
    o1.z = static_cast<float>(acc[6] / inv); o1.w = static_cast<float>(acc[7] / inv);
    reinterpret_cast<float4*>(out)[0] = o0;
    reinterpret_cast<float4*>(out)[1] = o1;
  }
}

// ----------------------------------------------------------------------------
// K2: fp64 coarse scores, bit-identical to the reference's
//   s = scale * np.einsum("bhid,bhjd->bhij", qc.astype(f64), kc.astype(f64))
// (pipeline.py:180-182, coarse.py:126). numpy's einsum reduces d with its
// baseline-SIMD (SSE2, 2 x f64 lanes) sum_of_products_contig_contig_outstride0_two:
// per group of 8 d it chains acc = a0*b0 + (a1*b1 + (a2*b2 + (a3*b3 + acc)))
// over the 2-lane vectors a_m = x[8g + 2m .. 8g + 2m + 1], then adds the two
// lanes. So lane 0 accumulates d = 8g+6, 8g+4, 8g+2, 8g in that order, lane 1
// d = 8g+7, 8g+5, 8g+3, 8g+1, and the dot is 0 + (lane0 + lane1). qc/kc are
// fp32, so every product is exact in fp64 and numpy's separate mul + add equals
// one fp64 FMA: two-lane FMA chains reproduce numpy's bits exactly
// (tests/test_coarse_api.py pins s_coarse against the reference's np.einsum
// output bit for bit, D = 64 and 128).
//
// s_out[bh][i][j] = scale * <qc[bh][i], kc[bh][col(j)]> for i < rows, j < n,
// col(j) = kv_blk ? kv_blk[bh * n + j] : col0 + j, on the fp64 tensor cores
// (DMMA, mma.sync.m8n8k4 .f64).
// Measured on B200 (tools/ubench/dmma_order.cu): an m8n8k4 DMMA accumulates
// its k = 4 products as the sequential FMA chain k = 0, 1, 2, 3 into C, bit
// for bit (0 mismatches in 262,144 outputs with fp32-valued operands). So one
// DMMA per (numpy group, lane) with k ordered (6, 4, 2, 0) resp. (7, 5, 3, 1)
// continues numpy's lane chains exactly, with C = the running lane
// accumulator. Fragments come from shared memory once per 8 DMMAs of a warp
// (0.75 B per FMA; an FMA-pipe kernel with 8 x 8 register tiles needs 2 B
// and ran 330 vs 247 us at cfg3).
// CTA: 64 x 64 outputs, 8 warps (2 x 4), warp tile 32 rows x 16 columns =
// 4 x 2 m8n8 tiles x 2 lanes. d staged 16 at a time (two numpy groups), k-major
// in shared memory with a 66-double row stride (conflict-free fragment
// loads: 2 wavefronts, the minimum for 256 bytes), two stages.
// grid (ceil(n/64), ceil(rows/64), BH), 256 threads.
// k-row stride in doubles: 66 = 132 words = 4 banks mod 32, so the k rows
// (6, 4, 2, 0) resp. (7, 5, 3, 1) a half-warp's fragment load touches start 8
// banks apart and each half-warp's 16 doubles cover all 32 banks once
constexpr int kDmS = 66;
__device__ __forceinline__ void dmma_m8n8k4(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}
constexpr int kDmG = 2;  // numpy groups (of 8 d) staged per barrier
__global__ void __launch_bounds__(256, 2) coarse_dmma_kernel(const float* __restrict__ qc, long long q_hstride,
                                                             const float* __restrict__ kc, long long k_hstride,
                                                             const int* __restrict__ kv_blk, int col0, int rows,
                                                             int n, int D, double scale, double* __restrict__ s_out) {
  __shared__ __align__(16) double As[2][8 * kDmG][kDmS];  // [stage][d within the staged groups][row]
  __shared__ __align__(16) double Bs[2][8 * kDmG][kDmS];  // [stage][d within the staged groups][col]
  __shared__ int colrow[64];
  const int bh = blockIdx.z;
  const int i0 = blockIdx.y * 64, j0 = blockIdx.x * 64;
  const float* qb = qc + (long long)bh * q_hstride;
  const float* kb = kc + (long long)bh * k_hstride;
  if (threadIdx.x < 64) {
    const int j = j0 + threadIdx.x;
    colrow[threadIdx.x] = j < n ? (kv_blk ? kv_blk[(long long)bh * n + j] : col0 + j) : -1;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wr = (warp >> 2) * 32, wc = (warp & 3) * 16;  // warp tile origin (rows, cols)
  const int fr = lane >> 2, fk = lane & 3;                 // fragment row/col and k slot
  double acc[2][4][2][2];  // [numpy lane][m tile][n tile][2 values]
#pragma unroll
  for (int l = 0; l < 2; ++l)
#pragma unroll
    for (int m = 0; m < 4; ++m)
#pragma unroll
      for (int t = 0; t < 2; ++t) acc[l][m][t][0] = acc[l][m][t][1] = 0.0;
  // loaders: threads 0-127 stage A (row tid/2), 128-255 stage B (col (tid-128)/2); 4 d of each group
  const int lt = threadIdx.x & 127, lr = lt >> 1, ld = (lt & 1) * 4;
  const bool loads_a = threadIdx.x < 128;
  const float* src;
  if (loads_a) {
    const int gi = i0 + lr;
    src = gi < rows ? qb + (long long)gi * D + ld : nullptr;
  } else {
    const int gj = colrow[lr];
    src = gj >= 0 ? kb + (long long)gj * D + ld : nullptr;
  }
  const float4 zero4 = make_float4(0.f, 0.f, 0.f, 0.f);
  float4 x4[kDmG];
  auto fetch = [&](int st) {  // st-th stage: groups kDmG * st ...
#pragma unroll
    for (int h = 0; h < kDmG; ++h) x4[h] = src ? __ldg(reinterpret_cast<const float4*>(src + 8 * (kDmG * st + h))) : zero4;
  };
  auto stage_in = [&](int buf) {
    double(*dst)[kDmS] = loads_a ? As[buf] : Bs[buf];
#pragma unroll
    for (int h = 0; h < kDmG; ++h) {
      dst[8 * h + ld + 0][lr] = x4[h].x; dst[8 * h + ld + 1][lr] = x4[h].y;
      dst[8 * h + ld + 2][lr] = x4[h].z; dst[8 * h + ld + 3][lr] = x4[h].w;
    }
  };
  fetch(0);
  stage_in(0);
  __syncthreads();
  const int NS = D / (8 * kDmG);
  for (int st = 0; st < NS; ++st) {
    const int buf = st & 1;
    if (st + 1 < NS) fetch(st + 1);
#pragma unroll
    for (int h = 0; h < kDmG; ++h)
#pragma unroll
      for (int l = 0; l < 2; ++l) {
        const int kd = 8 * h + 6 - 2 * fk + l;  // k slot fk: d = 6, 4, 2, 0 (lane 0) / 7, 5, 3, 1 (lane 1)
        double af[4], bf[2];
#pragma unroll
        for (int m = 0; m < 4; ++m) af[m] = As[buf][kd][wr + 8 * m + fr];
#pragma unroll
        for (int t = 0; t < 2; ++t) bf[t] = Bs[buf][kd][wc + 8 * t + fr];
#pragma unroll
        for (int m = 0; m < 4; ++m)
#pragma unroll
          for (int t = 0; t < 2; ++t) dmma_m8n8k4(acc[l][m][t], af[m], bf[t]);
      }
    if (st + 1 < NS) stage_in(buf ^ 1);
    __syncthreads();
  }
  // C fragment: row 8m + lane/4, cols 8t + 2 (lane % 4) + {0, 1}; dot = 0 + (lane0 + lane1)
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    const int i = i0 + wr + 8 * m + fr;
    if (i >= rows) continue;
#pragma unroll
    for (int t = 0; t < 2; ++t)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int j = j0 + wc + 8 * t + 2 * fk + e;
        if (j < n)
          s_out[((long long)bh * rows + i) * n + j] =
              scale * __dadd_rn(0.0, __dadd_rn(acc[0][m][t][e], acc[1][m][t][e]));
      }
  }
}

// ----------------------------------------------------------------------------
// K2b: context saliency = s_coarse[:, :, :t_src, t_src:].mean(axis=2)
// (coarse.py:155) in numpy's order: the reduction over the (outer) query-block
// axis adds rows sequentially, ((s_0 + s_1) + s_2) + ..., then divides by
// t_src. `s_ctx` holds the t_src x t_ctx scores from coarse_dmma_kernel (same
// bits as the reference's s_coarse), so the means are bit-identical too.
// Element (bh, i, c) at s + bh * head_stride + i * row_stride + c. Thread per
// context column. grid (ceil(t_ctx/128), BH).
// ----------------------------------------------------------------------------
__global__ void __launch_bounds__(128) ctx_mean_kernel(const double* __restrict__ s, long long head_stride,
                                                       long long row_stride, int t_src, int t_ctx,
                                                       double* __restrict__ ctx) {
  const int c = blockIdx.x * 128 + threadIdx.x, bh = blockIdx.y;
  if (c >= t_ctx) return;
  const double* col = s + (long long)bh * head_stride + c;
  // the sum is one dependent chain per column: keep 2 x 16 rows of loads in
  // flight (the next batch is fetched while the current one is added)
  constexpr int kU = 16;
  double acc = col[0];
  double v[kU], w[kU];
  int i = 1;
  const int full = 1 + ((t_src - 1) / kU) * kU;  // rows [1, full) come in batches of kU
  if (i < full) {
#pragma unroll
    for (int u = 0; u < kU; ++u) v[u] = col[(long long)(i + u) * row_stride];
  }
  for (; i < full; i += kU) {
    if (i + kU < full) {
#pragma unroll
      for (int u = 0; u < kU; ++u) w[u] = col[(long long)(i + kU + u) * row_stride];
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) acc += v[u];
#pragma unroll
    for (int u = 0; u < kU; ++u) v[u] = w[u];
  }
  for (; i < t_src; ++i) acc += col[(long long)i * row_stride];
  ctx[(long long)bh * t_ctx + c] = acc / static_cast<double>(t_src);
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
// Stable rank selection (coarse.py:130-136, 196-200), parallel over elements:
// element i of a row is kept iff rank_i < kth where rank_i = #{j : (x_j, j)
// ranks before (x_i, i)} under (value desc, index asc). Values are mapped to
// order-preserving uint64 keys (-0.0 folded onto +0.0, NaN lowest) so each
// comparison is integer. grid (ceil(n/256), rows), block 256,
// dyn smem n * 8 bytes.
// ----------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long order_key(double x) {
  if (x != x) return 0ull;             // NaN ranks last
  if (x == 0.0) x = 0.0;               // -0.0 == +0.0 (numpy comparison semantics)
  const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x));
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__global__ void __launch_bounds__(256) rank_flags_kernel(const double* __restrict__ vals, int n, int kth,
                                                         uint8_t* __restrict__ flags) {
  extern __shared__ unsigned long long keys[];
  const int row = blockIdx.y;
  const double* v = vals + (long long)row * n;
  for (int j = threadIdx.x; j < n; j += blockDim.x) keys[j] = order_key(v[j]);
  __syncthreads();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const unsigned long long ki = keys[i];
  int rank = 0;
  int j = 0;
  for (; j < i; ++j) rank += keys[j] >= ki;  // earlier index wins ties
  for (++j; j < n; ++j) rank += keys[j] > ki;
  flags[(long long)row * n + i] = rank < kth;
}

// Ascending compaction of the kept (flag = 1) and dropped (flag = 0) indices of
// each row. grid rows, block 1024.
__global__ void __launch_bounds__(1024) compact_kernel(const uint8_t* __restrict__ flags, int n, int n_kept,
                                                       int* __restrict__ kept, int64_t* __restrict__ kept64,
                                                       int* __restrict__ dropped, int64_t* __restrict__ dropped64) {
  extern __shared__ int pos[];  // n ints
  __shared__ int scratch[40];
  const int row = blockIdx.x;
  const uint8_t* f = flags + (long long)row * n;
  block_exclusive_scan(f, pos, n, scratch);
  const int n_drop = n - n_kept;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    if (f[i]) {
      const int p = pos[i];
      if (kept) kept[(long long)row * n_kept + p] = i;
      if (kept64) kept64[(long long)row * n_kept + p] = i;
    } else {
      const int p = i - pos[i];
      if (dropped) dropped[(long long)row * n_drop + p] = i;
      if (dropped64) dropped64[(long long)row * n_drop + p] = i;
    }
  }
}

// ----------------------------------------------------------------------------
// K4a: sharpness of every query block: population variance over the source
// columns of the row-softmax (softmax_first) or of the raw scaled scores
// (coarse.py:193-195; softmax_rows util.py:32-40; numpy var = mean((x-mean)^2)).
// One warp per row; the row lives in registers (MAXV values per lane), so the
// fp64 exp runs once per element. grid ceil(rows/8), block 256.
// ----------------------------------------------------------------------------
template <int MAXV>
#ifndef ISA_SHARP_MINB
#define ISA_SHARP_MINB 6  // 6 CTAs per SM (40 registers, small L1 spills): 98 -> 72 us at cfg3, same results
#endif
__global__ void __launch_bounds__(256, MAXV <= 16 ? ISA_SHARP_MINB : 1) sharpness_kernel(const double* __restrict__ s, long long row_stride, int rows,
                                                        int n, int softmax_first, double* __restrict__ out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = blockIdx.x * 8 + warp;
  if (row >= rows) return;
  const double* x = s + (long long)row * row_stride;
  double val[MAXV];
  double mx = -INFINITY;
#pragma unroll
  for (int m = 0; m < MAXV; ++m) {
    const int j = lane + 32 * m;
    val[m] = j < n ? x[j] : -INFINITY;
    mx = fmax(mx, val[m]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (softmax_first) {
    double se = 0.0;
#pragma unroll
    for (int m = 0; m < MAXV; ++m) {
      val[m] = (lane + 32 * m < n) ? exp(val[m] - mx) : 0.0;
      se += val[m];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
    const double rz = 1.0 / se;
#pragma unroll
    for (int m = 0; m < MAXV; ++m) val[m] = val[m] * rz;
  }
  double sum = 0.0;
#pragma unroll
  for (int m = 0; m < MAXV; ++m) sum += (lane + 32 * m < n) ? val[m] : 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  const double mean = sum / n;
  double sq = 0.0;
#pragma unroll
  for (int m = 0; m < MAXV; ++m) {
    const double dv = val[m] - mean;
    sq += (lane + 32 * m < n) ? dv * dv : 0.0;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
  if (lane == 0) out[row] = sq / n;
}

// ----------------------------------------------------------------------------
// K5: block mask for the flat query blocks (pipeline.py:219-225,
// coarse.py:160-170): the fp64 scores of the flat block against every K_new
// block are row u of S_new; keep the top k (desc, ties -> lower index) by k
// rounds of warp arg-max over order-preserving keys in shared memory, emit
// them ascending plus a membership bitmask (W words) for the Taylor kernel.
// Row r reads scores + (row_map ? row_map[r] : r) * n. One warp per row,
// 4 warps per CTA; dyn smem 4 * (n * 8 + W * 4).
// ----------------------------------------------------------------------------
__global__ void __launch_bounds__(128) block_mask_kernel(const double* __restrict__ scores, int rows, int n,
                                                         const int* __restrict__ flat, int n_flat, int T, int k,
                                                         int W, int* __restrict__ mask_idx,
                                                         int64_t* __restrict__ mask64,
                                                         uint32_t* __restrict__ member_bits) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = blockIdx.x * 4 + warp;
  unsigned long long* sv = reinterpret_cast<unsigned long long*>(sm) + (long long)warp * n;
  uint32_t* bits = reinterpret_cast<uint32_t*>(sm + sizeof(double) * 4 * n) + warp * W;
  if (row >= rows) return;
  long long src_row = row;
  if (flat) {
    const int bh = row / n_flat, f = row % n_flat;
    src_row = (long long)bh * T + flat[(long long)bh * n_flat + f];
  }
  const double* srow = scores + src_row * n;
  for (int j = lane; j < n; j += 32) sv[j] = order_key(srow[j]);
  for (int w = lane; w < W; w += 32) bits[w] = 0u;
  __syncwarp();
  for (int r = 0; r < k; ++r) {
    unsigned long long best = 0ull;
    int bi = 0x7fffffff;
    for (int j = lane; j < n; j += 32) {
      const bool taken = (bits[j >> 5] >> (j & 31)) & 1u;
      const unsigned long long kj = sv[j];
      if (!taken && (bi == 0x7fffffff || kj > best)) {  // ascending j per lane: ties keep the lower index
        best = kj;
        bi = j;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (oi != 0x7fffffff && (bi == 0x7fffffff || ob > best || (ob == best && oi < bi))) {
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

// K5 (fast path, n <= 32*MAXM): same selection as block_mask_kernel, by a
// bitwise threshold search instead of k arg-max rounds. With ordered keys
// (hi:lo 32-bit halves) the k-th largest key is found MSB-first on hi, then
// on lo among the hi ties; elements above it are kept and exact key ties are
// taken in ascending index order (the stable tie rule). Element j of the row
// is (lane j%32, register j/32), so membership word m is one ballot.
// ----------------------------------------------------------------------------
#ifndef ISA_MASK_MINB
#define ISA_MASK_MINB 8  // 64 registers, 8 CTAs per SM: 143 -> 135 us at cfg3, same masks
#endif
template <int MAXM>
__global__ void __launch_bounds__(128, ISA_MASK_MINB) block_mask_thr_kernel(const double* __restrict__ scores, int rows, int n,
                                                             const int* __restrict__ flat, int n_flat, int T, int k,
                                                             int W, int* __restrict__ mask_idx,
                                                             int64_t* __restrict__ mask64,
                                                             uint32_t* __restrict__ member_bits) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = blockIdx.x * 4 + warp;
  if (row >= rows) return;
  long long src_row = row;
  if (flat) {
    const int bh = row / n_flat, f = row % n_flat;
    src_row = (long long)bh * T + flat[(long long)bh * n_flat + f];
  }
  const double* srow = scores + src_row * n;
  uint32_t hi[MAXM], lo[MAXM];
#pragma unroll
  for (int m = 0; m < MAXM; ++m) {
    const int j = lane + 32 * m;
    const unsigned long long key = j < n ? order_key(srow[j]) : 0ull;
    hi[m] = static_cast<uint32_t>(key >> 32);
    lo[m] = static_cast<uint32_t>(key);
  }
  auto valid = [&](int m) { return lane + 32 * m < n; };
  // hi threshold: largest th with #(hi >= th) >= k
  uint32_t th = 0;
#pragma unroll 1
  for (int b = 31; b >= 0; --b) {
    const uint32_t cand = th | (1u << b);
    int c = 0;
#pragma unroll
    for (int m = 0; m < MAXM; ++m) c += (valid(m) && hi[m] >= cand) ? 1 : 0;
    if (__reduce_add_sync(0xffffffffu, c) >= k) th = cand;
  }
  int c_gt = 0, c_eq = 0;
#pragma unroll
  for (int m = 0; m < MAXM; ++m) {
    c_gt += (valid(m) && hi[m] > th) ? 1 : 0;
    c_eq += (valid(m) && hi[m] == th) ? 1 : 0;
  }
  c_gt = __reduce_add_sync(0xffffffffu, c_gt);
  c_eq = __reduce_add_sync(0xffffffffu, c_eq);
  const int need = k - c_gt;  // >= 1 and <= c_eq
  uint32_t tl = 0;
  int need2 = 0;  // ties at exactly (th, tl) to take in index order
  if (c_eq == need) {
    tl = 0;
    need2 = 0x7fffffff;  // every hi tie is kept (lo >= 0 always)
  } else {
#pragma unroll 1
    for (int b = 31; b >= 0; --b) {
      const uint32_t cand = tl | (1u << b);
      int c = 0;
#pragma unroll
      for (int m = 0; m < MAXM; ++m) c += (valid(m) && hi[m] == th && lo[m] >= cand) ? 1 : 0;
      if (__reduce_add_sync(0xffffffffu, c) >= need) tl = cand;
    }
    int c_gt2 = 0;
#pragma unroll
    for (int m = 0; m < MAXM; ++m) c_gt2 += (valid(m) && hi[m] == th && lo[m] > tl) ? 1 : 0;
    need2 = need - __reduce_add_sync(0xffffffffu, c_gt2);
  }
  const uint32_t lt_mask = (1u << lane) - 1u;
  int taken = 0, base = 0;
#pragma unroll
  for (int m = 0; m < MAXM; ++m) {
    const bool v = valid(m);
    bool sel = v && (hi[m] > th || (hi[m] == th && lo[m] > tl));
    const bool tie = v && hi[m] == th && lo[m] == tl;
    const uint32_t tb = __ballot_sync(0xffffffffu, tie);
    sel = sel || (tie && taken + __popc(tb & lt_mask) < need2);
    taken += __popc(tb);
    const uint32_t word = __ballot_sync(0xffffffffu, sel);
    if (sel) {
      const int p = base + __popc(word & lt_mask);
      const int j = lane + 32 * m;
      if (mask_idx) mask_idx[(long long)row * k + p] = j;
      if (mask64) mask64[(long long)row * k + p] = j;
    }
    base += __popc(word);
    if (lane == 0 && member_bits && m < W) member_bits[(long long)row * W + m] = word;
  }
  if (member_bits)
    for (int m = MAXM + lane; m < W; m += 32) member_bits[(long long)row * W + m] = 0u;
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
  } else {
    for (int d = threadIdx.x; d < D; d += blockDim.x) {
      kc_bf[o + d] = __float2bfloat16_rn(0.f);
      vc_bf[o + d] = __float2bfloat16_rn(0.f);
    }
  }
}

// ----------------------------------------------------------------------------
// Taylor work plan. A CTA item holds 4 flat query blocks: Q tile s (stage)
// = blocks (4*item + 2s, 4*item + 2s + 1). For each stage, merge the two
// exact lists (bitmask OR) into an ascending union stream paired into
// 128-key tiles; each half carries the visibility bits of the CTA's query
// blocks (bit qb = 2s + row-half). The shorter stream is padded with empty
// tiles (kn = -1) so both stages share one step count. grid (n_items, BH),
// block 64 (one warp per stage).
// ----------------------------------------------------------------------------
// Entries are resolved for the attention kernel's TMA producer: {tok0, tok1,
// meta0, meta1} with tok = first source token row of the K_new block (-1 =
// none) and meta = visibility bits (bits 0-3, one per query block of the CTA)
// | valid key rows << 8, so the producer issues its loads with no dependent
// table lookups.
__device__ __forceinline__ void plan_entry(int* e, int half, int j, int vis, const int* kv_tab, int t_src, int l_src,
                                           int l_ctx) {
  int tok = -1, valid = 0;
  if (j >= 0) {
    const int u = kv_tab[j];
    tok = u < t_src ? u * 64 : l_src + (u - t_src) * 64;
    const int r = u < t_src ? l_src - u * 64 : l_ctx - (u - t_src) * 64;
    valid = r < 64 ? r : 64;
  }
  e[half] = tok;
  e[2 + half] = vis | (valid << 8);
}

__global__ void __launch_bounds__(64) taylor_plan_kernel(const uint32_t* __restrict__ member_bits, int n_flat,
                                                         int W, int n_items, int max_tiles, const int* __restrict__ kv_blk,
                                                         int t_new, int t_src, int l_src, int l_ctx,
                                                         int4* __restrict__ tiles, int* __restrict__ n_tiles) {
  __shared__ int counts[2];
  const int item = blockIdx.x, bh = blockIdx.y;
  const int s = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t* mb[2];
  for (int h = 0; h < 2; ++h) {
    const int f = item * 4 + 2 * s + h;
    mb[h] = f < n_flat ? member_bits + ((long long)bh * n_flat + f) * W : nullptr;
  }
  int4* out = tiles + (((long long)bh * n_items + item) * 2 + s) * max_tiles;
  const int* kv_tab = kv_blk + (long long)bh * t_new;
  int base = 0;
  for (int w0 = 0; w0 < W; w0 += 32) {
    const int w = w0 + lane;
    uint32_t wq[2] = {0u, 0u};
    if (w < W) {
      for (int h = 0; h < 2; ++h)
        if (mb[h]) wq[h] = mb[h][w];
    }
    const uint32_t uni = wq[0] | wq[1];
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
      const int vis = (int)(((wq[0] >> bpos) & 1u) | (((wq[1] >> bpos) & 1u) << 1)) << (2 * s);
      plan_entry(reinterpret_cast<int*>(out + (p >> 1)), p & 1, j, vis, kv_tab, t_src, l_src, l_ctx);
      ++p;
    }
    base += __shfl_sync(0xffffffffu, incl, 31);
  }
  if (lane == 0) counts[s] = base;
  __syncthreads();
  const int nt = max((counts[0] + 1) >> 1, (counts[1] + 1) >> 1);
  // close this stage's stream: odd tail half, then empty padding tiles
  const int mine = counts[s];
  if (lane == 0 && (mine & 1)) plan_entry(reinterpret_cast<int*>(out + (mine >> 1)), 1, -1, 0, kv_tab, t_src, l_src, l_ctx);
  for (int t = ((mine + 1) >> 1) + lane; t < nt; t += 32) out[t] = make_int4(-1, -1, 0, 0);
  if (threadIdx.x == 0) n_tiles[bh * n_items + item] = nt;
}

// ----------------------------------------------------------------------------
// Coarse residual O_coarse (pipeline.py:261-267): per query block u,
//   softmax variant  O_u = sum_j softmax_j(scale * qc_u . kc_j) vc_j
//   raw variant      O_u = sum_j (qc_u . kc_j) vc_j
// over all T key blocks, added to every row of block u as out += gamma * O_u
// in the attention epilogues (pipeline.py:354-356). Register-tiled fp32 flash
// attention of the T block means per head. CTA = 64 query
// blocks x all T key blocks in tiles of 64, 256 threads; thread (ty, tx) owns
// query rows 4ty..4ty+3, keys tx + 16kk (kk < 4) of S and output columns
// 4tx + 64cc (cc < D/64) of O. Q/K/V tiles are row-major in shared memory
// (row stride D+4 floats: the float4 reads of 8 consecutive tx hit 8
// distinct bank quads, the Q reads broadcast); P^T is written into the dead
// K tile. 16 FMA per 2 LDS.128 in both products. Rows / keys past T are
// zero-filled; softmax masks keys past T with -inf (raw: zero K and V rows
// contribute 0). grid (ceil(T/64), BH), 101 KB smem at D=128 (2 CTAs / SM).
// ----------------------------------------------------------------------------
template <int D>
struct ResidTile {
  static constexpr int kRow = D + 4;            // padded row, floats
  static constexpr int kQ = 0;                  // Q tile [64][kRow]
  static constexpr int kK = 64 * kRow;          // K tile [64][kRow]; P^T [64][68] after S
  static constexpr int kV = 2 * 64 * kRow;      // V tile [64][kRow]
  static constexpr int kFloats = 3 * 64 * kRow;
  static constexpr size_t kBytes = sizeof(float) * kFloats;
};

template <int D>
__device__ __forceinline__ void resid_load_rows(float* dst, const float* __restrict__ src, int row0, int T) {
  constexpr int kV4 = D / 4;
#pragma unroll 4
  for (int e = threadIdx.x; e < 64 * kV4; e += 256) {
    const int r = e / kV4, c = (e % kV4) * 4;
    float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
    if (row0 + r < T) x = *reinterpret_cast<const float4*>(src + (long long)(row0 + r) * D + c);
    *reinterpret_cast<float4*>(dst + r * ResidTile<D>::kRow + c) = x;
  }
}

template <int D>
__global__ void __launch_bounds__(256, 2) coarse_residual_tiled_kernel(const float* __restrict__ qc,
                                                                     const float* __restrict__ kc,
                                                                     const float* __restrict__ vc, int T,
                                                                     float scale, int use_softmax,
                                                                     float* __restrict__ out) {
  using L = ResidTile<D>;
  constexpr int kCC = D / 64;  // float4 output column groups per thread
  constexpr int kPRow = 68;    // P^T row stride
  extern __shared__ __align__(16) float rsm[];
  float* sq = rsm + L::kQ;
  float* sk = rsm + L::kK;
  float* sv = rsm + L::kV;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const long long base = (long long)blockIdx.y * T * D;
  const int u0 = blockIdx.x * 64;
  resid_load_rows<D>(sq, qc + base, u0, T);
  float o[4][kCC][4], m[4], l[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    m[r] = -INFINITY;
    l[r] = 0.f;
#pragma unroll
    for (int cc = 0; cc < kCC; ++cc)
#pragma unroll
      for (int j = 0; j < 4; ++j) o[r][cc][j] = 0.f;
  }
  for (int j0 = 0; j0 < T; j0 += 64) {
    __syncthreads();  // previous tile's P^T / V reads done
    resid_load_rows<D>(sk, kc + base, j0, T);
    resid_load_rows<D>(sv, vc + base, j0, T);
    __syncthreads();
    float s[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) s[r][kk] = 0.f;
#pragma unroll 4
    for (int d = 0; d < D; d += 4) {
      float4 qv[4], kv[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) qv[r] = *reinterpret_cast<const float4*>(sq + (4 * ty + r) * L::kRow + d);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) kv[kk] = *reinterpret_cast<const float4*>(sk + (tx + 16 * kk) * L::kRow + d);
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          s[r][kk] = fmaf(qv[r].x, kv[kk].x, s[r][kk]);
          s[r][kk] = fmaf(qv[r].y, kv[kk].y, s[r][kk]);
          s[r][kk] = fmaf(qv[r].z, kv[kk].z, s[r][kk]);
          s[r][kk] = fmaf(qv[r].w, kv[kk].w, s[r][kk]);
        }
    }
    if (use_softmax) {
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        float mx = -INFINITY;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          s[r][kk] = j0 + tx + 16 * kk < T ? s[r][kk] * scale : -INFINITY;
          mx = fmaxf(mx, s[r][kk]);
        }
#pragma unroll
        for (int off = 1; off < 16; off <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
        const float mn = fmaxf(m[r], mx);
        const float corr = __expf(m[r] - mn);  // m = -inf -> 0
        float ps = 0.f;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          s[r][kk] = __expf(s[r][kk] - mn);
          ps += s[r][kk];
        }
        l[r] = l[r] * corr + ps;  // this thread's partial row sum
        m[r] = mn;
#pragma unroll
        for (int cc = 0; cc < kCC; ++cc)
#pragma unroll
          for (int j = 0; j < 4; ++j) o[r][cc][j] *= corr;
      }
    }  // raw variant: p = unscaled dot; keys past T have zero K rows
    __syncthreads();  // every thread is done reading the K tile
#pragma unroll
    for (int kk = 0; kk < 4; ++kk)
      *reinterpret_cast<float4*>(sk + (tx + 16 * kk) * kPRow + 4 * ty) =
          make_float4(s[0][kk], s[1][kk], s[2][kk], s[3][kk]);
    __syncthreads();
#pragma unroll 4
    for (int j = 0; j < 64; ++j) {
      const float4 p = *reinterpret_cast<const float4*>(sk + j * kPRow + 4 * ty);
      const float pr[4] = {p.x, p.y, p.z, p.w};
#pragma unroll
      for (int cc = 0; cc < kCC; ++cc) {
        const float4 v = *reinterpret_cast<const float4*>(sv + j * L::kRow + 64 * cc + 4 * tx);
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          o[r][cc][0] = fmaf(pr[r], v.x, o[r][cc][0]);
          o[r][cc][1] = fmaf(pr[r], v.y, o[r][cc][1]);
          o[r][cc][2] = fmaf(pr[r], v.z, o[r][cc][2]);
          o[r][cc][3] = fmaf(pr[r], v.w, o[r][cc][3]);
        }
      }
    }
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    float inv = 1.f;
    if (use_softmax) {
      float lt = l[r];
#pragma unroll
      for (int off = 1; off < 16; off <<= 1) lt += __shfl_xor_sync(0xffffffffu, lt, off);
      inv = 1.f / lt;
    }
    const int u = u0 + 4 * ty + r;
    if (u >= T) continue;
#pragma unroll
    for (int cc = 0; cc < kCC; ++cc)
      *reinterpret_cast<float4*>(out + base + (long long)u * D + 64 * cc + 4 * tx) =
          make_float4(o[r][cc][0] * inv, o[r][cc][1] * inv, o[r][cc][2] * inv, o[r][cc][3] * inv);
  }
}

// ----------------------------------------------------------------------------
// Decoupled RoPE (pipeline.py:469-490): position = token index within its
// segment (source 0..L_src-1, context 0..L_ctx-1); pair i of D/2 rotates by
// pos * base^(-2i/D). One thread per (token, 4 pairs): the angles are formed
// once in fp64 and applied to every (b, h) row; HBM-bound streaming.
// ----------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(256) decoupled_rope_kernel(const T* __restrict__ x, T* __restrict__ out, int B,
                                                            int H, int S, int D, int l_src, long long xb,
                                                            long long xh, long long xs, long long ob, long long oh,
                                                            long long os, double log2_base) {
  const int per_tok = D / 8;
  const long long gid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (gid >= (long long)S * per_tok) return;
  const int tok = static_cast<int>(gid / per_tok);
  const int c0 = static_cast<int>(gid % per_tok) * 8;  // first element of this thread's 4 pairs
  const double pos = tok < l_src ? tok : tok - l_src;
  float cs[4], sn[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int i = c0 / 2 + j;
    const double theta = pos * exp2(-log2_base * (2.0 * i) / D);  // pos * base^(-2i/D)
    double sd, cd;
    sincos(theta, &sd, &cd);
    cs[j] = static_cast<float>(cd);
    sn[j] = static_cast<float>(sd);
  }
  for (int b = 0; b < B; ++b) {
    for (int h = 0; h < H; ++h) {
      const T* src = x + b * xb + h * xh + tok * xs + c0;
      T* dst = out + b * ob + h * oh + tok * os + c0;
      float v[8];
      if constexpr (sizeof(T) == 2) {
        const uint4 w = *reinterpret_cast<const uint4*>(src);
        const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          v[2 * j] = __uint_as_float(ws[j] << 16);
          v[2 * j + 1] = __uint_as_float(ws[j] & 0xffff0000u);
        }
      } else {
        const float4 a = *reinterpret_cast<const float4*>(src);
        const float4 c = *reinterpret_cast<const float4*>(src + 4);
        v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = c.x; v[5] = c.y; v[6] = c.z; v[7] = c.w;
      }
      float r[8];
#pragma unroll
      for (int j = 0; j < 4; ++j) rope_pair(v[2 * j], v[2 * j + 1], cs[j], sn[j], r[2 * j], r[2 * j + 1]);
      if constexpr (sizeof(T) == 2) {
        uint4 w;
        w.x = pack_bf16x2(r[0], r[1]);
        w.y = pack_bf16x2(r[2], r[3]);
        w.z = pack_bf16x2(r[4], r[5]);
        w.w = pack_bf16x2(r[6], r[7]);
        *reinterpret_cast<uint4*>(dst) = w;
      } else {
        *reinterpret_cast<float4*>(dst) = make_float4(r[0], r[1], r[2], r[3]);
        *reinterpret_cast<float4*>(dst + 4) = make_float4(r[4], r[5], r[6], r[7]);
      }
    }
  }
}

// int32 -> int64 export of routing lists (caller-facing int64 API, pipeline types).
__global__ void widen_kernel(const int* __restrict__ src, int64_t* __restrict__ dst, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    dst[i] = src[i];
}
// int64 -> int32 import of pinned routing.
// int64 -> int32 index narrowing, clamped into [0, hi): an out-of-range
// caller index (reported by routing_check_kernel) can never address memory
// outside the workspace / output on the way to the error.
__global__ void narrow_kernel(const int64_t* __restrict__ src, int* __restrict__ dst, long long n, int hi) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long x = src[i];
    dst[i] = static_cast<int>(x < 0 ? 0 : (x >= hi ? hi - 1 : x));
  }
}

// Pinned routing checks (isa_forward_with_routing / isa_backward(routing=)),
// the reference's index contracts: selection and the sharp/flat lists are
// gathered with _normalize_block_index (tensor.py:120-133: out of range ->
// BlockIndexError, not strictly ascending -> ContractError); the flat mask
// goes through TaylorKernelInput (taylor.py:80-84: range and order ->
// ContractError); sharp and flat must partition the T query blocks (the
// reference scatters both into one output, pipeline.py:351-353). Error bits
// (atomicOr into err): see ISA_ERRBIT_* in include/isa_b200.h.
// grid BH, block 256, dyn smem ceil(T/32) words.
__global__ void __launch_bounds__(256) routing_check_kernel(const int64_t* __restrict__ sel, int k_ctx, int t_ctx,
                                                            const int64_t* __restrict__ sharp, int n_sharp,
                                                            const int64_t* __restrict__ flat, int n_flat, int T,
                                                            const int64_t* __restrict__ mask, int k, int t_new,
                                                            int32_t* __restrict__ err) {
  extern __shared__ uint32_t seen[];
  const long long bh = blockIdx.x;
  const int W = (T + 31) >> 5;
  for (int w = threadIdx.x; w < W; w += blockDim.x) seen[w] = 0u;
  __syncthreads();
  int bits = 0;
  if (sel)
    for (int i = threadIdx.x; i < k_ctx; i += blockDim.x) {
      const long long x = sel[bh * k_ctx + i];
      if (x < 0 || x >= t_ctx) bits |= ISA_ERRBIT_SEL_RANGE;
      if (i > 0 && x <= sel[bh * k_ctx + i - 1]) bits |= ISA_ERRBIT_SEL_ORDER;
    }
  for (int part = 0; part < 2; ++part) {
    const int64_t* lst = part ? flat : sharp;
    const int n = part ? n_flat : n_sharp;
    if (!lst) continue;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const long long x = lst[bh * n + i];
      if (x < 0 || x >= T) {
        bits |= ISA_ERRBIT_SPLIT_RANGE;
        continue;
      }
      if (i > 0 && x <= lst[bh * n + i - 1]) bits |= ISA_ERRBIT_SPLIT_ORDER;
      if (atomicOr(&seen[x >> 5], 1u << (x & 31)) & (1u << (x & 31))) bits |= ISA_ERRBIT_SPLIT_ORDER;
    }
  }
  if (mask)
    for (long long e = threadIdx.x; e < (long long)n_flat * k; e += blockDim.x) {
      const long long x = mask[bh * n_flat * k + e];
      if (x < 0 || x >= t_new) bits |= ISA_ERRBIT_MASK;
      if (e % k && x <= mask[bh * n_flat * k + e - 1]) bits |= ISA_ERRBIT_MASK;
    }
  if (bits) atomicOr(err, bits);
}

// Per-head completion counters when the attention ran as separate launches:
// stream-ordered after them, one increment per head.
__global__ void head_bump_kernel(int* __restrict__ head_done, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    __threadfence();
    atomicAdd(head_done + i, 1);
  }
}

__global__ void fill_i32_kernel(int* __restrict__ out, int v, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = v;
}

// out[i] = i mod n: per-(b, h) lists 0..n-1 (the standalone Taylor kernel's flat list).
__global__ void iota_rows_kernel(int* __restrict__ out, int n, long long total) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x)
    out[i] = static_cast<int>(i % n);
}

// Pinned selection -> K_new block table.
// Also records the K_new index of the short last context block when it was
// selected (-1 otherwise): the only K_new block besides t_src-1 whose valid
// row count can be < 64 (ragged segments, pipeline.py:199-209).
__global__ void kvblk_from_sel_kernel(const int* __restrict__ sel, int t_src, int k_ctx, int t_ctx, int l_ctx,
                                      int* __restrict__ kv_blk, int* __restrict__ ctx_short_j) {
  const int bh = blockIdx.x;
  if (threadIdx.x == 0) {
    int js = -1;
    if (l_ctx & 63)
      for (int c = 0; c < k_ctx; ++c)
        if (sel[(long long)bh * k_ctx + c] == t_ctx - 1) js = t_src + c;
    ctx_short_j[bh] = js;
  }
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
