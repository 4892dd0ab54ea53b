// tcgen05 key-major dK/dV kernel of the ISA backward (exact K_new blocks):
// the sharp-branch (reference.py:173-225) and Taylor exact-slot
// (taylor.py:262-273) contributions to dK_new / dV_new, plus the centroid
// block-mean adjoint (taylor.py:290-292) and the K_new gather adjoint
// (pipeline.py:423-433) fused into the epilogue.
//
// CTA = 128 keys = K_new blocks (2x, 2x+1); it streams 64-row query units
// (query blocks: all sharp blocks, then the flat blocks whose exact list
// holds either key block). K/V stay resident in shared memory, Q/dO units
// stream through a kSlots TMA ring. TMEM holds two S^T/dP^T buffers, so the
// MMA warp computes unit i+1's S^T and dP^T while the softmax warps turn
// unit i into P^T / dS^T:
//   S^T  = K Q^T     (SS, M=128 N=64, TMEM (i&1)*128 + [0,64))
//   dP^T = V dO^T    (SS, TMEM (i&1)*128 + [64,128))
//   softmax (8 warps: thread = key row x 32-query half, packed f32x2 math):
//     P^T = exp2(S^T*sl2 - lse), dS^T = P^T (dP^T - rho), bf16 over the first
//     16 columns of the warp's own S^T / dP^T half (no cross-warp overlap)
//   dV  += P^T dO    (TS, TMEM [256,384); dO unit read MN-major)
//   dK  += dS^T Q    (TS, TMEM [384,512); Q unit read MN-major)
// The 128-query form (N=128, one buffer) ran MMA and softmax back to back
// (~4400 clk per 128 queries); here per 64-query unit the tensor pipe does
// 2 x 8 N=64 MMAs (~45 clk each, tools/ubench/mma.cu) + 2 x 4 N=D ones
// (~1230 clk) under 32 exp2 per thread (512 MUFU clk per SM sub-partition).
// Warps: 0-7 softmax + epilogue, 8 TMEM alloc + MMA issue, 9 TMA producer
// (+ per-query lse/rho rows into shared memory).
//
// CENT = true: the Taylor centroid adjoint (taylor.py:286-289) on the same
// pipeline. CTA = 128 K_new centroids (kc/vc rows c0..c0+127); units = every
// flat query block (a 1/gridDim.z share of them); key row c carries the bias
// log2(valid rows of block c) (taylor.py:156) and is masked for the query
// blocks that hold block c exactly (taylor.py:154, member bits). Writes
// scale * dK_c / dV_c into the blockIdx.z partial slab of dkc / dvc.
#pragma once
#include <type_traits>

#include "isa_bwd.cuh"

namespace isa {

struct BwdTcParams {
  BwdParams b;
  int n_list_max;  // n_sharp + n_flat (query-list capacity)
};

template <int D>
struct BwdTcSmem {
  static constexpr int kSlots = 4;
  static constexpr int kTile = 128 * D * 2;  // K / V: 128 key rows, [plane][128 rows][64 d]
  static constexpr int kUnit = 64 * D * 2;   // Q / dO: 64 query rows, [plane][64 rows][64 d]
  static constexpr int kK = 0;
  static constexpr int kV = kTile;
  static constexpr int kQO = 2 * kTile;                       // [kSlots][Q, dO]
  static constexpr int kStats = kQO + kSlots * 2 * kUnit;     // [kSlots][-lse 64 | -rho 64] floats
  static constexpr int kMem = kStats + kSlots * 128 * 4;     // [kSlots][4] member words (CENT)
  static constexpr int kBar = kMem + kSlots * 16;
  static constexpr int kList = kBar + 256;                    // int list (query-block positions) + vis flags
  static constexpr int bytes(int n_list) { return kList + 8 * n_list + 1024; }
};

template <int D, bool CENT>
__global__ void __launch_bounds__(320, 1) bwd_dkv_tc_kernel(const __grid_constant__ CUtensorMap tm_q,
                                                            const __grid_constant__ CUtensorMap tm_k,
                                                            const __grid_constant__ CUtensorMap tm_v,
                                                            const __grid_constant__ CUtensorMap tm_do,
                                                            const BwdTcParams tp) {
  using L = BwdTcSmem<D>;
  constexpr int NS = L::kSlots;
  const BwdParams& p = tp.b;
  extern __shared__ uint8_t smem_raw[];
  // 1024-aligned by pointer arithmetic on the shared array, so list / stats reads stay ld.shared
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBar);
  uint64_t* kv_full = bars + 0;
  uint64_t* d_full = bars + 1;
  uint64_t* s_full = bars + 2;               // [2] S^T / dP^T buffer written
  uint64_t* p_full = bars + 4;               // [2] P^T / dS^T of the buffer stored (per buffer: see bwd_dq)
  uint64_t* qo_full = bars + 6;              // [NS] Q / dO unit + stats landed
  uint64_t* qo_empty = bars + 6 + NS;        // [NS] dV / dK MMAs of the slot's unit done
  uint64_t* st_free = bars + 6 + 2 * NS;     // [NS] every softmax thread has read the slot's stats
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 6 + 3 * NS);
  int* s_count = reinterpret_cast<int*>(bars + 7 + 3 * NS);
  float* sStats = reinterpret_cast<float*>(smem + L::kStats);
  uint32_t* sMem = reinterpret_cast<uint32_t*>(smem + L::kMem);
  int* sList = reinterpret_cast<int*>(smem + L::kList);  // query-block position (x < n_sharp: sharp)
  int* sVis = sList + tp.n_list_max;                       // bit0: lists j0, bit1: lists j1

  const int bh = blockIdx.y;
  const int hh = bh % p.H, bb = bh / p.H;
  const int j0 = 2 * blockIdx.x, j1 = 2 * blockIdx.x + 1;
  const bool has1 = CENT || j1 < p.t_new;
  const int c0 = 128 * blockIdx.x;  // CENT: first centroid row
  // CENT: this CTA's share [f0, f1) of the flat query blocks
  const int f_per = CENT ? (p.n_flat + gridDim.z - 1) / gridDim.z : 0;
  const int f0 = CENT ? min(p.n_flat, (int)blockIdx.z * f_per) : 0;
  const int f1 = CENT ? min(p.n_flat, f0 + f_per) : 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int* tab = p.kv_blk + (long long)bh * p.t_new;

  // ---- query list (sharp blocks, then flat blocks listing j0 or j1)
  if (threadIdx.x == 0) {
    *s_count = 0;
    mbar_init(kv_full, 1);
    mbar_init(d_full, 1);
    for (int b2 = 0; b2 < 2; ++b2) {
      mbar_init(&s_full[b2], 1);
      mbar_init(&p_full[b2], 4);  // the four warps of unit parity b2
    }
    for (int s = 0; s < NS; ++s) {
      mbar_init(&qo_full[s], 32);  // every producer lane arrives after its own smem writes
      mbar_init(&qo_empty[s], 1);
      mbar_init(&st_free[s], 128);  // the four warps of the unit's parity
    }
    fence_barrier_init();
  }
  __syncthreads();
  if (CENT) {
    for (int f = f0 + threadIdx.x; f < f1; f += blockDim.x) {
      sList[f - f0] = p.n_sharp + f;
      sVis[f - f0] = 3;
    }
  } else {
  for (int x = threadIdx.x; x < p.n_sharp; x += blockDim.x) {
    sList[x] = x;
    sVis[x] = 3;
  }
  for (int f = threadIdx.x; f < p.n_flat; f += blockDim.x) {
    const uint32_t* mb = p.bits + ((long long)bh * p.n_flat + f) * p.W;
    const int v0 = (mb[j0 >> 5] >> (j0 & 31)) & 1u;
    const int v1 = has1 ? (mb[j1 >> 5] >> (j1 & 31)) & 1u : 0;
    if (v0 | v1) {
      const int at = p.n_sharp + atomicAdd(s_count, 1);
      sList[at] = p.n_sharp + f;
      sVis[at] = v0 | (v1 << 1);
    }
  }
  }
  if (warp == 8) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int n_units = CENT ? f1 - f0 : p.n_sharp + *s_count;

  if (warp == 9) {
    // ---------------------------------------------------------------- TMA producer
    const bool leader = elect_one();
    const uint64_t pol = policy_evict_last();
    if (leader) {
      mbar_arrive_expect_tx(kv_full, 2 * L::kTile);
      for (int half = 0; half < 2; ++half) {
        if (CENT) {  // kc / vc maps: {D, tn_pad, BH, 1}
          for (int pl = 0; pl < D / 64; ++pl) {
            tma_load_4d(smem + L::kK + pl * 16384 + half * 8192, &tm_k, kv_full, pl * 64, c0 + 64 * half, bh, 0, pol);
            tma_load_4d(smem + L::kV + pl * 16384 + half * 8192, &tm_v, kv_full, pl * 64, c0 + 64 * half, bh, 0, pol);
          }
          continue;
        }
        const int j = half ? (has1 ? j1 : j0) : j0;
        const int u = tab[j];
        const int tok = bw_tok0(p, u);
        for (int pl = 0; pl < D / 64; ++pl) {
          tma_load_4d(smem + L::kK + pl * 16384 + half * 8192, &tm_k, kv_full, pl * 64, tok, hh, bb, pol);
          tma_load_4d(smem + L::kV + pl * 16384 + half * 8192, &tm_v, kv_full, pl * 64, tok, hh, bb, pol);
        }
      }
    }
    // Per-unit query info (block id, lse/rho rows: lane holds rows lane, lane + 32)
    // is loaded one unit ahead into registers, so its dependent global loads
    // overlap the wait for the slot instead of delaying the TMA issue.
    struct Info {
      int u;
      float ls[2], rh[2];
    };
    auto fetch = [&](int t, Info& in) {
      in.u = -1;
      int vq = 0;
      if (t < n_units) {
        const int x = sList[t];
        in.u = x < p.n_sharp ? p.sharp[bh * p.n_sharp + x] : p.flat[bh * p.n_flat + (x - p.n_sharp)];
        vq = bw_valid(p, in.u);
      }
#pragma unroll
      for (int k2 = 0; k2 < 2; ++k2) {  // lse = -inf masks padded rows
        const int r = lane + 32 * k2;
        in.ls[k2] = -INFINITY;
        in.rh[k2] = 0.f;
        if (r < vq) {
          const long long row = (long long)bh * p.S + bw_tok0(p, in.u) + r;
          in.ls[k2] = p.lse[row];
          in.rh[k2] = p.rho[row];
        }
      }
    };
    Info cur, nxt;
    fetch(0, nxt);
    for (int t = 0; t < n_units; ++t) {
      const int slot = t % NS;
      cur = nxt;
      fetch(t + 1, nxt);  // loads in flight during the wait below
      if (t >= NS) {
        const uint32_t ph = ((t / NS) - 1) & 1;
        mbar_wait(&qo_empty[slot], ph);
        mbar_wait(&st_free[slot], ph);  // unit t-NS's stats read by every softmax thread
      }
      __syncwarp();
      float* st = sStats + slot * 128;
#pragma unroll
      for (int k2 = 0; k2 < 2; ++k2) {  // -lse (-inf for padded rows: p = 0 with no predicate), -rho
        st[lane + 32 * k2] = cur.ls[k2] > -INFINITY ? -cur.ls[k2] : -INFINITY;
        st[64 + lane + 32 * k2] = -cur.rh[k2];
      }
      if (CENT && lane < 4) {  // this query block's exact members among the 128 centroids
        const uint32_t* mb = p.bits + ((long long)bh * p.n_flat + (sList[t] - p.n_sharp)) * p.W;
        sMem[slot * 4 + lane] = (c0 >> 5) + lane < p.W ? mb[(c0 >> 5) + lane] : 0u;
      }
      __syncwarp();
      // each lane releases its own stats writes (the leader also arms the TMA bytes)
      if (!leader) mbar_arrive(&qo_full[slot]);
      if (leader) {
        mbar_arrive_expect_tx(&qo_full[slot], 2 * L::kUnit);
        uint8_t* dq_ = smem + L::kQO + slot * 2 * L::kUnit;
        const int tok = bw_tok0(p, cur.u);
        for (int pl = 0; pl < D / 64; ++pl) {
          tma_load_4d(dq_ + pl * 8192, &tm_q, &qo_full[slot], pl * 64, tok, hh, bb, pol);
          tma_load_4d(dq_ + L::kUnit + pl * 8192, &tm_do, &qo_full[slot], pl * 64, tok, hh, bb, pol);
        }
      }
    }
  } else if (warp == 8) {
    // ---------------------------------------------------------------- MMA issuer
    constexpr uint32_t idesc_s = idesc_bf16_f32(128, 64, 0, 0);
    constexpr uint32_t idesc_g = idesc_bf16_f32(128, D, 0, 1);
    const bool leader = elect_one();
    const uint64_t dk_base = sdesc_sw128_base(smem_u32(smem + L::kK), 16, 1024);
    const uint64_t dv_base = sdesc_sw128_base(smem_u32(smem + L::kV), 16, 1024);
    auto qo_desc = [&](int slot, int which, bool mn) {
      return sdesc_sw128_base(smem_u32(smem + L::kQO + (slot * 2 + which) * L::kUnit), mn ? 8192 : 16, 1024);
    };
    auto issue_sd = [&](int j) {  // S^T = K Q^T, dP^T = V dO^T of unit j into buffer j & 1
      const int slot = j % NS;
      mbar_wait(&qo_full[slot], (j / NS) & 1);
      if (leader) ISA_TSTAMP(j, 0, 5);
      __syncwarp();
      tc_fence_after();
      if (leader) {
        const uint32_t tb = tmem + (j & 1) * 128;
        const uint64_t dq = qo_desc(slot, 0, false), dd = qo_desc(slot, 1, false);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint64_t oa = ((kk >> 2) * 16384 + (kk & 3) * 32) >> 4;  // 128-row K / V planes
          const uint64_t ob = ((kk >> 2) * 8192 + (kk & 3) * 32) >> 4;   // 64-row Q / dO planes
          mma_ss(tb, dk_base + oa, dq + ob, idesc_s, kk > 0);
          mma_ss(tb + 64, dv_base + oa, dd + ob, idesc_s, kk > 0);
        }
        mma_commit(&s_full[j & 1]);
      }
      __syncwarp();
    };
    mbar_wait(kv_full, 0);
    if (n_units > 0) issue_sd(0);
    for (int i = 0; i < n_units; ++i) {
      // buffer (i+1)&1 last held unit i-1, whose softmax finished and whose
      // dV / dK MMAs were issued (in order, before these writes) last iteration
      if (i + 1 < n_units) issue_sd(i + 1);
      mbar_wait(&p_full[i & 1], (i >> 1) & 1);
      if (leader) ISA_TSTAMP(i, 0, 6);
      __syncwarp();
      tc_fence_after();
      if (leader) {
        const int slot = i % NS;
        const uint32_t tb = tmem + (i & 1) * 128;
        const uint64_t dq = qo_desc(slot, 0, true), dd = qo_desc(slot, 1, true);
        // P^T / dS^T (bf16): queries 0-31 at cols [0,16), 32-63 at [32,48) of each region
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          mma_ts(tmem + 256, tb + (kk >> 1) * 32 + (kk & 1) * 8, dd + (uint64_t)((kk * 2048) >> 4), idesc_g,
                 (i > 0) || kk > 0);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          mma_ts(tmem + 384, tb + 64 + (kk >> 1) * 32 + (kk & 1) * 8, dq + (uint64_t)((kk * 2048) >> 4), idesc_g,
                 (i > 0) || kk > 0);
        mma_commit(&qo_empty[slot]);
      }
      __syncwarp();
      if (leader) ISA_TSTAMP(i, 0, 7);
    }
    if (leader) mma_commit(d_full);
    __syncwarp();
  } else {
    // ---------------------------------------------------------------- softmax (thread = key row, unit parity = half)
    // the two warps of a TMEM lane quadrant take alternate units (buffer
    // half = unit & 1), all 64 query columns each, so both run at once on
    // their SM sub-partition and each has two units of MMA time per unit
    const int quad = warp & 3, half = warp >> 2;
    const int row = quad * 32 + lane;
    const int kh = row >> 6;  // key half (warp-uniform): 0 -> j0, 1 -> j1
    const int j = kh ? j1 : j0;
    const bool key_exists = kh == 0 || has1;
    const int uk = CENT ? 0 : (key_exists ? tab[j] : tab[j0]);
    // CENT: key row = centroid c0 + row, weighted by its block's valid rows
    const bool key_ok = CENT ? c0 + row < p.t_new : key_exists && (row & 63) < bw_valid(p, uk);
    const float cbias = (CENT && key_ok) ? __log2f((float)bw_valid(p, tab[c0 + row])) : 0.f;
    const uint32_t lane_base = static_cast<uint32_t>(quad * 32) << 16;
    const uint64_t sl2x2 = f32x2(p.sl2, p.sl2);
    for (int t = half; t < n_units; t += 2) {
      const int slot = t % NS;
      // per lane (a partial key block has invalid rows); the TMEM loads below are
      // warp-collective, so the branch is on the warp-wide OR
      mbar_wait(&qo_full[slot], (t / NS) & 1);  // the producer's lse/rho rows (+ member words) of this unit
      const bool vis = CENT ? key_ok && !((sMem[slot * 4 + (row >> 5)] >> (row & 31)) & 1u)
                            : key_ok && ((sVis[t] >> kh) & 1);
      const bool wvis = __any_sync(0xffffffffu, vis);
      mbar_wait(&s_full[half], (t >> 1) & 1);
      if ((warp & 3) == 0 && lane == 0) ISA_TSTAMP(t, 0, 0);
      __syncwarp();
      tc_fence_after();
      const uint32_t t_s = tmem + lane_base + half * 128, t_dp = t_s + 64;
#pragma unroll
      for (int ch = 0; ch < 2; ++ch) {
        uint32_t pk[16], dk[16];
        if (wvis) {
          uint32_t sr[32], dr[32];
          tmem_ld32(t_s + 32 * ch, sr);
          tmem_ld32(t_dp + 32 * ch, dr);
          tmem_ld_wait();
          const float2* nl = reinterpret_cast<const float2*>(sStats + slot * 128 + ch * 32);
          const float2* nr = reinterpret_cast<const float2*>(sStats + slot * 128 + 64 + ch * 32);
#pragma unroll
          for (int c = 0; c < 16; ++c) {
            const float2 l2 = nl[c], r2 = nr[c];  // broadcast reads: -lse, -rho of queries 2c, 2c + 1
            const uint64_t x = fma_f32x2(f32x2(__uint_as_float(sr[2 * c]), __uint_as_float(sr[2 * c + 1])), sl2x2,
                                         CENT ? f32x2(l2.x + cbias, l2.y + cbias) : f32x2(l2.x, l2.y));
            float x0, x1;
            f32x2_split(x, x0, x1);
            const float p0 = ex2_approx(x0), p1 = ex2_approx(x1);
            const uint64_t dd =
                add_f32x2(f32x2(__uint_as_float(dr[2 * c]), __uint_as_float(dr[2 * c + 1])), f32x2(r2.x, r2.y));
            float d0, d1;
            f32x2_split(mul_f32x2(f32x2(p0, p1), dd), d0, d1);
            pk[c] = vis ? pack_bf16x2(p0, p1) : 0u;
            dk[c] = vis ? pack_bf16x2(d0, d1) : 0u;
          }
        } else {
#pragma unroll
          for (int c = 0; c < 16; ++c) pk[c] = dk[c] = 0u;
        }
        tmem_st16(t_s + 32 * ch, pk);   // over this chunk's own (already read) S^T columns
        tmem_st16(t_dp + 32 * ch, dk);  // and dP^T columns
      }
      mbar_arrive(&st_free[slot]);  // this thread's reads of the slot's stats are done
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[half]);
      if ((warp & 3) == 0 && lane == 0) ISA_TSTAMP(t, 0, 4);
      if (lane == 0) ISA_TSTAMP(t, 1, warp & 3);  // P^T / dS^T stored, per lane quadrant of the group
    }
    // ---------------------------------------------------------------- epilogue
    mbar_wait(d_full, 0);
    __syncwarp();
    tc_fence_after();
    const long long orow = CENT ? 0 : (long long)bh * p.S + bw_tok0(p, uk) + (row & 63);
    const float invw = CENT ? 0.f : 1.f / (float)bw_valid(p, uk);
    const long long cb = ((long long)bh * p.t_new + j) * D;
#pragma unroll 1
    for (int c = half * (D / 64); c < (half + 1) * (D / 64); ++c) {  // each half stores half the columns
      uint32_t vr[32], kr[32];
      __syncwarp();
      tmem_ld32(tmem + lane_base + 256 + c * 32, vr);
      tmem_ld32(tmem + lane_base + 384 + c * 32, kr);
      tmem_ld_wait();
      if (n_units == 0) {  // no query block sees these keys: only the centroid part
#pragma unroll
        for (int e = 0; e < 32; ++e) vr[e] = kr[e] = 0u;
      }
      if (CENT) {  // partial slab blockIdx.z (reduced by bwd_centroid_reduce_kernel)
        if (key_ok) {
          const long long o = blockIdx.z * p.c_part + ((long long)bh * p.t_new + c0 + row) * D + c * 32;
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            p.dkc[o + e] = p.scale * __uint_as_float(kr[e]);
            p.dvc[o + e] = __uint_as_float(vr[e]);
          }
        }
      } else if (key_ok) {
        float* dkp = p.dk + orow * D + c * 32;
        float* dvp = p.dv + orow * D + c * 32;
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          float ck = 0.f, cv = 0.f;
          if (p.n_flat) {
            ck = p.dkc[cb + c * 32 + e] * invw;
            cv = p.dvc[cb + c * 32 + e] * invw;
          }
          dkp[e] = p.scale * __uint_as_float(kr[e]) + ck;
          dvp[e] = __uint_as_float(vr[e]) + cv;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 8) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// ---------------------------------------------------------------- dQ (query-major, tcgen05)
#ifdef ISA_TRACE_DQ  // tools/trace_dq.py: stamp the dQ kernel instead of dK/dV
#define DQ_TSTAMP(step, stage, slot) ISA_TSTAMP(step, stage, slot)
#else
#define DQ_TSTAMP(step, stage, slot) \
  do {                               \
  } while (0)
#endif
// CTA = 128 query rows = a pair of query blocks: sharp pairs stream every
// K_new block pair (reference.py:173-225); flat pairs (the Taylor plan's
// (item, stage) streams) stream their exact-union tiles, then every centroid
// tile (taylor.py:262-285). Key tiles are 128 keys = two 64-key blocks.
//
// tcgen05.mma costs ~45 clk per instruction at N=64 whatever the operand
// source (tools/ubench/mma.cu: 5.8 of 8.2 kFLOP/clk/SM), full rate only from
// N=128 up, so S and dP are N=128 MMAs. TMEM (512 columns) holds two S
// buffers, one dP buffer and dQ:
//   S  = Q K^T   (SS, M=128 N=128, TMEM (i&1)*128 + [0,128))
//   dP = dO V^T  (SS, TMEM [256,384)) -- rewritten for tile i+1 as soon as
//                every softmax warp has pulled tile i's dP into registers
//   softmax (8 warps: thread = query row x 64-key half, packed f32x2 math):
//                dS = P (dP - rho), bf16 over the first 32 columns of its own S half
//   dQ += dS K   (TS, K = 128 keys, TMEM [384, 384 + D); K tile read MN-major)
// so the tensor pipe runs S(i+1), dP(i+1) and dQ(i-1)... while the softmax
// warps work on tile i: per 128-key tile 3 x 512 clk of MMA (D=128) against
// 64 exp2 per thread (1024 MUFU clk per SM sub-partition) -- MMA-bound.
// Q/dO stay resident in shared memory; K streams through a 3-slot ring (it
// is read again by dQ(i), issued a tile after S(i)), V through 2 slots.
template <int D>
struct BwdDqSmem {
  static constexpr int kKSlots = 3, kVSlots = 2;
  static constexpr int kTile = 128 * D * 2;  // 128 rows: [plane][128 rows][64 d]
  static constexpr int kQ = 0;
  static constexpr int kO = kTile;
  static constexpr int kK = 2 * kTile;                     // [kKSlots]
  static constexpr int kV = kK + kKSlots * kTile;          // [kVSlots]
  static constexpr int kCol = kV + kVSlots * kTile;        // [kKSlots][128] column bias (centroid tiles) floats
  static constexpr int kMeta = kCol + kKSlots * 128 * 4;   // [kKSlots][4] ints: centroid flag, tile, meta0, meta1
  static constexpr int kBar = kMeta + 64;
  static constexpr int kBytes = kBar + 256 + 1024;
};

template <int D>
__global__ void __launch_bounds__(320, 1) bwd_dq_tc_kernel(const __grid_constant__ CUtensorMap tm_q,
                                                           const __grid_constant__ CUtensorMap tm_k,
                                                           const __grid_constant__ CUtensorMap tm_v,
                                                           const __grid_constant__ CUtensorMap tm_do,
                                                           const __grid_constant__ CUtensorMap tm_kc,
                                                           const __grid_constant__ CUtensorMap tm_vc,
                                                           const BwdParams p, const int4* __restrict__ tiles,
                                                           const int* __restrict__ n_tiles_f, int n_items,
                                                           int max_tiles, int x0) {
  using L = BwdDqSmem<D>;
  constexpr int NK = L::kKSlots, NV = L::kVSlots;
  extern __shared__ uint8_t smem_raw[];
  // 1024-aligned by pointer arithmetic on the shared array, so metadata reads stay ld.shared
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBar);
  uint64_t* qo_full = bars + 0;
  uint64_t* d_full = bars + 1;
  uint64_t* dp_full = bars + 2;              // dP of the current tile written
  uint64_t* dp_free = bars + 3;              // every softmax warp holds the tile's dP in registers
  // [2] dS of the S buffer's tile stored. Per buffer: a softmax warp may
  // finish tile i+1 before a slower one finishes tile i (dP(i+1) only waits
  // for tile i's dP loads), so one shared barrier would alias the two phases.
  uint64_t* p_full = bars + 4;
  uint64_t* s_full = bars + 6;               // [2] S buffer written
  uint64_t* kf_full = bars + 8;              // [NK] K tile + metadata landed
  uint64_t* kf_empty = bars + 8 + NK;        // [NK] dQ MMA of the slot's tile done
  uint64_t* meta_free = bars + 8 + 2 * NK;   // [NK] every softmax thread has read the slot's metadata
  uint64_t* vf_full = bars + 8 + 3 * NK;     // [NV]
  uint64_t* vf_empty = bars + 8 + 3 * NK + NV;  // [NV] dP MMA of the slot's tile done
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 8 + 3 * NK + 2 * NV);
  float* sCol = reinterpret_cast<float*>(smem + L::kCol);
  int* sMeta = reinterpret_cast<int*>(smem + L::kMeta);

  const int bh = blockIdx.y;
  const int hh = bh % p.H, bb = bh / p.H;
  const int n_sp = (p.n_sharp + 1) >> 1;  // sharp pairs
  const int bx = (int)blockIdx.x + x0;  // x0 = n_sp: a launch of the flat pairs only
  const bool flat = bx >= n_sp;
  const int pair = flat ? bx - n_sp : bx;
  const int item = pair >> 1, stg = pair & 1;  // flat: Taylor plan (item, stage)
  int u[2];
  for (int h = 0; h < 2; ++h) {
    if (!flat) {
      const int x = 2 * pair + h;
      u[h] = x < p.n_sharp ? p.sharp[bh * p.n_sharp + x] : -1;
    } else {
      const int f = 4 * item + 2 * stg + h;
      u[h] = f < p.n_flat ? p.flat[bh * p.n_flat + f] : -1;
    }
  }
  const int n_exact = flat ? n_tiles_f[bh * n_items + item] : (p.t_new + 1) >> 1;
  const int n_kv = n_exact + (flat ? p.tn_pad / 128 : 0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int* tab = p.kv_blk + (long long)bh * p.t_new;

  if (threadIdx.x == 0) {
    mbar_init(qo_full, 1);
    mbar_init(d_full, 1);
    mbar_init(dp_full, 1);
    mbar_init(dp_free, 8);
    for (int b2 = 0; b2 < 2; ++b2) {
      mbar_init(&p_full[b2], 8);
      mbar_init(&s_full[b2], 1);
    }
    for (int s2 = 0; s2 < NK; ++s2) {
      mbar_init(&kf_full[s2], 32);  // every producer lane arrives after its own smem writes
      mbar_init(&kf_empty[s2], 1);
      mbar_init(&meta_free[s2], 256);
    }
    for (int s2 = 0; s2 < NV; ++s2) {
      mbar_init(&vf_full[s2], 1);
      mbar_init(&vf_empty[s2], 1);
    }
    fence_barrier_init();
  }
  if (warp == 8) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 9) {
    // ---------------------------------------------------------------- TMA producer
    const bool leader = elect_one();
    const uint64_t pol = policy_evict_last();
    if (leader) {
      mbar_arrive_expect_tx(qo_full, 2 * L::kTile);
      for (int h = 0; h < 2; ++h) {
        const int tok = bw_tok0(p, u[h] >= 0 ? u[h] : u[0]);
        for (int pl = 0; pl < D / 64; ++pl) {
          tma_load_4d(smem + L::kQ + pl * 16384 + h * 8192, &tm_q, qo_full, pl * 64, tok, hh, bb, pol);
          tma_load_4d(smem + L::kO + pl * 16384 + h * 8192, &tm_do, qo_full, pl * 64, tok, hh, bb, pol);
        }
      }
    }
    const int4* tl = flat ? tiles + (((long long)bh * n_items + item) * 2 + stg) * max_tiles : nullptr;
    for (int i = 0; i < n_kv; ++i) {
      const int ks = i % NK, vs = i % NV;
      if (i >= NK) {
        const uint32_t ph = ((i / NK) - 1) & 1;
        mbar_wait(&kf_empty[ks], ph);
        mbar_wait(&meta_free[ks], ph);  // the slot's previous metadata read by every softmax thread
      }
      if (leader) DQ_TSTAMP(i, 1, 4);
      __syncwarp();
      int tok0, tok1, cent = 0, meta0 = 0xF | (64 << 8), meta1 = 0xF | (64 << 8);
      if (i < n_exact) {
        if (flat) {
          const int4 e = tl[i];
          tok0 = e.x >= 0 ? e.x : 0;
          tok1 = e.y >= 0 ? e.y : tok0;
          meta0 = e.z >> (2 * stg) & 3 | (e.z & ~0xFF);  // visibility bits of this pair's two blocks | valid << 8
          meta1 = e.w >> (2 * stg) & 3 | (e.w & ~0xFF);
        } else {
          const int u0 = tab[2 * i];
          tok0 = bw_tok0(p, u0);
          meta0 = 3 | (bw_valid(p, u0) << 8);
          if (2 * i + 1 < p.t_new) {
            const int u1 = tab[2 * i + 1];
            tok1 = bw_tok0(p, u1);
            meta1 = 3 | (bw_valid(p, u1) << 8);
          } else {
            tok1 = tok0;
            meta1 = 0;
          }
        }
      } else {
        cent = 1;
        tok0 = (i - n_exact) * 128;
        tok1 = tok0 + 64;
        // column weights log2(valid rows) of the 128 centroids (-inf past t_new), taylor.py:156
        for (int c = lane; c < 128; c += 32) {
          const int jj = tok0 + c;
          sCol[ks * 128 + c] = jj < p.t_new ? __log2f((float)bw_valid(p, tab[jj])) : -INFINITY;
        }
      }
      if (lane == 0) {
        sMeta[ks * 4 + 0] = cent;
        sMeta[ks * 4 + 1] = i - n_exact;
        sMeta[ks * 4 + 2] = meta0;
        sMeta[ks * 4 + 3] = meta1;
      }
      __syncwarp();
      // each lane releases its own metadata writes (the leader also arms the TMA bytes)
      if (!leader) mbar_arrive(&kf_full[ks]);
      if (leader) {
        mbar_arrive_expect_tx(&kf_full[ks], L::kTile);
        uint8_t* dk = smem + L::kK + ks * L::kTile;
        for (int h = 0; h < 2; ++h)
          for (int pl = 0; pl < D / 64; ++pl) {
            if (cent)
              tma_load_4d(dk + pl * 16384 + h * 8192, &tm_kc, &kf_full[ks], pl * 64, h ? tok1 : tok0, bh, 0, pol);
            else
              tma_load_4d(dk + pl * 16384 + h * 8192, &tm_k, &kf_full[ks], pl * 64, h ? tok1 : tok0, hh, bb, pol);
          }
        if (i >= NV) mbar_wait(&vf_empty[vs], ((i / NV) - 1) & 1);
        mbar_arrive_expect_tx(&vf_full[vs], L::kTile);
        uint8_t* dv = smem + L::kV + vs * L::kTile;
        for (int h = 0; h < 2; ++h)
          for (int pl = 0; pl < D / 64; ++pl) {
            if (cent)
              tma_load_4d(dv + pl * 16384 + h * 8192, &tm_vc, &vf_full[vs], pl * 64, h ? tok1 : tok0, bh, 0, pol);
            else
              tma_load_4d(dv + pl * 16384 + h * 8192, &tm_v, &vf_full[vs], pl * 64, h ? tok1 : tok0, hh, bb, pol);
          }
        DQ_TSTAMP(i, 1, 5);
      }
      __syncwarp();
    }
  } else if (warp == 8) {
    // ---------------------------------------------------------------- MMA issuer
    constexpr uint32_t idesc_s = idesc_bf16_f32(128, 128, 0, 0);
    constexpr uint32_t idesc_g = idesc_bf16_f32(128, D, 0, 1);
    const bool leader = elect_one();
    const uint64_t q_desc = sdesc_sw128_base(smem_u32(smem + L::kQ), 16, 1024);
    const uint64_t do_desc = sdesc_sw128_base(smem_u32(smem + L::kO), 16, 1024);
    const uint32_t kb0 = smem_u32(smem + L::kK), vb0 = smem_u32(smem + L::kV);
    auto issue_s = [&](int j) {  // S of tile j into buffer j & 1
      const int ks = j % NK;
      mbar_wait(&kf_full[ks], (j / NK) & 1);
      __syncwarp();
      tc_fence_after();
      if (leader) {
        const uint64_t dk = sdesc_sw128_base(kb0 + ks * L::kTile, 16, 1024);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint64_t o = ((kk >> 2) * 16384 + (kk & 3) * 32) >> 4;
          mma_ss(tmem + (j & 1) * 128, q_desc + o, dk + o, idesc_s, kk > 0);
        }
        mma_commit(&s_full[j & 1]);
      }
      __syncwarp();
    };
    auto issue_dp = [&](int j) {  // dP of tile j
      const int vs = j % NV;
      mbar_wait(&vf_full[vs], (j / NV) & 1);
      __syncwarp();
      tc_fence_after();
      if (leader) {
        const uint64_t dv = sdesc_sw128_base(vb0 + vs * L::kTile, 16, 1024);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint64_t o = ((kk >> 2) * 16384 + (kk & 3) * 32) >> 4;
          mma_ss(tmem + 256, do_desc + o, dv + o, idesc_s, kk > 0);
        }
        mma_commit(dp_full);
        mma_commit(&vf_empty[vs]);
      }
      __syncwarp();
    };
    mbar_wait(qo_full, 0);
    if (leader) {
      ISA_CTA_SPAN(0, global_ns());
      ISA_CTA_SPAN(2, 2 * n_kv);
      unsigned sm;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
      ISA_CTA_SPAN(3, sm);
    }
    if (n_kv > 0) {
      issue_s(0);
      issue_dp(0);
    }
    for (int i = 0; i < n_kv; ++i) {
      // S buffer (i+1)&1 last held tile i-1: its softmax finished and its dQ
      // MMA was issued (in order, before these writes) last iteration
      if (i + 1 < n_kv) {
        issue_s(i + 1);
        mbar_wait(dp_free, i & 1);  // tile i's dP is in the softmax registers
        issue_dp(i + 1);
      }
      if (leader) DQ_TSTAMP(i, 1, 2);
      mbar_wait(&p_full[i & 1], (i >> 1) & 1);
      if (leader) DQ_TSTAMP(i, 1, 3);
      __syncwarp();
      tc_fence_after();
      if (leader) {
        const int ks = i % NK;
        const uint64_t dkm = sdesc_sw128_base(kb0 + ks * L::kTile, 16384, 1024);  // K as the MN-major B
        const uint32_t ts = tmem + (i & 1) * 128;  // dS (bf16): keys 0-63 at cols [0,32), 64-127 at [64,96)
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)  // 128 keys = 8 x 16
          mma_ts(tmem + 384, ts + (kk >> 2) * 64 + (kk & 3) * 8, dkm + (uint64_t)((kk * 2048) >> 4), idesc_g,
                 (i > 0) || kk > 0);
        mma_commit(&kf_empty[ks]);
      }
      __syncwarp();
    }
    if (leader) mma_commit(d_full);
    __syncwarp();
  } else {
    // ---------------------------------------------------------------- softmax (thread = query row x key half)
    const int quad = warp & 3, half = warp >> 2;  // TMEM lane quadrant; keys [64 half, 64 half + 64) = one block
    const int row = quad * 32 + lane;
    const int qh = row >> 6;  // warp-uniform
    const int uq = u[qh];
    const int vq = uq >= 0 ? bw_valid(p, uq) : 0;
    const bool row_ok = (row & 63) < vq;
    const long long grow = row_ok ? (long long)bh * p.S + bw_tok0(p, uq) + (row & 63) : 0;
    const float lse = row_ok ? p.lse[grow] : -INFINITY;
    const float rho = row_ok ? p.rho[grow] : 0.f;
    const bool live = row_ok && lse > -INFINITY;
    const float lse_eff = live ? lse : INFINITY;  // dead rows: exp2(-inf) = 0, no per-element predicate
    const uint32_t* mb = (flat && uq >= 0) ? p.bits + ((long long)bh * p.n_flat + 4 * item + 2 * stg + qh) * p.W
                                           : nullptr;
    const uint32_t lane_base = static_cast<uint32_t>(quad * 32) << 16;
    const uint64_t sl2x2 = f32x2(p.sl2, p.sl2), nlse2 = f32x2(-lse_eff, -lse_eff), nrho2 = f32x2(-rho, -rho);
    const uint32_t t_dp = tmem + lane_base + 256 + half * 64;
    for (int i = 0; i < n_kv; ++i) {
      const int ks = i % NK;
      mbar_wait(&kf_full[ks], (i / NK) & 1);  // the producer's per-tile metadata
      if (threadIdx.x == 0) DQ_TSTAMP(i, 0, 2);
      const int cent = sMeta[ks * 4 + 0], cidx = sMeta[ks * 4 + 1], m = sMeta[ks * 4 + 2 + half];
      // exact tiles: valid keys of this half's block if this row's block sees it (warp-uniform)
      const int lc = ((m >> qh) & 1) ? (m >> 8) : 0;
      uint32_t cw[2] = {0u, 0u};
      float colb[2] = {0.f, 0.f};  // lane c holds column 32 ch + c's weight
      if (cent) {
        if (mb) {
          cw[0] = __ldg(mb + cidx * 4 + 2 * half);  // own exact members excluded
          cw[1] = __ldg(mb + cidx * 4 + 2 * half + 1);
        }
        colb[0] = sCol[ks * 128 + half * 64 + lane];
        colb[1] = sCol[ks * 128 + half * 64 + 32 + lane];
      }
      const uint32_t t_s = tmem + lane_base + (i & 1) * 128 + half * 64;
      mbar_wait(&s_full[i & 1], (i >> 1) & 1);
      mbar_wait(dp_full, i & 1);
      if (threadIdx.x == 0) DQ_TSTAMP(i, 0, 1);
      __syncwarp();
      tc_fence_after();
      if (!cent && lc <= 0) {
        // block invisible to this query block: dS = 0
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(dp_free);
        uint32_t z[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) z[c] = 0u;
        tmem_st16(t_s, z);
        tmem_st16(t_s + 16, z);
      } else {
        uint32_t dr[2][32];
        tmem_ld32(t_dp, dr[0]);
        tmem_ld32(t_dp + 32, dr[1]);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(dp_free);  // the MMA warp may overwrite dP with tile i+1's
#pragma unroll
        for (int ch = 0; ch < 2; ++ch) {
          uint32_t sr[32], pk[16];
          tmem_ld32(t_s + ch * 32, sr);
          tmem_ld_wait();
          if (!cent && lc >= 64) {
            // whole block visible: no masking, two columns per packed op
#pragma unroll
            for (int c = 0; c < 16; ++c) {
              const uint64_t x =
                  fma_f32x2(f32x2(__uint_as_float(sr[2 * c]), __uint_as_float(sr[2 * c + 1])), sl2x2, nlse2);
              float x0, x1;
              f32x2_split(x, x0, x1);
              const uint64_t pr = f32x2(ex2_approx(x0), ex2_approx(x1));
              const uint64_t dd =
                  add_f32x2(f32x2(__uint_as_float(dr[ch][2 * c]), __uint_as_float(dr[ch][2 * c + 1])), nrho2);
              float d0, d1;
              f32x2_split(mul_f32x2(pr, dd), d0, d1);
              pk[c] = pack_bf16x2(d0, d1);
            }
          } else {
            const int lcc = lc - 32 * ch;
#pragma unroll
            for (int c = 0; c < 16; ++c) {
              float dvv[2];
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const int cc = 2 * c + e;  // column within the chunk
                float bias;
                if (cent)
                  bias = ((cw[ch] >> cc) & 1u) ? -INFINITY : __shfl_sync(0xffffffffu, colb[ch], cc);
                else
                  bias = cc < lcc ? 0.f : -INFINITY;
                const float pr = ex2_approx(fmaf(__uint_as_float(sr[cc]), p.sl2, bias - lse_eff));
                dvv[e] = pr * (__uint_as_float(dr[ch][cc]) - rho);
              }
              pk[c] = pack_bf16x2(dvv[0], dvv[1]);
            }
          }
          tmem_st16(t_s + ch * 16, pk);  // over S columns this thread has already read
        }
      }
      mbar_arrive(&meta_free[ks]);  // this thread's reads of the tile's metadata are done
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (threadIdx.x == 0) DQ_TSTAMP(i, 0, 3);
      if (lane == 0) mbar_arrive(&p_full[i & 1]);
    }
    // ---------------------------------------------------------------- epilogue
    mbar_wait(d_full, 0);
    __syncwarp();
    tc_fence_after();
#pragma unroll 1
    for (int c = half * (D / 64); c < (half + 1) * (D / 64); ++c) {
      uint32_t qr[32];
      __syncwarp();
      tmem_ld32(tmem + lane_base + 384 + c * 32, qr);
      tmem_ld_wait();
      if (row_ok) {
        float* dst = p.dq + grow * D + c * 32;
#pragma unroll
        for (int e = 0; e < 32; ++e) dst[e] = n_kv ? p.scale * __uint_as_float(qr[e]) : 0.f;
      }
    }
  }
  if (threadIdx.x == 0) ISA_CTA_SPAN(1, global_ns());
  tc_fence_before();
  __syncthreads();
  if (warp == 8) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// ---------------------------------------------------------------- dQ of the sharp blocks on CTA pairs
#ifdef ISA_TRACE_DQP  // tools/trace_dq.py --pair: stamp the CTA-pair dQ kernel
#define DQP_TSTAMP(step, stage, slot) ISA_TSTAMP(step, stage, slot)
#else
#define DQP_TSTAMP(step, stage, slot) \
  do {                                \
  } while (0)
#endif
// The sharp pairs all stream every K_new tile, so two of them (a 2-CTA
// cluster, 256 query rows) share one tcgen05.mma.cta_group::2 stream: M = 256
// (each CTA's 128 rows, its own Q/dO and TMEM), the B operand split between
// the two CTAs' shared memory. Per 128-key tile, CTA r loads
//   K block 2i+r, both d planes (16 KB): its half of S = Q K^T's B (N = keys)
//   d plane r of both K blocks (16 KB):  its half of dQ += dS K's B (N = d)
//   V block 2i+r, both d planes (16 KB): its half of dP = dO V^T's B
// i.e. 48 KB of TMA and 48 + 48 + 16 KB of MMA operand reads per SM per tile
// instead of 64 and 64 + 64 + 32 (the single-CTA kernel is bound by that
// shared-memory traffic, ~1,750 clk per tile against 1,536 of MMA). The
// leader (rank 0) issues every MMA; commits are multicast to both CTAs; the
// full barriers of the TMA bytes and the softmax arrivals (dP pulled into
// registers, dS stored) live in the leader. Softmax and epilogue are those of
// bwd_dq_tc_kernel (sharp tiles only: no metadata slots, the valid rows come
// from the block table).
template <int D>
struct BwdDqPairLayout {
  static constexpr int kKSlots = 3, kVSlots = 2;
  static constexpr int kTile = 128 * D * 2;   // Q / dO: 128 rows
  static constexpr int kHalf = 64 * D * 2;    // 64 rows x D (two planes of 8 KB at D = 128)
  static constexpr int kKSlot = 2 * kHalf;    // [S part: own block, planes 0..][dQ part: plane r of both blocks]
  static constexpr int kVSlot = kHalf;        // own V block, planes 0..
  static constexpr int kQ = 0;
  static constexpr int kO = kTile;
  static constexpr int kK = 2 * kTile;
  static constexpr int kV = kK + kKSlots * kKSlot;
  static constexpr int kBar = kV + kVSlots * kVSlot;
  static constexpr int kValid = kBar + 256;  // [t_new] valid rows of each K_new block (softmax masks)
  static constexpr int bytes(int t_new) { return kValid + 4 * t_new + 1024; }
};

template <int D>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(320, 1)
    bwd_dq_pair_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                       const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_do,
                       const BwdParams p) {
  static_assert(D == 128, "the pair dQ kernel splits the d planes between the two CTAs");
  using L = BwdDqPairLayout<D>;
  constexpr int NK = L::kKSlots, NV = L::kVSlots;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBar);
  uint64_t* qo_full = bars + 0;               // leader: both CTAs' Q / dO bytes
  uint64_t* d_full = bars + 1;                // multicast commit
  uint64_t* dp_full = bars + 2;               // multicast commit
  uint64_t* dp_free = bars + 3;               // leader: 16 softmax warps hold dP
  uint64_t* p_full = bars + 4;                // [2] leader: 16 softmax warps stored dS
  uint64_t* s_full = bars + 6;                // [2] multicast commit
  uint64_t* kf_full = bars + 8;               // [NK] leader: both CTAs' K bytes
  uint64_t* kf_empty = bars + 8 + NK;         // [NK] multicast commit after dQ(i)
  uint64_t* vf_full = bars + 8 + 2 * NK;      // [NV] leader: both CTAs' V bytes
  uint64_t* vf_empty = bars + 8 + 2 * NK + NV;  // [NV] multicast commit after dP(i)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 8 + 2 * NK + 2 * NV);
  int* sValid = reinterpret_cast<int*>(smem + L::kValid);
  const uint32_t rank = cluster_ctarank();

  const int bh = blockIdx.y;
  const int hh = bh % p.H, bb = bh / p.H;
  const int pair = blockIdx.x;  // sharp pair index (query blocks 2 pair, 2 pair + 1)
  int u[2];
  for (int h = 0; h < 2; ++h) {
    const int x = 2 * pair + h;
    u[h] = x < p.n_sharp ? p.sharp[bh * p.n_sharp + x] : -1;
  }
  const int n_kv = (p.t_new + 1) >> 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int* tab = p.kv_blk + (long long)bh * p.t_new;

  if (threadIdx.x == 0) {
    mbar_init(qo_full, 1);
    mbar_init(d_full, 1);
    mbar_init(dp_full, 1);
    mbar_init(dp_free, 16);
    for (int b2 = 0; b2 < 2; ++b2) {
      mbar_init(&p_full[b2], 16);
      mbar_init(&s_full[b2], 1);
    }
    for (int s2 = 0; s2 < NK; ++s2) {
      mbar_init(&kf_full[s2], 1);
      mbar_init(&kf_empty[s2], 1);
    }
    for (int s2 = 0; s2 < NV; ++s2) {
      mbar_init(&vf_full[s2], 1);
      mbar_init(&vf_empty[s2], 1);
    }
    fence_barrier_init();
  }
  for (int j = threadIdx.x; j < p.t_new; j += blockDim.x) sValid[j] = bw_valid(p, __ldg(tab + j));
  if (warp == 8) tmem_alloc2<512>(tmem_slot);
  tc_fence_before();
  cluster_sync_all();  // both CTAs' barriers initialised before any cross-CTA signal (+ sValid)
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 9) {
    // ---------------------------------------------------------------- TMA producer (both CTAs)
    const bool leader = elect_one();
    const uint64_t pol = policy_evict_last();
    if (leader) {
      if (rank == 0) mbar_arrive_expect_tx(qo_full, 4 * L::kTile);
      for (int h = 0; h < 2; ++h) {
        const int tok = bw_tok0(p, u[h] >= 0 ? u[h] : (u[0] >= 0 ? u[0] : p.sharp[bh * p.n_sharp]));
        for (int pl = 0; pl < D / 64; ++pl) {
          tma_load_4d_pair(smem + L::kQ + pl * 16384 + h * 8192, &tm_q, qo_full, pl * 64, tok, hh, bb, pol);
          tma_load_4d_pair(smem + L::kO + pl * 16384 + h * 8192, &tm_do, qo_full, pl * 64, tok, hh, bb, pol);
        }
      }
    }
    int tok_nxt[2];
    auto tile_tok = [&](int i, int (&t)[2]) {
      const int u0 = __ldg(tab + 2 * i);
      t[0] = bw_tok0(p, u0);
      t[1] = 2 * i + 1 < p.t_new ? bw_tok0(p, __ldg(tab + 2 * i + 1)) : t[0];  // missing block: masked
    };
    tile_tok(0, tok_nxt);
    for (int i = 0; i < n_kv; ++i) {
      int tok[2] = {tok_nxt[0], tok_nxt[1]};
      if (i + 1 < n_kv) tile_tok(i + 1, tok_nxt);  // next lookups in flight during the waits
      const int ks = i % NK, vs = i % NV;
      if (i >= NK) mbar_wait(&kf_empty[ks], ((i / NK) - 1) & 1);
      if (leader) {
        uint8_t* dk = smem + L::kK + ks * L::kKSlot;
        if (rank == 0) mbar_arrive_expect_tx(&kf_full[ks], 2 * L::kKSlot);
        for (int pl = 0; pl < D / 64; ++pl)  // S part: own block 2i + rank, both planes
          tma_load_4d_pair(dk + pl * 8192, &tm_k, &kf_full[ks], pl * 64, tok[rank], hh, bb, pol);
        for (int h = 0; h < 2; ++h)  // dQ part: plane `rank` of both blocks, [128 keys][64 d]
          tma_load_4d_pair(dk + L::kHalf + h * 8192, &tm_k, &kf_full[ks], static_cast<int>(rank) * 64, tok[h], hh,
                           bb, pol);
      }
      if (i >= NV) mbar_wait(&vf_empty[vs], ((i / NV) - 1) & 1);
      if (leader) {
        uint8_t* dv = smem + L::kV + vs * L::kVSlot;
        if (rank == 0) mbar_arrive_expect_tx(&vf_full[vs], 2 * L::kVSlot);
        for (int pl = 0; pl < D / 64; ++pl)
          tma_load_4d_pair(dv + pl * 8192, &tm_v, &vf_full[vs], pl * 64, tok[rank], hh, bb, pol);
      }
      __syncwarp();
    }
    // drain: the leader's multicast releases of this CTA's slots have all landed
    for (int e = n_kv > NK ? n_kv - NK : 0; e < n_kv; ++e) mbar_wait(&kf_empty[e % NK], (e / NK) & 1);
    for (int e = n_kv > NV ? n_kv - NV : 0; e < n_kv; ++e) mbar_wait(&vf_empty[e % NV], (e / NV) & 1);
  } else if (warp == 8) {
    // ---------------------------------------------------------------- MMA issuer (leader CTA)
    if (rank == 0) {
      constexpr uint32_t idesc_s = idesc_bf16_f32(256, 128, 0, 0);
      constexpr uint32_t idesc_g = idesc_bf16_f32(256, D, 0, 1);
      const bool leader = elect_one();
      const uint64_t q_desc = sdesc_sw128_base(smem_u32(smem + L::kQ), 16, 1024);
      const uint64_t do_desc = sdesc_sw128_base(smem_u32(smem + L::kO), 16, 1024);
      const uint32_t kb0 = smem_u32(smem + L::kK), vb0 = smem_u32(smem + L::kV);
      auto issue_s = [&](int j) {  // S of tile j into buffer j & 1
        const int ks = j % NK;
        mbar_wait(&kf_full[ks], (j / NK) & 1);
        __syncwarp();
        tc_fence_after();
        if (leader) {
          const uint64_t dk = sdesc_sw128_base(kb0 + ks * L::kKSlot, 16, 1024);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint64_t oa = ((kk >> 2) * 16384 + (kk & 3) * 32) >> 4;  // 128-row Q planes
            const uint64_t ob = ((kk >> 2) * 8192 + (kk & 3) * 32) >> 4;   // 64-key K planes
            mma_ss2(tmem + (j & 1) * 128, q_desc + oa, dk + ob, idesc_s, kk > 0);
          }
          mma_commit_pair(&s_full[j & 1]);
        }
        __syncwarp();
      };
      auto issue_dp = [&](int j) {  // dP of tile j
        const int vs = j % NV;
        mbar_wait(&vf_full[vs], (j / NV) & 1);
        __syncwarp();
        tc_fence_after();
        if (leader) {
          const uint64_t dv = sdesc_sw128_base(vb0 + vs * L::kVSlot, 16, 1024);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint64_t oa = ((kk >> 2) * 16384 + (kk & 3) * 32) >> 4;
            const uint64_t ob = ((kk >> 2) * 8192 + (kk & 3) * 32) >> 4;
            mma_ss2(tmem + 256, do_desc + oa, dv + ob, idesc_s, kk > 0);
          }
          mma_commit_pair(dp_full);
          mma_commit_pair(&vf_empty[vs]);
        }
        __syncwarp();
      };
      mbar_wait(qo_full, 0);
      if (n_kv > 0) {
        issue_s(0);
        issue_dp(0);
      }
      for (int i = 0; i < n_kv; ++i) {
        if (i + 1 < n_kv) {
          issue_s(i + 1);
          mbar_wait(dp_free, i & 1);  // tile i's dP is in both CTAs' softmax registers
          issue_dp(i + 1);
        }
        if (leader) DQP_TSTAMP(i, 1, 2);
        mbar_wait(&p_full[i & 1], (i >> 1) & 1);
        if (leader) DQP_TSTAMP(i, 1, 3);
        __syncwarp();
        tc_fence_after();
        if (leader) {
          const int ks = i % NK;
          const uint64_t dkm = sdesc_sw128_base(kb0 + ks * L::kKSlot + L::kHalf, 16384, 1024);  // [128 keys][64 d]
          const uint32_t ts = tmem + (i & 1) * 128;  // dS (bf16): keys 0-63 at cols [0,32), 64-127 at [64,96)
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            mma_ts2(tmem + 384, ts + (kk >> 2) * 64 + (kk & 3) * 8, dkm + (uint64_t)((kk * 2048) >> 4), idesc_g,
                    (i > 0) || kk > 0);
          mma_commit_pair(&kf_empty[ks]);
        }
        __syncwarp();
      }
      if (leader) mma_commit_pair(d_full);
      __syncwarp();
    }
  } else {
    // ---------------------------------------------------------------- softmax (thread = query row x key half)
    const int quad = warp & 3, half = warp >> 2;  // TMEM lane quadrant; keys [64 half, 64 half + 64) = one block
    const int row = quad * 32 + lane;
    const int qh = row >> 6;
    const int uq = u[qh];
    const int vq = uq >= 0 ? bw_valid(p, uq) : 0;
    const bool row_ok = (row & 63) < vq;
    const long long grow = row_ok ? (long long)bh * p.S + bw_tok0(p, uq) + (row & 63) : 0;
    const float lse = row_ok ? p.lse[grow] : -INFINITY;
    const float rho = row_ok ? p.rho[grow] : 0.f;
    const bool live = row_ok && lse > -INFINITY;
    const float lse_eff = live ? lse : INFINITY;  // dead rows: exp2(-inf) = 0, no per-element predicate
    const uint32_t lane_base = static_cast<uint32_t>(quad * 32) << 16;
    const uint64_t sl2x2 = f32x2(p.sl2, p.sl2), nlse2 = f32x2(-lse_eff, -lse_eff), nrho2 = f32x2(-rho, -rho);
    const uint32_t t_dp = tmem + lane_base + 256 + half * 64;
    auto arrive_leader = [&](uint64_t* bar) {
      if (rank)
        mbar_arrive_leader(bar);
      else
        mbar_arrive(bar);
    };
    for (int i = 0; i < n_kv; ++i) {
      // valid keys of this half's K_new block (warp-uniform), from shared memory: a
      // dependent table load here sat on the softmax loop's critical path (~450 clk)
      const int lc = 2 * i + half < p.t_new ? sValid[2 * i + half] : 0;
      const uint32_t t_s = tmem + lane_base + (i & 1) * 128 + half * 64;
      if (threadIdx.x == 0) DQP_TSTAMP(i, 0, 2);
      mbar_wait(&s_full[i & 1], (i >> 1) & 1);
      mbar_wait(dp_full, i & 1);
      if (threadIdx.x == 0) DQP_TSTAMP(i, 0, 1);
      __syncwarp();
      tc_fence_after();
      if (lc <= 0) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) arrive_leader(dp_free);
        uint32_t z[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) z[c] = 0u;
        tmem_st16(t_s, z);
        tmem_st16(t_s + 16, z);
      } else {
        uint32_t dr[2][32], srr[2][32];  // the whole 64-key half row of dP and S: one TMEM round trip
        tmem_ld32(t_dp, dr[0]);
        tmem_ld32(t_dp + 32, dr[1]);
        tmem_ld32(t_s, srr[0]);
        tmem_ld32(t_s + 32, srr[1]);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) arrive_leader(dp_free);  // the MMA warp may overwrite dP with tile i+1's
#pragma unroll
        for (int ch = 0; ch < 2; ++ch) {
          uint32_t pk[16];
          const uint32_t (&sr)[32] = srr[ch];
          if (lc >= 64) {
#pragma unroll
            for (int c = 0; c < 16; ++c) {
              const uint64_t x =
                  fma_f32x2(f32x2(__uint_as_float(sr[2 * c]), __uint_as_float(sr[2 * c + 1])), sl2x2, nlse2);
              float x0, x1;
              f32x2_split(x, x0, x1);
              uint64_t pr;
              if (kEmuEvery > 0 && (c % kEmuEvery) == kEmuEvery - 1) {  // 1 in kEmuEvery pairs on the FMA pipe
                const float2 e = ex2_emu2(make_float2(x0, x1));
                pr = f32x2(e.x, e.y);
              } else {
                pr = f32x2(ex2_approx(x0), ex2_approx(x1));
              }
              const uint64_t dd =
                  add_f32x2(f32x2(__uint_as_float(dr[ch][2 * c]), __uint_as_float(dr[ch][2 * c + 1])), nrho2);
              float d0, d1;
              f32x2_split(mul_f32x2(pr, dd), d0, d1);
              pk[c] = pack_bf16x2(d0, d1);
            }
          } else {
            const int lcc = lc - 32 * ch;
#pragma unroll
            for (int c = 0; c < 16; ++c) {
              float dvv[2];
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const int cc = 2 * c + e;
                const float bias = cc < lcc ? 0.f : -INFINITY;
                const float pr = ex2_approx(fmaf(__uint_as_float(sr[cc]), p.sl2, bias - lse_eff));
                dvv[e] = pr * (__uint_as_float(dr[ch][cc]) - rho);
              }
              pk[c] = pack_bf16x2(dvv[0], dvv[1]);
            }
          }
          tmem_st16(t_s + ch * 16, pk);  // over S columns this thread has already read
        }
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (threadIdx.x == 0) DQP_TSTAMP(i, 0, 3);
      if (lane == 0) arrive_leader(&p_full[i & 1]);
    }
    // ---------------------------------------------------------------- epilogue
    mbar_wait(d_full, 0);
    __syncwarp();
    tc_fence_after();
#pragma unroll 1
    for (int c = half * (D / 64); c < (half + 1) * (D / 64); ++c) {
      uint32_t qr[32];
      __syncwarp();
      tmem_ld32(tmem + lane_base + 384 + c * 32, qr);
      tmem_ld_wait();
      if (row_ok) {
        float* dst = p.dq + grow * D + c * 32;
#pragma unroll
        for (int e = 0; e < 32; ++e) dst[e] = n_kv ? p.scale * __uint_as_float(qr[e]) : 0.f;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // the peer's MMAs / signals into this CTA are complete
  if (warp == 8) {
    tc_fence_after();
    tmem_dealloc2<512>(tmem);
  }
}

}  // namespace isa
