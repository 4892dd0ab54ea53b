// K7T: the Taylor branch (taylor.py:124-160) computed transposed, D = 128.
//
// The row-major K7 (isa_attn.cuh, MODE_TAYLOR) puts two flat query blocks in
// one 128-row MMA tile and streams the union of their exact lists: with
// unrelated lists half of every S tile belongs to the other block (50% MMA
// waste on iid routing). Here each query block u runs alone with its own
// exact blocks, and the tensor-core M dimension is carried by keys and by the
// head dim instead of by queries:
//
//   S^T (128 keys x 64 queries)  = K_tile . Q_u^T      SS MMA, M=128, N=64
//   O^T (128 d    x 64 queries) += V_tile^T . P^T      SS MMA, M=128, N=64
//
// (M=128/N=64 runs at the full tcgen05 rate: floor = max(M,128)*N/256 cycles
// per K=16 step.) A tile is a pair of u's exact K_new blocks (k/2 tiles), then
// the tn_pad/128 centroid tiles (128 centroids each, weights 2^log2(w) as a
// per-key bias, u's own exact members excluded, taylor.py:153-159).
//
// Softmax: TMEM lane = key, so each thread owns one key's 64 query scores.
// The per-query running max m[q] lives in shared memory. Speculative
// exponentiation against m (a tile whose scores exceed m + 8 anywhere —
// detected with one barrier.red.or across the stage's 4 warps — takes the slow
// path: per-query tile max by a recursive-halving warp reduction + a 4-warp
// combine, lazy rescale of O^T columns and of the row-sum partials). Row sums
// are kept as per-key partials (one register per query) and reduced once in
// the epilogue. P^T (bf16) goes to shared memory in the SW128 K-row layout the
// second MMA reads as an MN-major B operand.
//
// CTA: two query blocks (stages 0/1, ping-pong like the row-major kernel),
// warps 0-7 softmax (4 per stage, 208 registers), warp 8 MMA issuer, warp 9
// TMA producer, warps 10-11 idle (88 registers each for warps 8-11).
// TMEM: S^T stage s, buffer b at columns 128s + 64b; O^T at 256 + 64s.
// S^T is double-buffered per stage, so QK(i+2) overlaps the softmax of tile
// i; P^T has one buffer per stage (the softmax of tile i waits PV(i-1)).
#pragma once
#include "isa_attn.cuh"

namespace isa {

constexpr int kTThreads = 384;  // warps 10-11 only complete the register-donating warpgroup
#ifndef ISA_TT_KV_STAGES
#define ISA_TT_KV_STAGES 5
#endif
constexpr int kTKvStages = ISA_TT_KV_STAGES;  // K/V ring slots of 32 KB
#ifndef ISA_TT_EMU
#define ISA_TT_EMU ISA_EMU_EVERY
#endif
constexpr int kTTEmu = ISA_TT_EMU;  // 1 in kTTEmu exp2 pairs on the FMA pipe (0 = none)

template <int D>
struct TaylorTSmem {
  static_assert(D == 128, "the transposed Taylor kernel is instantiated for D = 128");
  static constexpr int kQStage = 64 * D * 2;   // one 64-row query block, 2 planes of 8 KB
  static constexpr int kTile = 128 * D * 2;    // 128 keys, 2 planes of 16 KB
  static constexpr int kPT = 128 * 64 * 2;     // P^T: 128 key rows x 64 queries (bf16, SW128)
  static constexpr int kQOff = 0;
  static constexpr int kKvOff = 2 * kQStage;
  static constexpr int kPOff = kKvOff + kTKvStages * kTile;  // P^T [stage][buffer]
  static constexpr int kBarOff = kPOff + 2 * kPT;
  static constexpr int kBytes = kBarOff + 256;
  static constexpr int kAlloc = kBytes + 1024;
};

// After the call, v[0] / v[1] hold the reduction over the warp's 32 lanes for
// queries 2*lane and 2*lane + 1 (recursive halving: 62 shuffles for 64 values).
template <bool kMax>
__device__ __forceinline__ void warp_halve64(float (&v)[64], const int lane) {
#pragma unroll
  for (int h = 64, off = 16; h > 2; h >>= 1, off >>= 1) {
    const bool low = !(lane & off);
#pragma unroll
    for (int j = 0; j < h / 2; ++j) {
      const float send = low ? v[j + h / 2] : v[j];
      const float keep = low ? v[j] : v[j + h / 2];
      const float recv = __shfl_xor_sync(0xffffffffu, send, off);
      v[j] = kMax ? fmaxf(keep, recv) : keep + recv;
    }
  }
}

struct TTileSrc {
  int tok0, tok1, centroid;
};

constexpr int kTTokRegs = 3;  // exact blocks resolved up front: k <= 32 * kTTokRegs (larger k: lookups per tile)

// Token row of exact block j of a stage from the producer warp's registers
// (lane j % 32 holds entry j in tok[j / 32]); every lane must participate.
__device__ __forceinline__ int tt_tok(const int (&tok)[kTTokRegs], int j) {
  int v = tok[0];
#pragma unroll
  for (int r = 1; r < kTTokRegs; ++r)
    if ((j >> 5) == r) v = tok[r];
  return __shfl_sync(0xffffffffu, v, j & 31);
}

// Tile i of stage (flat position) pos: exact pair (mask[2i], mask[2i+1]) or
// centroid tile i - n_ex. With `tok` the stage's exact blocks were resolved
// once before the loop (mask -> K_new block table -> token row), so the
// producer issues loads without dependent global lookups.
__device__ __forceinline__ TTileSrc tt_tile(const AttnParams& p, int bh, int pos, int i, int n_ex, bool table,
                                            const int (&tok)[kTTokRegs]) {
  TTileSrc t;
  if (i >= n_ex) {
    t.centroid = 1;
    t.tok0 = (i - n_ex) * 128;
    t.tok1 = t.tok0 + 64;
    return t;
  }
  t.centroid = 0;
  if (table) {
    t.tok0 = tt_tok(tok, 2 * i);
    t.tok1 = tt_tok(tok, 2 * i + 1 < p.kmask ? 2 * i + 1 : 2 * i);
    return t;
  }
  const int* mrow = p.mask + ((long long)bh * p.n_qblk + pos) * p.kmask;
  const int* tab = p.kv_blk + (long long)bh * p.t_new;
  const int j0 = __ldg(mrow + 2 * i);
  const int j1 = 2 * i + 1 < p.kmask ? __ldg(mrow + 2 * i + 1) : -1;
  t.tok0 = blk_tok0(p, __ldg(tab + j0));
  t.tok1 = j1 >= 0 ? blk_tok0(p, __ldg(tab + j1)) : t.tok0;  // missing half: reload (finite), masked
  return t;
}

template <int D>
__device__ __forceinline__ void taylor_t_body(const CUtensorMap& tm_q, const CUtensorMap& tm_k,
                                              const CUtensorMap& tm_v, const CUtensorMap& tm_kc,
                                              const CUtensorMap& tm_vc, const AttnParams& p, const int item,
                                              const int bh) {
  using L = TaylorTSmem<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem + L::kQOff;
  uint8_t* sKV = smem + L::kKvOff;
  uint8_t* sP = smem + L::kPOff;
  // per-stage query vectors in static shared memory (LDS/STS addressing; the
  // dynamic-smem pointers above go through an integer alignment round trip)
  __shared__ __align__(16) float sM_all[2][64];   // running max per query (log2 domain)
  __shared__ __align__(16) float sA_all[2][64];   // rescale factors of the last slow path
  __shared__ __align__(16) float sI_all[2][64];   // 1 / row sum
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBarOff);
  uint64_t* q_full = bars + 0;                      // [2]
  uint64_t* kv_full = bars + 2;                     // [kTKvStages]
  uint64_t* kv_empty = bars + 2 + kTKvStages;       // [kTKvStages]
  uint64_t* s_full = bars + 2 + 2 * kTKvStages;     // [stage][buffer]: S^T(i) in buffer i&1
  uint64_t* p_full = bars + 6 + 2 * kTKvStages;     // [stage][buffer]: P^T(i) written (S^T buffer read)
  uint64_t* pv_done = bars + 10 + 2 * kTKvStages;   // [stage][buffer]: PV(i) complete (P^T buffer free)
  uint64_t* o_full = bars + 14 + 2 * kTKvStages;    // [stage]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 16 + 2 * kTKvStages);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_ex = (p.kmask + 1) >> 1;
  const int n_kv = n_ex + p.tn_pad / 128;

  if (threadIdx.x == 0) {
    mbar_init(&q_full[0], 1);
    mbar_init(&q_full[1], 1);
    for (int s = 0; s < kTKvStages; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int s = 0; s < 4; ++s) {
      mbar_init(&s_full[s], 1);
      mbar_init(&p_full[s], 4);
      mbar_init(&pv_done[s], 1);
    }
    mbar_init(&o_full[0], 1);
    mbar_init(&o_full[1], 1);
    fence_barrier_init();
  }
  if (warp == 8) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp >= 8) {
    setmaxnreg_dec<kOtherRegs>();
    if (warp == 9) {
      // ------------------------------------------------------------ TMA producer
      const bool leader = elect_one();
      if (leader) {
        tma_prefetch_desc(&tm_q);
        tma_prefetch_desc(&tm_k);
        tma_prefetch_desc(&tm_v);
        tma_prefetch_desc(&tm_kc);
        tma_prefetch_desc(&tm_vc);
      }
      const uint64_t pol_q = policy_evict_first();
      const uint64_t pol_kv = policy_evict_last();
      const int hh = bh % p.H, bb = bh / p.H;
      int pos[2];
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        pos[s] = 2 * item + s;
        if (pos[s] >= p.n_qblk) pos[s] = 2 * item;  // absent stage: a copy of stage 0, never written
      }
      if (leader) {
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          mbar_arrive_expect_tx(&q_full[s], L::kQStage);
          const int tok = blk_tok0(p, p.qlist[(long long)bh * p.n_qblk + pos[s]]);
          for (int pl = 0; pl < 2; ++pl)
            tma_load_4d(sQ + s * L::kQStage + pl * 8192, &tm_q, &q_full[s], pl * 64, tok, hh, bb, pol_q);
        }
      }
      int tokr[2][kTTokRegs];
      const bool table = p.kmask <= 32 * kTTokRegs;
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const int* mrow = p.mask + ((long long)bh * p.n_qblk + pos[s]) * p.kmask;
        const int* tab = p.kv_blk + (long long)bh * p.t_new;
#pragma unroll
        for (int r = 0; r < kTTokRegs; ++r) {
          const int j = 32 * r + lane;
          tokr[s][r] = (table && j < p.kmask) ? blk_tok0(p, __ldg(tab + __ldg(mrow + j))) : 0;
        }
      }
      int c = 0;
      auto push = [&](const TTileSrc& t, int is_v) {
        const int slot = c % kTKvStages;
        const int use = c / kTKvStages;
        if (use > 0) mbar_wait(&kv_empty[slot], (use - 1) & 1);
        __syncwarp();
        if (leader) {
          mbar_arrive_expect_tx(&kv_full[slot], L::kTile);
          uint8_t* dst = sKV + slot * L::kTile;
          const CUtensorMap* tm = t.centroid ? (is_v ? &tm_vc : &tm_kc) : (is_v ? &tm_v : &tm_k);
          const int c2 = t.centroid ? bh : hh, c3 = t.centroid ? 0 : bb;
          for (int half = 0; half < 2; ++half) {
            const int tok = half ? t.tok1 : t.tok0;
            for (int pl = 0; pl < 2; ++pl)
              tma_load_4d(dst + pl * 16384 + half * 8192, tm, &kv_full[slot], pl * 64, tok, c2, c3, pol_kv);
          }
        }
        ++c;
      };
      // ring order = MMA consumption order: K_0, K_1 of both stages, then per
      // step i and stage: V_i, K_{i+2}. Centroid tiles (i >= n_ex) are the
      // same for both stages: loaded once (stage 0's entry) and used by both.
      auto own = [&](int i, int s) { return s == 0 || i < n_ex; };
      for (int i = 0; i < 2 && i < n_kv; ++i)
#pragma unroll
        for (int s = 0; s < 2; ++s)
          if (own(i, s)) push(tt_tile(p, bh, pos[s], i, n_ex, table, tokr[s]), 0);
      for (int i = 0; i < n_kv; ++i) {
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          if (own(i, s)) push(tt_tile(p, bh, pos[s], i, n_ex, table, tokr[s]), 1);
          if (i + 2 < n_kv && own(i + 2, s)) push(tt_tile(p, bh, pos[s], i + 2, n_ex, table, tokr[s]), 0);
        }
      }
    } else if (warp == 8) {
      // ------------------------------------------------------------ MMA issuer
      constexpr uint32_t idesc_s = idesc_bf16_f32(128, 64, 0, 0);  // S^T = K . Q^T   (K-major both)
      constexpr uint32_t idesc_o = idesc_bf16_f32(128, 64, 1, 1);  // O^T = V^T . P^T (MN-major both)
      const bool leader = elect_one();
      const uint64_t dq_base = sdesc_sw128_base(smem_u32(sQ), 16, 1024);
      const uint64_t dk_base = sdesc_sw128_base(smem_u32(sKV), 16, 1024);
      const uint64_t dv_base = sdesc_sw128_base(smem_u32(sKV), 16384, 1024);
      const uint64_t dp_base = sdesc_sw128_base(smem_u32(sP), 16, 1024);
      auto issue_s = [&](int s, int b, int slot) {
        if (leader) {
          const uint64_t da = dk_base + static_cast<uint64_t>((slot * L::kTile) >> 4);
          const uint64_t db = dq_base + static_cast<uint64_t>((s * L::kQStage) >> 4);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint64_t oa = ((kk >> 2) * 16384 + (kk & 3) * 32) >> 4;
            const uint64_t ob = ((kk >> 2) * 8192 + (kk & 3) * 32) >> 4;
            mma_ss(tmem + s * 128 + b * 64, da + oa, db + ob, idesc_s, kk > 0);
          }
        }
        __syncwarp();
      };
      auto issue_o = [&](int s, int b, int slot, uint32_t acc) {
        if (leader) {
          const uint64_t da = dv_base + static_cast<uint64_t>((slot * L::kTile) >> 4);
          const uint64_t db = dp_base + static_cast<uint64_t>((s * L::kPT) >> 4);
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const uint64_t o = (kk * 2048) >> 4;
            mma_ss(tmem + 256 + s * 64, da + o, db + o, idesc_o, (acc | kk) != 0);
          }
        }
        __syncwarp();
      };
      auto commit = [&](uint64_t* bar) {
        if (leader) mma_commit(bar);
        __syncwarp();
      };
      int e = 0;  // next ring entry
      auto take = [&]() {
        const int slot = e % kTKvStages;
        mbar_wait(&kv_full[slot], (e / kTKvStages) & 1);
        __syncwarp();
        tc_fence_after();
        ++e;
        return slot;
      };
      auto release = [&](int slot) { commit(&kv_empty[slot]); };
      // a centroid tile's slot is taken by stage 0, reused by stage 1, then released
      int held_k = 0, held_v = 0;
      auto get = [&](int i, int s, int& held) { return (s == 1 && i >= n_ex) ? held : take(); };
      auto put = [&](int i, int s, int slot, int& held) {
        if (s == 0 && i >= n_ex)
          held = slot;
        else
          release(slot);
      };
      mbar_wait(&q_full[0], 0);
      mbar_wait(&q_full[1], 0);
      for (int i = 0; i < 2 && i < n_kv; ++i)
        for (int s = 0; s < 2; ++s) {
          const int slot = get(i, s, held_k);
          issue_s(s, i, slot);
          commit(&s_full[2 * s + i]);
          put(i, s, slot, held_k);
        }
      for (int i = 0; i < n_kv; ++i) {
        const int b = i & 1;
        for (int s = 0; s < 2; ++s) {
          mbar_wait(&p_full[2 * s + b], (i >> 1) & 1);  // P^T(i) written, S^T buffer b read
          if (leader) ISA_TSTAMP(i + 1, s, 6);
          __syncwarp();
          tc_fence_after();
          const int vs = get(i, s, held_v);
          if (leader) ISA_TSTAMP(i + 1, s, 5);
          issue_o(s, b, vs, i > 0);
          commit(&pv_done[2 * s + b]);
          if (i + 1 == n_kv) commit(&o_full[s]);
          put(i, s, vs, held_v);
          if (i + 2 < n_kv) {
            const int ks = get(i + 2, s, held_k);
            issue_s(s, b, ks);
            commit(&s_full[2 * s + b]);
            put(i + 2, s, ks, held_k);
            if (leader) ISA_TSTAMP(i + 1, s, 7);
          }
        }
      }
    }
    __syncwarp();
  } else {
    // -------------------------------------------------------------- softmax
    setmaxnreg_inc<kSoftmaxRegs>();
    const int s = warp >> 2, wq = warp & 3;
    const int r = wq * 32 + lane;  // TMEM lane: key row of S^T, head-dim row of O^T
    const uint32_t lane_base = static_cast<uint32_t>(wq * 32) << 16;
    const uint32_t t_s0 = tmem + lane_base + s * 128;  // S^T buffers at +0 / +64
    const uint32_t t_o = tmem + lane_base + 256 + s * 64;
    const uint32_t bar_id = 1 + s;
    float* sM = sM_all[s];
    float* sA = sA_all[s];
    float* sI = sI_all[s];
    uint8_t* sPs = sP + s * L::kPT;
    const float sl2 = p.scale_log2;
    const int pos = 2 * item + s;
    const bool present = pos < p.n_qblk;
    const int posr = present ? pos : 2 * item;
    const int u = present ? p.qlist[(long long)bh * p.n_qblk + pos] : -1;
    const uint32_t* mbits = p.member_bits + ((long long)bh * p.n_qblk + posr) * p.W;
    const int* mrow = p.mask + ((long long)bh * p.n_qblk + posr) * p.kmask;
    // K_new blocks with fewer than 64 rows: the last source block, the selected short context block
    const int jsrc = (p.l_src & 63) ? p.t_src - 1 : -1;
    const int jctx = (p.l_ctx & 63) ? p.ctx_short_j[bh] : -1;
    auto kn_valid = [&](int j) -> int {
      if (j < 0 || j >= p.t_new) return 0;
      if (j == jsrc) return p.l_src & 63;
      if (j == jctx) return p.l_ctx & 63;
      return 64;
    };
    if (r < 64) sM[r] = -INFINITY;
    named_bar_sync(bar_id, 128);
    float2 lp[32];  // row-sum partials of this key lane, query pairs
#pragma unroll
    for (int q = 0; q < 32; ++q) lp[q] = make_float2(0.f, 0.f);
    for (int i = 0; i < n_kv; ++i) {
      // per-key bias (log2 domain): 0 / log2(w) for live keys, -inf for padded or excluded ones
      float bias;
      if (i < n_ex) {
        const int j = (r < 64) ? __ldg(mrow + 2 * i) : (2 * i + 1 < p.kmask ? __ldg(mrow + 2 * i + 1) : -1);
        bias = (r & 63) < kn_valid(j) ? 0.f : -INFINITY;
      } else {
        const int j = (i - n_ex) * 128 + r;
        const bool excl = j >= p.t_new || ((__ldg(mbits + (j >> 5)) >> (j & 31)) & 1u);
        const int w = excl ? 0 : kn_valid(j);
        bias = w == 64 ? 6.f : (w > 0 ? __log2f(static_cast<float>(w)) : -INFINITY);
      }
      const int b = i & 1;
      const uint32_t t_s = t_s0 + b * 64;
      float* sRed = reinterpret_cast<float*>(sPs);  // slow-path scratch, before this tile's P^T
      mbar_wait(&s_full[2 * s + b], (i >> 1) & 1);
      tc_fence_after();
      if (wq == 0 && lane == 0) ISA_TSTAMP(i, s, 0);
      // the P^T buffer is free once PV(i-1) completed
      if (i >= 1) mbar_wait(&pv_done[2 * s + (b ^ 1)], ((i - 1) >> 1) & 1);
      float t[64];
      // t <- scaled score + key bias (- running max per query when kSub)
      auto load_t = [&](auto sub_tag) {
        constexpr bool kSub = decltype(sub_tag)::value;
        const float2 sl2x2 = make_float2(sl2, sl2), b2 = make_float2(bias, bias);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          uint32_t a[32];
          tmem_ld32(t_s + 32 * h, a);
          tmem_ld_wait();
#pragma unroll
          for (int q = 0; q < 32; q += 4) {
            float2 u0 = ffma2(make_float2(__uint_as_float(a[q]), __uint_as_float(a[q + 1])), sl2x2, b2);
            float2 u1 = ffma2(make_float2(__uint_as_float(a[q + 2]), __uint_as_float(a[q + 3])), sl2x2, b2);
            if (kSub) {
              const float4 m4 = *reinterpret_cast<const float4*>(sM + 32 * h + q);
              u0 = fsub2(u0, make_float2(m4.x, m4.y));
              u1 = fsub2(u1, make_float2(m4.z, m4.w));
            }
            t[32 * h + q] = u0.x;
            t[32 * h + q + 1] = u0.y;
            t[32 * h + q + 2] = u1.x;
            t[32 * h + q + 3] = u1.y;
          }
        }
      };
      load_t(std::true_type{});
      if (wq == 0 && lane == 0) ISA_TSTAMP(i, s, 1);
      // speculative check: any live key above m + 8 (m = -inf on the first
      // tile gives +inf and forces the slow path; masked keys carry -inf)
      float tmax = -INFINITY;
#pragma unroll
      for (int q = 0; q < 64; q += 2) tmax = fmax3(tmax, t[q], t[q + 1]);
      if (named_bar_red_or(bar_id, 128, !(tmax <= 8.f) && bias > -INFINITY)) {
        load_t(std::false_type{});  // raw scaled scores
        warp_halve64<true>(t, lane);
        sRed[wq * 64 + 2 * lane] = t[0];
        sRed[wq * 64 + 2 * lane + 1] = t[1];
        named_bar_sync(bar_id, 128);
        if (r < 64) {
          const float mo = sM[r];
          const float mt = fmaxf(fmaxf(sRed[r], sRed[64 + r]), fmaxf(sRed[128 + r], sRed[192 + r]));
          float mn = fmaxf(mo, mt);
          if (mo > -INFINITY && mn <= mo + 8.f) mn = mo;  // lazy: keep the old max within 2^8
          sA[r] = mo == mn ? 1.f : (mo == -INFINITY ? 0.f : ex2_approx(mo - mn));
          sM[r] = mn;
        }
        named_bar_sync(bar_id, 128);
        bool any = false;
#pragma unroll
        for (int q = 0; q < 64; q += 4) {
          const float4 a4 = *reinterpret_cast<const float4*>(sA + q);
          lp[q >> 1].x *= a4.x;
          lp[q >> 1].y *= a4.y;
          lp[(q >> 1) + 1].x *= a4.z;
          lp[(q >> 1) + 1].y *= a4.w;
          any |= (a4.x != 1.f) | (a4.y != 1.f) | (a4.z != 1.f) | (a4.w != 1.f);
        }
        if (i > 0 && any) {  // O^T columns (queries) * alpha (PV(i-1) completed above)
          tc_fence_after();
#pragma unroll 1
          for (int h = 0; h < 2; ++h) {
            uint32_t o[32];
            tmem_ld32(t_o + 32 * h, o);
            tmem_ld_wait();
#pragma unroll
            for (int q = 0; q < 32; ++q) o[q] = __float_as_uint(__uint_as_float(o[q]) * sA[32 * h + q]);
            tmem_st32(t_o + 32 * h, o);
          }
          tmem_st_wait();
        }
        load_t(std::true_type{});
      }
      if (wq == 0 && lane == 0) ISA_TSTAMP(i, s, 2);
      // P = exp2(t) (1 in kEmuEvery pairs on the FMA pipe), row-sum partials, P^T row -> smem
      uint32_t pk[32];
#pragma unroll
      for (int q = 0; q < 64; q += 2) {
        const float2 tt = make_float2(t[q], t[q + 1]);
        float2 pp;
        if (kTTEmu > 0 && ((q >> 1) % kTTEmu) == kTTEmu - 1) {
          pp = ex2_emu2(tt);
          if (bias == -INFINITY) pp = make_float2(0.f, 0.f);
        } else {
          pp.x = ex2_approx(tt.x);
          pp.y = ex2_approx(tt.y);
        }
        lp[q >> 1] = fadd2(lp[q >> 1], pp);
        pk[q >> 1] = pack_bf16x2(pp.x, pp.y);
      }
      {
        uint8_t* rowp = sPs + r * 128;
#pragma unroll
        for (int ch = 0; ch < 8; ++ch)
          *reinterpret_cast<uint4*>(rowp + ((ch ^ (r & 7)) << 4)) =
              make_uint4(pk[4 * ch], pk[4 * ch + 1], pk[4 * ch + 2], pk[4 * ch + 3]);
      }
      if (wq == 0 && lane == 0) ISA_TSTAMP(i, s, 3);
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[2 * s + b]);
      if (wq == 0 && lane == 0) ISA_TSTAMP(i, s, 4);
    }
    // -------------------------------------------------------------- epilogue
    mbar_wait(&o_full[s], 0);  // every PV of this stage complete: both P^T buffers are free
    __syncwarp();
    tc_fence_after();
    // the P^T buffer is reused as scratch: order every warp's last P^T row
    // stores before any warp's scratch stores (the o_full chain runs through
    // the async proxy, which racecheck does not see)
    named_bar_sync(bar_id, 128);
    float* sRed = reinterpret_cast<float*>(sPs);
    {
      float v[64];
#pragma unroll
      for (int q = 0; q < 32; ++q) {
        v[2 * q] = lp[q].x;
        v[2 * q + 1] = lp[q].y;
      }
      warp_halve64<false>(v, lane);
      sRed[wq * 64 + 2 * lane] = v[0];
      sRed[wq * 64 + 2 * lane + 1] = v[1];
    }
    named_bar_sync(bar_id, 128);
    const int vq = present ? blk_valid(p, u) : 0;
    const int tok = present ? blk_tok0(p, u) : 0;
    if (r < 64) {
      const float l = (sRed[r] + sRed[64 + r]) + (sRed[128 + r] + sRed[192 + r]);
      sI[r] = l > 0.f ? 1.f / l : 0.f;
      if (r < vq) {
        if (!(l > 0.f) && p.err_flag) atomicOr(p.err_flag, 2);
        if (p.lse) p.lse[(long long)bh * p.S + tok + r] = l > 0.f ? sM[r] + log2f(l) : -INFINITY;
      }
    }
    named_bar_sync(bar_id, 128);
    // O^T (lane = d, column = query) -> out: transposed through the stage's
    // (now idle) P^T buffer so the global stores are 16-byte row chunks
    const float res = (p.resid && present) ? p.gamma * __ldg(p.resid + ((long long)bh * p.T + u) * D + r) : 0.f;
    const int hh = bh % p.H, bb = bh / p.H;
    if (p.out_fp32) {
      const long long obase = bb * p.o_sb + hh * p.o_sh + (long long)tok * p.o_ss + r;
#pragma unroll 1
      for (int h = 0; h < 2; ++h) {
        uint32_t o[32];
        tmem_ld32(t_o + 32 * h, o);
        tmem_ld_wait();
#pragma unroll
        for (int qq = 0; qq < 32; ++qq) {
          const int q = 32 * h + qq;
          if (q < vq)
            reinterpret_cast<float*>(p.out)[obase + (long long)q * p.o_ss] =
                fmaf(__uint_as_float(o[qq]), sI[q], res);
        }
      }
    } else {
      __nv_bfloat16* stage_buf = reinterpret_cast<__nv_bfloat16*>(sPs);  // [64 q][128 d] bf16 = 16 KB
#pragma unroll 1
      for (int h = 0; h < 2; ++h) {
        uint32_t o[32];
        tmem_ld32(t_o + 32 * h, o);
        tmem_ld_wait();
#pragma unroll
        for (int qq = 0; qq < 32; ++qq) {
          const int q = 32 * h + qq;
          stage_buf[q * 128 + r] = __float2bfloat16_rn(fmaf(__uint_as_float(o[qq]), sI[q], res));
        }
      }
      named_bar_sync(bar_id, 128);
      // 64 rows x 256 B: 1024 16-byte chunks, 8 per thread
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const int idx = c * 128 + r;
        const int q = idx >> 4, ch = idx & 15;
        if (q < vq) {
          const uint4 w = *reinterpret_cast<const uint4*>(stage_buf + q * 128 + ch * 8);
          *reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(p.out) + bb * p.o_sb + hh * p.o_sh +
                                    (long long)(tok + q) * p.o_ss + ch * 8) = w;
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

template <int D>
__global__ void __launch_bounds__(kTThreads, 1)
    gba_taylor_t_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                        const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_kc,
                        const __grid_constant__ CUtensorMap tm_vc, const AttnParams p) {
  taylor_t_body<D>(tm_q, tm_k, tm_v, tm_kc, tm_vc, p, blockIdx.x, blockIdx.y);
}

// Per head: row-major K7 (pair-of-blocks union tiles, one K/V load serves
// both blocks of a pair, but every union tile costs a full 128x128 MMA pair)
// or K7T (each block's own tiles, no MMA waste, no load sharing). Operand
// traffic decides (both kernels are bound by it): K7 streams 2 * n_tiles
// tiles per 4-block item, K7T ceil(k/2) per block. K7 is taken when its tile
// count is below 0.9 x K7T's (tuned on cfg3: iid inputs keep K7T, clustered
// inputs match a forced K7). mode >= 0 forces the choice.
__global__ void taylor_pick_kernel(const int* __restrict__ n_tiles, int n_items, int n_flat, int k, int mode,
                                   int* __restrict__ pick) {
  const int bh = blockIdx.x;
  long long sum = 0;
  for (int i = threadIdx.x; i < n_items; i += blockDim.x) sum += n_tiles[(long long)bh * n_items + i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  __shared__ long long part[4];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = sum;
  __syncthreads();
  if (threadIdx.x == 0) {
    const long long k7 = 2 * (part[0] + part[1] + part[2] + part[3]);
    const long long k7t = (long long)n_flat * ((k + 1) / 2);
    pick[bh] = mode >= 0 ? mode : (10 * k7 < 9 * k7t ? 0 : 1);
  }
}

template <int D>
__global__ void __launch_bounds__(kTThreads, 1)
    gba_isa_hybrid_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                          const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_kc,
                          const __grid_constant__ CUtensorMap tm_vc, const AttnParams pe, const AttnParams pt,
                          const int n_exact, const int n_k7, const int* __restrict__ pick) {
  const int x = blockIdx.x, bh = blockIdx.y;
  if (x < n_exact) {
    gba_body<D, MODE_EXACT>(tm_q, tm_k, tm_v, tm_kc, tm_vc, pe, x, bh);
  } else if (x < n_exact + n_k7) {
    if (__ldg(pick + bh) == 0) gba_body<D, MODE_TAYLOR>(tm_q, tm_k, tm_v, tm_kc, tm_vc, pt, x - n_exact, bh);
  } else {
    if (__ldg(pick + bh) == 1) taylor_t_body<D>(tm_q, tm_k, tm_v, tm_kc, tm_vc, pt, x - n_exact - n_k7, bh);
  }
  if (pe.head_done) {  // head bh's output rows of this CTA are final: publish (release) for the comm stream
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) atomicAdd(pe.head_done + bh, 1);
  }
}

}  // namespace isa
