// Gathered-block attention on sm_100a (tcgen05 + TMEM + TMA, warp-specialised).
//
// One kernel body serves three hot-path branches of the ISA forward:
//   MODE_DENSE  (K8)  dense non-causal attention, identity block tables.
//                     Reference: full_attention (reference.py:79-123).
//   MODE_EXACT  (K6)  the sharp query blocks over K_new = source blocks + the
//                     selected context blocks, addressed through the per-head
//                     block table (no K_new / gathered-Q materialisation).
//                     Reference: gather_blocks + online_softmax_attention +
//                     OnlineState (pipeline.py:338-343, reference.py:126-170).
//   MODE_TAYLOR (K7)  the flat query blocks: online softmax over their exact
//                     K_new blocks (union stream of the CTA's 4 query blocks,
//                     per-(row-block, key-block) visibility bits) followed by
//                     all K_new centroids with additive log2(valid_rows)
//                     weights and -inf for the row block's own exact members.
//                     Reference: taylor_sparse_forward/_head_state
//                     (taylor.py:124-194), semantics SPEC.md:304.
// The stage-5 scatter (pipeline.py:350-357) is fused: each output row is
// written straight to its original token position.
//
// CTA = 4 query blocks of 64 rows = two 128-row Q tiles ("stages") sharing one
// K/V tile stream (128 keys per tile = two 64-row key blocks).
// Warp roles (384 threads):
//   warps 0-3   softmax / rescale / epilogue for Q tile 0 (TMEM lanes 0-127)
//   warps 4-7   same for Q tile 1
//   warp  8     TMEM allocator + single-thread tcgen05.mma issuer
//   warp  9     TMA producer (Q once, then the K/V ring)
// TMEM (512 columns): S0 [0,128) S1 [128,256) O0 [256,384) O1 [384,512);
// P_s (bf16 pairs) overwrites the upper 64 columns of S_s.
#pragma once
#include <type_traits>

#include "isa_ptx.cuh"

namespace isa {

enum AttnMode : int { MODE_DENSE = 0, MODE_EXACT = 1, MODE_TAYLOR = 2 };

struct AttnParams {
  int H;           // heads; bh = b*H + h
  int l_src, l_ctx;
  int t_src, t_ctx;
  int t_new;       // K_new blocks (T for DENSE)
  int n_qblk;      // query blocks per head in the list (n_sharp / n_flat / T)
  float scale_log2;
  const int* qlist;    // [BH][n_qblk] original query block ids (EXACT/TAYLOR)
  const int* kv_blk;   // [BH][t_new] original block id of K_new block j (EXACT/TAYLOR)
  // TAYLOR only
  const int4* tiles;   // [BH][n_items][max_tiles] {kn0, kn1, bits0, bits1}
  const int* n_tiles;  // [BH][n_items] exact tiles per item
  int n_items;
  int max_tiles;
  const uint32_t* member_bits;  // [BH][n_qblk][W]
  int W;
  const int* ctx_short_j;  // [BH]: K_new index of the selected short context block or -1
  int tn_pad;              // centroid rows, multiple of 128
  // output (token-major, D contiguous)
  void* out;
  int out_fp32;
  long long o_sb, o_sh, o_ss;
  int* err_flag;
  // gamma coarse residual (pipeline.py:354-356): out += gamma * resid[bh][u]
  const float* resid;  // [BH][T][D] or null
  float gamma;
  int T;
  // backward support: per-row log2-domain normaliser m + log2(l) of the
  // (surrogate) softmax, [BH][S] by original token row, or null
  float* lse;
  int S;
  // transposed Taylor kernel (isa_taylor_t.cuh): exact K_new lists [BH][n_qblk][kmask]
  const int* mask;
  int kmask;
  // per-head completion counters [BH] (multi-GPU overlap, isa_forward_signal):
  // every CTA of the hybrid grid adds 1 to its head's counter after its
  // output stores are visible device-wide; null = off
  int* head_done;
};

#ifndef ISA_TRACE_Q
#define ISA_TRACE_Q 0  // softmax warp quadrant stamped by ISA_TRACE builds
#endif
#ifndef ISA_TRACE_MODE
#define ISA_TRACE_MODE 0  // 2: stamp the Taylor branch instead of dense/exact
#endif
constexpr int kThreads = 384;
constexpr int kKvStages = 5;  // K/V ring slots (D=128: 64 KB Q + 5 x 32 KB = 224 KB)
constexpr int kSoftmaxRegs = 208;
constexpr int kOtherRegs = 88;
// setmaxnreg moves registers inside the CTA's pool only: the two softmax
// warpgroups may grow by no more than the third warpgroup shrinks from the
// launch allocation (65536 / 384 -> 168 per thread). Violating this starves
// a softmax warp in USETMAXREG.TRY_ALLOC forever (observed on B200).
constexpr int kLaunchRegs = 168;
static_assert(2 * (kSoftmaxRegs - kLaunchRegs) <= (kLaunchRegs - kOtherRegs), "register pool overcommitted");
constexpr int kLdCols = 16;   // tcgen05.ld width (columns) for the S row
#ifndef ISA_EMU_EVERY
#define ISA_EMU_EVERY 4
#endif
constexpr int kEmuEvery = ISA_EMU_EVERY;  // 1 in kEmuEvery exp2 pairs of the plain softmax path on the FMA pipe

template <int D>
struct AttnSmem {
  static constexpr int kPlanes = D / 64;
  static constexpr int kTileBytes = 128 * D * 2;  // one 128-row bf16 tile
  static constexpr int kQOff = 0;
  static constexpr int kKvOff = 2 * kTileBytes;
  static constexpr int kBarOff = kKvOff + kKvStages * kTileBytes;
  static constexpr int kBytes = kBarOff + 256;
  static constexpr int kAlloc = kBytes + 1024;  // slack for 1024-B alignment
};

__device__ __forceinline__ int blk_tok0(const AttnParams& p, int u) {
  return u < p.t_src ? u * 64 : p.l_src + (u - p.t_src) * 64;
}
__device__ __forceinline__ int blk_valid(const AttnParams& p, int u) {
  int r = u < p.t_src ? p.l_src - u * 64 : p.l_ctx - (u - p.t_src) * 64;
  return r < 64 ? r : 64;
}

struct TileInfo {
  int tok0, tok1;    // source rows (token index, or centroid row for centroid tiles)
  int valid0, valid1;  // valid key rows in each 64-row half (0 = missing)
  int bits0, bits1;    // TAYLOR: visibility bit per query block for each half
  int centroid;        // 1 = centroid tile, index in [0, tn_pad/128)
  int cidx;
};

template <int MODE>
__device__ __forceinline__ int num_kv_tiles(const AttnParams& p, int bh, int item) {
  if (MODE == MODE_TAYLOR) return p.n_tiles[bh * p.n_items + item] + p.tn_pad / 128;
  return (p.t_new + 1) >> 1;
}

// Source rows of K/V tile i of the stream that Q tile `s` consumes, for the
// TMA producer. DENSE/EXACT: one stream shared by both Q tiles (K_new blocks
// 2i, 2i+1, through the block table). TAYLOR: each Q tile (pair of flat query
// blocks) has its own exact-union stream of planned entries (token rows
// resolved by taylor_plan_kernel), padded to a common length with empty tiles,
// followed by the shared centroid tiles. The raw table words are loaded one
// tile ahead of use (tile_raw), so no dependent global load sits between two
// TMA issues.
struct TileSrc {
  int tok0, tok1;  // first token row per 64-row half (or centroid row); a missing half repeats tok0
  int centroid;
};

template <int MODE>
__device__ __forceinline__ int4 tile_raw(const AttnParams& p, int bh, int item, int i, int s, int ne) {
  if (MODE == MODE_TAYLOR) {
    if (i < ne) return __ldg(p.tiles + (((long long)bh * p.n_items + item) * 2 + s) * p.max_tiles + i);
    return make_int4(0, 0, 0, 0);
  }
  if (MODE == MODE_EXACT) {
    const int* tab = p.kv_blk + (long long)bh * p.t_new;
    const int kn0 = 2 * i, kn1 = 2 * i + 1;
    return make_int4(kn0 < p.t_new ? __ldg(tab + kn0) : 0, kn1 < p.t_new ? __ldg(tab + kn1) : -1, 0, 0);
  }
  return make_int4(2 * i, 2 * i + 1 < p.t_new ? 2 * i + 1 : -1, 0, 0);
}

template <int MODE>
__device__ __forceinline__ TileSrc tile_src(const AttnParams& p, int4 raw, int i, int ne) {
  TileSrc t;
  t.centroid = 0;
  if (MODE == MODE_TAYLOR) {
    if (i >= ne) {
      t.centroid = 1;
      t.tok0 = (i - ne) * 128;
      t.tok1 = t.tok0 + 64;
      return t;
    }
    t.tok0 = raw.x >= 0 ? raw.x : 0;  // empty padding tile: load rows 0.., fully masked
    t.tok1 = raw.y >= 0 ? raw.y : t.tok0;
    return t;
  }
  t.tok0 = blk_tok0(p, raw.x);
  t.tok1 = raw.y >= 0 ? blk_tok0(p, raw.y) : t.tok0;  // missing half: reload (finite), masked
  return t;
}

// Ring entry e in consumption order -> (tile, stage, is_v).
// Shared stream: K_0 | V_0 K_1 | V_1 K_2 | ... | V_{n-1}.
// Per-stage (TAYLOR): K0_0 K1_0 | V0_0 K0_1 V1_0 K1_1 | ... | V0_{n-1} V1_{n-1}.
struct Entry {
  int tile, stage, is_v;
};
template <int MODE>
__device__ __forceinline__ Entry ring_entry(int e, int n) {
  Entry r;
  if (MODE == MODE_TAYLOR) {
    if (e < 2) {
      r.tile = 0; r.stage = e; r.is_v = 0;
    } else if (e >= 4 * n - 2) {
      r.tile = n - 1; r.stage = e - (4 * n - 2); r.is_v = 1;
    } else {
      const int q = e - 2, step = q / 4 + 1, w = q % 4;
      r.stage = w >> 1;
      r.is_v = (w & 1) == 0;
      r.tile = r.is_v ? step - 1 : step;
    }
  } else {
    r.stage = 0;
    if (e == 0) {
      r.tile = 0; r.is_v = 0;
    } else {
      r.is_v = (e & 1);
      r.tile = r.is_v ? (e - 1) / 2 : e / 2;
    }
  }
  return r;
}

template <int MODE>
__device__ __forceinline__ int query_block(const AttnParams& p, int bh, int item, int q) {
  const int pos = item * 4 + q;
  if (pos >= p.n_qblk) return -1;
  if (MODE == MODE_DENSE) return pos;
  return p.qlist[(long long)bh * p.n_qblk + pos];
}

template <int D, int MODE, bool kPair = false>
__device__ __forceinline__ void gba_body(const CUtensorMap& tm_q, const CUtensorMap& tm_k, const CUtensorMap& tm_v,
                                         const CUtensorMap& tm_kc, const CUtensorMap& tm_vc, const AttnParams& p,
                                         const int item, const int bh) {
  using L = AttnSmem<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem + L::kQOff;
  uint8_t* sKV = smem + L::kKvOff;
  // kPair (cta_group::2, K6/K8 at D = 128): every K/V ring entry is a half
  // tile in each CTA of the pair (K: one 64-key block; V: one 64-column d
  // plane of both blocks), so the same ring bytes hold twice the slots.
  static_assert(!kPair || (MODE != MODE_TAYLOR && D == 128), "CTA pairs run the exact/dense branch at D = 128");
  constexpr int kSlots = kPair ? 2 * kKvStages : kKvStages;
  constexpr int kSlotBytes = kPair ? L::kTileBytes / 2 : L::kTileBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBarOff);
  uint64_t* q_full = bars + 0;           // [2]
  uint64_t* kv_full = bars + 2;          // [kSlots]
  uint64_t* kv_empty = bars + 2 + kSlots;  // [kSlots]
  uint64_t* s_full = bars + 2 + 2 * kSlots;     // [2]
  uint64_t* p_full = bars + 4 + 2 * kSlots;     // [2]
  uint64_t* o_full = bars + 6 + 2 * kSlots;     // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 8 + 2 * kSlots);
  static_assert((8 + 2 * kSlots) * 8 + 4 <= 256, "barrier area");
  const uint32_t rank = kPair ? cluster_ctarank() : 0u;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int n_kv = num_kv_tiles<MODE>(p, bh, item);

  if (threadIdx.x == 0) {
    mbar_init(&q_full[0], 1);
    mbar_init(&q_full[1], 1);
    for (int s = 0; s < kSlots; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&s_full[s], 1);
      mbar_init(&p_full[s], kPair ? 8 : 4);  // pair: the leader's copy counts both CTAs' softmax warps
      mbar_init(&o_full[s], 1);
    }
    fence_barrier_init();
  }
  if (warp == 8) {
    if constexpr (kPair)
      tmem_alloc2<512>(tmem_slot);
    else
      tmem_alloc<512>(tmem_slot);
  }
  tc_fence_before();
  if constexpr (kPair)
    cluster_sync_all();  // both CTAs' barriers initialised before any cross-CTA signal
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp >= 8) {
    setmaxnreg_dec<kOtherRegs>();
    if (warp == 9) {
      // ------------------------------------------------------------ TMA producer
      // The whole warp walks the schedule (uniform values); one lane issues.
      const bool leader = elect_one();
      if (leader) {
        tma_prefetch_desc(&tm_q);
        tma_prefetch_desc(&tm_k);
        tma_prefetch_desc(&tm_v);
        if (MODE == MODE_TAYLOR) {
          tma_prefetch_desc(&tm_kc);
          tma_prefetch_desc(&tm_vc);
        }
      }
      const uint64_t pol_q = policy_evict_first();
      const uint64_t pol_kv = policy_evict_last();
      const int hh = bh % p.H, bb = bh / p.H;
      int first_u = query_block<MODE>(p, bh, item, 0);
      if (first_u < 0) first_u = query_block<MODE>(p, bh, 0, 0);  // pair padding CTA: load any valid rows
      if (leader) {
        for (int s = 0; s < 2; ++s) {
          if (!kPair || rank == 0) mbar_arrive_expect_tx(&q_full[s], kPair ? 2 * L::kTileBytes : L::kTileBytes);
          for (int half = 0; half < 2; ++half) {
            int u = query_block<MODE>(p, bh, item, 2 * s + half);
            if (u < 0) u = first_u;
            const int tok = blk_tok0(p, u);
            for (int pl = 0; pl < L::kPlanes; ++pl) {
              uint8_t* dst = sQ + s * L::kTileBytes + pl * 16384 + half * 8192;
              if constexpr (kPair)
                tma_load_4d_pair(dst, &tm_q, &q_full[s], pl * 64, tok, hh, bb, pol_q);
              else
                tma_load_4d(dst, &tm_q, &q_full[s], pl * 64, tok, hh, bb, pol_q);
            }
          }
        }
      }
      // Entries in ring order (see ring_entry): per step i the V tiles of
      // step i-1 and the K tiles of step i; tile descriptors one step ahead.
      const int ne = (MODE == MODE_TAYLOR) ? p.n_tiles[bh * p.n_items + item] : 0;
      constexpr int kStages = (MODE == MODE_TAYLOR) ? 2 : 1;
      int c = 0;
      auto push = [&](const TileSrc& t, int is_v) {
        const int slot = c % kSlots;
        const int use = c / kSlots;
        if (use > 0) mbar_wait(&kv_empty[slot], (use - 1) & 1);
        __syncwarp();
        if (leader) {
          uint8_t* dst = sKV + slot * kSlotBytes;
          const CUtensorMap* tm;
          int c2, c3;
          if (t.centroid) {
            tm = is_v ? &tm_vc : &tm_kc;
            c2 = bh;
            c3 = 0;
          } else {
            tm = is_v ? &tm_v : &tm_k;
            c2 = hh;
            c3 = bb;
          }
          if constexpr (kPair) {
            // K: this CTA's 64-key block, both d planes ([plane][64 keys][64 d]);
            // V: this CTA's d plane of both blocks ([128 keys][64 d])
            if (rank == 0) mbar_arrive_expect_tx(&kv_full[slot], 2 * kSlotBytes);
            if (!is_v) {
              const int tok = rank ? t.tok1 : t.tok0;
              for (int pl = 0; pl < L::kPlanes; ++pl)
                tma_load_4d_pair(dst + pl * 8192, tm, &kv_full[slot], pl * 64, tok, c2, c3, pol_kv);
            } else {
              for (int half = 0; half < 2; ++half)
                tma_load_4d_pair(dst + half * 8192, tm, &kv_full[slot], static_cast<int>(rank) * 64,
                                 half ? t.tok1 : t.tok0, c2, c3, pol_kv);
            }
          } else {
            mbar_arrive_expect_tx(&kv_full[slot], L::kTileBytes);
            for (int half = 0; half < 2; ++half) {
              const int tok = half ? t.tok1 : t.tok0;
              for (int pl = 0; pl < L::kPlanes; ++pl)
                tma_load_4d(dst + pl * 16384 + half * 8192, tm, &kv_full[slot], pl * 64, tok, c2, c3, pol_kv);
            }
          }
          progress(0, c + 1);
        }
        ++c;
      };
      int4 raw[kStages];
#pragma unroll
      for (int st = 0; st < kStages; ++st) raw[st] = tile_raw<MODE>(p, bh, item, 0, st, ne);
      TileSrc cur[kStages], prv[kStages];
#pragma unroll
      for (int st = 0; st < kStages; ++st) cur[st] = prv[st] = TileSrc{0, 0, 0};
      for (int i = 0; i <= n_kv; ++i) {
        if (i < n_kv) {
#pragma unroll
          for (int st = 0; st < kStages; ++st) {
            prv[st] = cur[st];
#ifdef ISA_PRODUCER_NOPREFETCH
            raw[st] = tile_raw<MODE>(p, bh, item, i, st, ne);
#endif
            cur[st] = tile_src<MODE>(p, raw[st], i, ne);
#ifndef ISA_PRODUCER_NOPREFETCH
            if (i + 1 < n_kv) raw[st] = tile_raw<MODE>(p, bh, item, i + 1, st, ne);
#endif
          }
        }
#pragma unroll
        for (int st = 0; st < kStages; ++st) {
          if (i == n_kv) {
            push(cur[st], 1);  // last V
          } else {
            if (i > 0) push(prv[st], 1);
            push(cur[st], 0);
          }
        }
      }
      if constexpr (kPair) {  // drain: the leader's multicast releases of our slots have all landed
        for (int e = c > kSlots ? c - kSlots : 0; e < c; ++e) mbar_wait(&kv_empty[e % kSlots], (e / kSlots) & 1);
      }
    } else if (warp == 8 && (!kPair || rank == 0)) {
      // ------------------------------------------------------------ MMA issuer
      // Whole warp waits; one elected lane issues tcgen05.mma / commit.
      constexpr uint32_t idesc_qk = idesc_bf16_f32(kPair ? 256 : 128, 128, 0, 0);
      constexpr uint32_t idesc_pv = idesc_bf16_f32(kPair ? 256 : 128, D, 0, 1);
      const uint32_t sq = smem_u32(sQ);
      const uint32_t skv = smem_u32(sKV);
      const bool leader = elect_one();
      // Shared-memory descriptors: one base per operand tile, per-k steps are
      // constant 64-bit adds (keeps the issuing warp's instruction count low;
      // it shares an SM sub-partition with two softmax warps).
      const uint64_t dq_base = sdesc_sw128_base(sq, 16, 1024);
      const uint64_t dk_base = sdesc_sw128_base(skv, 16, 1024);
      const uint64_t dv_base = sdesc_sw128_base(skv, 16384, 1024);
      constexpr int kKPlane = kPair ? 8192 : 16384;  // K tile d-plane stride (pair: 64-key half tiles)
      auto issue_qk = [&](int s, int slot) {
        if (leader) {
          const uint64_t da = dq_base + static_cast<uint64_t>((s * L::kTileBytes) >> 4);
          const uint64_t db = dk_base + static_cast<uint64_t>((slot * kSlotBytes) >> 4);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint64_t oa = ((kk >> 2) * 16384 + (kk & 3) * 32) >> 4;
            const uint64_t ob = ((kk >> 2) * kKPlane + (kk & 3) * 32) >> 4;
            if constexpr (kPair)
              mma_ss2(tmem + s * 128, da + oa, db + ob, idesc_qk, kk > 0);
            else
              mma_ss(tmem + s * 128, da + oa, db + ob, idesc_qk, kk > 0);
          }
        }
        __syncwarp();
      };
      auto issue_pv = [&](int s, int slot, uint32_t acc) {
        if (leader) {
          const uint64_t db = dv_base + static_cast<uint64_t>((slot * kSlotBytes) >> 4);
          const uint32_t ta = tmem + s * 128 + 64;
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            if constexpr (kPair)
              mma_ts2(tmem + 256 + s * 128, ta + kk * 8, db + static_cast<uint64_t>((kk * 2048) >> 4), idesc_pv,
                      (acc | kk) != 0);
            else
              mma_ts(tmem + 256 + s * 128, ta + kk * 8, db + static_cast<uint64_t>((kk * 2048) >> 4), idesc_pv,
                     (acc | kk) != 0);
          }
        }
        __syncwarp();
      };
      auto commit = [&](uint64_t* bar) {
        if (leader) {
          if constexpr (kPair)
            mma_commit_pair(bar);
          else
            mma_commit(bar);
        }
        __syncwarp();
      };
      auto wait_p = [&](int s, uint32_t parity) { mbar_wait(&p_full[s], parity); };
      auto wait_entry = [&](int e) { mbar_wait(&kv_full[e % kSlots], (e / kSlots) & 1); };
      auto release = [&](int e) { commit(&kv_empty[e % kSlots]); };
      mbar_wait(&q_full[0], 0);
      mbar_wait(&q_full[1], 0);
      if (MODE == MODE_TAYLOR) {
        for (int s = 0; s < 2; ++s) {
          wait_entry(s);
          __syncwarp();
          tc_fence_after();
          issue_qk(s, s % kSlots);
          commit(&s_full[s]);
          release(s);
        }
        for (int i = 1; i < n_kv; ++i) {
          const int base = 2 + 4 * (i - 1);
          for (int s = 0; s < 2; ++s) {
            const int ev = base + 2 * s, ek = ev + 1;
            wait_p(s, (i - 1) & 1);
            if (leader && ISA_TRACE_MODE == 2) ISA_TSTAMP(i, s, 6);
            wait_entry(ev);
            if (leader && ISA_TRACE_MODE == 2) ISA_TSTAMP(i, s, 5);
            __syncwarp();
            tc_fence_after();
            issue_pv(s, ev % kSlots, i > 1);
            release(ev);
            wait_entry(ek);
            __syncwarp();
            tc_fence_after();
            issue_qk(s, ek % kSlots);
            commit(&s_full[s]);
            if (leader && ISA_TRACE_MODE == 2) ISA_TSTAMP(i, s, 7);
            release(ek);
          }
          if (leader) progress(1, 1000 * i + 1);
        }
        for (int s = 0; s < 2; ++s) {
          const int ev = 4 * n_kv - 2 + s;
          wait_p(s, (n_kv - 1) & 1);
          wait_entry(ev);
          __syncwarp();
          tc_fence_after();
          issue_pv(s, ev % kSlots, n_kv > 1);
          commit(&o_full[s]);
          release(ev);
        }
      } else {
        wait_entry(0);
        __syncwarp();
        tc_fence_after();
        issue_qk(0, 0);
        commit(&s_full[0]);
        issue_qk(1, 0);
        commit(&s_full[1]);
        release(0);
        for (int i = 1; i < n_kv; ++i) {
          const int ev = 2 * i - 1, ek = 2 * i;
          wait_entry(ev);
          wait_entry(ek);
          if (leader && ISA_TRACE_MODE != 2) ISA_TSTAMP(i, 0, 5);
          if (leader) progress(1, 1000 * i + 1);
          for (int s = 0; s < 2; ++s) {
            wait_p(s, (i - 1) & 1);
            if (leader && ISA_TRACE_MODE != 2) ISA_TSTAMP(i, s, 6);
            __syncwarp();
            tc_fence_after();
            issue_pv(s, ev % kSlots, i > 1);
            issue_qk(s, ek % kSlots);
            commit(&s_full[s]);
            if (leader && ISA_TRACE_MODE != 2) ISA_TSTAMP(i, s, 7);
          }
          release(ev);
          release(ek);
        }
        const int ev = 2 * n_kv - 1;
        wait_entry(ev);
        for (int s = 0; s < 2; ++s) {
          wait_p(s, (n_kv - 1) & 1);
          __syncwarp();
          tc_fence_after();
          issue_pv(s, ev % kSlots, n_kv > 1);
          commit(&o_full[s]);
        }
        release(ev);
      }
    }
    __syncwarp();
  } else {
    // -------------------------------------------------------------- softmax
    setmaxnreg_inc<kSoftmaxRegs>();
    auto arrive_p = [&](int st) {  // P(i) of stage st written to TMEM
      if constexpr (kPair) {
        if (rank) {
          mbar_arrive_leader(&p_full[st]);
          return;
        }
      }
      mbar_arrive(&p_full[st]);
    };
    const int s = warp >> 2;                  // Q tile (stage)
    const int row = (warp & 3) * 32 + lane;   // row in the 128-row tile == TMEM lane
    const int qb = 2 * s + (row >> 6);        // query block 0..3 of this CTA
    const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const uint32_t t_s = tmem + lane_base + s * 128;
    const uint32_t t_p = t_s + 64;
    const uint32_t t_o = tmem + lane_base + 256 + s * 128;
    const float sl2 = p.scale_log2;
    float m = -INFINITY;  // running max, log2 domain (already scaled)
    float l = 0.f;
    const uint32_t* mbits = nullptr;
    uint32_t mreg[4] = {0u, 0u, 0u, 0u};  // member words (W <= 128, checked on the host)
    int jsrc = -1, jctx = -1;
    float lwsrc = 6.f, lwctx = 6.f;
    if (MODE == MODE_TAYLOR) {
      int pos = item * 4 + qb;
      if (pos >= p.n_qblk) pos = item * 4;
      mbits = p.member_bits + ((long long)bh * p.n_qblk + pos) * p.W;
      // the row block's member words live in registers across the warp
      // (lane w holds words w and w + 32): centroid tiles fetch theirs with
      // shuffles instead of a dependent global load on the S -> P path
#pragma unroll
      for (int r = 0; r < 4; ++r) mreg[r] = lane + 32 * r < p.W ? __ldg(mbits + lane + 32 * r) : 0u;
      if (p.l_src & 63) {  // short last source block = K_new block t_src-1
        jsrc = p.t_src - 1;
        lwsrc = log2f(static_cast<float>(p.l_src & 63));
      }
      if (p.l_ctx & 63) {  // short last context block, if it was selected
        jctx = p.ctx_short_j[bh];
        lwctx = log2f(static_cast<float>(p.l_ctx & 63));
      }
    }
    // Column validity of the current K/V tile, computed without the block
    // table: only K_new block t_src-1 and the selected short context block can
    // hold fewer than 64 rows. TAYLOR tile descriptors are prefetched one
    // tile ahead so their load latency hides behind the current tile.
    const int jshort = (MODE != MODE_DENSE && (p.l_ctx & 63)) ? p.ctx_short_j[bh] : -1;
    auto kn_valid = [&](int kn) -> int {
      if (kn < 0 || kn >= p.t_new) return 0;
      if (MODE == MODE_DENSE) return blk_valid(p, kn);
      if ((p.l_src & 63) && kn == p.t_src - 1) return p.l_src & 63;
      if (kn == jshort) return p.l_ctx & 63;
      return 64;
    };
    const int n_exact = (MODE == MODE_TAYLOR) ? p.n_tiles[bh * p.n_items + item] : 0;
    const int4* tlist = (MODE == MODE_TAYLOR)
                            ? p.tiles + (((long long)bh * p.n_items + item) * 2 + s) * p.max_tiles
                            : nullptr;
    int4 e_next = (MODE == MODE_TAYLOR && n_exact > 0) ? tlist[0] : make_int4(0, 0, 0, 0);
    for (int i = 0; i < n_kv; ++i) {
      TileInfo t;
      t.centroid = 0;
      t.cidx = 0;
      if (MODE == MODE_TAYLOR) {
        if (i < n_exact) {
          const int4 e = e_next;
          if (i + 1 < n_exact) e_next = tlist[i + 1];
          t.valid0 = e.z >> 8;  // planned: visibility bits | valid rows << 8
          t.valid1 = e.w >> 8;
          t.bits0 = e.z & 0xF;
          t.bits1 = e.w & 0xF;
        } else {
          t.centroid = 1;
          t.cidx = i - n_exact;
          t.valid0 = t.valid1 = 64;
          t.bits0 = t.bits1 = 0xF;
        }
      } else {
        t.valid0 = kn_valid(2 * i);
        t.valid1 = kn_valid(2 * i + 1);
        t.bits0 = t.bits1 = 0xF;
      }
      mbar_wait(&s_full[s], i & 1);
      if ((warp & 3) == ISA_TRACE_Q && lane == 0 && (MODE == MODE_TAYLOR) == (ISA_TRACE_MODE == 2)) ISA_TSTAMP(i, s, 0);
      __syncwarp();  // reconverge before .sync.aligned tcgen05 ops
      tc_fence_after();
#ifdef ISA_EXP_NOSOFTMAX
      // Experiment: MMA/TMA ceiling with the softmax reduced to a P store.
      {
        uint32_t pk[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) pk[c] = 0x3c003c00u;
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) tmem_st16(t_p + 16 * ch, pk);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) arrive_p(s);
        if ((warp & 3) == ISA_TRACE_Q && lane == 0 && (MODE == MODE_TAYLOR) == (ISA_TRACE_MODE == 2)) ISA_TSTAMP(i, s, 4);
        l += 1.f;
        continue;
      }
#endif
      uint32_t sr[128];
#ifdef ISA_EXP_NOLOAD
      // Experiment: skip the TMEM read of S (synthetic scores).
#pragma unroll
      for (int c = 0; c < 128; ++c) sr[c] = __float_as_uint(0.001f * (float)((c * 7 + lane + i) & 63));
#else
#pragma unroll
      for (int c = 0; c < 128 / kLdCols; ++c) {
        if (kLdCols == 16) tmem_ld16(t_s + c * 16, sr + c * 16);
        else tmem_ld8(t_s + c * 8, sr + c * 8);
      }
      tmem_ld_wait();
#endif
      if ((warp & 3) == ISA_TRACE_Q && lane == 0 && (MODE == MODE_TAYLOR) == (ISA_TRACE_MODE == 2)) ISA_TSTAMP(i, s, 1);
#ifdef ISA_EXP_LOADONLY
      {
        float mm = -INFINITY;
#pragma unroll
        for (int c = 0; c < 128; c += 2) mm = fmax3(mm, __uint_as_float(sr[c]), __uint_as_float(sr[c + 1]));
        uint32_t pk[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) pk[c] = __float_as_uint(mm) & 0x3c003c00u;
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) tmem_st16(t_p + 16 * ch, pk);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) arrive_p(s);
        if ((warp & 3) == ISA_TRACE_Q && lane == 0 && (MODE == MODE_TAYLOR) == (ISA_TRACE_MODE == 2)) ISA_TSTAMP(i, s, 4);
        l += 1.f;
        continue;
      }
#endif
      float* x = reinterpret_cast<float*>(sr);
      // Column masks of this tile for this row's query block, one word per 32
      // columns (1 = excluded), plus an additive log2 weight: 0 for key
      // blocks, log2(64) for centroid columns (taylor.py:156). Masks are
      // warp-uniform (a warp's 32 rows belong to one query block), so wholly
      // masked halves skip their exponentials.
      uint32_t mw[4];
      float bias = 0.f;
      bool special = false;  // centroid tile holding a short block's centroid (per-column weight)
      if (!t.centroid) {
        const int v0 = ((t.bits0 >> qb) & 1) ? t.valid0 : 0;
        const int v1 = ((t.bits1 >> qb) & 1) ? t.valid1 : 0;
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          const int lim = (w < 2 ? v0 : v1) - 32 * (w & 1);
          mw[w] = lim >= 32 ? 0u : (lim <= 0 ? 0xffffffffu : ~((1u << lim) - 1u));
        }
      } else {
        const int j0 = t.cidx * 128;
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          const int live = p.t_new - (j0 + 32 * w);  // columns < t_new in this word
          const uint32_t oob = live >= 32 ? 0u : (live <= 0 ? 0xffffffffu : ~((1u << live) - 1u));
          mw[w] = oob;  // the row block's own members are ORed in where needed (add_members)
        }
        bias = 6.f;
        special = (jsrc >= j0 && jsrc < j0 + 128) || (jctx >= j0 && jctx < j0 + 128);
      }
      // centroid tiles: exclude the row block's own exact members
      // (taylor.py:154); words fetched from the warp's registers by shuffles,
      // only on the paths that process a centroid tile
      auto add_members = [&]() {
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          const int wi = t.cidx * 4 + w;
          uint32_t word = 0u;
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            const uint32_t xw = __shfl_sync(0xffffffffu, mreg[r], wi & 31);
            word = (wi >> 5) == r ? xw : word;
          }
          mw[w] |= word;
        }
      };
      bool skip0 = (mw[0] & mw[1]) == 0xffffffffu;
      bool skip1 = (mw[2] & mw[3]) == 0xffffffffu;
      bool dense = (mw[0] | mw[1] | mw[2] | mw[3]) == 0u;
      float mx[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) mx[j] = -INFINITY;
      bool force_rescale = false;
#ifndef ISA_NO_SPEC_MAX
      // Speculative hot path (dense tiles after the first): exponentiate
      // against the running max m right away; the tile max is reduced in the
      // same pass (off the S -> P dependency chain) and checked once at the
      // end. If it exceeds m + 8 (the lazy-rescale threshold below; rare after
      // the first tiles) the tile is redone by the general path with a
      // rescale to the new max (x[] still holds the raw scores).
      // Each 64-column half must be wholly kept or wholly excluded (always
      // true for K6 tiles and for the Taylor union tiles of full blocks: the
      // visibility bits are per (query block, key block)); excluded halves
      // get P = 0 with no exponentials.
      const bool half0 = (mw[0] | mw[1]) == 0u, half1 = (mw[2] | mw[3]) == 0u;
      // (K6/K8 take only fully dense tiles here: their code has a single,
      // straight-line schedule; partial tiles use the general path.)
      const bool halfwise =
          MODE == MODE_TAYLOR ? ((half0 || skip0) && (half1 || skip1) && (half0 || half1)) : dense;
      if (MODE == MODE_TAYLOR && !t.centroid && skip0 && skip1) {
        // Union tile none of whose blocks this row block lists: P = 0, no
        // state change (warp-uniform).
        uint32_t pk[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) pk[c] = 0u;
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) tmem_st16(t_p + 16 * ch, pk);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) arrive_p(s);
        ISA_COUNT(MODE, 3);
        continue;
      }
      // Taylor centroid tiles (taylor.py:153-159) also take the speculative
      // path: excluded centroids (the row block's own exact members, columns
      // past t_new) are set to -inf first, so they contribute p = 0.
#ifdef ISA_TAYLOR_FULLMASK
      const bool cmask = MODE == MODE_TAYLOR && (t.centroid || (halfwise && !dense));
#else
      const bool cmask = MODE == MODE_TAYLOR && t.centroid;
#endif
      if (i > 0 && (halfwise || cmask) && !special) {
        const float2 sl2x2 = make_float2(sl2, sl2), nb2 = make_float2(bias - m, bias - m);
        float2 sp2[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
        // masked_tag: std::true_type only on the centroid path, so the per-column
        // exclusion selects exist in that copy of the code alone (a runtime flag
        // gets if-converted into 128 SELs on every tile)
        auto chunk = [&](const int ch, auto masked_tag, auto emu_tag) {
          constexpr bool kMasked = decltype(masked_tag)::value;
          constexpr int kEmu = decltype(emu_tag)::value;
          uint32_t pk[16];
#pragma unroll
          for (int c = 0; c < 16; ++c) {
            const int cc = 32 * ch + 2 * c;
            float xa = x[cc], xb = x[cc + 1];
            if (kMasked) {  // excluded centroids (own exact members, past t_new) -> p = 0
              const uint32_t w = mw[ch];
              xa = ((w >> (2 * c)) & 1u) ? -INFINITY : xa;
              xb = ((w >> (2 * c + 1)) & 1u) ? -INFINITY : xb;
            }
#ifndef ISA_SPEC_SUMCHECK
            mx[c & 7] = fmax3(mx[c & 7], xa, xb);
#endif
            const float2 tt = ffma2(make_float2(xa, xb), sl2x2, nb2);
            float2 pp;
            if (kEmu > 0 && (c % kEmu) == kEmu - 1) {
              pp = ex2_emu2(tt);
            } else {
              pp.x = ex2_approx(tt.x);
              pp.y = ex2_approx(tt.y);
            }
            sp2[c & 3] = fadd2(sp2[c & 3], pp);
            pk[c] = pack_p(pp.x, pp.y);
          }
          tmem_st16(t_p + 16 * ch, pk);
        };
        using EmuStd = std::integral_constant<int, kEmuEvery>;
        auto zero = [&](const int ch) {
          uint32_t pk[16];
#pragma unroll
          for (int c = 0; c < 16; ++c) pk[c] = 0u;
          tmem_st16(t_p + 16 * ch, pk);
        };
        const std::false_type plain{};
        if (MODE == MODE_TAYLOR && cmask) {  // Taylor centroid tile
          add_members();
#pragma unroll
          for (int ch = 0; ch < 4; ++ch) chunk(ch, std::true_type{}, EmuStd{});
        } else if (MODE != MODE_TAYLOR || dense) {  // every K6/K8 tile: one straight-line schedule
#pragma unroll
          for (int ch = 0; ch < 4; ++ch) chunk(ch, plain, EmuStd{});
        } else if (half0) {  // Taylor union tile, only the first 64 keys listed (warp-uniform):
          chunk(0, plain, EmuStd{});  // straight-line code per case so the two chunks interleave
          chunk(1, plain, EmuStd{});
          zero(2);
          zero(3);
        } else {
          zero(0);
          zero(1);
          chunk(2, plain, EmuStd{});
          chunk(3, plain, EmuStd{});
        }
#ifdef ISA_TRACE_SPEC
        if ((warp & 3) == ISA_TRACE_Q && lane == 0 && (MODE == MODE_TAYLOR) == (ISA_TRACE_MODE == 2)) ISA_TSTAMP(i, s, 2);
#endif
#ifdef ISA_SPEC_SUMCHECK
        // every p <= sum: sum <= 2^8 bounds the tile max by m + 8
        const float2 s2c = fadd2(fadd2(sp2[0], sp2[1]), fadd2(sp2[2], sp2[3]));
        const bool redo = !(s2c.x + s2c.y <= 256.f);
#else
        const float mt = fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])), fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7])));
        const bool redo = (m == -INFINITY) || (fmaf(mt, sl2, bias) > m + 8.f);
#endif
        tmem_st_wait();
#ifdef ISA_TRACE_SPEC
        if ((warp & 3) == ISA_TRACE_Q && lane == 0 && (MODE == MODE_TAYLOR) == (ISA_TRACE_MODE == 2)) ISA_TSTAMP(i, s, 3);
#endif
        if (!__any_sync(0xffffffffu, redo)) {
          ISA_COUNT(MODE, 0);
          tc_fence_before();
          __syncwarp();
          if (lane == 0) arrive_p(s);
          if ((warp & 3) == ISA_TRACE_Q && lane == 0 && (MODE == MODE_TAYLOR) == (ISA_TRACE_MODE == 2)) ISA_TSTAMP(i, s, 4);
          const float2 s2 = fadd2(fadd2(sp2[0], sp2[1]), fadd2(sp2[2], sp2[3]));
          l += s2.x + s2.y;
          if ((threadIdx.x & 127) == 0) progress(2 + s, i + 1);
          continue;
        }
        // rare: the general path below recomputes the max and P from x[]
        ISA_COUNT(MODE, 1);
        force_rescale = true;
#pragma unroll
        for (int j = 0; j < 8; ++j) mx[j] = -INFINITY;
      }
#endif
      if (MODE == MODE_TAYLOR && t.centroid) {  // general path on a centroid tile (first tile / redo)
        add_members();
        skip0 = (mw[0] & mw[1]) == 0xffffffffu;
        skip1 = (mw[2] & mw[3]) == 0xffffffffu;
        dense = (mw[0] | mw[1] | mw[2] | mw[3]) == 0u;
      }
      if (special) {  // rare: per-column weights, scaled in place
        const int j0 = t.cidx * 128;
#pragma unroll
        for (int cc = 0; cc < 128; ++cc) {
          const int j = j0 + cc;
          const float bj = j == jsrc ? lwsrc : (j == jctx ? lwctx : 6.f);
          x[cc] = ((mw[cc >> 5] >> (cc & 31)) & 1) ? -INFINITY : fmaf(x[cc], sl2, bj);
          mx[cc & 7] = fmaxf(mx[cc & 7], x[cc]);
        }
      } else if (dense) {  // raw scores, scaled inside the exp2 FMA below
#pragma unroll
        for (int c = 0; c < 128; c += 2) mx[(c >> 1) & 7] = fmax3(mx[(c >> 1) & 7], x[c], x[c + 1]);
      } else {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (h == 0 ? skip0 : skip1) continue;
#pragma unroll
          for (int c = 64 * h; c < 64 * h + 64; c += 2) {
            const uint32_t w = mw[c >> 5];
            const float a0 = ((w >> (c & 31)) & 1) ? -INFINITY : x[c];
            const float a1 = ((w >> ((c + 1) & 31)) & 1) ? -INFINITY : x[c + 1];
            mx[(c >> 1) & 7] = fmax3(mx[(c >> 1) & 7], a0, a1);
          }
        }
      }
      float mt = fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])), fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7])));
      if (!special) mt = fmaf(mt, sl2, bias);  // max(x*sl2 + b) over the kept columns
      // running max with lazy rescale (threshold 8 in log2 units)
      ISA_COUNT(MODE, 2);
      float m_new = fmaxf(m, mt);
      float o_scale = 1.f;
      bool need = false;
      if (i == 0) {
        m = m_new;
      } else if (m_new > m + (force_rescale ? 0.f : 8.f)) {
        o_scale = ex2_approx(m - m_new);  // m == -inf -> 0 (O and l are 0 then)
        need = true;
        m = m_new;
      }
      if (__any_sync(0xffffffffu, need)) {
        l *= o_scale;
#pragma unroll 1
        for (int c = 0; c < D / 32; ++c) {
          uint32_t orr[32];
          tmem_ld32(t_o + c * 32, orr);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j) orr[j] = __float_as_uint(__uint_as_float(orr[j]) * o_scale);
          tmem_st32(t_o + c * 32, orr);
        }
      }
      if ((warp & 3) == ISA_TRACE_Q && lane == 0 && (MODE == MODE_TAYLOR) == (ISA_TRACE_MODE == 2)) ISA_TSTAMP(i, s, 2);
      const float mu = (m == -INFINITY) ? 0.f : m;
      float sm[4] = {0.f, 0.f, 0.f, 0.f};
      float2 sm2[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
      // P in 4 chunks of 32 columns, each stored to TMEM right away so the
      // live register set stays ~ S row + 16 packed words.
      const float2 sl2x2 = make_float2(sl2, sl2), nb2 = make_float2(bias - mu, bias - mu);
      if (dense && !special) {
        // hot path (every K6/K8 tile): FFMA2 scale-subtract; 1 in kEmuEvery
        // pairs takes the FMA-pipe polynomial exp2, the rest the MUFU (SFU).
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) {
          uint32_t pk[16];
#pragma unroll
          for (int c = 0; c < 16; ++c) {
            const float2 tt = ffma2(make_float2(x[32 * ch + 2 * c], x[32 * ch + 2 * c + 1]), sl2x2, nb2);
            float2 pp;
            if (kEmuEvery > 0 && (c % kEmuEvery) == kEmuEvery - 1) {
              pp = ex2_emu2(tt);
            } else {
              pp.x = ex2_approx(tt.x);
              pp.y = ex2_approx(tt.y);
            }
            sm2[c & 3] = fadd2(sm2[c & 3], pp);
            pk[c] = pack_bf16x2(pp.x, pp.y);
          }
          tmem_st16(t_p + 16 * ch, pk);
        }
      } else if (special) {
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) {
          uint32_t pk[16];
#pragma unroll
          for (int c = 0; c < 16; ++c) {
            const float p0 = ex2_approx(x[32 * ch + 2 * c] - mu);
            const float p1 = ex2_approx(x[32 * ch + 2 * c + 1] - mu);
            sm[c & 3] += p0 + p1;
            pk[c] = pack_bf16x2(p0, p1);
          }
          tmem_st16(t_p + 16 * ch, pk);
        }
      } else {
        // masked tiles (Taylor unions, centroids, ragged/missing halves):
        // wholly excluded halves write P = 0 with no exponentials; partial
        // words zero their excluded columns after the MUFU exp2.
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) {
          uint32_t pk[16];
          const uint32_t w = mw[ch];
          if (ch < 2 ? skip0 : skip1) {
#pragma unroll
            for (int c = 0; c < 16; ++c) pk[c] = 0u;
          } else {
#pragma unroll
            for (int c = 0; c < 16; ++c) {
              const float2 tt = ffma2(make_float2(x[32 * ch + 2 * c], x[32 * ch + 2 * c + 1]), sl2x2, nb2);
              float2 pp;
              pp.x = ((w >> (2 * c)) & 1) ? 0.f : ex2_approx(tt.x);
              pp.y = ((w >> (2 * c + 1)) & 1) ? 0.f : ex2_approx(tt.y);
              sm2[c & 3] = fadd2(sm2[c & 3], pp);
              pk[c] = pack_bf16x2(pp.x, pp.y);
            }
          }
          tmem_st16(t_p + 16 * ch, pk);
        }
      }
      if ((warp & 3) == ISA_TRACE_Q && lane == 0 && (MODE == MODE_TAYLOR) == (ISA_TRACE_MODE == 2)) ISA_TSTAMP(i, s, 3);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) arrive_p(s);
      if ((warp & 3) == ISA_TRACE_Q && lane == 0 && (MODE == MODE_TAYLOR) == (ISA_TRACE_MODE == 2)) ISA_TSTAMP(i, s, 4);
      const float2 s2 = fadd2(fadd2(sm2[0], sm2[1]), fadd2(sm2[2], sm2[3]));
      l += ((sm[0] + sm[1]) + (sm[2] + sm[3])) + (s2.x + s2.y);
      if ((threadIdx.x & 127) == 0) progress(2 + s, i + 1);
    }
    // -------------------------------------------------------------- epilogue
    mbar_wait(&o_full[s], 0);
    __syncwarp();
    tc_fence_after();
    const int u = query_block<MODE>(p, bh, item, qb);
    const int rr = row & 63;
    const bool write = u >= 0 && rr < blk_valid(p, u);
    if (write && !(l > 0.f) && p.err_flag) atomicOr(p.err_flag, 2);
    if (write && p.lse) p.lse[(long long)bh * p.S + blk_tok0(p, u) + rr] = l > 0.f ? m + log2f(l) : -INFINITY;
    const float inv = l > 0.f ? 1.f / l : 0.f;
    const int hh = bh % p.H, bb = bh / p.H;
    const long long obase =
        bb * p.o_sb + hh * p.o_sh + (long long)(write ? blk_tok0(p, u) + rr : 0) * p.o_ss;
    const float* res_row = (p.resid && write) ? p.resid + ((long long)bh * p.T + u) * D : nullptr;
#pragma unroll 1
    for (int c = 0; c < D / 32; ++c) {
      uint32_t orr[32];
      __syncwarp();
      tmem_ld32(t_o + c * 32, orr);
      tmem_ld_wait();
      if (res_row) {  // O/l + gamma * O_coarse, folded so the stores below stay unchanged
#pragma unroll
        for (int j = 0; j < 32; ++j)
          orr[j] = __float_as_uint(__uint_as_float(orr[j]) + p.gamma * __ldg(res_row + c * 32 + j) * l);
      }
      if (write) {
        if (p.out_fp32) {
          float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(p.out) + obase + c * 32);
#pragma unroll
          for (int j = 0; j < 8; ++j)
            dst[j] = make_float4(__uint_as_float(orr[4 * j]) * inv, __uint_as_float(orr[4 * j + 1]) * inv,
                                 __uint_as_float(orr[4 * j + 2]) * inv, __uint_as_float(orr[4 * j + 3]) * inv);
        } else {
          uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(p.out) + obase + c * 32);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            uint4 w;
            w.x = pack_bf16x2(__uint_as_float(orr[8 * j + 0]) * inv, __uint_as_float(orr[8 * j + 1]) * inv);
            w.y = pack_bf16x2(__uint_as_float(orr[8 * j + 2]) * inv, __uint_as_float(orr[8 * j + 3]) * inv);
            w.z = pack_bf16x2(__uint_as_float(orr[8 * j + 4]) * inv, __uint_as_float(orr[8 * j + 5]) * inv);
            w.w = pack_bf16x2(__uint_as_float(orr[8 * j + 6]) * inv, __uint_as_float(orr[8 * j + 7]) * inv);
            dst[j] = w;
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (kPair) cluster_sync_all();  // the peer's MMAs / signals into this CTA are complete
  if (warp == 8) {
    tc_fence_after();
    if constexpr (kPair)
      tmem_dealloc2<512>(tmem);
    else
      tmem_dealloc<512>(tmem);
  }
}

// K6 / K8 on CTA pairs (cta_group::2, cluster of 2 along x): items 2c and
// 2c+1 of a head run as one M = 256 MMA stream; each SM loads half of every
// K/V tile and feeds half of each MMA's B operand.
template <int D, int MODE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    gba_attention_pair_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                              const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_kc,
                              const __grid_constant__ CUtensorMap tm_vc, const AttnParams p) {
  gba_body<D, MODE, true>(tm_q, tm_k, tm_v, tm_kc, tm_vc, p, blockIdx.x, blockIdx.y);
  if (p.head_done) {
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) atomicAdd(p.head_done + blockIdx.y, 1);
  }
}

// One branch per launch (K6 exact, K7 Taylor or K8 dense).
template <int D, int MODE>
__global__ void __launch_bounds__(kThreads, 1)
    gba_attention_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                         const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_kc,
                         const __grid_constant__ CUtensorMap tm_vc, const AttnParams p) {
  gba_body<D, MODE>(tm_q, tm_k, tm_v, tm_kc, tm_vc, p, blockIdx.x, blockIdx.y);
  if (p.head_done) {  // this CTA's output rows are final: publish for the comm stream (parallel.py)
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) atomicAdd(p.head_done + blockIdx.y, 1);
  }
}

// Both ISA branches in one launch: CTAs [0, n_exact) run the sharp items (288
// K/V steps each at cfg3), the rest the Taylor items (~41 steps). The short
// Taylor CTAs fill the tail wave of the long exact ones instead of a second
// kernel ramping up after a ~60%-occupied last wave.
template <int D>
__global__ void __launch_bounds__(kThreads, 1)
    gba_isa_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                   const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_kc,
                   const __grid_constant__ CUtensorMap tm_vc, const AttnParams pe, const AttnParams pt,
                   const int n_exact) {
  if ((int)blockIdx.x < n_exact)
    gba_body<D, MODE_EXACT>(tm_q, tm_k, tm_v, tm_kc, tm_vc, pe, blockIdx.x, blockIdx.y);
  else
    gba_body<D, MODE_TAYLOR>(tm_q, tm_k, tm_v, tm_kc, tm_vc, pt, blockIdx.x - n_exact, blockIdx.y);
}

}  // namespace isa
