// Double-buffered variant of the exact/dense attention body (K6/K8):
// 64-key K/V tiles (one K_new block each) and TWO S buffers per Q tile, so the
// MMA warp can issue QK(i+2) as soon as PV(i) is issued — the softmax of tile
// i+1 never waits for the MMA round trip of tile i (distance-2 pipelining).
//
// TMEM per Q tile s (256 columns): S_s[0] [0,64) S_s[1] [64,128) O_s [128,256);
// P_s[b] (bf16 pairs, 32 columns) overwrites the upper half of S_s[b].
// Ring entries (16 KB each, 10 slots = 160 KB + 64 KB Q): K_0 K_1 | V_0 K_2 |
// V_1 K_3 | ... | V_{n-2} V_{n-1}; producer and MMA walk the same loop.
// The O rescale (rare, threshold 2^8) waits on o_ready for PV(i-1), which
// S(i) no longer implies.
#pragma once
#include "isa_attn.cuh"

namespace isa {

constexpr int kP2Slots = 10;

template <int D>
struct P2Smem {
  static constexpr int kPlanes = D / 64;
  static constexpr int kQBytes = 128 * D * 2;   // one 128-row Q tile
  static constexpr int kKVBytes = 64 * D * 2;   // one 64-row K or V block
  static constexpr int kQOff = 0;
  static constexpr int kKvOff = 2 * kQBytes;
  static constexpr int kBarOff = kKvOff + kP2Slots * kKVBytes;
  static constexpr int kBytes = kBarOff + 512;
  static constexpr int kAlloc = kBytes + 1024;
};

template <int D, int MODE>
__device__ __forceinline__ void gba_body_p2(const CUtensorMap& tm_q, const CUtensorMap& tm_k,
                                            const CUtensorMap& tm_v, const AttnParams& p, const int item,
                                            const int bh) {
  static_assert(MODE == MODE_DENSE || MODE == MODE_EXACT, "p2 pipeline serves the exact/dense branches");
  using L = P2Smem<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem + L::kQOff;
  uint8_t* sKV = smem + L::kKvOff;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBarOff);
  uint64_t* q_full = bars + 0;                  // [2]
  uint64_t* kv_full = bars + 2;                 // [kP2Slots]
  uint64_t* kv_empty = bars + 2 + kP2Slots;     // [kP2Slots]
  uint64_t* s_full = bars + 2 + 2 * kP2Slots;   // [2 stages][2 buffers]
  // p_full per (stage, buffer): the softmax can run two tiles ahead of the MMA
  // warp, so one barrier per stage would alias phases i and i+2.
  uint64_t* p_full = bars + 6 + 2 * kP2Slots;   // [2 stages][2 buffers]
  uint64_t* o_ready = bars + 10 + 2 * kP2Slots; // [2] one phase per PV (rescale waits)
  uint64_t* o_full = bars + 12 + 2 * kP2Slots;  // [2] after the last PV (epilogue)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 14 + 2 * kP2Slots);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int n_kv = p.t_new;  // one K_new block per tile

  if (threadIdx.x == 0) {
    mbar_init(&q_full[0], 1);
    mbar_init(&q_full[1], 1);
    for (int s = 0; s < kP2Slots; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int s = 0; s < 4; ++s) {
      mbar_init(&s_full[s], 1);
      mbar_init(&p_full[s], 4);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&o_ready[s], 1);
      mbar_init(&o_full[s], 1);
    }
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
      }
      const uint64_t pol_q = policy_evict_first();
      const uint64_t pol_kv = policy_evict_last();
      const int hh = bh % p.H, bb = bh / p.H;
      const int first_u = query_block<MODE>(p, bh, item, 0);
      const int* tab = MODE == MODE_EXACT ? p.kv_blk + (long long)bh * p.t_new : nullptr;
      if (leader) {
        for (int s = 0; s < 2; ++s) {
          mbar_arrive_expect_tx(&q_full[s], L::kQBytes);
          for (int half = 0; half < 2; ++half) {
            int u = query_block<MODE>(p, bh, item, 2 * s + half);
            if (u < 0) u = first_u;
            const int tok = blk_tok0(p, u);
            for (int pl = 0; pl < L::kPlanes; ++pl)
              tma_load_4d(sQ + s * L::kQBytes + pl * 16384 + half * 8192, &tm_q, &q_full[s], pl * 64, tok, hh,
                          bb, pol_q);
          }
        }
      }
      int c = 0;
      auto load = [&](int j, bool is_v) {
        const int slot = c % kP2Slots;
        const int use = c / kP2Slots;
        if (use > 0) mbar_wait(&kv_empty[slot], (use - 1) & 1);
        __syncwarp();
        if (leader) {
          const int u = tab ? tab[j] : j;
          const int tok = blk_tok0(p, u);
          mbar_arrive_expect_tx(&kv_full[slot], L::kKVBytes);
          uint8_t* dst = sKV + slot * L::kKVBytes;
          const CUtensorMap* tm = is_v ? &tm_v : &tm_k;
          for (int pl = 0; pl < L::kPlanes; ++pl)
            tma_load_4d(dst + pl * 8192, tm, &kv_full[slot], pl * 64, tok, hh, bb, pol_kv);
        }
        ++c;
      };
      load(0, false);
      if (n_kv > 1) load(1, false);
      for (int i = 0; i < n_kv; ++i) {
        load(i, true);
        if (i + 2 < n_kv) load(i + 2, false);
      }
    } else if (warp == 8) {
      // ------------------------------------------------------------ MMA issuer
      constexpr uint32_t idesc_qk = idesc_bf16_f32(128, 64, 0, 0);
      constexpr uint32_t idesc_pv = idesc_bf16_f32(128, D, 0, 1);
      const uint32_t sq = smem_u32(sQ);
      const uint32_t skv = smem_u32(sKV);
      const bool leader = elect_one();
      auto issue_qk = [&](int s, int buf, int slot) {
        if (leader) {
          const uint32_t a0 = sq + s * L::kQBytes;
          const uint32_t b0 = skv + slot * L::kKVBytes;
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t ao = (kk >> 2) * 16384 + (kk & 3) * 32;
            const uint32_t bo = (kk >> 2) * 8192 + (kk & 3) * 32;
            mma_ss(tmem + 256 * s + 64 * buf, sdesc_sw128(a0 + ao, 16, 1024), sdesc_sw128(b0 + bo, 16, 1024),
                   idesc_qk, kk > 0);
          }
        }
        __syncwarp();
      };
      auto issue_pv = [&](int s, int buf, int slot, uint32_t acc) {
        if (leader) {
          const uint32_t b0 = skv + slot * L::kKVBytes;
          const uint32_t ta = tmem + 256 * s + 64 * buf + 32;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            mma_ts(tmem + 256 * s + 128, ta + kk * 8, sdesc_sw128(b0 + kk * 2048, 8192, 1024), idesc_pv,
                   (acc | kk) != 0);
        }
        __syncwarp();
      };
      auto commit = [&](uint64_t* bar) {
        if (leader) mma_commit(bar);
        __syncwarp();
      };
      auto wait_entry = [&](int e) { mbar_wait(&kv_full[e % kP2Slots], (e / kP2Slots) & 1); };
      auto release = [&](int e) { commit(&kv_empty[e % kP2Slots]); };
      mbar_wait(&q_full[0], 0);
      mbar_wait(&q_full[1], 0);
      int c = 0;
      for (int j = 0; j < (n_kv > 1 ? 2 : 1); ++j) {  // QK(0), QK(1) into buffers 0, 1
        wait_entry(c);
        __syncwarp();
        tc_fence_after();
        for (int s = 0; s < 2; ++s) {
          issue_qk(s, j, c % kP2Slots);
          commit(&s_full[2 * s + j]);
        }
        release(c);
        ++c;
      }
      for (int i = 0; i < n_kv; ++i) {
        const int buf = i & 1;
        const int cv = c++;
        const int ck = (i + 2 < n_kv) ? c++ : -1;
        wait_entry(cv);
        if (ck >= 0) wait_entry(ck);
        for (int s = 0; s < 2; ++s) {
          mbar_wait(&p_full[2 * s + buf], (i >> 1) & 1);
          __syncwarp();
          tc_fence_after();
          issue_pv(s, buf, cv % kP2Slots, i > 0);
          commit(&o_ready[s]);
          if (i == n_kv - 1) commit(&o_full[s]);
          if (ck >= 0) {
            issue_qk(s, buf, ck % kP2Slots);  // S_s[buf] is free once PV(i) is in the pipe
            commit(&s_full[2 * s + buf]);
          }
        }
        release(cv);
        if (ck >= 0) release(ck);
        if (leader) progress(1, i + 1);
      }
    }
    __syncwarp();
  } else {
    // -------------------------------------------------------------- softmax
    setmaxnreg_inc<kSoftmaxRegs>();
    const int s = warp >> 2;
    const int row = (warp & 3) * 32 + lane;
    const int qb = 2 * s + (row >> 6);
    const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const uint32_t t_st = tmem + lane_base + 256 * s;  // S_s[0]
    const uint32_t t_o = t_st + 128;
    const float sl2 = p.scale_log2;
    float m = -INFINITY;
    float l = 0.f;
    const int jshort = (MODE == MODE_EXACT && (p.l_ctx & 63)) ? p.ctx_short_j[bh] : -1;
    auto kn_valid = [&](int kn) -> int {
      if (MODE == MODE_DENSE) return blk_valid(p, kn);
      if ((p.l_src & 63) && kn == p.t_src - 1) return p.l_src & 63;
      if (kn == jshort) return p.l_ctx & 63;
      return 64;
    };
    for (int i = 0; i < n_kv; ++i) {
      const int buf = i & 1;
      const int valid = kn_valid(i);
      mbar_wait(&s_full[2 * s + buf], (i >> 1) & 1);
      __syncwarp();
      tc_fence_after();
      const uint32_t t_s = t_st + 64 * buf;
      uint32_t sr[64];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld16(t_s + c * 16, sr + c * 16);
      tmem_ld_wait();
      float* x = reinterpret_cast<float*>(sr);
      float mx[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) mx[j] = -INFINITY;
      const bool dense = valid == 64;
      if (dense) {
#pragma unroll
        for (int c = 0; c < 64; c += 2) mx[(c >> 1) & 7] = fmax3(mx[(c >> 1) & 7], x[c], x[c + 1]);
      } else {
#pragma unroll
        for (int c = 0; c < 64; ++c) {
          x[c] = c < valid ? x[c] : -INFINITY;
          mx[c & 7] = fmaxf(mx[c & 7], x[c]);
        }
      }
      float mt = fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])), fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7])));
      mt *= sl2;
      float m_new = fmaxf(m, mt);
      float o_scale = 1.f;
      bool need = false;
      if (i == 0) {
        m = m_new;
      } else if (m_new > m + 8.f) {
        o_scale = ex2_approx(m - m_new);
        need = true;
        m = m_new;
      }
      if (__any_sync(0xffffffffu, need)) {
        // O must hold PV(i-1) before it is rescaled (S(i) only implies PV(i-2))
        mbar_wait(&o_ready[s], (i - 1) & 1);
        __syncwarp();
        tc_fence_after();
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
      const float mu = (m == -INFINITY) ? 0.f : m;
      const float2 sl2x2 = make_float2(sl2, sl2), nb2 = make_float2(-mu, -mu);
      float2 sm2[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
      const uint32_t t_p = t_s + 32;
#pragma unroll
      for (int ch = 0; ch < 2; ++ch) {
        uint32_t pk[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          const float2 tt = ffma2(make_float2(x[32 * ch + 2 * c], x[32 * ch + 2 * c + 1]), sl2x2, nb2);
          float2 pp;
          if (dense && kEmuEvery > 0 && (c % kEmuEvery) == kEmuEvery - 1) {
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
      const float2 s2 = fadd2(fadd2(sm2[0], sm2[1]), fadd2(sm2[2], sm2[3]));
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[2 * s + buf]);
      l += s2.x + s2.y;
    }
    // -------------------------------------------------------------- epilogue
    // S(n-1) only implies PV(n-3), and o_ready's parity cannot tell phase n-2
    // from n: the last PV has its own barrier.
    mbar_wait(&o_full[s], 0);
    __syncwarp();
    tc_fence_after();
    const int u = query_block<MODE>(p, bh, item, qb);
    const int rr = row & 63;
    const bool write = u >= 0 && rr < blk_valid(p, u);
    if (write && !(l > 0.f) && p.err_flag) atomicOr(p.err_flag, 2);
    const float inv = l > 0.f ? 1.f / l : 0.f;
    const int hh = bh % p.H, bb = bh / p.H;
    const long long obase =
        bb * p.o_sb + hh * p.o_sh + (long long)(write ? blk_tok0(p, u) + rr : 0) * p.o_ss;
#pragma unroll 1
    for (int c = 0; c < D / 32; ++c) {
      uint32_t orr[32];
      __syncwarp();
      tmem_ld32(t_o + c * 32, orr);
      tmem_ld_wait();
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
  if (warp == 8) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

template <int D, int MODE>
__global__ void __launch_bounds__(kThreads, 1)
    gba_attention_p2_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                            const __grid_constant__ CUtensorMap tm_v, const AttnParams p) {
  gba_body_p2<D, MODE>(tm_q, tm_k, tm_v, p, blockIdx.x, blockIdx.y);
}

// Fused ISA grid with the double-buffered exact branch.
template <int D>
__global__ void __launch_bounds__(kThreads, 1)
    gba_isa_p2_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                      const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_kc,
                      const __grid_constant__ CUtensorMap tm_vc, const AttnParams pe, const AttnParams pt,
                      const int n_exact) {
  if ((int)blockIdx.x < n_exact)
    gba_body_p2<D, MODE_EXACT>(tm_q, tm_k, tm_v, pe, blockIdx.x, blockIdx.y);
  else
    gba_body<D, MODE_TAYLOR>(tm_q, tm_k, tm_v, tm_kc, tm_vc, pt, blockIdx.x - n_exact, blockIdx.y);
}

}  // namespace isa
