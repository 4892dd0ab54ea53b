// C ABI and native orchestration of the ISA forward on sm_100a.
//
// isa_forward runs the five reference stages (pipeline.py:133-370) as one
// stream-ordered sequence of kernels with no host synchronisation:
//   stage 1 "coarse"  K1 pool_means, K2 coarse_dmma (fp64 S of the source rows
//                     vs the context columns), K2b ctx_mean  pipeline.py:176-184
//   stage 2 "select"  K3 topk_rank (context), K_new block table, bf16 K_new
//                     centroids + log2 weights              pipeline.py:186-212
//   stage 3 "split"   K4a sharpness, K4b split, K5 block mask, Taylor plan
//                                                            pipeline.py:214-228
//   stage 4 "kernel"  K6 exact (sharp) and K7 Taylor (flat) tcgen05 attention,
//                     stage-5 scatter fused into their epilogues
//                                                            pipeline.py:331-358
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>

#include "../../include/isa_b200.h"
#include "isa_attn.cuh"
#include "isa_bwd.cuh"
#include "isa_bwd_tc.cuh"
#include "isa_route.cuh"
#include "isa_taylor_t.cuh"

namespace {

thread_local std::string g_last_error;
thread_local int g_launches = 0;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

#define ISA_CUDA(call)                                                                         \
  do {                                                                                         \
    cudaError_t e_ = (call);                                                                   \
    if (e_ != cudaSuccess) return fail(ISA_ERR_CUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
  } while (0)

#define ISA_LAUNCHED(name)                                                                             \
  do {                                                                                                 \
    ++g_launches;                                                                                      \
    cudaError_t e_ = cudaGetLastError();                                                               \
    if (e_ != cudaSuccess) return fail(ISA_ERR_CUDA, "launch %s: %s", name, cudaGetErrorString(e_)); \
  } while (0)

// Dynamic shared memory opt-in. cudaFuncSetAttribute applies to the current
// device's context only, so the granted size is remembered per (kernel,
// device) and grown on demand (a process may drive several GPUs).
int ensure_smem(const void* fn, size_t bytes) {
  if (bytes <= 48 * 1024) return ISA_OK;
  int dev = 0;
  ISA_CUDA(cudaGetDevice(&dev));
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> granted;
  std::lock_guard<std::mutex> lock(mu);
  size_t& cur = granted[{fn, dev}];
  if (bytes > cur) {
    ISA_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    cur = bytes;
  }
  return ISA_OK;
}

// ---------------------------------------------------------------- TMA maps
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}

// bf16 4-D map {D, d1, d2, d3} with byte strides s1..s3; box {64, 64, 1, 1}, 128B swizzle.
int make_map(CUtensorMap* m, const void* ptr, int D, long long d1, long long d2, long long d3, long long s1,
             long long s2, long long s3) {
  EncodeFn enc = encode_fn();
  if (!enc) return fail(ISA_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  if ((reinterpret_cast<uintptr_t>(ptr) & 15) || (s1 & 15) || (s2 & 15) || (s3 & 15))
    return fail(ISA_ERR_LAYOUT, "TMA needs 16-byte aligned base and strides (got strides %lld,%lld,%lld bytes)",
                s1, s2, s3);
  cuuint64_t dims[4] = {(cuuint64_t)D, (cuuint64_t)d1, (cuuint64_t)d2, (cuuint64_t)d3};
  cuuint64_t strides[3] = {(cuuint64_t)s1, (cuuint64_t)s2, (cuuint64_t)s3};
  cuuint32_t box[4] = {64, 64, 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(ISA_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return ISA_OK;
}

// ---------------------------------------------------------------- geometry
struct Dims {
  int B, H, S, D, BH;
  int l_src, l_ctx, t_src, t_ctx, T;
  int k_ctx, t_new, n_flat, n_sharp, k;
  int tn_pad, W, items_s, items_f, max_tiles;
  double scale;
  double gamma;       // coarse residual weight (0 = off)
  int resid_softmax;  // residual weights softmax(S_coarse) (1) or raw Qc.Kc (0)
  double rope_base;   // > 0: decoupled RoPE fused into the pooling pass
};

int derive(const IsaShape* sh, const IsaKnobs* kn, Dims* d) {
  if (!sh || !kn) return fail(ISA_ERR_CONFIG, "null shape/knobs");
  if (sh->block != 64) return fail(ISA_ERR_CONFIG, "block_size=%d not supported (only 64)", sh->block);
  if (sh->head_dim != 64 && sh->head_dim != 128)
    return fail(ISA_ERR_CONFIG, "head_dim=%d not supported (64 or 128)", sh->head_dim);
  if (sh->batch < 1 || sh->heads < 1 || sh->seq_len < 1)
    return fail(ISA_ERR_LAYOUT, "all dims must be >= 1");
  if (sh->l_src < 1 || sh->l_ctx < 0) return fail(ISA_ERR_LAYOUT, "l_src must be >= 1 and l_ctx >= 0");
  if (sh->l_src + sh->l_ctx != sh->seq_len)
    return fail(ISA_ERR_LAYOUT, "sequence length %d != icl total %d", sh->seq_len, sh->l_src + sh->l_ctx);
  if (sh->dtype != ISA_DTYPE_BF16 && sh->dtype != ISA_DTYPE_F32) return fail(ISA_ERR_CONFIG, "bad dtype");
  if (!(kn->scale > 0.0)) return fail(ISA_ERR_CONFIG, "scale must be > 0");
  d->B = sh->batch;
  d->H = sh->heads;
  d->S = sh->seq_len;
  d->D = sh->head_dim;
  d->BH = d->B * d->H;
  d->l_src = sh->l_src;
  d->l_ctx = sh->l_ctx;
  d->t_src = (sh->l_src + 63) / 64;
  d->t_ctx = (sh->l_ctx + 63) / 64;
  d->T = d->t_src + d->t_ctx;
  d->k_ctx = kn->k_ctx;
  if (d->k_ctx < 0 || d->k_ctx > d->t_ctx) return fail(ISA_ERR_CONFIG, "k_ctx=%d out of [0, %d]", d->k_ctx, d->t_ctx);
  d->t_new = d->t_src + d->k_ctx;
  d->n_flat = kn->n_flat;
  if (d->n_flat < 0 || d->n_flat > d->T) return fail(ISA_ERR_CONFIG, "n_flat=%d out of [0, %d]", d->n_flat, d->T);
  d->n_sharp = d->T - d->n_flat;
  d->k = d->n_flat ? kn->k_mask : 0;
  if (d->n_flat && (d->k < 1 || d->k > d->t_new))
    return fail(ISA_ERR_CONFIG, "k_mask=%d out of [1, %d]", d->k, d->t_new);
  d->tn_pad = ((d->t_new + 127) / 128) * 128;
  d->W = d->tn_pad / 32;
  if (d->n_flat && d->W > 128)  // the Taylor kernel keeps a row block's member words in 4 registers per lane
    return fail(ISA_ERR_CONFIG, "t_new=%d K_new blocks exceed the Taylor kernel's limit (4096)", d->t_new);
  d->items_s = (d->n_sharp + 3) / 4;
  d->items_f = (d->n_flat + 3) / 4;
  int u = 2 * d->k < d->t_new ? 2 * d->k : d->t_new;  // union of a pair of exact lists
  d->max_tiles = (u + 1) / 2;
  if (d->max_tiles < 1) d->max_tiles = 1;
  d->scale = kn->scale;
  if (!(kn->gamma >= 0.0)) return fail(ISA_ERR_CONFIG, "gamma must be >= 0, got %g", kn->gamma);
  d->gamma = kn->gamma;
  d->resid_softmax = kn->residual_softmax != 0;
  d->rope_base = kn->rope_base;
  if (d->rope_base < 0.0 || d->rope_base != d->rope_base) return fail(ISA_ERR_CONFIG, "rope base must be > 0");
  if (d->rope_base > 0.0 && sh->dtype != ISA_DTYPE_BF16)
    return fail(ISA_ERR_CONFIG, "fused decoupled RoPE takes bf16 Q/K/V");
  return ISA_OK;
}

struct Workspace {
  int32_t* err;
  float* means;  // [3][BH][T][D]
  __nv_bfloat16* bf;  // [3][BH][S][D] (fp32 inputs; [2] rotated Q, K with fused RoPE)
  float2* rope_tab;   // [S][D/2] (cos, sin) with fused RoPE
  double* s_new;      // [BH][T][t_new]  fp64 coarse scores vs K_new blocks
  double* s_ctx;      // [BH][t_src][t_ctx] fp64 source-row x context-column scores
  uint8_t* flags;     // [BH][max(T, t_ctx)]
  double* ctx;        // [BH][t_ctx]
  int* sel;           // [BH][k_ctx]
  int* kv_blk;        // [BH][t_new]
  double* sharpness;  // [BH][T]
  int* sharp;         // [BH][n_sharp]
  int* flat;          // [BH][n_flat]
  int* mask;          // [BH][n_flat][k]
  uint32_t* bits;     // [BH][n_flat][W]
  __nv_bfloat16* kc_bf;  // [BH][tn_pad][D]
  __nv_bfloat16* vc_bf;
  int* ctx_short;     // [BH]
  int4* tiles;        // [BH][items_f][max_tiles]
  int* n_tiles;       // [BH][items_f]
  int* taylor_pick;   // [BH]: 0 = row-major K7 (union tiles), 1 = transposed K7T
  float* resid;       // [BH][T][D] coarse residual rows (gamma > 0 only)
  size_t bytes;
};

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

Workspace carve(const Dims& d, int dtype, uint8_t* base) {
  Workspace w{};
  size_t off = 0;
  auto take = [&](size_t n) {
    uint8_t* p = base ? base + off : nullptr;
    off += align256(n ? n : 1);
    return p;
  };
  const long long BH = d.BH;
  w.err = reinterpret_cast<int32_t*>(take(16));
  w.means = reinterpret_cast<float*>(take(3ull * BH * d.T * d.D * 4));
  w.bf = dtype == ISA_DTYPE_F32 ? reinterpret_cast<__nv_bfloat16*>(take(3ull * BH * d.S * d.D * 2))
         : d.rope_base > 0.0     ? reinterpret_cast<__nv_bfloat16*>(take(2ull * BH * d.S * d.D * 2))
                                 : nullptr;
  w.rope_tab = d.rope_base > 0.0 ? reinterpret_cast<float2*>(take(8ull * d.S * (d.D / 2))) : nullptr;
  w.s_new = reinterpret_cast<double*>(take(8ull * BH * d.T * d.t_new));
  w.s_ctx = reinterpret_cast<double*>(take(8ull * BH * d.t_src * d.t_ctx));
  w.flags = reinterpret_cast<uint8_t*>(take((size_t)BH * (d.T > d.t_ctx ? d.T : d.t_ctx)));
  w.ctx = reinterpret_cast<double*>(take(8ull * BH * d.t_ctx));
  w.sel = reinterpret_cast<int*>(take(4ull * BH * d.k_ctx));
  w.kv_blk = reinterpret_cast<int*>(take(4ull * BH * d.t_new));
  w.sharpness = reinterpret_cast<double*>(take(8ull * BH * d.T));
  w.sharp = reinterpret_cast<int*>(take(4ull * BH * d.n_sharp));
  w.flat = reinterpret_cast<int*>(take(4ull * BH * d.n_flat));
  w.mask = reinterpret_cast<int*>(take(4ull * BH * d.n_flat * d.k));
  w.bits = reinterpret_cast<uint32_t*>(take(4ull * BH * d.n_flat * d.W));
  w.kc_bf = reinterpret_cast<__nv_bfloat16*>(take(2ull * BH * d.tn_pad * d.D));
  w.vc_bf = reinterpret_cast<__nv_bfloat16*>(take(2ull * BH * d.tn_pad * d.D));
  w.ctx_short = reinterpret_cast<int*>(take(4ull * BH));
  w.tiles = reinterpret_cast<int4*>(take(16ull * BH * d.items_f * 2 * d.max_tiles));
  w.n_tiles = reinterpret_cast<int*>(take(4ull * BH * d.items_f));
  w.resid = d.gamma > 0.0 ? reinterpret_cast<float*>(take(4ull * BH * d.T * d.D)) : nullptr;
  w.taylor_pick = reinterpret_cast<int*>(take(4ull * BH));
  w.bytes = off;
  return w;
}

unsigned grid1d(long long n, int threads) {
  long long g = (n + threads - 1) / threads;
  return static_cast<unsigned>(g < 1 ? 1 : (g > 65535 * 16 ? 65535 * 16 : g));
}

template <int D>
int launch_resid_tiled(dim3 g, const float* qc, const float* kc, const float* vc, const Dims& d, float* out,
                       cudaStream_t st) {
  if (int rc_ = ensure_smem((const void*)isa::coarse_residual_tiled_kernel<D>, isa::ResidTile<D>::kBytes)) return rc_;
  isa::coarse_residual_tiled_kernel<D><<<g, 256, isa::ResidTile<D>::kBytes, st>>>(qc, kc, vc, d.T, (float)d.scale,
                                                                                 d.resid_softmax, out);
  return ISA_OK;
}

// K6 / K8 at D = 128 run on CTA pairs (cta_group::2, isa_attn.cuh) unless
// the call sets ISA_FLAG_SINGLE_CTA (or the process sets ISA_PAIR=0): A/B.
thread_local bool g_single_cta = false;
bool pair_mode() {
  static bool env_off = [] {
    const char* e = getenv("ISA_PAIR");
    return e && e[0] == '0';
  }();
  return !env_off && !g_single_cta;
}

template <int D, int MODE>
int launch_attention(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv, const CUtensorMap& tkc,
                     const CUtensorMap& tvc, const isa::AttnParams& p, int items, int BH, cudaStream_t st) {
  using L = isa::AttnSmem<D>;
  if (items < 1) return ISA_OK;
  if constexpr (D == 128 && MODE != isa::MODE_TAYLOR) {
    if (pair_mode()) {
      if (int rc_ = ensure_smem((const void*)isa::gba_attention_pair_kernel<D, MODE>, L::kAlloc)) return rc_;
      isa::gba_attention_pair_kernel<D, MODE><<<dim3((items + 1) & ~1, BH), isa::kThreads, L::kAlloc, st>>>(
          tq, tk, tv, tkc, tvc, p);
      ISA_LAUNCHED("gba_attention_pair_kernel");
      return ISA_OK;
    }
  }
  if (int rc_ = ensure_smem((const void*)isa::gba_attention_kernel<D, MODE>, L::kAlloc)) return rc_;
  dim3 grid(items, BH);
  isa::gba_attention_kernel<D, MODE><<<grid, isa::kThreads, L::kAlloc, st>>>(tq, tk, tv, tkc, tvc, p);
  ISA_LAUNCHED("gba_attention_kernel");
  return ISA_OK;
}

template <int D>
int launch_isa_fused_t(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv, const CUtensorMap& tkc,
                       const CUtensorMap& tvc, const isa::AttnParams& pe, const isa::AttnParams& pt, int items_e,
                       int items_t, int BH, cudaStream_t st) {
  using L = isa::AttnSmem<D>;
  if (int rc_ = ensure_smem((const void*)isa::gba_isa_kernel<D>, L::kAlloc)) return rc_;
  dim3 grid(items_e + items_t, BH);
  isa::gba_isa_kernel<D><<<grid, isa::kThreads, L::kAlloc, st>>>(tq, tk, tv, tkc, tvc, pe, pt, items_e);
  ISA_LAUNCHED("gba_isa_kernel");
  return ISA_OK;
}

// Transposed Taylor kernel (isa_taylor_t.cuh, D = 128): on by default,
// ISA_TAYLOR_T=0 selects the row-major K7 (fused with K6 in one launch).
bool taylor_t_mode() {
  static bool v = [] {
    const char* e = getenv("ISA_TAYLOR_T");
    return !(e && e[0] == '0');
  }();
  return v;
}

// Taylor-branch kernel choice per head (ISA_TAYLOR_PICK): -1 = auto (plan
// statistics), 0 = always the row-major K7, 1 = always K7T.
int taylor_pick_mode() {
  static int v = [] {
    const char* e = getenv("ISA_TAYLOR_PICK");
    if (e && e[0] == '7' && e[1] == 't') return 1;
    if (e && e[0] == '7') return 0;
    return -1;
  }();
  return v;
}

// K6 + (per head) K7 or K7T items in one grid (D = 128).
int launch_isa_hybrid(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv, const CUtensorMap& tkc,
                      const CUtensorMap& tvc, const isa::AttnParams& pe, const isa::AttnParams& pt, int items_e,
                      int items_k7, const int* pick, int BH, cudaStream_t st) {
  constexpr int kA = isa::TaylorTSmem<128>::kAlloc > isa::AttnSmem<128>::kAlloc ? isa::TaylorTSmem<128>::kAlloc
                                                                                : isa::AttnSmem<128>::kAlloc;
  if (int rc_ = ensure_smem((const void*)isa::gba_isa_hybrid_kernel<128>, kA)) return rc_;
  const int items_t = (pt.n_qblk + 1) / 2;
  isa::gba_isa_hybrid_kernel<128><<<dim3(items_e + items_k7 + items_t, BH), isa::kTThreads, kA, st>>>(
      tq, tk, tv, tkc, tvc, pe, pt, items_e, items_k7, pick);
  ISA_LAUNCHED("gba_isa_hybrid_kernel");
  return ISA_OK;
}

int launch_taylor_t(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv, const CUtensorMap& tkc,
                    const CUtensorMap& tvc, const isa::AttnParams& p, int BH, cudaStream_t st) {
  using L = isa::TaylorTSmem<128>;
  if (int rc_ = ensure_smem((const void*)isa::gba_taylor_t_kernel<128>, L::kAlloc)) return rc_;
  const int items = (p.n_qblk + 1) / 2;
  if (items < 1) return ISA_OK;
  isa::gba_taylor_t_kernel<128><<<dim3(items, BH), isa::kTThreads, L::kAlloc, st>>>(tq, tk, tv, tkc, tvc, p);
  ISA_LAUNCHED("gba_taylor_t_kernel");
  return ISA_OK;
}

int launch_isa_fused(int D, const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                     const CUtensorMap& tkc, const CUtensorMap& tvc, const isa::AttnParams& pe,
                     const isa::AttnParams& pt, int items_e, int items_t, int BH, cudaStream_t st) {
  if (D == 128) return launch_isa_fused_t<128>(tq, tk, tv, tkc, tvc, pe, pt, items_e, items_t, BH, st);
  return launch_isa_fused_t<64>(tq, tk, tv, tkc, tvc, pe, pt, items_e, items_t, BH, st);
}

template <int MODE>
int launch_attention_d(int D, const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                       const CUtensorMap& tkc, const CUtensorMap& tvc, const isa::AttnParams& p, int items, int BH,
                       cudaStream_t st) {
  if (D == 128) return launch_attention<128, MODE>(tq, tk, tv, tkc, tvc, p, items, BH, st);
  return launch_attention<64, MODE>(tq, tk, tv, tkc, tvc, p, items, BH, st);
}

// Q/K/V TMA maps (bf16): either the caller's tensors (with strides) or the workspace bf16 copy.
int qkv_maps(const IsaShape* sh, const Dims& d, const void* q, const void* k, const void* v, const Workspace& w,
             CUtensorMap* tq, CUtensorMap* tk, CUtensorMap* tv) {
  const void* ptr[3] = {q, k, v};
  CUtensorMap* maps[3] = {tq, tk, tv};
  for (int i = 0; i < 3; ++i) {
    int rc;
    if (sh->dtype == ISA_DTYPE_BF16 && !(d.rope_base > 0.0 && i < 2)) {
      rc = make_map(maps[i], ptr[i], d.D, d.S, d.H, d.B, sh->stride_s * 2, sh->stride_h * 2, sh->stride_b * 2);
    } else {  // the workspace bf16 copy: fp32 inputs, or Q / K rotated by the fused RoPE
      const __nv_bfloat16* base = w.bf + (long long)i * d.BH * d.S * d.D;
      rc = make_map(maps[i], base, d.D, d.S, d.H, d.B, (long long)d.D * 2, (long long)d.S * d.D * 2,
                    (long long)d.H * d.S * d.D * 2);
    }
    if (rc) return rc;
  }
  return ISA_OK;
}

int check_io(const IsaShape* sh, const void* q, const void* k, const void* v) {
  if (!q || !k || !v) return fail(ISA_ERR_LAYOUT, "null q/k/v");
  const int elem = sh->dtype == ISA_DTYPE_BF16 ? 2 : 4;
  for (const void* p : {q, k, v})
    if (reinterpret_cast<uintptr_t>(p) & 15) return fail(ISA_ERR_LAYOUT, "q/k/v must be 16-byte aligned");
  const long long st[3] = {sh->stride_b, sh->stride_h, sh->stride_s};
  for (long long s : st)
    if ((s * elem) & 15) return fail(ISA_ERR_LAYOUT, "q/k/v strides must be multiples of 16 bytes");
  return ISA_OK;
}

// Output element strides: caller's (D contiguous) or contiguous (B,H,S,D).
void out_strides(const IsaShape* sh, const Dims& d, isa::AttnParams* p) {
  if (sh->out_stride_b || sh->out_stride_h || sh->out_stride_s) {
    p->o_sb = sh->out_stride_b;
    p->o_sh = sh->out_stride_h;
    p->o_ss = sh->out_stride_s;
  } else {
    p->o_sh = (long long)d.S * d.D;
    p->o_sb = (long long)d.H * d.S * d.D;
    p->o_ss = d.D;
  }
}

int check_out(const IsaShape* sh, const void* out) {
  const int elem = sh->dtype == ISA_DTYPE_BF16 ? 2 : 4;
  if (!out || (reinterpret_cast<uintptr_t>(out) & 15)) return fail(ISA_ERR_LAYOUT, "out must be 16-byte aligned");
  const long long st[3] = {sh->out_stride_b, sh->out_stride_h, sh->out_stride_s};
  for (long long s : st)
    if ((s * elem) & 15) return fail(ISA_ERR_LAYOUT, "out strides must be multiples of 16 bytes");
  return ISA_OK;
}

void record(const IsaEvents* ev, int i, cudaStream_t st) {
  if (ev && ev->ev[i]) cudaEventRecord(reinterpret_cast<cudaEvent_t>(ev->ev[i]), st);
}

// fp64 coarse scores, numpy einsum bits (coarse_dmma_kernel)
int launch_coarse(const float* qc, long long q_hs, const float* kc, long long k_hs, const int* kv_blk, int col0,
                  int rows, int n, int D, double scale, double* out, int BH, cudaStream_t st) {
  dim3 g((n + 63) / 64, (rows + 63) / 64, BH);
  isa::coarse_dmma_kernel<<<g, 256, 0, st>>>(qc, q_hs, kc, k_hs, kv_blk, col0, rows, n, D, scale, out);
  ISA_LAUNCHED("coarse_dmma_kernel");
  return ISA_OK;
}

int run_pool(const IsaShape* sh, const Dims& d, const void* q, const void* k, const void* v, float* means,
             __nv_bfloat16* bf, int32_t* err, cudaStream_t st, float2* rope_tab = nullptr) {
  isa::SegInfo seg{d.l_src, d.l_ctx, d.t_src, d.t_ctx};
  dim3 grid((d.T + 3) / 4, d.BH, 3);
  if (sh->dtype == ISA_DTYPE_BF16) {
    auto* qq = static_cast<const __nv_bfloat16*>(q);
    auto* kk = static_cast<const __nv_bfloat16*>(k);
    auto* vv = static_cast<const __nv_bfloat16*>(v);
    const float2* tab = nullptr;
    if (d.rope_base > 0.0) {  // fused decoupled RoPE: angle table, then rotate + pool Q / K
      const long long n = (long long)d.S * (d.D / 2);
      isa::rope_table_kernel<<<grid1d(n, 256), 256, 0, st>>>(rope_tab, d.S, d.D, d.l_src, std::log2(d.rope_base));
      ISA_LAUNCHED("rope_table_kernel");
      tab = rope_tab;
    }
    if (d.D == 128)
      isa::pool_means_kernel<__nv_bfloat16, 128><<<grid, 128, 0, st>>>(qq, kk, vv, sh->stride_b, sh->stride_h,
                                                                       sh->stride_s, d.H, seg, d.T, means, bf,
                                                                       d.S, err, tab);
    else
      isa::pool_means_kernel<__nv_bfloat16, 64><<<grid, 128, 0, st>>>(qq, kk, vv, sh->stride_b, sh->stride_h,
                                                                      sh->stride_s, d.H, seg, d.T, means, bf,
                                                                      d.S, err, tab);
  } else {
    auto* qq = static_cast<const float*>(q);
    auto* kk = static_cast<const float*>(k);
    auto* vv = static_cast<const float*>(v);
    if (d.D == 128)
      isa::pool_means_kernel<float, 128><<<grid, 128, 0, st>>>(qq, kk, vv, sh->stride_b, sh->stride_h, sh->stride_s,
                                                               d.H, seg, d.T, means, bf, d.S, err);
    else
      isa::pool_means_kernel<float, 64><<<grid, 128, 0, st>>>(qq, kk, vv, sh->stride_b, sh->stride_h, sh->stride_s,
                                                              d.H, seg, d.T, means, bf, d.S, err);
  }
  ISA_LAUNCHED("pool_means_kernel");
  return ISA_OK;
}

// Stable top-`kth` selection of each row of a (rows, n) fp64 matrix into
// ascending kept / dropped index lists (rank flags + compaction).
int select_rows(const double* vals, int rows, int n, int kth, uint8_t* flags, int* kept, int64_t* kept64,
                int* dropped, int64_t* dropped64, cudaStream_t st) {
  int rc;
  if ((rc = ensure_smem((const void*)isa::rank_flags_kernel, (size_t)n * 8))) return rc;
  if ((rc = ensure_smem((const void*)isa::compact_kernel, (size_t)n * 4))) return rc;
  isa::rank_flags_kernel<<<dim3((n + 255) / 256, rows), 256, (size_t)n * 8, st>>>(vals, n, kth, flags);
  ISA_LAUNCHED("rank_flags_kernel");
  isa::compact_kernel<<<rows, 1024, (size_t)n * 4, st>>>(flags, n, kth, kept, kept64, dropped, dropped64);
  ISA_LAUNCHED("compact_kernel");
  return ISA_OK;
}

int launch_sharpness(const double* s, long long stride, int rows, int n, int softmax_first, double* out,
                     cudaStream_t st) {
  const unsigned g = (unsigned)((rows + 7) / 8);
  if (n <= 512)
    isa::sharpness_kernel<16><<<g, 256, 0, st>>>(s, stride, rows, n, softmax_first, out);
  else if (n <= 1024)
    isa::sharpness_kernel<32><<<g, 256, 0, st>>>(s, stride, rows, n, softmax_first, out);
  else if (n <= 2048)
    isa::sharpness_kernel<64><<<g, 256, 0, st>>>(s, stride, rows, n, softmax_first, out);
  else
    return fail(ISA_ERR_CONFIG, "source blocks %d > 2048 not supported", n);
  ISA_LAUNCHED("sharpness_kernel");
  return ISA_OK;
}

int launch_mask(const double* scores, int rows, int n, const int* flat, int n_flat, int T, int k, int W,
                int* mask_idx, int64_t* mask64, uint32_t* bits, cudaStream_t st) {
  const unsigned g = (unsigned)((rows + 3) / 4);
#define ISA_MASK_THR(M)                                                                                           \
  if (n <= 32 * M) {                                                                                             \
    isa::block_mask_thr_kernel<M><<<g, 128, 0, st>>>(scores, rows, n, flat, n_flat, T, k, W, mask_idx, mask64, bits); \
    ISA_LAUNCHED("block_mask_thr_kernel");                                                                        \
    return ISA_OK;                                                                                                \
  }
  ISA_MASK_THR(4)
  ISA_MASK_THR(8)
  ISA_MASK_THR(12)
  ISA_MASK_THR(16)
  ISA_MASK_THR(20)
  ISA_MASK_THR(24)
  ISA_MASK_THR(32)
#undef ISA_MASK_THR
  const size_t sm = 4 * ((size_t)n * 8 + (size_t)W * 4);
  int rc;
  if ((rc = ensure_smem((const void*)isa::block_mask_kernel, sm))) return rc;
  isa::block_mask_kernel<<<(rows + 3) / 4, 128, sm, st>>>(scores, rows, n, flat, n_flat, T, k, W, mask_idx, mask64,
                                                          bits);
  ISA_LAUNCHED("block_mask_kernel");
  return ISA_OK;
}

// Stages 1-3 (+ routing export). Leaves sel/kv_blk/sharp/flat/mask/bits/centroids in the workspace.
int run_routing(const IsaShape* sh, const Dims& d, const IsaKnobs* kn, const void* q, const void* k, const void* v,
                const Workspace& w, const IsaRoutingIn* pinned, IsaRoutingOut* ro, int32_t* err,
                const IsaEvents* ev, cudaStream_t st) {
  int rc;
  const long long BH = d.BH;
  float* qc = w.means;
  float* kc = w.means + BH * d.T * d.D;
  float* vc = w.means + 2 * BH * d.T * d.D;
  // ---- stage 1: coarse (pooled means, context saliency)
  if ((rc = run_pool(sh, d, q, k, v, w.means, w.bf, err, st, w.rope_tab))) return rc;
  const bool need_scores = !pinned;
  if (need_scores && d.t_ctx) {
    // context saliency in the reference's order: fp64 scores of the source
    // rows against the context columns (numpy einsum bits), sequential mean
    if ((rc = launch_coarse(qc, (long long)d.T * d.D, kc, (long long)d.T * d.D, nullptr, d.t_src, d.t_src, d.t_ctx,
                            d.D, d.scale, w.s_ctx, d.BH, st)))
      return rc;
    isa::ctx_mean_kernel<<<dim3((d.t_ctx + 127) / 128, d.BH), 128, 0, st>>>(w.s_ctx, (long long)d.t_src * d.t_ctx,
                                                                          d.t_ctx, d.t_src, d.t_ctx, w.ctx);
    ISA_LAUNCHED("ctx_mean_kernel");
  }
  if (d.gamma > 0.0) {  // coarse residual rows (pipeline.py:261-267), consumed by the attention epilogues
    dim3 g((d.T + 63) / 64, d.BH);
    if ((rc = d.D == 128 ? launch_resid_tiled<128>(g, qc, kc, vc, d, w.resid, st)
                         : launch_resid_tiled<64>(g, qc, kc, vc, d, w.resid, st)))
      return rc;
    ISA_LAUNCHED("coarse_residual_tiled_kernel");
  }
  record(ev, 1, st);
  // ---- stage 2: select (context top-k, K_new block table, fp64 scores vs K_new, centroids)
  if (pinned) {
    if (d.k_ctx && !pinned->selection) return fail(ISA_ERR_CONTRACT, "pinned routing lacks selection");
    if ((d.n_sharp && !pinned->sharp) || (d.n_flat && !pinned->flat))
      return fail(ISA_ERR_CONTRACT, "pinned routing lacks split");
    if (d.n_flat && !pinned->mask) return fail(ISA_ERR_CONTRACT, "pinned routing lacks mask");
    // the reference's index contracts, reported through err (the narrowing
    // below clamps, so a bad index never addresses memory out of bounds)
    const size_t seen = 4ull * ((d.T + 31) / 32);
    if ((rc = ensure_smem((const void*)isa::routing_check_kernel, seen))) return rc;
    isa::routing_check_kernel<<<d.BH, 256, seen, st>>>(d.k_ctx ? pinned->selection : nullptr, d.k_ctx, d.t_ctx,
                                                       d.n_sharp ? pinned->sharp : nullptr, d.n_sharp,
                                                       d.n_flat ? pinned->flat : nullptr, d.n_flat, d.T,
                                                       d.n_flat ? pinned->mask : nullptr, d.k, d.t_new, err);
    ISA_LAUNCHED("routing_check_kernel");
    if (d.k_ctx) {
      isa::narrow_kernel<<<grid1d(BH * d.k_ctx, 256), 256, 0, st>>>(pinned->selection, w.sel, BH * d.k_ctx, d.t_ctx);
      ISA_LAUNCHED("narrow_kernel");
    }
  } else if (d.k_ctx) {
    if ((rc = select_rows(w.ctx, d.BH, d.t_ctx, d.k_ctx, w.flags, w.sel, ro ? ro->selection : nullptr, nullptr,
                          nullptr, st)))
      return rc;
  }
  isa::kvblk_from_sel_kernel<<<d.BH, 256, 0, st>>>(w.sel, d.t_src, d.k_ctx, d.t_ctx, d.l_ctx, w.kv_blk,
                                                   w.ctx_short);
  ISA_LAUNCHED("kvblk_from_sel_kernel");
  if (need_scores) {
    if ((rc = launch_coarse(qc, (long long)d.T * d.D, kc, (long long)d.T * d.D, w.kv_blk, 0, d.T, d.t_new, d.D,
                            d.scale, w.s_new, d.BH, st)))
      return rc;
  }
  if (d.n_flat) {
    isa::SegInfo seg{d.l_src, d.l_ctx, d.t_src, d.t_ctx};
    isa::centroid_kernel<<<dim3(d.tn_pad, d.BH), d.D, 0, st>>>(kc, vc, w.kv_blk, d.T, d.t_new, d.tn_pad, d.D, seg,
                                                                w.kc_bf, w.vc_bf, w.ctx_short);
    ISA_LAUNCHED("centroid_kernel");
  }
  if (ro && ro->ctx_scores && need_scores && d.t_ctx)
    ISA_CUDA(cudaMemcpyAsync(ro->ctx_scores, w.ctx, 8ull * BH * d.t_ctx, cudaMemcpyDeviceToDevice, st));
  if (ro && ro->selection && pinned && d.k_ctx)
    ISA_CUDA(cudaMemcpyAsync(ro->selection, pinned->selection, 8ull * BH * d.k_ctx, cudaMemcpyDeviceToDevice, st));
  record(ev, 2, st);
  // ---- stage 3: split + block mask
  if (pinned) {
    if (d.n_sharp) {
      isa::narrow_kernel<<<grid1d(BH * d.n_sharp, 256), 256, 0, st>>>(pinned->sharp, w.sharp, BH * d.n_sharp, d.T);
      ISA_LAUNCHED("narrow_kernel");
    }
    if (d.n_flat) {
      isa::narrow_kernel<<<grid1d(BH * d.n_flat, 256), 256, 0, st>>>(pinned->flat, w.flat, BH * d.n_flat, d.T);
      ISA_LAUNCHED("narrow_kernel");
      isa::narrow_kernel<<<grid1d(BH * d.n_flat * d.k, 256), 256, 0, st>>>(pinned->mask, w.mask,
                                                                         BH * d.n_flat * d.k, d.t_new);
      ISA_LAUNCHED("narrow_kernel");
      isa::bits_from_mask_kernel<<<BH * d.n_flat, 128, 0, st>>>(w.mask, d.k, d.W, w.bits);
      ISA_LAUNCHED("bits_from_mask_kernel");
    }
  } else {
    if ((rc = launch_sharpness(w.s_new, d.t_new, (int)(BH * d.T), d.t_src, kn->softmax_first, w.sharpness, st)))
      return rc;
    if ((rc = select_rows(w.sharpness, d.BH, d.T, d.n_sharp, w.flags, w.sharp, ro ? ro->sharp : nullptr, w.flat,
                          ro ? ro->flat : nullptr, st)))
      return rc;
    if (ro && ro->sharpness)
      ISA_CUDA(cudaMemcpyAsync(ro->sharpness, w.sharpness, 8ull * BH * d.T, cudaMemcpyDeviceToDevice, st));
    if (d.n_flat) {
      if ((rc = launch_mask(w.s_new, (int)(BH * d.n_flat), d.t_new, w.flat, d.n_flat, d.T, d.k, d.W, w.mask,
                            ro ? ro->mask : nullptr, w.bits, st)))
        return rc;
    }
  }
  if (pinned && ro) {
    if (ro->sharp && d.n_sharp)
      ISA_CUDA(cudaMemcpyAsync(ro->sharp, pinned->sharp, 8ull * BH * d.n_sharp, cudaMemcpyDeviceToDevice, st));
    if (ro->flat && d.n_flat)
      ISA_CUDA(cudaMemcpyAsync(ro->flat, pinned->flat, 8ull * BH * d.n_flat, cudaMemcpyDeviceToDevice, st));
    if (ro->mask && d.n_flat)
      ISA_CUDA(cudaMemcpyAsync(ro->mask, pinned->mask, 8ull * BH * d.n_flat * d.k, cudaMemcpyDeviceToDevice, st));
  }
  if (d.n_flat) {
    isa::taylor_plan_kernel<<<dim3(d.items_f, d.BH), 64, 0, st>>>(w.bits, d.n_flat, d.W, d.items_f, d.max_tiles,
                                                                   w.kv_blk, d.t_new, d.t_src, d.l_src, d.l_ctx,
                                                                   w.tiles, w.n_tiles);
    ISA_LAUNCHED("taylor_plan_kernel");
    const int pick = (kn->flags & ISA_FLAG_TAYLOR_K7) ? 0 : (kn->flags & ISA_FLAG_TAYLOR_K7T) ? 1 : taylor_pick_mode();
    isa::taylor_pick_kernel<<<d.BH, 128, 0, st>>>(w.n_tiles, d.items_f, d.n_flat, d.k, pick,
                                                  w.taylor_pick);
    ISA_LAUNCHED("taylor_pick_kernel");
  }
  record(ev, 3, st);
  return ISA_OK;
}

// ---------------------------------------------------------------- host-streamed execution
// isa_forward_host: Q/K/V/out live in host memory. The flattened (b, h) range
// is cut into chunks of `hc` heads; each chunk is an independent (1, hc, S, D)
// problem (every stage is per head: reference.py:159-160, taylor.py:176-177).
// Three streams overlap the PCIe traffic with the pipeline: H2D of chunk c+1
// (streams[1]) and D2H of chunk c-1 (streams[2]) run under the pipeline of
// chunk c (streams[0]). Device staging holds kSlots chunks of 3 inputs + 1
// output, recycled through events.
constexpr int kHostSlots = 2;

struct HostPlan {
  Dims d;            // whole problem
  int hc, n_chunks;  // heads per chunk, chunks
  size_t elem, chunk_bytes, stage_bytes, ws_bytes;
};

IsaShape chunk_shape(const IsaShape* sh, int heads) {
  IsaShape c = *sh;
  c.batch = 1;
  c.heads = heads;
  c.stride_s = sh->head_dim;
  c.stride_h = (long long)sh->seq_len * sh->head_dim;
  c.stride_b = c.stride_h * heads;
  c.out_stride_b = c.out_stride_h = c.out_stride_s = 0;
  return c;
}

int host_plan(const IsaShape* sh, const IsaKnobs* kn, int heads_per_chunk, HostPlan* hp) {
  int rc = derive(sh, kn, &hp->d);
  if (rc) return rc;
  const Dims& d = hp->d;
  const long long sd = (long long)d.S * d.D;
  if (sh->stride_s != d.D || sh->stride_h != sd || sh->stride_b != sd * d.H)
    return fail(ISA_ERR_LAYOUT, "host-streamed q/k/v must be contiguous (B,H,S,D)");
  // default chunk: ~150 MB of inputs (measured at cfg3: 3 heads = 150 MB gives
  // 40.7 ms e2e vs 43.0 with B*H/8 = 5 heads; the first H2D and the last
  // pipeline + D2H are the exposed parts)
  const double head_in = 3.0 * sd * (sh->dtype == ISA_DTYPE_BF16 ? 2 : 4);
  int hc = heads_per_chunk > 0 ? heads_per_chunk : (int)(150e6 / head_in + 0.5);
  if (hc > d.BH) hc = d.BH;
  if (hc < 1) hc = 1;
  hp->hc = hc;
  hp->n_chunks = (d.BH + hc - 1) / hc;
  hp->elem = sh->dtype == ISA_DTYPE_BF16 ? 2 : 4;
  hp->chunk_bytes = align256((size_t)hc * sd * hp->elem);
  hp->stage_bytes = (size_t)kHostSlots * 4 * hp->chunk_bytes;
  IsaShape cs = chunk_shape(sh, hc);
  Dims cd;
  if ((rc = derive(&cs, kn, &cd))) return rc;
  hp->ws_bytes = carve(cd, sh->dtype, nullptr).bytes;
  return ISA_OK;
}

// Per-thread, per-device event ring (created on first use; timing disabled).
constexpr int kMaxDevices = 16;
cudaEvent_t* host_events() {
  thread_local cudaEvent_t ev[kMaxDevices][3 * kHostSlots + 1] = {};
  thread_local bool made[kMaxDevices] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return nullptr;
  if (!made[dev]) {
    for (auto& e : ev[dev])
      if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return nullptr;
    made[dev] = true;
  }
  return ev[dev];
}

}  // namespace

extern "C" {

int isa_abi_version(void) { return ISA_ABI_VERSION; }

int isa_last_launch_count(void) { return g_launches; }

const char* isa_last_error(void) { return g_last_error.c_str(); }

int isa_workspace_bytes(const IsaShape* shape, const IsaKnobs* knobs, size_t* bytes) {
  Dims d;
  int rc = derive(shape, knobs, &d);
  if (rc) return rc;
  if (!bytes) return fail(ISA_ERR_CONFIG, "null bytes");
  *bytes = carve(d, shape->dtype, nullptr).bytes;
  return ISA_OK;
}

int isa_routing(const IsaShape* shape, const IsaKnobs* knobs, const void* q, const void* k, const void* v,
                void* workspace, size_t workspace_bytes, IsaRoutingOut* routing, int32_t* err_word, void* stream) {
  g_launches = 0;
  Dims d;
  int rc = derive(shape, knobs, &d);
  if (rc) return rc;
  if ((rc = check_io(shape, q, k, v))) return rc;
  Workspace w = carve(d, shape->dtype, static_cast<uint8_t*>(workspace));
  if (!workspace || workspace_bytes < w.bytes)
    return fail(ISA_ERR_CONFIG, "workspace too small (%zu < %zu)", workspace_bytes, w.bytes);
  return run_routing(shape, d, knobs, q, k, v, w, nullptr, routing, err_word, nullptr,
                     static_cast<cudaStream_t>(stream));
}

}  // extern "C"

namespace {

// Stages 1-5 into `out`; `lse` (nullable, [BH][S] fp32) receives the per-row
// log2-domain softmax normaliser for the backward.
int forward_impl(const IsaShape* shape, const IsaKnobs* knobs, const Dims& d, const void* q, const void* k,
                 const void* v, void* out, const Workspace& w, const IsaRoutingIn* pinned, IsaRoutingOut* routing,
                 int32_t* err_word, const IsaEvents* events, float* lse, cudaStream_t st,
                 int32_t* head_done = nullptr, int32_t* done_inc = nullptr) {
  int rc;
  g_single_cta = (knobs->flags & ISA_FLAG_SINGLE_CTA) != 0;
  record(events, 0, st);
  if ((rc = run_routing(shape, d, knobs, q, k, v, w, pinned, routing, err_word, events, st))) return rc;
  // ---- stage 4 (+ fused stage 5)
  CUtensorMap tq, tk, tv, tkc, tvc;
  if ((rc = qkv_maps(shape, d, q, k, v, w, &tq, &tk, &tv))) return rc;
  isa::AttnParams p{};
  p.H = d.H;
  p.l_src = d.l_src;
  p.l_ctx = d.l_ctx;
  p.t_src = d.t_src;
  p.t_ctx = d.t_ctx;
  p.t_new = d.t_new;
  p.scale_log2 = static_cast<float>(d.scale * 1.4426950408889634);
  p.kv_blk = w.kv_blk;
  p.out = out;
  p.out_fp32 = shape->dtype == ISA_DTYPE_F32;
  out_strides(shape, d, &p);
  p.err_flag = err_word;
  p.resid = w.resid;  // null unless gamma > 0
  p.gamma = static_cast<float>(d.gamma);
  p.T = d.T;
  p.lse = lse;
  p.S = d.S;
  isa::AttnParams ps = p;
  ps.n_qblk = d.n_sharp;
  ps.qlist = w.sharp;
  ps.ctx_short_j = w.ctx_short;
  isa::AttnParams pf = p;
  if (d.n_flat) {
    if ((rc = make_map(&tkc, w.kc_bf, d.D, d.tn_pad, d.BH, 1, (long long)d.D * 2, (long long)d.tn_pad * d.D * 2,
                       (long long)d.BH * d.tn_pad * d.D * 2)))
      return rc;
    if ((rc = make_map(&tvc, w.vc_bf, d.D, d.tn_pad, d.BH, 1, (long long)d.D * 2, (long long)d.tn_pad * d.D * 2,
                       (long long)d.BH * d.tn_pad * d.D * 2)))
      return rc;
    pf.n_qblk = d.n_flat;
    pf.qlist = w.flat;
    pf.tiles = w.tiles;
    pf.n_tiles = w.n_tiles;
    pf.n_items = d.items_f;
    pf.max_tiles = d.max_tiles;
    pf.member_bits = w.bits;
    pf.W = d.W;
    pf.ctx_short_j = w.ctx_short;
    pf.tn_pad = d.tn_pad;
    pf.mask = w.mask;
    pf.kmask = d.k;
  }
  const bool taylor_t = d.n_flat && d.D == 128 && taylor_t_mode();
  const bool fuse = d.n_sharp && d.n_flat && !taylor_t && !(knobs->flags & ISA_FLAG_SEPARATE_BRANCHES);
  if (taylor_t && (knobs->flags & ISA_FLAG_FUSED_GRID)) {
    // K6 + Taylor items in one grid (the short Taylor CTAs fill the tail of
    // the last K6 wave); per head the Taylor branch runs as K7T or, when the
    // paired exact lists overlap enough that the union tiles cost less, K7
    ps.head_done = head_done;  // in-kernel per-head completion (every CTA of the grid counts)
    if (done_inc) *done_inc = d.items_s + d.items_f + (pf.n_qblk + 1) / 2;
    if ((rc = launch_isa_hybrid(tq, tk, tv, tkc, tvc, ps, pf, d.items_s, d.items_f, w.taylor_pick, d.BH, st)))
      return rc;
    head_done = nullptr;
    record(events, 4, st);
  } else if (taylor_t) {
    // Shipped (D = 128): K6 over the sharp blocks, then one grid of Taylor
    // items run per head as K7T or K7 (taylor_pick_kernel). Two launches beat
    // the single K6 + Taylor grid at cfg3 in an alternating same-clock loop
    // (22.15 vs 23.12 ms): K6 runs alone at full tensor rate, the L2-bound
    // Taylor items no longer contend with it. Both grids count per-head
    // completion when signalling (isa_forward_signal).
    ps.head_done = head_done;
    pf.head_done = head_done;
    const int k6_ctas = d.n_sharp ? (pair_mode() ? (d.items_s + 1) & ~1 : d.items_s) : 0;  // CTAs of the K6 grid
    if (done_inc) *done_inc = k6_ctas + d.items_f + (pf.n_qblk + 1) / 2;
    if (d.n_sharp)
      if ((rc = launch_attention_d<isa::MODE_EXACT>(d.D, tq, tk, tv, tq, tq, ps, d.items_s, d.BH, st))) return rc;
    record(events, 4, st);
    if ((rc = launch_isa_hybrid(tq, tk, tv, tkc, tvc, pf, pf, 0, d.items_f, w.taylor_pick, d.BH, st))) return rc;
    head_done = nullptr;
  } else if (fuse) {
    // K6 + K7 in one grid: exact items first, Taylor items fill the tail.
    if ((rc = launch_isa_fused(d.D, tq, tk, tv, tkc, tvc, ps, pf, d.items_s, d.items_f, d.BH, st))) return rc;
    record(events, 4, st);
  } else {
    if (d.n_sharp)
      if ((rc = launch_attention_d<isa::MODE_EXACT>(d.D, tq, tk, tv, tq, tq, ps, d.items_s, d.BH, st))) return rc;
    record(events, 4, st);
    if (d.n_flat)
      if ((rc = launch_attention_d<isa::MODE_TAYLOR>(d.D, tq, tk, tv, tkc, tvc, pf, d.items_f, d.BH, st)))
        return rc;
  }
  record(events, 5, st);
  if (head_done) {  // separate launches: one stream-ordered increment per head after them
    isa::head_bump_kernel<<<grid1d(d.BH, 128), 128, 0, st>>>(head_done, d.BH);
    ISA_LAUNCHED("head_bump_kernel");
    if (done_inc) *done_inc = 1;
  }
  if (routing && routing->taylor_kernel) {  // which Taylor-branch kernel ran per head (test hook)
    if (taylor_t) {
      ISA_CUDA(cudaMemcpyAsync(routing->taylor_kernel, w.taylor_pick, 4ull * d.BH, cudaMemcpyDeviceToDevice, st));
    } else {
      isa::fill_i32_kernel<<<grid1d(d.BH, 256), 256, 0, st>>>(routing->taylor_kernel, taylor_t ? 1 : 0, d.BH);
      ISA_LAUNCHED("fill_i32_kernel");
    }
  }
  return ISA_OK;
}

// Backward workspace: forward workspace, then O (bf16), lse, rho, dkc, dvc.
struct BwdWs {
  Workspace fw;
  __nv_bfloat16* o;
  float *lse, *rho, *dkc, *dvc;
  float *g_doc, *g_stats, *g_dqc, *g_dkc, *g_dvc;  // gamma residual (gamma > 0 only)
  size_t bytes;
};

// Centroid dK/dV kernel: split the flat query list over gridDim.z so the grid
// covers ~4 CTAs per SM (tn_pad/64 centroid tiles x BH is only 360 CTAs at
// cfg3), keeping >= 16 query blocks per split. ISA_BWD_CSPLIT=n overrides.
int centroid_splits(const Dims& d) {
  if (!d.n_flat) return 1;
  static int forced = [] {
    const char* e = getenv("ISA_BWD_CSPLIT");
    return e ? atoi(e) : 0;
  }();
  const int tiles = (d.tn_pad / 128) * d.BH;  // centroid CTAs per split (128 centroids each)
  int s = forced > 0 ? forced : (4 * 148 + tiles - 1) / tiles;
  const int cap = d.n_flat / 16 > 1 ? d.n_flat / 16 : 1;
  if (s > cap) s = cap;
  if (s > 16) s = 16;
  return s < 1 ? 1 : s;
}

BwdWs carve_bwd(const Dims& d0, uint8_t* base) {
  BwdWs b{};
  Dims d = d0;
  d.gamma = 0.0;  // the forward recompute runs without the residual (rho uses the attention output)
  b.fw = carve(d, ISA_DTYPE_BF16, base);
  size_t off = b.fw.bytes;
  auto take = [&](size_t n) {
    uint8_t* p = base ? base + off : nullptr;
    off += align256(n ? n : 1);
    return p;
  };
  const long long BH = d.BH;
  b.o = reinterpret_cast<__nv_bfloat16*>(take(2ull * BH * d.S * d.D));
  b.lse = reinterpret_cast<float*>(take(4ull * BH * d.S));
  b.rho = reinterpret_cast<float*>(take(4ull * BH * d.S));
  const int cs = centroid_splits(d);
  b.dkc = reinterpret_cast<float*>(take(4ull * cs * BH * d.t_new * d.D));
  b.dvc = reinterpret_cast<float*>(take(4ull * cs * BH * d.t_new * d.D));
  if (d0.gamma > 0.0) {
    b.g_doc = reinterpret_cast<float*>(take(4ull * BH * d.T * d.D));
    b.g_stats = reinterpret_cast<float*>(take(12ull * BH * d.T));
    b.g_dqc = reinterpret_cast<float*>(take(4ull * BH * d.T * d.D));
    b.g_dkc = reinterpret_cast<float*>(take(4ull * BH * d.T * d.D));
    b.g_dvc = reinterpret_cast<float*>(take(4ull * BH * d.T * d.D));
  }
  b.bytes = off;
  return b;
}

template <int D>
int launch_bwd(const isa::BwdParams& bp, const Dims& d, const CUtensorMap* maps, const Workspace& w,
               cudaStream_t st) {
  using TL = isa::BwdTcSmem<D>;
  const int n_list = d.n_sharp + d.n_flat;
  const size_t sm_tc = TL::bytes(n_list);
  isa::BwdTcParams tp{bp, n_list};
  int rc;
  CUtensorMap tkc = maps[0], tvc = maps[0];  // centroid maps (unused without flat blocks)
  if (d.n_flat) {
    if ((rc = make_map(&tkc, w.kc_bf, d.D, d.tn_pad, d.BH, 1, (long long)d.D * 2, (long long)d.tn_pad * d.D * 2,
                       (long long)d.BH * d.tn_pad * d.D * 2)))
      return rc;
    if ((rc = make_map(&tvc, w.vc_bf, d.D, d.tn_pad, d.BH, 1, (long long)d.D * 2, (long long)d.tn_pad * d.D * 2,
                       (long long)d.BH * d.tn_pad * d.D * 2)))
      return rc;
    // centroid adjoint (taylor.py:286-289): 128 centroids per CTA, flat list split over gridDim.z
    const int cs = bp.c_splits;
    if ((rc = ensure_smem((const void*)isa::bwd_dkv_tc_kernel<D, true>, sm_tc))) return rc;
    isa::bwd_dkv_tc_kernel<D, true><<<dim3(d.tn_pad / 128, d.BH, cs), 320, sm_tc, st>>>(maps[0], tkc, tvc, maps[3],
                                                                                         tp);
    ISA_LAUNCHED("bwd_dkv_tc_kernel<centroid>");
    if (cs > 1) {
      isa::bwd_centroid_reduce_kernel<<<grid1d(bp.c_part, 256), 256, 0, st>>>(bp.dkc, bp.dvc, bp.c_part, cs);
      ISA_LAUNCHED("bwd_centroid_reduce_kernel");
    }
  }
  if ((rc = ensure_smem((const void*)isa::bwd_dkv_tc_kernel<D, false>, sm_tc))) return rc;
  isa::bwd_dkv_tc_kernel<D, false><<<dim3((d.t_new + 1) / 2, d.BH), 320, sm_tc, st>>>(maps[0], maps[1], maps[2],
                                                                                        maps[3], tp);
  ISA_LAUNCHED("bwd_dkv_tc_kernel");
  {
    using QL = isa::BwdDqSmem<D>;
    const int n_sp = (d.n_sharp + 1) / 2;  // sharp pairs (128 query rows each)
    int x0 = 0;
    if constexpr (D == 128) {
      using PL = isa::BwdDqPairLayout<D>;
      // sharp pairs on CTA pairs (same K_new stream), flat pairs below; the per-block
      // valid-row table must fit next to the operand rings (t_new <= ~8K blocks)
      if (d.n_sharp && pair_mode() && PL::bytes(d.t_new) <= 232448) {
        const size_t bytes = PL::bytes(d.t_new);
        if ((rc = ensure_smem((const void*)isa::bwd_dq_pair_kernel<D>, bytes))) return rc;
        isa::bwd_dq_pair_kernel<D><<<dim3((n_sp + 1) & ~1, d.BH), 320, bytes, st>>>(maps[0], maps[1], maps[2], maps[3],
                                                                                   bp);
        ISA_LAUNCHED("bwd_dq_pair_kernel");
        x0 = n_sp;
      }
    }
    const int grid_x = n_sp - x0 + 2 * d.items_f;
    if (grid_x > 0) {
      if ((rc = ensure_smem((const void*)isa::bwd_dq_tc_kernel<D>, QL::kBytes))) return rc;
      isa::bwd_dq_tc_kernel<D><<<dim3(grid_x, d.BH), 320, QL::kBytes, st>>>(
          maps[0], maps[1], maps[2], maps[3], tkc, tvc, bp, w.tiles, w.n_tiles, d.items_f, d.max_tiles, x0);
      ISA_LAUNCHED("bwd_dq_tc_kernel");
    }
  }
  return ISA_OK;
}

}  // namespace

extern "C" {

int isa_forward(const IsaShape* shape, const IsaKnobs* knobs, const void* q, const void* k, const void* v, void* out,
                void* workspace, size_t workspace_bytes, const IsaRoutingIn* pinned, IsaRoutingOut* routing,
                int32_t* err_word, const IsaEvents* events, void* stream) {
  g_launches = 0;
  Dims d;
  int rc = derive(shape, knobs, &d);
  if (rc) return rc;
  if ((rc = check_io(shape, q, k, v))) return rc;
  if ((rc = check_out(shape, out))) return rc;
  Workspace w = carve(d, shape->dtype, static_cast<uint8_t*>(workspace));
  if (!workspace || workspace_bytes < w.bytes)
    return fail(ISA_ERR_CONFIG, "workspace too small (%zu < %zu)", workspace_bytes, w.bytes);
  return forward_impl(shape, knobs, d, q, k, v, out, w, pinned, routing, err_word, events, nullptr,
                      static_cast<cudaStream_t>(stream));
}

int isa_forward_signal(const IsaShape* shape, const IsaKnobs* knobs, const void* q, const void* k, const void* v,
                       void* out, void* workspace, size_t workspace_bytes, int32_t* err_word, int32_t* head_done,
                       int32_t* done_inc, void* stream) {
  g_launches = 0;
  if (!head_done || !done_inc) return fail(ISA_ERR_CONFIG, "isa_forward_signal needs head_done and done_inc");
  Dims d;
  int rc = derive(shape, knobs, &d);
  if (rc) return rc;
  if ((rc = check_io(shape, q, k, v))) return rc;
  if ((rc = check_out(shape, out))) return rc;
  Workspace w = carve(d, shape->dtype, static_cast<uint8_t*>(workspace));
  if (!workspace || workspace_bytes < w.bytes)
    return fail(ISA_ERR_CONFIG, "workspace too small (%zu < %zu)", workspace_bytes, w.bytes);
  return forward_impl(shape, knobs, d, q, k, v, out, w, nullptr, nullptr, err_word, nullptr, nullptr,
                      static_cast<cudaStream_t>(stream), head_done, done_inc);
}

int isa_stream_wait_geq(void* stream, const int32_t* addr, int32_t value) {
  using WaitFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
  static WaitFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<WaitFn>(p);
  });
  if (!fn) return fail(ISA_ERR_CUDA, "cuStreamWaitValue32 unavailable");
  // GEQ on a monotonically growing counter: no reset between steps, so a
  // wait can never be satisfied by an earlier step's completions
  CUresult r = fn(static_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(addr), (cuuint32_t)value,
                  CU_STREAM_WAIT_VALUE_GEQ);
  if (r != CUDA_SUCCESS) return fail(ISA_ERR_CUDA, "cuStreamWaitValue32 failed (%d)", (int)r);
  return ISA_OK;
}

int isa_backward_workspace_bytes(const IsaShape* shape, const IsaKnobs* knobs, size_t* bytes) {
  Dims d;
  int rc = derive(shape, knobs, &d);
  if (rc) return rc;
  if (!bytes) return fail(ISA_ERR_CONFIG, "null bytes");
  *bytes = carve_bwd(d, nullptr).bytes;
  return ISA_OK;
}

int isa_backward(const IsaShape* shape, const IsaKnobs* knobs, const void* q, const void* k, const void* v,
                 const void* dout, float* dq, float* dk, float* dv, void* workspace, size_t workspace_bytes,
                 const IsaRoutingIn* pinned, int32_t* err_word, void* stream) {
  g_launches = 0;
  Dims d;
  int rc = derive(shape, knobs, &d);
  if (rc) return rc;
  if (shape->dtype != ISA_DTYPE_BF16) return fail(ISA_ERR_CONFIG, "isa_backward takes bf16 q/k/v/dO");
  if ((rc = check_io(shape, q, k, v))) return rc;
  if ((rc = check_io(shape, dout, dout, dout))) return rc;
  if (!dq || !dk || !dv) return fail(ISA_ERR_LAYOUT, "null gradient buffers");
  BwdWs b = carve_bwd(d, static_cast<uint8_t*>(workspace));
  if (!workspace || workspace_bytes < b.bytes)
    return fail(ISA_ERR_CONFIG, "workspace too small (%zu < %zu)", workspace_bytes, b.bytes);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // forward recompute with the softmax statistics (routing frozen by determinism or `pinned`);
  // without the gamma residual: rho must see the attention output alone (taylor.py:274)
  IsaShape os = *shape;
  os.out_stride_b = os.out_stride_h = os.out_stride_s = 0;  // O into the workspace, contiguous
  IsaKnobs kf = *knobs;
  kf.gamma = 0.0;
  Dims df = d;
  df.gamma = 0.0;
  if ((rc = forward_impl(&os, &kf, df, q, k, v, b.o, b.fw, pinned, nullptr, err_word, nullptr, b.lse, st)))
    return rc;
  int launches = g_launches;
  // rows of unselected context blocks get no gradient: zero the context rows of every head
  // (the dK/dV epilogue writes every source row and every selected context row)
  if (d.l_ctx) {
    const size_t pitch = 4ull * d.S * d.D, width = 4ull * d.l_ctx * d.D;
    ISA_CUDA(cudaMemset2DAsync(static_cast<float*>(dk) + (size_t)d.l_src * d.D, pitch, 0, width, d.BH, st));
    ISA_CUDA(cudaMemset2DAsync(static_cast<float*>(dv) + (size_t)d.l_src * d.D, pitch, 0, width, d.BH, st));
  }
  const long long n_rows = (long long)d.BH * d.S;
  isa::bwd_rho_kernel<<<grid1d(n_rows * (d.D / 8), 256), 256, 0, st>>>(
      static_cast<const __nv_bfloat16*>(dout), shape->stride_b, shape->stride_h, shape->stride_s, b.o, d.H, d.S, d.D,
      b.rho, n_rows);
  ++launches;
  ISA_CUDA(cudaGetLastError());
  isa::BwdParams bp{};
  bp.H = d.H;
  bp.S = d.S;
  bp.D = d.D;
  bp.l_src = d.l_src;
  bp.l_ctx = d.l_ctx;
  bp.t_src = d.t_src;
  bp.t_ctx = d.t_ctx;
  bp.t_new = d.t_new;
  bp.n_sharp = d.n_sharp;
  bp.n_flat = d.n_flat;
  bp.k = d.k;
  bp.W = d.W;
  bp.tn_pad = d.tn_pad;
  bp.sl2 = static_cast<float>(d.scale * 1.4426950408889634);
  bp.scale = static_cast<float>(d.scale);
  bp.q = static_cast<const __nv_bfloat16*>(q);
  bp.kx = static_cast<const __nv_bfloat16*>(k);
  bp.v = static_cast<const __nv_bfloat16*>(v);
  bp.dout = static_cast<const __nv_bfloat16*>(dout);
  bp.sb = shape->stride_b;
  bp.sh = shape->stride_h;
  bp.ss = shape->stride_s;
  bp.db = shape->stride_b;
  bp.dh = shape->stride_h;
  bp.ds = shape->stride_s;
  bp.lse = b.lse;
  bp.rho = b.rho;
  bp.sharp = b.fw.sharp;
  bp.flat = b.fw.flat;
  bp.mask = b.fw.mask;
  bp.kv_blk = b.fw.kv_blk;
  bp.bits = b.fw.bits;
  bp.kc = b.fw.kc_bf;
  bp.vc = b.fw.vc_bf;
  bp.dkc = b.dkc;
  bp.dvc = b.dvc;
  bp.c_splits = centroid_splits(d);
  bp.c_part = (long long)d.BH * d.t_new * d.D;
  bp.dq = dq;
  bp.dk = dk;
  bp.dv = dv;
  CUtensorMap maps[4];  // q, k, v, dO (bf16, the shape's strides)
  const void* srcs[4] = {q, k, v, dout};
  for (int i = 0; i < 4; ++i)
    if ((rc = make_map(&maps[i], srcs[i], d.D, d.S, d.H, d.B, shape->stride_s * 2, shape->stride_h * 2,
                       shape->stride_b * 2)))
      return rc;
  g_launches = 0;
  rc = d.D == 128 ? launch_bwd<128>(bp, d, maps, b.fw, st) : launch_bwd<64>(bp, d, maps, b.fw, st);
  g_launches += launches;
  if (rc || !(d.gamma > 0.0)) return rc;
  // gamma coarse residual (pipeline.py:435-452) on the block means of the recompute
  isa::GammaBwdParams gp{};
  gp.H = d.H;
  gp.S = d.S;
  gp.D = d.D;
  gp.T = d.T;
  gp.t_src = d.t_src;
  gp.l_src = d.l_src;
  gp.l_ctx = d.l_ctx;
  gp.gamma = static_cast<float>(d.gamma);
  gp.scale = static_cast<float>(d.scale);
  gp.softmax = d.resid_softmax;
  gp.dout = static_cast<const __nv_bfloat16*>(dout);
  gp.db = shape->stride_b;
  gp.dh = shape->stride_h;
  gp.ds = shape->stride_s;
  gp.qc = b.fw.means;
  gp.kc = b.fw.means + (long long)d.BH * d.T * d.D;
  gp.vc = b.fw.means + 2ll * d.BH * d.T * d.D;
  gp.doc = b.g_doc;
  gp.m = b.g_stats;
  gp.l = b.g_stats + (long long)d.BH * d.T;
  gp.rho = b.g_stats + 2ll * d.BH * d.T;
  gp.dqc = b.g_dqc;
  gp.dkc = b.g_dkc;
  gp.dvc = b.g_dvc;
  gp.dq = dq;
  gp.dk = dk;
  gp.dv = dv;
  isa::gamma_doc_kernel<<<dim3(d.T, d.BH), d.D, 0, st>>>(gp);
  ISA_LAUNCHED("gamma_doc_kernel");
  isa::gamma_row_kernel<<<dim3((d.T + 3) / 4, d.BH), 128, 0, st>>>(gp);
  ISA_LAUNCHED("gamma_row_kernel");
  isa::gamma_col_kernel<<<dim3((d.T + 3) / 4, d.BH), 128, 0, st>>>(gp);
  ISA_LAUNCHED("gamma_col_kernel");
  isa::gamma_spread_kernel<<<dim3(d.T, d.BH), d.D, 0, st>>>(gp);
  ISA_LAUNCHED("gamma_spread_kernel");
  return ISA_OK;
}

int isa_dense_attention(const IsaShape* shape, double scale, const void* q, const void* k, const void* v, void* out,
                        void* stream) {
  g_launches = 0;
  IsaKnobs kn{scale, 0, 0, 1, 1, 0};
  Dims d;
  int rc = derive(shape, &kn, &d);
  if (rc) return rc;
  if (shape->dtype != ISA_DTYPE_BF16) return fail(ISA_ERR_CONFIG, "dense attention takes bf16 inputs");
  if ((rc = check_io(shape, q, k, v))) return rc;
  Workspace w{};
  CUtensorMap tq, tk, tv;
  if ((rc = qkv_maps(shape, d, q, k, v, w, &tq, &tk, &tv))) return rc;
  isa::AttnParams p{};
  p.H = d.H;
  p.l_src = d.l_src;
  p.l_ctx = d.l_ctx;
  p.t_src = d.t_src;
  p.t_ctx = d.t_ctx;
  p.t_new = d.T;
  p.n_qblk = d.T;
  p.scale_log2 = static_cast<float>(scale * 1.4426950408889634);
  p.out = out;
  p.out_fp32 = 0;
  out_strides(shape, d, &p);
  return launch_attention_d<isa::MODE_DENSE>(d.D, tq, tk, tv, tq, tq, p, (d.T + 3) / 4, d.BH,
                                             static_cast<cudaStream_t>(stream));
}

// ---------------------------------------------------------------- dense attention, S_q != S_k
// full_attention / online_softmax_attention (reference.py:79-170) for a
// query length different from the key length, on the K8 (DENSE) kernel. The
// kernel's two-segment geometry carries both sides: segment 1 = the t_q query
// blocks (l_src = S_q, a multiple of 64, so key block j sits at row 64j in
// either segment), segment 2 length S_k - S_q, so key block j's valid rows
// are min(64, S_k - 64j) for j >= t_q. Hence either S_k is a multiple of 64
// or t_k > t_q (the ragged block must lie in segment 2).
int isa_cross_attention(const IsaShape* q_shape, int32_t k_len, const int64_t* k_strides, double scale,
                        const void* q, const void* k, const void* v, void* out, void* stream) {
  g_launches = 0;
  const IsaShape* sh = q_shape;
  if (!sh || !k_strides) return fail(ISA_ERR_CONFIG, "null shape/strides");
  if (sh->head_dim != 64 && sh->head_dim != 128)
    return fail(ISA_ERR_CONFIG, "head_dim=%d not supported (64 or 128)", sh->head_dim);
  if (sh->dtype != ISA_DTYPE_BF16) return fail(ISA_ERR_CONFIG, "dense attention takes bf16 inputs");
  if (sh->batch < 1 || sh->heads < 1 || sh->seq_len < 1 || k_len < 1)
    return fail(ISA_ERR_LAYOUT, "all dims must be >= 1");
  if (sh->seq_len % 64) return fail(ISA_ERR_LAYOUT, "query length %d must be a multiple of 64", sh->seq_len);
  const int t_q = sh->seq_len / 64, t_k = (k_len + 63) / 64;
  if ((k_len % 64) && t_k <= t_q)
    return fail(ISA_ERR_LAYOUT, "a ragged key length needs more key blocks (%d) than query blocks (%d)", t_k, t_q);
  if (!(scale > 0.0)) return fail(ISA_ERR_CONFIG, "scale must be > 0");
  if (!q || !k || !v) return fail(ISA_ERR_CONFIG, "null operand");
  int rc;
  if ((rc = check_out(sh, out))) return rc;
  Dims d{};
  d.B = sh->batch;
  d.H = sh->heads;
  d.S = sh->seq_len;
  d.D = sh->head_dim;
  d.BH = d.B * d.H;
  CUtensorMap tq, tk, tv;
  if ((rc = make_map(&tq, q, d.D, d.S, d.H, d.B, sh->stride_s * 2, sh->stride_h * 2, sh->stride_b * 2))) return rc;
  if ((rc = make_map(&tk, k, d.D, k_len, d.H, d.B, k_strides[2] * 2, k_strides[1] * 2, k_strides[0] * 2))) return rc;
  if ((rc = make_map(&tv, v, d.D, k_len, d.H, d.B, k_strides[2] * 2, k_strides[1] * 2, k_strides[0] * 2))) return rc;
  isa::AttnParams p{};
  p.H = d.H;
  p.l_src = d.S;
  p.t_src = t_q;
  p.l_ctx = k_len - d.S;  // only read for key blocks j >= t_q, i.e. when k_len > S_q
  p.t_ctx = t_k > t_q ? t_k - t_q : 0;
  p.t_new = t_k;
  p.n_qblk = t_q;
  p.scale_log2 = static_cast<float>(scale * 1.4426950408889634);
  p.out = out;
  p.out_fp32 = 0;
  out_strides(sh, d, &p);
  return launch_attention_d<isa::MODE_DENSE>(d.D, tq, tk, tv, tq, tq, p, (t_q + 3) / 4, d.BH,
                                             static_cast<cudaStream_t>(stream));
}

// ---------------------------------------------------------------- standalone Taylor kernel
// taylor_sparse_forward (taylor.py:163-194): every query block of q is flat,
// its exact K_new blocks are the caller's mask rows, the centroids the
// caller's kc/vc. Same K7 kernel as the pipeline: identity block table over
// k (K_new = k), flat list 0..t_q-1, member words from the mask, the Taylor
// work plan, kc/vc rounded to the bf16 centroid rows. The query geometry goes
// in the attention params (l_src = S_q), the key geometry in the plan
// (l_src = S_k); full 64-row blocks on both sides.
struct TaylorWs {
  int *kv_blk, *flat, *mask, *ctx_short, *n_tiles;
  uint32_t* bits;
  __nv_bfloat16 *kc_bf, *vc_bf;
  int4* tiles;
  size_t bytes;
};

int taylor_dims(const IsaShape* sh, int k_len, int k_mask, Dims* d) {
  if (!sh) return fail(ISA_ERR_CONFIG, "null shape");
  if (sh->block != 64) return fail(ISA_ERR_CONFIG, "block_size=%d not supported (only 64)", sh->block);
  if (sh->head_dim != 64 && sh->head_dim != 128)
    return fail(ISA_ERR_CONFIG, "head_dim=%d not supported (64 or 128)", sh->head_dim);
  if (sh->dtype != ISA_DTYPE_BF16) return fail(ISA_ERR_CONFIG, "the standalone Taylor kernel takes bf16 q/k/v");
  if (sh->batch < 1 || sh->heads < 1 || sh->seq_len < 1 || k_len < 1)
    return fail(ISA_ERR_LAYOUT, "all dims must be >= 1");
  if (sh->seq_len % 64) return fail(ISA_ERR_LAYOUT, "query length %d not divisible by block size 64", sh->seq_len);
  if (k_len % 64) return fail(ISA_ERR_LAYOUT, "key length %d not divisible by block size 64", k_len);
  *d = Dims{};
  d->B = sh->batch;
  d->H = sh->heads;
  d->S = sh->seq_len;
  d->D = sh->head_dim;
  d->BH = d->B * d->H;
  d->l_src = sh->seq_len;
  d->t_src = d->T = d->n_flat = sh->seq_len / 64;
  d->t_new = k_len / 64;
  d->k = k_mask;
  if (k_mask < 1 || k_mask > d->t_new)
    return fail(ISA_ERR_CONTRACT, "mask width %d out of [1, %d]", k_mask, d->t_new);
  d->tn_pad = ((d->t_new + 127) / 128) * 128;
  d->W = d->tn_pad / 32;
  if (d->W > 128) return fail(ISA_ERR_CONFIG, "%d key blocks exceed the Taylor kernel's limit (4096)", d->t_new);
  d->items_f = (d->n_flat + 3) / 4;
  const int u = 2 * d->k < d->t_new ? 2 * d->k : d->t_new;
  d->max_tiles = (u + 1) / 2;
  return ISA_OK;
}

TaylorWs carve_taylor(const Dims& d, uint8_t* base) {
  TaylorWs w{};
  size_t off = 0;
  auto take = [&](size_t n) {
    uint8_t* p = base ? base + off : nullptr;
    off += align256(n ? n : 1);
    return p;
  };
  const long long BH = d.BH;
  w.kv_blk = reinterpret_cast<int*>(take(4ull * BH * d.t_new));
  w.flat = reinterpret_cast<int*>(take(4ull * BH * d.n_flat));
  w.mask = reinterpret_cast<int*>(take(4ull * BH * d.n_flat * d.k));
  w.bits = reinterpret_cast<uint32_t*>(take(4ull * BH * d.n_flat * d.W));
  w.kc_bf = reinterpret_cast<__nv_bfloat16*>(take(2ull * BH * d.tn_pad * d.D));
  w.vc_bf = reinterpret_cast<__nv_bfloat16*>(take(2ull * BH * d.tn_pad * d.D));
  w.ctx_short = reinterpret_cast<int*>(take(4ull * BH));
  w.tiles = reinterpret_cast<int4*>(take(16ull * BH * d.items_f * 2 * d.max_tiles));
  w.n_tiles = reinterpret_cast<int*>(take(4ull * BH * d.items_f));
  w.bytes = off;
  return w;
}

int isa_taylor_workspace_bytes(const IsaShape* q_shape, int32_t k_len, int32_t k_mask, size_t* bytes) {
  Dims d;
  int rc = taylor_dims(q_shape, k_len, k_mask, &d);
  if (rc) return rc;
  if (!bytes) return fail(ISA_ERR_CONFIG, "null bytes");
  *bytes = carve_taylor(d, nullptr).bytes;
  return ISA_OK;
}

int isa_taylor_forward(const IsaShape* q_shape, int32_t k_len, const int64_t* k_strides, int32_t k_mask,
                       double scale, const void* q, const void* k, const void* v, const float* kc, const float* vc,
                       const int64_t* mask, void* out, void* workspace, size_t workspace_bytes, int32_t* err_word,
                       void* stream) {
  g_launches = 0;
  Dims d;
  int rc = taylor_dims(q_shape, k_len, k_mask, &d);
  if (rc) return rc;
  if (!(scale > 0.0)) return fail(ISA_ERR_CONFIG, "scale must be > 0");
  if (!q || !k || !v || !kc || !vc || !mask || !k_strides) return fail(ISA_ERR_CONFIG, "null operand");
  if ((rc = check_out(q_shape, out))) return rc;
  TaylorWs w = carve_taylor(d, static_cast<uint8_t*>(workspace));
  if (!workspace || workspace_bytes < w.bytes)
    return fail(ISA_ERR_CONFIG, "workspace too small (%zu < %zu)", workspace_bytes, w.bytes);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const long long BH = d.BH;
  // identity K_new table (ctx_short = -1), flat list 0..t_q-1, member words
  isa::kvblk_from_sel_kernel<<<d.BH, 256, 0, st>>>(nullptr, d.t_new, 0, 0, 0, w.kv_blk, w.ctx_short);
  ISA_LAUNCHED("kvblk_from_sel_kernel");
  isa::iota_rows_kernel<<<grid1d(BH * d.n_flat, 256), 256, 0, st>>>(w.flat, d.n_flat, BH * d.n_flat);
  ISA_LAUNCHED("iota_rows_kernel");
  isa::narrow_kernel<<<grid1d(BH * d.n_flat * d.k, 256), 256, 0, st>>>(mask, w.mask, BH * d.n_flat * d.k, d.t_new);
  ISA_LAUNCHED("narrow_kernel");
  isa::bits_from_mask_kernel<<<BH * d.n_flat, 128, 0, st>>>(w.mask, d.k, d.W, w.bits);
  ISA_LAUNCHED("bits_from_mask_kernel");
  isa::SegInfo seg{k_len, 0, d.t_new, 0};
  isa::centroid_kernel<<<dim3(d.tn_pad, d.BH), d.D, 0, st>>>(kc, vc, w.kv_blk, d.t_new, d.t_new, d.tn_pad, d.D, seg,
                                                              w.kc_bf, w.vc_bf, w.ctx_short);
  ISA_LAUNCHED("centroid_kernel");
  isa::taylor_plan_kernel<<<dim3(d.items_f, d.BH), 64, 0, st>>>(w.bits, d.n_flat, d.W, d.items_f, d.max_tiles,
                                                                 w.kv_blk, d.t_new, d.t_new, k_len, 0, w.tiles,
                                                                 w.n_tiles);
  ISA_LAUNCHED("taylor_plan_kernel");
  CUtensorMap tq, tk, tv, tkc, tvc;
  const IsaShape* sh = q_shape;
  if ((rc = make_map(&tq, q, d.D, d.S, d.H, d.B, sh->stride_s * 2, sh->stride_h * 2, sh->stride_b * 2))) return rc;
  if ((rc = make_map(&tk, k, d.D, k_len, d.H, d.B, k_strides[2] * 2, k_strides[1] * 2, k_strides[0] * 2))) return rc;
  if ((rc = make_map(&tv, v, d.D, k_len, d.H, d.B, k_strides[2] * 2, k_strides[1] * 2, k_strides[0] * 2))) return rc;
  const long long cr = (long long)d.D * 2, ch = (long long)d.tn_pad * d.D * 2;
  if ((rc = make_map(&tkc, w.kc_bf, d.D, d.tn_pad, d.BH, 1, cr, ch, BH * ch))) return rc;
  if ((rc = make_map(&tvc, w.vc_bf, d.D, d.tn_pad, d.BH, 1, cr, ch, BH * ch))) return rc;
  isa::AttnParams p{};
  p.H = d.H;
  p.l_src = d.S;  // query geometry: one segment of t_q full blocks
  p.t_src = d.t_src;
  p.t_new = d.t_new;
  p.scale_log2 = static_cast<float>(scale * 1.4426950408889634);
  p.kv_blk = w.kv_blk;
  p.out = out;
  p.out_fp32 = 0;
  out_strides(sh, d, &p);
  p.err_flag = err_word;
  p.T = d.T;
  p.S = d.S;
  p.n_qblk = d.n_flat;
  p.qlist = w.flat;
  p.tiles = w.tiles;
  p.n_tiles = w.n_tiles;
  p.n_items = d.items_f;
  p.max_tiles = d.max_tiles;
  p.member_bits = w.bits;
  p.W = d.W;
  p.ctx_short_j = w.ctx_short;
  p.tn_pad = d.tn_pad;
  p.mask = w.mask;
  p.kmask = d.k;
  if (d.D == 128 && taylor_t_mode()) return launch_taylor_t(tq, tk, tv, tkc, tvc, p, d.BH, st);
  return launch_attention_d<isa::MODE_TAYLOR>(d.D, tq, tk, tv, tkc, tvc, p, d.items_f, d.BH, st);
}

int isa_decoupled_rope(const IsaShape* shape, double base, const void* x, void* out, void* stream) {
  g_launches = 0;
  if (!shape) return fail(ISA_ERR_CONFIG, "null shape");
  const IsaShape* sh = shape;
  if (sh->batch < 1 || sh->heads < 1 || sh->seq_len < 1 || sh->head_dim < 8 || sh->head_dim % 8)
    return fail(ISA_ERR_CONFIG, "decoupled rope needs D a multiple of 8, got D=%d", sh->head_dim);
  if (sh->l_src < 0 || sh->l_ctx < 0 || sh->l_src + sh->l_ctx != sh->seq_len)
    return fail(ISA_ERR_LAYOUT, "sequence length %d != icl total %d", sh->seq_len, sh->l_src + sh->l_ctx);
  if (!(base > 0.0)) return fail(ISA_ERR_CONFIG, "rope base must be > 0");
  if (sh->dtype != ISA_DTYPE_BF16 && sh->dtype != ISA_DTYPE_F32) return fail(ISA_ERR_CONFIG, "bad dtype");
  int rc;
  if ((rc = check_io(sh, x, x, x))) return rc;
  if ((rc = check_out(sh, out))) return rc;
  const long long D = sh->head_dim, S = sh->seq_len, H = sh->heads;
  const long long ob = sh->out_stride_b ? sh->out_stride_b : H * S * D;
  const long long oh = sh->out_stride_h ? sh->out_stride_h : S * D;
  const long long os = sh->out_stride_s ? sh->out_stride_s : D;
  const long long n = S * (D / 8);
  const unsigned grid = static_cast<unsigned>((n + 255) / 256);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const double lb = std::log2(base);
  if (sh->dtype == ISA_DTYPE_BF16)
    isa::decoupled_rope_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>(
        static_cast<const __nv_bfloat16*>(x), static_cast<__nv_bfloat16*>(out), sh->batch, sh->heads, sh->seq_len,
        sh->head_dim, sh->l_src, sh->stride_b, sh->stride_h, sh->stride_s, ob, oh, os, lb);
  else
    isa::decoupled_rope_kernel<float><<<grid, 256, 0, st>>>(static_cast<const float*>(x), static_cast<float*>(out),
                                                           sh->batch, sh->heads, sh->seq_len, sh->head_dim,
                                                           sh->l_src, sh->stride_b, sh->stride_h, sh->stride_s, ob,
                                                           oh, os, lb);
  ISA_LAUNCHED("decoupled_rope_kernel");
  return ISA_OK;
}

int isa_pool_means(const IsaShape* shape, const void* q, const void* k, const void* v, float* means,
                   int32_t* err_word, void* stream) {
  IsaKnobs kn{1.0, 0, 0, 1, 1, 0};
  Dims d;
  int rc = derive(shape, &kn, &d);
  if (rc) return rc;
  if ((rc = check_io(shape, q, k, v))) return rc;
  return run_pool(shape, d, q, k, v, means, nullptr, err_word, static_cast<cudaStream_t>(stream));
}

int isa_topk_rows_f64(const double* scores, int32_t rows, int32_t n, int32_t k, int64_t* out_idx, int32_t method,
                      void* stream) {
  g_launches = 0;
  if (rows < 0 || n < 1 || k < 0 || k > n) return fail(ISA_ERR_CONFIG, "bad topk geometry");
  if (rows == 0 || k == 0) return ISA_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (method == 0) {
    uint8_t* flags = nullptr;
    ISA_CUDA(cudaMallocAsync(&flags, (size_t)rows * n, st));
    int rc = select_rows(scores, rows, n, k, flags, nullptr, out_idx, nullptr, nullptr, st);
    cudaFreeAsync(flags, st);
    return rc;
  }
  const int W = (n + 31) / 32;
  if (method == 2) {  // generic arg-max-rounds kernel (n > 1024 path)
    const size_t sm = 4 * ((size_t)n * 8 + (size_t)W * 4);
    int rc;
    if ((rc = ensure_smem((const void*)isa::block_mask_kernel, sm))) return rc;
    isa::block_mask_kernel<<<(rows + 3) / 4, 128, sm, st>>>(scores, rows, n, nullptr, 1, 0, k, W, nullptr, out_idx,
                                                            nullptr);
    ISA_LAUNCHED("block_mask_kernel");
    return ISA_OK;
  }
  return launch_mask(scores, rows, n, nullptr, 1, 0, k, W, nullptr, out_idx, nullptr, st);
}

int isa_sharpness_rows_f64(const double* s, int32_t rows, int32_t n, int32_t softmax_first, double* out,
                           void* stream) {
  g_launches = 0;
  if (rows < 0 || n < 1) return fail(ISA_ERR_CONFIG, "bad sharpness geometry");
  if (rows == 0) return ISA_OK;
  return launch_sharpness(s, n, rows, n, softmax_first, out, static_cast<cudaStream_t>(stream));
}

int isa_split_rows_f64(const double* m, int32_t rows, int32_t n, int32_t n_flat, int64_t* sharp, int64_t* flat,
                       void* stream) {
  g_launches = 0;
  if (rows < 0 || n < 1 || n_flat < 0 || n_flat > n) return fail(ISA_ERR_CONFIG, "bad split geometry");
  if (rows == 0) return ISA_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint8_t* flags = nullptr;
  ISA_CUDA(cudaMallocAsync(&flags, (size_t)rows * n, st));
  int rc = select_rows(m, rows, n, n - n_flat, flags, nullptr, sharp, nullptr, flat, st);
  cudaFreeAsync(flags, st);
  return rc;
}

int isa_coarse_scores(int32_t bh, int32_t t_q, int32_t t_k, int32_t d, double scale, const float* qc,
                      const float* kc, double* s, void* stream) {
  g_launches = 0;
  if (bh < 0 || t_q < 0 || t_k < 0 || d < 8 || d % 8) return fail(ISA_ERR_CONFIG, "bad coarse geometry (d %% 8 != 0?)");
  if (!bh || !t_q || !t_k) return ISA_OK;
  if (!qc || !kc || !s || (reinterpret_cast<uintptr_t>(qc) & 15) || (reinterpret_cast<uintptr_t>(kc) & 15))
    return fail(ISA_ERR_LAYOUT, "qc/kc must be 16-byte aligned");
  return launch_coarse(qc, (long long)t_q * d, kc, (long long)t_k * d, nullptr, 0, t_q, t_k, d, scale, s, bh,
                       static_cast<cudaStream_t>(stream));
}

int isa_ctx_saliency_f64(const double* s, int32_t bh, int64_t head_stride, int64_t row_stride, int32_t n_src,
                         int32_t n_ctx, double* out, void* stream) {
  g_launches = 0;
  if (bh < 0 || n_src < 1 || n_ctx < 0) return fail(ISA_ERR_CONFIG, "bad saliency geometry");
  if (!bh || !n_ctx) return ISA_OK;
  isa::ctx_mean_kernel<<<dim3((n_ctx + 127) / 128, bh), 128, 0, static_cast<cudaStream_t>(stream)>>>(
      s + n_src, head_stride, row_stride, n_src, n_ctx, out);
  ISA_LAUNCHED("ctx_mean_kernel");
  return ISA_OK;
}

int isa_forward_host_bytes(const IsaShape* shape, const IsaKnobs* knobs, int32_t heads_per_chunk,
                           size_t* stage_bytes, size_t* workspace_bytes) {
  HostPlan hp;
  int rc = host_plan(shape, knobs, heads_per_chunk, &hp);
  if (rc) return rc;
  if (!stage_bytes || !workspace_bytes) return fail(ISA_ERR_CONFIG, "null byte counts");
  *stage_bytes = hp.stage_bytes;
  *workspace_bytes = hp.ws_bytes;
  return ISA_OK;
}

int isa_forward_host(const IsaShape* shape, const IsaKnobs* knobs, const void* q_host, const void* k_host,
                     const void* v_host, void* out_host, int32_t heads_per_chunk, void* stage, size_t stage_bytes,
                     void* workspace, size_t workspace_bytes, const IsaRoutingIn* pinned, IsaRoutingOut* routing,
                     int32_t* err_word, void* const* streams) {
  HostPlan hp;
  int rc = host_plan(shape, knobs, heads_per_chunk, &hp);
  if (rc) return rc;
  if (!q_host || !k_host || !v_host || !out_host) return fail(ISA_ERR_LAYOUT, "null host q/k/v/out");
  if (!stage || stage_bytes < hp.stage_bytes)
    return fail(ISA_ERR_CONFIG, "staging buffer too small (%zu < %zu)", stage_bytes, hp.stage_bytes);
  if (!workspace || workspace_bytes < hp.ws_bytes)
    return fail(ISA_ERR_CONFIG, "workspace too small (%zu < %zu)", workspace_bytes, hp.ws_bytes);
  if (!streams) return fail(ISA_ERR_CONFIG, "null streams");
  cudaStream_t s_comp = static_cast<cudaStream_t>(streams[0]);
  cudaStream_t s_in = static_cast<cudaStream_t>(streams[1]);
  cudaStream_t s_out = static_cast<cudaStream_t>(streams[2]);
  cudaEvent_t* ev = host_events();
  if (!ev) return fail(ISA_ERR_CUDA, "cudaEventCreate failed");
  cudaEvent_t* in_done = ev;                 // [slot] inputs resident
  cudaEvent_t* comp_done = ev + kHostSlots;  // [slot] pipeline finished (inputs free, output ready)
  cudaEvent_t* out_done = ev + 2 * kHostSlots;  // [slot] output copied back (output slot free)
  cudaEvent_t start = ev[3 * kHostSlots];
  // the copy streams must not run ahead of work already queued on the caller's stream
  ISA_CUDA(cudaEventRecord(start, s_comp));
  ISA_CUDA(cudaStreamWaitEvent(s_in, start, 0));
  ISA_CUDA(cudaStreamWaitEvent(s_out, start, 0));
  const Dims& d = hp.d;
  const size_t head_bytes = (size_t)d.S * d.D * hp.elem;
  const uint8_t* src[3] = {static_cast<const uint8_t*>(q_host), static_cast<const uint8_t*>(k_host),
                           static_cast<const uint8_t*>(v_host)};
  int launches = 0;
  for (int c = 0; c < hp.n_chunks; ++c) {
    const int slot = c % kHostSlots;
    const int bh0 = c * hp.hc;
    const int nh = d.BH - bh0 < hp.hc ? d.BH - bh0 : hp.hc;
    uint8_t* base = static_cast<uint8_t*>(stage) + (size_t)slot * 4 * hp.chunk_bytes;
    uint8_t* dq = base;
    uint8_t* dout = base + 3 * hp.chunk_bytes;
    // H2D: the slot's inputs are free once the pipeline two chunks back is done
    if (c >= kHostSlots) ISA_CUDA(cudaStreamWaitEvent(s_in, comp_done[slot], 0));
    for (int t = 0; t < 3; ++t)
      ISA_CUDA(cudaMemcpyAsync(dq + t * hp.chunk_bytes, src[t] + bh0 * head_bytes, nh * head_bytes,
                               cudaMemcpyHostToDevice, s_in));
    ISA_CUDA(cudaEventRecord(in_done[slot], s_in));
    // pipeline on the chunk; its output slot is free once its last D2H finished
    ISA_CUDA(cudaStreamWaitEvent(s_comp, in_done[slot], 0));
    if (c >= kHostSlots) ISA_CUDA(cudaStreamWaitEvent(s_comp, out_done[slot], 0));
    IsaShape cs = chunk_shape(shape, nh);
    IsaRoutingOut ro{};
    if (routing) {
      ro.selection = routing->selection ? routing->selection + (long long)bh0 * d.k_ctx : nullptr;
      ro.sharp = routing->sharp ? routing->sharp + (long long)bh0 * d.n_sharp : nullptr;
      ro.flat = routing->flat ? routing->flat + (long long)bh0 * d.n_flat : nullptr;
      ro.mask = routing->mask ? routing->mask + (long long)bh0 * d.n_flat * d.k : nullptr;
      ro.sharpness = routing->sharpness ? routing->sharpness + (long long)bh0 * d.T : nullptr;
      ro.ctx_scores = routing->ctx_scores ? routing->ctx_scores + (long long)bh0 * d.t_ctx : nullptr;
      ro.taylor_kernel = routing->taylor_kernel ? routing->taylor_kernel + bh0 : nullptr;
    }
    IsaRoutingIn pi{};
    if (pinned) {
      pi.selection = pinned->selection ? pinned->selection + (long long)bh0 * d.k_ctx : nullptr;
      pi.sharp = pinned->sharp ? pinned->sharp + (long long)bh0 * d.n_sharp : nullptr;
      pi.flat = pinned->flat ? pinned->flat + (long long)bh0 * d.n_flat : nullptr;
      pi.mask = pinned->mask ? pinned->mask + (long long)bh0 * d.n_flat * d.k : nullptr;
    }
    rc = isa_forward(&cs, knobs, dq, dq + hp.chunk_bytes, dq + 2 * hp.chunk_bytes, dout, workspace,
                     workspace_bytes, pinned ? &pi : nullptr, routing ? &ro : nullptr, err_word, nullptr, s_comp);
    if (rc) return rc;
    launches += g_launches;
    ISA_CUDA(cudaEventRecord(comp_done[slot], s_comp));
    // D2H of the chunk's output
    ISA_CUDA(cudaStreamWaitEvent(s_out, comp_done[slot], 0));
    ISA_CUDA(cudaMemcpyAsync(static_cast<uint8_t*>(out_host) + bh0 * head_bytes, dout, nh * head_bytes,
                             cudaMemcpyDeviceToHost, s_out));
    ISA_CUDA(cudaEventRecord(out_done[slot], s_out));
  }
  // join: the caller's stream completes only after the last D2H
  ISA_CUDA(cudaStreamWaitEvent(s_comp, out_done[(hp.n_chunks - 1) % kHostSlots], 0));
  g_launches = launches;
  return ISA_OK;
}

#ifdef ISA_TRACE
// Debug build only (not in the header): copy the timeline stamps to host.
int isa_debug_count_copy(void* host, int reset) {
  ISA_CUDA(cudaMemcpyFromSymbol(host, isa::g_isa_count, sizeof(isa::g_isa_count)));
  if (reset) {
    static const unsigned long long z[3][4] = {};
    ISA_CUDA(cudaMemcpyToSymbol(isa::g_isa_count, z, sizeof(z)));
  }
  return ISA_OK;
}
int isa_debug_trace_copy(void* host, size_t bytes) {
  ISA_CUDA(cudaMemcpyFromSymbol(host, isa::g_isa_trace, bytes < sizeof(isa::g_isa_trace) ? bytes : sizeof(isa::g_isa_trace)));
  return ISA_OK;
}
int isa_debug_cta_copy(void* host, size_t bytes) {
  ISA_CUDA(cudaMemcpyFromSymbol(host, isa::g_isa_cta, bytes < sizeof(isa::g_isa_cta) ? bytes : sizeof(isa::g_isa_cta)));
  return ISA_OK;
}
#endif

}  // extern "C"
