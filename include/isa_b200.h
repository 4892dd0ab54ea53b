/*
 * isa_b200.h — C ABI of the B200 (sm_100a) ISA forward operator.
 *
 * This is the drop-in boundary for the reference operator
 *   isa_forward(q, k, v, icl, cfg, collect_trace=True) -> (out, IsaTrace)
 *     /root/reference/pkg/src/isattn/pipeline.py:307-316
 * and its routing hooks
 *   isa_routing(q, k, v, icl, cfg) -> IsaRouting            pipeline.py:302-304
 *   isa_forward_with_routing(q, k, v, icl, cfg, routing)     pipeline.py:319-328
 * The reference is pure Python/numpy with no FFI of its own; the Python host
 * layer (paper_2605_04569_b200/pipeline.py) binds these symbols with ctypes
 * exactly as INTEGRATION.md shows a maintainer would.
 *
 * Conventions: plain C types only; every pointer to tensor data is a CUDA
 * device pointer (except the host-streamed isa_forward_host, whose q/k/v/out
 * are host pointers); every call is asynchronous and ordered on `stream`; the
 * caller owns all buffers (inputs, outputs, workspace, routing arrays); no
 * hidden allocations (isa_forward_host keeps a per-thread ring of 5 CUDA
 * events) and no host synchronisation. Thread-safe for distinct
 * streams/workspaces. Every entry point returns an IsaStatus; on failure
 * isa_last_error() (thread-local) describes it. Status codes map 1:1 onto the
 * reference exception classes (errors.py:4-37).
 */
#ifndef ISA_B200_H
#define ISA_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ISA_ABI_VERSION 4

typedef enum IsaStatus {
  ISA_OK = 0,
  ISA_ERR_LAYOUT = 1,         /* LayoutError         errors.py:8  */
  ISA_ERR_CONFIG = 2,         /* ConfigError         errors.py:24 */
  ISA_ERR_NUMERIC = 3,        /* NumericError        errors.py:36 */
  ISA_ERR_FORMAT = 4,         /* FormatError (reserved) errors.py:28 */
  ISA_ERR_CONTRACT = 5,       /* ContractError       errors.py:20 */
  ISA_ERR_BLOCK_INDEX = 6,    /* BlockIndexError     errors.py:16 */
  ISA_ERR_INPUT = 7,          /* InputError          errors.py:12 */
  ISA_ERR_DEGENERATE_ROW = 8, /* DegenerateRowError  errors.py:32 */
  ISA_ERR_CUDA = 9            /* launch / driver failure          */
} IsaStatus;

typedef enum IsaDtype { ISA_DTYPE_BF16 = 0, ISA_DTYPE_F32 = 1 } IsaDtype;

/* Geometry of Q/K/V (B,H,S,D) and the IclLayout (tensor.py:78-93). Q, K and V
 * share shape and element strides; the D stride must be 1. `out` is written
 * in the input dtype with the out_stride_* element strides (D contiguous; all
 * zero = contiguous (B,H,S,D)), e.g. straight into a (B,S,H*D) activation. */
typedef struct IsaShape {
  int32_t batch, heads, seq_len, head_dim;
  int32_t l_src, l_ctx;  /* source tokens first, then context */
  int32_t block;         /* b (only 64 is implemented) */
  int32_t dtype;         /* IsaDtype of q, k, v and out */
  int64_t stride_b, stride_h, stride_s; /* element strides of q, k, v */
  int64_t out_stride_b, out_stride_h, out_stride_s; /* element strides of out; all 0 = contiguous (B,H,S,D) */
} IsaShape;

/* Host-derived integers, computed by the caller with the reference's float
 * expressions: k_ctx = floor(alpha_s*T_ctx) (coarse.py:156), n_flat =
 * floor(alpha_f*T) (coarse.py:197), k_mask = min(t_new, max(1,
 * floor(alpha_ns*t_new))) (coarse.py:169). */
typedef struct IsaKnobs {
  double scale;          /* cfg.scale or 1/sqrt(D) (pipeline.py:154) */
  int32_t k_ctx;
  int32_t n_flat;
  int32_t k_mask;
  int32_t softmax_first; /* coarse.py:194 */
  int32_t flags;         /* ISA_FLAG_* bits, 0 = defaults */
  double gamma;          /* coarse residual weight, 0 = off (pipeline.py:354-356) */
  int32_t residual_softmax; /* residual weights: 1 softmax(S_coarse), 0 raw Qc.Kc (pipeline.py:261-267) */
  int32_t reserved;      /* 0 */
  double rope_base;      /* > 0: apply decoupled RoPE (pipeline.py:469-490) to Q and K inside the pooling
                            pass (bf16 inputs; same bits as isa_decoupled_rope then isa_forward); 0 = off */
} IsaKnobs;

/* IsaKnobs.flags: launch the exact (sharp) and Taylor (flat) attention
 * branches as two kernels (the default at D = 128; at D = 64 it replaces the
 * fused K6 + K7 grid). */
#define ISA_FLAG_SEPARATE_BRANCHES 1
/* D = 128: the sharp and flat items in ONE grid (gba_isa_hybrid_kernel)
 * instead of the default K6 launch + Taylor launch (A/B measurements). */
#define ISA_FLAG_FUSED_GRID 8
/* D = 128: run K6 on single CTAs instead of CTA pairs (cta_group::2; A/B). */
#define ISA_FLAG_SINGLE_CTA 16
/* Force the D = 128 Taylor-branch kernel for every head instead of the
 * per-head automatic choice (taylor_pick_kernel): K7 = row-major pair-union
 * tiles, K7T = transposed per-block tiles. Same operator, test/A-B hooks. */
#define ISA_FLAG_TAYLOR_K7 2
#define ISA_FLAG_TAYLOR_K7T 4

/* Optional routing export (device pointers; any may be NULL). */
typedef struct IsaRoutingOut {
  int64_t* selection;  /* (B,H,k_ctx)      SelectionIndex.indices coarse.py:56 */
  int64_t* sharp;      /* (B,H,n_sharp)    SharpnessSplit.sharp   coarse.py:95 */
  int64_t* flat;       /* (B,H,n_flat)     SharpnessSplit.flat    coarse.py:96 */
  int64_t* mask;       /* (B,H,n_flat,k)   BlockMask.indices      coarse.py:76 */
  double* sharpness;   /* (B,H,T)          SharpnessSplit.sharpness coarse.py:97 */
  double* ctx_scores;  /* (B,H,T_ctx)      context saliency s_coarse[:, :, :T_src, T_src:].mean(2)
                          (coarse.py:155), bit-identical to numpy */
  int32_t* taylor_kernel; /* (B,H) Taylor-branch kernel run per head (D = 128): 0 = row-major K7
                             (pair-union tiles), 1 = transposed K7T; written by isa_forward only */
} IsaRoutingOut;

/* err_word bits (device int32, OR-ed by the kernels; the caller zeroes it
 * and reads it after the stream completes). Pinned-routing checks follow the
 * reference's index contracts (tensor.py:120-133, taylor.py:80-84). */
#define ISA_ERRBIT_INPUT 1u          /* non-finite Q/K/V          -> InputError */
#define ISA_ERRBIT_DEGENERATE 2u     /* row with an empty key set -> DegenerateRowError */
#define ISA_ERRBIT_SEL_RANGE 4u      /* pinned selection out of [0, T_ctx)       -> BlockIndexError */
#define ISA_ERRBIT_SEL_ORDER 8u      /* pinned selection not strictly ascending  -> ContractError */
#define ISA_ERRBIT_SPLIT_RANGE 16u   /* pinned sharp/flat out of [0, T)          -> BlockIndexError */
#define ISA_ERRBIT_SPLIT_ORDER 32u   /* sharp/flat not ascending or not a partition of [0, T) -> ContractError */
#define ISA_ERRBIT_MASK 64u          /* pinned mask out of [0, t_new) or not ascending -> ContractError */

/* Pinned routing for isa_forward_with_routing (device int64, all required
 * except mask when n_flat == 0). */
typedef struct IsaRoutingIn {
  const int64_t* selection;
  const int64_t* sharp;
  const int64_t* flat;
  const int64_t* mask;
} IsaRoutingIn;

/* Optional per-stage CUDA events (cudaEvent_t handles cast to void*):
 * ev[0] start, ev[1] after stage 1 "coarse", ev[2] after stage 2 "select",
 * ev[3] after stage 3 "split", ev[4] after the exact (sharp) attention kernel,
 * ev[5] after the Taylor (flat) kernel (pipeline.py:157-348; stage 5
 * "reconstruct" is fused into the stage-4 epilogues). NULL entries skip. */
typedef struct IsaEvents {
  void* ev[6];
} IsaEvents;

int isa_abi_version(void);
const char* isa_last_error(void);

/* Number of kernels the calling thread's last isa_forward / isa_routing /
 * isa_dense_attention call launched (thread-local; for launch accounting). */
int isa_last_launch_count(void);

/* Workspace needed by isa_forward / isa_routing for this geometry. */
int isa_workspace_bytes(const IsaShape* shape, const IsaKnobs* knobs, size_t* bytes);

/* Full pipeline (stages 1-5). `pinned` == NULL computes routing on device,
 * otherwise uses it (isa_forward_with_routing). `routing` may be NULL.
 * `err_word` (device int32, may be NULL) receives ISA_ERRBIT_* bits; the
 * caller zeroes it beforehand and reads it after the stream completes.
 * `stream` is a cudaStream_t. */
int isa_forward(const IsaShape* shape, const IsaKnobs* knobs, const void* q, const void* k, const void* v,
                void* out, void* workspace, size_t workspace_bytes, const IsaRoutingIn* pinned,
                IsaRoutingOut* routing, int32_t* err_word, const IsaEvents* events, void* stream);

/* isa_forward (computed routing, no trace) that also publishes per-head
 * completion for multi-GPU overlap: head_done (device int32 [B*H], zeroed
 * once by the caller, never reset) grows by *done_inc per call for every
 * head, the increments landing as that head's output rows become final (the
 * fused attention grid counts its CTAs per head in-kernel). A comm stream
 * then waits with isa_stream_wait_geq(comm, head_done + h, calls * inc)
 * before moving head h (parallel.py). *done_inc is written on the host. */
int isa_forward_signal(const IsaShape* shape, const IsaKnobs* knobs, const void* q, const void* k, const void* v,
                       void* out, void* workspace, size_t workspace_bytes, int32_t* err_word, int32_t* head_done,
                       int32_t* done_inc, void* stream);

/* Stream-ordered wait until *addr >= value (cuStreamWaitValue32 GEQ). */
int isa_stream_wait_geq(void* stream, const int32_t* addr, int32_t value);

/* Host-streamed pipeline: q/k/v/out are HOST pointers (contiguous (B,H,S,D);
 * page-locked for copy/compute overlap). The flattened (b,h) range is processed
 * in chunks of `heads_per_chunk` heads (<= 0: about 150 MB of inputs); the H2D copy of
 * chunk c+1 (streams[1]) and the D2H copy of chunk c-1 (streams[2]) overlap the
 * device pipeline of chunk c (streams[0]). streams[0] completes after the last
 * D2H. `stage` (device, caller-owned) and `workspace` are sized by
 * isa_forward_host_bytes. `pinned`/`routing` are device arrays for all B*H
 * heads, as in isa_forward. Same operator as isa_forward (pipeline.py:307-328):
 * heads are independent (reference.py:159-160, taylor.py:176-177). */
int isa_forward_host_bytes(const IsaShape* shape, const IsaKnobs* knobs, int32_t heads_per_chunk,
                           size_t* stage_bytes, size_t* workspace_bytes);
int isa_forward_host(const IsaShape* shape, const IsaKnobs* knobs, const void* q_host, const void* k_host,
                     const void* v_host, void* out_host, int32_t heads_per_chunk, void* stage, size_t stage_bytes,
                     void* workspace, size_t workspace_bytes, const IsaRoutingIn* pinned, IsaRoutingOut* routing,
                     int32_t* err_word, void* const* streams);

/* Backward with frozen routing (isa_backward, pipeline.py:373-466, incl. the
 * gamma coarse residual through the block means, pipeline.py:435-452):
 * recomputes the forward (routing from q/k, or `pinned`) with its per-row
 * softmax statistics, then the sharp-branch (reference.py:173-225) and Taylor
 * (taylor.py:225-296) gradients, scattered back through the K_new gather
 * (pipeline.py:423-433). q/k/v/dout: bf16 with the shape's strides; dq/dk/dv:
 * fp32 contiguous (B,H,S,D), fully written (rows of unselected context blocks
 * get 0). Workspace sized by isa_backward_workspace_bytes. */
int isa_backward_workspace_bytes(const IsaShape* shape, const IsaKnobs* knobs, size_t* bytes);
int isa_backward(const IsaShape* shape, const IsaKnobs* knobs, const void* q, const void* k, const void* v,
                 const void* dout, float* dq, float* dk, float* dv, void* workspace, size_t workspace_bytes,
                 const IsaRoutingIn* pinned, int32_t* err_word, void* stream);

/* Stages 1-3 only (isa_routing, pipeline.py:302-304). */
int isa_routing(const IsaShape* shape, const IsaKnobs* knobs, const void* q, const void* k, const void* v,
                void* workspace, size_t workspace_bytes, IsaRoutingOut* routing, int32_t* err_word,
                void* stream);

/* Dense non-causal attention on the same sm_100a kernel (identity block
 * tables): the speed-up denominator and the full_attention oracle
 * (reference.py:79-123). Requires L_src, L_ctx multiples of 64 unless the
 * sequence is a single segment. */
int isa_dense_attention(const IsaShape* shape, double scale, const void* q, const void* k, const void* v,
                        void* out, void* stream);

/* Dense attention with a query length S_q different from the key length
 * k_len (full_attention / online_softmax_attention without a key mask,
 * reference.py:79-170). q_shape describes q and out (bf16, seq_len = S_q a
 * multiple of 64); k and v share k_strides {b, h, s} (elements). A ragged
 * k_len (not a multiple of 64) needs ceil(k_len/64) > S_q/64. */
int isa_cross_attention(const IsaShape* q_shape, int32_t k_len, const int64_t* k_strides, double scale,
                        const void* q, const void* k, const void* v, void* out, void* stream);

/* Decoupled rotary embedding (pipeline.py:469-490, apply_decoupled_rope):
 * pairs (2i, 2i+1) of each token rotate by pos * base^(-2i/D) with positions
 * 0..L_src-1 for the source segment and 0..L_ctx-1 for the context segment.
 * x and out share shape (B,H,S,D); x uses the shape's strides, out the out
 * strides; dtype bf16 or fp32; angles in fp64, rotation in fp32. */
int isa_decoupled_rope(const IsaShape* shape, double base, const void* x, void* out, void* stream);

/* Standalone Taylor kernel (taylor_sparse_forward, taylor.py:163-194, with
 * TaylorKernelInput, taylor.py:45-109): every 64-row query block of q is
 * flat; mask[b][h][u][0..k_mask) (int64, ascending, in [0, k_len/64)) are its
 * exact key blocks of k/v; kc/vc (fp32 contiguous (B,H,k_len/64,D)) are the
 * key-block centroids. q_shape describes q and out (seq_len = S_q, bf16,
 * l_src = seq_len, l_ctx = 0); k and v share k_strides {b, h, s} (elements).
 * Full blocks only (S_q, k_len multiples of 64). */
int isa_taylor_workspace_bytes(const IsaShape* q_shape, int32_t k_len, int32_t k_mask, size_t* bytes);
int isa_taylor_forward(const IsaShape* q_shape, int32_t k_len, const int64_t* k_strides, int32_t k_mask,
                       double scale, const void* q, const void* k, const void* v, const float* kc, const float* vc,
                       const int64_t* mask, void* out, void* workspace, size_t workspace_bytes, int32_t* err_word,
                       void* stream);

/* ---- stage primitives (test hooks; same kernels as the pipeline) ---- */

/* K1: block means (B,H,T,D) fp32 of q, k, v into means[3][B][H][T][D]. */
int isa_pool_means(const IsaShape* shape, const void* q, const void* k, const void* v, float* means,
                   int32_t* err_word, void* stream);

/* Top-k of each row of a float64 (rows, n) matrix, ties to the lower index,
 * emitted ascending (coarse.py:130-136). method 0 = CTA rank selection
 * (context pre-selection kernel), 1 = warp arg-max rounds (block-mask kernel). */
int isa_topk_rows_f64(const double* scores, int32_t rows, int32_t n, int32_t k, int64_t* out_idx,
                      int32_t method, void* stream);

/* Coarse scores s[bh][i][j] = scale * <qc[bh][i], kc[bh][j]> in float64,
 * bit-identical to the reference's np.einsum("bhid,bhjd->bhij") over fp64
 * copies of fp32 means (coarse.py:126, pipeline.py:180-182; head dims that
 * are multiples of 8). qc (bh, t_q, d), kc (bh, t_k, d) fp32 contiguous;
 * s (bh, t_q, t_k) fp64 contiguous. */
int isa_coarse_scores(int32_t bh, int32_t t_q, int32_t t_k, int32_t d, double scale, const float* qc,
                      const float* kc, double* s, void* stream);

/* Context saliency (coarse.py:155): out[bh][c] = mean over i < n_src of
 * s[bh][i][n_src + c] for c < n_ctx, summed in numpy's order. Element
 * (bh, i, j) of s sits at s + bh * head_stride + i * row_stride + j. */
int isa_ctx_saliency_f64(const double* s, int32_t bh, int64_t head_stride, int64_t row_stride, int32_t n_src,
                         int32_t n_ctx, double* out, void* stream);

/* Sharpness per row (coarse.py:193-195): population variance of the row
 * softmax (softmax_first) or of the raw row. */
int isa_sharpness_rows_f64(const double* s, int32_t rows, int32_t n, int32_t softmax_first, double* out,
                           void* stream);

/* Sharp/flat split of each row of sharpness values (coarse.py:196-200). */
int isa_split_rows_f64(const double* m, int32_t rows, int32_t n, int32_t n_flat, int64_t* sharp, int64_t* flat,
                       void* stream);

#ifdef __cplusplus
}
#endif
#endif /* ISA_B200_H */
