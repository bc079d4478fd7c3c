/*
 * specpipe_b200 — C ABI of the B200-native PipeInfer hot path.
 *
 * The reference (``specpipe``, a pure-Python package) has no FFI; the
 * boundary this library sits behind is its Python API.  Each
 * entry point below names the reference function it replaces.  The Python
 * host (``paper_2407_11798_b200``) binds these with ctypes; see
 * INTEGRATION.md for the binding a reference maintainer would add.
 *
 * Conventions
 *  - every function returns an ``int`` status (SP_OK or an SP_ERR_* code);
 *  - all tensor arguments are caller-owned DEVICE pointers unless the name
 *    says ``host``; nothing on the hot path allocates;
 *  - ``stream`` is a ``cudaStream_t`` passed as ``void*``; work is enqueued,
 *    never synchronised, except the explicitly blocking ``*_sync`` queries;
 *  - numerical errors detected on the device (bad token id, position beyond
 *    max_context, non-finite activations, NaN logits, coverage violations)
 *    set bits in a sticky device error word that the host reads when it
 *    collects a run's result (no per-layer host synchronisation).
 *
 * Build: nvcc -gencode arch=compute_100a,code=sm_100a (B200 only).
 */
#ifndef SPECPIPE_B200_H
#define SPECPIPE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (map to the reference's exception types) ------------ */
enum {
  SP_OK = 0,
  SP_ERR_MODEL = 1,     /* ModelError      model.py:35-36      */
  SP_ERR_CACHE = 2,     /* CacheError      kvcache.py:25-26    */
  SP_ERR_PROTOCOL = 3,  /* ProtocolError   transport.py:34-35  */
  SP_ERR_CUDA = 4,      /* CUDA runtime failure                 */
  SP_ERR_ARG = 5,       /* invalid argument to the C ABI        */
  SP_ERR_CAPACITY = 6   /* cell pool / descriptor capacity      */
};

/* ---- sticky device error bits ----------------------------------------- */
enum {
  SP_DEV_BAD_TOKEN = 1,      /* model.py:355-356 */
  SP_DEV_BAD_POS = 2,        /* model.py:357-358, kvcache.py:142-143 */
  SP_DEV_NONFINITE = 4,      /* model.py:419-420 */
  SP_DEV_NAN_LOGITS = 8,     /* model.py:441-442 */
  SP_DEV_COVERAGE = 16,      /* engine.py:625-633 */
  SP_DEV_BAD_SEQ = 32,       /* kvcache.py:144-146 */
  SP_DEV_PLAN_OVERFLOW = 64  /* visible list longer than the launch bound */
};

enum { SP_ARCH_REF = 0, SP_ARCH_LLAMA = 1 };
enum { SP_DTYPE_F32 = 0, SP_DTYPE_BF16 = 1 };
enum { SP_KIND_PREFILL = 0, SP_KIND_NONSPEC = 1, SP_KIND_SPEC = 2 };
enum { SP_STATUS_VALID = 0, SP_STATUS_PLACEHOLDER = 1 };

/* forward flags */
enum {
  SP_FWD_CHECK_COVERAGE = 1,  /* chain batches: token at pos p sees p cells */
  SP_FWD_SKIPPABLE = 2,       /* speculative: honour cancel / placeholder  */
  SP_FWD_CONTINUE = 4,        /* same run, next layer sub-range: reuse the
                                 descriptor, cells and plan (split
                                 evaluation, model.py:5-11)               */
  SP_FWD_CHAIN = 8            /* draft chain step: token 0 = tip argmax,
                                 gated by the chain gate                  */
};

/* Model shape (ModelConfig, model.py:39-64, extended with the llama arch). */
typedef struct sp_model_dims {
  int32_t arch;        /* SP_ARCH_*                                     */
  int32_t vocab;
  int32_t d_model;
  int32_t n_layers;
  int32_t n_heads;
  int32_t n_kv_heads;
  int32_t head_dim;
  int32_t ffn_dim;     /* ref: 4*d_model                                */
  int32_t max_context;
  int32_t w_dtype;     /* SP_DTYPE_* of weights and KV cache            */
  float norm_eps;      /* ref: 1e-8 inside the mean; llama: 1e-5         */
  float rope_theta;
  int32_t w_layout;    /* SP_LAYOUT_*: bf16 llama stages with TC-tiled
                          weights run on tcgen05, natural ones on the
                          CUDA-core GEMV (latency-bound drafts)          */
} sp_model_dims;

/* SWZ8: row-major bf16 rows whose 16-byte units are XOR-permuted within each
 * 128-byte group, unit u of row r stored at u ^ (r & 7): a contiguous copy of
 * any row block into shared memory is then bank-conflict-free for 8-row
 * ldmatrix / LDS access (the persistent draft kernels); requires K % 64 == 0. */
enum { SP_LAYOUT_NATURAL = 0, SP_LAYOUT_TC_TILED = 1, SP_LAYOUT_SWZ8 = 2 };

/* One BatchToken (model.py:67-75); seq sets are bitmasks (P <= 32). */
typedef struct sp_token {
  int32_t token;
  int32_t pos;
  uint32_t seq_mask;
  int32_t want_logits;
} sp_token;

/* Fused LM-head result per flagged row (model.py:438-457 on device). */
typedef struct sp_row_result {
  int32_t argmax;      /* greedy_sample: lowest id on ties   */
  int32_t second;      /* second_best                         */
  float conf;          /* max_softmax                         */
  float max_logit;
} sp_row_result;

/* ======================================================================
 * Low-level kernels
 * ====================================================================== */

/* K1: x[i] = E[tok_i] (+ P[pos_i] for the ref arch).  model.py:352-359 */
int sp_embed(const sp_model_dims* dims, const void* emb, const float* pos_table,
             const sp_token* toks, int n, float* x, int* err, void* stream);

/* Epilogues of the weight-streaming GEMV family (K2/K6/K7/K9). */
enum {
  SP_EPI_STORE = 0,   /* y = norm(x) @ W^T                                  */
  SP_EPI_RESID = 1,   /* out += x @ W^T (+ finite check)   model.py:416,418 */
  SP_EPI_QKV = 2,     /* q -> out; k,v -> cache rows (+RoPE) model.py:387-393 */
  SP_EPI_GELU = 3,    /* out = gelu(norm(x) @ W^T)          model.py:417-418 */
  SP_EPI_SWIGLU = 4,  /* out = silu(g)*u, rows interleaved (g,u)            */
  SP_EPI_LMHEAD = 5   /* greedy head: per token argmax / second / max-softmax
                         over all rows (tile partials + a fixed-order merge);
                         logits to out when out != NULL   model.py:424-457  */
};

typedef struct sp_gemv_args {
  const void* w;          /* [n_rows, k] row-major, K contiguous          */
  int32_t w_dtype;        /* SP_DTYPE_*                                   */
  int32_t n_rows;
  int32_t k;
  const float* x;         /* [m, ldx]                                     */
  int32_t m;
  int32_t ldx;
  int32_t norm;           /* fuse RMSNorm of x                           */
  float norm_eps;
  const float* gain;      /* optional RMSNorm gain [k]                   */
  int32_t epi;            /* SP_EPI_*                                     */
  void* out;              /* fp32 [m, ldo]                                */
  int32_t ldo;
  /* QKV epilogue */
  int32_t q_rows;         /* rows [0,q_rows) -> q; then k; then v        */
  int32_t kv_rows;
  void* k_cache;          /* [cap, kv_rows] (w_dtype)                    */
  void* v_cache;
  int32_t cache_row0;     /* cell row of token 0; token i -> row0+i       */
  int32_t rope;           /* rows are pair-interleaved per head          */
  int32_t head_dim;
  float rope_theta;
  const sp_token* toks;   /* positions for RoPE                          */
  int* err;
  const int* run_state;   /* non-zero => skip (cancelled / placeholder)  */
  /* early inference cancellation (K14): CTA 0 reads *cancel_word and, if it
   * names run_id, sets *run_state_w so every LATER kernel of the run skips.
   * Only kernels without cross-CTA state may observe it (a mid-kernel flip
   * must not strand split-merge tickets). */
  int* run_state_w;
  const int* cancel_word;
  int32_t run_id;
  const int32_t* cache_row0_dev;  /* if set, overrides cache_row0 (run header) */
  int32_t w_swz;          /* bf16 rows in the SWZ8 layout (see SP_LAYOUT_SWZ8) */
} sp_gemv_args;

int sp_gemv(const sp_gemv_args* a, void* stream);

/* Skinny tensor-core GEMM (tcgen05 + TMEM + TMA, bf16 weights/activations,
 * fp32 accumulate) used for every bf16 run: D[rows, tokens] = W . X^T with
 * split-K merged in fixed order and the epilogues of the GEMV family.
 * RMSNorm enters as a per-token scale from sum-of-squares partials
 * (ss_in[p * ss_ld + token], p < ss_nparts); the residual epilogue emits the
 * next norm's bf16 input (xb_next = x * gain_next) and its partials. */
typedef struct sp_tc_args {
  const void* w;           /* bf16 weights in the TILED layout: [n_rows/128]
                              [k/64] tiles of 128 x 64, each stored as the
                              128B-swizzled K-major smem image (16 KB)      */
  int32_t n_rows;          /* multiple of 128                               */
  int32_t k;               /* multiple of 64                                */
  int32_t m;               /* tokens                                        */
  int32_t tok0;            /* first token of the launch (internal)          */
  int32_t epi;             /* SP_EPI_STORE | QKV | SWIGLU | RESID            */
  int32_t norm;
  float norm_eps;
  void* out;               /* STORE/QKV-q: f32; SWIGLU: bf16; RESID: f32 x  */
  int32_t ldo;
  int32_t q_rows, kv_rows; /* QKV                                           */
  void* k_cache;           /* bf16 [cap, kv_rows]                           */
  void* v_cache;
  int32_t cache_row0;
  int32_t head_dim;
  float rope_theta;
  const sp_token* toks;
  const float* ss_in;      /* norm statistic partials                       */
  int32_t ss_nparts;
  int32_t ss_ld;
  float* ss_out;           /* RESID: per-128-row-tile partials              */
  void* xb_next;           /* RESID: bf16 [tokens, ldo]                     */
  const float* gain_next;  /* RESID: gain of the next RMSNorm (or NULL)     */
  float* scratch;          /* split-K partials                              */
  int* tickets;            /* per row tile, zero-initialised                */
  int32_t ksplit;          /* 0 = auto                                      */
  int32_t max_ctas;        /* CTA budget for auto split-K (0 = 2 per SM);
                              a smaller budget leaves SMs free for a
                              co-scheduled stream (the draft)              */
  int* err;
  const int* run_state;
  const int32_t* cache_row0_dev;  /* if set, overrides cache_row0 (run header) */
  /* SP_EPI_LMHEAD (tensor-core LM head) */
  sp_row_result* lm_out;   /* [m] records (argmax, second, conf, max logit) */
  void* lm_part;           /* >= m * n_rows/128 partials of 32 bytes        */
  int* lm_ticket;          /* zero-initialised; reset by the merging CTA    */
  int* lm_err_out;         /* *err copied here when the head finishes       */
  int* lm_status_out;      /* SP_STATUS_VALID, or PLACEHOLDER when skipped  */
  int* lm_tip;             /* [argmax, conf bits, valid] of the last row    */
  int* lm_gate;            /* chain gate (conf >= cutoff), with lm_chain_gate */
  int32_t lm_chain_gate;
  float lm_cutoff;
  const void* lm_hdr;      /* run header (its cutoff wins when set)         */
} sp_tc_args;

/* Low-level form (tests): a->w tiled bf16; X bf16 [x_rows, k] row-major
 * with x_rows >= 128 allocated rows. */
int sp_tc_gemm(const sp_tc_args* a, const void* x, int x_rows, void* stream);

/* K4: per query, the position-ordered visible cell rows (ties by row),
 * the query's own row appended last.  model.py:287-323.  Rows >= row0
 * are the batch's own cells (described by ``toks``).                     */
int sp_build_plan(const int32_t* cell_pos, const uint32_t* cell_mask,
                  int n_old, int row0, const sp_token* toks, int n,
                  int max_context, int32_t* vis, int32_t* vis_len, int ld_vis,
                  int check_coverage, int* err, void* stream);

/* K5: tree-masked attention over the plan.  model.py:394-415 */
int sp_attention(const float* q, const void* k_cache, const void* v_cache,
                 int kv_dtype, const int32_t* vis, const int32_t* vis_len,
                 int ld_vis, int n, int n_heads, int n_kv_heads, int head_dim,
                 int max_vis, float* out, float* scratch, int* tickets,
                 const int* run_state, void* stream);

/* K3/K10/K11: cell metadata (layer-uniform, one table per stage). */
int sp_kv_meta_write(int32_t* cell_pos, uint32_t* cell_mask, int row0,
                     const sp_token* toks, int n, int n_seq_ids,
                     int max_context, int* err, void* stream);
int sp_kv_copy(int32_t* cell_pos, uint32_t* cell_mask, int n_cells, int src,
               uint32_t dst_mask, int end_pos, int max_context, void* stream);
int sp_kv_remove(const int32_t* cell_pos, uint32_t* cell_mask, int n_cells,
                 uint32_t seq_mask, int from_pos, void* stream);
int sp_kv_keep(uint32_t* cell_mask, int n_cells, int seq, void* stream);

/* K9: fused final RMSNorm + LM head + argmax/second/max-softmax. */
int sp_lmhead(const void* w_out, int w_dtype, int vocab, int d, const float* x,
              const int32_t* rows, int n_rows, int norm, float norm_eps,
              const float* gain, sp_row_result* out, float* logits_out,
              float* scratch, int* tickets, int* err, const int* run_state,
              void* stream);

/* ======================================================================
 * Stage runtime: one pipeline stage (contiguous layer range) on one GPU.
 * Replaces _Worker._on_activations + eval_layers (engine.py:563-623,
 * model.py:326-421) and owns the stage's KV cells (kvcache.py:94-283).
 * ====================================================================== */
typedef struct sp_stage sp_stage;

int sp_stage_create(const sp_model_dims* dims, int layer_lo, int layer_hi,
                    int cell_capacity, int max_tokens, int n_seq_ids,
                    sp_stage** out);
int sp_stage_destroy(sp_stage* s);
int sp_stage_set_embedding(sp_stage* s, const void* emb, const float* pos_table);
int sp_stage_set_layer(sp_stage* s, int layer, const void* w_qkv,
                       const void* w_o, const void* w_up, const void* w_down,
                       const float* attn_norm, const float* mlp_norm);
int sp_stage_set_head(sp_stage* s, const void* w_out, const float* final_norm);
/* The LM head in the tensor-core tiled layout (model.tile_weight of w_out,
 * vocab % 128 == 0): graph-replayed steps of a tiled stage then run the
 * head as one tcgen05 GEMM with the fused greedy epilogue (SP_EPI_LMHEAD),
 * flat in the number of rows up to 16 (the CUDA-core head re-streams per
 * 8-row tile).  NULL restores the CUDA-core head. */
int sp_stage_set_head_tiled(sp_stage* s, const void* w_out_tiled);
/* device-visible cancel words: table[run_id % size] == run_id => cancelled */
int sp_stage_set_cancel_table(sp_stage* s, const int* table, int size);
/* CTA budget of this stage's tensor-core GEMMs (0 = whole GPU). */
int sp_stage_set_cta_budget(sp_stage* s, int ctas);

/* Enqueue layers [lo,hi) for one run.  ``host_toks`` is copied into a
 * stream-ordered device descriptor (RUN_CONFIG, engine.py:231-251).
 * ``x_in``: device activations (NULL on stage 0); ``in_status``: device
 * status word of the upstream message (NULL if none).  ``x_out`` receives
 * the stage output (the layers run in place on it) and ``out_status`` the
 * placeholder flag (engine.py:545-554).  ``chain`` != 0: token 0 is the
 * draft chain's tip argmax and the run is gated by the chain gate (the
 * device-side speculate_microbatch loop, speculation.py:185-211). */
int sp_stage_forward(sp_stage* s, const sp_token* host_toks, int n, int run_id,
                     int kind, int flags, const float* x_in, const int* in_status,
                     float* x_out, int* out_status, int chain, void* stream);

/* Same, restricted to layers [layer_a, layer_b) of the stage (-1: all).
 * With SP_FWD_CONTINUE the call continues the previous run of this stage. */
int sp_stage_forward_range(sp_stage* s, const sp_token* host_toks, int n,
                           int run_id, int kind, int flags, const float* x_in,
                           const int* in_status, float* x_out, int* out_status,
                           int chain, int layer_a, int layer_b, void* stream);

/* K9 over the flagged rows ``host_rows`` of ``x`` (the last forward's
 * output): writes ``out[n_rows]``, optionally full logits, and a copy of the
 * sticky error word into ``err_out``.  ``update_tip``: remember the last
 * row's (argmax, conf) as the draft tip; ``chain_gate``: gate &= conf >=
 * cutoff (one step of speculate_microbatch). */
int sp_stage_lmhead(sp_stage* s, const float* x, const int32_t* host_rows,
                    int n_rows, sp_row_result* out, float* logits_out,
                    int* err_out, int update_tip, int chain_gate, float cutoff,
                    void* stream);

/* One decode / verification stage-run (+ the fused LM head when n_rows > 0)
 * replayed from a per-shape CUDA graph: every per-run scalar travels in one
 * small H2D header copy.  Inputs: x_in/in_status (device, NULL on layer 0;
 * pointers are part of the graph key, so pass fixed buffers); outputs land in
 * the stage's fixed buffers (sp_stage_io): activations + status word at
 * x_out[n*d], result block [status, err, -, -] + n_rows sp_row_result.
 * ``res_copy``: optional destination (device or pinned host) for the result
 * block.  head_flags: SP_STEP_TIP (remember the tip), SP_STEP_CHAIN (draft
 * chain step: token 0 = tip argmax, gated; gate &= conf >= cutoff). */
enum { SP_STEP_TIP = 1, SP_STEP_CHAIN = 2 };
int sp_stage_step(sp_stage* s, const sp_token* host_toks, int n, int run_id, int kind,
                  int flags, const int32_t* host_rows, int n_rows, int head_flags,
                  float cutoff, const float* x_in, const int* in_status, void* res_copy,
                  void* stream);
int sp_stage_io(sp_stage* s, float** x_out, sp_row_result** res);

/* A whole draft request as ONE persistent cooperative kernel (K15): feed
 * n_feed <= 4 tokens at positions pos0.. (their forward + LM head on the
 * last -> out[0]; with n_feed == 0, out[0] = the current tip), then `steps`
 * single-token forwards, step j (1-based) -> out[j].  step_tokens == NULL:
 * chain mode (token = previous argmax; stops once conf < cutoff, remaining
 * cells dead, like sp_stage_step with SP_STEP_CHAIN); else the given tokens.
 * Requires a llama bf16 stage with natural-layout weights holding every
 * layer + head, one sequence, rows == positions (pos0 == n_cells; see
 * sp_stage_truncate).  Appends n_feed + steps cells.  Replaces the draft
 * node's per-token loop (engine.py:640-688, speculation.py:142-195). */
/* 1 if this stage's shape runs on the persistent draft kernels (else the
 * caller uses one sp_stage_step per forward). */
int sp_stage_decode_chain_ok(const sp_stage* s);
/* Which persistent draft kernel sp_stage_decode_chain launches: the cluster
 * form (16 SMs; leaves the rest of the GPU to a co-resident target stage) or
 * the grid form (every SM; for a draft whose GPU is otherwise idle -- a
 * dedicated draft GPU, or a shared one while no target run is queued).
 * AUTO follows the SP_DRAFT_KERNEL environment variable (cluster default). */
#define SP_DRAFT_KIND_AUTO 0
#define SP_DRAFT_KIND_CLUSTER 1
#define SP_DRAFT_KIND_GRID 2
int sp_stage_set_draft_kernel(sp_stage* s, int kind);
/* Whether captured stage-runs put the layers inside a conditional (IF) graph
 * body set by the gate kernel (1, default): a run cancelled before it starts
 * then skips every layer (~0.06 ms instead of ~0.45 ms for a 7B stage), but
 * the body's device-side launch adds ~80-250 us to every full run (it grows
 * with the body's node count).  Off (0) when no run can be cancelled (sync,
 * iterative, and the 1-stage folding policy).  Replaces no reference call. */
int sp_stage_set_skip_graphs(sp_stage* s, int on);
/* Text of the last CUDA failure behind an SP_ERR_CUDA status on this thread
 * ("runtime.cu:<line>: <call> -> <cudaGetErrorString>"), "" if none. */
const char* sp_last_error(void);
int sp_stage_decode_chain(sp_stage* s, const int32_t* feed, int n_feed, int pos0,
                          const int32_t* step_tokens, int steps, float cutoff,
                          sp_row_result* out, int* err_out, void* stream);
/* Position-addressed stages: drop rows >= n_cells (they are rewritten by the
 * next tokens; the draft's truncate, kvcache.py:120-149 for one sequence). */
int sp_stage_truncate(sp_stage* s, int n_cells);
/* Reclaim the rows of dead cells (stable compaction of the bounded cell
 * pool; the reference's cache is unbounded).  Synchronises the stream;
 * returns the new cell count or -error.  Not for position-addressed stages. */
int sp_stage_compact(sp_stage* s, void* stream);
/* Diagnostics (env SP_DRAFT_PROF=1): %globaltimer stamps of CTA 0 at every
 * phase edge of the last decode_chain; returns the count (or -error). */
int sp_stage_draft_profile(sp_stage* s, long long* host, int max);

/* Draft chain: gate = tip.valid && tip.conf >= cutoff; out <- tip. */
int sp_stage_chain_begin(sp_stage* s, float cutoff, sp_row_result* out,
                         void* stream);
int sp_stage_chain_state(sp_stage* s, int** tip, int** gate);
/* SerialDecoder.truncate nulls the tip logits (model.py:507-512). */
int sp_stage_invalidate_tip(sp_stage* s, void* stream);

/* Sequence ops on the stage's cell table (CACHE_COPY / CACHE_REMOVE). */
int sp_stage_cache_copy(sp_stage* s, int src, uint32_t dst_mask, int end_pos,
                        void* stream);
int sp_stage_cache_remove(sp_stage* s, int seq, int from_pos, void* stream);
int sp_stage_cache_keep(sp_stage* s, int seq, void* stream);
int sp_stage_reset(sp_stage* s, void* stream);
/* Append cells (metadata only) — KVCache.insert for trace-replay tests. */
int sp_stage_cache_insert_meta(sp_stage* s, const sp_token* host_toks, int n,
                               void* stream);

/* Queries (blocking, for tests/diagnostics and run-completion checks). */
int sp_stage_n_cells(const sp_stage* s);
int sp_stage_meta_sync(sp_stage* s, int32_t* host_pos, uint32_t* host_mask,
                       int cap, void* stream);
int sp_stage_read_kv_sync(sp_stage* s, int layer, int row, float* host_k,
                          float* host_v, void* stream);
int sp_stage_error_sync(sp_stage* s, int clear, void* stream);
int sp_stage_error_ptr(sp_stage* s, int** dev_err);
int sp_stage_plan_sync(sp_stage* s, int32_t* host_vis, int32_t* host_len,
                       int n, void* stream);
int sp_stage_ld_vis(const sp_stage* s);
/* eval_layers(..., mask=TreeAttentionMask) (model.py:326-373): install a
 * caller-built plan -- per query ``host_len[i]`` rows of ``host_vis`` (row
 * stride sp_stage_ld_vis), cache rows and this batch's rows
 * (n_cells + j) in gather order, the query's own row last -- for the next
 * non-continuation forward, which then skips building the plan (K4). */
int sp_stage_set_plan(sp_stage* s, const int32_t* host_vis, const int32_t* host_len,
                      int n, void* stream);
/* K4/K11: build the plan ``host_toks`` would get against the current table
 * (without inserting its cells); visible counts = plan lengths - 1. */
int sp_stage_plan_only(sp_stage* s, const sp_token* host_toks, int n,
                       int check_coverage, void* stream);

/* Cross-process control plane (distributed pipeline): page-lock a host
 * region (e.g. POSIX shared memory) and map it into the device address space
 * so kernels can read cancel words and results can be written into it;
 * ``sp_signal`` stores ``value`` to a mapped flag after all prior work on
 * ``stream`` (CANCEL / LOGITS transport.py:265-271, engine.py:619-623). */
int sp_host_register(void* ptr, size_t bytes, void** dev_ptr);
int sp_host_unregister(void* ptr);
int sp_signal(int* dev_flag, int value, void* stream);
int sp_copy_async(void* dst, const void* src, size_t bytes, void* stream);

/* Library info. */
const char* sp_version(void);
int sp_device_arch(void);

#ifdef __cplusplus
}
#endif
#endif /* SPECPIPE_B200_H */
