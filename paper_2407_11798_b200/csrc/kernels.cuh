// Launch interfaces shared by the kernel translation units and the runtime.
#pragma once

#include <cuda.h>

#include "common.cuh"

namespace sp {

typedef sp_tc_args TcArgs;

// a stage's tensor-core GEMM scratch (split-K partials) and tile tickets;
// launchers that pass TcArgs::scratch / tickets provide at least this much
static constexpr int TC_SCRATCH_FLOATS = 8 << 20;
static constexpr int TC_TICKETS = 4096;

// Per-run scalars read by the kernels of a stage-run (one small H2D copy per
// run); followed in memory by int32 rows[max_tokens] and sp_token
// toks[max_tokens].  Keeping them out of kernel arguments makes a stage-run
// replayable as a CUDA graph.
struct RunHdr {
  int32_t row0;        // first cell row of the run's tokens
  int32_t n;           // tokens
  int32_t run_id;
  int32_t kind;
  int32_t flags;       // SP_FWD_*
  int32_t nrows;       // flagged rows for the LM head
  int32_t cancel_idx;  // run_id % cancel table size, -1 if none
  float cutoff;        // draft chain: conf >= cutoff keeps the gate open
};

struct AttnArgs {
  const float* q;
  const void* k;
  const void* v;
  const int32_t* vis;
  const int32_t* vis_len;
  int ld_vis;
  int n, H, KH, nsplit;
  float scale;
  float* out;
  float* scratch;
  int* tickets;
  const int* run_state;
  int* run_state_w;        // written by CTA (0,0,0) when the cancel word fires
  const int* cancel_word;  // device-visible cancel word of this run (or null)
  int run_id;
  int* err;
  int out_bf16;            // write the output as bf16 (tensor-core path input)
  int merge_smem;   // set by the launcher: merge partials through shared memory
  // cache rows >= this are written by the kernel the launch depends on (the
  // run's own cells); older rows may be read before the dependency wait
  const int32_t* fresh_row0_dev;
  int fresh_row0;
  int diag_empty;   // diagnostics only (SP_ATT_DIAG=1): return after the dependency wait
  // the run's tokens and header (tensor-core kernel: in a run whose
  // coverage is checked -- every token sees exactly one cell per earlier
  // position -- a query on the reference query's sequence set has a plan
  // that is a prefix of the reference's), or null
  const sp_token* toks;
  const RunHdr* hdr;
  int max_context;   // the model's context cap (a per-stage constant: kernel choice)
};

struct LmPartial {
  float v1; int i1; float v2; int i2; float mx; float se; int nan; int pad;
};

struct LmArgs {
  const void* w;
  int V, d;
  const float* x;   // gathered flagged rows [n_rows, d]
  int n_rows;
  int norm;
  float eps;
  const float* gain;
  sp_row_result* out;
  float* logits;    // optional [n_rows, V]
  LmPartial* scratch;
  int* ticket;
  int* err;
  int* err_out;     // optional: copy of *err after the merge
  const int* run_state;
  int* tip;         // device-side draft chain: [argmax, conf bits, valid]
  int* status_out;  // optional: run status (valid / placeholder)
  const RunHdr* hdr;  // optional: cutoff from the run header
  int swz;            // weights in the SWZ8 layout
  int* gate;
  int chain_gate;
  float cutoff;
};

// ---- K15: persistent draft chain (draft.cu) --------------------------------
constexpr int DR_NT = 4;          // max fed tokens per launch
constexpr int DR_MAX_STEPS = 64;  // max chained steps per launch
constexpr int DR_MAX_LAYERS = 64;

struct DraftLayer {
  const __nv_bfloat16* qkv;
  const __nv_bfloat16* o;
  const __nv_bfloat16* up;
  const __nv_bfloat16* down;
  const float* g_attn;
  const float* g_mlp;
};

struct DraftHdr {                 // per-launch run header (one H2D copy)
  int32_t n_feed, steps, pos0, row0, chain, pad0, pad1, pad2;
  float cutoff;
  int32_t pad3[3];
  int32_t tok[DR_NT + DR_MAX_STEPS];   // fed tokens, then explicit step tokens
};

struct DraftArgs {
  const DraftLayer* layers;
  int L, V, d, H, KH, hd, f;
  float eps, theta;
  const __nv_bfloat16* emb;
  const __nv_bfloat16* w_out;
  const float* g_final;
  __nv_bfloat16* kc;
  __nv_bfloat16* vc;
  size_t kv_layer_elems;
  int32_t* cell_pos;
  uint32_t* cell_mask;
  const DraftHdr* hdr;
  int* tip;
  int* gate;
  float* x;          // [DR_NT, d]
  float* q;          // [DR_NT, H*hd]
  float* attn;       // [DR_NT, H*hd]
  float* h;          // [DR_NT, f]
  float* att_part;   // [DR_NT, H, max_split, hd + 2]
  int* att_tick;     // [DR_NT * H]
  int max_split;
  LmPartial* lm_part;  // [grid]
  unsigned* bar;
  sp_row_result* out;  // [steps + 1]
  int* err;
  int* err_out;
  long long* prof;     // optional: CTA 0's clock64 at every phase edge
  float* xb;           // [DR_NT, d] x after attention (residual owners' rows)
  float* opart;        // [DR_NT, H, d] per-head O projections
  int bufA, bufD, bufE;  // per-CTA weight staging buffers (bytes)
  int kmax;
  int ring_stages, ring_bytes;  // cluster form: weight ring per CTA
  int nt;                       // cluster form: token rows of the activation buffers
  int use_mma;                  // cluster form: mma.sync GEMV for 16-row chunks
  unsigned spin_ns;             // grid form: barrier poll back-off
  int diag_nocompute;           // cluster form, diagnostics only: skip the GEMV math
};

size_t draft_smem_bytes(const DraftArgs& a);
cudaError_t launch_draft_chain(const DraftArgs& a, int ctas, cudaStream_t st);
int draft_max_ctas(const DraftArgs& a);
void draft_buffers(DraftArgs& a, int ctas);
size_t draft2_smem_bytes(const DraftArgs& a, int cl);
size_t draft2_act_bytes(const DraftArgs& a, int cl, int nt);
int draft2_cluster_size(const DraftArgs& a, int want);
cudaError_t launch_draft_cluster(const DraftArgs& a, int cl, cudaStream_t st);

cudaError_t launch_plan(const int32_t* cell_pos, const uint32_t* cell_mask,
                        int n_old, int row0, const sp_token* toks, int n,
                        int max_context, int32_t* vis, int32_t* vis_len,
                        int ld_vis, int check_cov, int* err, cudaStream_t st,
                        const int* run_state = nullptr, const RunHdr* hdr = nullptr);
cudaError_t launch_attention(const AttnArgs& a, int kv_dtype, int hd,
                             cudaStream_t st);
int attn_splits(int max_len);
// flash-decoding attention over bf16 caches, decode-sized runs (attention_fd.cu)
bool attn_fd_ok(int kv_dtype, int hd, int n, int max_context);
cudaError_t launch_attention_fd(const AttnArgs& a, int hd, cudaStream_t st);
// tensor-core attention over bf16 caches (attention_tc.cu)
bool attn_tc_ok(int kv_dtype, int hd, int n);
cudaError_t launch_attention_tc(const AttnArgs& a, int hd, cudaStream_t st);
cudaError_t launch_lmhead(const LmArgs& a, int w_dtype, cudaStream_t st);
int lmhead_grid(int V);
cudaError_t launch_meta_write(int32_t* pos, uint32_t* mask, int row0,
                              const sp_token* toks, int n, int n_seq,
                              int max_context, int* err, cudaStream_t st);
cudaError_t launch_copy(const int32_t* pos, uint32_t* mask, int n, int src,
                        uint32_t dst_mask, int end_pos, int max_context,
                        cudaStream_t st);
cudaError_t launch_remove(const int32_t* pos, uint32_t* mask, int n,
                          uint32_t seq_mask, int from_pos, cudaStream_t st);
cudaError_t launch_keep(uint32_t* mask, int n, int seq, cudaStream_t st);
cudaError_t launch_compact_scan(const int32_t* pos, const uint32_t* mask, int n, int32_t* src_of,
                                int32_t* pos2, uint32_t* mask2, int* live, cudaStream_t st);
cudaError_t launch_compact_gather(const void* src, void* dst, const int32_t* src_of,
                                  const int* live, int row_bytes, int n_max, cudaStream_t st);
bool make_map_bf16(CUtensorMap* map, const void* base, long rows, long cols, long ld_elems,
                   int box_rows);
// Persistent decode stage (stagemk.cu): every layer of a stage-run in one
// cooperative launch, phases separated by grid barriers.
struct MkLayer {
  const void* qkv; const void* o; const void* up; const void* down;   // tiled bf16
  const float* mlp_norm;     // gain of the MLP RMSNorm (O epilogue emits xb)
  const float* gain_next;    // attn_norm of the next layer of the stage (or null)
  void* kc; void* vc;        // this layer's K/V cell rows (bf16)
};
struct MkArgs {
  const MkLayer* layers;
  int nl, m;
  int d, ffn, q_dim, kv_dim, head_dim, H, KH;
  float eps, rope_theta, scale;
  float* x;                  // residual stream f32 [m, d]
  __nv_bfloat16* xb; __nv_bfloat16* attnb; __nv_bfloat16* hb;
  float* q;
  float* ss; int ss_ld, ss_parts0;
  const sp_token* toks; const int32_t* row0_dev;
  const int32_t* vis; const int32_t* vis_len; int ld_vis, nsplit;
  float* att_scratch; int* att_tickets; int att_tstride;   // tickets one L2 line apart when room
  float* scratch; int* tickets; int maxseg;                // (tile tickets: 16 ints apart)
  int* run_state; const int* cancel_table; const RunHdr* hdr;
  unsigned* bar;
  int* err;
  long long* prof;           // SP_MK_PROF: CTA 0's phase edges (site << 56 | clock64)
};
size_t stage_mk_smem();
void stage_mk_occupancy_report();
cudaError_t launch_stage_mk(const CUtensorMap& mxb, const CUtensorMap& mattn,
                            const CUtensorMap& mhb, const MkArgs& a, int ctas, cudaStream_t st);

cudaError_t launch_tc_gemm(const CUtensorMap* xmaps, TcArgs a, cudaStream_t st);
int tc_nt_for(int m);
int tc_gemm_occupancy();
int tc_ksplit(int n_rows, int k, int target_ctas);

}  // namespace sp
