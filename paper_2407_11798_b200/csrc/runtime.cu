// Stage runtime: one pipeline stage (contiguous layer range) on one GPU.
//
// Replaces the stage worker's evaluation path (engine.py:563-623 calling
// model.py:326-421): per run it enqueues, on one in-order stream,
//   gate (cancel/placeholder/chain gate + cell metadata, K3/K14)
//   embed (stage 0, K1) | activation copy
//   plan (K4, once per stage-run, shared by all layers)
//   per layer: QKV GEMV (+norm, RoPE, KV write) -> attention (K5)
//              -> O GEMV (+residual) -> up GEMV (+norm, GELU/SwiGLU)
//              -> down GEMV (+residual, finite check)
//   epilogue (purge of skipped runs, placeholder status)
// and never synchronises with the host.  Cell rows are handed out in run
// order by the host, identically on every stage.
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include <cstdio>
#include <cstring>

#include "kernels.cuh"

namespace sp {

// ---- small kernels ---------------------------------------------------------

// K1 (model.py:352-359): x[i] = E[tok] (+ P[pos]).
template <typename T>
__global__ void embed_kernel(const T* __restrict__ emb,
                             const float* __restrict__ pos_table,
                             const sp_token* __restrict__ toks, int n, int d,
                             int vocab, int max_context, float* __restrict__ x,
                             int* err, const int* run_state) {
  pdl_wait();
  pdl_trigger();
  if (run_skipped(run_state)) return;
  const int i = blockIdx.x;
  const sp_token t = toks[i];
  const bool ok_t = t.token >= 0 && t.token < vocab;
  const bool ok_p = t.pos >= 0 && t.pos < max_context;
  if (threadIdx.x == 0) {
    if (!ok_t) set_error(err, SP_DEV_BAD_TOKEN);
    if (!ok_p) set_error(err, SP_DEV_BAD_POS);
  }
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    float v = ok_t ? to_f32(emb[(size_t)t.token * d + c]) : 0.f;
    if (pos_table != nullptr && ok_p) v = __fadd_rn(v, pos_table[(size_t)t.pos * d + c]);
    x[(size_t)i * d + c] = v;
  }
}

// K1 fused with the tensor-core path's stage input (bf16-only stages whose
// first layer is layer 0): x = E[tok] and, from the same registers, the
// RMSNorm statistic (fixed-order block reduction) and xb = bf16(x * gain) --
// the exact arithmetic of embed_kernel followed by prep_kernel at 256 threads.
__global__ void embed_prep_kernel(const __nv_bfloat16* __restrict__ emb,
                                  const sp_token* __restrict__ toks, int d, int vocab,
                                  int max_context, float* __restrict__ x,
                                  const float* __restrict__ gain, __nv_bfloat16* __restrict__ xb,
                                  float* __restrict__ ss, int* err, const int* run_state) {
  pdl_wait();
  pdl_trigger();
  __shared__ float red[8];
  if (run_skipped(run_state)) return;
  const int i = blockIdx.x;
  const sp_token t = toks[i];
  const bool ok_t = t.token >= 0 && t.token < vocab;
  const bool ok_p = t.pos >= 0 && t.pos < max_context;
  if (threadIdx.x == 0) {
    if (!ok_t) set_error(err, SP_DEV_BAD_TOKEN);
    if (!ok_p) set_error(err, SP_DEV_BAD_POS);
  }
  float s = 0.f;
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    const float v = ok_t ? to_f32(emb[(size_t)t.token * d + c]) : 0.f;
    x[(size_t)i * d + c] = v;
    s = __fmaf_rn(v, v, s);
    xb[(size_t)i * d + c] = __float2bfloat16_rn(gain ? __fmul_rn(v, gain[c]) : v);
  }
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    float tot = red[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) tot = __fadd_rn(tot, red[w]);
    ss[i] = tot;
  }
}

// Stage-run prologue: fold cancel word / upstream placeholder / draft-chain
// gate into run_state, take token 0 from the chain if asked, write metadata.
// Every per-run scalar comes from the device run header, so the same launch
// (or captured graph) serves every run.
__global__ void gate_kernel(const RunHdr* hdr, sp_token* toks, const int* cancel_table,
                            const int* in_status, const int* gate, const int* chain_tip,
                            int* run_state, int32_t* cell_pos, uint32_t* cell_mask,
                            int n_seq, int max_context, int* err,
                            unsigned long long cond) {
  pdl_wait();
  pdl_trigger();
  __shared__ int skip;
  const int n = hdr->n, row0 = hdr->row0, flags = hdr->flags;
  if (threadIdx.x == 0) {
    int s = 0;
    if ((flags & SP_FWD_SKIPPABLE) && hdr->kind == SP_KIND_SPEC) {
      if (cancel_table && hdr->cancel_idx >= 0 &&
          ld_volatile(cancel_table + hdr->cancel_idx) == hdr->run_id)
        s = 1;
      if (in_status && ld_volatile(in_status) == SP_STATUS_PLACEHOLDER) s = 1;
    }
    if ((flags & SP_FWD_CHAIN) && gate && ld_volatile(gate) == 0) s = 1;
    if ((flags & SP_FWD_CHAIN) && chain_tip) toks[0].token = chain_tip[0];
    *run_state = s;
    skip = s;
    // graph-replayed runs: the layers sit in a conditional node that a
    // skipped run does not execute at all
    if (cond) cudaGraphSetConditional((cudaGraphConditionalHandle)cond, s ? 0u : 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const sp_token t = toks[i];
    uint32_t m = t.seq_mask;
    if (n_seq < 32) m &= (1u << n_seq) - 1;
    cell_pos[row0 + i] = t.pos;
    cell_mask[row0 + i] = skip ? 0u : m;
  }
}

// Stage-run epilogue: a skipped/abandoned speculative run purges the
// partitions it wrote under (engine.py:556-561, 581-585, 602-612) and its
// own cells; the outgoing message is a placeholder (engine.py:545-554).
__global__ void epilogue_kernel(const RunHdr* hdr, const sp_token* toks,
                                const int* run_state, const int32_t* cell_pos,
                                uint32_t* cell_mask, int* out_status) {
  pdl_wait();
  pdl_trigger();
  const int skip = ld_volatile(run_state);
  if (!skip) {
    if (out_status && blockIdx.x == 0 && threadIdx.x == 0) *out_status = SP_STATUS_VALID;
    return;
  }
  const int n = hdr->n, row0 = hdr->row0, n_cells = row0 + n;
  uint32_t purge = 0;
  for (int i = 0; i < n; ++i) purge |= toks[i].seq_mask;
  purge &= ~1u;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n_cells;
       r += gridDim.x * blockDim.x) {
    if (r >= row0 && r < row0 + n) cell_mask[r] = 0u;
    else if (purge) cell_mask[r] &= ~purge;
  }
  if (out_status && blockIdx.x == 0 && threadIdx.x == 0) *out_status = SP_STATUS_PLACEHOLDER;
}

__global__ void gather_rows_kernel(const float* __restrict__ x, int d,
                                   const int32_t* __restrict__ rows,
                                   float* __restrict__ out, const int* run_state) {
  pdl_wait();
  pdl_trigger();
  if (run_skipped(run_state)) return;
  const int r = blockIdx.x;
  const float* src = x + (size_t)rows[r] * d;
  for (int c = threadIdx.x; c < d; c += blockDim.x) out[(size_t)r * d + c] = src[c];
}

// Stage input for the tensor-core path: per token, the RMSNorm statistic of
// x (fixed-order block reduction) and the bf16 normed-input row x * gain.
__global__ void prep_kernel(const float* __restrict__ x, int d,
                            const float* __restrict__ gain, __nv_bfloat16* __restrict__ xb,
                            float* __restrict__ ss, const int* run_state,
                            const int32_t* __restrict__ rows) {
  pdl_wait();
  pdl_trigger();
  __shared__ float red[8];
  if (run_skipped(run_state)) return;
  const int t = blockIdx.x;
  const float* xr = x + (size_t)(rows ? rows[t] : t) * d;   // (rows: the LM head's gather)
  float s = 0.f;
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    const float v = xr[c];
    s = __fmaf_rn(v, v, s);
    xb[(size_t)t * d + c] = __float2bfloat16_rn(gain ? __fmul_rn(v, gain[c]) : v);
  }
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    float tot = red[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) tot = __fadd_rn(tot, red[w]);
    ss[t] = tot;
  }
}

// Early inference cancellation (K14): one thread per observation point
// folds the device-visible cancel word into run_state; kernels launched
// after it skip.  A dedicated launch keeps every multi-CTA kernel's view of
// run_state consistent (no mid-kernel flips).
__global__ void observe_kernel(const RunHdr* hdr, const int* cancel_table, int* run_state,
                               unsigned long long cond) {
  pdl_wait();
  pdl_trigger();
  int skip = ld_volatile(run_state);
  if ((hdr->flags & SP_FWD_SKIPPABLE) && hdr->kind == SP_KIND_SPEC && hdr->cancel_idx >= 0 &&
      ld_volatile(cancel_table + hdr->cancel_idx) == hdr->run_id) {
    *run_state = 1;
    skip = 1;
  }
  // graph-replayed runs: the next block of layers sits in its own
  // conditional node -- a run cancelled mid-flight skips the rest outright
  if (cond) cudaGraphSetConditional((cudaGraphConditionalHandle)cond, skip ? 0u : 1u);
}

__global__ void chain_begin_kernel(const int* tip, int* gate, float cutoff,
                                   sp_row_result* out) {
  const int valid = tip[2];
  const float conf = valid ? __int_as_float(tip[1]) : -1.0f;
  *gate = (valid && conf >= cutoff) ? 1 : 0;
  if (out) {
    sp_row_result r;
    r.argmax = valid ? tip[0] : -1;
    r.second = -1;
    r.conf = conf;
    r.max_logit = 0.f;
    *out = r;
  }
}

}  // namespace sp

using namespace sp;

bool sp::pdl_enabled() {
  static const bool on = getenv("SP_NO_PDL") == nullptr;
  return on;
}

struct LayerW {
  const void* qkv = nullptr;
  const void* o = nullptr;
  const void* up = nullptr;
  const void* down = nullptr;
  const float* attn_norm = nullptr;
  const float* mlp_norm = nullptr;
};

// layers between cancel observations / per conditional graph node (each
// observation and IF node breaks the PDL chain: 7B stage-run 2.64 ms at 4/8,
// 2.60 ms at 8/16, and a run cancelled 1 ms in still ends 0.3 ms later)
static int observe_every() {
  static const int v = getenv("SP_OBSERVE_EVERY") ? atoi(getenv("SP_OBSERVE_EVERY")) : 8;
  return v > 0 ? v : 1;
}
static int cond_block() {
  static const int v = getenv("SP_COND_BLOCK") ? atoi(getenv("SP_COND_BLOCK")) : 16;
  return v > 0 ? v : 1;
}

static constexpr int DESC_RING = 64;

struct sp_stage {
  sp_model_dims dims{};
  int lo = 0, hi = 0, cap = 0, max_tokens = 0, n_seq = 0;
  int q_dim = 0, kv_dim = 0, up_rows = 0;
  std::vector<LayerW> layers;
  const void* emb = nullptr;
  const float* pos_table = nullptr;
  const void* w_out = nullptr;
  const void* w_out_tc = nullptr;        // tiled LM head (tensor-core head)
  const float* final_norm = nullptr;
  const int* cancel_table = nullptr;
  int cancel_size = 0;

  bool tc = false;                       // bf16 llama path on tcgen05
  int swz = 0;                           // row-major bf16 weights in SWZ8 layout
  int tc_ctas = 0;                       // CTA budget of the GEMMs (0 = all SMs)
  __nv_bfloat16* xb = nullptr;           // [mt, d]   normed input (x * gain)
  __nv_bfloat16* attnb = nullptr;        // [mt, q]   attention output
  __nv_bfloat16* hb = nullptr;           // [mt, ffn] SwiGLU output
  float* ss = nullptr;                   // [d/128, mt] sum-of-squares partials
  float* tc_scratch = nullptr;
  int* tc_tickets = nullptr;
  CUtensorMap m_xb[2], m_attnb[2], m_hb[2];

  int32_t* cell_pos = nullptr;
  uint32_t* cell_mask = nullptr;
  int n_cells = 0;
  void* kc = nullptr;
  void* vc = nullptr;
  size_t kv_layer_elems = 0;

  float* q = nullptr;
  float* attn = nullptr;
  float* h = nullptr;
  float* xg = nullptr;
  int32_t* vis = nullptr;
  int32_t* vis_len = nullptr;
  int ld_vis = 0;
  float* att_scratch = nullptr;
  size_t att_scratch_floats = 0;
  int* att_tickets = nullptr;
  LmPartial* lm_scratch = nullptr;
  int* lm_ticket = nullptr;
  int* err = nullptr;
  int* run_state = nullptr;
  int* tip = nullptr;   // [argmax, conf bits, valid]
  int* gate = nullptr;

  // run header (device) + its pinned host staging ring
  RunHdr* hdr = nullptr;
  int32_t* hdr_rows = nullptr;           // inside hdr
  sp_token* hdr_toks = nullptr;          // inside hdr
  size_t hdr_bytes = 0;
  uint8_t* hdr_host = nullptr;           // [DESC_RING][hdr_bytes]
  cudaEvent_t ev[DESC_RING];
  int slot = 0;

  // fixed outputs of graph-replayed steps
  float* gx_out = nullptr;               // [max_tokens * d + 4] (x then status)
  sp_row_result* gres = nullptr;         // [1 + max_tokens]: header row + rows
  std::map<std::vector<long>, cudaGraphExec_t> graphs;
  std::map<std::vector<long>, int> seen;
  bool use_graphs = true;
  bool use_cond = true;                  // conditional (IF) body in captured steps
  cudaStream_t body_st = nullptr;

  // K15 draft chain (persistent kernel)
  DraftLayer* dlayers = nullptr;         // device copy of the layer table
  bool dlayers_dirty = true;
  DraftHdr* dhdr = nullptr;
  unsigned* dbar = nullptr;
  int draft_ctas = 0;
  int draft_cluster = 0;
  int draft_kernel = 0;   // SP_DRAFT_KIND_*: 0 = SP_DRAFT_KERNEL env (cluster default)
  int draft_stages = 0;
  long long* dprof = nullptr;            // SP_DRAFT_PROF: phase timestamps
  float* dxb = nullptr;
  float* dopart = nullptr;
  // persistent decode stage (stagemk.cu)
  MkLayer* mklayers = nullptr;           // device copy of the layer table
  bool mk_dirty = true;
  unsigned* mkbar = nullptr;             // grid barrier counter
  int mk_maxseg = 0;
  // cell-pool compaction scratch (lazy)
  int32_t* cp_src = nullptr;
  int32_t* cp_pos = nullptr;
  uint32_t* cp_mask = nullptr;
  int* cp_live = nullptr;
  void* cp_rows = nullptr;

  // last forward (split evaluation continues it)
  int cur_n = 0;
  int cur_row0 = 0;
  int cur_max_pos = 0;
  int cur_flags = 0;
  bool cur_valid = false;
  // caller-supplied attention plan (eval_layers(mask=...)): the next
  // forward uses s->vis/vis_len as uploaded instead of building them
  bool host_plan = false;
};

static int cuda_status(cudaError_t e) { return e == cudaSuccess ? SP_OK : SP_ERR_CUDA; }
// the first failing call of the last failed entry point, for sp_last_error()
static thread_local char g_last_error[320];
static void note_cuda_error(cudaError_t e, const char* what, int line) {
  snprintf(g_last_error, sizeof(g_last_error), "runtime.cu:%d: %s -> %s", line, what,
           cudaGetErrorString(e));
}
extern "C" const char* sp_last_error(void) { return g_last_error; }

#define SP_CHECK(call)                                   \
  do {                                                   \
    cudaError_t _e = (call);                             \
    if (_e != cudaSuccess) {                             \
      note_cuda_error(_e, #call, __LINE__);              \
      return SP_ERR_CUDA;                                \
    }                                                    \
  } while (0)

static size_t wbytes(const sp_model_dims& d) { return d.w_dtype == SP_DTYPE_BF16 ? 2 : 4; }

extern "C" int sp_stage_create(const sp_model_dims* dims, int layer_lo,
                               int layer_hi, int cell_capacity, int max_tokens,
                               int n_seq_ids, sp_stage** out) {
  if (!dims || !out || layer_lo < 0 || layer_hi <= layer_lo ||
      layer_hi > dims->n_layers || cell_capacity <= 0 || max_tokens <= 0 ||
      n_seq_ids < 1 || n_seq_ids > 32)
    return SP_ERR_ARG;
  const sp_model_dims& d = *dims;
  if (d.n_kv_heads <= 0 || d.n_heads % d.n_kv_heads || d.head_dim <= 0)
    return SP_ERR_ARG;
  if (d.head_dim != 8 && d.head_dim != 16 && d.head_dim != 32 && d.head_dim != 64 &&
      d.head_dim != 128)
    return SP_ERR_ARG;
  sp_stage* s = new sp_stage();
  s->dims = d;
  s->lo = layer_lo; s->hi = layer_hi;
  s->cap = cell_capacity; s->max_tokens = max_tokens; s->n_seq = n_seq_ids;
  s->q_dim = d.n_heads * d.head_dim;
  s->kv_dim = d.n_kv_heads * d.head_dim;
  s->up_rows = d.arch == SP_ARCH_LLAMA ? 2 * d.ffn_dim : d.ffn_dim;
  s->layers.resize(layer_hi - layer_lo);
  const int nl = layer_hi - layer_lo;
  s->kv_layer_elems = (size_t)cell_capacity * s->kv_dim;
  s->ld_vis = cell_capacity + 1;
  const size_t wb = wbytes(d);
  const int mt = max_tokens;
  bool ok = true;
  auto alloc = [&](void** p, size_t bytes) {
    if (ok && cudaMalloc(p, bytes) != cudaSuccess) ok = false;
    if (ok) cudaMemset(*p, 0, bytes);
  };
  alloc((void**)&s->cell_pos, sizeof(int32_t) * cell_capacity);
  alloc((void**)&s->cell_mask, sizeof(uint32_t) * cell_capacity);
  alloc(&s->kc, wb * s->kv_layer_elems * nl);
  alloc(&s->vc, wb * s->kv_layer_elems * nl);
  alloc((void**)&s->q, sizeof(float) * (size_t)mt * s->q_dim);
  alloc((void**)&s->attn, sizeof(float) * (size_t)mt * s->q_dim);
  alloc((void**)&s->h, sizeof(float) * (size_t)mt * d.ffn_dim);
  alloc((void**)&s->xg, sizeof(float) * (size_t)mt * d.d_model);
  alloc((void**)&s->vis, sizeof(int32_t) * (size_t)mt * s->ld_vis);
  alloc((void**)&s->vis_len, sizeof(int32_t) * mt);
  s->att_scratch_floats = (size_t)mt * d.n_heads *
                          attn_splits(d.max_context + mt) * (d.head_dim + 2);
  alloc((void**)&s->att_scratch, sizeof(float) * s->att_scratch_floats);
  alloc((void**)&s->att_tickets, sizeof(int) * (size_t)mt * d.n_heads);
  alloc((void**)&s->lm_scratch, sizeof(LmPartial) * (size_t)mt * lmhead_grid(d.vocab));
  alloc((void**)&s->lm_ticket, sizeof(int));
  alloc((void**)&s->err, sizeof(int));
  alloc((void**)&s->run_state, sizeof(int));
  alloc((void**)&s->tip, sizeof(int) * 4);
  alloc((void**)&s->gate, sizeof(int));
  // bf16 (llama) stages run on the tensor-core path with tiled weights
  s->tc = d.arch == SP_ARCH_LLAMA && d.w_dtype == SP_DTYPE_BF16 &&
          d.w_layout == SP_LAYOUT_TC_TILED;
  if (d.w_layout == SP_LAYOUT_TC_TILED && !s->tc) {
    delete s;
    return SP_ERR_ARG;
  }
  if (d.w_layout == SP_LAYOUT_SWZ8) {
    if (d.w_dtype != SP_DTYPE_BF16 || d.d_model % 64 || d.ffn_dim % 64 ||
        (d.n_heads * d.head_dim) % 64) {
      delete s;
      return SP_ERR_ARG;
    }
    s->swz = 1;
  }
  if (s->tc && (d.d_model % 128 || s->q_dim % 128 || (s->q_dim + 2 * s->kv_dim) % 128 ||
                d.ffn_dim % 64)) {
    delete s;
    return SP_ERR_ARG;
  }
  if (s->tc) {
    const int mtp = mt < 128 ? 128 : mt;   // TMA boxes of 128 rows
    alloc((void**)&s->xb, 2 * (size_t)mtp * d.d_model);
    alloc((void**)&s->attnb, 2 * (size_t)mtp * s->q_dim);
    alloc((void**)&s->hb, 2 * (size_t)mtp * d.ffn_dim);
    alloc((void**)&s->ss, sizeof(float) * (size_t)mt * (d.d_model / 128 + 1));
    alloc((void**)&s->tc_scratch, sizeof(float) * (size_t)TC_SCRATCH_FLOATS);
    alloc((void**)&s->tc_tickets, sizeof(int) * TC_TICKETS);
    if (ok) {
      const int boxes[2] = {16, 128};
      for (int i = 0; i < 2 && ok; ++i) {
        ok = make_map_bf16(&s->m_xb[i], s->xb, mtp, d.d_model, d.d_model, boxes[i]) &&
             make_map_bf16(&s->m_attnb[i], s->attnb, mtp, s->q_dim, s->q_dim, boxes[i]) &&
             make_map_bf16(&s->m_hb[i], s->hb, mtp, d.ffn_dim, d.ffn_dim, boxes[i]);
      }
    }
  }
  s->hdr_bytes = sizeof(RunHdr) + sizeof(int32_t) * (size_t)mt + sizeof(sp_token) * (size_t)mt;
  alloc((void**)&s->hdr, s->hdr_bytes);
  if (ok) {
    s->hdr_rows = reinterpret_cast<int32_t*>(s->hdr + 1);
    s->hdr_toks = reinterpret_cast<sp_token*>(s->hdr_rows + mt);
  }
  if (ok && cudaMallocHost((void**)&s->hdr_host, s->hdr_bytes * DESC_RING) != cudaSuccess) ok = false;
  alloc((void**)&s->gx_out, sizeof(float) * ((size_t)mt * d.d_model + 4));
  alloc((void**)&s->gres, sizeof(sp_row_result) * (size_t)(mt + 1));
  s->use_graphs = getenv("SP_NO_GRAPHS") == nullptr;
  s->use_cond = getenv("SP_NO_COND_GRAPH") == nullptr;
  for (int i = 0; ok && i < DESC_RING; ++i)
    if (cudaEventCreateWithFlags(&s->ev[i], cudaEventDisableTiming) != cudaSuccess) ok = false;
  if (ok) ok = cudaDeviceSynchronize() == cudaSuccess;
  if (!ok) {
    sp_stage_destroy(s);
    return SP_ERR_CUDA;
  }
  *out = s;
  return SP_OK;
}

extern "C" int sp_stage_destroy(sp_stage* s) {
  if (!s) return SP_OK;
  cudaDeviceSynchronize();
  void* ptrs[] = {s->cell_pos, s->cell_mask, s->kc, s->vc, s->q, s->attn, s->h,
                  s->xg, s->vis, s->vis_len, s->att_scratch, s->att_tickets,
                  s->lm_scratch, s->lm_ticket, s->err, s->run_state, s->tip,
                  s->gate, s->hdr, s->xb, s->attnb, s->hb, s->ss,
                  s->tc_scratch, s->tc_tickets, s->gx_out, s->gres,
                  s->dlayers, s->dhdr, s->dbar, s->dprof, s->dxb, s->dopart,
                  s->cp_src, s->cp_pos, s->cp_mask, s->cp_live, s->cp_rows,
                  s->mklayers, s->mkbar};
  for (auto& kv : s->graphs) cudaGraphExecDestroy(kv.second);
  if (s->body_st) cudaStreamDestroy(s->body_st);
  for (void* p : ptrs) if (p) cudaFree(p);
  if (s->hdr_host) cudaFreeHost(s->hdr_host);
  for (int i = 0; i < DESC_RING; ++i) if (s->ev[i]) cudaEventDestroy(s->ev[i]);
  delete s;
  return SP_OK;
}

extern "C" int sp_stage_set_embedding(sp_stage* s, const void* emb,
                                      const float* pos_table) {
  if (!s) return SP_ERR_ARG;
  s->emb = emb;
  s->pos_table = pos_table;
  return SP_OK;
}

extern "C" int sp_stage_set_layer(sp_stage* s, int layer, const void* w_qkv,
                                  const void* w_o, const void* w_up,
                                  const void* w_down, const float* attn_norm,
                                  const float* mlp_norm) {
  if (!s || layer < s->lo || layer >= s->hi) return SP_ERR_ARG;
  LayerW& L = s->layers[layer - s->lo];
  L.qkv = w_qkv; L.o = w_o; L.up = w_up; L.down = w_down;
  L.attn_norm = attn_norm; L.mlp_norm = mlp_norm;
  s->dlayers_dirty = true;
  s->mk_dirty = true;
  return SP_OK;
}

extern "C" int sp_stage_set_head(sp_stage* s, const void* w_out,
                                 const float* final_norm) {
  if (!s) return SP_ERR_ARG;
  s->w_out = w_out;
  s->final_norm = final_norm;
  return SP_OK;
}

static void drop_graphs(sp_stage* s);

extern "C" int sp_stage_set_head_tiled(sp_stage* s, const void* w_out_tiled) {
  if (!s) return SP_ERR_ARG;
  if (w_out_tiled && (!s->tc || s->dims.vocab % 128 || s->dims.d_model % 64 ||
                      s->dims.w_dtype != SP_DTYPE_BF16))
    return SP_ERR_ARG;
  if (w_out_tiled != s->w_out_tc) drop_graphs(s);   // captured heads hold the other path
  s->w_out_tc = w_out_tiled;
  return SP_OK;
}

static void drop_graphs(sp_stage* s) {
  for (auto& kv : s->graphs) cudaGraphExecDestroy(kv.second);
  s->graphs.clear();
  s->seen.clear();
}

extern "C" int sp_stage_set_cta_budget(sp_stage* s, int ctas) {
  if (!s || ctas < 0) return SP_ERR_ARG;
  s->tc_ctas = ctas;
  s->mk_dirty = true;   // the persistent stage's grid follows the budget
  drop_graphs(s);
  return SP_OK;
}

extern "C" int sp_stage_set_cancel_table(sp_stage* s, const int* table, int size) {
  if (!s || (table && size <= 0)) return SP_ERR_ARG;
  drop_graphs(s);
  s->cancel_table = table;
  s->cancel_size = size;
  return SP_OK;
}

static int next_slot(sp_stage* s) {
  const int k = s->slot;
  s->slot = (s->slot + 1) % DESC_RING;
  cudaEventSynchronize(s->ev[k]);  // slot reuse: its H2D copy has completed
  return k;
}

// RUN_CONFIG (engine.py:231-251): per-run scalars + descriptor -> the device
// run header, one stream-ordered H2D copy from a pinned ring slot.
static cudaError_t write_hdr(sp_stage* s, const sp_token* toks, int n, int run_id, int kind,
                             int flags, const int32_t* rows, int nrows, float cutoff,
                             cudaStream_t st) {
  const int k = next_slot(s);
  uint8_t* h = s->hdr_host + (size_t)k * s->hdr_bytes;
  RunHdr* rh = reinterpret_cast<RunHdr*>(h);
  int32_t* hr = reinterpret_cast<int32_t*>(rh + 1);
  sp_token* ht = reinterpret_cast<sp_token*>(hr + s->max_tokens);
  rh->row0 = s->n_cells;
  rh->n = n;
  rh->run_id = run_id;
  rh->kind = kind;
  rh->flags = flags;
  rh->nrows = nrows;
  rh->cancel_idx = (s->cancel_table && (flags & SP_FWD_SKIPPABLE) && kind == SP_KIND_SPEC)
                       ? run_id % s->cancel_size : -1;
  rh->cutoff = cutoff;
  for (int i = 0; i < nrows; ++i) hr[i] = rows[i];
  for (int i = 0; i < n; ++i) ht[i] = toks[i];
  const size_t bytes = (const uint8_t*)(ht + n) - h;
  cudaError_t e = cudaMemcpyAsync(s->hdr, h, bytes, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaEventRecord(s->ev[k], st);
  return e;
}

struct RunIO {
  const float* x_in;       // stage input activations (NULL on layer 0)
  const int* in_status;
  float* x_out;
  int* out_status;
};

struct HeadIO {            // fused LM head over the header's rows
  int nrows = 0;
  sp_row_result* out = nullptr;
  int* err_out = nullptr;
  int* status_out = nullptr;
  float* logits = nullptr;
  int update_tip = 0;
  int chain_gate = 0;
};

static int sm_count() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

// The persistent stage kernel (opt-in, SP_STAGE_MK=1) serves decode runs
// (<= 16 tokens) of bf16 llama stages.  Parity-green, but not yet faster than
// the one-GEMM-per-launch chain on the 7B stage.
static bool mk_enabled(const sp_stage* s, int n) {
  static const char* e = getenv("SP_STAGE_MK");
  if (!e || atoi(e) == 0) return false;
  const sp_model_dims& D = s->dims;
  return s->tc && n <= 16 && (D.head_dim == 128 || D.head_dim == 64) && s->mk_maxseg > 0;
}

static int mk_ctas(const sp_stage* s) {
  static const bool noncoop = getenv("SP_MK_NONCOOP") != nullptr;
  if (noncoop) return 2 * sm_count();
  static bool reported = false;
  if (!reported && getenv("SP_MK_VERBOSE")) { reported = true; stage_mk_occupancy_report(); }
  const int sms = sm_count();
  const int c = s->tc_ctas > 0 ? s->tc_ctas / 2 : sms;
  return c < 1 ? 1 : (c > sms ? sms : c);
}

// (Re)build the device layer table; sizes the stream-K merge slots.
static int mk_prepare(sp_stage* s) {
  if (!s->tc) return SP_OK;
  const sp_model_dims& D = s->dims;
  const int nl = s->hi - s->lo;
  if (!s->mkbar) SP_CHECK(cudaMalloc((void**)&s->mkbar, sizeof(unsigned)));
  if (!s->mklayers) SP_CHECK(cudaMalloc((void**)&s->mklayers, sizeof(MkLayer) * nl));
  const size_t wb = wbytes(D);
  std::vector<MkLayer> t(nl);
  for (int i = 0; i < nl; ++i) {
    const LayerW& L = s->layers[i];
    t[i].qkv = L.qkv; t[i].o = L.o; t[i].up = L.up; t[i].down = L.down;
    t[i].mlp_norm = L.mlp_norm;
    t[i].gain_next = i + 1 < nl ? s->layers[i + 1].attn_norm : nullptr;
    t[i].kc = (char*)s->kc + wb * s->kv_layer_elems * i;
    t[i].vc = (char*)s->vc + wb * s->kv_layer_elems * i;
  }
  SP_CHECK(cudaMemcpy(s->mklayers, t.data(), sizeof(MkLayer) * nl, cudaMemcpyHostToDevice));
  // merge slots: a tile of C chunks meets at most ceil(C / q) + 1 ranges
  const int G = mk_ctas(s), d = D.d_model, f = D.ffn_dim;
  const int shapes[4][2] = {{(s->q_dim + 2 * s->kv_dim) / 128, d / 64}, {d / 128, s->q_dim / 64},
                            {2 * f / 128, d / 64}, {d / 128, f / 64}};
  int maxseg = 1, maxtiles = 1;
  for (auto& sh : shapes) {
    const long total = (long)sh[0] * sh[1];
    const long q = total / G;
    if (q < 1) { s->mk_maxseg = 0; s->mk_dirty = false; return SP_OK; }   // too small a stage
    const int segs = (int)((sh[1] + q - 1) / q) + 1;
    maxseg = segs > maxseg ? segs : maxseg;
    maxtiles = sh[0] > maxtiles ? sh[0] : maxtiles;
  }
  const bool fits = (size_t)maxtiles * maxseg * 16 * 128 <= (size_t)TC_SCRATCH_FLOATS &&
                    maxtiles * 16 <= TC_TICKETS && maxseg <= 16;   // MK_MAXSEG
  s->mk_maxseg = fits ? maxseg : 0;
  s->mk_dirty = false;
  return SP_OK;
}

// Enqueue one stage-run (layers [layer_a, layer_b)) reading every per-run
// scalar from the device header.  ``graphable``: no host-dependent launch
// shapes (the attention bound is the context cap) so the sequence can be
// captured once and replayed for any run of the same token count.
static int enqueue_run(sp_stage* s, int n, int layer_a, int layer_b, bool cont,
                       int max_pos, bool coverage, bool graphable, const RunIO& io,
                       const HeadIO* head, cudaStream_t st, cudaStream_t body_st = nullptr) {
  const sp_model_dims& D = s->dims;
  const int d = D.d_model;
  // body_st (capture only): the gate kernel is followed by an IF node whose
  // body -- captured on body_st -- holds the layers; the epilogue and the
  // LM head stay outside (a skipped run still purges and reports)
  unsigned long long cond = 0;
  cudaGraph_t cap_graph = nullptr;
  if (body_st) {
    cudaStreamCaptureStatus cs;
    if (cudaStreamGetCaptureInfo(st, &cs, nullptr, &cap_graph, nullptr, nullptr) != cudaSuccess ||
        cs != cudaStreamCaptureStatusActive)
      return SP_ERR_CUDA;
    cudaGraphConditionalHandle h;
    SP_CHECK(cudaGraphConditionalHandleCreate(&h, cap_graph, 0, 0));
    cond = (unsigned long long)h;
  }
  if (!cont) {
    SP_CHECK(launch_pdl(gate_kernel, dim3(1), dim3(128), 0, st, (const RunHdr*)s->hdr,
                        s->hdr_toks, s->cancel_table, io.in_status,
                        (const int*)s->gate, (const int*)s->tip, s->run_state, s->cell_pos,
                        s->cell_mask, s->n_seq, D.max_context, s->err, cond));
  }
  cudaStream_t outer = st;
  if (body_st) {
    cudaStreamCaptureStatus cs;
    const cudaGraphNode_t* deps = nullptr;
    size_t nd = 0;
    SP_CHECK(cudaStreamGetCaptureInfo(st, &cs, nullptr, nullptr, &deps, &nd));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = (cudaGraphConditionalHandle)cond;
    cp.conditional.type = cudaGraphCondTypeIf;
    cp.conditional.size = 1;
    cudaGraphNode_t cn;
    SP_CHECK(cudaGraphAddNode(&cn, cap_graph, deps, nd, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    SP_CHECK(cudaStreamUpdateCaptureDependencies(st, &cn, 1, cudaStreamSetCaptureDependencies));
    SP_CHECK(cudaStreamBeginCaptureToGraph(body_st, body, nullptr, nullptr, 0,
                                           cudaStreamCaptureModeThreadLocal));
    st = body_st;
  }
  void* stream = reinterpret_cast<void*>(st);
  // tensor-core stages starting at layer 0: embedding + stage input in one pass
  const bool fused_prep = s->tc && layer_a == 0 && s->pos_table == nullptr && d >= 256;
  if (fused_prep) {
    SP_CHECK(launch_pdl(embed_prep_kernel, dim3(n), dim3(256), 0, st,
                        (const __nv_bfloat16*)s->emb, (const sp_token*)s->hdr_toks, d, D.vocab,
                        D.max_context, io.x_out, s->layers[0].attn_norm, s->xb, s->ss, s->err,
                        (const int*)s->run_state));
  } else if (layer_a == 0) {
    const int threads = d >= 256 ? 256 : 64;
    if (D.w_dtype == SP_DTYPE_BF16)
      SP_CHECK(launch_pdl(embed_kernel<__nv_bfloat16>, dim3(n), dim3(threads), 0, st,
                          (const __nv_bfloat16*)s->emb, s->pos_table,
                          (const sp_token*)s->hdr_toks, n, d, D.vocab, D.max_context,
                          io.x_out, s->err, (const int*)s->run_state));
    else
      SP_CHECK(launch_pdl(embed_kernel<float>, dim3(n), dim3(threads), 0, st,
                          (const float*)s->emb, s->pos_table, (const sp_token*)s->hdr_toks,
                          n, d, D.vocab, D.max_context, io.x_out, s->err,
                          (const int*)s->run_state));
  } else if (io.x_in != io.x_out) {
    SP_CHECK(cudaMemcpyAsync(io.x_out, io.x_in, sizeof(float) * (size_t)n * d,
                             cudaMemcpyDeviceToDevice, st));
  }
  if (!cont && !s->host_plan)
    SP_CHECK(launch_plan(s->cell_pos, s->cell_mask, 0, 0, s->hdr_toks, n, D.max_context,
                         s->vis, s->vis_len, s->ld_vis, 0, s->err, st, s->run_state,
                         s->hdr));
  if (!cont) s->host_plan = false;
  // launch bound on visible entries per query (+ self): chain batches see
  // exactly pos cells; a graph must hold for any run (context cap)
  const int bound = graphable ? (D.max_context + s->max_tokens)
                              : (coverage ? (max_pos + 1) : (s->n_cells));
  const int nsplit = attn_splits(bound);
  const size_t need = (size_t)n * D.n_heads * nsplit * (D.head_dim + 2);
  if (need > s->att_scratch_floats) {
    cudaStreamCaptureStatus cs;
    if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone)
      return SP_ERR_CAPACITY;  // the eager first occurrence sizes it
    cudaStreamSynchronize(st);
    drop_graphs(s);  // captured graphs hold the old scratch pointer
    cudaFree(s->att_scratch);
    if (cudaMalloc((void**)&s->att_scratch, sizeof(float) * need) != cudaSuccess)
      return SP_ERR_CUDA;
    s->att_scratch_floats = need;
  }

  const bool llama = D.arch == SP_ARCH_LLAMA;
  const size_t wb = wbytes(D);
  float* x_out = io.x_out;
  const int32_t* row0_dev = &s->hdr->row0;
  if (s->tc && !fused_prep) {
    // bf16 normed input of layer_a's attention norm + its statistic
    SP_CHECK(launch_pdl(prep_kernel, dim3(n), dim3(256), 0, st, (const float*)x_out, d,
                        s->layers[layer_a - s->lo].attn_norm, s->xb, s->ss,
                        (const int*)s->run_state, (const int32_t*)nullptr));
  }
  int ss_parts = 1;
  if (s->tc && s->mk_dirty) {   // layer table + merge slots (never inside a capture)
    cudaStreamCaptureStatus cs;
    if (cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusNone) {
      const int rc = mk_prepare(s);
      if (rc) return rc;
    }
  }
  const bool mk = mk_enabled(s, n);
  if (mk) {
    MkArgs k{};
    k.layers = s->mklayers + (layer_a - s->lo); k.nl = layer_b - layer_a; k.m = n;
    k.d = d; k.ffn = D.ffn_dim; k.q_dim = s->q_dim; k.kv_dim = s->kv_dim;
    k.head_dim = D.head_dim; k.H = D.n_heads; k.KH = D.n_kv_heads;
    k.eps = D.norm_eps; k.rope_theta = D.rope_theta; k.scale = 1.0f / sqrtf((float)D.head_dim);
    k.x = x_out; k.xb = s->xb; k.attnb = s->attnb; k.hb = s->hb; k.q = s->q;
    k.ss = s->ss; k.ss_ld = s->max_tokens; k.ss_parts0 = 1;
    k.toks = s->hdr_toks; k.row0_dev = row0_dev;
    k.vis = s->vis; k.vis_len = s->vis_len; k.ld_vis = s->ld_vis; k.nsplit = nsplit;
    k.att_scratch = s->att_scratch; k.att_tickets = s->att_tickets;
    k.att_tstride = s->max_tokens >= 16 * 16 ? 16 : 1;   // (m <= 16 queries x H heads)
    k.scratch = s->tc_scratch; k.tickets = s->tc_tickets; k.maxseg = s->mk_maxseg;
    k.run_state = s->run_state; k.cancel_table = s->cancel_table; k.hdr = s->hdr;
    k.bar = s->mkbar; k.err = s->err;
    static const bool prof = getenv("SP_MK_PROF") != nullptr;
    if (prof) {
      if (!s->dprof) SP_CHECK(cudaMalloc((void**)&s->dprof, sizeof(long long) * 16384));
      k.prof = s->dprof;
    }
    SP_CHECK(cudaMemsetAsync(s->mkbar, 0, sizeof(unsigned), st));
    SP_CHECK(launch_stage_mk(s->m_xb[0], s->m_attnb[0], s->m_hb[0], k, mk_ctas(s), st));
  }
  for (int l = layer_a; l < (mk ? layer_a : layer_b); ++l) {
    const LayerW& L = s->layers[l - s->lo];
    void* kl = (char*)s->kc + wb * s->kv_layer_elems * (l - s->lo);
    void* vl = (char*)s->vc + wb * s->kv_layer_elems * (l - s->lo);
    AttnArgs a{};
    a.q = s->q; a.k = kl; a.v = vl; a.vis = s->vis; a.vis_len = s->vis_len;
    a.ld_vis = s->ld_vis; a.n = n; a.H = D.n_heads; a.KH = D.n_kv_heads;
    a.nsplit = nsplit; a.scale = 1.0f / sqrtf((float)D.head_dim);
    a.out = s->attn; a.scratch = s->att_scratch; a.tickets = s->att_tickets;
    a.run_state = s->run_state; a.run_state_w = nullptr;
    a.cancel_word = nullptr; a.run_id = 0; a.err = s->err;
    a.fresh_row0_dev = row0_dev;   // the QKV epilogue writes rows row0 .. row0 + n
    a.toks = s->hdr_toks;
    a.hdr = (const RunHdr*)s->hdr;
    a.max_context = D.max_context;
    if (s->tc) {
      // ---- tensor-core path (tcgen05, bf16 activations, fp32 accumulate) ----
      TcArgs t{};
      t.m = n; t.toks = s->hdr_toks; t.err = s->err; t.run_state = s->run_state;
      t.scratch = s->tc_scratch; t.tickets = s->tc_tickets; t.norm_eps = D.norm_eps;
      t.max_ctas = s->tc_ctas;
      t.ss_ld = s->max_tokens;
      // q, k, v (+RoPE, K/V into the cell rows): model.py:387-393
      t.n_rows = s->q_dim + 2 * s->kv_dim; t.k = d; t.epi = SP_EPI_QKV; t.norm = 1;
      t.ss_in = s->ss; t.ss_nparts = ss_parts; t.out = s->q; t.ldo = s->q_dim;
      t.q_rows = s->q_dim; t.kv_rows = s->kv_dim; t.k_cache = kl; t.v_cache = vl;
      t.cache_row0_dev = row0_dev; t.head_dim = D.head_dim; t.rope_theta = D.rope_theta;
      t.w = L.qkv;
      SP_CHECK(launch_tc_gemm(s->m_xb, t, st));
      a.out = reinterpret_cast<float*>(s->attnb); a.out_bf16 = 1;
      SP_CHECK(launch_attention(a, D.w_dtype, D.head_dim, st));
      // x += attn @ Wo, emit bf16(x * mlp_norm) and its statistic
      TcArgs o = t;
      o.n_rows = d; o.k = s->q_dim; o.epi = SP_EPI_RESID; o.norm = 0; o.out = x_out;
      o.ldo = d; o.ss_out = s->ss; o.xb_next = s->xb; o.gain_next = L.mlp_norm;
      o.w = L.o;
      SP_CHECK(launch_tc_gemm(s->m_attnb, o, st));
      ss_parts = d / 128;
      // h = silu(g) * u of rmsnorm(x)
      TcArgs u = t;
      u.n_rows = 2 * D.ffn_dim; u.k = d; u.epi = SP_EPI_SWIGLU; u.norm = 1;
      u.ss_in = s->ss; u.ss_nparts = ss_parts; u.out = s->hb; u.ldo = D.ffn_dim;
      u.w = L.up;
      SP_CHECK(launch_tc_gemm(s->m_xb, u, st));
      // x += h @ Wd (+ finite check), emit the next layer's normed input
      TcArgs dn = t;
      dn.n_rows = d; dn.k = D.ffn_dim; dn.epi = SP_EPI_RESID; dn.norm = 0; dn.out = x_out;
      dn.ldo = d; dn.ss_out = s->ss; dn.xb_next = s->xb;
      dn.gain_next = (l + 1 < s->hi) ? s->layers[l + 1 - s->lo].attn_norm : nullptr;
      dn.w = L.down;
      SP_CHECK(launch_tc_gemm(s->m_hb, dn, st));
    } else {
      // ---- CUDA-core path (fp32 ref arch): weight-streaming GEMV ----
      sp_gemv_args g{};
      g.w_dtype = D.w_dtype;
      g.w_swz = s->swz;
      g.run_state = s->run_state;
      g.err = s->err;
      g.toks = s->hdr_toks;
      g.m = n;
      // q, k, v (model.py:387-393): rmsnorm fused, k/v into cell rows
      g.w = L.qkv; g.n_rows = s->q_dim + 2 * s->kv_dim; g.k = d;
      g.x = x_out; g.ldx = d; g.norm = 1; g.norm_eps = D.norm_eps;
      g.gain = llama ? L.attn_norm : nullptr;
      g.epi = SP_EPI_QKV; g.out = s->q; g.ldo = s->q_dim;
      g.q_rows = s->q_dim; g.kv_rows = s->kv_dim; g.k_cache = kl; g.v_cache = vl;
      g.cache_row0_dev = row0_dev; g.rope = llama ? 1 : 0; g.head_dim = D.head_dim;
      g.rope_theta = D.rope_theta;
      int rc = sp_gemv(&g, stream);
      if (rc) return rc;
      // attention over the plan (model.py:394-415)
      SP_CHECK(launch_attention(a, D.w_dtype, D.head_dim, st));
      // x += attn @ Wo (model.py:416)
      g = sp_gemv_args{};
      g.w_dtype = D.w_dtype; g.w_swz = s->swz; g.run_state = s->run_state; g.err = s->err;
      g.toks = s->hdr_toks;
      g.m = n; g.w = L.o; g.n_rows = d; g.k = s->q_dim; g.x = s->attn; g.ldx = s->q_dim;
      g.norm = 0; g.epi = SP_EPI_RESID; g.out = x_out; g.ldo = d;
      rc = sp_gemv(&g, stream);
      if (rc) return rc;
      // h = act(rmsnorm(x) @ W1) (model.py:417-418)
      g.w = L.up; g.n_rows = s->up_rows; g.k = d; g.x = x_out; g.ldx = d;
      g.norm = 1; g.norm_eps = D.norm_eps; g.gain = llama ? L.mlp_norm : nullptr;
      g.epi = llama ? SP_EPI_SWIGLU : SP_EPI_GELU; g.out = s->h; g.ldo = D.ffn_dim;
      rc = sp_gemv(&g, stream);
      if (rc) return rc;
      // x += h @ W2 (+ finite check, model.py:418-420)
      g.w = L.down; g.n_rows = d; g.k = D.ffn_dim; g.x = s->h; g.ldx = D.ffn_dim;
      g.norm = 0; g.gain = nullptr; g.epi = SP_EPI_RESID; g.out = x_out; g.ldo = d;
      rc = sp_gemv(&g, stream);
      if (rc) return rc;
    }
    // early inference cancellation: observe the cancel word between layers
    // (engine.py:602-612 drains cancels between layers); a no-op for runs
    // that are not cancellable (read from the header)
    if (s->cancel_table && l + 1 < layer_b && ((l + 1 - layer_a) % observe_every()) == 0) {
      const bool block_edge = body_st && ((l + 1 - layer_a) % cond_block()) == 0;
      unsigned long long next = 0;
      if (block_edge) {   // handle of the next block's IF node (resets to 0 per launch)
        cudaGraphConditionalHandle h;
        SP_CHECK(cudaGraphConditionalHandleCreate(&h, cap_graph, 0,
                                                  cudaGraphCondAssignDefault));
        next = (unsigned long long)h;
      }
      SP_CHECK(launch_pdl(observe_kernel, dim3(1), dim3(1), 0, st, (const RunHdr*)s->hdr,
                          s->cancel_table, s->run_state, next));
      if (block_edge) {
        // close this block's body, chain the next IF node in the outer graph
        cudaGraph_t g;
        SP_CHECK(cudaStreamEndCapture(body_st, &g));
        cudaStreamCaptureStatus cs;
        const cudaGraphNode_t* deps = nullptr;
        size_t nd = 0;
        SP_CHECK(cudaStreamGetCaptureInfo(outer, &cs, nullptr, nullptr, &deps, &nd));
        cudaGraphNodeParams cp = {};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = (cudaGraphConditionalHandle)next;
        cp.conditional.type = cudaGraphCondTypeIf;
        cp.conditional.size = 1;
        cudaGraphNode_t cn;
        SP_CHECK(cudaGraphAddNode(&cn, cap_graph, deps, nd, &cp));
        SP_CHECK(cudaStreamUpdateCaptureDependencies(outer, &cn, 1,
                                                     cudaStreamSetCaptureDependencies));
        SP_CHECK(cudaStreamBeginCaptureToGraph(body_st, cp.conditional.phGraph_out[0], nullptr,
                                               nullptr, 0, cudaStreamCaptureModeThreadLocal));
      }
    }
  }
  if (body_st) {
    cudaGraph_t g;
    SP_CHECK(cudaStreamEndCapture(body_st, &g));
    st = outer;
  }
  SP_CHECK(launch_pdl(epilogue_kernel, dim3(max(1, min(148, (s->cap + 255) / 256))),
                      dim3(256), 0, st, (const RunHdr*)s->hdr, (const sp_token*)s->hdr_toks,
                      (const int*)s->run_state, (const int32_t*)s->cell_pos, s->cell_mask,
                      io.out_status));
  if (head && head->nrows > 0) {
    const bool tc_head = s->tc && s->w_out_tc && head->nrows <= s->max_tokens;
    if (!tc_head)
      SP_CHECK(launch_pdl(gather_rows_kernel, dim3(head->nrows), dim3(128), 0, st,
                          (const float*)x_out, d, (const int32_t*)s->hdr_rows, s->xg,
                          (const int*)s->run_state));
    LmArgs m{};
    m.w = s->w_out; m.V = D.vocab; m.d = d; m.x = s->xg; m.n_rows = head->nrows;
    m.norm = 1; m.eps = D.norm_eps;
    m.gain = D.arch == SP_ARCH_LLAMA ? s->final_norm : nullptr;
    m.out = head->out; m.logits = head->logits; m.scratch = s->lm_scratch;
    m.ticket = s->lm_ticket; m.err = s->err; m.err_out = head->err_out;
    m.status_out = head->status_out; m.run_state = s->run_state;
    m.tip = head->update_tip ? s->tip : nullptr;
    m.gate = head->update_tip ? s->gate : nullptr;
    m.chain_gate = head->chain_gate;
    m.hdr = s->hdr;
    m.swz = s->swz;
    if (tc_head) {
      // tensor-core head: the flagged rows gathered as bf16 x*g_final (+ their
      // statistic) into the stage's xb / ss, one tcgen05 GEMM over the tiled
      // head with the fused greedy epilogue -- flat in rows (<= 16 per pass)
      SP_CHECK(launch_pdl(prep_kernel, dim3(head->nrows), dim3(256), 0, st, (const float*)x_out,
                          d, m.gain, s->xb, s->ss, (const int*)s->run_state,
                          (const int32_t*)s->hdr_rows));
      TcArgs h{};
      h.w = s->w_out_tc; h.n_rows = D.vocab; h.k = d; h.m = head->nrows;
      h.epi = SP_EPI_LMHEAD; h.norm = 1; h.norm_eps = D.norm_eps;
      h.out = head->logits; h.ldo = D.vocab;
      h.ss_in = s->ss; h.ss_nparts = 1; h.ss_ld = s->max_tokens;
      h.scratch = s->tc_scratch; h.tickets = s->tc_tickets; h.ksplit = 1;
      h.max_ctas = s->tc_ctas; h.err = s->err; h.run_state = s->run_state;
      h.lm_out = head->out; h.lm_part = s->lm_scratch; h.lm_ticket = s->lm_ticket;
      h.lm_err_out = head->err_out; h.lm_status_out = head->status_out;
      h.lm_tip = m.tip; h.lm_gate = m.gate; h.lm_chain_gate = head->chain_gate;
      h.lm_hdr = s->hdr;
      SP_CHECK(launch_tc_gemm(s->m_xb, h, st));
    } else {
      SP_CHECK(launch_lmhead(m, D.w_dtype, st));
    }
  }
  return SP_OK;
}

static int check_run(sp_stage* s, const sp_token* toks, int n, int layer_a, int layer_b,
                     const float* x_in) {
  if (!s || n <= 0) return SP_ERR_ARG;
  if (layer_a < s->lo || layer_b > s->hi || layer_b <= layer_a) return SP_ERR_MODEL;
  if (n > s->max_tokens) return SP_ERR_CAPACITY;
  if (layer_a == 0 && !s->emb) return SP_ERR_ARG;
  if (layer_a > 0 && !x_in) return SP_ERR_MODEL;  // model.py:361-362
  for (int l = layer_a; l < layer_b; ++l)
    if (!s->layers[l - s->lo].qkv) return SP_ERR_ARG;
  // host-visible token ids and positions are rejected eagerly (the device
  // checks stay for chain-fed tokens): an out-of-range position would index
  // past the RoPE / cache tables before the sticky error is read
  if (toks)
    for (int i = 0; i < n; ++i)
      if (toks[i].pos < 0 || toks[i].pos >= s->dims.max_context || toks[i].token < 0 ||
          toks[i].token >= s->dims.vocab)
        return SP_ERR_MODEL;
  return SP_OK;
}

extern "C" int sp_stage_forward_range(sp_stage* s, const sp_token* host_toks,
                                      int n, int run_id, int kind, int flags,
                                      const float* x_in, const int* in_status,
                                      float* x_out, int* out_status, int chain,
                                      int layer_a, int layer_b, void* stream) {
  if (!s || !x_out) return SP_ERR_ARG;
  if (layer_a < 0) { layer_a = s->lo; layer_b = s->hi; }
  int rc = check_run(s, host_toks, n, layer_a, layer_b, x_in);
  if (rc) return rc;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const bool cont = (flags & SP_FWD_CONTINUE) != 0;
  if (cont && (!s->cur_valid || s->cur_n != n)) return SP_ERR_PROTOCOL;
  if (chain) flags |= SP_FWD_CHAIN;
  int max_pos = 0;
  if (!cont) {
    if (!host_toks || s->n_cells + n > s->cap) return SP_ERR_CAPACITY;
    for (int i = 0; i < n; ++i) max_pos = host_toks[i].pos > max_pos ? host_toks[i].pos : max_pos;
    SP_CHECK(write_hdr(s, host_toks, n, run_id, kind, flags & ~SP_FWD_CONTINUE, nullptr, 0,
                       0.f, st));
    s->cur_n = n; s->cur_row0 = s->n_cells; s->cur_max_pos = max_pos;
    s->cur_flags = flags & ~SP_FWD_CONTINUE; s->cur_valid = true;
    s->n_cells += n;
  } else {
    max_pos = s->cur_max_pos;
  }
  const bool cov = ((cont ? s->cur_flags : flags) & SP_FWD_CHECK_COVERAGE) != 0;
  RunIO io{x_in, in_status, x_out, out_status};
  return enqueue_run(s, n, layer_a, layer_b, cont, max_pos, cov, false, io, nullptr, st);
}

extern "C" int sp_stage_forward(sp_stage* s, const sp_token* host_toks, int n,
                                int run_id, int kind, int flags,
                                const float* x_in, const int* in_status,
                                float* x_out, int* out_status, int chain,
                                void* stream) {
  return sp_stage_forward_range(s, host_toks, n, run_id, kind,
                                flags & ~SP_FWD_CONTINUE, x_in, in_status, x_out,
                                out_status, chain, -1, -1, stream);
}

extern "C" int sp_stage_lmhead(sp_stage* s, const float* x,
                               const int32_t* host_rows, int n_rows,
                               sp_row_result* out, float* logits_out,
                               int* err_out, int update_tip, int chain_gate,
                               float cutoff, void* stream) {
  if (!s || !x || !host_rows || n_rows <= 0 || !out) return SP_ERR_ARG;
  if (s->hi != s->dims.n_layers || !s->w_out) return SP_ERR_ARG;
  if (n_rows > s->max_tokens) return SP_ERR_CAPACITY;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const sp_model_dims& D = s->dims;
  // rows + cutoff into the header (the forward's scalars stay as written)
  const int k = next_slot(s);
  uint8_t* h = s->hdr_host + (size_t)k * s->hdr_bytes;
  int32_t* hr = reinterpret_cast<int32_t*>(h);
  for (int i = 0; i < n_rows; ++i) hr[i] = host_rows[i];
  float* hc = reinterpret_cast<float*>(hr + s->max_tokens);
  *hc = cutoff;
  SP_CHECK(cudaMemcpyAsync(s->hdr_rows, hr, sizeof(int32_t) * n_rows, cudaMemcpyHostToDevice, st));
  SP_CHECK(cudaMemcpyAsync(&s->hdr->cutoff, hc, sizeof(float), cudaMemcpyHostToDevice, st));
  SP_CHECK(cudaEventRecord(s->ev[k], st));
  SP_CHECK(launch_pdl(gather_rows_kernel, dim3(n_rows), dim3(128), 0, st, x, D.d_model,
                      (const int32_t*)s->hdr_rows, s->xg, (const int*)s->run_state));
  LmArgs a{};
  a.w = s->w_out; a.V = D.vocab; a.d = D.d_model; a.x = s->xg; a.n_rows = n_rows;
  a.norm = 1; a.eps = D.norm_eps;
  a.gain = D.arch == SP_ARCH_LLAMA ? s->final_norm : nullptr;
  a.out = out; a.logits = logits_out; a.scratch = s->lm_scratch;
  a.ticket = s->lm_ticket; a.err = s->err; a.err_out = err_out;
  a.run_state = s->run_state;
  a.tip = update_tip ? s->tip : nullptr;
  a.gate = update_tip ? s->gate : nullptr;
  a.chain_gate = chain_gate;
  a.hdr = s->hdr;
  a.swz = s->swz;
  SP_CHECK(launch_lmhead(a, D.w_dtype, st));
  return SP_OK;
}

// One decode/verification stage-run (+ fused LM head) replayed from a
// cached CUDA graph: the run's scalars travel in the header copy, the graph
// reads x_in/in_status (pointers fixed per key) and writes the stage's fixed
// buffers (sp_stage_io).  The first occurrence of a shape runs eagerly, the
// second is captured.
extern "C" int sp_stage_step(sp_stage* s, const sp_token* host_toks, int n, int run_id,
                             int kind, int flags, const int32_t* host_rows, int n_rows,
                             int head_flags, float cutoff, const float* x_in,
                             const int* in_status, void* res_copy, void* stream) {
  int rc = check_run(s, host_toks, n, s ? s->lo : 0, s ? s->hi : 0, x_in);
  if (rc) return rc;
  if (!host_toks || s->n_cells + n > s->cap) return SP_ERR_CAPACITY;
  if (n_rows > 0 && (s->hi != s->dims.n_layers || !s->w_out || !host_rows)) return SP_ERR_ARG;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int d = s->dims.d_model;
  if (head_flags & SP_STEP_CHAIN) flags |= SP_FWD_CHAIN;
  SP_CHECK(write_hdr(s, host_toks, n, run_id, kind, flags & ~SP_FWD_CONTINUE, host_rows,
                     n_rows, cutoff, st));
  s->cur_valid = false;
  int max_pos = 0;
  for (int i = 0; i < n; ++i) max_pos = host_toks[i].pos > max_pos ? host_toks[i].pos : max_pos;
  s->n_cells += n;
  RunIO io{x_in, in_status, s->gx_out, reinterpret_cast<int*>(s->gx_out + (size_t)n * d)};
  HeadIO head;
  head.nrows = n_rows;
  head.out = s->gres + 1;
  head.err_out = &reinterpret_cast<int*>(s->gres)[1];
  head.status_out = &reinterpret_cast<int*>(s->gres)[0];
  head.update_tip = (head_flags & (SP_STEP_TIP | SP_STEP_CHAIN)) ? 1 : 0;
  head.chain_gate = (head_flags & SP_STEP_CHAIN) ? 1 : 0;
  const bool graphable = s->use_graphs && n <= 16;
  if (!graphable) {
    rc = enqueue_run(s, n, s->lo, s->hi, false, max_pos,
                     (flags & SP_FWD_CHECK_COVERAGE) != 0, false, io, &head, st);
  } else {
    const std::vector<long> key = {n, n_rows, head.update_tip, head.chain_gate,
                                   (long)(uintptr_t)x_in, (long)(uintptr_t)in_status};
    auto it = s->graphs.find(key);
    if (it != s->graphs.end()) {
      SP_CHECK(cudaGraphLaunch(it->second, st));
    } else if (s->seen[key]++ == 0) {
      rc = enqueue_run(s, n, s->lo, s->hi, false, max_pos, true, true, io, &head, st);
    } else {
      // capture; the layers go into a conditional (IF) node that the gate
      // kernel switches off for a cancelled run (SP_NO_COND_GRAPH=1: plain)
      cudaGraphExec_t ex = nullptr;
      if (s->use_cond && !s->body_st &&
          cudaStreamCreateWithFlags(&s->body_st, cudaStreamNonBlocking) != cudaSuccess)
        s->use_cond = false;
      for (int attempt = s->use_cond ? 0 : 1; attempt < 2 && !ex; ++attempt) {
        cudaGraph_t g = nullptr;
        SP_CHECK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        rc = enqueue_run(s, n, s->lo, s->hi, false, max_pos, true, true, io, &head, st,
                         attempt == 0 ? s->body_st : nullptr);
        if (rc && attempt == 0) {        // leave both captures cleanly, then plain
          cudaGraph_t junk;
          cudaStreamCaptureStatus cs;
          if (cudaStreamIsCapturing(s->body_st, &cs) == cudaSuccess &&
              cs != cudaStreamCaptureStatusNone)
            cudaStreamEndCapture(s->body_st, &junk);
        }
        cudaError_t e = cudaStreamEndCapture(st, &g);
        if (rc == SP_OK && e == cudaSuccess &&
            cudaGraphInstantiate(&ex, g, 0) == cudaSuccess) {
          cudaGraphDestroy(g);
          break;
        }
        if (g) cudaGraphDestroy(g);
        ex = nullptr;
        cudaGetLastError();
        if (attempt == 1) {
          if (rc) return rc;
          return SP_ERR_CUDA;
        }
        s->use_cond = false;             // conditional capture unsupported here
        rc = SP_OK;
      }
      s->graphs[key] = ex;
      SP_CHECK(cudaGraphLaunch(ex, st));
    }
  }
  if (rc) return rc;
  if (res_copy && n_rows > 0)
    SP_CHECK(cudaMemcpyAsync(res_copy, s->gres, sizeof(sp_row_result) * (1 + n_rows),
                             cudaMemcpyDefault, st));
  return SP_OK;
}

extern "C" int sp_stage_io(sp_stage* s, float** x_out, sp_row_result** res) {
  if (!s) return SP_ERR_ARG;
  if (x_out) *x_out = s->gx_out;
  if (res) *res = s->gres;
  return SP_OK;
}

extern "C" int sp_stage_chain_begin(sp_stage* s, float cutoff, sp_row_result* out,
                                    void* stream) {
  if (!s) return SP_ERR_ARG;
  chain_begin_kernel<<<1, 1, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      s->tip, s->gate, cutoff, out);
  return cuda_status(cudaGetLastError());
}

extern "C" int sp_stage_chain_state(sp_stage* s, int** tip, int** gate) {
  if (!s) return SP_ERR_ARG;
  if (tip) *tip = s->tip;
  if (gate) *gate = s->gate;
  return SP_OK;
}

extern "C" int sp_stage_invalidate_tip(sp_stage* s, void* stream) {
  if (!s) return SP_ERR_ARG;
  return cuda_status(cudaMemsetAsync(s->tip + 2, 0, sizeof(int),
                                     reinterpret_cast<cudaStream_t>(stream)));
}

extern "C" int sp_stage_cache_copy(sp_stage* s, int src, uint32_t dst_mask,
                                   int end_pos, void* stream) {
  if (!s || src < 0 || src >= s->n_seq) return SP_ERR_CACHE;
  if (s->n_seq < 32 && (dst_mask >> s->n_seq)) return SP_ERR_CACHE;
  return cuda_status(launch_copy(s->cell_pos, s->cell_mask, s->n_cells, src,
                                 dst_mask, end_pos, s->dims.max_context,
                                 reinterpret_cast<cudaStream_t>(stream)));
}

extern "C" int sp_stage_cache_remove(sp_stage* s, int seq, int from_pos,
                                     void* stream) {
  if (!s || seq < 0 || seq >= s->n_seq) return SP_ERR_CACHE;
  return cuda_status(launch_remove(s->cell_pos, s->cell_mask, s->n_cells,
                                   1u << seq, from_pos,
                                   reinterpret_cast<cudaStream_t>(stream)));
}

extern "C" int sp_stage_cache_keep(sp_stage* s, int seq, void* stream) {
  if (!s || seq < 0 || seq >= s->n_seq) return SP_ERR_CACHE;
  return cuda_status(launch_keep(s->cell_mask, s->n_cells, seq,
                                 reinterpret_cast<cudaStream_t>(stream)));
}

extern "C" int sp_stage_cache_insert_meta(sp_stage* s, const sp_token* host_toks,
                                          int n, void* stream) {
  // test/diagnostic helper: append cells (metadata only, K/V untouched)
  if (!s || !host_toks || n <= 0) return SP_ERR_ARG;
  if (n > s->max_tokens || s->n_cells + n > s->cap) return SP_ERR_CAPACITY;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  SP_CHECK(write_hdr(s, host_toks, n, 0, SP_KIND_PREFILL, 0, nullptr, 0, 0.f, st));
  s->cur_valid = false;
  SP_CHECK(launch_meta_write(s->cell_pos, s->cell_mask, s->n_cells, s->hdr_toks, n,
                             s->n_seq, s->dims.max_context, s->err, st));
  s->n_cells += n;
  return SP_OK;
}

extern "C" int sp_stage_plan_only(sp_stage* s, const sp_token* host_toks, int n,
                                  int check_coverage, void* stream) {
  // K4/K11 query: the plan a batch WOULD get against the current table
  // (visible rows per query, position order, own row last) without
  // inserting its cells.  Read back with sp_stage_plan_sync.
  if (!s || !host_toks || n <= 0) return SP_ERR_ARG;
  if (n > s->max_tokens || s->n_cells + n > s->cap) return SP_ERR_CAPACITY;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  SP_CHECK(write_hdr(s, host_toks, n, 0, SP_KIND_PREFILL, 0, nullptr, 0, 0.f, st));
  s->cur_valid = false;
  SP_CHECK(launch_plan(s->cell_pos, s->cell_mask, s->n_cells, s->n_cells, s->hdr_toks, n,
                       s->dims.max_context, s->vis, s->vis_len, s->ld_vis,
                       check_coverage, s->err, st));
  return SP_OK;
}

extern "C" int sp_stage_reset(sp_stage* s, void* stream) {
  if (!s) return SP_ERR_ARG;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  SP_CHECK(cudaMemsetAsync(s->cell_mask, 0, sizeof(uint32_t) * s->cap, st));
  SP_CHECK(cudaMemsetAsync(s->tip, 0, sizeof(int) * 4, st));
  s->n_cells = 0;
  s->cur_valid = false;
  return SP_OK;
}

extern "C" int sp_stage_n_cells(const sp_stage* s) { return s ? s->n_cells : -1; }

extern "C" int sp_stage_meta_sync(sp_stage* s, int32_t* host_pos,
                                  uint32_t* host_mask, int cap, void* stream) {
  if (!s || cap < s->n_cells) return SP_ERR_ARG;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (s->n_cells) {
    SP_CHECK(cudaMemcpyAsync(host_pos, s->cell_pos, 4 * s->n_cells, cudaMemcpyDeviceToHost, st));
    SP_CHECK(cudaMemcpyAsync(host_mask, s->cell_mask, 4 * s->n_cells, cudaMemcpyDeviceToHost, st));
  }
  SP_CHECK(cudaStreamSynchronize(st));
  return SP_OK;
}

extern "C" int sp_stage_read_kv_sync(sp_stage* s, int layer, int row,
                                     float* host_k, float* host_v, void* stream) {
  if (!s || layer < s->lo || layer >= s->hi || row < 0 || row >= s->cap)
    return SP_ERR_ARG;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const size_t wb = wbytes(s->dims);
  const size_t off = wb * (s->kv_layer_elems * (layer - s->lo) + (size_t)row * s->kv_dim);
  std::vector<uint16_t> tmp;
  if (wb == 4) {
    SP_CHECK(cudaMemcpyAsync(host_k, (char*)s->kc + off, 4 * s->kv_dim, cudaMemcpyDeviceToHost, st));
    SP_CHECK(cudaMemcpyAsync(host_v, (char*)s->vc + off, 4 * s->kv_dim, cudaMemcpyDeviceToHost, st));
    SP_CHECK(cudaStreamSynchronize(st));
  } else {
    tmp.resize(2 * s->kv_dim);
    SP_CHECK(cudaMemcpyAsync(tmp.data(), (char*)s->kc + off, 2 * s->kv_dim, cudaMemcpyDeviceToHost, st));
    SP_CHECK(cudaMemcpyAsync(tmp.data() + s->kv_dim, (char*)s->vc + off, 2 * s->kv_dim, cudaMemcpyDeviceToHost, st));
    SP_CHECK(cudaStreamSynchronize(st));
    for (int i = 0; i < s->kv_dim; ++i) {
      uint32_t a = (uint32_t)tmp[i] << 16, b = (uint32_t)tmp[s->kv_dim + i] << 16;
      memcpy(host_k + i, &a, 4);
      memcpy(host_v + i, &b, 4);
    }
  }
  return SP_OK;
}

extern "C" int sp_stage_error_sync(sp_stage* s, int clear, void* stream) {
  if (!s) return -1;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  int v = 0;
  if (cudaMemcpyAsync(&v, s->err, sizeof(int), cudaMemcpyDeviceToHost, st) != cudaSuccess) return -1;
  if (cudaStreamSynchronize(st) != cudaSuccess) return -1;
  if (clear) cudaMemsetAsync(s->err, 0, sizeof(int), st);
  return v;
}

extern "C" int sp_stage_error_ptr(sp_stage* s, int** dev_err) {
  if (!s || !dev_err) return SP_ERR_ARG;
  *dev_err = s->err;
  return SP_OK;
}

extern "C" int sp_stage_plan_sync(sp_stage* s, int32_t* host_vis,
                                  int32_t* host_len, int n, void* stream) {
  if (!s || n <= 0 || n > s->max_tokens) return SP_ERR_ARG;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  SP_CHECK(cudaMemcpyAsync(host_len, s->vis_len, 4 * n, cudaMemcpyDeviceToHost, st));
  SP_CHECK(cudaMemcpyAsync(host_vis, s->vis, 4 * (size_t)n * s->ld_vis, cudaMemcpyDeviceToHost, st));
  SP_CHECK(cudaStreamSynchronize(st));
  return SP_OK;
}

extern "C" int sp_stage_ld_vis(const sp_stage* s) { return s ? s->ld_vis : -1; }

extern "C" int sp_stage_set_plan(sp_stage* s, const int32_t* host_vis, const int32_t* host_len,
                                 int n, void* stream) {
  // caller-supplied TreeAttentionMask (model.py:369-373): per query, the
  // rows it attends to in gather order, its own row last; consumed by the
  // next non-continuation forward of this stage (which skips K4)
  if (!s || !host_vis || !host_len || n <= 0 || n > s->max_tokens) return SP_ERR_ARG;
  for (int i = 0; i < n; ++i) {
    if (host_len[i] < 1 || host_len[i] > s->ld_vis || host_len[i] > s->n_cells + n)
      return SP_ERR_ARG;
    for (int j = 0; j < host_len[i]; ++j) {
      const int r = host_vis[(size_t)i * s->ld_vis + j];
      if (r < 0 || r >= s->n_cells + n) return SP_ERR_ARG;
    }
  }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  SP_CHECK(cudaMemcpyAsync(s->vis, host_vis, 4 * (size_t)n * s->ld_vis, cudaMemcpyHostToDevice,
                           st));
  SP_CHECK(cudaMemcpyAsync(s->vis_len, host_len, 4 * (size_t)n, cudaMemcpyHostToDevice, st));
  SP_CHECK(cudaStreamSynchronize(st));   // host buffers are the caller's
  s->host_plan = true;
  return SP_OK;
}

extern "C" int sp_embed(const sp_model_dims* dims, const void* emb,
                        const float* pos_table, const sp_token* toks, int n,
                        float* x, int* err, void* stream) {
  if (!dims || !emb || !toks || n <= 0 || !x) return SP_ERR_ARG;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int d = dims->d_model;
  if (dims->w_dtype == SP_DTYPE_BF16)
    embed_kernel<__nv_bfloat16><<<n, 128, 0, st>>>((const __nv_bfloat16*)emb, pos_table,
                                                   toks, n, d, dims->vocab,
                                                   dims->max_context, x, err, nullptr);
  else
    embed_kernel<float><<<n, 128, 0, st>>>((const float*)emb, pos_table, toks, n, d,
                                           dims->vocab, dims->max_context, x, err,
                                           nullptr);
  return cuda_status(cudaGetLastError());
}

extern "C" int sp_lmhead(const void* w_out, int w_dtype, int vocab, int d,
                         const float* x, const int32_t* rows, int n_rows, int norm,
                         float norm_eps, const float* gain, sp_row_result* out,
                         float* logits_out, float* scratch, int* tickets,
                         int* err, const int* run_state, void* stream) {
  // low-level form: ``rows`` must be NULL (x already holds the n_rows rows
  // contiguously); ``scratch`` needs n_rows * ceil(vocab/8) * 32 bytes.
  if (!w_out || !x || rows || n_rows <= 0 || !out || !scratch || !tickets)
    return SP_ERR_ARG;
  LmArgs a{};
  a.w = w_out; a.V = vocab; a.d = d; a.x = x; a.n_rows = n_rows; a.norm = norm;
  a.eps = norm_eps; a.gain = gain; a.out = out; a.logits = logits_out;
  a.scratch = reinterpret_cast<LmPartial*>(scratch); a.ticket = tickets;
  a.err = err; a.run_state = run_state;
  return cuda_status(launch_lmhead(a, w_dtype, reinterpret_cast<cudaStream_t>(stream)));
}

extern "C" int sp_tc_gemm(const sp_tc_args* a, const void* x, int x_rows, void* stream) {
  if (!a || !a->w || !x || a->n_rows % 128 || a->k % 64 || a->m <= 0 || x_rows < 128)
    return SP_ERR_ARG;
  CUtensorMap mx[2];
  if (!make_map_bf16(&mx[0], x, x_rows, a->k, a->k, 16) ||
      !make_map_bf16(&mx[1], x, x_rows, a->k, a->k, 128))
    return SP_ERR_CUDA;
  return cuda_status(launch_tc_gemm(mx, *a, reinterpret_cast<cudaStream_t>(stream)));
}

extern "C" const char* sp_version(void) { return "specpipe_b200 0.1 sm_100a"; }

extern "C" int sp_device_arch(void) {
  int dev = 0, major = 0, minor = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  return major * 10 + minor;
}

// ---------------------------------------------------------------------------
// Cross-process control plumbing (distributed pipeline, dist.py).
// ---------------------------------------------------------------------------

namespace sp {
// Completion signal for a result block copied into host-mapped memory: the
// copy precedes this kernel in stream order; the flag store is made visible
// system-wide after it (the head polls the flag, then reads the block).
__global__ void signal_kernel(volatile int* flag, int value) {
  __threadfence_system();
  *flag = value;
  __threadfence_system();
}
}  // namespace sp

extern "C" int sp_host_register(void* ptr, size_t bytes, void** dev_ptr) {
  if (!ptr || !bytes || !dev_ptr) return SP_ERR_ARG;
  SP_CHECK(cudaHostRegister(ptr, bytes, cudaHostRegisterPortable | cudaHostRegisterMapped));
  SP_CHECK(cudaHostGetDevicePointer(dev_ptr, ptr, 0));
  return SP_OK;
}

extern "C" int sp_host_unregister(void* ptr) {
  return cuda_status(cudaHostUnregister(ptr));
}

extern "C" int sp_signal(int* dev_flag, int value, void* stream) {
  if (!dev_flag) return SP_ERR_ARG;
  sp::signal_kernel<<<1, 1, 0, reinterpret_cast<cudaStream_t>(stream)>>>(dev_flag, value);
  return cuda_status(cudaGetLastError());
}

extern "C" int sp_copy_async(void* dst, const void* src, size_t bytes, void* stream) {
  return cuda_status(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault,
                                     reinterpret_cast<cudaStream_t>(stream)));
}

// ---------------------------------------------------------------------------
// K15 host side: one cooperative launch per draft request (draft.cu).
// ---------------------------------------------------------------------------
extern "C" int sp_stage_truncate(sp_stage* s, int n_cells) {
  // position-addressed single-sequence stages (the draft): rows >= n_cells
  // are discarded and will be overwritten by the next tokens
  if (!s || n_cells < 0 || n_cells > s->n_cells) return SP_ERR_CACHE;
  s->n_cells = n_cells;
  s->cur_valid = false;
  return SP_OK;
}

// Shapes the persistent draft kernels (draft.cu / draft2.cu) take: a whole
// llama bf16 model with row-major SWZ8 weights, head dim 64/128, and widths
// whose per-CTA slices fit the shared-memory plan (the 160M draft does;
// TinyLlama's ffn 5632 does not -- it runs the per-forward path).
static bool decode_chain_shape_ok(const sp_stage* s) {
  const sp_model_dims& D = s->dims;
  if (D.arch != SP_ARCH_LLAMA || D.w_dtype != SP_DTYPE_BF16 || !s->swz || s->lo != 0 ||
      s->hi != D.n_layers || !s->emb || !s->w_out || !s->final_norm || s->n_seq != 1 ||
      (D.head_dim != 64 && D.head_dim != 128) || D.d_model % 8 || D.ffn_dim % 8 ||
      D.d_model > 2048 || D.ffn_dim > 4096 || D.n_layers > DR_MAX_LAYERS)
    return false;
  for (const LayerW& L : s->layers)
    if (!L.qkv || !L.attn_norm || !L.mlp_norm) return false;
  return true;
}

extern "C" int sp_stage_decode_chain_ok(const sp_stage* s) {
  return s && decode_chain_shape_ok(s) ? 1 : 0;
}

extern "C" int sp_stage_decode_chain(sp_stage* s, const int32_t* feed, int n_feed, int pos0,
                                     const int32_t* step_tokens, int steps, float cutoff,
                                     sp_row_result* out, int* err_out, void* stream) {
  if (!s || !out || n_feed < 0 || n_feed > DR_NT || steps < 0 || steps > DR_MAX_STEPS ||
      (n_feed > 0 && !feed))
    return SP_ERR_ARG;
  const sp_model_dims& D = s->dims;
  if (!decode_chain_shape_ok(s)) return SP_ERR_ARG;
  if (pos0 != s->n_cells) return SP_ERR_PROTOCOL;   // rows == positions
  const int total = n_feed + steps;
  if (s->n_cells + total > s->cap || pos0 + total > D.max_context) return SP_ERR_CAPACITY;
  for (int i = 0; i < n_feed; ++i)
    if (feed[i] < 0 || feed[i] >= D.vocab) return SP_ERR_MODEL;
  if (step_tokens)
    for (int i = 0; i < steps; ++i)
      if (step_tokens[i] < 0 || step_tokens[i] >= D.vocab) return SP_ERR_MODEL;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int L = D.n_layers;
  const int max_split = (s->cap + 127) / 128;
  const size_t need = (size_t)DR_NT * D.n_heads * max_split * (D.head_dim + 2);
  if (!s->dhdr) {
    SP_CHECK(cudaMalloc((void**)&s->dxb, sizeof(float) * DR_NT * D.d_model));
    SP_CHECK(cudaMalloc((void**)&s->dopart, sizeof(float) * DR_NT * D.n_heads * D.d_model));
    SP_CHECK(cudaMalloc((void**)&s->dhdr, sizeof(DraftHdr)));
    SP_CHECK(cudaMalloc((void**)&s->dbar, sizeof(unsigned)));
    SP_CHECK(cudaMalloc((void**)&s->dlayers, sizeof(DraftLayer) * L));
  }
  if (need > s->att_scratch_floats) {
    SP_CHECK(cudaStreamSynchronize(st));
    drop_graphs(s);
    cudaFree(s->att_scratch);
    if (cudaMalloc((void**)&s->att_scratch, sizeof(float) * need) != cudaSuccess)
      return SP_ERR_CUDA;
    s->att_scratch_floats = need;
  }
  const int k = next_slot(s);
  uint8_t* h = s->hdr_host + (size_t)k * s->hdr_bytes;
  if (sizeof(DraftHdr) > s->hdr_bytes) return SP_ERR_CAPACITY;  // max_tokens too small
  if (s->dlayers_dirty) {
    // the layer table rides in the same pinned slot, after the header
    DraftLayer* hl = reinterpret_cast<DraftLayer*>(h + sizeof(DraftHdr));
    if (sizeof(DraftHdr) + sizeof(DraftLayer) * L > s->hdr_bytes) {
      std::vector<DraftLayer> tmp(L);
      for (int l = 0; l < L; ++l) {
        const LayerW& W = s->layers[l];
        tmp[l] = DraftLayer{(const __nv_bfloat16*)W.qkv, (const __nv_bfloat16*)W.o,
                            (const __nv_bfloat16*)W.up, (const __nv_bfloat16*)W.down,
                            W.attn_norm, W.mlp_norm};
      }
      SP_CHECK(cudaStreamSynchronize(st));
      SP_CHECK(cudaMemcpy(s->dlayers, tmp.data(), sizeof(DraftLayer) * L,
                          cudaMemcpyHostToDevice));
    } else {
      for (int l = 0; l < L; ++l) {
        const LayerW& W = s->layers[l];
        hl[l] = DraftLayer{(const __nv_bfloat16*)W.qkv, (const __nv_bfloat16*)W.o,
                           (const __nv_bfloat16*)W.up, (const __nv_bfloat16*)W.down,
                           W.attn_norm, W.mlp_norm};
      }
      SP_CHECK(cudaMemcpyAsync(s->dlayers, hl, sizeof(DraftLayer) * L, cudaMemcpyHostToDevice,
                               st));
    }
    s->dlayers_dirty = false;
  }
  DraftHdr* hh = reinterpret_cast<DraftHdr*>(h);
  std::memset(hh, 0, sizeof(DraftHdr));
  hh->n_feed = n_feed;
  hh->steps = steps;
  hh->pos0 = pos0;
  hh->row0 = s->n_cells;
  hh->chain = step_tokens ? 0 : 1;
  hh->cutoff = cutoff;
  for (int i = 0; i < n_feed; ++i) hh->tok[i] = feed[i];
  if (step_tokens)
    for (int i = 0; i < steps; ++i) hh->tok[n_feed + i] = step_tokens[i];
  SP_CHECK(cudaMemcpyAsync(s->dhdr, hh, sizeof(DraftHdr), cudaMemcpyHostToDevice, st));
  SP_CHECK(cudaMemsetAsync(s->dbar, 0, sizeof(unsigned), st));
  SP_CHECK(cudaEventRecord(s->ev[k], st));

  DraftArgs a{};
  a.layers = s->dlayers; a.L = L; a.V = D.vocab; a.d = D.d_model; a.H = D.n_heads;
  a.KH = D.n_kv_heads; a.hd = D.head_dim; a.f = D.ffn_dim; a.eps = D.norm_eps;
  a.theta = D.rope_theta;
  a.emb = (const __nv_bfloat16*)s->emb; a.w_out = (const __nv_bfloat16*)s->w_out;
  a.g_final = s->final_norm;
  a.kc = (__nv_bfloat16*)s->kc; a.vc = (__nv_bfloat16*)s->vc;
  a.kv_layer_elems = s->kv_layer_elems;
  a.cell_pos = s->cell_pos; a.cell_mask = s->cell_mask;
  a.hdr = s->dhdr; a.tip = s->tip; a.gate = s->gate;
  a.x = s->xg; a.q = s->q; a.attn = s->attn; a.h = s->h;
  a.att_part = s->att_scratch; a.att_tick = s->att_tickets; a.max_split = max_split;
  a.lm_part = s->lm_scratch; a.bar = s->dbar;
  a.xb = s->dxb; a.opart = s->dopart;
  a.out = out; a.err = s->err; a.err_out = err_out;
  if (getenv("SP_DRAFT_PROF")) {
    if (!s->dprof) SP_CHECK(cudaMalloc((void**)&s->dprof, sizeof(long long) * 16384));
    a.prof = s->dprof;
  }
  a.spin_ns = getenv("SP_DRAFT_SPIN_NS") ? (unsigned)atoi(getenv("SP_DRAFT_SPIN_NS")) : 32u;
  const char* kind = getenv("SP_DRAFT_KERNEL");
  const bool grid = s->draft_kernel == SP_DRAFT_KIND_GRID ||
                    (s->draft_kernel == SP_DRAFT_KIND_AUTO && kind && std::strcmp(kind, "grid") == 0);
  if (grid) {
    if (s->draft_ctas <= 0) {
      int dev = 0, sms = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      const char* env = getenv("SP_DRAFT_CTAS");
      int want = env ? atoi(env) : sms;
      if (want <= 0 || want > sms) want = sms;
      draft_buffers(a, want);
      if (draft_smem_bytes(a) > 200 * 1024) return SP_ERR_ARG;   // shape too wide
      if (draft_max_ctas(a) < want) return SP_ERR_ARG;
      s->draft_ctas = want;
    }
    draft_buffers(a, s->draft_ctas);
    SP_CHECK(launch_draft_chain(a, s->draft_ctas, st));
  } else {
    // cluster form (default): one cluster of 16 (else 8) SMs
    if (s->q_dim + 2 * s->kv_dim > D.ffn_dim) return SP_ERR_ARG;   // q|k|v staging in h
    {   // a stage holds 16 padded rows of the short matrices (one tensor-core
        // tile) and at least a pair of the long (down) rows
      const long kx = s->q_dim > D.d_model ? s->q_dim : D.d_model;
      long rb = 16 * (2 * kx);
      const long rl = 2 * (2L * D.ffn_dim);
      if (rl > rb) rb = rl;
      a.ring_bytes = (int)((rb + 127) / 128 * 128);
    }
    const size_t budget = 200 * 1024;
    if (s->draft_cluster <= 0) {
      // size the ring for the widest launch (4 fed tokens) to pick the cluster
      const size_t act4 = draft2_act_bytes(a, 16, DR_NT);
      if (act4 + 2 * (size_t)a.ring_bytes > budget) return SP_ERR_ARG;   // shape too wide
      a.ring_stages = (int)((budget - act4) / a.ring_bytes);
      a.nt = DR_NT;
      const char* env = getenv("SP_DRAFT_CLUSTER");
      s->draft_cluster = draft2_cluster_size(a, env ? atoi(env) : 16);
      if (s->draft_cluster <= 0) return SP_ERR_ARG;
    }
    // a launch with one fed token (every chain launch) gets a deeper ring
    const int nt = n_feed > 1 ? n_feed : 1;
    const size_t act = draft2_act_bytes(a, s->draft_cluster, nt);
    a.ring_stages = (int)((budget - act) / a.ring_bytes);
    if (a.ring_stages > 16) a.ring_stages = 16;
    a.nt = nt;
    a.use_mma = getenv("SP_DRAFT_MMA") && atoi(getenv("SP_DRAFT_MMA")) == 1;
    a.diag_nocompute = getenv("SP_DRAFT_DIAG_NOCOMPUTE") != nullptr;
    SP_CHECK(launch_draft_cluster(a, s->draft_cluster, st));
  }
  s->n_cells += total;
  s->cur_valid = false;
  return SP_OK;
}

extern "C" int sp_stage_set_skip_graphs(sp_stage* s, int on) {
  if (!s) return SP_ERR_ARG;
  const bool want = on != 0 && getenv("SP_NO_COND_GRAPH") == nullptr;
  if (want != s->use_cond) {
    if (cudaDeviceSynchronize() != cudaSuccess) return SP_ERR_CUDA;
    drop_graphs(s);     // captured steps hold the other structure
    s->use_cond = want;
  }
  return SP_OK;
}

extern "C" int sp_stage_set_draft_kernel(sp_stage* s, int kind) {
  if (!s || kind < SP_DRAFT_KIND_AUTO || kind > SP_DRAFT_KIND_GRID) return SP_ERR_ARG;
  s->draft_kernel = kind;
  return SP_OK;
}

extern "C" int sp_stage_draft_profile(sp_stage* s, long long* host, int max) {
  // diagnostics: timestamps (ns) of the last decode_chain's phase edges
  if (!s || !host || max <= 0) return SP_ERR_ARG;
  if (!s->dprof) return 0;
  if (cudaDeviceSynchronize() != cudaSuccess) return -SP_ERR_CUDA;
  long long n = 0;
  if (cudaMemcpy(&n, s->dprof, sizeof(n), cudaMemcpyDeviceToHost) != cudaSuccess)
    return -SP_ERR_CUDA;
  if (n > max) n = max;
  if (cudaMemcpy(host, s->dprof + 1, sizeof(long long) * n, cudaMemcpyDeviceToHost) !=
      cudaSuccess)
    return -SP_ERR_CUDA;
  return (int)n;
}

// ---------------------------------------------------------------------------
// Cell-pool compaction: the reference's cache grows without bound; here the
// pool is bounded, so dead cells (purged / removed runs) are reclaimed by a
// stable compaction at a quiescent point of the stage's stream.  Synchronous:
// returns the new cell count (>= 0) or -error.
// ---------------------------------------------------------------------------
extern "C" int sp_stage_compact(sp_stage* s, void* stream) {
  if (!s) return -SP_ERR_ARG;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (s->n_cells == 0) return 0;
  const size_t kvrow = wbytes(s->dims) * (size_t)s->kv_dim;
  if (!s->cp_src) {
    if (cudaMalloc((void**)&s->cp_src, sizeof(int32_t) * s->cap) != cudaSuccess ||
        cudaMalloc((void**)&s->cp_pos, sizeof(int32_t) * s->cap) != cudaSuccess ||
        cudaMalloc((void**)&s->cp_mask, sizeof(uint32_t) * s->cap) != cudaSuccess ||
        cudaMalloc((void**)&s->cp_live, sizeof(int)) != cudaSuccess ||
        cudaMalloc(&s->cp_rows, kvrow * s->cap) != cudaSuccess)
      return -SP_ERR_CUDA;
  }
  if (launch_compact_scan(s->cell_pos, s->cell_mask, s->n_cells, s->cp_src, s->cp_pos,
                          s->cp_mask, s->cp_live, st) != cudaSuccess)
    return -SP_ERR_CUDA;
  int live = 0;
  if (cudaMemcpyAsync(&live, s->cp_live, sizeof(int), cudaMemcpyDeviceToHost, st) !=
          cudaSuccess || cudaStreamSynchronize(st) != cudaSuccess)
    return -SP_ERR_CUDA;
  if (cudaMemcpyAsync(s->cell_pos, s->cp_pos, sizeof(int32_t) * live, cudaMemcpyDeviceToDevice,
                      st) != cudaSuccess ||
      cudaMemcpyAsync(s->cell_mask, s->cp_mask, sizeof(uint32_t) * live,
                      cudaMemcpyDeviceToDevice, st) != cudaSuccess ||
      cudaMemsetAsync(s->cell_mask + live, 0, sizeof(uint32_t) * (s->n_cells - live), st) !=
          cudaSuccess)
    return -SP_ERR_CUDA;
  const int nl = s->hi - s->lo;
  for (int l = 0; l < nl; ++l) {
    for (int kv = 0; kv < 2; ++kv) {
      char* base = (char*)(kv ? s->vc : s->kc) + wbytes(s->dims) * s->kv_layer_elems * l;
      if (launch_compact_gather(base, s->cp_rows, s->cp_src, s->cp_live, (int)kvrow, live, st) !=
              cudaSuccess ||
          cudaMemcpyAsync(base, s->cp_rows, kvrow * live, cudaMemcpyDeviceToDevice, st) !=
              cudaSuccess)
        return -SP_ERR_CUDA;
    }
  }
  if (cudaStreamSynchronize(st) != cudaSuccess) return -SP_ERR_CUDA;
  s->n_cells = live;
  s->cur_valid = false;
  return live;
}
