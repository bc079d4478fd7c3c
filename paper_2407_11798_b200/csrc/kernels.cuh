// Launch interfaces shared by the kernel translation units and the runtime.
#pragma once

#include <cuda.h>

#include "common.cuh"

namespace sp {

typedef sp_tc_args TcArgs;

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
  int* gate;
  int chain_gate;
  float cutoff;
};

cudaError_t launch_plan(const int32_t* cell_pos, const uint32_t* cell_mask,
                        int n_old, int row0, const sp_token* toks, int n,
                        int max_context, int32_t* vis, int32_t* vis_len,
                        int ld_vis, int check_cov, int* err, cudaStream_t st,
                        const int* run_state = nullptr);
cudaError_t launch_attention(const AttnArgs& a, int kv_dtype, int hd,
                             cudaStream_t st);
int attn_splits(int max_len);
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
bool make_map_bf16(CUtensorMap* map, const void* base, long rows, long cols, long ld_elems,
                   int box_rows);
cudaError_t launch_tc_gemm(const CUtensorMap* xmaps, TcArgs a, cudaStream_t st);
int tc_nt_for(int m);
int tc_ksplit(int n_rows, int k, int target_ctas);

}  // namespace sp
