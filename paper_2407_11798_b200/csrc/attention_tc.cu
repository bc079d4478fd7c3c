// K5 (bf16 KV cache, head dim 64/128): tree-masked attention on the tensor
// cores, one CTA per (KV head, chunk of 64 plan entries).
//
// model.py:394-415 per query q and head h: softmax(q.K_vis^T * scale) V_vis
// over the query's visible rows in plan order.  Layout on B200:
//
//  * the unit of work is (kv head kh, chunk c): plan entries [64c, 64c+64)
//    of every query of the run.  Within a run the plans of a chain are
//    nested (query j's plan is the first len_j entries of the longest one),
//    so the chunk's K and V rows are gathered ONCE into shared memory
//    (cp.async 16 B, XOR-swizzled for conflict-free ldmatrix) and serve
//    every query and every q head of kh (GQA: H/KH heads share the K/V
//    bytes).  Queries whose chunk differs (tree siblings) get their own
//    staging pass;
//  * the rows (query j, q head) of kh are M tiles of 16: scores
//    S = Q K^T and O = P V run as mma.sync m16n8k16 bf16 with fp32
//    accumulation.  q (fp32) and P are split into bf16 hi + lo parts (two
//    MMAs each), so the products carry ~2^-16 relative error, not bf16's;
//  * each (row, chunk) leaves a partial (max, sum, O) -- the last CTA of a
//    KV head merges the chunks of each row in chunk order.  A row's result
//    depends only on its own plan (fixed 64-entry chunks, fixed MMA and
//    shuffle order): batch-, tree- and split-invariant, like the CUDA-core
//    kernel it replaces for bf16 caches.
#include "kernels.cuh"

namespace sp {

constexpr int AT_C = 64;          // plan entries per chunk
constexpr int AT_THREADS = 128;   // 4 warps

__device__ __forceinline__ uint32_t at_s(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void at_cp16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void at_cp_commit_wait() {
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&v);
}
// hi/lo split of two floats into packed bf16x2 pairs
__device__ __forceinline__ void split2(float a, float b, uint32_t& hi, uint32_t& lo) {
  const __nv_bfloat16 ah = __float2bfloat16_rn(a), bh = __float2bfloat16_rn(b);
  __nv_bfloat162 h;
  h.x = ah;
  h.y = bh;
  hi = *reinterpret_cast<const uint32_t*>(&h);
  lo = pack_bf16(__fsub_rn(a, __bfloat162float(ah)), __fsub_rn(b, __bfloat162float(bh)));
}
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// One 16-row tile against the staged chunk, all four warps: warp w owns
// chunk entries [16w, 16w+16) -- its scores (2 n-tiles), its share of the
// chunk max / sum, and its k-step of P V; the four partial O's are summed
// in warp order through shared memory.  Row r of the tile is (query j,
// head h); entries >= the row's plan length are masked.  Writes each live
// row's partial (max, sum, O) to scratch, or its final output when the
// row's plan has a single chunk.
template <int HD>
__device__ __forceinline__ void at_tile(const AttnArgs& a, uint32_t kbase, uint32_t vbase, int c,
                                        int row0, int nrows, int G, int kh,
                                        const int* __restrict__ mem, int grp,
                                        float (*sred)[2][16], float* sO) {
  constexpr int U = HD / 8;         // 16-byte units per K/V row
  constexpr int KS = HD / 16;       // k steps of the score MMA
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  int rj[2], rh[2], rlen[2];
  bool live[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int r = row0 + g + 8 * q;
    live[q] = r < nrows;
    rj[q] = live[q] ? r / G : 0;
    rh[q] = kh * G + (live[q] ? r % G : 0);
    rlen[q] = live[q] ? a.vis_len[rj[q]] - c * AT_C : 0;   // entries of this chunk it sees
    if (live[q] && mem[rj[q]] != grp) rlen[q] = 0;          // another staging group's row
    if (rlen[q] <= 0) live[q] = false;
  }
  // Q fragments (scaled, split hi/lo) straight from the fp32 q rows
  uint32_t qa_h[KS][4], qa_l[KS][4];
#pragma unroll
  for (int k = 0; k < KS; ++k)
#pragma unroll
    for (int hf = 0; hf < 2; ++hf)         // columns 2t.. (a0/a1) and 2t+8.. (a2/a3)
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        float x0 = 0.f, x1 = 0.f;
        if (live[q]) {
          const float2 v = *reinterpret_cast<const float2*>(
              a.q + (size_t)rj[q] * a.H * HD + (size_t)rh[q] * HD + 16 * k + 8 * hf + 2 * t);
          x0 = v.x * a.scale;
          x1 = v.y * a.scale;
        }
        split2(x0, x1, qa_h[k][hf * 2 + q], qa_l[k][hf * 2 + q]);
      }
  // S for this warp's 16 entries (n-tiles 2w, 2w+1)
  float s[2][4];
#pragma unroll
  for (int nn = 0; nn < 2; ++nn)
#pragma unroll
    for (int i = 0; i < 4; ++i) s[nn][i] = 0.f;
#pragma unroll
  for (int nn = 0; nn < 2; ++nn) {
#pragma unroll
    for (int k = 0; k < KS; k += 2) {
      const int er = (2 * w + nn) * 8 + (lane & 7);
      const int uu = 2 * k + (lane >> 3);
      uint32_t b[4];
      asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                   : "=r"(b[0]), "=r"(b[1]), "=r"(b[2]), "=r"(b[3])
                   : "r"(kbase + (uint32_t)(er * U + (uu ^ (er & 7))) * 16));
      mma16816(s[nn], qa_h[k], b[0], b[1]);
      mma16816(s[nn], qa_l[k], b[0], b[1]);
      mma16816(s[nn], qa_h[k + 1], b[2], b[3]);
      mma16816(s[nn], qa_l[k + 1], b[2], b[3]);
    }
  }
  float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
  for (int nn = 0; nn < 2; ++nn)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int q = i >> 1, e = (2 * w + nn) * 8 + 2 * t + (i & 1);
      if (e >= rlen[q]) s[nn][i] = -INFINITY;
      mx[q] = fmaxf(mx[q], s[nn][i]);
    }
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    mx[q] = fmaxf(mx[q], __shfl_xor_sync(0xffffffffu, mx[q], 1));
    mx[q] = fmaxf(mx[q], __shfl_xor_sync(0xffffffffu, mx[q], 2));
  }
  if (t == 0) {
    sred[w][0][g] = mx[0];
    sred[w][0][g + 8] = mx[1];
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < 2; ++q) {    // chunk max, warps in order
    float m = sred[0][0][g + 8 * q];
#pragma unroll
    for (int ww = 1; ww < 4; ++ww) m = fmaxf(m, sred[ww][0][g + 8 * q]);
    mx[q] = m;
  }
  float ls[2] = {0.f, 0.f};
  uint32_t ph[4], pl[4];           // P of this warp's 16 entries: one A fragment
#pragma unroll
  for (int nn = 0; nn < 2; ++nn) {
    float p[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int q = i >> 1;
      p[i] = (s[nn][i] == -INFINITY) ? 0.f : __expf(s[nn][i] - mx[q]);
      ls[q] = __fadd_rn(ls[q], p[i]);
    }
    split2(p[0], p[1], ph[nn * 2 + 0], pl[nn * 2 + 0]);
    split2(p[2], p[3], ph[nn * 2 + 1], pl[nn * 2 + 1]);
  }
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    ls[q] = __fadd_rn(ls[q], __shfl_xor_sync(0xffffffffu, ls[q], 1));
    ls[q] = __fadd_rn(ls[q], __shfl_xor_sync(0xffffffffu, ls[q], 2));
  }
  if (t == 0) {
    sred[w][1][g] = ls[0];
    sred[w][1][g + 8] = ls[1];
  }
  // this warp's P V over all HD dims -> sO[w][row][dim]
#pragma unroll
  for (int nd = 0; nd < HD / 8; nd += 2) {
    const int er = 16 * w + (lane & 15);
    const int uu = nd + (lane >> 4);
    uint32_t b[4];
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(b[0]), "=r"(b[1]), "=r"(b[2]), "=r"(b[3])
                 : "r"(vbase + (uint32_t)(er * U + (uu ^ (er & 7))) * 16));
    float o[2][4];
#pragma unroll
    for (int x = 0; x < 2; ++x)
#pragma unroll
      for (int i = 0; i < 4; ++i) o[x][i] = 0.f;
    mma16816(o[0], ph, b[0], b[1]);
    mma16816(o[0], pl, b[0], b[1]);
    mma16816(o[1], ph, b[2], b[3]);
    mma16816(o[1], pl, b[2], b[3]);
#pragma unroll
    for (int x = 0; x < 2; ++x) {
      const int d0 = (nd + x) * 8 + 2 * t;
      *reinterpret_cast<float2*>(sO + ((size_t)w * 16 + g) * HD + d0) = make_float2(o[x][0], o[x][1]);
      *reinterpret_cast<float2*>(sO + ((size_t)w * 16 + g + 8) * HD + d0) =
          make_float2(o[x][2], o[x][3]);
    }
  }
  __syncthreads();
  // warps in order: O and sum of each row; partial or final output
  for (int idx = tid; idx < 16 * HD; idx += AT_THREADS) {
    const int rr = idx / HD, dd = idx % HD;
    const int r = row0 + rr;
    if (r >= nrows) continue;
    const int j = r / G, h = kh * G + r % G;
    if (mem[j] != grp || a.vis_len[j] <= c * AT_C) continue;
    float o = sO[(size_t)rr * HD + dd];
    float l = sred[0][1][rr];
#pragma unroll
    for (int ww = 1; ww < 4; ++ww) {
      o = __fadd_rn(o, sO[((size_t)ww * 16 + rr) * HD + dd]);
      l = __fadd_rn(l, sred[ww][1][rr]);
    }
    const size_t row = (size_t)j * a.H + h;
    const int nch = (a.vis_len[j] + AT_C - 1) / AT_C;
    if (nch == 1) {   // = the chunk-order merge of one partial (weights exp(0) = 1)
      const float v = o / l;
      if (a.out_bf16) reinterpret_cast<__nv_bfloat16*>(a.out)[row * HD + dd] = __float2bfloat16_rn(v);
      else a.out[row * HD + dd] = v;
    } else {
      float* sp = a.scratch + (row * a.nsplit + c) * (HD + 2);
      sp[2 + dd] = o;
      if (dd == 0) {
        float m = sred[0][0][rr];
#pragma unroll
        for (int ww = 1; ww < 4; ++ww) m = fmaxf(m, sred[ww][0][rr]);
        sp[0] = m;
        sp[1] = l;
      }
    }
  }
  __syncthreads();   // sred / sO are reused by the next tile
}

template <int HD>
__global__ void __launch_bounds__(AT_THREADS) attn_tc_kernel(const AttnArgs a) {
  constexpr int U = HD / 8;
  constexpr int CHUNK_BYTES = AT_C * HD * 2;
  extern __shared__ __align__(128) uint8_t at_smem[];
  uint8_t* KV = at_smem;                                              // [2 bufs][K | V]
  float* sO = reinterpret_cast<float*>(at_smem + 4 * CHUNK_BYTES);     // [4][16][HD]
  int* mem = reinterpret_cast<int*>(sO + 4 * 16 * HD);                // [n] staging group
  __shared__ int srows[2][AT_C];
  __shared__ float sred[4][2][16];
  __shared__ int s_ref, s_last;

  const int kh = blockIdx.x;
  const int G = a.H / a.KH;
  const int kvd = a.KH * HD;
  const int nrows = a.n * G;
  const int tid = threadIdx.x, warp = tid >> 5;
  const __nv_bfloat16* Kc = reinterpret_cast<const __nv_bfloat16*>(a.k) + (size_t)kh * HD;
  const __nv_bfloat16* Vc = reinterpret_cast<const __nv_bfloat16*>(a.v) + (size_t)kh * HD;

  // Before the dependency wait: the plan (built at the start of the
  // stage-run) and the K/V rows of cells older than this run are final; only
  // rows >= fresh0 come from the QKV kernel this launch depends on.  The old
  // rows of this CTA's first chunk stream in while QKV drains.
  if (tid == 0) {   // reference query: the longest plan (ties: the last)
    int best = 0, bl = -1;
    for (int j = 0; j < a.n; ++j) {
      const int l = a.vis_len[j];
      if (l >= bl) { bl = l; best = j; }
    }
    s_ref = best;
  }
  __syncthreads();
  const int ref = s_ref;
  const int ref_len = a.vis_len[ref];
  const int nch = (ref_len + AT_C - 1) / AT_C;
  if ((int)blockIdx.y >= nch) {
    if (blockIdx.y == 0 && tid == 0) set_error(a.err, SP_DEV_PLAN_OVERFLOW);   // (empty plan)
    return;
  }
  const int32_t* pref = a.vis + (size_t)ref * a.ld_vis;
  const int fresh0 = a.fresh_row0_dev ? *a.fresh_row0_dev : a.fresh_row0;

  // gather chunk c of ``plan`` into buffer b (cp.async, not waited here);
  // part 1 = rows < fresh0 only, 2 = rows >= fresh0 only, 0 = all
  auto issue = [&](const int32_t* plan, int len, int c, int b, int part) {
    const int e0 = c * AT_C;
    if (part != 2) {
      for (int e = tid; e < AT_C; e += AT_THREADS)
        srows[b][e] = e0 + e < len ? plan[e0 + e] : plan[e0];
      __syncthreads();
    }
    const uint32_t kb = at_s(KV + (size_t)b * 2 * CHUNK_BYTES), vb = kb + CHUNK_BYTES;
    for (int i = tid; i < AT_C * U; i += AT_THREADS) {
      const int er = i / U, u = i % U;
      const int row = srows[b][er];
      if ((part == 1 && row >= fresh0) || (part == 2 && row < fresh0)) continue;
      const size_t off = (size_t)row * kvd + u * 8;
      const uint32_t pu = (uint32_t)(er * U + (u ^ (er & 7))) * 16;
      at_cp16(kb + pu, Kc + off);
      at_cp16(vb + pu, Vc + off);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };

  const bool pre = fresh0 > 0 && !run_skipped(a.run_state);   // (a stale 0 only wastes a load)
  if (pre) issue(pref, ref_len, blockIdx.y, 0, 1);
  pdl_wait();
  pdl_trigger();
  if (a.diag_empty || run_skipped(a.run_state)) {
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    return;
  }
  if (blockIdx.y == 0 && tid == 0 && nch > a.nsplit) set_error(a.err, SP_DEV_PLAN_OVERFLOW);
  issue(pref, ref_len, blockIdx.y, 0, pre ? 2 : 0);

  int buf = 0;
  for (int c = blockIdx.y; c < nch; c += gridDim.y) {
    // staging groups: 0 = queries whose chunk entries equal the reference's
    const int e0 = c * AT_C;
    for (int j = warp; j < a.n; j += AT_THREADS / 32) {
      const int lj = a.vis_len[j];
      const int32_t* pj = a.vis + (size_t)j * a.ld_vis;
      const int hi = min(lj, e0 + AT_C);
      bool same = true;
      for (int e = e0 + (tid & 31); e < hi; e += 32) same &= pj[e] == pref[e];
      same = __all_sync(0xffffffffu, same);
      if ((tid & 31) == 0) mem[j] = (lj <= e0) ? -1 : (same ? 0 : 1 + j);
    }
    const int cn = c + gridDim.y;
    if (cn < nch) {      // next chunk's rows stream in while this one computes
      issue(pref, ref_len, cn, buf ^ 1, 0);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const uint32_t kb = at_s(KV + (size_t)buf * 2 * CHUNK_BYTES), vb = kb + CHUNK_BYTES;
    for (int t0 = 0; t0 < nrows; t0 += 16)
      at_tile<HD>(a, kb, vb, c, t0, nrows, G, kh, mem, 0, sred, sO);
    // queries with a chunk of their own (tree siblings): one staging each
    for (int j = 0; j < a.n; ++j) {
      if (mem[j] != 1 + j) continue;            // (uniform across the CTA)
      asm volatile("cp.async.wait_group 0;" ::: "memory");
      issue(a.vis + (size_t)j * a.ld_vis, a.vis_len[j], c, buf, 0);
      asm volatile("cp.async.wait_group 0;" ::: "memory");
      __syncthreads();
      for (int t0 = j * G; t0 < (j + 1) * G; t0 += 16)
        at_tile<HD>(a, kb, vb, c, t0, (j + 1) * G, G, kh, mem, 1 + j, sred, sO);
    }
    buf ^= 1;
  }

  if (nch <= 1) return;     // single-chunk rows were written directly
  // the last CTA of this KV head merges the multi-chunk rows in chunk order
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = atomicAdd(&a.tickets[kh], 1) == min((int)gridDim.y, nch) - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // (1) every row's chunk statistics into shared memory (the K/V buffers
  // are free now), loads all in flight; (2) per row the chunk weights
  // exp(m_c - M) and L in chunk order; (3) per (row, dim) the weighted sum,
  // loads batched 8 at a time.  Same arithmetic order as before: a row's
  // bits do not depend on which CTA merges.
  const bool fits = ((size_t)2 * nrows * a.nsplit + nrows) * sizeof(float) <= 4 * (size_t)CHUNK_BYTES;
  const int rbmax = fits ? nrows : 1;                 // rows per merge batch
  float* smw = reinterpret_cast<float*>(KV);          // [rbmax][nsplit] m -> weight
  float* sml = smw + (size_t)rbmax * a.nsplit;        // [rbmax][nsplit] l
  float* sL = sml + (size_t)rbmax * a.nsplit;         // [rbmax] L
  for (int r0 = 0; r0 < nrows; r0 += 1) {
    // rows are merged in batches that fit the buffers (all rows when decoding)
    int rb = nrows - r0;
    if (!fits) rb = 1;
    for (int idx = tid; idx < rb * a.nsplit; idx += AT_THREADS) {
      const int rr = idx / a.nsplit, cc = idx % a.nsplit;
      const int r = r0 + rr, j = r / G, h = kh * G + r % G;
      const int nc = (a.vis_len[j] + AT_C - 1) / AT_C;
      if (nc <= 1 || cc >= nc) continue;
      const float* b = a.scratch + (((size_t)j * a.H + h) * a.nsplit + cc) * (HD + 2);
      smw[(size_t)rr * a.nsplit + cc] = __ldcg(b);
      sml[(size_t)rr * a.nsplit + cc] = __ldcg(b + 1);
    }
    __syncthreads();
    for (int rr = tid; rr < rb; rr += AT_THREADS) {
      const int r = r0 + rr, j = r / G;
      const int nc = (a.vis_len[j] + AT_C - 1) / AT_C;
      if (nc <= 1) continue;
      float* wv = smw + (size_t)rr * a.nsplit;
      const float* lv = sml + (size_t)rr * a.nsplit;
      float M = -INFINITY;
      for (int cc = 0; cc < nc; ++cc) M = fmaxf(M, wv[cc]);
      float L = 0.f;
      for (int cc = 0; cc < nc; ++cc) {
        const float wgt = __expf(wv[cc] - M);
        wv[cc] = wgt;
        L = __fadd_rn(L, __fmul_rn(lv[cc], wgt));
      }
      sL[rr] = L;
    }
    __syncthreads();
    for (int idx = tid; idx < rb * HD; idx += AT_THREADS) {
      const int rr = idx / HD, dd = idx % HD;
      const int r = r0 + rr, j = r / G, h = kh * G + r % G;
      const int nc = (a.vis_len[j] + AT_C - 1) / AT_C;
      if (nc <= 1) continue;
      const size_t row = (size_t)j * a.H + h;
      const float* base = a.scratch + row * a.nsplit * (HD + 2) + 2 + dd;
      const float* wv = smw + (size_t)rr * a.nsplit;
      float o = 0.f;
      for (int c0 = 0; c0 < nc; c0 += 8) {
        float v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k)
          v[k] = c0 + k < nc ? __ldcg(base + (size_t)(c0 + k) * (HD + 2)) : 0.f;
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (c0 + k < nc) o = __fadd_rn(o, __fmul_rn(v[k], wv[c0 + k]));
      }
      const float val = o / sL[rr];
      if (a.out_bf16) reinterpret_cast<__nv_bfloat16*>(a.out)[row * HD + dd] = __float2bfloat16_rn(val);
      else a.out[row * HD + dd] = val;
    }
    __syncthreads();
    r0 += rb - 1;
  }
  if (tid == 0) a.tickets[kh] = 0;
}

template <int HD>
static cudaError_t launch_tc_hd(const AttnArgs& a, cudaStream_t st) {
  const size_t smem = 4 * (size_t)AT_C * HD * 2 + sizeof(float) * 4 * 16 * HD +
                      sizeof(int) * (size_t)a.n;
  static size_t configured = 0;
  if (configured < smem) {
    cudaError_t e = cudaFuncSetAttribute(attn_tc_kernel<HD>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  // one CTA per (KV head, chunk) up to ~8 per SM of work units; longer
  // contexts loop in-CTA (double-buffered), so one launch shape serves any
  // context (graph replay); CTAs past the run's chunk count exit at once
  const int z = max(1, min(a.nsplit, (8 * 148 + a.KH - 1) / a.KH));
  return launch_pdl(attn_tc_kernel<HD>, dim3(a.KH, z), dim3(AT_THREADS), smem, st, a);
}

// Which kernel a launch of n queries takes.  Measured (tools/attn_bench.py,
// profiles/r02_attention.txt): on decode-sized runs the CUDA-core kernel is
// faster (7B ctx 1024: 15.1 vs 20.6 us; 70B GQA: 20.8 vs 30.9 us) -- one
// 16-row MMA tile is mostly padding there and the chunk's phases do not
// overlap -- so the tensor-core kernel takes prefill-sized runs (n >= 32),
// where it also holds at any context.  The switch depends on n only and
// lies above every speculative run (<= 10 tokens), so verification and
// iterative decoding stay bit-identical.  SP_ATT_TC=1 / SP_ATT_LEGACY=1 force
// one kernel (experiments).
bool attn_tc_ok(int kv_dtype, int hd, int n) {
  static const bool legacy = getenv("SP_ATT_LEGACY") != nullptr;
  static const bool force = getenv("SP_ATT_TC") != nullptr;
  if (legacy || kv_dtype != SP_DTYPE_BF16 || (hd != 64 && hd != 128)) return false;
  return force || n >= 32;
}

cudaError_t launch_attention_tc(const AttnArgs& a, int hd, cudaStream_t st) {
  return hd == 64 ? launch_tc_hd<64>(a, st) : launch_tc_hd<128>(a, st);
}

}  // namespace sp
