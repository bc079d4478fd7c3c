// K5 (bf16 KV cache, head dim 64/128): tree-masked attention on the tensor
// cores for prefill-sized runs (see attn_tc_ok for the measured split with
// the CUDA-core kernel).
//
// model.py:394-415 per query q and head h: softmax(q.K_vis^T * scale) V_vis
// over the query's visible rows in plan order.  Layout on B200:
//
//  * grid (KV head kh, z): each of a CTA's four warps walks its own chunks
//    of 64 plan entries (chunk wz, wz + W, ...; W warps per KV head).  Within
//    a run the plans of a chain are nested (a query on the reference
//    query's sequence set sees a prefix of its plan), so the chunk's K and V
//    rows are gathered ONCE into the warp's shared memory (cp.async 16 B,
//    XOR-swizzled for conflict-free ldmatrix; the old rows of the first
//    chunk before the dependency wait) and serve every query and every q
//    head of kh (GQA: H/KH heads share the K/V bytes).  Queries whose chunk
//    differs (tree siblings) get their own gather;
//  * the rows (query j, q head) of kh are M tiles of 16: S = Q K^T and
//    O = P V run as mma.sync m16n8k16 bf16 with fp32 accumulation; q (fp32)
//    and P are split into bf16 hi + lo parts (two MMAs each), so products
//    carry ~2^-16 relative error, not bf16's (max |err| vs fp32 <= 1e-6,
//    tools/attn_bench.py);
//  * each (row, chunk) leaves a partial (max, sum, O); the rows are merged
//    in chunk order -- by the last CTA of the KV head for <= 32 rows, else by
//    attn_merge_kernel, one CTA per row, same arithmetic.  A row's result
//    depends only on its own plan (fixed 64-entry chunks, fixed MMA and
//    shuffle order): batch-, tree- and split-invariant.
#include "kernels.cuh"

namespace sp {

constexpr int AT_C = 64;          // plan entries per chunk
constexpr int AT_MERGE_ROWS = 32; // (query, head) rows per KV head merged in-kernel
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
  asm(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// Staging group of query j for chunk c: 0 when its chunk entries are the
// reference query's (always so for a query on the reference's sequence
// set: its plan is a prefix of the reference's), -1 when its plan ends
// before the chunk, else 1 + j (its own gather).
__device__ __forceinline__ int at_group(const AttnArgs& a, int j, int c, int ref_mask,
                                        const int32_t* pref) {
  const int lj = a.vis_len[j];
  const int e0 = c * AT_C;
  if (lj <= e0) return -1;
  if (ref_mask != 0 && (int)a.toks[j].seq_mask == ref_mask) return 0;
  const int32_t* pj = a.vis + (size_t)j * a.ld_vis;
  const int hi = min(lj, e0 + AT_C);
  bool same = true;
  for (int e = e0 + (threadIdx.x & 31); e < hi; e += 32) same &= pj[e] == pref[e];
  return __all_sync(0xffffffffu, same) ? 0 : 1 + j;
}

// One warp, one 16-row tile against its staged chunk (64 entries).  Row r
// of the tile is (query j, head h) = (r / G, kh*G + r % G); entries >= the
// row's plan length are masked.  Leaves each live row's partial (max, sum,
// O) for chunk c in scratch, or its final output when the row's plan has a
// single chunk.  The arithmetic of a (row, chunk) is fixed: it does not
// depend on the tile's other rows, on which warp / CTA runs it or on n.
template <int HD>
__device__ __forceinline__ void at_tile(const AttnArgs& a, uint32_t kbase, uint32_t vbase, int c,
                                        int row0, int nrows, int G, int kh, int grp,
                                        int ref_mask, const int32_t* pref) {
  constexpr int U = HD / 8;         // 16-byte units per K/V row
  constexpr int KS = HD / 16;       // k steps of the score MMA
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  // staging group of each query in the tile (warp-uniform calls)
  int rgrp[2] = {-2, -2};
  {
    int prev_j = -1, prev_g = -2;
    for (int rr = 0; rr < 16; ++rr) {
      const int r = row0 + rr;
      if (r >= nrows) break;
      const int jj = r / G;
      if (jj != prev_j) {
        prev_g = at_group(a, jj, c, ref_mask, pref);
        prev_j = jj;
      }
      if (rr == g) rgrp[0] = prev_g;
      if (rr == g + 8) rgrp[1] = prev_g;
    }
  }
  int rj[2], rh[2], rlen[2];
  bool live[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int r = row0 + g + 8 * q;
    live[q] = r < nrows;
    rj[q] = live[q] ? r / G : 0;
    rh[q] = kh * G + (live[q] ? r % G : 0);
    rlen[q] = live[q] ? a.vis_len[rj[q]] - c * AT_C : 0;   // entries of this chunk it sees
    if (live[q] && rgrp[q] != grp) rlen[q] = 0;              // another staging group's row
    if (rlen[q] <= 0) live[q] = false;
  }
  if (!__any_sync(0xffffffffu, live[0] || live[1])) return;
  uint32_t qa_h[KS][4], qa_l[KS][4];   // Q fragments (scaled, split hi/lo)
#pragma unroll
  for (int k = 0; k < KS; ++k)
#pragma unroll
    for (int hf = 0; hf < 2; ++hf)
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
  // S = Q K^T: k steps outer, the 8 independent n-tile accumulators inner
  float s[8][4];
#pragma unroll
  for (int n = 0; n < 8; ++n)
#pragma unroll
    for (int i = 0; i < 4; ++i) s[n][i] = 0.f;
#pragma unroll
  for (int k = 0; k < KS; k += 2) {
    uint32_t b[8][4];
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      const int er = n * 8 + (lane & 7);
      const int uu = 2 * k + (lane >> 3);
      asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                   : "=r"(b[n][0]), "=r"(b[n][1]), "=r"(b[n][2]), "=r"(b[n][3])
                   : "r"(kbase + (uint32_t)(er * U + (uu ^ (er & 7))) * 16));
    }
#pragma unroll
    for (int n = 0; n < 8; ++n) mma16816(s[n], qa_h[k], b[n][0], b[n][1]);
#pragma unroll
    for (int n = 0; n < 8; ++n) mma16816(s[n], qa_l[k], b[n][0], b[n][1]);
#pragma unroll
    for (int n = 0; n < 8; ++n) mma16816(s[n], qa_h[k + 1], b[n][2], b[n][3]);
#pragma unroll
    for (int n = 0; n < 8; ++n) mma16816(s[n], qa_l[k + 1], b[n][2], b[n][3]);
  }
  float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
  for (int n = 0; n < 8; ++n)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int q = i >> 1, e = n * 8 + 2 * t + (i & 1);
      if (e >= rlen[q]) s[n][i] = -INFINITY;
      mx[q] = fmaxf(mx[q], s[n][i]);
    }
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    mx[q] = fmaxf(mx[q], __shfl_xor_sync(0xffffffffu, mx[q], 1));
    mx[q] = fmaxf(mx[q], __shfl_xor_sync(0xffffffffu, mx[q], 2));
  }
  float ls[2] = {0.f, 0.f};
  uint32_t ph[4][4], pl[4][4];      // P as A fragments, 4 k steps of 16 entries
#pragma unroll
  for (int n = 0; n < 8; ++n) {
    float p[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int q = i >> 1;
      p[i] = (s[n][i] == -INFINITY) ? 0.f : __expf(s[n][i] - mx[q]);
      ls[q] = __fadd_rn(ls[q], p[i]);
    }
    const int k = n >> 1, hf = n & 1;
    split2(p[0], p[1], ph[k][hf * 2 + 0], pl[k][hf * 2 + 0]);
    split2(p[2], p[3], ph[k][hf * 2 + 1], pl[k][hf * 2 + 1]);
  }
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    ls[q] = __fadd_rn(ls[q], __shfl_xor_sync(0xffffffffu, ls[q], 1));
    ls[q] = __fadd_rn(ls[q], __shfl_xor_sync(0xffffffffu, ls[q], 2));
  }
  int nchr[2];
  size_t rowi[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    nchr[q] = live[q] ? (a.vis_len[rj[q]] + AT_C - 1) / AT_C : 0;
    rowi[q] = (size_t)rj[q] * a.H + rh[q];
    if (live[q] && t == 0 && nchr[q] > 1) {
      float* sp = a.scratch + (rowi[q] * a.nsplit + c) * (HD + 2);
      sp[0] = mx[q];
      sp[1] = ls[q];
    }
  }
  // O = P V, 16 dims at a time (4 independent accumulators per step)
#pragma unroll
  for (int nd = 0; nd < HD / 8; nd += 2) {
    float o[2][2][4];   // [n-tile][hi/lo][4]: hi and lo chains accumulate apart
#pragma unroll
    for (int x = 0; x < 2; ++x)
#pragma unroll
      for (int y = 0; y < 2; ++y)
#pragma unroll
        for (int i = 0; i < 4; ++i) o[x][y][i] = 0.f;
    uint32_t b[4][4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int er = 16 * k + (lane & 15);
      const int uu = nd + (lane >> 4);
      asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                   : "=r"(b[k][0]), "=r"(b[k][1]), "=r"(b[k][2]), "=r"(b[k][3])
                   : "r"(vbase + (uint32_t)(er * U + (uu ^ (er & 7))) * 16));
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      mma16816(o[0][0], ph[k], b[k][0], b[k][1]);
      mma16816(o[1][0], ph[k], b[k][2], b[k][3]);
      mma16816(o[0][1], pl[k], b[k][0], b[k][1]);
      mma16816(o[1][1], pl[k], b[k][2], b[k][3]);
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      if (!live[q]) continue;
#pragma unroll
      for (int x = 0; x < 2; ++x) {
        const int d0 = (nd + x) * 8 + 2 * t;
        const float v0 = __fadd_rn(o[x][0][q * 2 + 0], o[x][1][q * 2 + 0]);
        const float v1 = __fadd_rn(o[x][0][q * 2 + 1], o[x][1][q * 2 + 1]);
        if (nchr[q] == 1) {   // = the chunk-order merge of one partial (weight exp(0) = 1)
          const float f0 = v0 / ls[q], f1 = v1 / ls[q];
          if (a.out_bf16)
            *reinterpret_cast<uint32_t*>(reinterpret_cast<__nv_bfloat16*>(a.out) + rowi[q] * HD + d0) =
                pack_bf16(f0, f1);
          else
            *reinterpret_cast<float2*>(a.out + rowi[q] * HD + d0) = make_float2(f0, f1);
        } else {
          float* sp = a.scratch + (rowi[q] * a.nsplit + c) * (HD + 2);
          *reinterpret_cast<float2*>(sp + 2 + d0) = make_float2(v0, v1);
        }
      }
    }
  }
}

template <int HD>
__global__ void __launch_bounds__(AT_THREADS) attn_tc_kernel(const AttnArgs a) {
  constexpr int U = HD / 8;
  constexpr int CHUNK_BYTES = AT_C * HD * 2;
  constexpr int NW = AT_THREADS / 32;
  extern __shared__ __align__(128) uint8_t at_smem[];   // per warp: [K | V] of one chunk
  __shared__ int s_ref, s_last;

  const int kh = blockIdx.x;
  const int G = a.H / a.KH;
  const int kvd = a.KH * HD;
  const int nrows = a.n * G;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const __nv_bfloat16* Kc = reinterpret_cast<const __nv_bfloat16*>(a.k) + (size_t)kh * HD;
  const __nv_bfloat16* Vc = reinterpret_cast<const __nv_bfloat16*>(a.v) + (size_t)kh * HD;
  const uint32_t kb = at_s(at_smem + (size_t)warp * 2 * CHUNK_BYTES), vb = kb + CHUNK_BYTES;

  // Before the dependency wait: the plan (built at the start of the
  // stage-run) and the K/V rows of cells older than this run are final; only
  // rows >= fresh0 come from the QKV kernel this launch depends on.  Each
  // warp's first chunk streams its old rows in while QKV drains.
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
  // (0: compare plans; a coverage-checked run's masks decide nesting)
  const int ref_mask = (a.toks != nullptr && a.hdr != nullptr &&
                        (a.hdr->flags & SP_FWD_CHECK_COVERAGE))
                           ? (int)a.toks[ref].seq_mask : 0;
  const int nch = (ref_len + AT_C - 1) / AT_C;
  const int wz = blockIdx.y * NW + warp, W = gridDim.y * NW;   // this warp's chunks: wz + i*W
  // row blocks (grid z, prefill-sized runs): this CTA's 16-row tiles
  // [tb0, tb1); every (row, chunk) is still computed exactly once
  const int ntiles = (nrows + 15) / 16;
  const int tpb = (ntiles + gridDim.z - 1) / gridDim.z;
  const int tb0 = blockIdx.z * tpb, tb1 = min(ntiles, tb0 + tpb);
  if ((int)blockIdx.y * NW >= nch) return;                      // no chunk for this CTA
  const int32_t* pref = a.vis + (size_t)ref * a.ld_vis;
  const int fresh0 = a.fresh_row0_dev ? *a.fresh_row0_dev : a.fresh_row0;

  // gather chunk c of ``plan`` into this warp's buffer; part 1 = rows <
  // fresh0 only, 2 = rows >= fresh0 only, 0 = all (cp.async, committed)
  auto issue = [&](const int32_t* plan, int len, int c, int part) {
    const int e0 = c * AT_C;
    // the chunk's 64 row indices: two loads per lane, all in flight at once
    const int i0 = e0 + lane, i1 = e0 + 32 + lane;
    const int rw0 = plan[i0 < len ? i0 : e0], rw1 = plan[i1 < len ? i1 : e0];
    // lanes [0, U) copy K units, [U, 2U) V units; 32 / 2U entries per step
    constexpr int EPS = 32 / (2 * U);
    const int sub = lane / (2 * U), l2 = lane % (2 * U);
    const bool isv = l2 >= U;
    const int u = isv ? l2 - U : l2;
    const __nv_bfloat16* base = isv ? Vc : Kc;
    const uint32_t dst = isv ? vb : kb;
#pragma unroll 4
    for (int e = 0; e < AT_C; e += EPS) {
      const int ee = e + sub;
      const int src = __shfl_sync(0xffffffffu, ee < 32 ? rw0 : rw1, ee & 31);
      if ((part == 1 && src >= fresh0) || (part == 2 && src < fresh0)) continue;
      at_cp16(dst + (uint32_t)(ee * U + (u ^ (ee & 7))) * 16, base + (size_t)src * kvd + u * 8);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };

  const bool pre = wz < nch && fresh0 > 0 && !run_skipped(a.run_state);
  if (pre) issue(pref, ref_len, wz, 1);
  pdl_wait();
  pdl_trigger();
  if (a.diag_empty || run_skipped(a.run_state)) {
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    return;
  }
  if (blockIdx.y == 0 && blockIdx.z == 0 && tid == 0 && nch > a.nsplit)
    set_error(a.err, SP_DEV_PLAN_OVERFLOW);

  for (int c = wz; c < nch; c += W) {
    issue(pref, ref_len, c, (c == wz && pre) ? 2 : 0);
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncwarp();
    for (int t0 = tb0 * 16; t0 < tb1 * 16; t0 += 16)
      at_tile<HD>(a, kb, vb, c, t0, nrows, G, kh, 0, ref_mask, pref);
    // queries with a chunk of their own (tree siblings): one gather each
    for (int j = 0; j < a.n; ++j) {
      if ((j * G) / 16 < tb0 || (j * G) / 16 >= tb1) continue;   // another row block's query
      const int gj = at_group(a, j, c, ref_mask, pref);
      if (gj != 1 + j) continue;
      __syncwarp();
      issue(a.vis + (size_t)j * a.ld_vis, a.vis_len[j], c, 0);
      asm volatile("cp.async.wait_group 0;" ::: "memory");
      __syncwarp();
      for (int t0 = j * G; t0 < (j + 1) * G; t0 += 16)
        at_tile<HD>(a, kb, vb, c, t0, (j + 1) * G, G, kh, 1 + j, ref_mask, pref);
    }
    __syncwarp();
  }

  if (nch <= 1) return;     // single-chunk rows were written directly
  if (nrows > AT_MERGE_ROWS) return;   // many rows: attn_merge_kernel merges them
  // the last CTA of this KV head merges the multi-chunk rows in chunk order
  __threadfence();
  __syncthreads();
  const int active = min((int)gridDim.y, (nch + NW - 1) / NW);
  if (tid == 0) s_last = atomicAdd(&a.tickets[kh], 1) == active - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // (1) every row's chunk statistics into shared memory, loads all in
  // flight; (2) per row the chunk weights exp(m_c - M) and L in chunk order;
  // (3) per (row, dim) the weighted sum, loads batched 8 at a time
  const size_t room = (size_t)NW * 2 * CHUNK_BYTES;
  const bool fits = ((size_t)2 * nrows * a.nsplit + nrows) * sizeof(float) <= room;
  const int rbmax = fits ? nrows : 1;                 // rows per merge batch
  float* smw = reinterpret_cast<float*>(at_smem);     // [rbmax][nsplit] m -> weight
  float* sml = smw + (size_t)rbmax * a.nsplit;        // [rbmax][nsplit] l
  float* sL = sml + (size_t)rbmax * a.nsplit;         // [rbmax] L
  for (int r0 = 0; r0 < nrows; r0 += rbmax) {
    const int rb = min(rbmax, nrows - r0);
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
  }
  if (tid == 0) a.tickets[kh] = 0;
}

// Chunk merge for runs with many rows (prefill): one CTA per (query, head)
// row; the same order and formula as the in-kernel merge (chunk weights
// exp(m_c - M) in chunk order, L, then the weighted sum per dim).
template <int HD>
__global__ void __launch_bounds__(HD) attn_merge_kernel(const AttnArgs a) {
  pdl_wait();
  pdl_trigger();
  if (run_skipped(a.run_state)) return;
  extern __shared__ float wts[];     // [nsplit]
  __shared__ float sL;
  const int row = blockIdx.x;       // j * H + h
  const int j = row / a.H;
  const int nc = (a.vis_len[j] + AT_C - 1) / AT_C;
  if (nc <= 1) return;
  const float* base = a.scratch + (size_t)row * a.nsplit * (HD + 2);
  for (int cc = threadIdx.x; cc < nc; cc += blockDim.x) wts[cc] = __ldcg(base + (size_t)cc * (HD + 2));
  __syncthreads();
  if (threadIdx.x == 0) {
    float M = -INFINITY;
    for (int cc = 0; cc < nc; ++cc) M = fmaxf(M, wts[cc]);
    float L = 0.f;
    for (int cc = 0; cc < nc; ++cc) {
      const float wgt = __expf(wts[cc] - M);
      wts[cc] = wgt;
      L = __fadd_rn(L, __fmul_rn(__ldcg(base + (size_t)cc * (HD + 2) + 1), wgt));
    }
    sL = L;
  }
  __syncthreads();
  const int dd = threadIdx.x;
  const float* bd = base + 2 + dd;
  float o = 0.f;
  for (int c0 = 0; c0 < nc; c0 += 8) {
    float v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = c0 + k < nc ? __ldcg(bd + (size_t)(c0 + k) * (HD + 2)) : 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (c0 + k < nc) o = __fadd_rn(o, __fmul_rn(v[k], wts[c0 + k]));
  }
  const float val = o / sL;
  if (a.out_bf16) reinterpret_cast<__nv_bfloat16*>(a.out)[(size_t)row * HD + dd] = __float2bfloat16_rn(val);
  else a.out[(size_t)row * HD + dd] = val;
}

template <int HD>
static cudaError_t launch_tc_hd(const AttnArgs& a, cudaStream_t st) {
  const size_t smem = (size_t)(AT_THREADS / 32) * 2 * AT_C * HD * 2;   // one chunk per warp
  static size_t configured = 0;
  if (configured < smem) {
    cudaError_t e = cudaFuncSetAttribute(attn_tc_kernel<HD>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  // one CTA per SM in total over the KV heads (four independent warp
  // streams each); chunks loop in-warp, so one launch shape serves any
  // context (graph replay) and CTAs past the run's chunks exit at once
  const int per_sm = HD == 64 ? 3 : 1;
  const int chunks4 = (a.nsplit + 1) / 2 / (AT_THREADS / 32) + 1;   // (nsplit counts 32-entry splits)
  const int z = max(1, min(chunks4, (per_sm * 148 + a.KH - 1) / a.KH));
  // many rows (prefill): their 16-row tiles spread over up to 8 row blocks
  // (a warp otherwise walks every tile of its chunk in sequence); the
  // in-kernel merge of <= 32 rows keeps one block
  const int nrows = a.n * (a.H / a.KH);
  static const int rb_max = getenv("SP_ATT_TC_RB") ? max(1, atoi(getenv("SP_ATT_TC_RB"))) : 8;
  const int rb = nrows > AT_MERGE_ROWS ? max(1, min(rb_max, (nrows + 15) / 16)) : 1;
  cudaError_t e = launch_pdl(attn_tc_kernel<HD>, dim3(a.KH, z, rb), dim3(AT_THREADS), smem, st, a);
  if (e != cudaSuccess || a.n * (a.H / a.KH) <= AT_MERGE_ROWS) return e;
  const size_t msmem = sizeof(float) * (size_t)a.nsplit;
  static size_t mconf = 0;
  if (mconf < msmem) {
    e = cudaFuncSetAttribute(attn_merge_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)msmem);
    if (e != cudaSuccess) return e;
    mconf = msmem;
  }
  return launch_pdl(attn_merge_kernel<HD>, dim3(a.n * a.H), dim3(HD), msmem, st, a);
}

// Which kernel a launch of n queries takes.  Measured (tools/attn_bench.py,
// profiles/r02_attention.txt): on decode-sized runs the CUDA-core kernel is
// faster (7B ctx 640: 11.7 vs 15.7 us; 4096: 55.6 vs 64.6 us; 70B GQA ctx
// 640: 14.8 vs 30.2 us) -- a 16-row MMA tile is mostly padding there and a
// warp's gather does not overlap its math -- so the tensor-core kernel takes
// prefill-sized runs (n >= 32: 7B n=128 ctx 4096 1.14 vs 3.49 ms; the
// CUDA-core kernel re-reads the plan per query and head).  The switch depends on n only and
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
