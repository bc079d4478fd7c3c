// K5 (bf16 KV cache, decode-sized runs): flash-decoding attention with
// shared-memory K/V staging, every query of the run in each CTA.
//
// model.py:394-415 per query q and head h: softmax(q.K_vis^T * scale) V_vis
// over the query's visible rows in plan order.  Layout on B200:
//
//  * grid (head h, z): CTA z owns plan chunks z, z+Z, ... (64 entries each)
//    of the run's longest plan; Z depends on the head count only.  Each
//    chunk's K and V rows are gathered into a two-stage shared-memory ring
//    with cp.async (the next chunk streams in while this one computes; the
//    old rows of the first chunk before the dependency wait);
//  * every query of the run reads the staged rows: a verification run's
//    queries share their prefix, so its K/V cross HBM once, not once per
//    query.  A query whose plan is not nested in the longest one (tree
//    siblings) reads its diverging entries from global memory;
//  * 16 (hd 128) or 8 (hd 64) lanes per row, the row groups of a CTA walk
//    their entries of each chunk in order with an online softmax per query;
//    the groups merge in group order into a CTA partial, the CTA partials
//    merge in z order (the last CTA of the head).  A query's arithmetic
//    never depends on the other queries, on n or on the context: batch-,
//    tree- and split-invariant.
#include "kernels.cuh"

namespace sp {

constexpr int FD_C = 64;          // plan entries per chunk
constexpr int FD_THREADS = 128;
#ifndef SP_FD_QB
#define SP_FD_QB 4
#endif
constexpr int FD_QB = SP_FD_QB;   // queries per register batch

__device__ __forceinline__ uint32_t fd_s(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void fd_cp16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}

template <int HD>
__global__ void __launch_bounds__(FD_THREADS) attn_fd_kernel(const AttnArgs a) {
  constexpr int U = HD / 8;                 // 16-byte units per row
  constexpr int LPR = U;                    // lanes per row (one unit each)
  constexpr int G = FD_THREADS / LPR;       // row groups
  constexpr int EPG = FD_C / G;             // entries per group per chunk
  constexpr int CB = FD_C * HD * 2;         // bytes of K (or V) per chunk
  extern __shared__ __align__(128) uint8_t fd_smem[];   // [2 stages][K | V]
  __shared__ int srows[2][FD_C];
  __shared__ unsigned char sdiv[FD_QB][FD_C];   // entry differs from the staged row
  __shared__ float gst[G][HD + 2];          // per-group (m, l, acc) of one query
  __shared__ int s_last;

  const int h = blockIdx.x, z = blockIdx.y, Z = gridDim.y;
  const int kh = h / (a.H / a.KH);
  const int kvd = a.KH * HD;
  const int tid = threadIdx.x, g = tid / LPR, l = tid % LPR;
  const __nv_bfloat16* Kc = reinterpret_cast<const __nv_bfloat16*>(a.k) + (size_t)kh * HD;
  const __nv_bfloat16* Vc = reinterpret_cast<const __nv_bfloat16*>(a.v) + (size_t)kh * HD;

  // before the dependency wait: plans, lengths and old K/V rows are final
  int ref = 0, ref_len = -1;
  for (int j = 0; j < a.n; ++j) {
    const int lj = a.vis_len[j];
    if (lj >= ref_len) { ref_len = lj; ref = j; }
  }
  const int nch = (ref_len + FD_C - 1) / FD_C;
  if (z >= nch) return;                     // no chunk here (not counted below)
  const int32_t* pref = a.vis + (size_t)ref * a.ld_vis;
  const int fresh0 = a.fresh_row0_dev ? *a.fresh_row0_dev : a.fresh_row0;
  // a query on the reference's sequence set in a coverage-checked run has a
  // plan that is a prefix of the reference's (one cell per position)
  const int ref_mask = (a.toks != nullptr && a.hdr != nullptr &&
                        (a.hdr->flags & SP_FWD_CHECK_COVERAGE))
                           ? (int)a.toks[ref].seq_mask : 0;

  // chunk c of the reference plan into stage b; part 1 = rows < fresh0,
  // 2 = rows >= fresh0, 0 = all.  One commit group per call.
  auto issue = [&](int c, int b, int part) {
    const int e0 = c * FD_C;
    if (part != 2) {
      if (tid < FD_C) srows[b][tid] = e0 + tid < ref_len ? pref[e0 + tid] : pref[e0];
      __syncthreads();
    }
    const uint32_t kb = fd_s(fd_smem + (size_t)b * 2 * CB), vb = kb + CB;
    for (int i = tid; i < FD_C * U; i += FD_THREADS) {
      const int e = i / U, u = i % U;
      const int row = srows[b][e];
      if ((part == 1 && row >= fresh0) || (part == 2 && row < fresh0)) continue;
      const size_t off = (size_t)row * kvd + u * 8;
      fd_cp16(kb + (uint32_t)i * 16, Kc + off);
      fd_cp16(vb + (uint32_t)i * 16, Vc + off);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };

  const bool pre = fresh0 > 0 && !run_skipped(a.run_state);
  if (pre) issue(z, 0, 1);
  pdl_wait();
  pdl_trigger();
  if (a.diag_empty || run_skipped(a.run_state)) {
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    return;
  }
  if (z == 0 && tid == 0 && nch > a.nsplit) set_error(a.err, SP_DEV_PLAN_OVERFLOW);
  const int nz = (nch - z + Z - 1) / Z;     // this CTA's chunks
  const int active = min(Z, nch);           // CTAs holding a partial
  const bool single = active == 1;

  for (int q0 = 0; q0 < a.n; q0 += FD_QB) {
    const int nq = min(FD_QB, a.n - q0);
    float qv[FD_QB][8], m[FD_QB], ls[FD_QB], acc[FD_QB][8];
    int qlen[FD_QB];
    bool nested[FD_QB];
#pragma unroll
    for (int q = 0; q < FD_QB; ++q) {
      m[q] = -INFINITY;
      ls[q] = 0.f;
      qlen[q] = 0;
      nested[q] = true;
#pragma unroll
      for (int t = 0; t < 8; ++t) { acc[q][t] = 0.f; qv[q][t] = 0.f; }
      if (q < nq) {
        const int j = q0 + q;
        qlen[q] = a.vis_len[j];
        nested[q] = j == ref || (ref_mask != 0 && (int)a.toks[j].seq_mask == ref_mask);
        const float* qp = a.q + (size_t)j * a.H * HD + (size_t)h * HD + l * 8;
#pragma unroll
        for (int t = 0; t < 8; ++t) qv[q][t] = qp[t] * a.scale;
      }
    }
    // ring: chunk k of this CTA (c = z + k*Z) in stage k & 1
    if (q0 == 0) {
      issue(z, 0, pre ? 2 : 0);
    } else {
      issue(z, 0, 0);
    }
    if (nz > 1) issue(z + Z, 1, 0);
    for (int k = 0; k < nz; ++k) {
      const int c = z + k * Z, b = k & 1;
      if (k + 1 < nz) asm volatile("cp.async.wait_group 1;" ::: "memory");
      else asm volatile("cp.async.wait_group 0;" ::: "memory");
      __syncthreads();
      const uint8_t* Ks = fd_smem + (size_t)b * 2 * CB;
      const uint8_t* Vs = Ks + CB;
      const int e0 = c * FD_C;
      // queries not known to be nested: which of their entries diverge from
      // the staged rows (one parallel compare per query and chunk)
      bool any_div = false;
#pragma unroll
      for (int q = 0; q < FD_QB; ++q) {
        if (q >= nq || nested[q]) continue;
        any_div = true;
        if (tid < FD_C) {
          const int e = e0 + tid;
          sdiv[q][tid] = e < qlen[q] ? (a.vis[(size_t)(q0 + q) * a.ld_vis + e] != srows[b][tid])
                                     : 0;
        }
      }
      if (any_div) __syncthreads();
#pragma unroll
      for (int q = 0; q < FD_QB; ++q) {
        if (q >= nq) break;
        const int lim = qlen[q] - e0;          // entries of this chunk the query sees
        if (lim <= 0) continue;                // (uniform: depends on the query only)
        const int32_t* pj = a.vis + (size_t)(q0 + q) * a.ld_vis;
#pragma unroll 2
        for (int i = 0; i < EPG; ++i) {
          const int e = g + G * i;             // this group's entries, in order
          uint4 kr, vr;
          bool own = true;
          if (!nested[q] && e < lim && sdiv[q][e]) {   // diverging entry: from L2/HBM
            const int row = pj[e0 + e];
            own = false;
            kr = __ldcg(reinterpret_cast<const uint4*>(Kc + (size_t)row * kvd + l * 8));
            vr = __ldcg(reinterpret_cast<const uint4*>(Vc + (size_t)row * kvd + l * 8));
          }
          if (own) {
            kr = *reinterpret_cast<const uint4*>(Ks + ((size_t)e * U + l) * 16);
            vr = *reinterpret_cast<const uint4*>(Vs + ((size_t)e * U + l) * 16);
          }
          float kf[8];
          bf16x8_to_f32(kr, kf);
          float d = 0.f;
#pragma unroll
          for (int t = 0; t < 8; ++t) d = __fmaf_rn(qv[q][t], kf[t], d);
#pragma unroll
          for (int o = LPR / 2; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
          if (e < lim) {
            float vf[8];
            bf16x8_to_f32(vr, vf);
            if (d > m[q]) {
              const float cc = __expf(m[q] - d);
              ls[q] = __fmul_rn(ls[q], cc);
#pragma unroll
              for (int t = 0; t < 8; ++t) acc[q][t] = __fmul_rn(acc[q][t], cc);
              m[q] = d;
            }
            const float p = __expf(d - m[q]);
            ls[q] = __fadd_rn(ls[q], p);
#pragma unroll
            for (int t = 0; t < 8; ++t) acc[q][t] = __fmaf_rn(p, vf[t], acc[q][t]);
          }
        }
      }
      __syncthreads();                         // stage b is free again
      if (k + 2 < nz) issue(z + (k + 2) * Z, b, 0);
    }
    // groups -> CTA partial (group order), per query
#pragma unroll
    for (int q = 0; q < FD_QB; ++q) {
      if (q >= nq) break;
      const int j = q0 + q;
      if (l == 0) { gst[g][0] = m[q]; gst[g][1] = ls[q]; }
#pragma unroll
      for (int t = 0; t < 8; ++t) gst[g][2 + l * 8 + t] = acc[q][t];
      __syncthreads();
      const size_t row = (size_t)j * a.H + h;
      for (int dd = tid; dd < HD; dd += FD_THREADS) {
        float M = -INFINITY;
        for (int gg = 0; gg < G; ++gg) M = fmaxf(M, gst[gg][0]);
        float L = 0.f, o = 0.f;
        if (M != -INFINITY) {
          for (int gg = 0; gg < G; ++gg) {
            if (gst[gg][0] == -INFINITY) continue;
            const float w = __expf(gst[gg][0] - M);
            L = __fadd_rn(L, __fmul_rn(gst[gg][1], w));
            o = __fadd_rn(o, __fmul_rn(gst[gg][2 + dd], w));
          }
        }
        if (single) {    // = the z-order merge of one partial (weight exp(0) = 1)
          const float v = o / L;
          if (a.out_bf16) reinterpret_cast<__nv_bfloat16*>(a.out)[row * HD + dd] = __float2bfloat16_rn(v);
          else a.out[row * HD + dd] = v;
        } else {
          float* sp = a.scratch + (row * a.nsplit + z) * (HD + 2);
          sp[2 + dd] = o;
          if (dd == 0) { sp[0] = M; sp[1] = L; }
        }
      }
      __syncthreads();
    }
  }
  if (single) return;
  // the last CTA of the head merges the CTA partials of every query, z order
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = atomicAdd(&a.tickets[h], 1) == active - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  for (int idx = tid; idx < a.n * HD; idx += FD_THREADS) {
    const int j = idx / HD, dd = idx % HD;
    const size_t row = (size_t)j * a.H + h;
    const float* base = a.scratch + row * a.nsplit * (HD + 2);
    float M = -INFINITY;
    for (int zz = 0; zz < active; ++zz) M = fmaxf(M, __ldcg(base + (size_t)zz * (HD + 2)));
    float L = 0.f, o = 0.f;
    for (int z0 = 0; z0 < active; z0 += 8) {
      float mv[8], lv[8], ov[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const float* b = base + (size_t)(z0 + u) * (HD + 2);
        const bool ok = z0 + u < active;
        mv[u] = ok ? __ldcg(b) : -INFINITY;
        lv[u] = ok ? __ldcg(b + 1) : 0.f;
        ov[u] = ok ? __ldcg(b + 2 + dd) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (mv[u] == -INFINITY) continue;
        const float w = __expf(mv[u] - M);
        L = __fadd_rn(L, __fmul_rn(lv[u], w));
        o = __fadd_rn(o, __fmul_rn(ov[u], w));
      }
    }
    const float v = o / L;
    if (a.out_bf16) reinterpret_cast<__nv_bfloat16*>(a.out)[row * HD + dd] = __float2bfloat16_rn(v);
    else a.out[row * HD + dd] = v;
  }
  if (tid == 0) a.tickets[h] = 0;
}

template <int HD>
static cudaError_t launch_fd_hd(const AttnArgs& a, cudaStream_t st) {
  const size_t smem = 2 * 2 * (size_t)FD_C * HD * 2;   // two stages of K and V
  static size_t configured = 0;
  if (configured < smem) {
    const cudaError_t e = cudaFuncSetAttribute(
        attn_fd_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  // Z CTAs per head: about two per SM in total (a fixed function of the head
  // count, so one captured shape serves any run and context)
  static const int per_sm = getenv("SP_ATT_FD_PER_SM") ? atoi(getenv("SP_ATT_FD_PER_SM")) : 2;
  const int z = max(1, min((a.nsplit + 1) / 2, (per_sm * 148 + a.H - 1) / a.H));
  return launch_pdl(attn_fd_kernel<HD>, dim3(a.H, z), dim3(FD_THREADS), smem, st, a);
}

// Decode-sized runs of long-context stages (max_context >= 4096) take this
// kernel; shorter ones keep the CUDA-core per-query kernel.  The choice is
// a per-stage constant -- never a function of the run -- so a token's bits
// do not depend on how many tokens share its run.  Measured (7B 1-token
// stage-run, tools/stage_timeline.py): ctx 4096 60.4 -> 31.0 us per layer,
// 16384 209 -> 90.6; but ctx 384 8.8 -> 9.7 and a 5-token run 16.5 -> 28.7
// (the query batches walk the chunk in sequence).  SP_ATT_FD=1/0 forces.
bool attn_fd_ok(int kv_dtype, int hd, int n, int max_context) {
  static const char* env = getenv("SP_ATT_FD");
  if (kv_dtype != SP_DTYPE_BF16 || (hd != 64 && hd != 128) || n >= 32) return false;
  if (env) return atoi(env) != 0;
  return max_context >= 4096;
}

cudaError_t launch_attention_fd(const AttnArgs& a, int hd, cudaStream_t st) {
  return hd == 64 ? launch_fd_hd<64>(a, st) : launch_fd_hd<128>(a, st);
}

}  // namespace sp
