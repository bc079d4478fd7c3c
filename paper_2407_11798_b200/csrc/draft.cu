// K15: the draft request as ONE persistent kernel.
//
// A draft request (DraftRequestPayload, engine.py:313-322; served by
// _DraftNode, engine.py:640-688) feeds a few tokens, then speculates while
// the draft's confidence stays >= cutoff (speculate_microbatch with
// microbatch 1, speculation.py:142-195).  With one launch per layer-GEMV a
// 160M-shape forward is ~60 dependent launches whose fill/drain dominates
// (the weights are only ~0.28 GB).  Here one cooperative grid (one CTA per
// SM) runs every step of the request:
//
//   per step:  embed -> L x [A: rmsnorm+QKV+RoPE+KV write | B: attention |
//              C: O + residual | D: rmsnorm+gate/up+SwiGLU | E: down +
//              residual] -> H: final norm + LM head + top-2/softmax stats
//
// with a grid barrier between phases.  Every CTA owns a fixed contiguous
// slice of each weight matrix and prefetches its NEXT phase's slice into L2
// (cp.async.bulk.prefetch) while the current phase runs, so HBM streams
// behind the barriers.  The LM head's partials are merged redundantly by
// every CTA (fixed order), so all CTAs know the argmax / confidence and the
// chain continues (token = argmax, gate = conf >= cutoff) without a host
// round trip.
//
// Cache discipline: the draft is one sequence whose cell rows equal token
// positions (the host truncates before feeding), so a token at row r
// attends to rows [0, r] — no plan needed.
//
// Determinism: every reduction has a fixed order (per-lane chunk order,
// butterflies, warps/CTAs/splits in index order), so a request's proposals
// are reproducible run to run.
#include "gemv_core.cuh"
#include "kernels.cuh"

namespace sp {

constexpr int DR_THREADS = 256;
constexpr int DR_WARPS = DR_THREADS / 32;

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Grid barrier over a counter zeroed before the launch (monotonic targets).
__device__ __forceinline__ void grid_sync(unsigned* bar, unsigned& target,
                                          unsigned a_spin_ns = 32) {
  __syncthreads();
  target += gridDim.x;
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
    unsigned spins = 0;
    // poll with a short back-off: 148 pollers on one L2 line otherwise
    // queue behind each other at its slice (SP_DRAFT_SPIN_NS, default 32)
    while (ld_acquire_u32(bar) < target) {
      __nanosleep(a_spin_ns);
      if (++spins > (1u << 28)) __trap();  // a lost CTA: fail loudly, never hang
    }
  }
  __syncthreads();
}

__device__ __forceinline__ long long gtime() {
  long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void l2_prefetch(const void* p, size_t bytes) {
  // bulk L2 prefetch of a contiguous slice, in <= 1 MiB pieces
  const char* c = reinterpret_cast<const char*>(p);
  while (bytes >= 16) {
    const unsigned n = (unsigned)(bytes > (1u << 20) ? (1u << 20) : (bytes & ~size_t(15)));
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(c), "r"(n) : "memory");
    c += n;
    bytes -= n;
  }
}

__device__ __forceinline__ uint4 ldcg16(const void* p) {
  return __ldcg(reinterpret_cast<const uint4*>(p));
}

// ---- shared-memory weight staging (1D bulk copies on an mbarrier) --------
__device__ __forceinline__ uint32_t dr_smem(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void dr_mbar_init(uint64_t* b) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(dr_smem(b)));
}
__device__ __forceinline__ void dr_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(dr_smem(b)),
               "r"(bytes) : "memory");
}
__device__ __forceinline__ void dr_wait(uint64_t* b, uint32_t parity) {
  for (uint32_t it = 0;; ++it) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}"
        : "=r"(ok) : "r"(dr_smem(b)), "r"(parity), "r"(1000u) : "memory");
    if (ok) return;
    if (it > (1u << 22)) __trap();
  }
}
__device__ __forceinline__ void dr_bulk(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(dr_smem(dst)), "l"(src), "r"(bytes), "r"(dr_smem(b)) : "memory");
}

__device__ __forceinline__ void slice(int R, int& u0, int& u1) {
  u0 = (int)(((long long)R * blockIdx.x) / gridDim.x);
  u1 = (int)(((long long)R * (blockIdx.x + 1)) / gridDim.x);
}

// y[r][m] = sum_k W[row_r][k] * xs[m][k] for R rows (row pointers) and n <= NT
// tokens held in shared memory.  Lane l takes 8-element chunks l, l+32, ...
// (ascending), then a butterfly: a fixed order.
template <int NT, int R>
__device__ __forceinline__ void warp_dot(const __nv_bfloat16* const (&w)[R], const float* xs,
                                         int K, int n, float (&y)[R][NT], int row0g) {
  const int lane = threadIdx.x & 31;
  const int nch = K >> 3;
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int m = 0; m < NT; ++m) y[r][m] = 0.f;
  constexpr int U = (R >= 8) ? 3 : (R >= 4) ? 2 : 4;
  for (int c0 = lane; c0 < nch; c0 += 32 * U) {
    uint4 wv[U][R];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int c = c0 + 32 * u;
#pragma unroll
      for (int r = 0; r < R; ++r)
        wv[u][r] = (c < nch && w[r])
                       ? ld_stream16(w[r] + (size_t)(c ^ ((row0g + r) & 7)) * 8)   // SWZ8
                       : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int c = c0 + 32 * u;
      if (c >= nch) break;
      float wf[R][8];
#pragma unroll
      for (int r = 0; r < R; ++r) bf16x8_to_f32(wv[u][r], wf[r]);
#pragma unroll
      for (int m = 0; m < NT; ++m) {
        if (m >= n) break;
        const float4 x0 = *reinterpret_cast<const float4*>(xs + (size_t)m * K + c * 8);
        const float4 x1 = *reinterpret_cast<const float4*>(xs + (size_t)m * K + c * 8 + 4);
        const float xv[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
          for (int j = 0; j < 8; ++j) y[r][m] = __fmaf_rn(wf[r][j], xv[j], y[r][m]);
      }
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int m = 0; m < NT; ++m)
      if (m < n) y[r][m] = warp_sum(y[r][m]);
}

// Same contraction with the weight rows in shared memory (staged by bulk
// copies ahead of the phase): no global round trip on the critical path.
template <int NT, int R>
__device__ __forceinline__ void warp_dot_s(const __nv_bfloat16* const (&w)[R], const float* xs,
                                           int K, int n, float (&y)[R][NT], int row0g) {
  const int lane = threadIdx.x & 31;
  const int nch = K >> 3;
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int m = 0; m < NT; ++m) y[r][m] = 0.f;
#pragma unroll 4
  for (int c = lane; c < nch; c += 32) {
    float wf[R][8];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const uint4 u = w[r] ? *reinterpret_cast<const uint4*>(
                                 w[r] + (size_t)(c ^ ((row0g + r) & 7)) * 8)   // SWZ8
                           : make_uint4(0, 0, 0, 0);
      bf16x8_to_f32(u, wf[r]);
    }
#pragma unroll
    for (int m = 0; m < NT; ++m) {
      if (m >= n) break;
      const float4 x0 = *reinterpret_cast<const float4*>(xs + (size_t)m * K + c * 8);
      const float4 x1 = *reinterpret_cast<const float4*>(xs + (size_t)m * K + c * 8 + 4);
      const float xv[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int j = 0; j < 8; ++j) y[r][m] = __fmaf_rn(wf[r][j], xv[j], y[r][m]);
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int m = 0; m < NT; ++m)
      if (m < n) y[r][m] = warp_sum(y[r][m]);
}

// Stage n rows of a [*, K] fp32 activation into shared memory (times gain),
// and (norm) each row's RMS scale.  The statistic's order is fixed: thread
// t sums elements t, t+256, ... ascending, then warps 0..7.
__device__ void stage_rows(float* xs, const float* src, int ld, int K, int n, const float* gain,
                           bool norm, float eps, float* scale, float (&red)[DR_WARPS][DR_NT]) {
  const int tid = threadIdx.x;
  float ss[DR_NT];
#pragma unroll
  for (int m = 0; m < DR_NT; ++m) ss[m] = 0.f;
  for (int m = 0; m < n; ++m) {
    const float* s = src + (size_t)m * ld;
    for (int k = tid * 4; k < K; k += DR_THREADS * 4) {
      const float4 v = __ldcg(reinterpret_cast<const float4*>(s + k));
      if (norm) {
        ss[m] = __fmaf_rn(v.x, v.x, ss[m]);
        ss[m] = __fmaf_rn(v.y, v.y, ss[m]);
        ss[m] = __fmaf_rn(v.z, v.z, ss[m]);
        ss[m] = __fmaf_rn(v.w, v.w, ss[m]);
      }
      float4 o = v;
      if (gain) {
        const float4 g = __ldg(reinterpret_cast<const float4*>(gain + k));
        o.x = __fmul_rn(v.x, g.x); o.y = __fmul_rn(v.y, g.y);
        o.z = __fmul_rn(v.z, g.z); o.w = __fmul_rn(v.w, g.w);
      }
      *reinterpret_cast<float4*>(xs + (size_t)m * K + k) = o;
    }
  }
  if (norm) {
    const int warp = tid >> 5, lane = tid & 31;
#pragma unroll
    for (int m = 0; m < DR_NT; ++m) {
      const float v = warp_sum(ss[m]);
      if (lane == 0) red[warp][m] = v;
    }
    __syncthreads();
    if (tid < DR_NT) {
      float t = red[0][tid];
#pragma unroll
      for (int w = 1; w < DR_WARPS; ++w) t = __fadd_rn(t, red[w][tid]);
      scale[tid] = rms_scale(t, K, eps);
    }
  }
  __syncthreads();
}

struct DTop2 { float v1; int i1; float v2; int i2; };
__device__ __forceinline__ bool dbetter(float va, int ia, float vb, int ib) {
  return va > vb || (va == vb && ia < ib);
}
__device__ __forceinline__ void dpush(DTop2& t, float v, int i) {
  if (dbetter(v, i, t.v1, t.i1)) { t.v2 = t.v1; t.i2 = t.i1; t.v1 = v; t.i1 = i; }
  else if (dbetter(v, i, t.v2, t.i2)) { t.v2 = v; t.i2 = i; }
}
// online (max, sum of exp) update with a fixed visiting order
__device__ __forceinline__ void online_add(float& mx, float& se, float v) {
  if (v > mx) { se = __fadd_rn(__fmul_rn(se, __expf(mx - v)), 1.0f); mx = v; }
  else se = __fadd_rn(se, __expf(v - mx));
}
__device__ __forceinline__ void online_merge(float& mx, float& se, float m2, float s2) {
  if (m2 == -INFINITY) return;
  if (mx == -INFINITY) { mx = m2; se = s2; return; }
  const float M = fmaxf(mx, m2);
  se = __fadd_rn(__fmul_rn(se, __expf(mx - M)), __fmul_rn(s2, __expf(m2 - M)));
  mx = M;
}

template <int HD>
__global__ void __launch_bounds__(DR_THREADS, 1) draft_chain_kernel(const DraftArgs a) {
  // dynamic smem: three weight buffers (QKV / gate-up / down slices, each
  // staged by bulk copies two phases ahead), the scaled activations xs
  // [DR_NT][Kmax] and the raw rows xr [DR_NT][d] (for the RMS statistic)
  extern __shared__ __align__(128) uint8_t dsm[];
  __nv_bfloat16* const bufA = reinterpret_cast<__nv_bfloat16*>(dsm);
  __nv_bfloat16* const bufD = reinterpret_cast<__nv_bfloat16*>(dsm + a.bufA);
  __nv_bfloat16* const bufE = reinterpret_cast<__nv_bfloat16*>(dsm + a.bufA + a.bufD);
  float* const xs = reinterpret_cast<float*>(dsm + a.bufA + a.bufD + a.bufE);
  float* const xr = xs + (size_t)DR_NT * a.kmax;
  __shared__ __align__(8) uint64_t wbar[3];
  __shared__ DraftLayer lw_s[DR_MAX_LAYERS];
  __shared__ float inv_s[HD / 2];
  __shared__ float part[DR_THREADS / (HD / 8)][HD];
  __shared__ float attn_s[HD];
  __shared__ float gstat[DR_THREADS / (HD / 8)][2];
  __shared__ float wred[DR_WARPS];
  __shared__ int last;
  __shared__ float lm_w[DR_WARPS][4];
  __shared__ int lm_wi[DR_WARPS][3];
  __shared__ int s_next_tok, s_gate;

  const DraftHdr& H = *a.hdr;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int d = a.d, f = a.f, qd = a.H * HD, kvd = a.KH * HD;
  const int n_feed = H.n_feed, steps = H.steps, pos0 = H.pos0, row0 = H.row0;
  const int chain = H.chain;
  const float cutoff = H.cutoff;
  unsigned target = 0;
  int nprof = 0;
  // stamp = (site << 56) | clock64 (diagnostics, SP_DRAFT_PROF)
  auto mark = [&](long long site) {
    if (a.prof && blockIdx.x == 0 && tid == 0 && nprof < 4095)
      a.prof[1 + nprof++] = (site << 56) | (clock64() & ((1ll << 56) - 1));
  };
  mark(0);
  const float att_scale = 1.0f / sqrtf((float)HD);
  uint64_t pol_stream, pol_keep;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_stream));
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_keep));

  // row slices (fixed per CTA for the whole launch)
  int qkv0, qkv1, d0, d1, up0, up1, v0, v1;
  slice((qd + 2 * kvd) / 2, qkv0, qkv1);   // QKV row pairs
  slice(d, d0, d1);                         // down rows = residual owners
  slice(f, up0, up1);                       // gate/up row pairs
  slice(a.V, v0, v1);                       // LM head rows

  uint32_t wpar[3] = {0u, 0u, 0u};
  int wpend[3] = {0, 0, 0};
  for (int l = tid; l < a.L; l += DR_THREADS) lw_s[l] = a.layers[l];
  for (int j = tid; j < HD / 2; j += DR_THREADS)
    inv_s[j] = powf(a.theta, -2.0f * (float)j / (float)HD);
  if (tid == 0) {
    for (int i = 0; i < 3; ++i) dr_mbar_init(&wbar[i]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // which: 0 = QKV (bufA), 1 = gate/up (bufD), 2 = down (bufE)
  auto wload = [&](int which, int l) {
    wpend[which] = 1;
    if (tid != 0) return;
    const DraftLayer& Lw = lw_s[l];
    const __nv_bfloat16* src;
    size_t bytes;
    __nv_bfloat16* dst;
    if (which == 0) {
      src = Lw.qkv + (size_t)2 * qkv0 * d; bytes = (size_t)2 * (qkv1 - qkv0) * d * 2; dst = bufA;
    } else if (which == 1) {
      src = Lw.up + (size_t)2 * up0 * d; bytes = (size_t)2 * (up1 - up0) * d * 2; dst = bufD;
    } else {
      src = Lw.down + (size_t)d0 * f; bytes = (size_t)(d1 - d0) * f * 2; dst = bufE;
    }
    // the previous phase's generic reads of dst precede these async writes
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    dr_expect(&wbar[which], (uint32_t)bytes);
    char* dc = reinterpret_cast<char*>(dst);
    const char* sc_ = reinterpret_cast<const char*>(src);
    for (size_t off = 0; off < bytes; off += 32768) {
      const uint32_t nb = (uint32_t)(bytes - off < 32768 ? bytes - off : 32768);
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
          " [%0], [%1], %2, [%3], %4;" ::"r"(dr_smem(dc + off)), "l"(sc_ + off), "r"(nb),
          "r"(dr_smem(&wbar[which])), "l"(pol_stream) : "memory");
    }
  };
  auto wwait = [&](int which) {
    dr_wait(&wbar[which], wpar[which]);
    wpar[which] ^= 1u;
    wpend[which] = 0;
  };
  // the LM head slice streams into L2 (evict_last) a piece per layer
  auto head_prefetch = [&](int l) {
    if (tid != 0) return;
    const size_t rows = (size_t)(v1 - v0);
    const size_t r0 = rows * l / a.L, r1 = rows * (l + 1) / a.L;
    const char* c = reinterpret_cast<const char*>(a.w_out + (size_t)(v0 + r0) * d);
    size_t bytes = (r1 - r0) * d * 2;
    while (bytes >= 16) {
      const unsigned nb = (unsigned)(bytes > (1u << 20) ? (1u << 20) : (bytes & ~size_t(15)));
      asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(c),
                   "r"(nb), "l"(pol_keep) : "memory");
      c += nb;
      bytes -= nb;
    }
  };
  // per-warp RMS scales of the staged raw rows xr (every warp computes the
  // same statistic in the same order: lane-strided, then a butterfly)
  auto warp_scales = [&](int K, int n, float (&scl)[DR_NT]) {
#pragma unroll
    for (int m = 0; m < DR_NT; ++m) {
      scl[m] = 1.0f;
      if (m < n) {
        float ss = 0.f;
        for (int k = lane * 4; k < K; k += 128) {
          const float4 v = *reinterpret_cast<const float4*>(xr + (size_t)m * a.d + k);
          ss = __fmaf_rn(v.x, v.x, ss); ss = __fmaf_rn(v.y, v.y, ss);
          ss = __fmaf_rn(v.z, v.z, ss); ss = __fmaf_rn(v.w, v.w, ss);
        }
        scl[m] = rms_scale(warp_sum(ss), K, a.eps);
      }
    }
  };
  if (n_feed > 0 || steps > 0) {
    wload(0, 0);
    wload(1, 0);
  }

  int tip_tok = 0;
  int gate = 1;
  int row = row0;      // next cell row
  int pos = pos0;      // next position
  for (int k = 0; k <= steps; ++k) {
    int n;
    int toks[DR_NT];
    if (k == 0) {
      if (n_feed == 0) {
        // no feed: the chain starts from the current tip (sp_stage_chain_begin)
        const int valid = __ldcg(a.tip + 2);
        const float conf = valid ? __int_as_float(__ldcg(a.tip + 1)) : -1.0f;
        tip_tok = valid ? __ldcg(a.tip) : 0;
        gate = (valid && conf >= cutoff) ? 1 : 0;
        if (blockIdx.x == 0 && tid == 0) {
          sp_row_result r;
          r.argmax = valid ? tip_tok : -1;
          r.second = -1;
          r.conf = conf;
          r.max_logit = 0.f;
          a.out[0] = r;
          if (chain) *a.gate = gate;
        }
        continue;
      }
      n = n_feed;
      for (int i = 0; i < DR_NT; ++i) toks[i] = i < n ? H.tok[i] : 0;
    } else {
      if (chain && !gate) {
        // gate closed: the remaining steps' cells are dead (sp_stage_step's
        // gate_kernel skip); rows are still consumed
        if (blockIdx.x == 0)
          for (int j = tid; j <= steps - k; j += DR_THREADS) {
            a.cell_pos[row + j] = pos + j;
            a.cell_mask[row + j] = 0u;
          }
        break;
      }
      n = 1;
      toks[0] = chain ? tip_tok : H.tok[n_feed + k - 1];
      for (int i = 1; i < DR_NT; ++i) toks[i] = 0;
    }
    const int rowA = row;   // rows rowA .. rowA+n-1, positions posA ..
    const int posA = pos;
    if (blockIdx.x == 0)
      for (int i = tid; i < n; i += DR_THREADS) {
        a.cell_pos[rowA + i] = posA + i;
        a.cell_mask[rowA + i] = 1u;
      }

    for (int l = 0; l < a.L; ++l) {
      const DraftLayer& Lw = lw_s[l];
      __nv_bfloat16* Kc = a.kc + a.kv_layer_elems * l;
      __nv_bfloat16* Vc = a.vc + a.kv_layer_elems * l;
      // ------------- A: rmsnorm + QKV + RoPE + K/V cell write ---------------
      wload(2, l);
      mark(40);
      if (tid == 0) l2_prefetch(Lw.o + (size_t)d0 * qd, (size_t)(d1 - d0) * qd * 2);
      mark(41);
      for (int m = 0; m < n && l == 0; ++m) {
        {   // embedding rows; the residual owners keep theirs in x
          const __nv_bfloat16* e = a.emb + (size_t)toks[m] * d;
          for (int c = tid; c < d; c += DR_THREADS) {
            const float v = __bfloat162float(e[c]);
            xr[(size_t)m * d + c] = v;
            xs[(size_t)m * d + c] = __fmul_rn(v, Lw.g_attn[c]);
            if (c >= d0 && c < d1) a.x[(size_t)m * d + c] = v;
          }
        }
      }
      if (l > 0) {
        // all loads first (one round trip), then the shared-memory stores
        constexpr int MAXV = DR_NT * 2;     // d <= 2048 -> <= 2 float4 per thread per token
        float4 v[MAXV], g[2];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int c = (tid + i * DR_THREADS) * 4;
          g[i] = c < d ? __ldg(reinterpret_cast<const float4*>(Lw.g_attn + c)) : make_float4(0, 0, 0, 0);
#pragma unroll
          for (int m = 0; m < DR_NT; ++m)
            v[m * 2 + i] = (m < n && c < d)
                               ? __ldcg(reinterpret_cast<const float4*>(a.x + (size_t)m * d + c))
                               : make_float4(0, 0, 0, 0);
        }
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int c = (tid + i * DR_THREADS) * 4;
          if (c >= d) break;
#pragma unroll
          for (int m = 0; m < DR_NT; ++m) {
            if (m >= n) break;
            const float4 x = v[m * 2 + i];
            *reinterpret_cast<float4*>(xr + (size_t)m * d + c) = x;
            *reinterpret_cast<float4*>(xs + (size_t)m * d + c) =
                make_float4(__fmul_rn(x.x, g[i].x), __fmul_rn(x.y, g[i].y),
                            __fmul_rn(x.z, g[i].z), __fmul_rn(x.w, g[i].w));
          }
        }
      }
      mark(42);
      __syncthreads();
      mark(43);
      {
        float scl[DR_NT];
        warp_scales(d, n, scl);
        mark(33); wwait(0); mark(49);
        for (int u = qkv0 + warp; u < qkv1; u += DR_WARPS) {
          const __nv_bfloat16* const w2[2] = {bufA + (size_t)(2 * (u - qkv0)) * d,
                                              bufA + (size_t)(2 * (u - qkv0) + 1) * d};
          float y[2][DR_NT];
          warp_dot_s<DR_NT, 2>(w2, xs, d, n, y, 2 * u);
          if (lane < n) {
            const int m = lane;
            float y0 = 0.f, y1 = 0.f;
#pragma unroll
            for (int mm = 0; mm < DR_NT; ++mm)
              if (mm == m) { y0 = __fmul_rn(y[0][mm], scl[mm]); y1 = __fmul_rn(y[1][mm], scl[mm]); }
            const int R = 2 * u;
            int sec, off;
            if (R < qd) { sec = 0; off = R; }
            else if (R < qd + kvd) { sec = 1; off = R - qd; }
            else { sec = 2; off = R - qd - kvd; }
            int e0 = off, e1 = off + 1;
            float o0 = y0, o1 = y1;
            if (sec < 2) {  // pair-interleaved rows -> rotate-half dims
              const int head = off / HD, j = (off % HD) >> 1;
              e0 = head * HD + j;
              e1 = e0 + (HD >> 1);
              const float inv = inv_s[j];
              float sn, cs;
              sincosf((float)(posA + m) * inv, &sn, &cs);
              o0 = y0 * cs - y1 * sn;
              o1 = y1 * cs + y0 * sn;
            }
            if (sec == 0) {
              a.q[(size_t)m * qd + e0] = o0;
              a.q[(size_t)m * qd + e1] = o1;
            } else {
              __nv_bfloat16* c = (sec == 1 ? Kc : Vc) + (size_t)(rowA + m) * kvd;
              c[e0] = __float2bfloat16_rn(o0);
              c[e1] = __float2bfloat16_rn(o1);
            }
          }
        }
      }
      mark(1); grid_sync(a.bar, target, a.spin_ns); mark(9);

      // ------ B: attention over rows [0, row_m] + this head's O partial ------
      if (l + 1 < a.L) wload(0, l + 1);
      else if (k < steps) wload(0, 0);
      head_prefetch(l);
      if (n == 1 && (int)gridDim.x >= 2 * a.H) {
        // single token: head groups of GS CTAs; every CTA of a group runs the
        // head's whole attention (redundantly, K/V stream from L2) and then
        // its own d/GS rows of the head's W_o columns -- no split merge, no
        // idle CTAs
        constexpr int LPR = HD / 8;
        constexpr int RPP = DR_THREADS / LPR;    // row groups (rows per pass)
        constexpr int PASSES = 8;                // rows in flight per chunk: RPP*8
        const int GS = (int)gridDim.x / a.H;
        const int hh = blockIdx.x / GS, jm = blockIdx.x % GS;
        if (hh < a.H) {
          const int grp = tid / LPR, li = tid % LPR;
          const int kh = hh / (a.H / a.KH);
          const int len = rowA + 1;
          // this member's W_o rows do not depend on the attention: their
          // loads go out first and land while it runs (one HBM round trip
          // off the phase)
          const int r0 = (int)(((long)d * jm) / GS), r1 = (int)(((long)d * (jm + 1)) / GS);
          constexpr int LR = HD / 8, RW = 32 / LR;
          constexpr int WB = 4;
          const int lr = lane % LR, rw = lane / LR;
          const bool wone = r1 - r0 <= DR_WARPS * RW * WB;   // one batch covers the slice
          uint4 wpre[WB];
          if (wone) {
#pragma unroll
            for (int b = 0; b < WB; ++b) {
              const int r = r0 + warp * RW + b * DR_WARPS * RW + rw;
              const int un = (hh * HD) / 8 + lr;
              wpre[b] = r < r1 ? ld_stream16(Lw.o + (size_t)r * qd + (size_t)(un ^ (r & 7)) * 8)
                               : make_uint4(0, 0, 0, 0);
            }
          }
          // q is scaled only after the first chunk's K/V loads are out (the
          // loads share one round trip)
          const float* qp = a.q + hh * HD + li * 8;
          const float4 q0 = __ldcg(reinterpret_cast<const float4*>(qp));
          const float4 q1 = __ldcg(reinterpret_cast<const float4*>(qp + 4));
          float qv[8];
          // per row-group online softmax over rows grp, grp+RPP, ... (fixed order)
          float mx = -INFINITY, ls = 0.f, acc[8];
#pragma unroll
          for (int t = 0; t < 8; ++t) acc[t] = 0.f;
          for (int c0 = 0; c0 < len; c0 += RPP * PASSES) {
            uint4 kr[PASSES], vr[PASSES];
#pragma unroll
            for (int p = 0; p < PASSES; ++p) {
              const int r = c0 + p * RPP + grp;
              const size_t off = (size_t)r * kvd + kh * HD + li * 8;
              kr[p] = r < len ? ldcg16(Kc + off) : make_uint4(0, 0, 0, 0);
              vr[p] = r < len ? ldcg16(Vc + off) : make_uint4(0, 0, 0, 0);
            }
            qv[0] = q0.x * att_scale; qv[1] = q0.y * att_scale;
            qv[2] = q0.z * att_scale; qv[3] = q0.w * att_scale;
            qv[4] = q1.x * att_scale; qv[5] = q1.y * att_scale;
            qv[6] = q1.z * att_scale; qv[7] = q1.w * att_scale;
#pragma unroll
            for (int p = 0; p < PASSES; ++p) {
              const int r = c0 + p * RPP + grp;
              float kf[8];
              bf16x8_to_f32(kr[p], kf);
              float sdot = 0.f;
#pragma unroll
              for (int t = 0; t < 8; ++t) sdot = __fmaf_rn(qv[t], kf[t], sdot);
#pragma unroll
              for (int o = LPR / 2; o > 0; o >>= 1) sdot += __shfl_xor_sync(0xffffffffu, sdot, o);
              if (r < len) {
                float vf[8];
                bf16x8_to_f32(vr[p], vf);
                if (sdot > mx) {
                  const float cc = __expf(mx - sdot);
                  ls = __fmul_rn(ls, cc);
#pragma unroll
                  for (int t = 0; t < 8; ++t) acc[t] = __fmul_rn(acc[t], cc);
                  mx = sdot;
                }
                const float pr = __expf(sdot - mx);
                ls = __fadd_rn(ls, pr);
#pragma unroll
                for (int t = 0; t < 8; ++t) acc[t] = __fmaf_rn(pr, vf[t], acc[t]);
              }
            }
          }
          // row groups -> head output in group order (shared memory)
          if (li == 0) { gstat[grp][0] = mx; gstat[grp][1] = ls; }
#pragma unroll
          for (int t = 0; t < 8; ++t) part[grp][li * 8 + t] = acc[t];
          __syncthreads();
          for (int e = tid; e < HD; e += DR_THREADS) {
            float M = -INFINITY;
            for (int q = 0; q < RPP; ++q) M = fmaxf(M, gstat[q][0]);
            float L = 0.f, o = 0.f;
            for (int q = 0; q < RPP; ++q) {
              if (gstat[q][0] == -INFINITY) continue;
              const float cc = __expf(gstat[q][0] - M);
              L = __fadd_rn(L, __fmul_rn(gstat[q][1], cc));
              o = __fadd_rn(o, __fmul_rn(part[q][e], cc));
            }
            attn_s[e] = o / L;
          }
          __syncthreads();
          // this member's rows of the head's O columns (SWZ8 units)
          float av[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) av[j] = attn_s[lr * 8 + j];
          float* op = a.opart + (size_t)hh * d;
          for (int rb = r0 + warp * RW; rb < r1; rb += DR_WARPS * RW * WB) {
            uint4 wv[WB];
#pragma unroll
            for (int b = 0; b < WB; ++b) {
              const int r = rb + b * DR_WARPS * RW + rw;
              const int un = (hh * HD) / 8 + lr;
              wv[b] = wone ? wpre[b]
                      : r < r1 ? ld_stream16(Lw.o + (size_t)r * qd + (size_t)(un ^ (r & 7)) * 8)
                               : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
            for (int b = 0; b < WB; ++b) {
              float wf[8];
              bf16x8_to_f32(wv[b], wf);
              float t = 0.f;
#pragma unroll
              for (int j = 0; j < 8; ++j) t = __fmaf_rn(wf[j], av[j], t);
#pragma unroll
              for (int o = LR / 2; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
              const int r = rb + b * DR_WARPS * RW + rw;
              if (lr == 0 && r < r1) op[r] = t;
            }
          }
        }
      } else
      {
        // one CTA per (token, head, split of ACH rows); each thread issues
        // ALL of its K and V loads up front (one round trip)
        constexpr int LPR = HD / 8;              // lanes per K/V row
        constexpr int RPP = DR_THREADS / LPR;    // rows per pass
        constexpr int PASSES = 8;
        constexpr int ACH = RPP * PASSES;        // 256 (hd 64) / 128 (hd 128)
        const int grp = tid / LPR, li = tid % LPR;
        const int rows_last = rowA + n;          // rows visible to the last token
        const int nsplit = (rows_last + ACH - 1) / ACH;
        const int items = n * a.H * nsplit;
        for (int it = blockIdx.x; it < items; it += gridDim.x) {
          const int m = it / (a.H * nsplit);
          const int hh = (it / nsplit) % a.H;
          const int s = it % nsplit;
          const int len = rowA + m + 1;
          const int ns = (len + ACH - 1) / ACH;
          if (s >= ns) continue;
          const int kh = hh / (a.H / a.KH);
          const int e0 = s * ACH, e1 = min(len, e0 + ACH);
          uint4 kr[PASSES], vr[PASSES];
#pragma unroll
          for (int p = 0; p < PASSES; ++p) {
            const int r = e0 + p * RPP + grp;
            const size_t off = (size_t)r * kvd + kh * HD + li * 8;
            kr[p] = r < e1 ? ldcg16(Kc + off) : make_uint4(0, 0, 0, 0);
            vr[p] = r < e1 ? ldcg16(Vc + off) : make_uint4(0, 0, 0, 0);
          }
          mark(60);
          float qv[8];
          {
            const float* qp = a.q + (size_t)m * qd + hh * HD + li * 8;
            const float4 q0 = __ldcg(reinterpret_cast<const float4*>(qp));
            const float4 q1 = __ldcg(reinterpret_cast<const float4*>(qp + 4));
            qv[0] = q0.x * att_scale; qv[1] = q0.y * att_scale;
            qv[2] = q0.z * att_scale; qv[3] = q0.w * att_scale;
            qv[4] = q1.x * att_scale; qv[5] = q1.y * att_scale;
            qv[6] = q1.z * att_scale; qv[7] = q1.w * att_scale;
          }
          float scv[PASSES];
          float mx = -INFINITY;
#pragma unroll
          for (int p = 0; p < PASSES; ++p) {
            float kf[8];
            bf16x8_to_f32(kr[p], kf);
            float dsum = 0.f;
#pragma unroll
            for (int j = 0; j < 8; ++j) dsum = __fmaf_rn(qv[j], kf[j], dsum);
#pragma unroll
            for (int o = LPR / 2; o > 0; o >>= 1) dsum += __shfl_xor_sync(0xffffffffu, dsum, o);
            const int r = e0 + p * RPP + grp;
            scv[p] = r < e1 ? dsum : -INFINITY;
            mx = fmaxf(mx, scv[p]);
          }
          mark(61);
          mx = warp_max(mx);
          if (lane == 0) wred[warp] = mx;
          __syncthreads();
          mark(62);
          mx = wred[0];
#pragma unroll
          for (int w = 1; w < DR_WARPS; ++w) mx = fmaxf(mx, wred[w]);
          __syncthreads();
          float acc[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[j] = 0.f;
          float psum = 0.f;
#pragma unroll
          for (int p = 0; p < PASSES; ++p) {
            const float pr = scv[p] == -INFINITY ? 0.f : __expf(scv[p] - mx);
            psum += pr;
            float vf[8];
            bf16x8_to_f32(vr[p], vf);
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[j] = __fmaf_rn(pr, vf[j], acc[j]);
          }
          float sum = warp_sum(li == 0 ? psum : 0.f);   // one lane per row group
          if (lane == 0) wred[warp] = sum;
#pragma unroll
          for (int j = 0; j < 8; ++j) part[grp][li * 8 + j] = acc[j];
          __syncthreads();
          sum = wred[0];
#pragma unroll
          for (int w = 1; w < DR_WARPS; ++w) sum += wred[w];
          mark(63);
          bool have = false;
          if (ns == 1) {
            for (int e = tid; e < HD; e += DR_THREADS) {
              float o = part[0][e];
              for (int g = 1; g < RPP; ++g) o += part[g][e];
              attn_s[e] = o / sum;
            }
            have = true;
          } else {
            float* pp = a.att_part + (((size_t)m * a.H + hh) * a.max_split + s) * (HD + 2);
            for (int e = tid; e < HD; e += DR_THREADS) {
              float o = part[0][e];
              for (int g = 1; g < RPP; ++g) o += part[g][e];
              pp[2 + e] = o;
            }
            if (tid == 0) { pp[0] = mx; pp[1] = sum; }
            __threadfence();
            __syncthreads();
            if (tid == 0) last = (atomicAdd(a.att_tick + m * a.H + hh, 1) == ns - 1);
            __syncthreads();
            if (last) {
              __threadfence();
              const float* base = a.att_part + ((size_t)m * a.H + hh) * a.max_split * (HD + 2);
              float M = -INFINITY;
              for (int t = 0; t < ns; ++t) M = fmaxf(M, __ldcg(base + t * (HD + 2)));
              float Ls = 0.f;
              for (int t = 0; t < ns; ++t)
                Ls += __ldcg(base + t * (HD + 2) + 1) * __expf(__ldcg(base + t * (HD + 2)) - M);
              for (int e = tid; e < HD; e += DR_THREADS) {
                float o = 0.f;
                for (int t = 0; t < ns; ++t)
                  o += __ldcg(base + t * (HD + 2) + 2 + e) * __expf(__ldcg(base + t * (HD + 2)) - M);
                attn_s[e] = o / Ls;
              }
              if (tid == 0) a.att_tick[m * a.H + hh] = 0;
              have = true;
            }
          }
          mark(64);
          if (have) {
            // O partial of this head: opart[m][hh][r] = Wo[r, hh*HD:(hh+1)*HD] . attn_h
            // (8 lanes per row, 16 B each for hd 64; batches of 8 rows per lane)
            __syncthreads();
            constexpr int LR = HD / 8;                // lanes per Wo row segment
            constexpr int RW = 32 / LR;               // rows per warp pass
            const int lr = lane % LR, rw = lane / LR;
            float av[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) av[j] = attn_s[lr * 8 + j];
            float* op = a.opart + ((size_t)m * a.H + hh) * d;
            constexpr int OB = 24;                    // rows per lane per batch
            for (int r0 = warp * RW; r0 < d; r0 += DR_WARPS * RW * OB) {
              uint4 wv[OB];
#pragma unroll
              for (int b = 0; b < OB; ++b) {
                const int r = r0 + b * DR_WARPS * RW + rw;
                const int un = (hh * HD) / 8 + lr;            // SWZ8 unit of row r
                wv[b] = r < d ? ld_stream16(Lw.o + (size_t)r * qd + (size_t)(un ^ (r & 7)) * 8)
                              : make_uint4(0, 0, 0, 0);
              }
              mark(65);
#pragma unroll
              for (int b = 0; b < OB; ++b) {
                float wf[8];
                bf16x8_to_f32(wv[b], wf);
                float t = 0.f;
#pragma unroll
                for (int j = 0; j < 8; ++j) t = __fmaf_rn(wf[j], av[j], t);
#pragma unroll
                for (int o = LR / 2; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
                const int r = r0 + b * DR_WARPS * RW + rw;
                if (lr == 0 && r < d) op[r] = t;
              }
            }
            mark(66);
          }
          __syncthreads();
        }
      }
      mark(2); grid_sync(a.bar, target, a.spin_ns); mark(10);

      // --- D: x += sum_h O partials; h = silu(g) * u of rmsnorm(x) ----------
      for (int m = 0; m < n; ++m) {
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int c = (tid + i * DR_THREADS) * 4;
          if (c >= d) break;
          // x + sum of the heads' O partials in ascending head order; all
          // loads of a 16-head group are issued before the adds
          float4 v = __ldcg(reinterpret_cast<const float4*>(a.x + (size_t)m * d + c));
          const float4 g = __ldg(reinterpret_cast<const float4*>(Lw.g_mlp + c));
          const float* op = a.opart + (size_t)m * a.H * d + c;
          for (int h0 = 0; h0 < a.H; h0 += 16) {
            float4 o[16];
#pragma unroll
            for (int j = 0; j < 16; ++j)
              o[j] = h0 + j < a.H ? __ldcg(reinterpret_cast<const float4*>(op + (size_t)(h0 + j) * d))
                                  : make_float4(0, 0, 0, 0);
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              if (h0 + j >= a.H) break;
              v.x = __fadd_rn(v.x, o[j].x); v.y = __fadd_rn(v.y, o[j].y);
              v.z = __fadd_rn(v.z, o[j].z); v.w = __fadd_rn(v.w, o[j].w);
            }
          }
          *reinterpret_cast<float4*>(xr + (size_t)m * d + c) = v;
          *reinterpret_cast<float4*>(xs + (size_t)m * d + c) =
              make_float4(__fmul_rn(v.x, g.x), __fmul_rn(v.y, g.y), __fmul_rn(v.z, g.z),
                          __fmul_rn(v.w, g.w));
          if (!isfinite(v.x) || !isfinite(v.y) || !isfinite(v.z) || !isfinite(v.w))
            set_error(a.err, SP_DEV_NONFINITE);
        }
      }
      __syncthreads();
      {
        float scl[DR_NT];
        warp_scales(d, n, scl);
        mark(36); wwait(1); mark(52);
        for (int u = up0 + 3 * warp; u < up1; u += 3 * DR_WARPS) {
          // three gate/up pairs per warp at once (ILP across rows)
          const __nv_bfloat16* w6[6];
#pragma unroll
          for (int j = 0; j < 3; ++j) {
            const bool ok = u + j < up1;
            w6[2 * j] = ok ? bufD + (size_t)(2 * (u + j - up0)) * d : nullptr;
            w6[2 * j + 1] = ok ? bufD + (size_t)(2 * (u + j - up0) + 1) * d : nullptr;
          }
          float y[6][DR_NT];
          warp_dot_s<DR_NT, 6>(reinterpret_cast<const __nv_bfloat16* const(&)[6]>(w6), xs, d, n, y,
                               2 * u);
          if (lane < n) {
#pragma unroll
            for (int j = 0; j < 3; ++j) {
              if (u + j >= up1) break;
              float g = 0.f, uu = 0.f;
#pragma unroll
              for (int mm = 0; mm < DR_NT; ++mm)
                if (mm == lane) {
                  g = __fmul_rn(y[2 * j][mm], scl[mm]);
                  uu = __fmul_rn(y[2 * j + 1][mm], scl[mm]);
                }
              a.h[(size_t)lane * f + u + j] = __fmul_rn(silu(g), uu);
            }
          }
        }
      }
      mark(4); grid_sync(a.bar, target, a.spin_ns); mark(12);

      // ---------------- E: x = x_attn + h @ Wd (row owners) -----------------
      if (l + 1 < a.L) wload(1, l + 1);
      else if (k < steps) wload(1, 0);
      {
        float4 hv[DR_NT][4];            // f <= 4096
#pragma unroll
        for (int m = 0; m < DR_NT; ++m)
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int c = (tid + i * DR_THREADS) * 4;
            hv[m][i] = (m < n && c < f)
                           ? __ldcg(reinterpret_cast<const float4*>(a.h + (size_t)m * f + c))
                           : make_float4(0, 0, 0, 0);
          }
#pragma unroll
        for (int m = 0; m < DR_NT; ++m)
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int c = (tid + i * DR_THREADS) * 4;
            if (m < n && c < f) *reinterpret_cast<float4*>(xs + (size_t)m * f + c) = hv[m][i];
          }
      }
      __syncthreads();
      mark(37); wwait(2); mark(53);
      for (int r = d0 + 2 * warp; r < d1; r += 2 * DR_WARPS) {
        const __nv_bfloat16* const w2[2] = {
            bufE + (size_t)(r - d0) * f, r + 1 < d1 ? bufE + (size_t)(r + 1 - d0) * f : nullptr};
        float y[2][DR_NT];
        warp_dot_s<DR_NT, 2>(w2, xs, f, n, y, r);
        if (lane < 2 * n) {
          const int m = lane >> 1, rr = r + (lane & 1);
          if (rr < d1) {
            float v = 0.f;
#pragma unroll
            for (int mm = 0; mm < DR_NT; ++mm)
              if (mm == m) v = (lane & 1) ? y[1][mm] : y[0][mm];
            const float nv = __fadd_rn(xr[(size_t)m * d + rr], v);
            a.x[(size_t)m * d + rr] = nv;
            if (!isfinite(nv)) set_error(a.err, SP_DEV_NONFINITE);
          }
        }
      }
      mark(5); grid_sync(a.bar, target, a.spin_ns); mark(13);
    }

    // ---------------- H: final norm + LM head over the last token ----------
    {
      const int m = n - 1;
      for (int c = tid * 4; c < d; c += DR_THREADS * 4) {
        const float4 v = __ldcg(reinterpret_cast<const float4*>(a.x + (size_t)m * d + c));
        const float4 g = __ldg(reinterpret_cast<const float4*>(a.g_final + c));
        *reinterpret_cast<float4*>(xr + c) = v;
        *reinterpret_cast<float4*>(xs + c) =
            make_float4(__fmul_rn(v.x, g.x), __fmul_rn(v.y, g.y), __fmul_rn(v.z, g.z),
                        __fmul_rn(v.w, g.w));
      }
      __syncthreads();
      float scl[DR_NT];
      warp_scales(d, 1, scl);
      DTop2 t{-INFINITY, 0x7fffffff, -INFINITY, 0x7fffffff};
      float mx = -INFINITY, se = 0.f;
      int nan = 0;
      const float sc0 = scl[0];
      for (int r = v0 + 8 * warp; r < v1; r += 8 * DR_WARPS) {
        const __nv_bfloat16* w8[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) w8[j] = r + j < v1 ? a.w_out + (size_t)(r + j) * d : nullptr;
        float y[8][1];
        warp_dot<1, 8>(reinterpret_cast<const __nv_bfloat16* const(&)[8]>(w8), xs, d, 1, y, r);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (r + j >= v1) break;
          const float v = __fmul_rn(y[j][0], sc0);
          if (isnan(v)) { nan = 1; continue; }
          dpush(t, v, r + j);
          online_add(mx, se, v);
        }
      }
      if (lane == 0) {
        lm_w[warp][0] = t.v1; lm_w[warp][1] = t.v2; lm_w[warp][2] = mx; lm_w[warp][3] = se;
        lm_wi[warp][0] = t.i1; lm_wi[warp][1] = t.i2; lm_wi[warp][2] = nan;
      }
      __syncthreads();
      if (tid == 0) {
        DTop2 c{-INFINITY, 0x7fffffff, -INFINITY, 0x7fffffff};
        float cm = -INFINITY, cs = 0.f;
        int cn = 0;
        for (int w = 0; w < DR_WARPS; ++w) {
          dpush(c, lm_w[w][0], lm_wi[w][0]);
          dpush(c, lm_w[w][1], lm_wi[w][1]);
          online_merge(cm, cs, lm_w[w][2], lm_w[w][3]);
          cn |= lm_wi[w][2];
        }
        LmPartial p{c.v1, c.i1, c.v2, c.i2, cm, cs, cn, 0};
        a.lm_part[blockIdx.x] = p;
      }
    }
    mark(6); grid_sync(a.bar, target, a.spin_ns); mark(14);
    {
      // every CTA merges all partials in the same fixed order: thread t
      // takes partial t (one round trip), then butterflies and warps 0..7
      DTop2 t{-INFINITY, 0x7fffffff, -INFINITY, 0x7fffffff};
      float pm = -INFINITY, ps = 0.f;
      int nan = 0;
      for (int c = tid; c < (int)gridDim.x; c += DR_THREADS) {
        const LmPartial* P = a.lm_part + c;
        const float4 lo = __ldcg(reinterpret_cast<const float4*>(P));
        const float4 hi = __ldcg(reinterpret_cast<const float4*>(P) + 1);
        dpush(t, lo.x, __float_as_int(lo.y));
        dpush(t, lo.z, __float_as_int(lo.w));
        online_merge(pm, ps, hi.x, hi.y);
        nan |= __float_as_int(hi.z);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const float a1 = __shfl_xor_sync(0xffffffffu, t.v1, o);
        const int b1 = __shfl_xor_sync(0xffffffffu, t.i1, o);
        const float a2 = __shfl_xor_sync(0xffffffffu, t.v2, o);
        const int b2 = __shfl_xor_sync(0xffffffffu, t.i2, o);
        dpush(t, a1, b1);
        dpush(t, a2, b2);
        const float m2 = __shfl_xor_sync(0xffffffffu, pm, o);
        const float s2 = __shfl_xor_sync(0xffffffffu, ps, o);
        online_merge(pm, ps, m2, s2);   // symmetric: same result on both partners
        nan |= __shfl_xor_sync(0xffffffffu, nan, o);
      }
      if (lane == 0) {
        lm_w[warp][0] = t.v1; lm_w[warp][1] = t.v2; lm_w[warp][2] = pm; lm_w[warp][3] = ps;
        lm_wi[warp][0] = t.i1; lm_wi[warp][1] = t.i2; lm_wi[warp][2] = nan;
      }
      __syncthreads();
      if (tid == 0) {
        DTop2 c{-INFINITY, 0x7fffffff, -INFINITY, 0x7fffffff};
        float cm = -INFINITY, cs = 0.f;
        int cn = 0;
        for (int w = 0; w < DR_WARPS; ++w) {
          dpush(c, lm_w[w][0], lm_wi[w][0]);
          dpush(c, lm_w[w][1], lm_wi[w][1]);
          online_merge(cm, cs, lm_w[w][2], lm_w[w][3]);
          cn |= lm_wi[w][2];
        }
        const float conf = 1.0f / cs;
        s_next_tok = c.i1;
        s_gate = (conf >= cutoff) ? 1 : 0;
        if (blockIdx.x == 0) {
          sp_row_result r;
          r.argmax = c.i1;
          r.second = c.i2;
          r.conf = conf;
          r.max_logit = c.v1;
          a.out[k] = r;
          a.tip[0] = c.i1;
          a.tip[1] = __float_as_int(conf);
          a.tip[2] = 1;
          if (chain) *a.gate = s_gate;
          if (cn) set_error(a.err, SP_DEV_NAN_LOGITS);
        }
      }
    }
    __syncthreads();
    tip_tok = s_next_tok;
    gate = chain ? s_gate : 1;
    row += n;
    pos += n;
  }
  // never exit with a bulk copy still landing in shared memory
  for (int i = 0; i < 3; ++i)
    if (wpend[i]) wwait(i);
  if (a.prof && blockIdx.x == 0 && tid == 0) {
    a.prof[1 + nprof] = (15ll << 56) | (clock64() & ((1ll << 56) - 1));
    a.prof[0] = nprof + 1;
  }
  if (blockIdx.x == 0 && tid == 0 && a.err_out) {
    __threadfence();
    *a.err_out = *a.err;
  }
}

size_t draft_smem_bytes(const DraftArgs& a) {
  return (size_t)a.bufA + a.bufD + a.bufE + sizeof(float) * (size_t)DR_NT * (a.kmax + a.d);
}

void draft_buffers(DraftArgs& a, int ctas) {
  // per-CTA weight slices of the three staged phases (QKV, gate/up, down)
  auto per = [&](long units) { return (units + ctas - 1) / ctas; };
  auto r128 = [](long b) { return (int)((b + 127) / 128 * 128); };
  const long qd = (long)a.H * a.hd, kvd = (long)a.KH * a.hd;
  a.bufA = r128(per((qd + 2 * kvd) / 2) * 2 * a.d * 2);
  a.bufD = r128(per(a.f) * 2 * (long)a.d * 2);
  a.bufE = r128(per(a.d) * (long)a.f * 2);
  int kmax = a.d > a.f ? a.d : a.f;
  a.kmax = kmax > (int)qd ? kmax : (int)qd;
}

template <int HD>
static cudaError_t launch_hd(const DraftArgs& a, int ctas, cudaStream_t st) {
  const size_t smem = draft_smem_bytes(a);
  cudaError_t e = cudaFuncSetAttribute(draft_chain_kernel<HD>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ctas);
  cfg.blockDim = dim3(DR_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;   // co-residency for grid_sync
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, draft_chain_kernel<HD>, a);
}

template <int HD>
static int max_ctas_hd(const DraftArgs& a) {
  const size_t smem = draft_smem_bytes(a);
  if (cudaFuncSetAttribute(draft_chain_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem) != cudaSuccess)
    return 0;
  int per_sm = 0, dev = 0, sms = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, draft_chain_kernel<HD>, DR_THREADS,
                                                    smem) != cudaSuccess)
    return 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return per_sm * sms;
}

int draft_max_ctas(const DraftArgs& a) {
  if (a.hd == 64) return max_ctas_hd<64>(a);
  if (a.hd == 128) return max_ctas_hd<128>(a);
  return 0;
}

cudaError_t launch_draft_chain(const DraftArgs& a, int ctas, cudaStream_t st) {
  if (a.hd == 64) return launch_hd<64>(a, ctas, st);
  if (a.hd == 128) return launch_hd<128>(a, ctas, st);
  return cudaErrorInvalidValue;
}

}  // namespace sp
