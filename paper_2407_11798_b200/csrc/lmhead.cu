// K9: fused final RMSNorm + LM head + greedy_sample / second_best /
// max_softmax (model.py:424-457).  The output per flagged row is a 16-byte
// record instead of V logits; full logits are written only when requested
// (parity tests).  Per-CTA partials (top-2 by (value desc, id asc), running
// max, sum of exp) are merged by the last-arriving CTA in CTA order, so the
// result is independent of scheduling.
#include "gemv_core.cuh"
#include "kernels.cuh"

namespace sp {

struct Top2 {
  float v1; int i1; float v2; int i2;
};

// (a before b) iff a.v > b.v or (a.v == b.v and a.i < b.i); NaN never wins
__device__ __forceinline__ bool better(float va, int ia, float vb, int ib) {
  return va > vb || (va == vb && ia < ib);
}

__device__ __forceinline__ void push(Top2& t, float v, int i) {
  if (better(v, i, t.v1, t.i1)) { t.v2 = t.v1; t.i2 = t.i1; t.v1 = v; t.i1 = i; }
  else if (better(v, i, t.v2, t.i2)) { t.v2 = v; t.i2 = i; }
}

__device__ __forceinline__ void push_top2(LmPartial& s, const Top2& t) {
  Top2 u{s.v1, s.i1, s.v2, s.i2};
  push(u, t.v1, t.i1);
  push(u, t.v2, t.i2);
  s.v1 = u.v1; s.i1 = u.i1; s.v2 = u.v2; s.i2 = u.i2;
}





constexpr int LM_ROWS = 8;        // weight rows per block (gemv_core tile)
#ifndef LM_CTAS_DEF
#define LM_CTAS_DEF (4 * 148)
#endif
constexpr int LM_CTAS = LM_CTAS_DEF;  // persistent grid: a fixed constant, so the
                                  // per-CTA partition (and conf's summation
                                  // order) never depends on the device

__device__ __forceinline__ void lm_fold(LmPartial& s, const Top2& t, float mx, float se,
                                        int nan) {
  push_top2(s, t);
  if (mx != -INFINITY) {
    if (s.mx == -INFINITY) {
      s.mx = mx; s.se = se;
    } else {
      const float M = fmaxf(s.mx, mx);
      s.se = __fadd_rn(__fmul_rn(s.se, __expf(s.mx - M)), __fmul_rn(se, __expf(mx - M)));
      s.mx = M;
    }
  }
  s.nan |= nan;
}

// Persistent LM head: CTA b owns row blocks b, b + G, ... (ascending) and
// keeps a running (top-2, max, sum-exp) per token in shared memory; each
// weight block is read once for all tokens (token tiles reuse it from L1).
template <typename T, int MT>
__global__ void __launch_bounds__(GEMV_THREADS) lmhead_kernel(const LmArgs a) {
  pdl_wait();
  pdl_trigger();
  __shared__ GemvSmem<T, MT, LM_ROWS, true> sm;
  __shared__ int last;
  extern __shared__ LmPartial st[];  // [n_rows]
  if (run_skipped(a.run_state)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      if (a.gate) *a.gate = 0;
      if (a.err_out) *a.err_out = a.err ? *a.err : 0;
      if (a.status_out) *a.status_out = SP_STATUS_PLACEHOLDER;
    }
    return;
  }
  const int G = gridDim.x;
  for (int m = threadIdx.x; m < a.n_rows; m += blockDim.x)
    st[m] = LmPartial{-INFINITY, 0x7fffffff, -INFINITY, 0x7fffffff, -INFINITY, 0.f, 0, 0};
  __syncthreads();
  const T* W = reinterpret_cast<const T*>(a.w);
  const int nblk = (a.V + LM_ROWS - 1) / LM_ROWS;
  for (int b = blockIdx.x; b < nblk; b += G) {
    const int row0 = b * LM_ROWS;
    for (int mt0 = 0; mt0 < a.n_rows; mt0 += MT) {
      const int mv = min(MT, a.n_rows - mt0);
      gemv_core<T, MT, LM_ROWS, true>(W, a.V, a.d, a.x + (size_t)mt0 * a.d, a.d, mv,
                                      a.norm ? a.gain : nullptr, row0, sm, a.swz);
      if (threadIdx.x < mv) {
        const int m = threadIdx.x, mi = mt0 + m;
        const float sc = a.norm ? rms_scale(sm.ss[0][m], a.d, a.eps) : 1.0f;
        Top2 t{-INFINITY, 0x7fffffff, -INFINITY, 0x7fffffff};
        float mx = -INFINITY;
        int nan = 0;
        float vals[LM_ROWS];
#pragma unroll
        for (int r = 0; r < LM_ROWS; ++r) {
          vals[r] = -INFINITY;
          const int id = row0 + r;
          if (id < a.V) {
            const float v = __fmul_rn(sm.red[0][m][r], sc);
            vals[r] = v;
            if (a.logits) a.logits[(size_t)mi * a.V + id] = v;
            if (isnan(v)) nan = 1;
            else { push(t, v, id); mx = fmaxf(mx, v); }
          }
        }
        float se = 0.f;
#pragma unroll
        for (int r = 0; r < LM_ROWS; ++r)
          if (row0 + r < a.V && !isnan(vals[r])) se += __expf(vals[r] - mx);
        lm_fold(st[mi], t, mx, se, nan);
      }
      __syncthreads();
    }
  }
  for (int m = threadIdx.x; m < a.n_rows; m += blockDim.x)
    a.scratch[(size_t)m * G + blockIdx.x] = st[m];
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = (atomicAdd(a.ticket, 1) == G - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  // merge: one warp per row; lanes take CTA partials lane, lane+32, ... and
  // combine in a fixed order (top-2 and max are order-free; the sum of exp
  // is rescaled to the global max in a fixed lane order + butterfly)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int m = warp; m < a.n_rows; m += GEMV_WARPS) {
    const LmPartial* P = a.scratch + (size_t)m * G;
    Top2 t{-INFINITY, 0x7fffffff, -INFINITY, 0x7fffffff};
    float mx = -INFINITY;
    int nan = 0;
    constexpr int UN = 4;
    for (int c0 = lane; c0 < G; c0 += 32 * UN) {
      LmPartial q[UN];
#pragma unroll
      for (int u = 0; u < UN; ++u) {
        const int c = c0 + 32 * u;
        if (c < G) {
          const float4 lo = __ldcg(reinterpret_cast<const float4*>(P + c));
          const float4 hi = __ldcg(reinterpret_cast<const float4*>(P + c) + 1);
          q[u] = LmPartial{lo.x, __float_as_int(lo.y), lo.z, __float_as_int(lo.w),
                           hi.x, hi.y, __float_as_int(hi.z), 0};
        } else {
          q[u] = LmPartial{-INFINITY, 0x7fffffff, -INFINITY, 0x7fffffff, -INFINITY, 0.f, 0, 0};
        }
      }
#pragma unroll
      for (int u = 0; u < UN; ++u) {
        push(t, q[u].v1, q[u].i1);
        push(t, q[u].v2, q[u].i2);
        mx = fmaxf(mx, q[u].mx);
        nan |= q[u].nan;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float v1 = __shfl_xor_sync(0xffffffffu, t.v1, o);
      const int i1 = __shfl_xor_sync(0xffffffffu, t.i1, o);
      const float v2 = __shfl_xor_sync(0xffffffffu, t.v2, o);
      const int i2 = __shfl_xor_sync(0xffffffffu, t.i2, o);
      push(t, v1, i1);
      push(t, v2, i2);
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      nan |= __shfl_xor_sync(0xffffffffu, nan, o);
    }
    float se = 0.f;
    for (int c = lane; c < G; c += 32) {
      const float2 ms = __ldcg(reinterpret_cast<const float2*>(P + c) + 2);
      if (ms.x != -INFINITY) se += ms.y * __expf(ms.x - mx);
    }
    se = warp_sum(se);
    if (lane == 0) {
      sp_row_result r;
      r.argmax = t.i1;
      r.second = t.i2;
      r.conf = 1.0f / se;   // exp(max - max) / sum
      r.max_logit = t.v1;
      a.out[m] = r;
      if (nan) set_error(a.err, SP_DEV_NAN_LOGITS);
      if (a.tip && m == a.n_rows - 1) {
        a.tip[0] = r.argmax;
        a.tip[1] = __float_as_int(r.conf);
        a.tip[2] = 1;
        if (a.gate && a.chain_gate) {
          const int g = *a.gate;
          const float cut = a.hdr ? a.hdr->cutoff : a.cutoff;
          *a.gate = (g != 0 && r.conf >= cut) ? 1 : 0;
        }
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    *a.ticket = 0;
    if (a.err_out) *a.err_out = a.err ? *a.err : 0;
    if (a.status_out) *a.status_out = SP_STATUS_VALID;
  }
}

int lmhead_grid(int V) { return min((V + LM_ROWS - 1) / LM_ROWS, LM_CTAS); }

cudaError_t launch_lmhead(const LmArgs& a, int w_dtype, cudaStream_t st) {
  const dim3 grid(lmhead_grid(a.V));
  const dim3 blk(GEMV_THREADS);
  const size_t smem = sizeof(LmPartial) * (size_t)a.n_rows;
  if (smem > 48 * 1024) return cudaErrorInvalidValue;
  if (w_dtype == SP_DTYPE_BF16) {
    // one token tile per weight pass up to 8 rows (a verification run's rows
    // share every streamed weight chunk; two tiles re-stream the head:
    // measured 5 rows 251 us with 4-row tiles)
    if (a.n_rows <= 1) return launch_pdl(lmhead_kernel<__nv_bfloat16, 1>, grid, blk, smem, st, a);
    if (a.n_rows <= 8) return launch_pdl(lmhead_kernel<__nv_bfloat16, 8>, grid, blk, smem, st, a);
    return launch_pdl(lmhead_kernel<__nv_bfloat16, 4>, grid, blk, smem, st, a);
  }
  if (a.n_rows <= 1) return launch_pdl(lmhead_kernel<float, 1>, grid, blk, smem, st, a);
  return launch_pdl(lmhead_kernel<float, 4>, grid, blk, smem, st, a);
}

}  // namespace sp
