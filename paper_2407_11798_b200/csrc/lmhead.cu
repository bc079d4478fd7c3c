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





template <typename T, int MT, int ROWS>
__global__ void __launch_bounds__(GEMV_THREADS) lmhead_kernel(const LmArgs a) {
  pdl_wait();
  pdl_trigger();
  __shared__ GemvSmem<T, MT, ROWS, true> sm;
  __shared__ int last;
  if (run_skipped(a.run_state)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      if (a.gate) *a.gate = 0;
      if (a.err_out) *a.err_out = a.err ? *a.err : 0;
    }
    return;
  }
  const int row0 = blockIdx.x * ROWS;
  const T* W = reinterpret_cast<const T*>(a.w);
  for (int mt0 = 0; mt0 < a.n_rows; mt0 += MT) {
    const int mv = min(MT, a.n_rows - mt0);
    if (a.norm)
      gemv_core<T, MT, ROWS, true>(W, a.V, a.d, a.x + (size_t)mt0 * a.d, a.d, mv,
                                   a.gain, row0, sm);
    else
      gemv_core<T, MT, ROWS, true>(W, a.V, a.d, a.x + (size_t)mt0 * a.d, a.d, mv,
                                   nullptr, row0, sm);
    if (threadIdx.x < mv) {
      const int m = threadIdx.x, mi = mt0 + m;
      const float sc = a.norm ? rms_scale(sm.ss[0][m], a.d, a.eps) : 1.0f;
      Top2 t{-INFINITY, 0x7fffffff, -INFINITY, 0x7fffffff};
      float mx = -INFINITY;
      int nan = 0;
      float vals[ROWS];
#pragma unroll
      for (int r = 0; r < ROWS; ++r) {
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
      for (int r = 0; r < ROWS; ++r)
        if (row0 + r < a.V && !isnan(vals[r])) se += __expf(vals[r] - mx);
      a.scratch[(size_t)mi * gridDim.x + blockIdx.x] =
          LmPartial{t.v1, t.i1, t.v2, t.i2, mx, se, nan, 0};
    }
    __syncthreads();
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = (atomicAdd(a.ticket, 1) == (int)gridDim.x - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  // merge: one warp per flagged row, CTA partials in ascending order
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int m = warp; m < a.n_rows; m += GEMV_WARPS) {
    const volatile LmPartial* P = a.scratch + (size_t)m * gridDim.x;
    Top2 t{-INFINITY, 0x7fffffff, -INFINITY, 0x7fffffff};
    float mx = -INFINITY;
    int nan = 0;
    for (int c = lane; c < (int)gridDim.x; c += 32) {
      push(t, P[c].v1, P[c].i1);
      push(t, P[c].v2, P[c].i2);
      mx = fmaxf(mx, P[c].mx);
      nan |= P[c].nan;
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
    // sum of exp relative to the global max, fixed order per lane + butterfly
    float se = 0.f;
    for (int c = lane; c < (int)gridDim.x; c += 32) se += P[c].se * __expf(P[c].mx - mx);
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
          *a.gate = (g != 0 && r.conf >= a.cutoff) ? 1 : 0;
        }
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    *a.ticket = 0;
    if (a.err_out) *a.err_out = a.err ? *a.err : 0;
  }
}

cudaError_t launch_lmhead(const LmArgs& a, int w_dtype, cudaStream_t st) {
  constexpr int ROWS = 8;
  const dim3 grid((a.V + ROWS - 1) / ROWS);
  const dim3 blk(GEMV_THREADS);
  if (w_dtype == SP_DTYPE_BF16) {
    if (a.n_rows <= 1) return launch_pdl(lmhead_kernel<__nv_bfloat16, 1, ROWS>, grid, blk, 0, st, a);
    return launch_pdl(lmhead_kernel<__nv_bfloat16, 4, ROWS>, grid, blk, 0, st, a);
  }
  if (a.n_rows <= 1) return launch_pdl(lmhead_kernel<float, 1, ROWS>, grid, blk, 0, st, a);
  return launch_pdl(lmhead_kernel<float, 4, ROWS>, grid, blk, 0, st, a);
}

int lmhead_grid(int V) { return (V + 7) / 8; }

}  // namespace sp
