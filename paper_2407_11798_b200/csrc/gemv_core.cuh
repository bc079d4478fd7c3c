// Weight-streaming GEMV core shared by the layer GEMVs and the LM head.
//
// Computes, for one CTA's ROWS consecutive weight rows and up to MT tokens,
//     acc[m][r] = sum_k W[row0 + r][k] * (x[m][k] * gain[k])
// and, when NORM, ss[m] = sum_k x[m][k]^2 (the RMSNorm statistic, fused:
// rmsnorm(x) @ W == (x @ W) / sqrt(mean(x^2) + eps), model.py:188-189).
//
// Layout: W is [n_rows, K] row-major (K contiguous) so every lane issues
// 16-byte streaming loads; 8 warps split K into 32*VEC-element chunks
// (chunk c belongs to warp c % 8).  The reduction order for one (m, r) is
// fixed — chunks ascending per lane, fixed butterfly across lanes, warps
// 0..7 in order — and independent of MT and of the batch, so a token's
// result is bitwise identical whether it is evaluated alone or batched.
#pragma once

#include "common.cuh"

namespace sp {

constexpr int GEMV_THREADS = 256;
constexpr int GEMV_WARPS = GEMV_THREADS / 32;

template <typename T, int MT, int ROWS, bool NORM>
struct GemvSmem {
  float red[GEMV_WARPS][MT][ROWS];
  float ss[GEMV_WARPS][MT];
};

// After return (and a __syncthreads inside), sm.red[0][m][r] holds the full
// dot product and sm.ss[0][m] the sum of squares, for m < MT.
template <typename T, int MT, int ROWS, bool NORM>
__device__ __forceinline__ void gemv_core(const T* __restrict__ W, int n_rows,
                                          int K, const float* __restrict__ x,
                                          int ldx, int m_valid,
                                          const float* __restrict__ gain,
                                          int row0,
                                          GemvSmem<T, MT, ROWS, NORM>& sm, int swz = 0) {
  constexpr int VEC = VecTraits<T>::N;
  constexpr int CH = 32 * VEC;
  constexpr int U = (sizeof(T) == 2) ? 2 : 4;  // chunks in flight per lane
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nch = (K + CH - 1) / CH;
  const int rvalid = min(ROWS, n_rows - row0);

  float acc[MT][ROWS];
  float ss[MT];
#pragma unroll
  for (int m = 0; m < MT; ++m) {
    ss[m] = 0.f;
#pragma unroll
    for (int r = 0; r < ROWS; ++r) acc[m][r] = 0.f;
  }

  for (int c0 = warp; c0 < nch; c0 += GEMV_WARPS * U) {
    uint4 wv[U][ROWS];
    bool ok[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int c = c0 + GEMV_WARPS * u;
      const int k = c * CH + lane * VEC;
      ok[u] = (c < nch) && (k < K);
#pragma unroll
      for (int r = 0; r < ROWS; ++r) {
        wv[u][r] = make_uint4(0, 0, 0, 0);
        if (ok[u] && r < rvalid) {
          // SWZ8 (bf16): 16-byte unit k/8 of row R sits at (k/8) ^ (R & 7)
          const int kk = swz ? ((((k >> 3) ^ ((row0 + r) & 7))) << 3) : k;
          wv[u][r] = ld_stream16(W + (size_t)(row0 + r) * K + kk);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (!ok[u]) continue;
      const int k = (c0 + GEMV_WARPS * u) * CH + lane * VEC;
      float g[VEC];
      if (gain != nullptr) {
#pragma unroll
        for (int j = 0; j < VEC; j += 4) {
          const float4 gv = ld_act16(gain + k + j);
          g[j] = gv.x; g[j + 1] = gv.y; g[j + 2] = gv.z; g[j + 3] = gv.w;
        }
      }
      float wf[ROWS][VEC];
#pragma unroll
      for (int r = 0; r < ROWS; ++r) VecTraits<T>::unpack(wv[u][r], wf[r]);
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        if (m >= m_valid) break;
        float xv[VEC];
#pragma unroll
        for (int j = 0; j < VEC; j += 4) {
          const float4 t = ld_act16(x + (size_t)m * ldx + k + j);
          xv[j] = t.x; xv[j + 1] = t.y; xv[j + 2] = t.z; xv[j + 3] = t.w;
        }
        if (NORM) {
#pragma unroll
          for (int j = 0; j < VEC; ++j) ss[m] = __fmaf_rn(xv[j], xv[j], ss[m]);
        }
        if (gain != nullptr) {
#pragma unroll
          for (int j = 0; j < VEC; ++j) xv[j] = __fmul_rn(xv[j], g[j]);
        }
#pragma unroll
        for (int r = 0; r < ROWS; ++r) {
#pragma unroll
          for (int j = 0; j < VEC; ++j) acc[m][r] = __fmaf_rn(wf[r][j], xv[j], acc[m][r]);
        }
      }
    }
  }

#pragma unroll
  for (int m = 0; m < MT; ++m) {
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
      const float v = warp_sum(acc[m][r]);
      if (lane == 0) sm.red[warp][m][r] = v;
    }
    if (NORM) {
      const float v = warp_sum(ss[m]);
      if (lane == 0) sm.ss[warp][m] = v;
    }
  }
  __syncthreads();
  if (threadIdx.x < MT * ROWS) {
    const int m = threadIdx.x / ROWS, r = threadIdx.x % ROWS;
    float s = sm.red[0][m][r];
#pragma unroll
    for (int w = 1; w < GEMV_WARPS; ++w) s = __fadd_rn(s, sm.red[w][m][r]);
    sm.red[0][m][r] = s;
  }
  if (NORM && threadIdx.x >= 128 && threadIdx.x < 128 + MT) {
    const int m = threadIdx.x - 128;
    float s = sm.ss[0][m];
#pragma unroll
    for (int w = 1; w < GEMV_WARPS; ++w) s = __fadd_rn(s, sm.ss[w][m]);
    sm.ss[0][m] = s;
  }
  __syncthreads();
}

__device__ __forceinline__ float rms_scale(float ss, int K, float eps) {
  return __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(__fdiv_rn(ss, (float)K), eps)));
}

}  // namespace sp
