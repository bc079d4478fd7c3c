// K2/K6/K7: weight-streaming GEMV with fused RMSNorm prologue and
// QKV(+RoPE, KV-cache write) / residual / GELU / SwiGLU epilogues.
// Reference sites: model.py:387-393 (q,k,v + cache insert), 416 (out-proj
// residual), 417-418 (MLP), 419-420 (finite check).
#include "gemv_core.cuh"

namespace sp {

template <typename T>
__device__ __forceinline__ void store_cache(void* base, size_t idx, float v) {
  from_f32(v, reinterpret_cast<T*>(base) + idx);
}

template <typename T, int MT, int ROWS, int EPI, bool NORM>
__global__ void __launch_bounds__(GEMV_THREADS)
gemv_kernel(const sp_gemv_args a) {
  pdl_wait();
  pdl_trigger();
  __shared__ GemvSmem<T, MT, ROWS, NORM> sm;
  if (a.cancel_word != nullptr && blockIdx.x == 0 && threadIdx.x == 0 &&
      ld_volatile(a.cancel_word) == a.run_id)
    atomicExch(a.run_state_w, 1);  // observed once per layer (O projection)
  if (run_skipped(a.run_state)) return;
  const int row0 = blockIdx.x * ROWS;
  const T* W = reinterpret_cast<const T*>(a.w);
  float* out = reinterpret_cast<float*>(a.out);

  for (int mt0 = 0; mt0 < a.m; mt0 += MT) {
    const int mv = min(MT, a.m - mt0);
    gemv_core<T, MT, ROWS, NORM>(W, a.n_rows, a.k, a.x + (size_t)mt0 * a.ldx,
                                 a.ldx, mv, a.gain, row0, sm, a.w_swz);
    constexpr bool PAIRED = (EPI == SP_EPI_SWIGLU) || (EPI == SP_EPI_QKV);
    constexpr int PER = PAIRED ? 2 : 1;
    const int t = threadIdx.x;
    if (t < MT * ROWS / PER) {
      const int m = t / (ROWS / PER);
      const int r = (t % (ROWS / PER)) * PER;
      const int R = row0 + r;
      const int mi = mt0 + m;
      if (m < mv && R < a.n_rows) {
        const float sc = NORM ? rms_scale(sm.ss[0][m], a.k, a.norm_eps) : 1.0f;
        const float y0 = __fmul_rn(sm.red[0][m][r], sc);
        const float y1 = PAIRED ? __fmul_rn(sm.red[0][m][r + 1], sc) : 0.f;
        if (EPI == SP_EPI_STORE) {
          out[(size_t)mi * a.ldo + R] = y0;
        } else if (EPI == SP_EPI_RESID) {
          float* o = out + (size_t)mi * a.ldo + R;
          const float nv = __fadd_rn(*o, y0);
          *o = nv;
          if (!isfinite(nv)) set_error(a.err, SP_DEV_NONFINITE);
        } else if (EPI == SP_EPI_GELU) {
          out[(size_t)mi * a.ldo + R] = gelu_tanh(y0);
        } else if (EPI == SP_EPI_SWIGLU) {
          out[(size_t)mi * a.ldo + (R >> 1)] = __fmul_rn(silu(y0), y1);
        } else if (EPI == SP_EPI_QKV) {
          // rows: [q | k | v]; within q and k each head is pair-interleaved
          // when RoPE is on: row 2j <-> dim j, row 2j+1 <-> dim j + hd/2.
          const int hd = a.head_dim;
          int sec, off;
          if (R < a.q_rows) { sec = 0; off = R; }
          else if (R < a.q_rows + a.kv_rows) { sec = 1; off = R - a.q_rows; }
          else { sec = 2; off = R - a.q_rows - a.kv_rows; }
          int d0 = off, d1 = off + 1;
          float o0 = y0, o1 = y1;
          if (a.rope && sec < 2) {
            const int head = off / hd, j = (off % hd) >> 1;
            d0 = head * hd + j;
            d1 = d0 + (hd >> 1);
            const float inv = powf(a.rope_theta, -2.0f * (float)j / (float)hd);
            float sn, cs;
            sincosf((float)a.toks[mi].pos * inv, &sn, &cs);
            o0 = y0 * cs - y1 * sn;
            o1 = y1 * cs + y0 * sn;
          }
          if (sec == 0) {
            out[(size_t)mi * a.ldo + d0] = o0;
            out[(size_t)mi * a.ldo + d1] = o1;
          } else {
            void* cache = (sec == 1) ? a.k_cache : a.v_cache;
            const int crow = a.cache_row0_dev ? *a.cache_row0_dev : a.cache_row0;
            const size_t base = (size_t)(crow + mi) * a.kv_rows;
            store_cache<T>(cache, base + d0, o0);
            store_cache<T>(cache, base + d1, o1);
          }
        }
      }
    }
    __syncthreads();
  }
}

template <typename T, int MT, int ROWS, int EPI>
static cudaError_t launch_norm(const sp_gemv_args& a, cudaStream_t st) {
  const dim3 grid((a.n_rows + ROWS - 1) / ROWS);
  if (a.norm)
    return launch_pdl(gemv_kernel<T, MT, ROWS, EPI, true>, grid, dim3(GEMV_THREADS), 0, st, a);
  return launch_pdl(gemv_kernel<T, MT, ROWS, EPI, false>, grid, dim3(GEMV_THREADS), 0, st, a);
}

template <typename T, int EPI>
static cudaError_t launch_m(const sp_gemv_args& a, cudaStream_t st) {
  // MT = token tile; ROWS = rows per CTA.  ROWS is irrelevant to the
  // per-(token,row) reduction order, so it can be tuned per MT freely.
  if (a.m <= 1) return launch_norm<T, 1, 4, EPI>(a, st);
  if (a.m <= 2) return launch_norm<T, 2, 4, EPI>(a, st);
  if (a.m <= 4) return launch_norm<T, 4, 4, EPI>(a, st);
  return launch_norm<T, 8, 4, EPI>(a, st);
}

template <typename T>
static cudaError_t launch_epi(const sp_gemv_args& a, cudaStream_t st) {
  switch (a.epi) {
    case SP_EPI_STORE: return launch_m<T, SP_EPI_STORE>(a, st);
    case SP_EPI_RESID: return launch_m<T, SP_EPI_RESID>(a, st);
    case SP_EPI_QKV: return launch_m<T, SP_EPI_QKV>(a, st);
    case SP_EPI_GELU: return launch_m<T, SP_EPI_GELU>(a, st);
    case SP_EPI_SWIGLU: return launch_m<T, SP_EPI_SWIGLU>(a, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace sp

extern "C" int sp_gemv(const sp_gemv_args* a, void* stream) {
  if (!a || !a->w || !a->x || !a->out || a->m <= 0 || a->n_rows <= 0 || a->k <= 0)
    return SP_ERR_ARG;
  const int vec = a->w_dtype == SP_DTYPE_BF16 ? 8 : 4;
  if (a->k % vec || a->ldx % 4) return SP_ERR_ARG;
  if ((a->epi == SP_EPI_SWIGLU || a->epi == SP_EPI_QKV) && (a->n_rows & 1))
    return SP_ERR_ARG;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e = a->w_dtype == SP_DTYPE_BF16
                      ? sp::launch_epi<__nv_bfloat16>(*a, st)
                      : sp::launch_epi<float>(*a, st);
  return e == cudaSuccess ? SP_OK : SP_ERR_CUDA;
}
