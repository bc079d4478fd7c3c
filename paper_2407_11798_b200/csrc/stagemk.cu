// Persistent decode stage (llama, bf16, tcgen05): ONE launch runs every layer
// of a stage-run for up to 16 tokens -- q/k/v (+RMSNorm, RoPE, K/V cell
// rows), attention over the plan, out-projection + residual, gate/up +
// SwiGLU, down + residual -- with a grid barrier between phases instead of a
// kernel boundary (each boundary of the one-GEMM-per-launch chain costs the
// run ~2.5 us of dependency resolution, measured by tools/skip_cost.py).
//
// The weights of every phase are independent of the activations, so they
// stream continuously: warp 0 (one lane) walks this CTA's weight slabs of
// every phase of every layer through a shared-memory ring, gated only by
// free ring slots; warp 2 (one lane) loads the matching activation tiles
// after the phase's grid barrier; warp 1 (one lane) issues the UMMAs
// (D[128 rows, 16 tokens] += W[128, 64] . X[16, 64]^T, TMEM accumulators,
// two buffers); warps 3-6 drain the accumulators and run the epilogues and
// the attention phase.
//
// Work split: stream-K.  A GEMM of T row tiles and C 64-wide K chunks is the
// flat sequence of T*C (tile, chunk) units; CTA b of G takes the contiguous
// range [b*T*C/G, (b+1)*T*C/G) -- one contiguous slab of the tiled weight
// image, the same byte count for every CTA.  A tile cut by range borders is
// finished by its last-arriving segment, which sums the segments' partials
// in K order (deterministic) and runs the epilogue.
//
// Reference sites: model.py:387-393 (q,k,v + cache insert), 394-415
// (attention over the visibility plan), 416 (out-proj residual), 417-418
// (MLP, SwiGLU in the llama variant), 419-420 (finite check); RMSNorm
// (model.py:188-189) as a per-token scale from sum-of-squares partials;
// early cancellation between layers (engine.py:602-612).
#include <cuda.h>
#include <cstdio>

#include "gemv_core.cuh"
#include "kernels.cuh"
#include "tc_ptx.cuh"

namespace sp {

constexpr int MK_THREADS = 224;   // 7 warps
#ifndef MK_ST_DEF
#define MK_ST_DEF 10
#endif
constexpr int MK_ST = MK_ST_DEF;   // ring slots of (16 KB weights + 2 KB activations)
#ifndef MK_MRG_DEF
#define MK_MRG_DEF 8192
#endif
constexpr int MK_MRG = MK_MRG_DEF; // attention merge staging (floats): 63 splits at HD 128
constexpr int MK_MAXSEG = 16;     // stream-K segments per tile merged from registers
constexpr int MK_NT = 16;         // token columns (UMMA_N)
constexpr int MK_XTILE = MK_NT * TC_BK * 2;
constexpr int MK_STAGE = TC_WTILE + MK_XTILE;
constexpr int MK_EPI_THREADS = 128;   // warps 3..6
constexpr int MK_ATT_CH = 32;         // attention split (plan entries), as attn_kernel
constexpr int MK_PH = 5;              // phases per layer: QKV, ATTN, O, UP, DOWN

enum { PH_QKV = 0, PH_ATTN = 1, PH_O = 2, PH_UP = 3, PH_DOWN = 4 };

struct MkSmem {
  uint64_t fullw[MK_ST];
  uint64_t fullx[MK_ST];
  uint64_t empty[MK_ST];
  uint64_t accf[2];        // accumulator buffer b holds a finished segment
  uint64_t acce[2];        // accumulator buffer b drained by the epilogue
  uint32_t tmem_base;
  volatile int stop;       // the run was cancelled: every role winds down
  int consumed;            // ring index the MMA lane stopped at
  int issued;              // ring index the weight producer stopped at
  int last;                // segment/attention merge broadcast
  float inv_rms[MK_NT];
  float ssw[4][MK_NT];
  float sc[MK_ATT_CH];
  float part[1024];        // attention: [row group][HD] partial P.V
  float red[4];
  float mrg[MK_MRG];       // attention: the split partials of one (query, head)
};

__device__ __forceinline__ unsigned mk_ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void mk_arrive(unsigned* bar) {
  asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
}
__device__ __forceinline__ void mk_wait_epoch(const unsigned* bar, unsigned target) {
  unsigned spins = 0;
  while (mk_ld_acquire(bar) < target) {
    __nanosleep(32);
    if (++spins > (1u << 27)) __trap();   // a lost CTA: fail loudly, never hang
  }
}
__device__ __forceinline__ void epi_sync() {   // warps 3..6 only
  asm volatile("bar.sync 1, %0;" ::"n"(MK_EPI_THREADS) : "memory");
}
// mbarrier wait that gives up when the run is being wound down
__device__ __forceinline__ bool mbar_wait_or_stop(uint64_t* b, uint32_t parity, MkSmem* sm) {
  for (uint32_t it = 0;; ++it) {
    if (mbar_try(b, parity)) return true;
    if (sm->stop) return false;
    if (it > (1u << 24)) __trap();
  }
}

// phase geometry (GEMM phases)
struct MkGemm {
  const uint8_t* w;     // tiled weights
  int tiles, nchunk;
};
__device__ __forceinline__ MkGemm mk_gemm(const MkArgs& a, const MkLayer& L, int ph) {
  MkGemm g;
  switch (ph) {
    case PH_QKV: g.w = (const uint8_t*)L.qkv; g.tiles = (a.q_dim + 2 * a.kv_dim) / TC_BM;
                 g.nchunk = a.d / TC_BK; break;
    case PH_O:   g.w = (const uint8_t*)L.o; g.tiles = a.d / TC_BM; g.nchunk = a.q_dim / TC_BK; break;
    case PH_UP:  g.w = (const uint8_t*)L.up; g.tiles = 2 * a.ffn / TC_BM; g.nchunk = a.d / TC_BK;
                 break;
    default:     g.w = (const uint8_t*)L.down; g.tiles = a.d / TC_BM; g.nchunk = a.ffn / TC_BK;
                 break;
  }
  return g;
}
__device__ __forceinline__ long mk_start(long total, int b, int G) { return total * b / G; }
__device__ __forceinline__ int mk_owner(long f, long total, int G) {
  return (int)(((f + 1) * G - 1) / total);
}

// ---------------------------------------------------------------------------
// Epilogues (thread = weight row within the tile, acc = its NT token columns)
// ---------------------------------------------------------------------------
__device__ __forceinline__ void mk_epi_qkv(const MkArgs& a, const MkLayer& L, int R, int mv,
                                           const float* acc, const float* inv_rms) {
  const int hd = a.head_dim;
  int sec, off;
  if (R < a.q_dim) { sec = 0; off = R; }
  else if (R < a.q_dim + a.kv_dim) { sec = 1; off = R - a.q_dim; }
  else { sec = 2; off = R - a.q_dim - a.kv_dim; }
  const bool odd = (R & 1) != 0;
  int dim = off;
  float inv = 0.f;
  if (sec < 2) {                         // RoPE pair (j, j + hd/2) on rows (2j, 2j+1)
    const int head = off / hd, j = (off % hd) >> 1;
    dim = head * hd + j + (odd ? (hd >> 1) : 0);
    inv = powf(a.rope_theta, -2.0f * (float)j / (float)hd);
  }
  const int crow = *a.row0_dev;
#pragma unroll
  for (int c = 0; c < MK_NT; ++c) {
    const float y = __fmul_rn(acc[c], c < mv ? inv_rms[c] : 0.f);
    const float partner = __shfl_xor_sync(0xffffffffu, y, 1);
    if (c >= mv) continue;
    float o = y;
    if (sec < 2) {
      float sn, cs;
      sincosf((float)a.toks[c].pos * inv, &sn, &cs);
      o = odd ? (y * cs + partner * sn) : (y * cs - partner * sn);
    }
    if (sec == 0) {
      a.q[(size_t)c * a.q_dim + dim] = o;
    } else {
      __nv_bfloat16* cache = reinterpret_cast<__nv_bfloat16*>(sec == 1 ? L.kc : L.vc);
      cache[(size_t)(crow + c) * a.kv_dim + dim] = __float2bfloat16_rn(o);
    }
  }
}

__device__ __forceinline__ void mk_epi_swiglu(const MkArgs& a, int R, int mv, const float* acc,
                                              const float* inv_rms) {
  const bool odd = (R & 1) != 0;
#pragma unroll
  for (int c = 0; c < MK_NT; ++c) {
    const float y = __fmul_rn(acc[c], c < mv ? inv_rms[c] : 0.f);
    const float up = __shfl_xor_sync(0xffffffffu, y, 1);
    if (c >= mv || odd) continue;
    a.hb[(size_t)c * a.ffn + (R >> 1)] = __float2bfloat16_rn(__fmul_rn(silu(y), up));
  }
}

// x += acc; xb = bf16(x * gain_next); per-token sum of squares of the tile
__device__ __forceinline__ void mk_epi_resid(const MkArgs& a, int tile, int R, int mv,
                                             const float* acc, const float* gain_next,
                                             MkSmem* sm, int tq, int lane) {
  const float g = gain_next ? gain_next[R] : 1.0f;
  float sq[MK_NT];
#pragma unroll
  for (int c = 0; c < MK_NT; ++c) {
    sq[c] = 0.f;
    if (c < mv) {
      float* xp = a.x + (size_t)c * a.d + R;
      const float nv = __fadd_rn(*xp, acc[c]);
      *xp = nv;
      if (!isfinite(nv)) set_error(a.err, SP_DEV_NONFINITE);
      a.xb[(size_t)c * a.d + R] = __float2bfloat16_rn(__fmul_rn(nv, g));
      sq[c] = __fmul_rn(nv, nv);
    }
  }
#pragma unroll
  for (int c = 0; c < MK_NT; ++c) {
    const float s = warp_sum(sq[c]);
    if (lane == 0) sm->ssw[tq][c] = s;
  }
  epi_sync();
  const int t = threadIdx.x - 3 * 32;
  if (t < mv) {
    // warp order 0..3 = rows 0-31, 32-63, 64-95, 96-127 of the tile
    const float s = __fadd_rn(__fadd_rn(sm->ssw[0][t], sm->ssw[1][t]),
                              __fadd_rn(sm->ssw[2][t], sm->ssw[3][t]));
    a.ss[(size_t)tile * a.ss_ld + t] = s;
  }
  epi_sync();
}

// ---------------------------------------------------------------------------
// Attention phase: units (query i, head h, split s of MK_ATT_CH plan entries)
// spread over the grid; the last split of a (query, head) merges the split
// partials in split order (the arithmetic of attn_kernel).
// ---------------------------------------------------------------------------
template <int HD>
__device__ void mk_attention(const MkArgs& a, const MkLayer& L, MkSmem* sm, int b, int G,
                             int& pn, bool trace) {
  int unit_k = 0;
  auto stamp = [&](int site) {
    if (a.prof && b == 0 && threadIdx.x == 96 && pn < 2040)
      a.prof[1 + pn++] = ((long long)site << 56) | (clock64() & ((1ll << 56) - 1));
  };
  constexpr int VEC = 8;                 // bf16 x 8 per 16-byte load
  constexpr int LPR = HD / VEC;          // lanes per row
  constexpr int G8 = MK_EPI_THREADS / LPR;
  constexpr int U = 4;
  static_assert(MK_ATT_CH <= G8 * U, "one load pass per split");
  static_assert(G8 * HD <= 1024, "part[] size");
  const int tid = threadIdx.x - 3 * 32;
  const int g = tid / LPR, l = tid % LPR;
  const int kvd = a.KH * HD;
  // flat unit index over (i, h, s) with per-query split counts
  int total = 0;
  for (int i = 0; i < a.m; ++i) total += a.H * ((a.vis_len[i] + MK_ATT_CH - 1) / MK_ATT_CH);
  for (int u = b; u < total; u += G) {
    int i = 0, rem = u, ns = 0;
    for (;; ++i) {
      ns = (a.vis_len[i] + MK_ATT_CH - 1) / MK_ATT_CH;
      if (rem < a.H * ns) break;
      rem -= a.H * ns;
    }
    const int h = rem / ns, s = rem % ns;
    stamp(30);
    const int len = a.vis_len[i];
    const int kh = h / (a.H / a.KH);
    const int32_t* plan = a.vis + (size_t)i * a.ld_vis;
    const __nv_bfloat16* Kc = reinterpret_cast<const __nv_bfloat16*>(L.kc) + kh * HD + l * VEC;
    const __nv_bfloat16* Vc = reinterpret_cast<const __nv_bfloat16*>(L.vc) + kh * HD + l * VEC;
    float qv[VEC];
    {
      const float* qp = a.q + (size_t)i * a.H * HD + h * HD + l * VEC;
#pragma unroll
      for (int j = 0; j < VEC; ++j) qv[j] = qp[j] * a.scale;
    }
    const int e0 = s * MK_ATT_CH, e1 = min(len, e0 + MK_ATT_CH);
    uint4 kv[U], vv[U];
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const int e = e0 + q * G8 + g;
      const int row = e < e1 ? plan[e] : plan[e0];
      kv[q] = ld_stream16(Kc + (size_t)row * kvd);
      vv[q] = ld_stream16(Vc + (size_t)row * kvd);
    }
#pragma unroll
    for (int q = 0; q < U; ++q) {
      float kf[VEC];
      VecTraits<__nv_bfloat16>::unpack(kv[q], kf);
      float dd = 0.f;
#pragma unroll
      for (int j = 0; j < VEC; ++j) dd = __fmaf_rn(qv[j], kf[j], dd);
#pragma unroll
      for (int o = LPR / 2; o > 0; o >>= 1) dd += __shfl_xor_sync(0xffffffffu, dd, o);
      const int e = e0 + q * G8 + g;
      if (l == 0 && e < e1) sm->sc[e - e0] = dd;
    }
    epi_sync();
    stamp(31);
    const int cntv = e1 - e0;
    float mx = -INFINITY;
    for (int e = tid; e < cntv; e += MK_EPI_THREADS) mx = fmaxf(mx, sm->sc[e]);
    mx = warp_max(mx);
    if ((tid & 31) == 0) sm->red[tid >> 5] = mx;
    epi_sync();
    mx = fmaxf(fmaxf(sm->red[0], sm->red[1]), fmaxf(sm->red[2], sm->red[3]));
    epi_sync();
    float sum = 0.f;
    for (int e = tid; e < cntv; e += MK_EPI_THREADS) {
      const float p = __expf(sm->sc[e] - mx);
      sm->sc[e] = p;
      sum += p;
    }
    sum = warp_sum(sum);
    if ((tid & 31) == 0) sm->red[tid >> 5] = sum;
    epi_sync();
    sum = sm->red[0] + sm->red[1] + sm->red[2] + sm->red[3];
    float acc[VEC];
#pragma unroll
    for (int j = 0; j < VEC; ++j) acc[j] = 0.f;
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const int e = e0 + q * G8 + g;
      if (e < e1) {
        float vf[VEC];
        VecTraits<__nv_bfloat16>::unpack(vv[q], vf);
        const float p = sm->sc[e - e0];
#pragma unroll
        for (int j = 0; j < VEC; ++j) acc[j] = __fmaf_rn(p, vf[j], acc[j]);
      }
    }
#pragma unroll
    for (int j = 0; j < VEC; ++j) sm->part[g * HD + l * VEC + j] = acc[j];
    epi_sync();
    const size_t obase = (size_t)i * a.H * HD + h * HD;
    if (ns == 1) {
      for (int d = tid; d < HD; d += MK_EPI_THREADS) {
        float o = sm->part[d];
        for (int gg = 1; gg < G8; ++gg) o += sm->part[gg * HD + d];
        a.attnb[obase + d] = __float2bfloat16_rn(o / sum);
      }
      epi_sync();
      continue;
    }
    float* sp_ = a.att_scratch + (((size_t)i * a.H + h) * a.nsplit + s) * (HD + 2);
    for (int d = tid; d < HD; d += MK_EPI_THREADS) {
      float o = sm->part[d];
      for (int gg = 1; gg < G8; ++gg) o += sm->part[gg * HD + d];
      sp_[2 + d] = o;
    }
    if (tid == 0) { sp_[0] = mx; sp_[1] = sum; }
    stamp(32);
    epi_sync();
    if (tid == 0) {   // one fence per CTA: the barrier orders the other threads' stores
      __threadfence();
      const int t = atomicAdd(&a.att_tickets[(i * a.H + h) * a.att_tstride], 1);
      sm->last = (t == ns - 1);
      __threadfence();
    }
    epi_sync();
    stamp(33);
    if (trace && tid == 0 && unit_k < 4) {
      long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      a.prof[4096 + 1024 + b * 8 + 2 * unit_k] = t;
      a.prof[4096 + 1024 + b * 8 + 2 * unit_k + 1] = sm->last;
      ++unit_k;
    }
    if (sm->last) {
      // all partials of this (query, head) in one coalesced round trip, then
      // the split-order merge from shared memory
      const float* base = a.att_scratch + ((size_t)i * a.H + h) * a.nsplit * (HD + 2);
      const bool staged = ns * (HD + 2) <= MK_MRG;
      const float* src = base;
      if (staged) {
        const int tot = ns * (HD + 2);
        for (int i0 = 0; i0 < tot; i0 += 8 * MK_EPI_THREADS) {   // 8 loads in flight per thread
          float v[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int idx = i0 + k * MK_EPI_THREADS + tid;
            v[k] = idx < tot ? __ldcg(base + idx) : 0.f;
          }
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int idx = i0 + k * MK_EPI_THREADS + tid;
            if (idx < tot) sm->mrg[idx] = v[k];
          }
        }
        epi_sync();
        src = sm->mrg;
      }
      auto rd = [&](int idx) { return staged ? src[idx] : __ldcg(src + idx); };
      float M = -INFINITY;
      for (int ss = 0; ss < ns; ++ss) M = fmaxf(M, rd(ss * (HD + 2)));
      float Lsum = 0.f;
      for (int ss = 0; ss < ns; ++ss) Lsum += rd(ss * (HD + 2) + 1) * __expf(rd(ss * (HD + 2)) - M);
      for (int d = tid; d < HD; d += MK_EPI_THREADS) {
        float o = 0.f;
        for (int ss = 0; ss < ns; ++ss)
          o += rd(ss * (HD + 2) + 2 + d) * __expf(rd(ss * (HD + 2)) - M);
        a.attnb[obase + d] = __float2bfloat16_rn(o / Lsum);
      }
      if (tid == 0) a.att_tickets[(i * a.H + h) * a.att_tstride] = 0;
    }
    epi_sync();
  }
}

// ---------------------------------------------------------------------------
// The kernel
// ---------------------------------------------------------------------------
template <int HD>
__global__ void __launch_bounds__(MK_THREADS, 1)
stage_mk_kernel(const __grid_constant__ CUtensorMap mXb, const __grid_constant__ CUtensorMap mAttn,
                const __grid_constant__ CUtensorMap mHb, const MkArgs a) {
  extern __shared__ __align__(1024) uint8_t mk_smem_raw[];
  uint8_t* ring = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(mk_smem_raw) + 1023) & ~uintptr_t(1023));
  MkSmem* sm = reinterpret_cast<MkSmem*>(ring + MK_ST * MK_STAGE);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.x, G = gridDim.x;
  const int mv = a.m;

  if (threadIdx.x == 0) {
    for (int s = 0; s < MK_ST; ++s) {
      mbar_init(&sm->fullw[s], 1);
      mbar_init(&sm->fullx[s], 1);
      mbar_init(&sm->empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sm->accf[i], 1);
      mbar_init(&sm->acce[i], 1);
    }
    sm->stop = 0;
    sm->consumed = 0;
    sm->issued = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&sm->tmem_base)),
                 "r"(32));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm->tmem_base;
  // a run already known to be skipped streams nothing (a stale 0 only costs
  // a wasted prefetch; run_state never goes 1 -> 0 within a run)
  const bool pre_skip = run_skipped(a.run_state);

  if (warp == 0) {
    // ================= weight producer: never waits on activations ==========
    if (lane == 0 && !pre_skip) {
      const uint64_t pw = policy_evict_first();
      int idx = 0;
      for (int l = 0; l < a.nl && !sm->stop; ++l) {
        const MkLayer& L = a.layers[l];
        for (int ph = 0; ph < MK_PH; ++ph) {
          if (ph == PH_ATTN) continue;
          const MkGemm gm = mk_gemm(a, L, ph);
          const long total = (long)gm.tiles * gm.nchunk;
          const long f0 = mk_start(total, b, G), f1 = mk_start(total, b + 1, G);
          for (long f = f0; f < f1; ++f, ++idx) {
            const int s = idx % MK_ST;
            if (!mbar_wait_or_stop(&sm->empty[s], ((idx / MK_ST) & 1) ^ 1, sm)) goto wdone;
            mbar_expect_tx(&sm->fullw[s], TC_WTILE);
            bulk_load(ring + s * MK_STAGE, gm.w + (size_t)f * TC_WTILE, TC_WTILE, &sm->fullw[s], pw);
          }
        }
      }
    wdone:
      sm->issued = idx;
    }
  }
  // ---- programmatic dependency: activations, plan, run_state, ss
  pdl_wait();
  pdl_trigger();
  const bool skipped = run_skipped(a.run_state);   // grid-uniform after the wait
  if (skipped && threadIdx.x == 0) sm->stop = 1;

  if (warp == 2) {
    // ================= activation producer: after each phase's barrier =====
    if (lane == 0 && !skipped) {
      const uint64_t px = policy_evict_last();
      int idx = 0;
      for (int l = 0; l < a.nl; ++l) {
        const MkLayer& L = a.layers[l];
        if (l > 0) {                       // previous layer done; cancelled there?
          mk_wait_epoch(a.bar, (unsigned)G * (MK_PH * l));
          if (ld_volatile(a.run_state) != 0) { sm->stop = 1; break; }
        }
        for (int ph = 0; ph < MK_PH; ++ph) {
          if (ph == PH_ATTN) continue;
          if (ph > 0) mk_wait_epoch(a.bar, (unsigned)G * (MK_PH * l + ph));
          const MkGemm gm = mk_gemm(a, L, ph);
          const CUtensorMap* mp = ph == PH_O ? &mAttn : (ph == PH_DOWN ? &mHb : &mXb);
          const long total = (long)gm.tiles * gm.nchunk;
          const long f0 = mk_start(total, b, G), f1 = mk_start(total, b + 1, G);
          for (long f = f0; f < f1; ++f, ++idx) {
            const int s = idx % MK_ST;
            if (!mbar_wait_or_stop(&sm->empty[s], ((idx / MK_ST) & 1) ^ 1, sm)) goto xdone;
            mbar_expect_tx(&sm->fullx[s], MK_XTILE);
            tma_load_2d(ring + s * MK_STAGE + TC_WTILE, mp, &sm->fullx[s],
                        (int)(f % gm.nchunk) * TC_BK, 0, px);
          }
        }
      }
    xdone:;
    }
  } else if (warp == 1) {
    // ================= MMA issuer =================
    if (lane == 0 && !skipped) {
      constexpr uint32_t IDESC = idesc_bf16(TC_BM, MK_NT);
      int idx = 0, seg = 0;
      for (int l = 0; l < a.nl; ++l) {
        const MkLayer& L = a.layers[l];
        for (int ph = 0; ph < MK_PH; ++ph) {
          if (ph == PH_ATTN) continue;
          const MkGemm gm = mk_gemm(a, L, ph);
          const long total = (long)gm.tiles * gm.nchunk;
          const long f0 = mk_start(total, b, G), f1 = mk_start(total, b + 1, G);
          long f = f0;
          while (f < f1) {
            // one segment: the chunks of tile f / nchunk inside [f0, f1)
            const long tend = min(f1, (f / gm.nchunk + 1) * gm.nchunk);
            const int buf = seg & 1;
            if (!mbar_wait_or_stop(&sm->acce[buf], ((seg >> 1) & 1) ^ 1, sm)) goto mdone;
            tc_fence_after();
            const uint32_t td = tmem + (uint32_t)(buf * MK_NT);
            for (long c = f; c < tend; ++c, ++idx) {
              const int s = idx % MK_ST;
              const uint32_t par = (idx / MK_ST) & 1;
              if (!mbar_wait_or_stop(&sm->fullw[s], par, sm)) goto mdone;
              if (!mbar_wait_or_stop(&sm->fullx[s], par, sm)) {
                // weights of this slot landed; count it consumed for the drain
                sm->consumed = idx + 1;
                goto mdone;
              }
              tc_fence_after();
              const uint32_t sa = smem_u32(ring + s * MK_STAGE);
              const uint32_t sb = sa + TC_WTILE;
#pragma unroll
              for (int k = 0; k < TC_BK / 16; ++k)
                umma_bf16(td, umma_desc_sw128(sa + 32 * k), umma_desc_sw128(sb + 32 * k), IDESC,
                          (c > f || k > 0) ? 1u : 0u);
              umma_commit(&sm->empty[s]);
              sm->consumed = idx + 1;
            }
            umma_commit(&sm->accf[buf]);
            ++seg;
            f = tend;
          }
        }
      }
    mdone:;
    }
  } else if (warp >= 3) {
    // ================= epilogue + attention (128 threads) =================
    const int tq = warp & 3;                 // TMEM lane quarter = warp % 4
    const int row = tq * 32 + lane;          // row within the tile
    const int tid = threadIdx.x - 96;
    int seg = 0, pn = 0, nmerge = 0;
    float acc[MK_NT];
    if (!skipped) {
      for (int l = 0; l < a.nl; ++l) {
        const MkLayer& L = a.layers[l];
        if (l > 0) {
          // one poller per CTA (148 x 128 pollers on one line would queue
          // behind each other), then a named barrier
          if (tid == 0) mk_wait_epoch(a.bar, (unsigned)G * (MK_PH * l));
          epi_sync();
          if (ld_volatile(a.run_state) != 0) break;
        }
        for (int ph = 0; ph < MK_PH; ++ph) {
          if (ph > 0) {
            if (tid == 0) mk_wait_epoch(a.bar, (unsigned)G * (MK_PH * l + ph));
            epi_sync();
          }
          nmerge = 0;
          if (a.prof && b == 0 && tid == 0 && pn < 2040)   // phase start (barrier passed)
            a.prof[1 + pn++] = ((long long)(10 + ph) << 56) | (clock64() & ((1ll << 56) - 1));
          if (ph == PH_ATTN) {
            long long t0 = 0;
            if (a.prof && l == 5 && tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
            mk_attention<HD>(a, L, sm, b, G, pn, a.prof && l == 5);
            if (a.prof && l == 5 && tid == 0) {
              long long t1;
              asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
              a.prof[4096 + b] = t0;
              a.prof[4096 + 512 + b] = t1;
            }
          } else {
            const MkGemm gm = mk_gemm(a, L, ph);
            const bool norm = ph == PH_QKV || ph == PH_UP;
            if (norm) {                        // per-token RMSNorm scale
              const int parts = (l == 0 && ph == PH_QKV) ? a.ss_parts0 : a.d / TC_BM;
              for (int c = tid; c < mv; c += MK_EPI_THREADS) {
                float ssum = 0.f;
                for (int p = 0; p < parts; ++p) ssum = __fadd_rn(ssum, a.ss[(size_t)p * a.ss_ld + c]);
                sm->inv_rms[c] = rms_scale(ssum, a.d, a.eps);
              }
              epi_sync();
            }
            const long total = (long)gm.tiles * gm.nchunk;
            const long f0 = mk_start(total, b, G), f1 = mk_start(total, b + 1, G);
            long f = f0;
            while (f < f1) {
              const int tile = (int)(f / gm.nchunk);
              const long tb = (long)tile * gm.nchunk, te = tb + gm.nchunk;
              const long tend = min(f1, te);
              const int buf = seg & 1;
              mbar_wait(&sm->accf[buf], (seg >> 1) & 1);
              tc_fence_after();
              const uint32_t ta = tmem + ((uint32_t)(tq * 32) << 16) + (uint32_t)(buf * MK_NT);
              tmem_ld16(ta, acc);
              tc_fence_before();
              epi_sync();
              if (tid == 0) mbar_arrive(&sm->acce[buf]);
              ++seg;
              // segments of this tile: owners of its first and last chunk
              const int o0 = mk_owner(tb, total, G), o1 = mk_owner(te - 1, total, G);
              const int nseg = o1 - o0 + 1, j = b - o0;
              bool mine = nseg == 1;
              if (!mine) {
                float* slot = a.scratch + ((size_t)tile * a.maxseg + j) * (MK_NT * TC_BM);
#pragma unroll
                for (int c = 0; c < MK_NT; ++c)
                  if (c < mv) slot[c * TC_BM + row] = acc[c];
                epi_sync();
                if (tid == 0) {   // one fence per CTA: the barrier orders the stores
                  __threadfence();
                  const int t = atomicAdd(&a.tickets[tile * 16], 1);
                  sm->last = (t == nseg - 1);
                  __threadfence();
                }
                epi_sync();
                mine = sm->last != 0;
                if (mine) {
                  ++nmerge;
                  // K order: segments 0..nseg-1 (own partial from registers);
                  // every peer partial of a token column in flight at once
                  float sum[MK_NT];
#pragma unroll
                  for (int c = 0; c < MK_NT; ++c) {
                    sum[c] = 0.f;
                    if (c < mv) {
                      float v[MK_MAXSEG];
#pragma unroll
                      for (int jj = 0; jj < MK_MAXSEG; ++jj)
                        v[jj] = (jj < nseg && jj != j)
                                    ? __ldcg(a.scratch + ((size_t)tile * a.maxseg + jj) * (MK_NT * TC_BM) +
                                             c * TC_BM + row)
                                    : acc[c];
#pragma unroll
                      for (int jj = 0; jj < MK_MAXSEG; ++jj)
                        if (jj < nseg) sum[c] = jj == 0 ? v[jj] : __fadd_rn(sum[c], v[jj]);
                    }
                  }
#pragma unroll
                  for (int c = 0; c < MK_NT; ++c) acc[c] = sum[c];
                  if (tid == 0) a.tickets[tile * 16] = 0;
                }
              }
              if (mine) {
                const int R = tile * TC_BM + row;
                if (ph == PH_QKV) mk_epi_qkv(a, L, R, mv, acc, sm->inv_rms);
                else if (ph == PH_UP) mk_epi_swiglu(a, R, mv, acc, sm->inv_rms);
                else mk_epi_resid(a, tile, R, mv, acc, ph == PH_O ? L.mlp_norm : L.gain_next,
                                  sm, tq, lane);
              }
              f = tend;
            }
          }
          // phase done on this CTA: publish (early cancellation observed by
          // CTA 0 at the end of every layer but the last)
          epi_sync();
          if (a.prof && b == 0 && tid == 0 && pn < 2040)   // phase work done
            a.prof[1 + pn++] = ((long long)(20 + ph) << 56) | (clock64() & ((1ll << 56) - 1));
          if (a.prof && l == 5 && tid == 0 && b < 512) {   // per-CTA phase end (ns)
            long long tg;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tg));
            a.prof[10240 + ph * 512 + b] = tg;
            a.prof[12800 + ph * 512 + b] = nmerge;
          }
          if (tid == 0) {
            __threadfence();
            if (ph == PH_DOWN && b == 0 && l + 1 < a.nl && a.cancel_table) {
              const RunHdr* h = a.hdr;
              if ((h->flags & SP_FWD_SKIPPABLE) && h->kind == SP_KIND_SPEC && h->cancel_idx >= 0 &&
                  ld_volatile(a.cancel_table + h->cancel_idx) == h->run_id)
                *a.run_state = 1;
            }
            mk_arrive(a.bar);
          }
        }
      }
    }
    if (a.prof && b == 0 && tid == 0) { a.prof[0] = 16382; a.prof[16382] = pn; }
    if (tid == 0) sm->stop = 1;    // release any role still waiting
  }

  // ---- wind down: drain weight copies still in flight, free TMEM
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int idx = sm->consumed; idx < sm->issued; ++idx)
      mbar_wait(&sm->fullw[idx % MK_ST], (idx / MK_ST) & 1);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(32));
}

size_t stage_mk_smem() { return MK_ST * MK_STAGE + sizeof(MkSmem) + 1024; }

// diagnostics (SP_MK_VERBOSE): co-residency of the persistent kernel
void stage_mk_occupancy_report() {
  auto kern = stage_mk_kernel<128>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const int smems[4] = {0, 16 * 1024, 64 * 1024, 100 * 1024};
  const int thr[3] = {128, 224, 256};
  for (int t : thr)
    for (int sm : smems) {
      int n = -1;
      cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, t, sm);
      fprintf(stderr, "stage_mk occupancy: threads %d smem %d -> %d CTAs/SM (%s)\n", t, sm, n,
              cudaGetErrorString(e));
    }
  fprintf(stderr, "tc_gemm<16,QKV,norm,5> occupancy API: %d CTAs/SM\n", tc_gemm_occupancy());
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, kern);
  fprintf(stderr, "stage_mk attrs: regs %d local %zu const %zu maxThreads %d\n", fa.numRegs,
          fa.localSizeBytes, fa.constSizeBytes, fa.maxThreadsPerBlock);
}

cudaError_t launch_stage_mk(const CUtensorMap& mxb, const CUtensorMap& mattn,
                            const CUtensorMap& mhb, const MkArgs& a, int ctas, cudaStream_t st) {
  const size_t smem = stage_mk_smem();
  auto kern = a.head_dim == 128 ? stage_mk_kernel<128> : stage_mk_kernel<64>;
  static bool configured[2] = {false, false};
  const int ki = a.head_dim == 128 ? 1 : 0;
  if (!configured[ki]) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    configured[ki] = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ctas);
  cfg.blockDim = dim3(MK_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;   // co-residency for the grid barriers
  // (the occupancy API counts a TMEM kernel as one CTA per SM; SP_MK_NONCOOP=1
  // launches two per SM without the guarantee -- experiments only)
  static const bool noncoop = getenv("SP_MK_NONCOOP") != nullptr;
  attr[0].val.cooperative = noncoop ? 0 : 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, kern, mxb, mattn, mhb, a);
}

}  // namespace sp
