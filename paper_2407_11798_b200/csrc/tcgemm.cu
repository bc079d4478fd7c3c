// Skinny tensor-core GEMM for the bf16 (llama) decoder path: tcgen05.mma
// with TMEM accumulators, TMA-fed 4-stage mbarrier pipeline, split-K across
// CTAs and fused epilogues.  Replaces the CUDA-core GEMV for every llama run
// (single-token, speculative verification and prefill alike), so a token's
// result does not depend on how many tokens share the launch.
//
//   D[128 rows, NT tokens] += W[128 rows, 64 k] . X[NT tokens, 64 k]^T
//
// swap-AB: the weight tile is the A operand (UMMA_M = 128, K-major, SW128),
// the activation tile the B operand (UMMA_N = NT, K-major, SW128).  The
// CTA's K range is split into 64-element chunks; warp 0 lane 0 streams
// W and X chunks with cp.async.bulk.tensor into a ring of stages, warp 1
// lane 0 issues 4 UMMA_K=16 MMAs per chunk and commits each stage back to
// its "empty" barrier.  With ksplit > 1 each CTA parks its fp32 partial in
// global scratch and the last-arriving CTA of a row tile sums the splits in
// ascending order (deterministic) and runs the epilogue.
//
// Reference sites of the fused epilogues: model.py:387-393 (q,k,v + cache
// insert), 416 (out-proj residual), 417-418 (MLP, SwiGLU in the llama
// variant), 419-420 (finite check); RMSNorm (model.py:188-189) is applied
// as a per-token scale from the producer's sum-of-squares partials.
#include <cuda.h>

#include "gemv_core.cuh"
#include "kernels.cuh"
#include "tc_ptx.cuh"

namespace sp {

constexpr int TC_THREADS = 128;
// 128-token tiles run their epilogue on 8 warps: two per TMEM lane quarter,
// each over half the token columns (the per-element arithmetic is unchanged)
__host__ __device__ constexpr int tc_threads(int nt) { return nt > 16 ? 256 : TC_THREADS; }
constexpr int TC_STAGES = 4;

// greedy-head order: (a before b) iff a.v > b.v or (a.v == b.v and a.i < b.i)
__device__ __forceinline__ bool tc_better(float va, int ia, float vb, int ib) {
  return va > vb || (va == vb && ia < ib);
}
struct TcTop2 { float v1; int i1; float v2; int i2; };
__device__ __forceinline__ void tc_push(TcTop2& t, float v, int i) {
  if (tc_better(v, i, t.v1, t.i1)) { t.v2 = t.v1; t.i2 = t.i1; t.v1 = v; t.i1 = i; }
  else if (tc_better(v, i, t.v2, t.i2)) { t.v2 = v; t.i2 = i; }
}
__device__ __forceinline__ void tc_top2_butterfly(TcTop2& t, float& mx, int& nan) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float v1 = __shfl_xor_sync(0xffffffffu, t.v1, o);
    const int i1 = __shfl_xor_sync(0xffffffffu, t.i1, o);
    const float v2 = __shfl_xor_sync(0xffffffffu, t.v2, o);
    const int i2 = __shfl_xor_sync(0xffffffffu, t.i2, o);
    tc_push(t, v1, i1);
    tc_push(t, v2, i2);
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    nan |= __shfl_xor_sync(0xffffffffu, nan, o);
  }
}

template <int ST>
struct TcSmemTailT {
  uint64_t full[ST];
  uint64_t empty[ST];
  uint64_t done;
  uint64_t red;             // push merge: the peers' partials have landed
  uint32_t tmem_base;
  int npre;                 // weight stages prefetched before the dependency wait
  int last;
  float inv_rms[128];
  float ssw[4][128];
};

// ---- the kernel -------------------------------------------------------------
// ST = ring depth: 5 stages (2 CTAs/SM) for wide grids, 6 when the grid
// fits one CTA per SM.  Deeper rings were measured slower in the layer chain
// (7B stage-run: deep 10 -> 6 stages 2.71 -> 2.67 ms, 12 stages 2.74;
// shallow 4 -> 5 stages 2.67 -> 2.63 ms, 3 stages 2.93): a smaller footprint
// lets the next GEMM's CTAs become resident -- and prefetch their weights
// before the dependency wait -- while this one drains
template <int NT, int EPI, bool NORM, int ST>
__global__ void __launch_bounds__(tc_threads(NT))
tc_gemm_kernel(const __grid_constant__ CUtensorMap tmX, const TcArgs a, const int push) {
  constexpr int XTILE = NT * TC_BK * 2;
  constexpr int STAGE = TC_WTILE + XTILE;
  constexpr uint32_t TMEM_COLS = NT < 32 ? 32 : NT;
  extern __shared__ __align__(1024) uint8_t tc_smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(tc_smem_raw) + 1023) & ~uintptr_t(1023));
  TcSmemTailT<ST>* tail = reinterpret_cast<TcSmemTailT<ST>*>(smem + ST * STAGE);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int NC = NT > 16 ? NT / 2 : NT;          // token columns per thread
  const int q4 = warp & 3;                            // TMEM lane quarter (weight rows)
  const int cb = NT > 16 ? (warp >> 2) * NC : 0;      // this thread's first column
  const int tile = blockIdx.x, split = blockIdx.y, nsplit = gridDim.y;
  const int nchunk = a.k / TC_BK;
  const int c0 = (int)((long)nchunk * split / nsplit);
  const int c1 = (int)((long)nchunk * (split + 1) / nsplit);
  const int nloc = c1 - c0;
  const int npre = nloc < ST ? nloc : ST;
  // this CTA's weight tiles [tile][c0..c1) are one contiguous run
  const __nv_bfloat16* wtiles =
      reinterpret_cast<const __nv_bfloat16*>(a.w) + (size_t)tile * nchunk * (TC_WTILE / 2);

  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) {
      mbar_init(&tail->full[s], 1);
      mbar_init(&tail->empty[s], 1);
    }
    mbar_init(&tail->done, 1);
    mbar_init(&tail->red, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmX)) : "memory");
    // Weights do not depend on the previous kernel: start streaming the
    // first stages before the programmatic dependency is resolved -- unless
    // the run is already known to be skipped (a cancelled speculative run
    // would otherwise still pull 64 KB per CTA of every GEMM of every layer).
    // run_state only goes 0 -> 1 within a run and the run's gate kernel has
    // completed before any of its GEMMs start, so a stale read can only be
    // a 0 (a wasted prefetch), never a wrong skip.
    const bool pre = !run_skipped(a.run_state);
    tail->npre = pre ? npre : 0;
    if (pre) {
      const uint64_t pw = policy_evict_first();
      for (int i = 0; i < npre; ++i) {
        mbar_expect_tx_only(&tail->full[i], TC_WTILE);
        bulk_load(smem + i * STAGE, wtiles + (size_t)(c0 + i) * (TC_WTILE / 2), TC_WTILE,
                  &tail->full[i], pw);
      }
    }
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tail->tmem_base)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tail->tmem_base;
  // push merge: publish the initialised reduction barrier to the cluster
  // now, wait for the peers' arrivals only when the partials are ready
  if (push == 1) cluster_arrive();

  // ---- programmatic dependency: everything below may read the previous
  // kernel's outputs (activations, run_state, norm statistics)
  pdl_wait();
  pdl_trigger();
  const int npre_done = tail->npre;
  if (run_skipped(a.run_state)) {        // consistent for the whole grid (no one waits)
    if (EPI == SP_EPI_LMHEAD && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {
      if (a.lm_gate) *a.lm_gate = 0;     // (lmhead_kernel's skipped-run contract)
      if (a.lm_err_out) *a.lm_err_out = a.err ? *a.err : 0;
      if (a.lm_status_out) *a.lm_status_out = SP_STATUS_PLACEHOLDER;
    }
    if (threadIdx.x == 0) {              // drain the weight prefetch
      for (int i = 0; i < npre_done; ++i) {
        mbar_arrive(&tail->full[i]);
        mbar_wait(&tail->full[i], 0);
      }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                   "r"(TMEM_COLS));
    return;
  }

  // epilogue operands that do not depend on this GEMM, loaded while it
  // streams: per-token RMSNorm scales, the residual rows, the next gain
  const int row = q4 * 32 + lane;            // row within the tile
  const int R = tile * TC_BM + row;          // global weight row
  const int mv = min(NT, a.m - a.tok0);
  // the CTA that runs the epilogue (ticket merge: whichever split arrives
  // last, so every split loads the epilogue operands)
  const bool head = push != 1 || split == 0;
  if (NORM && head && threadIdx.x >= 64) {   // warps 2-3: not the producer / MMA lanes
    for (int c = threadIdx.x - 64; c < mv; c += tc_threads(NT) - 64) {
      float ssum = 0.f;
      for (int p = 0; p < a.ss_nparts; ++p)
        ssum = __fadd_rn(ssum, a.ss_in[(size_t)p * a.ss_ld + a.tok0 + c]);
      tail->inv_rms[c] = rms_scale(ssum, a.k, a.norm_eps);
    }
  }
  constexpr bool XEARLY = EPI == SP_EPI_RESID && NT <= 16;   // (registers)
  float xold[XEARLY ? NT : 1];
  float gnext = 1.0f;
  if (EPI == SP_EPI_RESID && head) {
    if (XEARLY) {
      const float* x = reinterpret_cast<const float*>(a.out);
#pragma unroll
      for (int c = 0; c < (XEARLY ? NT : 0); ++c)
        if (c < mv) xold[c] = x[(size_t)(a.tok0 + c) * a.ldo + R];
    }
    if (a.gain_next) gnext = a.gain_next[R];
  }

  constexpr bool QEARLY = EPI == SP_EPI_QKV && NT <= 16;    // token positions, cache row
  int pe[QEARLY ? NT : 1];
  int crow_e = 0;
  if (QEARLY && head) {
#pragma unroll
    for (int c = 0; c < (QEARLY ? NT : 0); ++c)
      if (c < mv) pe[c] = a.toks[a.tok0 + c].pos;
    crow_e = a.cache_row0_dev ? *a.cache_row0_dev : a.cache_row0;
  }

  if (warp == 0 && lane == 0) {
    // ---- TMA producer ----
    const uint64_t pw = policy_evict_first(), px = policy_evict_last();
    for (int i = 0; i < nloc; ++i) {
      const int s = i % ST;
      const uint32_t ph = (i / ST) & 1;
      uint8_t* st = smem + s * STAGE;
      if (i < npre_done) {               // weights already in flight
        mbar_expect_tx(&tail->full[s], XTILE);
      } else {
        mbar_wait(&tail->empty[s], ph ^ 1);
        mbar_expect_tx(&tail->full[s], STAGE);
        bulk_load(st, wtiles + (size_t)(c0 + i) * (TC_WTILE / 2), TC_WTILE, &tail->full[s], pw);
      }
      tma_load_2d(st + TC_WTILE, &tmX, &tail->full[s], (c0 + i) * TC_BK, a.tok0, px);
    }
  } else if (warp == 1 && lane == 0) {
    // ---- MMA issuer ----
    constexpr uint32_t IDESC = idesc_bf16(TC_BM, NT);
    for (int i = 0; i < nloc; ++i) {
      const int s = i % ST;
      const uint32_t ph = (i / ST) & 1;
      mbar_wait(&tail->full[s], ph);
      tc_fence_after();
      const uint32_t sa = smem_u32(smem + s * STAGE);
      const uint32_t sb = sa + TC_WTILE;
#pragma unroll
      for (int k = 0; k < TC_BK / 16; ++k)
        umma_bf16(tmem, umma_desc_sw128(sa + 32 * k), umma_desc_sw128(sb + 32 * k), IDESC,
                  (i > 0 || k > 0) ? 1u : 0u);
      umma_commit(&tail->empty[s]);
    }
    umma_commit(&tail->done);
  }

  // ---- epilogue: TMEM -> registers (thread = weight row, NT token columns)
  mbar_wait(&tail->done, 0);
  tc_fence_after();
  float acc[NC];
  if (nloc > 0) {
#pragma unroll
    for (int c = 0; c < NC; c += 16)
      tmem_ld16(tmem + ((uint32_t)(q4 * 32) << 16) + cb + c, acc + c);
  } else {
#pragma unroll
    for (int c = 0; c < NC; ++c) acc[c] = 0.f;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(TMEM_COLS));

  if (push == 2) {
    // split-K merge through L2 (no cluster): each split parks its partial in
    // global scratch; the last to take the tile's ticket sums them in split
    // order from split 0 -- the same fp32 add sequence as the cluster merges,
    // so the bits do not depend on the merge path.  Used when a co-resident
    // draft cluster holds SMs of one GPC: clusters of split CTAs would no
    // longer all fit in one wave (measured: O / down 2x slower).
    if (nsplit > 1) {
      float* part = a.scratch + ((size_t)tile * nsplit + split) * (NT * TC_BM);
#pragma unroll
      for (int c = 0; c < NC; ++c)
        if (cb + c < mv) part[(cb + c) * TC_BM + row] = acc[c];
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0) tail->last = atomicAdd(a.tickets + tile, 1) == nsplit - 1;
      __syncthreads();
      if (!tail->last) return;
      __threadfence();
      const float* p0 = a.scratch + (size_t)tile * nsplit * (NT * TC_BM);
#pragma unroll
      for (int c = 0; c < NC; ++c)
        if (cb + c < mv) acc[c] = __ldcg(p0 + (cb + c) * TC_BM + row);
      for (int sp2 = 1; sp2 < nsplit; ++sp2) {
#pragma unroll
        for (int c = 0; c < NC; ++c)
          if (cb + c < mv)
            acc[c] = __fadd_rn(acc[c], __ldcg(p0 + ((size_t)sp2 * NT + cb + c) * TC_BM + row));
      }
      if (threadIdx.x == 0) a.tickets[tile] = 0;   // the next launch reuses it
    }
  } else if (push) {
    // split-K merge by push: the split CTAs of this row tile form one
    // cluster; each peer stores its partial rows straight into rank 0's
    // reduction buffer (st.async, completing on rank 0's barrier) and
    // leaves; rank 0 sums them in split order and runs the epilogue
    float* red = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(tail) +
                                          sizeof(TcSmemTailT<ST>));   // [nsplit-1][mv][128]
    cluster_wait();                      // rank 0's barrier is initialised
    if (split != 0) {
      const uint32_t rbar = map_rank(&tail->red, 0);
      const uint32_t rbase = map_rank(red, 0);
#pragma unroll
      for (int c = 0; c < NC; ++c)
        if (cb + c < mv)
          st_async_f32(rbase + (uint32_t)((((split - 1) * mv + cb + c) * TC_BM + row) * 4), acc[c],
                       rbar);
      return;
    }
    if (threadIdx.x == 0)
      mbar_expect_tx(&tail->red, (uint32_t)((nsplit - 1) * mv * TC_BM * 4));
    mbar_wait(&tail->red, 0);
    for (int sp2 = 1; sp2 < nsplit; ++sp2) {
#pragma unroll
      for (int c = 0; c < NC; ++c)
        if (cb + c < mv) acc[c] = __fadd_rn(acc[c], red[((sp2 - 1) * mv + cb + c) * TC_BM + row]);
    }
  } else if (nsplit > 1) {
    // split-K merge through distributed shared memory: the nsplit CTAs of
    // this row tile form one cluster (grid y = cluster y); each parks its
    // partial in its own (now idle) stage buffers, rank 0 sums them in split
    // order straight from the peers' shared memory and runs the epilogue
    float* part = reinterpret_cast<float*>(smem);          // [NT][TC_BM]
#pragma unroll
    for (int c = 0; c < NC; ++c) part[(cb + c) * TC_BM + row] = acc[c];
    asm volatile("barrier.cluster.arrive.release.aligned;\n\t"
                 "barrier.cluster.wait.acquire.aligned;" ::: "memory");
    uint32_t crank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
    if (crank == 0) {
      const uint32_t la = smem_u32(part);
      for (int sp2 = 1; sp2 < nsplit; ++sp2) {
        uint32_t ra;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(sp2));
        float v[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c)
          asm volatile("ld.shared::cluster.f32 %0, [%1];"
                       : "=f"(v[c]) : "r"(ra + (uint32_t)(((cb + c) * TC_BM + row) * 4)));
#pragma unroll
        for (int c = 0; c < NC; ++c) acc[c] = __fadd_rn(acc[c], v[c]);
      }
    }
    // peers keep their shared memory alive until rank 0 has read it
    asm volatile("barrier.cluster.arrive.release.aligned;\n\t"
                 "barrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (crank != 0) return;
  }

  // (per-token RMSNorm scales: computed before the main loop; the
  // __syncthreads after the accumulator load published them)

  if (EPI == SP_EPI_QKV) {
    const int hd = a.head_dim;
    int sec, off;
    if (R < a.q_rows) { sec = 0; off = R; }
    else if (R < a.q_rows + a.kv_rows) { sec = 1; off = R - a.q_rows; }
    else { sec = 2; off = R - a.q_rows - a.kv_rows; }
    const bool odd = (R & 1) != 0;
    int dim = off;
    float inv = 0.f;
    if (sec < 2) {                         // RoPE pair (j, j + hd/2) on rows (2j, 2j+1)
      const int head = off / hd, j = (off % hd) >> 1;
      dim = head * hd + j + (odd ? (hd >> 1) : 0);
      inv = powf(a.rope_theta, -2.0f * (float)j / (float)hd);
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int cc = cb + c;
      float y = acc[c];
      if (NORM) y = __fmul_rn(y, cc < mv ? tail->inv_rms[cc] : 0.f);
      const float partner = __shfl_xor_sync(0xffffffffu, y, 1);
      if (cc >= mv) continue;
      const int t = a.tok0 + cc;
      float o = y;
      if (sec < 2) {
        float sn, cs;
        sincosf((float)(QEARLY ? pe[QEARLY ? c : 0] : a.toks[t].pos) * inv, &sn, &cs);
        o = odd ? (y * cs + partner * sn) : (y * cs - partner * sn);
      }
      if (sec == 0) {
        reinterpret_cast<float*>(a.out)[(size_t)t * a.ldo + dim] = o;
      } else {
        __nv_bfloat16* cache = reinterpret_cast<__nv_bfloat16*>(sec == 1 ? a.k_cache : a.v_cache);
        const int crow = QEARLY ? crow_e : (a.cache_row0_dev ? *a.cache_row0_dev : a.cache_row0);
        cache[(size_t)(crow + t) * a.kv_rows + dim] = __float2bfloat16_rn(o);
      }
    }
  } else if (EPI == SP_EPI_SWIGLU) {
    const bool odd = (R & 1) != 0;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int cc = cb + c;
      float y = acc[c];
      if (NORM) y = __fmul_rn(y, cc < mv ? tail->inv_rms[cc] : 0.f);
      const float up = __shfl_xor_sync(0xffffffffu, y, 1);
      if (cc >= mv || odd) continue;
      const int t = a.tok0 + cc;
      reinterpret_cast<__nv_bfloat16*>(a.out)[(size_t)t * a.ldo + (R >> 1)] =
          __float2bfloat16_rn(__fmul_rn(silu(y), up));
    }
  } else if (EPI == SP_EPI_RESID) {
    float* x = reinterpret_cast<float*>(a.out);
    const float g = gnext;
    float sq[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      sq[c] = 0.f;
      if (cb + c < mv) {
        const int t = a.tok0 + cb + c;
        float* xp = x + (size_t)t * a.ldo + R;
        const float nv = __fadd_rn(XEARLY ? xold[XEARLY ? c : 0] : *xp, acc[c]);
        *xp = nv;
        if (!isfinite(nv)) set_error(a.err, SP_DEV_NONFINITE);
        if (a.xb_next)
          reinterpret_cast<__nv_bfloat16*>(a.xb_next)[(size_t)t * a.ldo + R] =
              __float2bfloat16_rn(__fmul_rn(nv, g));
        sq[c] = __fmul_rn(nv, nv);
      }
    }
    // per-token sum of squares of this tile's 128 rows (fixed order)
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const float s = warp_sum(sq[c]);
      if (lane == 0) tail->ssw[q4][cb + c] = s;
    }
    __syncthreads();
    if (threadIdx.x < mv) {
      const int c = threadIdx.x;
      const float s = __fadd_rn(__fadd_rn(tail->ssw[0][c], tail->ssw[1][c]),
                                __fadd_rn(tail->ssw[2][c], tail->ssw[3][c]));
      a.ss_out[(size_t)tile * a.ss_ld + a.tok0 + c] = s;
    }
  } else if (EPI == SP_EPI_LMHEAD) {
    // greedy head (model.py:424-457): per token the tile's top-2 (value
    // desc, id asc), max and sum of exp over its 128 vocabulary rows, then
    // the last tile CTA merges the tiles in tile order (fixed: the record
    // does not depend on scheduling or on how many tokens share the launch)
    float* tv = reinterpret_cast<float*>(smem);           // [NT][128]; stages are idle
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int cc = cb + c;
      if (cc >= mv) break;
      float y = acc[c];
      if (NORM) y = __fmul_rn(y, tail->inv_rms[cc]);
      tv[cc * TC_BM + row] = y;
      if (a.out) reinterpret_cast<float*>(a.out)[(size_t)(a.tok0 + cc) * a.ldo + R] = y;
    }
    __syncthreads();
    const int ntiles = gridDim.x;
    LmPartial* part = reinterpret_cast<LmPartial*>(a.lm_part);
    for (int c = warp; c < mv; c += tc_threads(NT) / 32) {
      float v[4];
      TcTop2 t{-INFINITY, 0x7fffffff, -INFINITY, 0x7fffffff};
      float mx = -INFINITY;
      int nan = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        v[i] = tv[c * TC_BM + lane + 32 * i];
        if (isnan(v[i])) nan = 1;
        else { tc_push(t, v[i], tile * TC_BM + lane + 32 * i); mx = fmaxf(mx, v[i]); }
      }
      tc_top2_butterfly(t, mx, nan);
      float se = 0.f;
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (!isnan(v[i]) && mx != -INFINITY) se = __fadd_rn(se, __expf(v[i] - mx));
      se = warp_sum(se);
      if (lane == 0)
        part[(size_t)(a.tok0 + c) * ntiles + tile] = LmPartial{t.v1, t.i1, t.v2, t.i2, mx, se, nan, 0};
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) tail->last = atomicAdd(a.lm_ticket, 1) == ntiles - 1;
    __syncthreads();
    if (!tail->last) return;
    __threadfence();
    for (int c = warp; c < mv; c += tc_threads(NT) / 32) {   // one warp per token
      const LmPartial* P = part + (size_t)(a.tok0 + c) * ntiles;
      TcTop2 t{-INFINITY, 0x7fffffff, -INFINITY, 0x7fffffff};
      float mx = -INFINITY;
      int nan = 0;
      for (int q = lane; q < ntiles; q += 32) {
        const float4 lo = __ldcg(reinterpret_cast<const float4*>(P + q));
        const float4 hi = __ldcg(reinterpret_cast<const float4*>(P + q) + 1);
        tc_push(t, lo.x, __float_as_int(lo.y));
        tc_push(t, lo.z, __float_as_int(lo.w));
        mx = fmaxf(mx, hi.x);
        nan |= __float_as_int(hi.z);
      }
      tc_top2_butterfly(t, mx, nan);
      float se = 0.f;
      for (int q = lane; q < ntiles; q += 32) {
        const float2 ms = __ldcg(reinterpret_cast<const float2*>(P + q) + 2);
        if (ms.x != -INFINITY) se = __fadd_rn(se, __fmul_rn(ms.y, __expf(ms.x - mx)));
      }
      se = warp_sum(se);
      if (lane == 0) {
        sp_row_result r;
        r.argmax = t.i1;
        r.second = t.i2;
        r.conf = 1.0f / se;        // exp(max - max) / sum
        r.max_logit = t.v1;
        a.lm_out[a.tok0 + c] = r;
        if (nan) set_error(a.err, SP_DEV_NAN_LOGITS);
        if (a.lm_tip && a.tok0 + c == a.m - 1) {
          a.lm_tip[0] = r.argmax;
          a.lm_tip[1] = __float_as_int(r.conf);
          a.lm_tip[2] = 1;
          if (a.lm_gate && a.lm_chain_gate) {
            const int g = *a.lm_gate;
            const float cut = a.lm_hdr ? reinterpret_cast<const RunHdr*>(a.lm_hdr)->cutoff
                                       : a.lm_cutoff;
            *a.lm_gate = (g != 0 && r.conf >= cut) ? 1 : 0;
          }
        }
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      *a.lm_ticket = 0;
      if (a.lm_err_out) *a.lm_err_out = a.err ? *a.err : 0;
      if (a.lm_status_out) *a.lm_status_out = SP_STATUS_VALID;
    }
  } else {  // SP_EPI_STORE
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int cc = cb + c;
      if (cc >= mv) break;
      float y = acc[c];
      if (NORM) y = __fmul_rn(y, tail->inv_rms[cc]);
      reinterpret_cast<float*>(a.out)[(size_t)(a.tok0 + cc) * a.ldo + R] = y;
    }
  }
}

// ---- host side --------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// 2D bf16 map over a row-major [rows, cols] matrix (cols contiguous) with a
// {64, box_rows} box and 128B swizzle.
bool make_map_bf16(CUtensorMap* map, const void* base, long rows, long cols, long ld_elems,
                   int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld_elems * 2};
  cuuint32_t box[2] = {(cuuint32_t)TC_BK, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
            box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

template <int NT, int EPI, bool NORM, int ST>
static cudaError_t launch_nt(const CUtensorMap& x, const TcArgs& a, int ksplit,
                             cudaStream_t st) {
  constexpr int STAGE = TC_WTILE + NT * TC_BK * 2;
  const int base = ST * STAGE + (int)sizeof(TcSmemTailT<ST>) + 1024;
  // decode tiles merge split-K by push into a reduction buffer behind the
  // tail ([ksplit-1][<=16 tokens][128 rows] f32) when it fits; prefill
  // tiles (and oversize splits) pull from the peers after the main loop
  const int mvl = a.m - a.tok0 < NT ? a.m - a.tok0 : NT;   // token columns of this tile
  const int red = NT == 16 && ksplit > 1 ? (ksplit - 1) * mvl * TC_BM * 4 : 0;
  static const bool nopush = getenv("SP_TC_PULL") != nullptr;   // experiments
  // opt-in (SP_TC_TICKET_MERGE=1, with a sharing budget): merge decode
  // splits through L2 instead of a cluster (see the kernel).  Measured on
  // the 7B stage: no slowdown beside a running draft cluster (3.18 vs 3.45
  // ms) but +0.35-0.55 ms per run without one, so the cluster merge stays
  // the default and the head keeps the draft off the GPU's SMs instead
  static const bool tk_merge = getenv("SP_TC_TICKET_MERGE") != nullptr;
  const bool ticket = NT == 16 && ksplit > 1 && a.max_ctas > 0 && a.max_ctas < 296 &&
                      tk_merge && a.scratch && a.tickets &&
                      (size_t)(a.n_rows / TC_BM) * ksplit * NT * TC_BM <= (size_t)TC_SCRATCH_FLOATS &&
                      a.n_rows / TC_BM <= TC_TICKETS;
  const int push = ticket ? 2 : red > 0 && !nopush && base + red <= 227 * 1024 ? 1 : 0;
  const int smem = base + (push == 1 ? red : 0);
  static int configured = 0;
  if (configured < smem) {
    cudaFuncSetAttribute(tc_gemm_kernel<NT, EPI, NORM, ST>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    configured = smem;
  }
  dim3 grid(a.n_rows / TC_BM, ksplit);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(tc_threads(NT));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  attr[1].id = cudaLaunchAttributeClusterDimension;   // the split-K CTAs of a tile
  attr[1].val.clusterDim.x = 1;
  attr[1].val.clusterDim.y = push == 2 ? 1 : ksplit;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, tc_gemm_kernel<NT, EPI, NORM, ST>, x, a, push);
}

template <int NT, int ST>
static cudaError_t launch_epi(const CUtensorMap& x, const TcArgs& a, int ksplit,
                              cudaStream_t st) {
  switch (a.epi) {
    case SP_EPI_QKV:
      return a.norm ? launch_nt<NT, SP_EPI_QKV, true, ST>(x, a, ksplit, st)
                    : launch_nt<NT, SP_EPI_QKV, false, ST>(x, a, ksplit, st);
    case SP_EPI_SWIGLU:
      return a.norm ? launch_nt<NT, SP_EPI_SWIGLU, true, ST>(x, a, ksplit, st)
                    : launch_nt<NT, SP_EPI_SWIGLU, false, ST>(x, a, ksplit, st);
    case SP_EPI_RESID:
      return launch_nt<NT, SP_EPI_RESID, false, ST>(x, a, ksplit, st);
    case SP_EPI_LMHEAD:
      return a.norm ? launch_nt<NT, SP_EPI_LMHEAD, true, ST>(x, a, ksplit, st)
                    : launch_nt<NT, SP_EPI_LMHEAD, false, ST>(x, a, ksplit, st);
    case SP_EPI_STORE:
      return a.norm ? launch_nt<NT, SP_EPI_STORE, true, ST>(x, a, ksplit, st)
                    : launch_nt<NT, SP_EPI_STORE, false, ST>(x, a, ksplit, st);
  }
  return cudaErrorInvalidValue;
}

int tc_nt_for(int m) { return m <= 16 ? 16 : 128; }

// diagnostics: the occupancy API's view of a decode GEMM instance
int tc_gemm_occupancy() {
  auto kern = tc_gemm_kernel<16, SP_EPI_QKV, true, 5>;
  constexpr int STAGE = TC_WTILE + 16 * TC_BK * 2;
  const int smem = 5 * STAGE + (int)sizeof(TcSmemTailT<5>) + 1024;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int n = -1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, TC_THREADS, smem);
  return n;
}

// Split-K factor: as many CTAs as fit in ONE wave (a second partial wave
// doubles the tail) but at least 16 chunks (256 KB of weights) per CTA so
// the fixed prologue/merge cost is amortised (measured on the 7B shapes:
// QKV 3, O 4, gate/up 1, down 9).
int tc_ksplit(int n_rows, int k, int target_ctas) {
  const int tiles = n_rows / TC_BM, nchunk = k / TC_BK;
  // the split CTAs of a tile merge as one cluster: at most 8 (portable size),
  // a power of two (odd clusters schedule badly: measured QKV 18.5 us at 2,
  // 26.5 at 3; O 11.0 at 4; down 18.7 at 8 on the 7B shapes)
  static const int min_chunks =
      getenv("SP_TC_MIN_CHUNKS") ? max(1, atoi(getenv("SP_TC_MIN_CHUNKS"))) : 16;   // experiments
  int ks = max(1, min(min(target_ctas / tiles, nchunk / min_chunks), 8));
  while (ks & (ks - 1)) ks &= ks - 1;
  return ks;
}

// ring depths (see tc_gemm_kernel); SP_TC_DEEP_ST=4..8|10 and
// SP_TC_SHALLOW_ST=3..5 select others for experiments
static int deep_st() {
  static const int v = getenv("SP_TC_DEEP_ST") ? atoi(getenv("SP_TC_DEEP_ST")) : 6;
  return v;
}
static int shallow_st() {
  static const int v = getenv("SP_TC_SHALLOW_ST") ? atoi(getenv("SP_TC_SHALLOW_ST")) : 5;
  return v;
}

// Launch over all tokens (token tiles of NT); maps[0] is the NT=16 X map,
// maps[1] the NT=128 one.
cudaError_t launch_tc_gemm(const CUtensorMap* xmaps, TcArgs a, cudaStream_t st) {
  const int nt = tc_nt_for(a.m);
  const int budget = a.max_ctas > 0 ? a.max_ctas : 296;   // at 2 CTAs per SM
  const int sms = budget / 2;                              // at 1 CTA per SM
  const int tiles = a.n_rows / TC_BM, nchunk = a.k / TC_BK;
  int ksplit;
  bool deep = false;
  // The split is a function of the GEMM shape only -- the same for the
  // 16-token and the 128-token tiles -- so a token's K-sum order (and bits)
  // does not depend on how many tokens share its run.
  // deep when the tile count leaves room to split at least 2-way within one
  // CTA per SM (measured on the 7B shapes: O 10.9 -> 10.4 us, down 18.7 ->
  // 17.4; QKV (96 tiles) stays faster at 2 shallow CTAs per SM)
  if (getenv("SP_TC_SHALLOW") == nullptr &&
      (a.ksplit > 0 ? tiles * a.ksplit <= sms : 2 * tiles <= sms)) {
    // one CTA per SM with a deep ring: split so the grid still fits one wave
    ksplit = a.ksplit > 0 ? a.ksplit
                          : max(1, min(min(sms / tiles, nchunk / 16), 8));
    static const int ks_cap = getenv("SP_TC_DEEP_KS_MAX") ? atoi(getenv("SP_TC_DEEP_KS_MAX")) : 8;
    if (a.ksplit <= 0 && ksplit > ks_cap) ksplit = ks_cap;
    while (ksplit & (ksplit - 1)) ksplit &= ksplit - 1;
    deep = nt == 16;
  } else {
    ksplit = a.ksplit > 0 ? a.ksplit : tc_ksplit(a.n_rows, a.k, budget);
  }
  if (ksplit > 8) ksplit = 8;
  for (int t0 = 0; t0 < a.m; t0 += nt) {
    a.tok0 = t0;
    cudaError_t e;
    if (nt == 16)
      e = !deep ? (shallow_st() == 3   ? launch_epi<16, 3>(xmaps[0], a, ksplit, st)
                   : shallow_st() == 5 ? launch_epi<16, 5>(xmaps[0], a, ksplit, st)
                                       : launch_epi<16, 4>(xmaps[0], a, ksplit, st))
          : deep_st() == 7 ? launch_epi<16, 7>(xmaps[0], a, ksplit, st)
          : deep_st() == 8 ? launch_epi<16, 8>(xmaps[0], a, ksplit, st)
          : deep_st() == 6 ? launch_epi<16, 6>(xmaps[0], a, ksplit, st)
          : deep_st() == 5 ? launch_epi<16, 5>(xmaps[0], a, ksplit, st)
          : deep_st() == 4 ? launch_epi<16, 4>(xmaps[0], a, ksplit, st)
                           : launch_epi<16, 10>(xmaps[0], a, ksplit, st);
    else
      e = launch_epi<128, 4>(xmaps[1], a, ksplit, st);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace sp
