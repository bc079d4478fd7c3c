// K4 + K5: visibility plan and tree-masked attention over the
// sequence-partitioned cell table.
//
// Visibility rule (model.py:197-206, 287-323): query q sees cell c iff
// c.pos < q.pos and c.seqs ∩ q.seqs ≠ ∅, plus itself.  The plan lists the
// visible rows of each query in ascending position order (ties by row, which
// equals the reference's cache-rows-then-batch-rows order because a run's
// own cells are appended after every existing row), followed by the query's
// own row.  It is built once per stage-run and reused by every layer of the
// stage (the reference reuses its gather plans the same way, model.py:378-380).
#include "kernels.cuh"

namespace sp {

constexpr int PLAN_THREADS = 512;

// ---------------------------------------------------------------------------
// K4: plan.  One CTA per query; counting sort over positions in smem.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(PLAN_THREADS)
plan_kernel(const int32_t* __restrict__ cell_pos,
            const uint32_t* __restrict__ cell_mask, int n_old, int row0,
            const sp_token* __restrict__ toks, int n, int max_context,
            int32_t* __restrict__ vis, int32_t* __restrict__ vis_len,
            int ld_vis, int check_cov, int* err, const int* run_state,
            const RunHdr* hdr) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ int cnt[];  // [max_context + 1]
  // a run skipped by its gate is never checked (engine.py:581-590: the
  // coverage check follows the cancellation test)
  if (run_skipped(run_state)) return;
  if (hdr != nullptr) {          // per-run scalars from the run header
    n_old = hdr->row0;
    row0 = hdr->row0;
    check_cov = (hdr->flags & SP_FWD_CHECK_COVERAGE) != 0;
  }
  __shared__ int wsum[PLAN_THREADS / 32];
  const int i = blockIdx.x;
  const int tid = threadIdx.x;
  const int qpos = toks[i].pos;
  const uint32_t qmask = toks[i].seq_mask;
  const int P = max(0, min(qpos, max_context));
  int32_t* out = vis + (size_t)i * ld_vis;

  for (int p = tid; p <= P; p += PLAN_THREADS) cnt[p] = 0;
  __syncthreads();
  for (int r = tid; r < n_old; r += PLAN_THREADS) {
    const int p = cell_pos[r];
    if ((cell_mask[r] & qmask) && p < qpos) atomicAdd(&cnt[p], 1);
  }
  for (int j = tid; j < n; j += PLAN_THREADS) {
    const int p = toks[j].pos;
    if (j != i && (toks[j].seq_mask & qmask) && p < qpos) atomicAdd(&cnt[p], 1);
  }
  __syncthreads();

  // exclusive scan of cnt[0..P) (each thread a contiguous segment)
  const int seg = (P + PLAN_THREADS - 1) / PLAN_THREADS;
  const int s0 = min(P, tid * seg), s1 = min(P, s0 + seg);
  int local = 0;
  for (int p = s0; p < s1; ++p) local += cnt[p];
  const int lane = tid & 31, warp = tid >> 5;
  int incl = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  int wbase = 0;
  for (int w = 0; w < warp; ++w) wbase += wsum[w];
  int total = 0;
  for (int w = 0; w < PLAN_THREADS / 32; ++w) total += wsum[w];
  int run = wbase + incl - local;
  __syncthreads();
  for (int p = s0; p < s1; ++p) {
    const int c = cnt[p];
    cnt[p] = run;
    run += c;
  }
  __syncthreads();

  // place (cursor per position); ties are ordered afterwards
  for (int r = tid; r < n_old; r += PLAN_THREADS) {
    const int p = cell_pos[r];
    if ((cell_mask[r] & qmask) && p < qpos) out[atomicAdd(&cnt[p], 1)] = r;
  }
  for (int j = tid; j < n; j += PLAN_THREADS) {
    const int p = toks[j].pos;
    if (j != i && (toks[j].seq_mask & qmask) && p < qpos)
      out[atomicAdd(&cnt[p], 1)] = row0 + j;
  }
  __syncthreads();
  // after placement cnt[p] is the END of position p's segment
  for (int p = tid; p < P; p += PLAN_THREADS) {
    const int b = p == 0 ? 0 : cnt[p - 1], e = cnt[p];
    for (int a = b + 1; a < e; ++a) {  // insertion sort of a (tiny) tie run
      const int v = out[a];
      int c = a - 1;
      while (c >= b && out[c] > v) { out[c + 1] = out[c]; --c; }
      out[c + 1] = v;
    }
  }
  if (tid == 0) {
    out[total] = row0 + i;
    vis_len[i] = total + 1;
    if (check_cov && total != qpos) set_error(err, SP_DEV_COVERAGE);
  }
}

// ---------------------------------------------------------------------------
// K5: attention.  grid = (heads, queries, splits); each CTA takes up to
// ATT_CH plan entries of one (query, head) and merges split partials in a
// fixed order (last-arriving CTA), so results do not depend on scheduling.
// ---------------------------------------------------------------------------
constexpr int ATT_THREADS = 128;
#ifndef SP_ATT_CH
#define SP_ATT_CH 32
#endif
constexpr int ATT_CH = SP_ATT_CH;   // plan entries per split: one load pass, K and V together
constexpr int ATT_UNROLL = 4;



template <typename T, int HD>
__global__ void __launch_bounds__(ATT_THREADS) attn_kernel(const AttnArgs a) {
  constexpr int VEC = 16 / sizeof(T);
  constexpr int LPR = HD / VEC;           // lanes per row
  constexpr int G = ATT_THREADS / LPR;    // rows in flight per pass
  static_assert(LPR >= 1 && LPR <= 32 && (32 % LPR) == 0, "bad head dim");
  constexpr bool ONE = ATT_CH <= G * ATT_UNROLL;   // a split is one pass, K and V together
  __shared__ float sc[ATT_CH];
  extern __shared__ float mrg[];   // [nsplit][HD + 2] split partials (merging CTA)
  __shared__ float part[G][HD];
  __shared__ float red[ATT_THREADS / 32];
  __shared__ int last;

  const int h = blockIdx.x, i = blockIdx.y;
  const int kh = h / (a.H / a.KH);
  const int kvd = a.KH * HD;
  const int tid = threadIdx.x, g = tid / LPR, l = tid % LPR;
  const int32_t* plan = a.vis + (size_t)i * a.ld_vis;
  const T* Kc = reinterpret_cast<const T*>(a.k) + kh * HD + l * VEC;
  const T* Vc = reinterpret_cast<const T*>(a.v) + kh * HD + l * VEC;

  // Before the dependency wait: the plan (built at the start of the
  // stage-run) and the K/V rows of cells older than this run are final;
  // only rows >= fresh0 come from the QKV kernel this launch depends on.
  // The old rows of this CTA's first split stream in while QKV drains.
  const int fresh0 = a.fresh_row0_dev ? *a.fresh_row0_dev : a.fresh_row0;
  const int len = a.vis_len[i];
  const bool pre = ONE && fresh0 > 0 && !run_skipped(a.run_state);
  uint4 kp[ATT_UNROLL], vp[ATT_UNROLL];
  if (pre) {
    const int e0 = blockIdx.z * ATT_CH, e1 = min(len, e0 + ATT_CH);
#pragma unroll
    for (int u = 0; u < ATT_UNROLL; ++u) {
      const int e = e0 + u * G + g;
      if (e < e1) {
        const int row = plan[e];
        if (row < fresh0) {
          kp[u] = ld_stream16(Kc + (size_t)row * kvd);
          vp[u] = ld_stream16(Vc + (size_t)row * kvd);
        }
      }
    }
  }
  pdl_wait();
  pdl_trigger();
  if (a.diag_empty) return;   // diagnostics: kernel-boundary cost only

  if (run_skipped(a.run_state)) return;

  const int ns = (len + ATT_CH - 1) / ATT_CH;
  if (blockIdx.z == 0 && threadIdx.x == 0 && ns > a.nsplit) set_error(a.err, SP_DEV_PLAN_OVERFLOW);
  const size_t obase = (size_t)i * a.H * HD + h * HD;
  auto store = [&](int d, float v) {
    if (a.out_bf16) reinterpret_cast<__nv_bfloat16*>(a.out)[obase + d] = __float2bfloat16_rn(v);
    else a.out[obase + d] = v;
  };

  float qv[VEC];
  {
    const float* qp = a.q + (size_t)i * a.H * HD + h * HD + l * VEC;
#pragma unroll
    for (int j = 0; j < VEC; ++j) qv[j] = qp[j] * a.scale;
  }

  // splits s = z, z + gridDim.z, ...: the grid is sized for the machine, not
  // the context, so one launch shape (and one captured graph) serves any
  // context length; each split's partial is independent of which CTA ran it
  for (int s = blockIdx.z; s < ns; s += gridDim.z) {
    const int e0 = s * ATT_CH, e1 = min(len, e0 + ATT_CH);
    // a split fits one pass for bf16 heads: its V rows are loaded together
    // with its K rows (one round trip instead of two)
    uint4 vpre[ATT_UNROLL];
    // scores
    for (int eb = e0; eb < e1; eb += G * ATT_UNROLL) {
      uint4 kv[ATT_UNROLL];
#pragma unroll
      for (int u = 0; u < ATT_UNROLL; ++u) {
        const int e = eb + u * G + g;
        const int row = e < e1 ? plan[e] : plan[e0];
        if (ONE && pre && s == (int)blockIdx.z && e < e1 && row < fresh0) {
          kv[u] = kp[u];           // streamed before the dependency wait
          vpre[u] = vp[u];
        } else {
          kv[u] = ld_stream16(Kc + (size_t)row * kvd);
          if (ONE) vpre[u] = ld_stream16(Vc + (size_t)row * kvd);
        }
      }
#pragma unroll
      for (int u = 0; u < ATT_UNROLL; ++u) {
        float kf[VEC];
        VecTraits<T>::unpack(kv[u], kf);
        float d = 0.f;
#pragma unroll
        for (int j = 0; j < VEC; ++j) d = __fmaf_rn(qv[j], kf[j], d);
#pragma unroll
        for (int o = LPR / 2; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
        const int e = eb + u * G + g;
        if (l == 0 && e < e1) sc[e - e0] = d;
      }
    }
    __syncthreads();
    const int cntv = e1 - e0;
    float mx = -INFINITY;
    for (int e = tid; e < cntv; e += ATT_THREADS) mx = fmaxf(mx, sc[e]);
    mx = warp_max(mx);
    if ((tid & 31) == 0) red[tid >> 5] = mx;
    __syncthreads();
    mx = red[0];
#pragma unroll
    for (int w = 1; w < ATT_THREADS / 32; ++w) mx = fmaxf(mx, red[w]);
    __syncthreads();
    float sum = 0.f;
    for (int e = tid; e < cntv; e += ATT_THREADS) {
      const float p = __expf(sc[e] - mx);
      sc[e] = p;
      sum += p;
    }
    sum = warp_sum(sum);
    if ((tid & 31) == 0) red[tid >> 5] = sum;
    __syncthreads();
    sum = red[0];
#pragma unroll
    for (int w = 1; w < ATT_THREADS / 32; ++w) sum += red[w];

    // P @ V
    float acc[VEC];
#pragma unroll
    for (int j = 0; j < VEC; ++j) acc[j] = 0.f;
    for (int eb = e0; eb < e1; eb += G * ATT_UNROLL) {
      uint4 vv[ATT_UNROLL];
#pragma unroll
      for (int u = 0; u < ATT_UNROLL; ++u) {
        if (ONE) {
          vv[u] = vpre[u];
        } else {
          const int e = eb + u * G + g;
          const int row = e < e1 ? plan[e] : plan[e0];
          vv[u] = ld_stream16(Vc + (size_t)row * kvd);
        }
      }
#pragma unroll
      for (int u = 0; u < ATT_UNROLL; ++u) {
        const int e = eb + u * G + g;
        if (e < e1) {
          float vf[VEC];
          VecTraits<T>::unpack(vv[u], vf);
          const float p = sc[e - e0];
#pragma unroll
          for (int j = 0; j < VEC; ++j) acc[j] = __fmaf_rn(p, vf[j], acc[j]);
        }
      }
    }
#pragma unroll
    for (int j = 0; j < VEC; ++j) part[g][l * VEC + j] = acc[j];
    __syncthreads();

    if (ns == 1) {
      for (int d = tid; d < HD; d += ATT_THREADS) {
        float o = part[0][d];
        for (int gg = 1; gg < G; ++gg) o += part[gg][d];
        store(d, o / sum);
      }
      return;
    }
    float* sp_ = a.scratch + (((size_t)i * a.H + h) * a.nsplit + s) * (HD + 2);
    for (int d = tid; d < HD; d += ATT_THREADS) {
      float o = part[0][d];
      for (int gg = 1; gg < G; ++gg) o += part[gg][d];
      sp_[2 + d] = o;
    }
    if (tid == 0) { sp_[0] = mx; sp_[1] = sum; }
    __threadfence();
    __syncthreads();
    if (tid == 0) {
      const int t = atomicAdd(&a.tickets[i * a.H + h], 1);
      last = (t == ns - 1);
    }
    __syncthreads();
    if (!last) continue;  // (sc/part/red are rewritten only after a barrier)
    __threadfence();
    // all partials of this (query, head) in one coalesced round trip, then
    // the fixed split-order merge from shared memory
    const float* base = a.scratch + ((size_t)i * a.H + h) * a.nsplit * (HD + 2);
    const float* src = base;
    if (a.merge_smem) {   // (else the partials are read from L2 directly)
      const int tot = ns * (HD + 2);
      for (int i0 = 0; i0 < tot; i0 += 8 * ATT_THREADS) {   // 8 loads in flight per thread
        float v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int idx = i0 + k * ATT_THREADS + tid;
          v[k] = idx < tot ? __ldcg(base + idx) : 0.f;
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int idx = i0 + k * ATT_THREADS + tid;
          if (idx < tot) mrg[idx] = v[k];
        }
      }
      __syncthreads();
      src = mrg;
    }
    float M = -INFINITY;
    for (int ss = 0; ss < ns; ++ss)
      M = fmaxf(M, a.merge_smem ? src[ss * (HD + 2)] : __ldcg(src + ss * (HD + 2)));
    float L = 0.f;
    for (int ss = 0; ss < ns; ++ss) {
      const float* b = src + ss * (HD + 2);
      const float m0 = a.merge_smem ? b[0] : __ldcg(b), l0 = a.merge_smem ? b[1] : __ldcg(b + 1);
      L = __fmaf_rn(l0, __expf(m0 - M), L);
    }
    for (int d = tid; d < HD; d += ATT_THREADS) {
      float o = 0.f;
      for (int ss = 0; ss < ns; ++ss) {
        const float* b = src + ss * (HD + 2);
        const float m0 = a.merge_smem ? b[0] : __ldcg(b);
        const float ov = a.merge_smem ? b[2 + d] : __ldcg(b + 2 + d);
        o = __fmaf_rn(ov, __expf(m0 - M), o);
      }
      store(d, o / L);
    }
    if (tid == 0) a.tickets[i * a.H + h] = 0;
    return;
  }
}


// Decode/verify attention without splits: one CTA per (head, query). The
// query's plan is staged in shared memory (one coalesced round trip); each
// row group walks plan entries g, g+G, ... with K and V of the next PF rows
// in flight while the current ones are folded into a per-group online
// softmax (running max, sum, accumulator); the G group states merge in
// group order at the end.  No partials, tickets or second pass: the launch
// is one load-latency chain long.  Order is fixed per query (batch
// invariant).
template <typename T, int HD>
__global__ void __launch_bounds__(ATT_THREADS) attn_flat_kernel(const AttnArgs a) {
  pdl_wait();
  pdl_trigger();
  constexpr int VEC = 16 / sizeof(T);
  constexpr int LPR = HD / VEC;
  constexpr int G = ATT_THREADS / LPR;
  constexpr int PF = 4;
  extern __shared__ int32_t splan[];          // [len]
  __shared__ float gm[G], gl[G];
  __shared__ float gacc[G][HD];
  if (run_skipped(a.run_state)) return;
  const int h = blockIdx.x, i = blockIdx.y;
  const int len = a.vis_len[i];
  const int kh = h / (a.H / a.KH);
  const int kvd = a.KH * HD;
  const int tid = threadIdx.x, g = tid / LPR, l = tid % LPR;
  const int32_t* plan = a.vis + (size_t)i * a.ld_vis;
  for (int e = tid; e < len; e += ATT_THREADS) splan[e] = plan[e];
  float qv[VEC];
  {
    const float* qp = a.q + (size_t)i * a.H * HD + h * HD + l * VEC;
#pragma unroll
    for (int j = 0; j < VEC; ++j) qv[j] = qp[j] * a.scale;
  }
  __syncthreads();
  const T* Kc = reinterpret_cast<const T*>(a.k) + kh * HD + l * VEC;
  const T* Vc = reinterpret_cast<const T*>(a.v) + kh * HD + l * VEC;
  float m = -INFINITY, lsum = 0.f, acc[VEC];
#pragma unroll
  for (int j = 0; j < VEC; ++j) acc[j] = 0.f;
  uint4 kb[2][PF], vb[2][PF];
  auto load = [&](int buf, int e0) {
#pragma unroll
    for (int p = 0; p < PF; ++p) {
      const int e = e0 + p * G;
      const int row = e < len ? splan[e] : splan[0];
      kb[buf][p] = ld_stream16(Kc + (size_t)row * kvd);
      vb[buf][p] = ld_stream16(Vc + (size_t)row * kvd);
    }
  };
  int cur = 0;
  load(0, g);
  // the trip count is the same for every group (shuffles need whole warps)
  for (int base = 0; base < len; base += G * PF) {
    const int e0 = base + g;
    if (base + G * PF < len) load(cur ^ 1, e0 + G * PF);   // next rows in flight
#pragma unroll
    for (int p = 0; p < PF; ++p) {
      const int e = e0 + p * G;
      float kf[VEC];
      VecTraits<T>::unpack(kb[cur][p], kf);
      float d = 0.f;
#pragma unroll
      for (int j = 0; j < VEC; ++j) d = __fmaf_rn(qv[j], kf[j], d);
#pragma unroll
      for (int o = LPR / 2; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
      if (e < len) {
        float vf[VEC];
        VecTraits<T>::unpack(vb[cur][p], vf);
        if (d > m) {
          const float c = __expf(m - d);
          lsum = __fmul_rn(lsum, c);
#pragma unroll
          for (int j = 0; j < VEC; ++j) acc[j] = __fmul_rn(acc[j], c);
          m = d;
        }
        const float pr = __expf(d - m);
        lsum = __fadd_rn(lsum, pr);
#pragma unroll
        for (int j = 0; j < VEC; ++j) acc[j] = __fmaf_rn(pr, vf[j], acc[j]);
      }
    }
    cur ^= 1;
  }
  if (l == 0) { gm[g] = m; gl[g] = lsum; }
#pragma unroll
  for (int j = 0; j < VEC; ++j) gacc[g][l * VEC + j] = acc[j];
  __syncthreads();
  const size_t obase = (size_t)i * a.H * HD + h * HD;
  for (int dd = tid; dd < HD; dd += ATT_THREADS) {
    float M = -INFINITY;
    for (int q = 0; q < G; ++q) M = fmaxf(M, gm[q]);
    float L = 0.f, o = 0.f;
    for (int q = 0; q < G; ++q) {
      if (gm[q] == -INFINITY) continue;
      const float c = __expf(gm[q] - M);
      L = __fadd_rn(L, __fmul_rn(gl[q], c));
      o = __fadd_rn(o, __fmul_rn(gacc[q][dd], c));
    }
    const float v = o / L;
    if (a.out_bf16) reinterpret_cast<__nv_bfloat16*>(a.out)[obase + dd] = __float2bfloat16_rn(v);
    else a.out[obase + dd] = v;
  }
}

template <typename T, int HD>
static cudaError_t launch_attn_flat(AttnArgs a, cudaStream_t st) {
  const size_t smem = sizeof(int32_t) * (size_t)a.ld_vis;
  if (smem > 200 * 1024) return cudaErrorInvalidValue;
  static size_t configured = 0;
  if (configured < smem) {
    const cudaError_t e = cudaFuncSetAttribute(
        attn_flat_kernel<T, HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  return launch_pdl(attn_flat_kernel<T, HD>, dim3(a.H, a.n), dim3(ATT_THREADS), smem, st, a);
}

template <typename T, int HD>
static cudaError_t launch_attn_hd(dim3 grid, AttnArgs a, cudaStream_t st) {
  // the unsplit variant is kept for experiments (SP_ATTN_FLAT=1): on the 7B
  // decode it is no faster than 32-entry splits (one CTA per head keeps too
  // few bytes in flight)
  static const bool flat = getenv("SP_ATTN_FLAT") != nullptr;
  if (flat && (size_t)a.ld_vis * 4 <= 200 * 1024) return launch_attn_flat<T, HD>(a, st);
  const size_t smem = sizeof(float) * (size_t)a.nsplit * (HD + 2);
  static const int msm = getenv("SP_ATT_MERGE_SMEM_KB") ? atoi(getenv("SP_ATT_MERGE_SMEM_KB")) : 96;
  a.merge_smem = smem <= (size_t)msm * 1024 ? 1 : 0;
  // (the 48 KB default covers static + dynamic shared memory together:
  // raise the limit before the first launch that could cross it)
  static bool configured = false;
  if (a.merge_smem && !configured) {
    const cudaError_t e = cudaFuncSetAttribute(
        attn_kernel<T, HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  return launch_pdl(attn_kernel<T, HD>, grid, dim3(ATT_THREADS), a.merge_smem ? smem : 0, st, a);
}

template <typename T>
static cudaError_t attn_dispatch(const AttnArgs& a, int hd, cudaStream_t st) {
  // a few CTAs per SM in total; splits beyond gridDim.z loop in-CTA
  // (8 per SM measured best on the 7B decode: ctx 640 11.8 -> 9.4 us; the
  // split partition is by plan index, so the grid never changes the bits)
  static const int per_sm = getenv("SP_ATT_CTAS_PER_SM") ? atoi(getenv("SP_ATT_CTAS_PER_SM")) : 8;
  const int want = (per_sm * 148 + a.H * a.n - 1) / (a.H * a.n);
  const dim3 grid(a.H, a.n, max(1, min(a.nsplit, want)));
  switch (hd) {
    case 8: return launch_attn_hd<T, 8>(grid, a, st);
    case 16: return launch_attn_hd<T, 16>(grid, a, st);
    case 32: return launch_attn_hd<T, 32>(grid, a, st);
    case 64: return launch_attn_hd<T, 64>(grid, a, st);
    case 128: return launch_attn_hd<T, 128>(grid, a, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_plan(const int32_t* cell_pos, const uint32_t* cell_mask,
                        int n_old, int row0, const sp_token* toks, int n,
                        int max_context, int32_t* vis, int32_t* vis_len,
                        int ld_vis, int check_cov, int* err, cudaStream_t st,
                        const int* run_state, const RunHdr* hdr) {
  const size_t smem = (size_t)(max_context + 1) * sizeof(int);
  static int configured = 0;
  if (configured < (int)smem) {   // (48 KB default covers static + dynamic)
    cudaFuncSetAttribute(plan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    configured = (int)smem;
  }
  return launch_pdl(plan_kernel, dim3(n), dim3(PLAN_THREADS), smem, st, cell_pos, cell_mask,
                    n_old, row0, toks, n, max_context, vis, vis_len, ld_vis, check_cov, err,
                    run_state, hdr);
}

cudaError_t launch_attention(const AttnArgs& a0, int kv_dtype, int hd,
                             cudaStream_t st) {
  static const bool nopre = getenv("SP_ATT_NOPRE") != nullptr;   // experiments
  static const int diag = getenv("SP_ATT_DIAG") ? atoi(getenv("SP_ATT_DIAG")) : 0;
  AttnArgs a = a0;
  if (nopre) { a.fresh_row0_dev = nullptr; a.fresh_row0 = 0; }
  if (diag == 2) return cudaSuccess;   // diagnostics: no attention launch at all
  a.diag_empty = diag == 1;
  if (attn_tc_ok(kv_dtype, hd, a.n)) return launch_attention_tc(a, hd, st);
  if (attn_fd_ok(kv_dtype, hd, a.n, a.max_context)) return launch_attention_fd(a, hd, st);
  return kv_dtype == SP_DTYPE_BF16 ? attn_dispatch<__nv_bfloat16>(a, hd, st)
                                   : attn_dispatch<float>(a, hd, st);
}

int attn_splits(int max_len) { return (max_len + ATT_CH - 1) / ATT_CH; }

}  // namespace sp

extern "C" int sp_build_plan(const int32_t* cell_pos, const uint32_t* cell_mask,
                             int n_old, int row0, const sp_token* toks, int n,
                             int max_context, int32_t* vis, int32_t* vis_len,
                             int ld_vis, int check_coverage, int* err,
                             void* stream) {
  if (n <= 0 || !toks || !vis || !vis_len) return SP_ERR_ARG;
  return sp::launch_plan(cell_pos, cell_mask, n_old, row0, toks, n, max_context,
                         vis, vis_len, ld_vis, check_coverage, err,
                         reinterpret_cast<cudaStream_t>(stream)) == cudaSuccess
             ? SP_OK
             : SP_ERR_CUDA;
}

extern "C" int sp_attention(const float* q, const void* k_cache,
                            const void* v_cache, int kv_dtype,
                            const int32_t* vis, const int32_t* vis_len,
                            int ld_vis, int n, int n_heads, int n_kv_heads,
                            int head_dim, int max_vis, float* out,
                            float* scratch, int* tickets, const int* run_state,
                            void* stream) {
  if (n <= 0 || n_kv_heads <= 0 || n_heads % n_kv_heads) return SP_ERR_ARG;
  sp::AttnArgs a{};
  a.q = q; a.k = k_cache; a.v = v_cache; a.vis = vis; a.vis_len = vis_len;
  a.ld_vis = ld_vis; a.n = n; a.H = n_heads; a.KH = n_kv_heads;
  a.nsplit = sp::attn_splits(max_vis);
  a.scale = 1.0f / sqrtf((float)head_dim);
  a.out = out; a.scratch = scratch; a.tickets = tickets; a.run_state = run_state;
  return sp::launch_attention(a, kv_dtype, head_dim,
                              reinterpret_cast<cudaStream_t>(stream)) == cudaSuccess
             ? SP_OK
             : SP_ERR_ARG;
}
