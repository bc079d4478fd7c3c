// K15 (cluster form): the draft request on ONE thread-block cluster.
//
// The grid form (draft.cu) spreads a draft forward over every SM and pays a
// grid barrier (~1.3 us) at each of the ~60 phase edges of a forward; it also
// takes the whole GPU away from the target stage it shares the device with.
// Here one cluster of CL CTAs (16 SMs, one CTA per SM) runs the request:
//
//  * a producer warp per CTA streams that CTA's fixed weight slices (QKV, O,
//    gate/up, down of every layer, then its LM-head rows) through a ring of
//    shared-memory stages with 1D bulk copies, running ahead across phase
//    edges (weights never depend on activations);
//  * eight consumer warps compute from the ring; results every CTA needs
//    (q/k/v for the attention CTAs, the attention output, x rows, h) are
//    pushed straight into the other CTAs' shared memory (DSMEM stores);
//  * a phase edge is an all-to-all mbarrier arrive (release.cluster) +
//    local acquire wait: ~0.3 us, and the ring keeps streaming through it.
//
// Same algorithm and per-row reduction orders as the grid form; every CTA
// keeps a full replica of x and normalises it itself (identical values in
// every CTA, so no broadcast of the statistic is needed).
#include "gemv_core.cuh"
#include "kernels.cuh"

namespace sp {

constexpr int K2_CW = 8;                    // consumer warps
constexpr int K2_CT = K2_CW * 32;           // consumer threads
constexpr int K2_THREADS = K2_CT + 32;      // + producer warp

// ---- PTX helpers -----------------------------------------------------------
__device__ __forceinline__ uint32_t k2_s(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t k2_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t k2_mapa(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void k2_st(uint32_t cl_addr, float v) {
  asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(cl_addr), "f"(v) : "memory");
}
__device__ __forceinline__ void k2_mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(k2_s(b)), "r"(count));
}
__device__ __forceinline__ void k2_arrive_local(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(k2_s(b)) : "memory");
}
__device__ __forceinline__ void k2_arrive_remote(uint32_t cl_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cl_addr)
               : "memory");
}
__device__ __forceinline__ void k2_wait(uint64_t* b, uint32_t parity) {
  for (uint32_t it = 0;; ++it) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}"
        : "=r"(ok) : "r"(k2_s(b)), "r"(parity) : "memory");
    if (ok) return;
    if (it > (1u << 24)) __trap();   // a protocol bug: fail loudly, never hang
  }
}
__device__ __forceinline__ void k2_wait_cluster(uint64_t* b, uint32_t parity) {
  for (uint32_t it = 0;; ++it) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}"
        : "=r"(ok) : "r"(k2_s(b)), "r"(parity) : "memory");
    if (ok) return;
    if (it > (1u << 24)) __trap();
  }
}
__device__ __forceinline__ void k2_cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\t"
               "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void k2_cons_sync() {   // consumer warps only
  asm volatile("bar.sync 1, %0;" ::"r"(K2_CT) : "memory");
}

__device__ __forceinline__ void k2_slice(int R, int rank, int cl, int& u0, int& u1) {
  u0 = (int)(((long long)R * rank) / cl);
  u1 = (int)(((long long)R * (rank + 1)) / cl);
}

// Weight segments of one forward, in stream order: per layer A (QKV row
// pairs), C (O rows), D (gate/up row pairs), E (down rows); then H (LM head
// rows).  Producer and consumers walk the same chunking.
struct K2Seg {
  const __nv_bfloat16* base;  // first row of this CTA's slice
  int rows;                   // rows in the slice
  int rb;                     // bytes per row
  int rs;                     // bytes per row in the ring (= rb: the SWZ8 layout
                              // keeps 8-row ldmatrix / LDS accesses conflict-free)
  int rc;                     // rows per chunk
  int row0g;                  // matrix row of the slice's first row (SWZ8 key)
};

__device__ __forceinline__ K2Seg k2_seg(const DraftArgs& a, const DraftLayer* lw, int l, int ph,
                                        int rank, int cl) {
  const int d = a.d, f = a.f, qd = a.H * a.hd, kvd = a.KH * a.hd;
  K2Seg s;
  int u0, u1;
  int pg = 1;
  if (ph == 0) {
    k2_slice((qd + 2 * kvd) / 2, rank, cl, u0, u1);
    s.base = lw[l].qkv + (size_t)2 * u0 * d; s.rows = 2 * (u1 - u0); s.rb = d * 2; pg = 2;
    s.row0g = 2 * u0;
  } else if (ph == 1) {
    k2_slice(d, rank, cl, u0, u1);
    s.base = lw[l].o + (size_t)u0 * qd; s.rows = u1 - u0; s.rb = qd * 2; s.row0g = u0;
  } else if (ph == 2) {
    k2_slice(f, rank, cl, u0, u1);
    s.base = lw[l].up + (size_t)2 * u0 * d; s.rows = 2 * (u1 - u0); s.rb = d * 2; pg = 2;
    s.row0g = 2 * u0;
  } else if (ph == 3) {
    k2_slice(d, rank, cl, u0, u1);
    s.base = lw[l].down + (size_t)u0 * f; s.rows = u1 - u0; s.rb = f * 2; s.row0g = u0;
  } else {
    k2_slice(a.V, rank, cl, u0, u1);
    s.base = a.w_out + (size_t)u0 * d; s.rows = u1 - u0; s.rb = d * 2; s.row0g = u0;
  }
  s.rs = s.rb;
  int rc = a.ring_bytes / s.rs;
  rc = rc / pg * pg;
  s.rc = rc < pg ? pg : rc;
  return s;
}

// y[r][m] = W_row_r . xs[m] for R rows resident in shared memory
template <int NT, int R>
__device__ __forceinline__ void k2_dot(const __nv_bfloat16* const (&w)[R], const float* xs,
                                       int ldx, int K, int n, float (&y)[R][NT]) {
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
      const uint4 u = w[r] ? *reinterpret_cast<const uint4*>(w[r] + (size_t)c * 8)
                           : make_uint4(0, 0, 0, 0);
      bf16x8_to_f32(u, wf[r]);
    }
#pragma unroll
    for (int m = 0; m < NT; ++m) {
      if (m >= n) break;
      const float4 x0 = *reinterpret_cast<const float4*>(xs + (size_t)m * ldx + c * 8);
      const float4 x1 = *reinterpret_cast<const float4*>(xs + (size_t)m * ldx + c * 8 + 4);
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

// R rows (R in {2,4,8}) of length K from shared memory (row stride K) against
// n <= DR_NT activation rows xs (stride ldx): lane l accumulates its K-slice
// (8-element chunks l, l+32, ...) for all R rows, then a transposed
// butterfly leaves row k2_row<R>(l)'s sum on the lanes whose low 5-log2(R)
// bits are zero (fixed order: deterministic).
template <int R>
__device__ __forceinline__ int k2_row(int lane) {
  int r = 0;
#pragma unroll
  for (int s = 0, h = R >> 1; h >= 1; ++s, h >>= 1)
    if (lane & (16 >> s)) r += h;
  return r;
}
template <int R, int NT>
__device__ __forceinline__ void k2_rows(const __nv_bfloat16* W, int ldw, int nr, int K,
                                        const float* xs, int ldx, int n, float (&res)[NT],
                                        int row0g) {
  const int lane = threadIdx.x & 31;
  const int nch = K >> 3;
  float acc[NT][R];
#pragma unroll
  for (int m = 0; m < NT; ++m)
#pragma unroll
    for (int r = 0; r < R; ++r) acc[m][r] = 0.f;
#pragma unroll 1
  for (int c = lane; c < nch; c += 32) {
    float xv[NT][8];
#pragma unroll
    for (int m = 0; m < NT; ++m) {
      if (NT > 1 && m >= n) break;
      const float4 x0 = *reinterpret_cast<const float4*>(xs + (size_t)m * ldx + c * 8);
      const float4 x1 = *reinterpret_cast<const float4*>(xs + (size_t)m * ldx + c * 8 + 4);
      xv[m][0] = x0.x; xv[m][1] = x0.y; xv[m][2] = x0.z; xv[m][3] = x0.w;
      xv[m][4] = x1.x; xv[m][5] = x1.y; xv[m][6] = x1.z; xv[m][7] = x1.w;
    }
    uint4 wv[R];
#pragma unroll
    for (int r = 0; r < R; ++r)
      wv[r] = r < nr ? *reinterpret_cast<const uint4*>(
                           W + (size_t)r * ldw + (size_t)(c ^ ((row0g + r) & 7)) * 8)   // SWZ8
                     : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      float wf[8];
      bf16x8_to_f32(wv[r], wf);
#pragma unroll
      for (int m = 0; m < NT; ++m) {
        if (NT > 1 && m >= n) break;
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[m][r] = __fmaf_rn(wf[j], xv[m][j], acc[m][r]);
      }
    }
  }
#pragma unroll
  for (int m = 0; m < NT; ++m) {
    if (NT == 1 || m < n) {
#pragma unroll
      for (int s = 0, h = R >> 1; h >= 1; ++s, h >>= 1) {
        const bool hi = lane & (16 >> s);
#pragma unroll
        for (int i = 0; i < h; ++i) {
          const float send = hi ? acc[m][i] : acc[m][i + h];
          const float keep = hi ? acc[m][i + h] : acc[m][i];
          acc[m][i] = __fadd_rn(keep, __shfl_xor_sync(0xffffffffu, send, 16 >> s));
        }
      }
      float v = acc[m][0];
#pragma unroll
      for (int sh = 16 / R; sh >= 1; sh >>= 1) v = __fadd_rn(v, __shfl_xor_sync(0xffffffffu, v, sh));
      res[m] = v;
    } else {
      res[m] = 0.f;
    }
  }
}

// 16 weight rows (ring, padded stride ldw) x one token on the tensor cores:
// mma.m16n8k16 with A = W rows (ldmatrix.x4), B = the token's activations
// split into bf16 hi + lo parts (two MMAs, fp32 accumulate: ~2^-16 relative
// to the fp32 product), column 0 of C = token 0.  Lanes with (lane & 3) == 0
// return row lane/4 in r0 and row lane/4 + 8 in r1.  Hardware accumulation
// order is fixed: deterministic.
__device__ __forceinline__ void k2_mma_rows16(const __nv_bfloat16* W, int ldw, int nr, int K,
                                              const __nv_bfloat16* xh, const __nv_bfloat16* xl,
                                              float& r0, float& r1, int row0g) {
  const int lane = threadIdx.x & 31;
  const int t = lane & 3;
  const bool col0 = lane < 4;   // only B column 0 (token 0) is non-zero
  const int arow = min(lane & 15, nr - 1);
  const uint32_t rbase = k2_s(W + (size_t)arow * ldw);
  const int rx = (row0g + arow) & 7;   // SWZ8: unit u of this row sits at u ^ rx
  const int uh = lane >> 4;            // this lane's 8-column half of the k-step
  float ch[4] = {0.f, 0.f, 0.f, 0.f}, cl[4] = {0.f, 0.f, 0.f, 0.f};
  // batches of KB k-steps: every shared-memory load of a batch is issued
  // before its MMAs (asm volatile keeps source order, so the batching is
  // what lets the loads overlap)
  constexpr int KB = 4;
  for (int kb = 0; kb < K; kb += 16 * KB) {
    uint32_t af[KB][4], bf[KB][4];
#pragma unroll
    for (int i = 0; i < KB; ++i) {
      const int k0 = kb + 16 * i;
      if (k0 < K) {
        const uint32_t pos = (uint32_t)(((k0 >> 3) + uh) ^ rx);
        asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                     : "=r"(af[i][0]), "=r"(af[i][1]), "=r"(af[i][2]), "=r"(af[i][3])
                     : "r"(rbase + pos * 16));
      }
      bf[i][0] = bf[i][1] = bf[i][2] = bf[i][3] = 0u;
      if (col0 && k0 < K) {
        bf[i][0] = *reinterpret_cast<const uint32_t*>(xh + k0 + 2 * t);
        bf[i][1] = *reinterpret_cast<const uint32_t*>(xh + k0 + 8 + 2 * t);
        bf[i][2] = *reinterpret_cast<const uint32_t*>(xl + k0 + 2 * t);
        bf[i][3] = *reinterpret_cast<const uint32_t*>(xl + k0 + 8 + 2 * t);
      }
    }
#pragma unroll
    for (int i = 0; i < KB; ++i) {
      if (kb + 16 * i >= K) break;
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
          "{%8,%9}, {%0,%1,%2,%3};"
          : "+f"(ch[0]), "+f"(ch[1]), "+f"(ch[2]), "+f"(ch[3])
          : "r"(af[i][0]), "r"(af[i][1]), "r"(af[i][2]), "r"(af[i][3]), "r"(bf[i][0]),
            "r"(bf[i][1]));
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
          "{%8,%9}, {%0,%1,%2,%3};"
          : "+f"(cl[0]), "+f"(cl[1]), "+f"(cl[2]), "+f"(cl[3])
          : "r"(af[i][0]), "r"(af[i][1]), "r"(af[i][2]), "r"(af[i][3]), "r"(bf[i][2]),
            "r"(bf[i][3]));
    }
  }
  r0 = __fadd_rn(ch[0], cl[0]);
  r1 = __fadd_rn(ch[2], cl[2]);
}

struct K2Top2 { float v1; int i1; float v2; int i2; };
__device__ __forceinline__ bool k2_better(float va, int ia, float vb, int ib) {
  return va > vb || (va == vb && ia < ib);
}
__device__ __forceinline__ void k2_push(K2Top2& t, float v, int i) {
  if (k2_better(v, i, t.v1, t.i1)) { t.v2 = t.v1; t.i2 = t.i1; t.v1 = v; t.i1 = i; }
  else if (k2_better(v, i, t.v2, t.i2)) { t.v2 = v; t.i2 = i; }
}
__device__ __forceinline__ void k2_online(float& mx, float& se, float v) {
  if (v > mx) { se = __fadd_rn(__fmul_rn(se, __expf(mx - v)), 1.0f); mx = v; }
  else se = __fadd_rn(se, __expf(v - mx));
}
__device__ __forceinline__ void k2_merge(float& mx, float& se, float m2, float s2) {
  if (m2 == -INFINITY) return;
  if (mx == -INFINITY) { mx = m2; se = s2; return; }
  const float M = fmaxf(mx, m2);
  se = __fadd_rn(__fmul_rn(se, __expf(mx - M)), __fmul_rn(s2, __expf(m2 - M)));
  mx = M;
}

template <int HD, int CL, int NT>
__global__ void __launch_bounds__(K2_THREADS, 1) draft_cluster_kernel(const DraftArgs a) {
  extern __shared__ __align__(128) uint8_t dsm[];
  const int d = a.d, f = a.f, qd = a.H * HD, kvd = a.KH * HD;
  const int HPC = (a.H + CL - 1) / CL;     // heads per CTA
  // dynamic smem layout (host computes the same sizes in draft2_smem_bytes)
  uint8_t* ring = dsm;
  float* xrep = reinterpret_cast<float*>(dsm + (size_t)a.ring_stages * a.ring_bytes);  // [NT][d]
  const int NTR = a.nt;                    // token rows of the activation buffers
  float* xn = xrep + NTR * d;              // [NTR][d]   normed input of A / D / H
  float* abuf = xn + NTR * d;              // [NTR][qd]  attention output (all heads)
  float* hbuf = abuf + NTR * qd;           // [NTR][f]   SwiGLU output (all rows)
  float* qkvb = hbuf + NTR * f;            // [HPC][NTR][3][HD] this CTA's heads' q, k, v
  float* lmp = qkvb + HPC * NTR * 3 * HD;  // [CL][8] LM-head partials of every CTA
  const int KX = d > qd ? d : qd;
  __nv_bfloat16* xh = reinterpret_cast<__nv_bfloat16*>(lmp + CL * 8);   // [KX] token-0 hi
  __nv_bfloat16* xl = xh + KX;                                          // [KX] token-0 lo

  __shared__ __align__(8) uint64_t full[16], empty[16];
  __shared__ int sdone[16];
  __shared__ volatile int srel[16];   // rounds of each stage released by the consumers
  __shared__ __align__(8) uint64_t pbar[2];   // phase edges alternate barriers
  __shared__ DraftLayer lw[DR_MAX_LAYERS];
  __shared__ float inv_s[HD / 2];
  __shared__ float gpart[K2_CW][HD + 2];  // attention: per-warp (m, l, acc[HD])
  __shared__ float wred[K2_CW][8];
  __shared__ volatile int go_fwd;
  __shared__ volatile int stop;
  __shared__ int s_tok, s_gate;

  const DraftHdr& Hd = *a.hdr;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int rank = (int)k2_rank();
  const int n_feed = Hd.n_feed, steps = Hd.steps, pos0 = Hd.pos0, row0 = Hd.row0;
  const int chain = Hd.chain;
  const float cutoff = Hd.cutoff;
  const float att_scale = 1.0f / sqrtf((float)HD);

  for (int l = tid; l < a.L; l += K2_THREADS) lw[l] = a.layers[l];
  for (int j = tid; j < HD / 2; j += K2_THREADS)
    inv_s[j] = powf(a.theta, -2.0f * (float)j / (float)HD);
  if (tid == 0) {
    for (int s = 0; s < a.ring_stages; ++s) {
      k2_mbar_init(&full[s], 1);
      k2_mbar_init(&empty[s], 1);
      sdone[s] = 0;
      srel[s] = 0;
    }
    k2_mbar_init(&pbar[0], CL);
    k2_mbar_init(&pbar[1], CL);
    go_fwd = (n_feed > 0) ? 0 : -1;
    stop = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  k2_cluster_sync_all();   // every CTA's barriers exist before any remote arrive

  // ======================= producer warp ===================================
  if (warp == K2_CW) {
    if (lane == 0) {
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      long it = 0;   // chunks issued (ring position)
      for (int fw = 0;; ++fw) {
        // wait for the consumers to confirm forward fw (or to stop)
        while (go_fwd < fw && !stop) __nanosleep(64);
        if (go_fwd < fw) break;
        for (int l = 0; l <= a.L; ++l) {
          for (int ph = 0; ph < (l < a.L ? 4 : 1); ++ph) {
            const K2Seg sg = k2_seg(a, lw, l < a.L ? l : 0, l < a.L ? ph : 4, rank, CL);
            {   // the next segment heads for L2 while this one streams into the ring
              const int nl = ph + 1 < 4 ? l : l + 1, nph = ph + 1 < 4 ? ph + 1 : 0;
              if (l < a.L) {
                const K2Seg nx = k2_seg(a, lw, nl < a.L ? nl : 0, nl < a.L ? nph : 4, rank, CL);
                const char* c = reinterpret_cast<const char*>(nx.base);
                size_t bytes = (size_t)nx.rows * nx.rb;
                while (bytes >= 16) {
                  const unsigned nb = (unsigned)(bytes > (1u << 20) ? (1u << 20) : (bytes & ~size_t(15)));
                  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(c), "r"(nb) : "memory");
                  c += nb;
                  bytes -= nb;
                }
              }
            }
            for (int r0 = 0; r0 < sg.rows; r0 += sg.rc) {
              const int nr = min(sg.rc, sg.rows - r0);
              const int st = (int)(it % a.ring_stages);
              const long round = it / a.ring_stages;
              if (round > 0) k2_wait(&empty[st], (uint32_t)((round - 1) & 1));
              const uint32_t bytes = (uint32_t)nr * sg.rb;
              asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                               k2_s(&full[st])), "r"(bytes) : "memory");
              asm volatile(
                  "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes"
                  ".L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
                      k2_s(ring + (size_t)st * a.ring_bytes)),
                  "l"(reinterpret_cast<const char*>(sg.base) + (size_t)r0 * sg.rb), "r"(bytes),
                  "r"(k2_s(&full[st])), "l"(pol) : "memory");
              ++it;
            }
          }
        }
      }
    }
    __syncwarp();
    k2_cluster_sync_all();   // matches the consumers' final cluster barrier
    return;
  }

  // ======================= consumer warps ==================================
  int nprof = 0;
  long long wait_cyc = 0;   // time the CTA-0 thread 0 spent waiting for ring chunks
  auto mark = [&](long long site) {
    if (a.prof && rank == 0 && tid == 0 && nprof < 4094) {
      a.prof[1 + nprof++] = (site << 56) | (clock64() & ((1ll << 56) - 1));
    }
  };
  long ct = 0;              // chunks consumed (ring position)
  uint32_t pedge = 0;       // phase edges passed
  // Run one weight phase: sub-slices of R rows (8 for short rows, fewer for
  // long ones) go to warps round-robin, so up to eight sub-slices (several
  // ring stages) are in flight; a stage is released when all its parts are
  // done.  epi(row_in_slice, res) runs on the lanes that hold a row's sums.
  auto run_phase = [&](const K2Seg& sg, int K, const float* xs, int ldx, int n, auto&& epi) {
    const int ldw = sg.rs / 2;
    if (NT == 1 && sg.rc >= 16 && a.use_mma) {
      // tensor-core path (opt-in, SP_DRAFT_MMA=1): one whole 16-row chunk per warp
      const int nchunks = (sg.rows + sg.rc - 1) / sg.rc;
      for (int c = warp; c < nchunks; c += K2_CW) {
        const long g = ct + c;
        const int st = (int)(g % a.ring_stages);
        const long long t0 = clock64();
        const int rnd = (int)(g / a.ring_stages);
        for (uint32_t it = 0; srel[st] < rnd; ++it) {
          __nanosleep(32);
          if (it > (1u << 26)) __trap();
        }
        k2_wait(&full[st], (uint32_t)(rnd & 1));
        wait_cyc += clock64() - t0;
        const int crow = c * sg.rc;
        const int rows_c = min(sg.rc, sg.rows - crow);
        const __nv_bfloat16* W = reinterpret_cast<const __nv_bfloat16*>(
            ring + (size_t)st * a.ring_bytes);
        for (int h0 = 0; h0 < rows_c; h0 += 16) {
          const int cnt = min(16, rows_c - h0);
          float r0, r1;
          k2_mma_rows16(W + (size_t)h0 * ldw, ldw, cnt, K, xh, xl, r0, r1, sg.row0g + crow + h0);
          const bool lead = (lane & 3) == 0;
          const int gr = lane >> 2;
          float res0[NT], res1[NT];
          res0[0] = r0;
          res1[0] = r1;
          epi(crow + h0 + gr, lead && gr < cnt, res0, 8);
          epi(crow + h0 + 8 + gr, lead && 8 + gr < cnt, res1, 8);
        }
        __syncwarp();
        if (lane == 0) {
          srel[st] = srel[st] + 1;
          k2_arrive_local(&empty[st]);
        }
      }
      ct += nchunks;
      return;
    }
    const int R = sg.rc >= 8 ? 8 : (sg.rc >= 4 ? 4 : 2);
    const int parts = (sg.rc + R - 1) / R;
    const int nchunks = (sg.rows + sg.rc - 1) / sg.rc;
    const int nsub = nchunks * parts;
    for (int j = warp; j < nsub; j += K2_CW) {
      const int c = j / parts, pt = j - c * parts;
      const long g = ct + c;
      const int st = (int)(g % a.ring_stages);
      const long long t0 = clock64();
      // a warp may run ahead of the others by several chunks; waiting on a
      // stage whose previous round is still in use would alias the barrier
      // phase (parity ABA), so first wait until that round is released
      const int rnd = (int)(g / a.ring_stages);
      for (uint32_t it = 0; srel[st] < rnd; ++it) {
        __nanosleep(32);
        if (it > (1u << 26)) __trap();
      }
      k2_wait(&full[st], (uint32_t)(rnd & 1));
      wait_cyc += clock64() - t0;
      const int crow = c * sg.rc;                                  // chunk's first row
      const int rows_c = min(sg.rc, sg.rows - crow);
      const int r_lo = pt * R;
      const int cnt = min(R, rows_c - r_lo);
      const __nv_bfloat16* W = reinterpret_cast<const __nv_bfloat16*>(
          ring + (size_t)st * a.ring_bytes) + (size_t)r_lo * ldw;
      float res[NT];
      if (cnt > 0 && a.diag_nocompute) {   // diagnostics: streaming/sync cost only
#pragma unroll
        for (int m = 0; m < NT; ++m) res[m] = 0.f;
        epi(crow + r_lo, false, res, R);
      } else if (cnt > 0) {
        const int rg = sg.row0g + crow + r_lo;
        if (R == 8) k2_rows<8, NT>(W, ldw, cnt, K, xs, ldx, n, res, rg);
        else if (R == 4) k2_rows<4, NT>(W, ldw, cnt, K, xs, ldx, n, res, rg);
        else k2_rows<2, NT>(W, ldw, cnt, K, xs, ldx, n, res, rg);
        const int rr = R == 8 ? k2_row<8>(lane) : R == 4 ? k2_row<4>(lane) : k2_row<2>(lane);
        const bool owner = (lane & (32 / R - 1)) == 0;
        epi(crow + r_lo + rr, owner && rr < cnt, res, R);
      }
      __syncwarp();
      if (lane == 0) {
        __threadfence_block();
        if (atomicAdd(&sdone[st], 1) == parts - 1) {
          sdone[st] = 0;
          srel[st] = srel[st] + 1;
          k2_arrive_local(&empty[st]);
        }
      }
    }
    ct += nchunks;
  };
  // all-to-all phase edge: everything pushed before it is visible after it
  auto phase_edge = [&]() {
    mark(1);
    k2_cons_sync();
    // edge e uses barrier e&1 (parity (e>>1)&1): an early arrival for edge
    // e+1 lands on the other barrier, and edge e+2's cannot come before this
    // CTA has passed edge e
    uint64_t* b = &pbar[pedge & 1];
    if (tid < CL) {   // one remote arrive per lane, in parallel
      asm volatile("fence.acq_rel.cluster;" ::: "memory");
      k2_arrive_remote(k2_mapa(k2_s(b), (uint32_t)tid));
    }
    k2_wait_cluster(b, (pedge >> 1) & 1u);
    ++pedge;
    mark(9);
  };
  // copy buf[m*ld + c], c in [c0, c1), m < n, from this CTA to every other
  // CTA's copy of buf: all consumer threads in parallel (one remote store
  // each per element), after the local values are complete
  auto push_range = [&](float* buf, int ld, int c0, int c1, int n) {
    k2_cons_sync();
    const int w = c1 - c0, per = n * w, tot = per * (CL - 1);
    for (int t = tid; t < tot; t += K2_CT) {
      int r = t / per;
      const int rem = t - r * per;
      const int m = rem / w, c = c0 + rem % w;
      r += (r >= rank);   // skip self
      const size_t off = (size_t)m * ld + c;
      k2_st(k2_mapa(k2_s(buf + off), (uint32_t)r), buf[off]);
    }
  };
  // per-warp RMS scales of the rows in xrep (same order in every warp / CTA)
  auto scales = [&](int n, float (&scl)[NT]) {
#pragma unroll
    for (int m = 0; m < NT; ++m) {
      scl[m] = 1.0f;
      if (m < n) {
        float ss = 0.f;
        for (int k = lane * 4; k < d; k += 128) {
          const float4 v = *reinterpret_cast<const float4*>(xrep + (size_t)m * d + k);
          ss = __fmaf_rn(v.x, v.x, ss); ss = __fmaf_rn(v.y, v.y, ss);
          ss = __fmaf_rn(v.z, v.z, ss); ss = __fmaf_rn(v.w, v.w, ss);
        }
        scl[m] = rms_scale(warp_sum(ss), d, a.eps);
      }
    }
  };
  // token-0 activations as bf16 hi + lo parts for the tensor-core GEMV
  auto split_hilo = [&](const float* src, int K) {
    if (NT != 1) return;
    for (int k = tid; k < K; k += K2_CT) {
      const float v = src[k];
      const __nv_bfloat16 h = __float2bfloat16_rn(v);
      xh[k] = h;
      xl[k] = __float2bfloat16_rn(__fsub_rn(v, __bfloat162float(h)));
    }
  };
  auto stage_norm = [&](int n, const float* gain) {
    for (int m = 0; m < n; ++m)
      for (int k = tid * 4; k < d; k += K2_CT * 4) {
        const float4 v = *reinterpret_cast<const float4*>(xrep + (size_t)m * d + k);
        const float4 g = __ldg(reinterpret_cast<const float4*>(gain + k));
        *reinterpret_cast<float4*>(xn + (size_t)m * d + k) =
            make_float4(__fmul_rn(v.x, g.x), __fmul_rn(v.y, g.y), __fmul_rn(v.z, g.z),
                        __fmul_rn(v.w, g.w));
      }
    k2_cons_sync();
    split_hilo(xn, d);
    k2_cons_sync();
  };

  int o0, o1;   // this CTA's residual rows (O and down)
  k2_slice(d, rank, CL, o0, o1);
  int tip_tok = 0, gate = 1, row = row0, pos = pos0, fw = 0;
  for (int k = 0; k <= steps; ++k) {
    int n;
    int toks[DR_NT];
    if (k == 0) {
      if (n_feed == 0) {
        const int valid = __ldcg(a.tip + 2);
        const float conf = valid ? __int_as_float(__ldcg(a.tip + 1)) : -1.0f;
        tip_tok = valid ? __ldcg(a.tip) : 0;
        gate = (valid && conf >= cutoff) ? 1 : 0;
        if (rank == 0 && tid == 0) {
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
      for (int i = 0; i < DR_NT; ++i) toks[i] = i < n ? Hd.tok[i] : 0;
    } else {
      if (chain && !gate) {
        if (rank == 0)
          for (int j = tid; j <= steps - k; j += K2_CT) {
            a.cell_pos[row + j] = pos + j;
            a.cell_mask[row + j] = 0u;
          }
        break;
      }
      n = 1;
      toks[0] = chain ? tip_tok : Hd.tok[n_feed + k - 1];
      for (int i = 1; i < DR_NT; ++i) toks[i] = 0;
    }
    if (tid == 0) go_fwd = fw;   // the producer may stream this forward
    const int rowA = row, posA = pos;
    if (rank == 0)
      for (int i = tid; i < n; i += K2_CT) {
        a.cell_pos[rowA + i] = posA + i;
        a.cell_mask[rowA + i] = 1u;
      }
    // embedding rows -> the local replica of x
    for (int m = 0; m < n; ++m) {
      const __nv_bfloat16* e = a.emb + (size_t)toks[m] * d;
      for (int c = tid * 8; c < d; c += K2_CT * 8) {
        float v[8];
        bf16x8_to_f32(__ldg(reinterpret_cast<const uint4*>(e + c)), v);
#pragma unroll
        for (int j = 0; j < 8; ++j) xrep[(size_t)m * d + c + j] = v[j];
      }
    }
    k2_cons_sync();

    for (int l = 0; l < a.L; ++l) {
      const DraftLayer& L = lw[l];
      __nv_bfloat16* Kc = a.kc + a.kv_layer_elems * l;
      __nv_bfloat16* Vc = a.vc + a.kv_layer_elems * l;
      // ---------------- A: rmsnorm + QKV + RoPE (row pairs) ------------------
      {
        float scl[NT];
        scales(n, scl);
        stage_norm(n, L.g_attn);
        const K2Seg sg = k2_seg(a, lw, l, 0, rank, CL);
        int p0, p1;
        k2_slice((qd + 2 * kvd) / 2, rank, CL, p0, p1);
        run_phase(sg, d, xn, d, n, [&](int rs, bool own, float (&res)[NT], int R) {
          const int px = R == 8 ? 4 : R == 4 ? 8 : 16;   // lane holding row rs + 1
          float odd[NT];
#pragma unroll
          for (int m = 0; m < NT; ++m) odd[m] = __shfl_xor_sync(0xffffffffu, res[m], px);
          if (!own || (rs & 1)) return;
          const int Rg = 2 * p0 + rs;
          int sec, off;
          if (Rg < qd) { sec = 0; off = Rg; }
          else if (Rg < qd + kvd) { sec = 1; off = Rg - qd; }
          else { sec = 2; off = Rg - qd - kvd; }
          const int j = (off % HD) >> 1;
          const int sbase = (sec == 0 ? 0 : sec == 1 ? qd : qd + kvd);
#pragma unroll
          for (int m = 0; m < NT; ++m) {
            if (m >= n) break;
            const float y0 = __fmul_rn(res[m], scl[m]), y1 = __fmul_rn(odd[m], scl[m]);
            int e0 = off, e1 = off + 1;
            float v0 = y0, v1 = y1;
            if (sec < 2) {   // pair-interleaved rows -> rotate-half dims
              e0 = (off / HD) * HD + j;
              e1 = e0 + (HD >> 1);
              float sn, cs;
              sincosf((float)(posA + m) * inv_s[j], &sn, &cs);
              v0 = y0 * cs - y1 * sn;
              v1 = y1 * cs + y0 * sn;
            }
            // staged locally in hbuf ([m][q | k | v], de-interleaved dims);
            // K/V also go to the cache rows (bf16) and are staged rounded
            if (sec == 0) {
              hbuf[(size_t)m * f + sbase + e0] = v0;
              hbuf[(size_t)m * f + sbase + e1] = v1;
            } else {
              const __nv_bfloat16 b0 = __float2bfloat16_rn(v0), b1 = __float2bfloat16_rn(v1);
              __nv_bfloat16* c = (sec == 1 ? Kc : Vc) + (size_t)(rowA + m) * kvd;
              c[e0] = b0;
              c[e1] = b1;
              hbuf[(size_t)m * f + sbase + e0] = __bfloat162float(b0);
              hbuf[(size_t)m * f + sbase + e1] = __bfloat162float(b1);
            }
          }
        });
        // route this CTA's q/k/v values to the CTAs whose heads use them
        k2_cons_sync();
        const int G = a.H / a.KH;
        const int npair = p1 - p0;
        for (int t = tid; t < n * npair * 2; t += K2_CT) {
          const int m = t / (npair * 2), rem = t % (npair * 2);
          const int R = 2 * (p0 + (rem >> 1)) + (rem & 1);
          int sec, off;
          if (R < qd) { sec = 0; off = R; }
          else if (R < qd + kvd) { sec = 1; off = R - qd; }
          else { sec = 2; off = R - qd - kvd; }
          int e = off;
          if (sec < 2) {
            const int j = (off % HD) >> 1;
            e = (off / HD) * HD + j + ((off & 1) ? (HD >> 1) : 0);
          }
          const int sbase = (sec == 0 ? 0 : sec == 1 ? qd : qd + kvd);
          const float v = hbuf[(size_t)m * f + sbase + e];
          const int hd0 = sec == 0 ? e / HD : (e / HD) * G;
          const int nh = sec == 0 ? 1 : G;
          for (int g = 0; g < nh; ++g) {
            const int hh = hd0 + g;
            const size_t b = (((size_t)(hh / CL) * NTR + m) * 3 + sec) * HD + (e % HD);
            k2_st(k2_mapa(k2_s(qkvb + b), (uint32_t)(hh % CL)), v);
          }
        }
      }
      phase_edge();

      // ---------------- B: attention for this CTA's heads -------------------
      {
        constexpr int LPR = HD / 8;
        constexpr int RPW = 32 / LPR;           // rows per warp pass
        constexpr int PB = 8;                   // passes per batch (loads in flight)
        const int grp = lane / LPR, li = lane % LPR;
        for (int j = 0; j < HPC; ++j) {
          const int hh = rank + j * CL;
          if (hh >= a.H) break;
          const int kh = hh / (a.H / a.KH);
          for (int m = 0; m < n; ++m) {
            const float* qb = qkvb + (((size_t)j * NTR + m) * 3) * HD;
            float qv[8];
#pragma unroll
            for (int t = 0; t < 8; ++t) qv[t] = qb[li * 8 + t] * att_scale;
            // warp w takes history rows w*RPW + grp + i*K2_CW*RPW (online softmax)
            float mx = -INFINITY, ls = 0.f, acc[8];
#pragma unroll
            for (int t = 0; t < 8; ++t) acc[t] = 0.f;
            const int hist = rowA;                 // rows [0, rowA) from the cache
            const int stride = K2_CW * RPW;
            for (int base = warp * RPW; base < hist; base += stride * PB) {   // warp-uniform
              const int b0 = base + grp;
              uint4 kr[PB], vr[PB];
#pragma unroll
              for (int p = 0; p < PB; ++p) {
                const int r = b0 + p * stride;
                const size_t off = (size_t)r * kvd + kh * HD + li * 8;
                kr[p] = r < hist ? __ldcg(reinterpret_cast<const uint4*>(Kc + off)) : make_uint4(0, 0, 0, 0);
                vr[p] = r < hist ? __ldcg(reinterpret_cast<const uint4*>(Vc + off)) : make_uint4(0, 0, 0, 0);
              }
#pragma unroll
              for (int p = 0; p < PB; ++p) {
                const int r = b0 + p * stride;
                float kf[8];
                bf16x8_to_f32(kr[p], kf);
                float s = 0.f;
#pragma unroll
                for (int t = 0; t < 8; ++t) s = __fmaf_rn(qv[t], kf[t], s);
#pragma unroll
                for (int o = LPR / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
                if (r < hist) {
                  float vf[8];
                  bf16x8_to_f32(vr[p], vf);
                  if (s > mx) {
                    const float c = __expf(mx - s);
                    ls = __fmul_rn(ls, c);
#pragma unroll
                    for (int t = 0; t < 8; ++t) acc[t] = __fmul_rn(acc[t], c);
                    mx = s;
                  }
                  const float p_ = __expf(s - mx);
                  ls = __fadd_rn(ls, p_);
#pragma unroll
                  for (int t = 0; t < 8; ++t) acc[t] = __fmaf_rn(p_, vf[t], acc[t]);
                }
              }
            }
            // this step's rows (tokens 0..m), from shared memory
            if (warp == 0 && grp == 0) {
              for (int i = 0; i <= m; ++i) {
                const float* kb = qkvb + (((size_t)j * NTR + i) * 3 + 1) * HD + li * 8;
                const float* vb = qkvb + (((size_t)j * NTR + i) * 3 + 2) * HD + li * 8;
                float s = 0.f;
#pragma unroll
                for (int t = 0; t < 8; ++t) s = __fmaf_rn(qv[t], kb[t], s);
#pragma unroll
                for (int o = LPR / 2; o > 0; o >>= 1) s += __shfl_xor_sync((1u << LPR) - 1, s, o);
                if (s > mx) {
                  const float c = __expf(mx - s);
                  ls = __fmul_rn(ls, c);
#pragma unroll
                  for (int t = 0; t < 8; ++t) acc[t] = __fmul_rn(acc[t], c);
                  mx = s;
                }
                const float p_ = __expf(s - mx);
                ls = __fadd_rn(ls, p_);
#pragma unroll
                for (int t = 0; t < 8; ++t) acc[t] = __fmaf_rn(p_, vb[t], acc[t]);
              }
            }
            // combine the row groups of the warp (fixed butterfly), then warps
#pragma unroll
            for (int o = LPR; o < 32; o <<= 1) {
              const float m2 = __shfl_xor_sync(0xffffffffu, mx, o);
              const float l2 = __shfl_xor_sync(0xffffffffu, ls, o);
              float a2[8];
#pragma unroll
              for (int t = 0; t < 8; ++t) a2[t] = __shfl_xor_sync(0xffffffffu, acc[t], o);
              const float M = fmaxf(mx, m2);
              if (M != -INFINITY) {
                const float c1 = __expf(mx - M), c2 = __expf(m2 - M);
                ls = __fadd_rn(__fmul_rn(ls, c1), __fmul_rn(l2, c2));
#pragma unroll
                for (int t = 0; t < 8; ++t)
                  acc[t] = __fadd_rn(__fmul_rn(acc[t], c1), __fmul_rn(a2[t], c2));
                mx = M;
              }
            }
            if (grp == 0) {
#pragma unroll
              for (int t = 0; t < 8; ++t) gpart[warp][2 + li * 8 + t] = acc[t];
              if (li == 0) { gpart[warp][0] = mx; gpart[warp][1] = ls; }
            }
            k2_cons_sync();
            if (tid < HD) {
              float M = -INFINITY;
              for (int w = 0; w < K2_CW; ++w) M = fmaxf(M, gpart[w][0]);
              float Ls = 0.f, o = 0.f;
              for (int w = 0; w < K2_CW; ++w) {
                if (gpart[w][0] == -INFINITY) continue;
                const float c = __expf(gpart[w][0] - M);
                Ls = __fadd_rn(Ls, __fmul_rn(gpart[w][1], c));
                o = __fadd_rn(o, __fmul_rn(gpart[w][2 + tid], c));
              }
              abuf[(size_t)m * qd + hh * HD + tid] = o / Ls;
            }
            k2_cons_sync();
          }
        }
        for (int j = 0; j < HPC; ++j) {
          const int hh = rank + j * CL;
          if (hh >= a.H) break;
          push_range(abuf, qd, hh * HD, (hh + 1) * HD, n);
        }
      }
      phase_edge();

      // ---------------- C: x += attn @ Wo (this CTA's rows) ------------------
      {
        const K2Seg sg = k2_seg(a, lw, l, 1, rank, CL);
        split_hilo(abuf, qd);
        k2_cons_sync();
        run_phase(sg, qd, abuf, qd, n, [&](int rs, bool own, float (&res)[NT], int) {
          if (!own) return;
          const int r = o0 + rs;
#pragma unroll
          for (int m = 0; m < NT; ++m) {
            if (m >= n) break;
            const float nv = __fadd_rn(xrep[(size_t)m * d + r], res[m]);
            if (!isfinite(nv)) set_error(a.err, SP_DEV_NONFINITE);
            xrep[(size_t)m * d + r] = nv;
          }
        });
        push_range(xrep, d, o0, o1, n);
      }
      phase_edge();

      // ---------------- D: h = silu(g) * u of rmsnorm(x) ---------------------
      {
        float scl[NT];
        scales(n, scl);
        mark(20);
        stage_norm(n, L.g_mlp);
        mark(21);
        const K2Seg sg = k2_seg(a, lw, l, 2, rank, CL);
        int u0, u1;
        k2_slice(f, rank, CL, u0, u1);
        run_phase(sg, d, xn, d, n, [&](int rs, bool own, float (&res)[NT], int R) {
          const int px = R == 8 ? 4 : R == 4 ? 8 : 16;
          float odd[NT];
#pragma unroll
          for (int m = 0; m < NT; ++m) odd[m] = __shfl_xor_sync(0xffffffffu, res[m], px);
          if (!own || (rs & 1)) return;
          const int col = u0 + (rs >> 1);
#pragma unroll
          for (int m = 0; m < NT; ++m) {
            if (m >= n) break;
            const float g = __fmul_rn(res[m], scl[m]), uu = __fmul_rn(odd[m], scl[m]);
            hbuf[(size_t)m * f + col] = __fmul_rn(silu(g), uu);
          }
        });
        mark(22);
        push_range(hbuf, f, u0, u1, n);
        mark(23);
      }
      phase_edge();

      // ---------------- E: x += h @ Wd (this CTA's rows) ---------------------
      {
        const K2Seg sg = k2_seg(a, lw, l, 3, rank, CL);
        run_phase(sg, f, hbuf, f, n, [&](int rs, bool own, float (&res)[NT], int) {
          if (!own) return;
          const int r = o0 + rs;
#pragma unroll
          for (int m = 0; m < NT; ++m) {
            if (m >= n) break;
            const float nv = __fadd_rn(xrep[(size_t)m * d + r], res[m]);
            if (!isfinite(nv)) set_error(a.err, SP_DEV_NONFINITE);
            xrep[(size_t)m * d + r] = nv;
          }
        });
        push_range(xrep, d, o0, o1, n);
      }
      phase_edge();
    }

    // ---------------- H: final norm + LM head (this CTA's rows) --------------
    {
      const int m = n - 1;
      float ss = 0.f;
      for (int kk = lane * 4; kk < d; kk += 128) {
        const float4 v = *reinterpret_cast<const float4*>(xrep + (size_t)m * d + kk);
        ss = __fmaf_rn(v.x, v.x, ss); ss = __fmaf_rn(v.y, v.y, ss);
        ss = __fmaf_rn(v.z, v.z, ss); ss = __fmaf_rn(v.w, v.w, ss);
      }
      const float sc0 = rms_scale(warp_sum(ss), d, a.eps);
      for (int kk = tid * 4; kk < d; kk += K2_CT * 4) {
        const float4 v = *reinterpret_cast<const float4*>(xrep + (size_t)m * d + kk);
        const float4 g = __ldg(reinterpret_cast<const float4*>(a.g_final + kk));
        *reinterpret_cast<float4*>(xn + kk) =
            make_float4(__fmul_rn(v.x, g.x), __fmul_rn(v.y, g.y), __fmul_rn(v.z, g.z),
                        __fmul_rn(v.w, g.w));
      }
      k2_cons_sync();
      split_hilo(xn, d);
      k2_cons_sync();
      int v0, v1;
      k2_slice(a.V, rank, CL, v0, v1);
      const K2Seg sg = k2_seg(a, lw, 0, 4, rank, CL);
      K2Top2 t{-INFINITY, 0x7fffffff, -INFINITY, 0x7fffffff};
      float mx = -INFINITY, se = 0.f;
      int nan = 0;
      run_phase(sg, d, xn, d, 1, [&](int rs, bool own, float (&res)[NT], int) {
        if (!own) return;
        const float v = __fmul_rn(res[0], sc0);
        if (isnan(v)) { nan = 1; return; }
        k2_push(t, v, v0 + rs);
        k2_online(mx, se, v);
      });
      // lanes -> warp (fixed butterfly), then warps 0..7 in order below
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const float a1 = __shfl_xor_sync(0xffffffffu, t.v1, o);
        const int b1 = __shfl_xor_sync(0xffffffffu, t.i1, o);
        const float a2 = __shfl_xor_sync(0xffffffffu, t.v2, o);
        const int b2 = __shfl_xor_sync(0xffffffffu, t.i2, o);
        k2_push(t, a1, b1);
        k2_push(t, a2, b2);
        const float m2 = __shfl_xor_sync(0xffffffffu, mx, o);
        const float s2 = __shfl_xor_sync(0xffffffffu, se, o);
        k2_merge(mx, se, m2, s2);
        nan |= __shfl_xor_sync(0xffffffffu, nan, o);
      }
      if (lane == 0) {
        wred[warp][0] = t.v1; wred[warp][1] = __int_as_float(t.i1);
        wred[warp][2] = t.v2; wred[warp][3] = __int_as_float(t.i2);
        wred[warp][4] = mx; wred[warp][5] = se; wred[warp][6] = __int_as_float(nan);
      }
      k2_cons_sync();
      if (tid < 7) {   // warps 0..7 in order -> this CTA's partial, pushed to all
        K2Top2 c{-INFINITY, 0x7fffffff, -INFINITY, 0x7fffffff};
        float cm = -INFINITY, cs = 0.f;
        int cn = 0;
        for (int w = 0; w < K2_CW; ++w) {
          k2_push(c, wred[w][0], __float_as_int(wred[w][1]));
          k2_push(c, wred[w][2], __float_as_int(wred[w][3]));
          k2_merge(cm, cs, wred[w][4], wred[w][5]);
          cn |= __float_as_int(wred[w][6]);
        }
        const float vals[7] = {c.v1, __int_as_float(c.i1), c.v2, __int_as_float(c.i2), cm, cs,
                               __int_as_float(cn)};
        lmp[(size_t)rank * 8 + tid] = vals[tid];
      }
      push_range(lmp, 0, rank * 8, rank * 8 + 7, 1);
    }
    phase_edge();
    if (tid == 0) {
      K2Top2 c{-INFINITY, 0x7fffffff, -INFINITY, 0x7fffffff};
      float cm = -INFINITY, cs = 0.f;
      int cn = 0;
      for (int r = 0; r < CL; ++r) {   // CTAs in rank order
        const float* p = lmp + r * 8;
        k2_push(c, p[0], __float_as_int(p[1]));
        k2_push(c, p[2], __float_as_int(p[3]));
        k2_merge(cm, cs, p[4], p[5]);
        cn |= __float_as_int(p[6]);
      }
      const float conf = 1.0f / cs;
      s_tok = c.i1;
      s_gate = conf >= cutoff ? 1 : 0;
      if (rank == 0) {
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
    k2_cons_sync();
    tip_tok = s_tok;
    gate = chain ? s_gate : 1;
    row += n;
    pos += n;
    ++fw;
  }
  if (tid == 0) stop = 1;
  if (a.prof && rank == 0 && tid == 0) {
    a.prof[1 + nprof] = (15ll << 56) | (wait_cyc & ((1ll << 56) - 1));
    a.prof[0] = nprof + 1;
  }
  // every chunk the producer issued has been consumed (it streams a forward
  // only after go_fwd names it, and each confirmed forward is fully consumed)
  if (rank == 0 && tid == 0 && a.err_out) {
    __threadfence();
    *a.err_out = *a.err;
  }
  k2_cluster_sync_all();   // no CTA leaves while others may still push into it
}

size_t draft2_act_bytes(const DraftArgs& a, int cl, int nt) {
  const int qd = a.H * a.hd;
  const int hpc = (a.H + cl - 1) / cl;
  const int kx = a.d > qd ? a.d : qd;
  return sizeof(float) * ((size_t)nt * (2 * a.d + qd + a.f) + (size_t)hpc * nt * 3 * a.hd +
                          (size_t)cl * 8) + 2 * sizeof(__nv_bfloat16) * (size_t)kx;
}

size_t draft2_smem_bytes(const DraftArgs& a, int cl) {
  return (size_t)a.ring_stages * a.ring_bytes + draft2_act_bytes(a, cl, a.nt);
}

template <int HD, int CL, int NT>
static cudaError_t launch_k2(const DraftArgs& a, cudaStream_t st) {
  const size_t smem = draft2_smem_bytes(a, CL);
  cudaError_t e = cudaFuncSetAttribute(draft_cluster_kernel<HD, CL, NT>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (CL > 8) {
    e = cudaFuncSetAttribute(draft_cluster_kernel<HD, CL, NT>,
                             cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CL);
  cfg.blockDim = dim3(K2_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, draft_cluster_kernel<HD, CL, NT>, a);
}

template <int HD, int CL, int NT>
static int clusters_k2(const DraftArgs& a) {
  const size_t smem = draft2_smem_bytes(a, CL);
  if (cudaFuncSetAttribute(draft_cluster_kernel<HD, CL, NT>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return 0;
  if (CL > 8 && cudaFuncSetAttribute(draft_cluster_kernel<HD, CL, NT>,
                                     cudaFuncAttributeNonPortableClusterSizeAllowed,
                                     1) != cudaSuccess)
    return 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CL);
  cfg.blockDim = dim3(K2_THREADS);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, draft_cluster_kernel<HD, CL, NT>, &cfg) != cudaSuccess)
    return 0;
  return n;
}

int draft2_cluster_size(const DraftArgs& a, int want) {
  // largest supported cluster (16 needs the non-portable opt-in) that fits
  if (want >= 16 && (a.hd == 64 ? clusters_k2<64, 16, DR_NT>(a) : clusters_k2<128, 16, DR_NT>(a)) > 0)
    return 16;
  if (want >= 8 && (a.hd == 64 ? clusters_k2<64, 8, DR_NT>(a) : clusters_k2<128, 8, DR_NT>(a)) > 0)
    return 8;
  return 0;
}

cudaError_t launch_draft_cluster(const DraftArgs& a, int cl, cudaStream_t st) {
  // one token per step (every chain launch) -> the single-token instantiation
  if (a.nt <= 1) {
    if (a.hd == 64) return cl == 16 ? launch_k2<64, 16, 1>(a, st) : launch_k2<64, 8, 1>(a, st);
    if (a.hd == 128) return cl == 16 ? launch_k2<128, 16, 1>(a, st) : launch_k2<128, 8, 1>(a, st);
  }
  if (a.hd == 64) return cl == 16 ? launch_k2<64, 16, DR_NT>(a, st) : launch_k2<64, 8, DR_NT>(a, st);
  if (a.hd == 128) return cl == 16 ? launch_k2<128, 16, DR_NT>(a, st) : launch_k2<128, 8, DR_NT>(a, st);
  return cudaErrorInvalidValue;
}

}  // namespace sp
