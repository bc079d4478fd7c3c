// Per-SM streaming bandwidth probe: each CTA pulls `per_cta` bytes of a
// large buffer through a 4-stage ring of 1D bulk copies (TMA) into shared
// memory, or with plain 16-byte loads.  Prints aggregate and per-SM GB/s for
// several grid sizes (one CTA per SM).  Diagnostic only.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bw_probe tools/bw_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t s32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int STAGES, int CHUNK>
__global__ void __launch_bounds__(128) bulk_stream(const char* src, size_t per_cta, int* sink) {
  extern __shared__ __align__(128) char buf[];
  __shared__ __align__(8) uint64_t bar[STAGES];
  const char* base = src + per_cta * blockIdx.x;
  const int nchunks = (int)(per_cta / CHUNK);
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  auto issue = [&](int c) {
    const int s = c % STAGES;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(&bar[s])),
                 "r"(CHUNK) : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(s32(buf + s * CHUNK)), "l"(base + (size_t)c * CHUNK), "r"(CHUNK),
        "r"(s32(&bar[s])) : "memory");
  };
  for (int c = 0; c < STAGES && c < nchunks; ++c) issue(c);
  int acc = 0;
  for (int c = 0; c < nchunks; ++c) {
    const int s = c % STAGES;
    const uint32_t par = (c / STAGES) & 1;
    uint32_t ok = 0;
    while (!ok)
      asm volatile(
          "{\n\t.reg .pred P1;\n\t"
          "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
          "selp.u32 %0, 1, 0, P1;\n\t}"
          : "=r"(ok) : "r"(s32(&bar[s])), "r"(par) : "memory");
    acc += buf[s * CHUNK];
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (c + STAGES < nchunks) issue(c + STAGES);
  }
  if (acc == 123456789) *sink = acc;
}

__global__ void __launch_bounds__(256) ldg_stream(const uint4* src, size_t per_cta, int* sink) {
  const uint4* base = src + (per_cta / 16) * blockIdx.x;
  const size_t n = per_cta / 16;
  uint32_t acc = 0;
  for (size_t i = threadIdx.x; i < n; i += 256 * 8) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const size_t j = i + (size_t)u * 256;
      v[u] = j < n ? __ldcs(base + j) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) acc ^= v[u].x;
  }
  if (acc == 0x12345678u) *sink = (int)acc;
}

int main() {
  const size_t total = (size_t)4 << 30;   // 4 GiB >> L2
  char* src;
  int* sink;
  cudaMalloc(&src, total);
  cudaMalloc(&sink, 4);
  cudaMemset(src, 1, total);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  constexpr int ST = 4, CH = 32768;
  cudaFuncSetAttribute(bulk_stream<ST, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, ST * CH);
  cudaFuncSetAttribute(bulk_stream<6, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * CH);
  // L2-resident: 16 CTAs x 2 MiB = 32 MiB, re-read (warm) -> L2 -> SM bandwidth
  for (int st = 4; st <= 6; st += 2) {
    const size_t per = (size_t)2 << 20;
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      if (st == 4) bulk_stream<4, CH><<<16, 128, 4 * CH>>>(src, per, sink);
      else bulk_stream<6, CH><<<16, 128, 6 * CH>>>(src, per, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    const double gbs = (double)per * 16 / (best * 1e-3) / 1e9;
    printf("L2-warm bulk stages %d grid 16: %8.1f GB/s total %7.1f per SM\n", st, gbs, gbs / 16);
  }
  const int grids[] = {1, 2, 4, 8, 16, 32, 64, 148};
  for (int g : grids) {
    const size_t per = (total / 148) / CH * CH;   // same bytes per CTA for every grid
    for (int kind = 0; kind < 2; ++kind) {
      float best = 1e30f;
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        if (kind == 0)
          bulk_stream<ST, CH><<<g, 128, ST * CH>>>(src, per, sink);
        else
          ldg_stream<<<g, 256>>>(reinterpret_cast<const uint4*>(src), per, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      const double gbs = (double)per * g / (best * 1e-3) / 1e9;
      printf("%-5s grid %3d: %8.1f GB/s total  %7.1f GB/s per SM\n", kind ? "ldg" : "bulk", g,
             gbs, gbs / g);
    }
  }
  cudaError_t e = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
