// K3/K10: cell-metadata kernels for the sequence-partitioned KV cache.
//
// One metadata table per stage (position int32, sequence bitmask uint32),
// shared by all of the stage's layers — the reference's per-layer tables
// evolve identically (kvcache.py:96-100), so keeping one removes pad_dead
// (kvcache.py:158-167) altogether.  K/V rows are written once by the QKV
// epilogue and never moved: copy/remove/keep only edit membership bits.
#include "kernels.cuh"

namespace sp {

constexpr int KV_THREADS = 1024;

// kvcache.py:135-156 (metadata half of insert, validated like the reference)
__global__ void meta_write_kernel(int32_t* pos, uint32_t* mask, int row0,
                                  const sp_token* toks, int n, int n_seq,
                                  int max_context, int* err) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const sp_token t = toks[i];
  uint32_t m = t.seq_mask;
  if (t.pos < 0 || t.pos >= max_context) set_error(err, SP_DEV_BAD_POS);
  if (n_seq < 32 && (m >> n_seq) != 0) { set_error(err, SP_DEV_BAD_SEQ); m &= (1u << n_seq) - 1; }
  if (m == 0) set_error(err, SP_DEV_BAD_SEQ);
  pos[row0 + i] = t.pos;
  mask[row0 + i] = m;
}

// kvcache.py:181-204.  For every destination the occupied-position set is
// taken before the copy, the candidate set (src member, pos < end) once; a
// destination never gains a second cell at a position it already holds.
// Single CTA: the occupied bitmap (one dst bitmask per position) lives in
// shared memory, so the two phases need only a CTA barrier.
__global__ void __launch_bounds__(KV_THREADS)
copy_kernel(const int32_t* __restrict__ pos, uint32_t* __restrict__ mask,
            int n, int src, uint32_t dst_mask, int end_pos, int max_context) {
  extern __shared__ uint32_t occ[];  // [max_context]
  dst_mask &= ~(1u << src);
  for (int p = threadIdx.x; p < max_context; p += KV_THREADS) occ[p] = 0;
  __syncthreads();
  for (int r = threadIdx.x; r < n; r += KV_THREADS) {
    const uint32_t m = mask[r] & dst_mask;
    if (m) atomicOr(&occ[pos[r]], m);
  }
  __syncthreads();
  const uint32_t sbit = 1u << src;
  for (int r = threadIdx.x; r < n; r += KV_THREADS) {
    const uint32_t m = mask[r];
    const int p = pos[r];
    if ((m & sbit) && p < end_pos) {
      const uint32_t add = dst_mask & ~occ[p];
      if (add) mask[r] = m | add;
    }
  }
}

// kvcache.py:206-216 (seq_mask may name several sequences: the stage purge)
__global__ void remove_kernel(const int32_t* __restrict__ pos,
                              uint32_t* __restrict__ mask, int n,
                              uint32_t seq_mask, int from_pos) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n;
       r += gridDim.x * blockDim.x)
    if (pos[r] >= from_pos) mask[r] &= ~seq_mask;
}

// llama.cpp seq_keep: cells of ``seq`` keep only ``seq``, all others die.
__global__ void keep_kernel(uint32_t* __restrict__ mask, int n, int seq) {
  const uint32_t b = 1u << seq;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n;
       r += gridDim.x * blockDim.x)
    mask[r] = (mask[r] & b) ? b : 0u;
}

static int grid_for(int n) { return max(1, min(148 * 4, (n + 255) / 256)); }

cudaError_t launch_meta_write(int32_t* pos, uint32_t* mask, int row0,
                              const sp_token* toks, int n, int n_seq,
                              int max_context, int* err, cudaStream_t st) {
  meta_write_kernel<<<(n + 127) / 128, 128, 0, st>>>(pos, mask, row0, toks, n,
                                                     n_seq, max_context, err);
  return cudaGetLastError();
}

// Stable compaction of the cell pool (reclaims rows of dead cells).  One
// CTA scans the live flags (mask != 0) in row order: live row r gets the new
// row new = #live rows before r, src_of[new] = r, and the metadata moves to
// scratch (pos2/mask2) -> copied back by the host.  Row order among live
// cells is preserved, so plan tie order (by row) and every result are
// unchanged.
__global__ void __launch_bounds__(KV_THREADS)
compact_scan_kernel(const int32_t* __restrict__ pos, const uint32_t* __restrict__ mask, int n,
                    int32_t* __restrict__ src_of, int32_t* __restrict__ pos2,
                    uint32_t* __restrict__ mask2, int* live_out) {
  __shared__ int wsum[KV_THREADS / 32];
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int b = 0; b < n; b += KV_THREADS) {
    const int r = b + threadIdx.x;
    const int live = (r < n && mask[r] != 0u) ? 1 : 0;
    int incl = live;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    int base = carry;
    for (int w = 0; w < warp; ++w) base += wsum[w];
    if (live) {
      const int nr = base + incl - 1;
      src_of[nr] = r;
      pos2[nr] = pos[r];
      mask2[nr] = mask[r];
    }
    __syncthreads();
    if (threadIdx.x == KV_THREADS - 1) carry = base + incl;
    __syncthreads();
  }
  if (threadIdx.x == 0) *live_out = carry;
}

// gather the live K or V rows of one layer into scratch (new row order)
__global__ void compact_gather_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                      const int32_t* __restrict__ src_of, const int* live,
                                      int vec_per_row) {
  const int nl = *live;
  const long total = (long)nl * vec_per_row;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total;
       i += (long)gridDim.x * blockDim.x) {
    const int r = (int)(i / vec_per_row), v = (int)(i % vec_per_row);
    dst[i] = src[(size_t)src_of[r] * vec_per_row + v];
  }
}

cudaError_t launch_compact_scan(const int32_t* pos, const uint32_t* mask, int n, int32_t* src_of,
                                int32_t* pos2, uint32_t* mask2, int* live, cudaStream_t st) {
  compact_scan_kernel<<<1, KV_THREADS, 0, st>>>(pos, mask, n, src_of, pos2, mask2, live);
  return cudaGetLastError();
}

cudaError_t launch_compact_gather(const void* src, void* dst, const int32_t* src_of,
                                  const int* live, int row_bytes, int n_max, cudaStream_t st) {
  const int vpr = row_bytes / 16;
  long total = (long)n_max * vpr;
  int grid = (int)((total + 255) / 256);
  if (grid > 4 * 148) grid = 4 * 148;
  if (grid < 1) grid = 1;
  compact_gather_kernel<<<grid, 256, 0, st>>>(reinterpret_cast<const uint4*>(src),
                                              reinterpret_cast<uint4*>(dst), src_of, live, vpr);
  return cudaGetLastError();
}

cudaError_t launch_copy(const int32_t* pos, uint32_t* mask, int n, int src,
                        uint32_t dst_mask, int end_pos, int max_context,
                        cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const size_t smem = (size_t)max_context * sizeof(uint32_t);
  static size_t configured = 0;
  if (configured < smem) {   // (48 KB default covers static + dynamic)
    cudaFuncSetAttribute(copy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    configured = smem;
  }
  copy_kernel<<<1, KV_THREADS, smem, st>>>(pos, mask, n, src, dst_mask, end_pos,
                                           max_context);
  return cudaGetLastError();
}

cudaError_t launch_remove(const int32_t* pos, uint32_t* mask, int n,
                          uint32_t seq_mask, int from_pos, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  remove_kernel<<<grid_for(n), 256, 0, st>>>(pos, mask, n, seq_mask, from_pos);
  return cudaGetLastError();
}

cudaError_t launch_keep(uint32_t* mask, int n, int seq, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  keep_kernel<<<grid_for(n), 256, 0, st>>>(mask, n, seq);
  return cudaGetLastError();
}

}  // namespace sp

static int status(cudaError_t e) { return e == cudaSuccess ? SP_OK : SP_ERR_CUDA; }

extern "C" int sp_kv_meta_write(int32_t* cell_pos, uint32_t* cell_mask, int row0,
                                const sp_token* toks, int n, int n_seq_ids,
                                int max_context, int* err, void* stream) {
  if (n <= 0) return SP_ERR_ARG;
  return status(sp::launch_meta_write(cell_pos, cell_mask, row0, toks, n,
                                      n_seq_ids, max_context, err,
                                      reinterpret_cast<cudaStream_t>(stream)));
}

extern "C" int sp_kv_copy(int32_t* cell_pos, uint32_t* cell_mask, int n_cells,
                          int src, uint32_t dst_mask, int end_pos,
                          int max_context, void* stream) {
  if (src < 0 || src >= 32) return SP_ERR_CACHE;
  return status(sp::launch_copy(cell_pos, cell_mask, n_cells, src, dst_mask,
                                end_pos, max_context,
                                reinterpret_cast<cudaStream_t>(stream)));
}

extern "C" int sp_kv_remove(const int32_t* cell_pos, uint32_t* cell_mask,
                            int n_cells, uint32_t seq_mask, int from_pos,
                            void* stream) {
  return status(sp::launch_remove(cell_pos, cell_mask, n_cells, seq_mask,
                                  from_pos, reinterpret_cast<cudaStream_t>(stream)));
}

extern "C" int sp_kv_keep(uint32_t* cell_mask, int n_cells, int seq, void* stream) {
  if (seq < 0 || seq >= 32) return SP_ERR_CACHE;
  return status(sp::launch_keep(cell_mask, n_cells, seq,
                                reinterpret_cast<cudaStream_t>(stream)));
}
