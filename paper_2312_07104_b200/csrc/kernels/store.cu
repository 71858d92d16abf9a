// KV store (rx_store_kv): k_pool[slot_i] = k_i, v_pool[slot_i] = v_i, bit-exact,
// plus the optional req_to_token append rtt_flat[idx_i] = slot_i.
// "KV cache tensors are stored in a non-contiguous, paged layout, where the
// size of each page is equivalent to one token" (§3): a token's
// page is one contiguous pool row of h_kv*head_dim bf16.
//
// Pure copy: 16-byte vector loads/stores, one warp per row chunk, grid sized
// to the row count.  HBM-bound: 2 * row_bytes read + written per token.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "params.cuh"

namespace rx {

__global__ void __launch_bounds__(256) store_kv_kernel(int64_t n, int row_vec, const int32_t* __restrict__ slots,
                                                       const int4* __restrict__ k, const int4* __restrict__ v,
                                                       int4* __restrict__ kpool, int4* __restrict__ vpool,
                                                       int32_t* __restrict__ rtt, const int64_t* __restrict__ rtt_idx) {
  // one thread per 16-byte vector; row i occupies vectors [i*row_vec, (i+1)*row_vec)
  const int64_t total = n * row_vec;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < total; t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = t / row_vec;
    const int c = int(t - i * row_vec);
    const int64_t slot = slots[i];
    if (k) {                                       // null k / v: table append only
      kpool[slot * row_vec + c] = k[t];
      vpool[slot * row_vec + c] = v[t];
    }
    if (rtt_idx && c == 0) rtt[rtt_idx[i]] = int32_t(slot);
  }
}

// Extend-side store (A5 of rx_extend): token i of the ragged batch belongs to
// the request b with qo[b] <= i < qo[b] + ext[b]; its slot is
// rtt[row_b][prefix[b] + i - qo[b]].  One warp per token row (all local heads,
// contiguous), 16-byte vectors, every warp independent (no serial chains).
__global__ void __launch_bounds__(256) extend_store_kernel(
    int64_t n, int batch, int row_vec, const int32_t* __restrict__ qo, const int32_t* __restrict__ ext,
    const int32_t* __restrict__ prefix, const int32_t* __restrict__ rows, const int32_t* __restrict__ rtt,
    int64_t rtt_stride, const int4* __restrict__ k, const int4* __restrict__ v, int4* __restrict__ kpool,
    int4* __restrict__ vpool) {
  const int lane = threadIdx.x & 31;
  for (int64_t i = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5; i < n;
       i += (int64_t(gridDim.x) * blockDim.x) >> 5) {
    int lo = 0, hi = batch - 1;                      // last b with qo[b] <= i
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (qo[mid] <= i) lo = mid; else hi = mid - 1;
    }
    const int b = lo;
    const int j = int(i - qo[b]);
    if (j >= ext[b]) continue;                       // (qo need not be dense)
    const int row = rows ? rows[b] : b;
    const int64_t slot = rtt[int64_t(row) * rtt_stride + prefix[b] + j];
    for (int c = lane; c < row_vec; c += 32) {
      kpool[slot * row_vec + c] = k[i * row_vec + c];
      vpool[slot * row_vec + c] = v[i * row_vec + c];
    }
  }
}

cudaError_t launch_extend_store(int64_t n, int batch, int row_bytes, const int32_t* qo, const int32_t* ext,
                                const int32_t* prefix, const int32_t* rows, const int32_t* rtt, int64_t rtt_stride,
                                const void* k, const void* v, void* kpool, void* vpool, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  int64_t blocks = (n * 32 + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  extend_store_kernel<<<int(blocks), 256, 0, st>>>(n, batch, row_bytes / 16, qo, ext, prefix, rows, rtt, rtt_stride,
                                                   static_cast<const int4*>(k), static_cast<const int4*>(v),
                                                   static_cast<int4*>(kpool), static_cast<int4*>(vpool));
  return cudaPeekAtLastError();
}

cudaError_t launch_store_kv(int64_t n, int row_bytes, const int32_t* slots, const void* k, const void* v,
                            void* kpool, void* vpool, int32_t* rtt, const int64_t* rtt_idx, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  const int row_vec = k ? row_bytes / 16 : 1;      // table only: one thread per row
  const int64_t total = n * row_vec;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  store_kv_kernel<<<int(blocks), 256, 0, st>>>(n, row_vec, slots, static_cast<const int4*>(k),
                                                static_cast<const int4*>(v), static_cast<int4*>(kpool),
                                                static_cast<int4*>(vpool), rtt, rtt_idx);
  return cudaPeekAtLastError();
}

// Host -> device copy of small metadata (slot tables, decode step records) by the SMs: the kernel
// reads pinned (UVA-mapped) host memory over PCIe itself, so the upload does not queue on the copy
// engines behind a large input prefetch of another stream (copy-engine work is served in
// submission order).  16-byte vectors when both pointers allow, bytes otherwise.
__global__ void __launch_bounds__(256) copy_h2d_kernel(char* __restrict__ dst, const char* __restrict__ src,
                                                       int64_t bytes) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  const int64_t t0 = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  const bool vec = ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15) == 0;
  const int64_t nv = vec ? bytes / 16 : 0;
  for (int64_t i = t0; i < nv; i += stride)
    reinterpret_cast<int4*>(dst)[i] = reinterpret_cast<const int4*>(src)[i];
  for (int64_t i = nv * 16 + t0; i < bytes; i += stride) dst[i] = src[i];
}

cudaError_t launch_copy_h2d(void* dst, const void* src, int64_t bytes, cudaStream_t st) {
  if (bytes <= 0) return cudaSuccess;
  int64_t blocks = (bytes / 16 + 255) / 256;
  blocks = blocks < 1 ? 1 : (blocks > 148 * 4 ? 148 * 4 : blocks);
  copy_h2d_kernel<<<int(blocks), 256, 0, st>>>(static_cast<char*>(dst), static_cast<const char*>(src), bytes);
  return cudaPeekAtLastError();
}

}  // namespace rx
