// TP output all-gather over peer memory (A9; §3 "each GPU maintains a sharded KV
// cache ... the tree operations are the same": the only exchange of a tensor-parallel attention
// call is reassembling the head shards of its output).
//
// Instead of an NCCL collective per call (~30-40 us of launch and proxy overhead even on one rank,
// the same order as a decode step's compute at P = 8), every rank maps its peers' gather buffers
// (CUDA IPC; NVLink / NVSwitch peer memory on a multi-GPU node) and one small kernel
//   (1) stores its own shard into every peer's buffer (16-byte vectors, P2P stores),
//   (2) publishes "call seq is in your buffer" to every peer (flag, release at system scope),
//   (3) waits until every peer's flag for seq has arrived in its own buffer (acquire),
// so when the kernel completes the rank holds the whole [P, bytes] gathered output.
// Buffer layout per rank (one IPC allocation): [flags int64 P | counter | pad to 256 B | slot 0 |
// slot 1], a slot = P shards of cap bytes; call seq uses slot seq & 1, so a peer that already
// runs call seq + 1 never overwrites the slot this rank still reads for call seq (it cannot reach
// seq + 2 before this rank signalled seq + 1, which is after this rank's reads of seq in stream
// order).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>

#include "../../../include/rx.h"
#include "params.cuh"

namespace rx {

constexpr int kTpThreads = 256;

__device__ __forceinline__ void st_release_sys(int64_t* p, int64_t v) {
  asm volatile("st.release.sys.global.b64 [%0], %1;\n" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ int64_t ld_acquire_sys(const int64_t* p) {
  int64_t v;
  asm volatile("ld.acquire.sys.global.b64 %0, [%1];\n" : "=l"(v) : "l"(p) : "memory");
  return v;
}

struct TpPeers {
  char* buf[8];        // every rank's buffer base, mapped into this process (buf[rank] = own)
};

__global__ void __launch_bounds__(kTpThreads) tp_allgather_kernel(const int4* __restrict__ src, int64_t vecs,
                                                                  const TpPeers peers, int P, int rank,
                                                                  int64_t cap, int64_t seq) {
  const int64_t slot_off = kTpHeader + (seq & 1) * int64_t(P) * cap + int64_t(rank) * cap;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < vecs; i += stride) {
    const int4 v = src[i];
#pragma unroll 8
    for (int p = 0; p < P; ++p) reinterpret_cast<int4*>(peers.buf[p] + slot_off)[i] = v;
  }
  // the last CTA to finish publishes seq to every peer, then waits for every peer's seq
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x != 0) return;
  int* counter = reinterpret_cast<int*>(peers.buf[rank] + 8 * kTpMaxRanks);
  if (atomicAdd(counter, 1) != int(gridDim.x) - 1) return;
  *counter = 0;
  __threadfence_system();
  for (int p = 0; p < P; ++p) st_release_sys(reinterpret_cast<int64_t*>(peers.buf[p]) + rank, seq);
  const int64_t* flags = reinterpret_cast<const int64_t*>(peers.buf[rank]);
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int p = 0; p < P; ++p) {
    while (ld_acquire_sys(flags + p) < seq) {
      __nanosleep(64);
      uint64_t t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > 30ull * 1000000000ull) __trap();   // a peer never arrived: fail loudly, never hang
    }
  }
}

}  // namespace rx

extern "C" {

size_t rx_tp_buffer_bytes(int32_t world, int64_t cap) {
  if (world < 1 || world > rx::kTpMaxRanks || cap < 0) return 0;
  return rx::kTpHeader + 2 * size_t(world) * size_t((cap + 15) / 16 * 16);
}

rx_status rx_tp_ipc_handle(void* d_buf, void* handle_out) {
  if (!d_buf || !handle_out) return RX_E_INVALID;
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, d_buf) != cudaSuccess) return RX_E_CUDA;
  static_assert(sizeof(h) == RX_TP_HANDLE_BYTES, "IPC handle size");
  memcpy(handle_out, &h, sizeof(h));
  return RX_OK;
}

int64_t rx_tp_ipc_offset(const void* d_buf) {
  // an IPC handle names the whole allocation that holds d_buf (a caching allocator may place the
  // buffer inside a larger segment): peers add this offset to the base they open
  typedef CUresult (*GetRangeFn)(CUdeviceptr*, size_t*, CUdeviceptr);
  static GetRangeFn fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &ptr, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return -1;
    fn = reinterpret_cast<GetRangeFn>(ptr);
  }
  if (!d_buf) return -1;
  CUdeviceptr base = 0;
  size_t size = 0;
  if (fn(&base, &size, reinterpret_cast<CUdeviceptr>(d_buf)) != CUDA_SUCCESS) return -1;
  return int64_t(reinterpret_cast<CUdeviceptr>(d_buf) - base);
}

rx_status rx_tp_ipc_open(const void* handle, void** d_ptr) {
  if (!handle || !d_ptr) return RX_E_INVALID;
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  if (cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) return RX_E_CUDA;
  return RX_OK;
}

rx_status rx_tp_ipc_close(void* d_ptr) {
  if (!d_ptr) return RX_E_INVALID;
  return cudaIpcCloseMemHandle(d_ptr) == cudaSuccess ? RX_OK : RX_E_CUDA;
}

rx_status rx_tp_allgather(const void* d_src, int64_t bytes, void* const* peer_bufs, int32_t world, int32_t rank,
                          int64_t cap, int64_t seq, void* stream) {
  if (world < 1 || world > rx::kTpMaxRanks || rank < 0 || rank >= world || bytes < 0 || bytes > cap ||
      bytes % 16 || cap % 16 || seq < 1 || !peer_bufs || (bytes > 0 && !d_src))
    return RX_E_INVALID;
  rx::TpPeers peers{};
  for (int p = 0; p < world; ++p) {
    if (!peer_bufs[p]) return RX_E_INVALID;
    peers.buf[p] = static_cast<char*>(peer_bufs[p]);
  }
  const int64_t vecs = bytes / 16;
  int64_t blocks = (vecs + rx::kTpThreads - 1) / rx::kTpThreads;
  blocks = blocks < 1 ? 1 : (blocks > 2 * 148 ? 2 * 148 : blocks);
  rx::tp_allgather_kernel<<<int(blocks), rx::kTpThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const int4*>(d_src), vecs, peers, world, rank, cap, seq);
  return cudaPeekAtLastError() == cudaSuccess ? RX_OK : RX_E_CUDA;
}

}  // extern "C"
