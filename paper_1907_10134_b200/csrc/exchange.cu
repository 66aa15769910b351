// exchange.cu — the carry exchange of the time-sharded scan (row a5, SURVEY
// 8(e)) over peer memory instead of an NCCL all-gather: each rank stores its
// up-sweep aggregate straight into every rank's mailbox (P2P stores over
// NVLink / NVSwitch; CUDA IPC mappings) and raises a per-rank flag there with
// a system-scope release; a rank's down-sweep starts after an acquire wait on
// the flags of the later ranks, whose aggregates its carry needs.
// Mailbox of a rank: [2][world][n] floats (epoch parity double buffer), flags
// [world] u32 (the last published epoch per sender, monotone), acks [world]
// u32 (the last epoch each reader finished reading from this rank's slot).
// Back-pressure: a writer publishing epoch e overwrites the slot of epoch
// e - 2, so it first waits until every reader (the earlier ranks) acked e - 2.
#include "common.cuh"

namespace bppsa {
namespace {

__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__global__ void publish_kernel(const float* __restrict__ src, long long n, int rank, int world,
                               float* const* __restrict__ peers, unsigned* const* __restrict__ peer_flags,
                               unsigned* __restrict__ counter, const unsigned* __restrict__ acks, unsigned epoch) {
  if (epoch > 2 && threadIdx.x == 0) {             // readers (ranks < rank) are done with epoch - 2's slot
    for (int r = 0; r < rank; ++r)
      while ((int)(ld_acquire_sys(acks + r) - (epoch - 2)) < 0) __nanosleep(256);
  }
  __syncthreads();
  const long long slot = ((long long)(epoch & 1u) * world + rank) * n;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride) {
    const float v = src[i];
    for (int p = 0; p < world; ++p) peers[p][slot + i] = v;
  }
  __threadfence_system();                          // this block's stores, before the count
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned done = atomicAdd(counter, 1u);
    if (done == gridDim.x - 1) {                   // the last block: every store is performed
      __threadfence_system();
      for (int p = 0; p < world; ++p)
        asm volatile("st.release.sys.global.u32 [%0], %1;\n" ::"l"(peer_flags[p] + rank), "r"(epoch) : "memory");
      *counter = 0u;                               // ready for the next epoch (stream-ordered)
    }
  }
}

__global__ void wait_kernel(const unsigned* __restrict__ flags, int rank, int world, unsigned epoch) {
  for (int r = rank + 1; r < world; ++r)
    while ((int)(ld_acquire_sys(flags + r) - epoch) < 0) __nanosleep(256);   // monotone epochs (wrap-safe)
  __threadfence_system();
}

// after this rank's reads of epoch `epoch` (ordered before on the stream):
// ack it in every later rank (writer) it read from
__global__ void ack_kernel(int rank, int world, unsigned* const* __restrict__ peer_acks, unsigned epoch) {
  __threadfence_system();
  for (int p = rank + 1; p < world; ++p)
    asm volatile("st.release.sys.global.u32 [%0], %1;\n" ::"l"(peer_acks[p] + rank), "r"(epoch) : "memory");
}

}  // namespace

cudaError_t launch_exchange_publish(const float* src, long long n, int rank, int world, float* const* peers,
                                    unsigned* const* peer_flags, unsigned* counter, const unsigned* acks,
                                    unsigned epoch, int num_sms, cudaStream_t st) {
  const long long want = (n + 255) / 256;
  const int grid = (int)std::max(1LL, std::min(want, 2LL * num_sms));
  publish_kernel<<<grid, 256, 0, st>>>(src, n, rank, world, peers, peer_flags, counter, acks, epoch);
  return cudaGetLastError();
}

cudaError_t launch_exchange_ack(int rank, int world, unsigned* const* peer_acks, unsigned epoch, cudaStream_t st) {
  ack_kernel<<<1, 1, 0, st>>>(rank, world, peer_acks, epoch);
  return cudaGetLastError();
}

cudaError_t launch_exchange_wait(const unsigned* flags, int rank, int world, unsigned epoch, cudaStream_t st) {
  wait_kernel<<<1, 1, 0, st>>>(flags, rank, world, epoch);
  return cudaGetLastError();
}

}  // namespace bppsa
