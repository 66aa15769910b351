// exchange.cu — the carry exchange of the time-sharded scan (row a5, SURVEY
// 8(e)) over peer memory instead of an NCCL all-gather: each rank stores its
// up-sweep aggregate straight into every rank's mailbox (P2P stores over
// NVLink / NVSwitch; CUDA IPC mappings) and raises a per-rank flag there with
// a system-scope release; a rank's down-sweep starts after an acquire wait on
// the flags of the later ranks, whose aggregates its carry needs.
// Mailbox of a rank: [2][world][n] floats (epoch parity double buffer: a rank
// may run at most one epoch ahead of a reader), flags [world] u32 (the last
// published epoch per sender, monotone).
#include "common.cuh"

namespace bppsa {
namespace {

__global__ void publish_kernel(const float* __restrict__ src, long long n, int rank, int world,
                               float* const* __restrict__ peers, unsigned* const* __restrict__ peer_flags,
                               unsigned* __restrict__ counter, unsigned epoch) {
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
  for (int r = rank + 1; r < world; ++r) {
    unsigned v;
    while (true) {
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];\n" : "=r"(v) : "l"(flags + r) : "memory");
      if ((int)(v - epoch) >= 0) break;            // monotone epochs (wrap-safe)
      __nanosleep(256);
    }
  }
  __threadfence_system();
}

}  // namespace

cudaError_t launch_exchange_publish(const float* src, long long n, int rank, int world, float* const* peers,
                                    unsigned* const* peer_flags, unsigned* counter, unsigned epoch, int num_sms,
                                    cudaStream_t st) {
  const long long want = (n + 255) / 256;
  const int grid = (int)std::max(1LL, std::min(want, 2LL * num_sms));
  publish_kernel<<<grid, 256, 0, st>>>(src, n, rank, world, peers, peer_flags, counter, epoch);
  return cudaGetLastError();
}

cudaError_t launch_exchange_wait(const unsigned* flags, int rank, int world, unsigned epoch, cudaStream_t st) {
  wait_kernel<<<1, 1, 0, st>>>(flags, rank, world, epoch);
  return cudaGetLastError();
}

}  // namespace bppsa
