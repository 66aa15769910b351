// Microbenchmark (dev aid): cycles per tcgen05.mma kind::tf32 (M = 128,
// cta_group::1) for N in {64, 128, 256}, A from SMEM (SS) or TMEM (TS).
// One CTA per SM issues NB batches of 24 MMAs, commit + wait per batch
// (like the scan's per-step dependency) or a single commit at the end.
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

template <int N, bool TS>
__global__ void rate(int nbatch, int wait_each, long long* cycles) {
  extern __shared__ uint8_t smem_raw[];
  char* smem = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  for (int i = threadIdx.x; i < (128 + N) * 64; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 0.001f;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(&tslot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tslot;
  long long t0 = clock64();
  if (threadIdx.x < 32) {
    uint32_t ph = 0;
    for (int b = 0; b < nbatch; ++b) {
      if (threadIdx.x == 0) {
        for (int i = 0; i < 24; ++i) {
          const uint32_t boff = (uint32_t)(((i & 7) >> 2) * N * 128 + (i & 3) * 32);
          const uint32_t aoff = (uint32_t)(((i & 7) >> 2) * 128 * 128 + (i & 3) * 32);
          const uint32_t bsm = su32(smem + 128 * 256) + boff;
          if (TS) {
            asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                         " tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem),
                         "r"(tmem + 256 + 8 * (i & 7)), "l"(sdesc(bsm)), "r"(IDESC), "r"(i));
          } else {
            asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                         " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                         "l"(sdesc(su32(smem) + aoff)), "l"(sdesc(bsm)), "r"(IDESC), "r"(i));
          }
        }
        if (wait_each || b == nbatch - 1)
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
              su32(&bar)) : "memory");
      }
      __syncwarp();
      if (wait_each || b == nbatch - 1) {
        asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" ::"r"(
                         su32(&bar)), "r"(ph) : "memory");
        ph ^= 1;
      }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512));
}

template <int N, bool TS>
void run(long long* d) {
  const int smem = 128 * 256 + 256 * 256 + 1024 + 64;
  cudaFuncSetAttribute(rate<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int we = 0; we < 2; ++we) {
    const int nb = 2000;
    rate<N, TS><<<148, 128, smem>>>(nb, we, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return; }
    long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; ++i) avg += h[i];
    avg /= 148;
    printf("N=%3d %s wait_each=%d: %.1f cycles per MMA (%.0f per 24-batch)\n", N, TS ? "TS" : "SS", we,
           avg / (nb * 24.0), avg / nb);
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  run<64, false>(d);
  run<64, true>(d);
  run<128, false>(d);
  run<128, true>(d);
  run<256, false>(d);
  run<256, true>(d);
  return 0;
}
