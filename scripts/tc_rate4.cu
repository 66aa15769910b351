// Dev aid: does tcgen05.commit cost tensor-pipe time?  One CTA per SM issues
// 64000 TS MMAs (M = 128, N = 128, K = 8, tf32) with a commit every C MMAs
// (C = 8 .. 64000) and never waits except at the end.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/r4 scripts/tc_rate4.cu && /tmp/r4
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

__global__ void rate(int total, int every, int dual, long long* cycles) {
  extern __shared__ uint8_t smem_raw[];
  char* smem = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  const uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  for (int i = threadIdx.x; i < 128 * 64; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 0.001f * (i % 7);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(&tslot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    long long t0 = clock64();
    int ncommit = 0;
    for (int i = 0; i < total; ++i) {
      const int kk = i & 7;
      const uint32_t d = dual ? tmem + 256 * ((i / every) & 1) : tmem;   // alternate D regions per batch
      const uint32_t boff = (uint32_t)(kk >> 2) * 128 * 128 + (kk & 3) * 32;
      asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                   " tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
                   "r"(d + 128 + 8 * kk), "l"(sdesc(su32(smem) + boff)), "r"(IDESC), "r"(i % every));
      if ((i + 1) % every == 0 && i + 1 < total) {
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(&bar))
                     : "memory");
        ++ncommit;
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(&bar))
                 : "memory");
    ++ncommit;
    // wait for the final phase: the barrier completes once per commit (count 1)
    const uint32_t ph = (ncommit - 1) & 1;
    asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" ::"r"(
                     su32(&bar)), "r"(ph) : "memory");
    cycles[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512));
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  const int smem = 128 * 64 * 4 + 2048;
  cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int total = 64000;
  const int evs[] = {8, 16, 32, 64, 256, 64000};
  for (int dual = 0; dual < 2; ++dual)
    for (int every : evs) {
      rate<<<148, 128, smem>>>(total, every, dual, d);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      long long h[148];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      double avg = 0;
      for (int i = 0; i < 148; ++i) avg += h[i];
      avg /= 148;
      printf("commit every %5d MMAs, %s D: %.1f cycles per MMA\n", every, dual ? "alternating" : "single", avg / total);
    }
  return 0;
}
