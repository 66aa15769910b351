// Dev aid: which feature of the level-0 fold's MMA stream slows tcgen05 tf32
// (M = 128, N = 128, K = 8, TS) below ~64 cycles per MMA on B200.
//   bit 0: batches alternate between two D regions (cols 0 / 256), A lo/hi regions
//   bit 1: two batches in flight (wait for batch k-1 after issuing batch k)
//   bit 2: 24 other warps spin on mbarrier.try_wait meanwhile
//   bit 3: 24 other warps spin on a shared-memory flag (plain loads) meanwhile
//   bits 4-5: A operand data: 0 uninitialised TMEM, 1 normal N(0,1)-ish, 2 denormal (~1e-39), 3 zero
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/r3 scripts/tc_rate3.cu && /tmp/r3
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
__device__ __forceinline__ void wait_bar(uint32_t bar, uint32_t ph) {
  asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" ::"r"(
                   bar), "r"(ph) : "memory");
}

__global__ void rate(int nbatch, int mode, long long* cycles) {
  extern __shared__ uint8_t smem_raw[];
  char* smem = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar[2], never;
  __shared__ uint32_t tslot;
  __shared__ volatile int done;
  const int warp = threadIdx.x >> 5;
  const uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  for (int i = threadIdx.x; i < 128 * 64; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 0.001f * (i % 7);
  if (threadIdx.x == 0) {
    done = 0;
    for (int i = 0; i < 2; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(&bar[i])), "r"(1));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(&never)), "r"(1));
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
  const int adata = (mode >> 4) & 3;
  if (adata && warp < 4) {       // A regions: cols 128..255 and 384..511
    uint32_t s = 977u * threadIdx.x + 13u * blockIdx.x + 1u;
    const uint32_t lb = tmem + ((uint32_t)(warp * 32) << 16);
    for (int c = 0; c < 512; c += 8) {
      if ((c & 255) < 128) continue;
      uint32_t v[8];
      for (int k = 0; k < 8; ++k) {
        s = s * 1664525u + 1013904223u;
        const float r = ((s >> 8) / 16777216.f) * 2.f - 1.f;
        v[k] = __float_as_uint(adata == 1 ? r : adata == 2 ? r * 1e-39f : 0.f);
      }
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(lb + c),
                   "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]) : "memory");
    }
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  if (warp == 0) {
    long long t0 = clock64();
    uint32_t ph[2] = {0, 0};
    for (int b = 0; b < nbatch; ++b) {
      const int sl = (mode & 1) ? (b & 1) : 0;
      const uint32_t d = tmem + 256 * sl;
      if ((threadIdx.x & 31) == 0) {
        for (int i = 0; i < 16; ++i) {
          const int kk = i & 7, pq = i >> 3;
          const uint32_t boff = (uint32_t)(kk >> 2) * 128 * 128 + (kk & 3) * 32;
          const uint32_t a = (mode & 1) ? d + (pq ? 128 : 192) + 8 * kk : tmem + 128 + 8 * kk;
          asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                       " tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
                       "r"(a), "l"(sdesc(su32(smem) + boff)), "r"(IDESC), "r"(i));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                         su32(&bar[b & 1])) : "memory");
      }
      __syncwarp();
      const int wb = (mode & 2) ? b - 1 : b;           // batch to wait for
      if (wb >= 0) {
        wait_bar(su32(&bar[wb & 1]), ph[wb & 1]);
        ph[wb & 1] ^= 1;
      }
    }
    if (mode & 2) wait_bar(su32(&bar[(nbatch - 1) & 1]), ph[(nbatch - 1) & 1]);
    if ((threadIdx.x & 31) == 0) {
      cycles[blockIdx.x] = clock64() - t0;
      done = 1;
    }
  } else if (mode & 4) {
    while (!done) {
      uint32_t ok;
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                   : "=r"(ok) : "r"(su32(&never)), "r"(0u) : "memory");
    }
  } else if ((mode & 8) && (!(mode & 64) || (warp & 3) != 0)) {   // bit 6: spinners off the issuer's SMSP
    while (!done) {
    }
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
  const int modes[] = {16, 19 + 8, 19 + 8 + 64, 19 + 8, 19 + 8 + 64};
  const int nts[] = {1024, 1024, 1024, 512, 512};
  for (int mi = 0; mi < 5; ++mi) {
    const int mode = modes[mi], nt = nts[mi];
    const int nb = 4000;
    rate<<<148, nt, smem>>>(nb, mode, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; ++i) avg += h[i];
    avg /= 148;
    const char* dn[] = {"garbage", "normal", "denormal", "zero"};
    printf("threads %4d mode %2d (two-D %d, pipelined %d, mbar-spin %d, flag-spin %d%s, A %s): %.1f cycles per MMA\n", nt, mode, mode & 1,
           (mode >> 1) & 1, (mode >> 2) & 1, (mode >> 3) & 1, (mode & 64) ? " off-SMSP0" : "", dn[(mode >> 4) & 3], avg / (nb * 16.0));
  }
  return 0;
}
