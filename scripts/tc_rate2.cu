// Dev aid: cycles per tcgen05.mma kind::tf32 (M = 128, N = 128, K = 8, TS form)
// on all 148 SMs under (a) constant vs random operands and (b) concurrent
// tcgen05.ld / tcgen05.st traffic from 8 other warps on disjoint TMEM columns.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/r2 scripts/tc_rate2.cu && /tmp/r2
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
__device__ __forceinline__ float frand(uint32_t& s) {
  s = s * 1664525u + 1013904223u;
  return ((s >> 8) / 16777216.f) * 2.f - 1.f;
}

// mode bit 0: random operands; bit 1: TMEM ld/st traffic; bit 2: exact-zero lo-like tiny values
__global__ void rate(int nbatch, int mode, long long* cycles) {
  extern __shared__ uint8_t smem_raw[];
  char* smem = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  __shared__ volatile int done;
  const int warp = threadIdx.x >> 5;
  const uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  uint32_t s = 12345u + threadIdx.x * 7919u + blockIdx.x * 104729u;
  for (int i = threadIdx.x; i < 128 * 64; i += blockDim.x)
    reinterpret_cast<float*>(smem)[i] = (mode & 1) ? frand(s) : 0.001f;
  if (threadIdx.x == 0) {
    done = 0;
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
  // A operand (cols 128..191) written by warps 0..3 (one lane quarter each)
  if (warp < 4) {
    const uint32_t lb = tmem + ((uint32_t)(warp * 32) << 16);
    for (int c = 0; c < 64; c += 8) {
      uint32_t v[8];
      for (int k = 0; k < 8; ++k) v[k] = __float_as_uint((mode & 1) ? frand(s) : 0.001f);
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(lb + 128 + c),
                   "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]) : "memory");
    }
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  if (warp == 8) {
    long long t0 = clock64();
    uint32_t ph = 0;
    for (int b = 0; b < nbatch; ++b) {
      if ((threadIdx.x & 31) == 0) {
        for (int i = 0; i < 16; ++i) {
          const uint32_t boff = (uint32_t)((i & 7) >> 2) * 128 * 128 + (i & 3) * 32;
          asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                       " tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem),
                       "r"(tmem + 128 + 8 * (i & 7)), "l"(sdesc(su32(smem) + boff)), "r"(IDESC), "r"(i));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(&bar))
                     : "memory");
      }
      __syncwarp();
      asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" ::"r"(
                       su32(&bar)), "r"(ph) : "memory");
      ph ^= 1;
    }
    if ((threadIdx.x & 31) == 0) {
      done = 1;
      cycles[blockIdx.x] = clock64() - t0;
    }
  } else if ((mode & 2) && warp < 8) {
    // traffic on cols 256..511 (disjoint from D [0,128) and A [128,192))
    const uint32_t lb = tmem + ((uint32_t)((warp & 3) * 32) << 16) + 256 + 128 * (warp >> 2);
    uint32_t v[32];
    for (int k = 0; k < 32; ++k) v[k] = k;
    while (!done) {
      for (int c = 0; c < 128; c += 32) {
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
            : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]), "+r"(v[7]),
              "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]), "+r"(v[12]), "+r"(v[13]), "+r"(v[14]), "+r"(v[15]),
              "+r"(v[16]), "+r"(v[17]), "+r"(v[18]), "+r"(v[19]), "+r"(v[20]), "+r"(v[21]), "+r"(v[22]), "+r"(v[23]),
              "+r"(v[24]), "+r"(v[25]), "+r"(v[26]), "+r"(v[27]), "+r"(v[28]), "+r"(v[29]), "+r"(v[30]), "+r"(v[31])
            : "r"(lb + c));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        for (int k = 0; k < 32; ++k) v[k] += 1;
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
            "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};\n" ::"r"(lb + c),
            "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
            "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
            "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
            "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]) : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
      }
    }
  }
  __syncthreads();
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512));
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  const int smem = 128 * 64 * 4 + 2048;
  cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names[] = {"const", "random", "const+traffic", "random+traffic"};
  for (int rep = 0; rep < 2; ++rep)
    for (int mode = 0; mode < 4; ++mode) {
      const int nb = 4000;
      rate<<<148, 288, smem>>>(nb, mode, d);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      long long h[148];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      double avg = 0;
      for (int i = 0; i < 148; ++i) avg += h[i];
      avg /= 148;
      printf("%-15s: %.1f cycles per MMA\n", names[mode], avg / (nb * 16.0));
    }
  return 0;
}
