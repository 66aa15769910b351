// Dev aid: tcgen05 kind::i8 MMA cost with INDEPENDENT accumulators.  The
// fold's 6 MMAs per step all accumulate into overlapping columns of one
// 256-column D (a dependent chain); tc_i8_probe.cu measured ~146-182 cycles
// per MMA for such chains whatever N.  This probe rotates D over R disjoint
// column ranges (MMA i -> D + (i % R) * N) to see whether independent
// accumulations pipeline, and times one 6-MMA batch issue -> commit.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/tc_i8_rate2.cu -o /tmp/r2 && /tmp/r2
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc64(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(512 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)4 << 61;
  return d;
}
// K-major SWIZZLE_128B: rows of 128 B, 8-row atoms of 1 KB
__device__ __forceinline__ uint64_t sdesc128(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t ph) {
  asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" ::"r"(
                   bar), "r"(ph) : "memory");
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, int acc) {
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
               "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_ss_f8(uint32_t d, uint64_t a, uint64_t b, uint32_t id, int acc) {
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
               "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_ss_f16(uint32_t d, uint64_t a, uint64_t b, uint32_t id, int acc) {
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
               "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, int acc) {
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
               "r"(a), "l"(b), "r"(id), "r"(acc));
}

__global__ void rate(int nbatch, int M, int N, int R, int nm, int ts, long long* cycles, int sw128, int zero, int kind) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 98304 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = zero ? 0u : (uint32_t)i * 2654435761u;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(su32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tslot;
  // f8f6f4: D f32 (bit 4), A/B e4m3 (format 0); f16: D f32, A/B f16 (format 0)
  const uint32_t id = (kind == 0 || kind == 3) ? idesc_i8(M, N) : ((1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24));
  const uint32_t bb = su32(smem), ab = su32(smem + 32768);
  // descriptors precomputed; 8 MMAs per batch, fully unrolled, one kind per launch
  uint64_t adv[2], bdv[2];
  for (int q = 0; q < 2; ++q) {
    adv[q] = sdesc64(ab + q * 32);
    bdv[q] = sdesc64(bb + q * 32);
  }
  long long t0 = clock64();
  if (threadIdx.x < 32) {
    uint32_t ph = 0;
    for (int b = 0; b < nbatch; ++b) {
      if (threadIdx.x == 0) {
        if (kind == 0) {
#pragma unroll
          for (int i = 0; i < 8; ++i) mma_ss(tmem, adv[i & 1], bdv[i & 1], id, i > 0);
        } else if (kind == 1) {
#pragma unroll
          for (int i = 0; i < 8; ++i) mma_ss_f8(tmem, adv[i & 1], bdv[i & 1], id, i > 0);
        } else if (kind == 2) {
#pragma unroll
          for (int i = 0; i < 8; ++i) mma_ss_f16(tmem, adv[i & 1], bdv[i & 1], id, i > 0);
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) mma_ts(tmem, tmem + 448 + 8 * (i & 1), bdv[i & 1], id, i > 0);
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
            su32(&bar)) : "memory");
      }
      __syncwarp();
      mbar_wait(su32(&bar), ph);
      ph ^= 1;
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

int main() {
  long long* dc;
  cudaMalloc(&dc, 148 * sizeof(long long));
  cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  auto run = [&](int N, int R, int nm, int ts, int nb, int sw128, int zero, int kind) {
    rate<<<148, 128, 100 * 1024>>>(nb, 128, N, R, nm, ts, dc, sw128, zero, kind);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); exit(1); }
    long long h[148];
    cudaMemcpy(h, dc, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; ++i) avg += h[i];
    avg /= 148;
    const char* kn[] = {"i8    ", "e4m3  ", "f16   ", "i8 TS "};
    printf("%s %s N=%3d nm=%2d: %7.1f cycles per MMA (K bytes 32), %7.1f per batch\n", kn[kind], ts ? "TS" : "SS", N,
           nm, avg / (nb * (double)nm), avg / nb);
  };
  for (int kind : {0, 1, 2, 3})
    for (int N : {64, 128, 256}) run(N, 1, 8, 0, 2000, 0, 1, kind);
  return 0;
}
