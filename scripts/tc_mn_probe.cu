// Dev aid: tcgen05 kind::tf32 with BOTH operands MN-major in shared memory
// (SWIZZLE_128B MN-major atoms: 8 K-rows x 128 B = 32 elements along M/N;
// atoms along M/N at LBO = 1024 B; one MMA (K = 8) per atom row, the next K
// group by advancing the start address by 4096 B).  D[m][n] = sum_k A[m][k]
// B[n][k], M = N = 128, K = 32, small integers -> exact; compared on the host.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/tc_mn_probe.cu -o /tmp/mn && /tmp/mn
#include <cstdint>
#include <cstdio>
#include <vector>
#include <cuda_fp16.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
// byte offset of (mn, k) in an MN-major SW128 tile of MN = 128, K = 32 (fp32)
__host__ __device__ inline uint32_t mn_off(int mn, int k) {
  const int atom = mn >> 5, kg = k >> 3, r = k & 7, chunk = (mn & 31) >> 2;
  return (uint32_t)(kg * 4096 + atom * 1024 + r * 128 + ((chunk ^ r) << 4) + (mn & 3) * 4);
}
// K-major SW128 (the wgrad kernel's B layout): rows of 128 B = 32 K-elements
__host__ __device__ inline uint32_t k_off(int mn, int k) {
  return (uint32_t)((mn >> 3) * 1024 + (mn & 7) * 128 + ((((k & 31) >> 2) ^ (mn & 7)) << 4) + (k & 3) * 4);
}
// MN-major SWIZZLE_NONE: core matrices of 8 K-rows x 16 B (4 elements along MN)
__host__ __device__ inline uint32_t mn_off_i(int mn, int k) {
  return (uint32_t)((mn >> 2) * 128 + (k >> 3) * 4096 + (k & 7) * 16 + (mn & 3) * 4);
}
__device__ __forceinline__ uint64_t sdesc_mn(uint32_t saddr, uint32_t lbo, uint32_t sbo, int swz = 2) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)swz << 61;   // 2 = SWIZZLE_128B, 0 = none
  return d;
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t ph) {
  asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" ::"r"(
                   bar), "r"(ph) : "memory");
}

__global__ void probe(const float* A, const float* B, float* D, uint32_t lbo, uint32_t sbo, int amaj, int bmaj, uint32_t kstep) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  float* sA = reinterpret_cast<float*>(smem);
  float* sB = reinterpret_cast<float*>(smem + 16384);
  for (int e = threadIdx.x; e < 128 * 32; e += blockDim.x) {
    const int mn = e / 32, k = e % 32;
    sA[(amaj == 2 ? mn_off_i(mn, k) : amaj ? mn_off(mn, k) : k_off(mn, k)) / 4] = A[mn * 32 + k];
    sB[(bmaj == 2 ? mn_off_i(mn, k) : bmaj ? mn_off(mn, k) : k_off(mn, k)) / 4] = B[mn * 32 + k];
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;\n" ::"r"(su32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tslot;
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(amaj != 0) << 15) | ((uint32_t)(bmaj != 0) << 16) |
                         ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  if (threadIdx.x == 0) {
    for (int kg = 0; kg < 4; ++kg) {
      const uint64_t ad = amaj == 2 ? sdesc_mn(su32(sA) + kg * 4096, lbo, sbo, 0)
                          : amaj ? sdesc_mn(su32(sA) + kg * kstep, lbo, sbo) : sdesc_mn(su32(sA) + kg * 32, 16, 1024);
      const uint64_t bd = bmaj == 2 ? sdesc_mn(su32(sB) + kg * 4096, lbo, sbo, 0)
                          : bmaj ? sdesc_mn(su32(sB) + kg * kstep, lbo, sbo) : sdesc_mn(su32(sB) + kg * 32, 16, 1024);
      asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(
                       tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(kg));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(&bar)) : "memory");
  }
  __syncwarp();
  if (threadIdx.x % 32 == 0) mbar_wait(su32(&bar), 0);
  __syncwarp();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int c = 0; c < 128; ++c) {
    uint32_t v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];\n" : "=r"(v) : "r"(tmem + ((uint32_t)(32 * w) << 16) + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
    D[(32 * w + lane) * 128 + c] = __uint_as_float(v);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;\n" ::"r"(tmem));
}


// ---- kind::f16, MN-major SW128: atom = 64 halves (128 B) along M/N x 8 K-rows;
// K = 16 per MMA = 2 K-groups at SBO; atoms along M/N at LBO
__host__ __device__ inline uint32_t mn16_off(int mn, int k, uint32_t lbo, uint32_t sbo) {
  const int atom = mn >> 6, kg = k >> 3, r = k & 7, chunk = (mn & 63) >> 3;
  return (uint32_t)(kg * sbo + atom * lbo + r * 128 + ((chunk ^ r) << 4) + (mn & 7) * 2);
}
__global__ void probe16(const float* A, const float* B, float* D, uint32_t lbo, uint32_t sbo) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  __half* sA = reinterpret_cast<__half*>(smem);
  __half* sB = reinterpret_cast<__half*>(smem + 16384);
  for (int e = threadIdx.x; e < 128 * 32; e += blockDim.x) {
    const int mn = e / 32, k = e % 32;
    sA[mn16_off(mn, k, lbo, sbo) / 2] = __float2half(A[mn * 32 + k]);
    sB[mn16_off(mn, k, lbo, sbo) / 2] = __float2half(B[mn * 32 + k]);
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;\n" ::"r"(su32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tslot;
  // D f32, A/B f16 (format 0), both MN-major (bits 15, 16), N = M = 128
  const uint32_t idesc = (1u << 4) | (1u << 15) | (1u << 16) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  if (threadIdx.x == 0) {
    for (int ks = 0; ks < 2; ++ks) {
      const uint64_t ad = sdesc_mn(su32(sA) + ks * 2 * sbo, lbo, sbo), bd = sdesc_mn(su32(sB) + ks * 2 * sbo, lbo, sbo);
      asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(
                       tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(ks));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(&bar)) : "memory");
  }
  __syncwarp();
  if (threadIdx.x % 32 == 0) mbar_wait(su32(&bar), 0);
  __syncwarp();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int c = 0; c < 128; ++c) {
    uint32_t v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];\n" : "=r"(v) : "r"(tmem + ((uint32_t)(32 * w) << 16) + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
    D[(32 * w + lane) * 128 + c] = __uint_as_float(v);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;\n" ::"r"(tmem));
}

int main() {
  std::vector<float> A(128 * 32), B(128 * 32), D(128 * 128);
  uint32_t s = 12345;
  auto rnd = [&]() { s = s * 1664525u + 1013904223u; return (float)((int)(s >> 24) % 17 - 8); };
  for (auto& v : A) v = rnd();
  for (auto& v : B) v = rnd();
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
  struct Cfg { uint32_t lbo, sbo; int am, bm; uint32_t kstep; } cfgs[] = {
      {0, 0, 0, 0, 0}, {1024, 4096, 1, 0, 4096}, {4096, 1024, 1, 0, 4096}, {1024, 4096, 0, 1, 4096},
      {4096, 1024, 0, 1, 4096}, {1024, 4096, 1, 1, 4096}, {4096, 1024, 1, 1, 4096}, {1024, 128, 1, 1, 4096},
      {4096, 128, 2, 0, 0}, {128, 4096, 2, 0, 0}, {4096, 128, 0, 2, 0}, {128, 4096, 0, 2, 0}};
  for (auto c : cfgs) {
    cudaMemset(dD, 0, D.size() * 4);
    probe<<<1, 128, 40 * 1024>>>(dA, dB, dD, c.lbo, c.sbo, c.am, c.bm, c.kstep);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    long bad = 0;
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < 128; ++n) {
        double r = 0;
        for (int k = 0; k < 32; ++k) r += (double)A[m * 32 + k] * B[n * 32 + k];
        if (r != D[m * 128 + n]) ++bad;
      }
    printf("A %s B %s LBO=%u SBO=%u: %s (%ld mismatches) D00 %g want %g\n", c.am == 2 ? "MNi" : c.am ? "MN" : "K",
           c.bm == 2 ? "MNi" : c.bm ? "MN" : "K", c.lbo, c.sbo, bad ? "FAIL" : "exact", bad, D[0], [&] {
             double r = 0; for (int k = 0; k < 32; ++k) r += (double)A[k] * B[k]; return r; }());
  }
  cudaFuncSetAttribute(probe16, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
  struct C16 { uint32_t lbo, sbo; } c16s[] = {{1024, 2048}, {2048, 1024}, {1024, 4096}, {4096, 1024}};
  for (auto c : c16s) {
    cudaMemset(dD, 0, D.size() * 4);
    probe16<<<1, 128, 40 * 1024>>>(dA, dB, dD, c.lbo, c.sbo);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    long bad = 0;
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < 128; ++n) {
        double r = 0;
        for (int k = 0; k < 32; ++k) r += (double)A[m * 32 + k] * B[n * 32 + k];
        if (r != D[m * 128 + n]) ++bad;
      }
    printf("f16 A MN B MN LBO=%u SBO=%u: %s (%ld mismatches) D00 %g\n", c.lbo, c.sbo, bad ? "FAIL" : "exact", bad, D[0]);
  }
  return 0;
}
