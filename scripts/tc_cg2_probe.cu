// Dev aid: validates the 2-CTA (cta_group::2) kind::f16 TS MMA used by the
// level-0 fold: cluster of 2, TMEM alloc cta_group::2, A (128 rows per CTA)
// in each CTA's TMEM, B = [W1 | W2] split along N (CTA0 holds W1, CTA1 W2),
// one leader thread issues M = 256, multicast commit to both CTAs.  Also the
// dispatch cost per MMA (M256 N128 K16) vs cta_group::1 M128 N128 K16.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/tc_cg2_probe.cu -o scripts/tc_cg2_probe.bin
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>
#include <cuda_fp16.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16; d |= (uint64_t)(1024 >> 4) << 32; d |= (uint64_t)1 << 46; d |= (uint64_t)2 << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) { return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24); }
__device__ __forceinline__ uint32_t sw16(int row, int k) {
  return (uint32_t)((row >> 3) * 1024 + (row & 7) * 128 + ((((k >> 3)) ^ (row & 7)) << 4) + (k & 7) * 2);
}
__device__ __forceinline__ uint32_t cta_rank() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t ph) {
  asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" ::"r"(bar), "r"(ph) : "memory");
}

__global__ void __cluster_dims__(2, 1, 1) probe(const float* X, const float* W, float* D, int nrep, long long* cyc) {
  extern __shared__ uint8_t smem_raw[];
  char* smem = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int t = threadIdx.x, warp = t >> 5;
  const uint32_t rank = cta_rank();
  // B half of this CTA: rank 0 rows n = W1[:, n], rank 1 rows n = W2[:, n] (n < 64), unscaled-ish test
  for (int e = t; e < 64 * 64; e += 128) {
    const int n = e / 64, k = e % 64;
    const float w = W[k * 64 + n] * 1024.f;
    const __half w1 = __float2half_rn(w);
    const __half w2 = __float2half_rn(w - __half2float(w1));
    *reinterpret_cast<__half*>(smem + sw16(n, k)) = rank == 0 ? w1 : w2;
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(su32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n" ::);
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tslot, lane_base = tmem + ((uint32_t)(warp * 32) << 16);
  // A: row t of this CTA (global row rank*128 + t), x1 / x2 split, scale 2^8
  const int grow = rank * 128 + t;
  uint32_t p1[32], p2[32];
  for (int c = 0; c < 32; ++c) {
    __half a1[2], a2[2];
    for (int h = 0; h < 2; ++h) {
      const float x = X[grow * 64 + 2 * c + h] * 256.f;
      a1[h] = __float2half_rn(x);
      a2[h] = __float2half_rn(x - __half2float(a1[h]));
    }
    p1[c] = (uint32_t)__half_as_ushort(a1[0]) | ((uint32_t)__half_as_ushort(a1[1]) << 16);
    p2[c] = (uint32_t)__half_as_ushort(a2[0]) | ((uint32_t)__half_as_ushort(a2[1]) << 16);
  }
  for (int c8 = 0; c8 < 4; ++c8) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(lane_base + 256 + 8 * c8),
                 "r"(p1[8 * c8]), "r"(p1[8 * c8 + 1]), "r"(p1[8 * c8 + 2]), "r"(p1[8 * c8 + 3]), "r"(p1[8 * c8 + 4]),
                 "r"(p1[8 * c8 + 5]), "r"(p1[8 * c8 + 6]), "r"(p1[8 * c8 + 7]) : "memory");
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(lane_base + 288 + 8 * c8),
                 "r"(p2[8 * c8]), "r"(p2[8 * c8 + 1]), "r"(p2[8 * c8 + 2]), "r"(p2[8 * c8 + 3]), "r"(p2[8 * c8 + 4]),
                 "r"(p2[8 * c8 + 5]), "r"(p2[8 * c8 + 6]), "r"(p2[8 * c8 + 7]) : "memory");
  }
  asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  long long t0 = clock64();
  uint32_t ph = 0;
  for (int rep = 0; rep < nrep; ++rep) {
    if (rank == 0 && t == 0) {
      int first = 1;
      for (int pass = 0; pass < 2; ++pass) {
        const uint32_t acol = pass == 0 ? 288 : 256;
        for (int kk = 0; kk < 4; ++kk) {
          asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                       " tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem),
                       "r"(tmem + acol + 8 * kk), "l"(sdesc(su32(smem) + 32 * kk)), "r"(idesc_f16(256, 128)), "r"(first ? 0 : 1));
          first = 0;
        }
      }
      asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n"
                   ::"r"(su32(&bar)), "h"((uint16_t)3) : "memory");
    }
    if (t == 0) mbar_wait(su32(&bar), ph);
    ph ^= 1;
    __syncthreads();
  }
  long long t1 = clock64();
  if (t == 0 && rank == 0 && blockIdx.x == 0) *cyc = t1 - t0;
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  for (int c8 = 0; c8 < 8; ++c8) {
    uint32_t a[8], b[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                 : "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3]), "=r"(a[4]), "=r"(a[5]), "=r"(a[6]), "=r"(a[7]) : "r"(lane_base + 8 * c8));
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                 : "=r"(b[0]), "=r"(b[1]), "=r"(b[2]), "=r"(b[3]), "=r"(b[4]), "=r"(b[5]), "=r"(b[6]), "=r"(b[7]) : "r"(lane_base + 64 + 8 * c8));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
    for (int i = 0; i < 8; ++i)
      D[(size_t)blockIdx.x / 2 * 0 + grow * 64 + 8 * c8 + i] = (__uint_as_float(a[i]) + __uint_as_float(b[i])) / (256.f * 1024.f);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  cluster_sync();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

int main() {
  std::mt19937 g(0);
  std::normal_distribution<float> nd;
  std::vector<float> X(256 * 64), W(64 * 64), D(256 * 64);
  for (auto& x : X) x = nd(g);
  for (auto& w : W) w = nd(g) / 8;
  float *dX, *dW, *dD;
  long long* dc;
  cudaMalloc(&dX, X.size() * 4); cudaMalloc(&dW, W.size() * 4); cudaMalloc(&dD, D.size() * 4); cudaMalloc(&dc, 8);
  cudaMemcpy(dX, X.data(), X.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dW, W.data(), W.size() * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
  for (int nrep : {1, 2000}) {
    probe<<<2, 128, 40 * 1024>>>(dX, dW, dD, nrep, dc);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    long long cyc;
    cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
    double worst = 0;
    for (int m = 0; m < 256; ++m) {
      double rowmax = 0, rowerr = 0;
      for (int n = 0; n < 64; ++n) {
        double ref = 0;
        for (int k = 0; k < 64; ++k) ref += (double)X[m * 64 + k] * W[k * 64 + n];
        rowmax = fmax(rowmax, fabs(ref));
        rowerr = fmax(rowerr, fabs(D[m * 64 + n] - ref));
      }
      worst = fmax(worst, rowerr / rowmax);
    }
    printf("nrep=%d: worst row rel err %.3e; %.1f cycles per 8-MMA batch (M256 N128 K16, wait each)\n", nrep, worst,
           (double)cyc / nrep);
  }
  return 0;
}
