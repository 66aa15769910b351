// Standalone probe (dev aid) of the kind::f16 tcgen05 path for the level-0
// fold: (1) the TMEM layout of a 16-bit A operand (TS form) and the accuracy
// of a row-scaled 2-term fp16 split (x = x1 + x2, W = W1 + W2, D = x1 W1 +
// x1 W2 + x2 W1 (+ x2 W2)) against fp64; (2) cycles per MMA for M = 128,
// K = 16, N in {64, 128, 256}, A in TMEM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/tc_f16_probe.cu -o /tmp/tc_f16_probe
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>

#include <cuda_fp16.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc_f16(int N) { return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24); }
// K-major SWIZZLE_128B tile of fp16 with K = 64 (one 128-byte row per N row)
__device__ __forceinline__ uint32_t sw16(int row, int k) {
  return (uint32_t)((row >> 3) * 1024 + (row & 7) * 128 + ((((k >> 3)) ^ (row & 7)) << 4) + (k & 7) * 2);
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(taddr), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float (&v)[8]) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t ph) {
  asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" ::"r"(
                   bar), "r"(ph) : "memory");
}

// variant bit 0: swap the two halves of each packed 32-bit column; bit 1: skip the x2 pass
__global__ void probe(const float* X, const float* W, float* D, int variant) {
  extern __shared__ uint8_t smem_raw[];
  char* smem = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  __shared__ int sw_s;
  const int t = threadIdx.x, warp = t >> 5;
  if (t == 0) {
    float m = 0.f;
    for (int i = 0; i < 64 * 64; ++i) m = fmaxf(m, fabsf(W[i]));
    int e;
    frexpf(m, &e);       // m = f 2^e, f in [0.5, 1)
    sw_s = 14 - e;       // max |W| 2^sw in [2^13, 2^14)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const int sw = sw_s;
  // B rows 0..63 = W1[:, n], 64..127 = W2[:, n]
  for (int e = t; e < 64 * 64; e += 128) {
    const int n = e / 64, k = e % 64;
    const float w = ldexpf(W[k * 64 + n], sw);
    const __half w1 = __float2half_rn(w);
    const __half w2 = __float2half_rn(w - __half2float(w1));
    *reinterpret_cast<__half*>(smem + sw16(n, k)) = w1;
    *reinterpret_cast<__half*>(smem + sw16(64 + n, k)) = w2;
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(su32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tslot, lane_base = tmem + ((uint32_t)(warp * 32) << 16);
  // row t: scale, split, pack into TMEM A1 (cols 256..287) / A2 (288..319)
  float m = 0.f;
  for (int k = 0; k < 64; ++k) m = fmaxf(m, fabsf(X[t * 64 + k]));
  int e;
  frexpf(m, &e);
  const int s = 14 - e;
  uint32_t p1[32], p2[32];
  for (int c = 0; c < 32; ++c) {
    __half a1[2], a2[2];
    for (int h = 0; h < 2; ++h) {
      const float x = ldexpf(X[t * 64 + 2 * c + h], s);
      a1[h] = __float2half_rn(x);
      a2[h] = __float2half_rn(x - __half2float(a1[h]));
    }
    const int lo = (variant & 1) ? 1 : 0;
    p1[c] = (uint32_t)__half_as_ushort(a1[lo]) | ((uint32_t)__half_as_ushort(a1[1 - lo]) << 16);
    p2[c] = (uint32_t)__half_as_ushort(a2[lo]) | ((uint32_t)__half_as_ushort(a2[1 - lo]) << 16);
  }
  for (int c8 = 0; c8 < 4; ++c8) {
    uint32_t r1[8], r2[8];
    for (int i = 0; i < 8; ++i) r1[i] = p1[8 * c8 + i], r2[i] = p2[8 * c8 + i];
    tmem_st8(lane_base + 256 + 8 * c8, r1);
    tmem_st8(lane_base + 288 + 8 * c8, r2);
  }
  asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  if (t == 0) {
    const uint32_t bsm = su32(smem);
    int first = 1;
    for (int pass = (variant & 2) ? 1 : 0; pass < 2; ++pass) {     // x2 (corrections) first, then x1
      const uint32_t acol = pass == 0 ? 288 : 256;
      for (int kk = 0; kk < 4; ++kk) {
        asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                     " tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem),
                     "r"(tmem + acol + 8 * kk), "l"(sdesc(bsm + 32 * kk)), "r"(idesc_f16(128)), "r"(first ? 0 : 1));
        first = 0;
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(&bar))
                 : "memory");
  }
  __syncwarp();
  mbar_wait(su32(&bar), 0);
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  for (int c8 = 0; c8 < 8; ++c8) {
    float a[8], b[8];
    tmem_ld8(lane_base + 8 * c8, a);
    tmem_ld8(lane_base + 64 + 8 * c8, b);
    for (int i = 0; i < 8; ++i) D[t * 64 + 8 * c8 + i] = ldexpf(a[i] + b[i], -(s + sw));
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

template <int N>
__global__ void rate(int nbatch, int wait_each, long long* cycles, int pattern = 0) {
  extern __shared__ uint8_t smem_raw[];
  char* smem = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  // operand patterns: 0 = constants, 1 = A random normal halves, 2 = A random incl. subnormal halves,
  // 3 = A and B random normal, 4 = A and B incl. subnormals
  for (int i = threadIdx.x; i < N * 32; i += blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u;
    uint32_t bn = ((h >> 3) & 0x03FF03FFu) | 0x3C003C00u;          // normal halves in [1, 2)
    uint32_t bs = (h & 0x83FF83FFu);                                // subnormal halves
    reinterpret_cast<uint32_t*>(smem)[i] = pattern == 3 ? bn : (pattern == 4 ? ((i & 1) ? bs : bn) : 0x1c001c00u);
  }
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
  if (pattern != 0) {
    const uint32_t lb = tmem + ((uint32_t)((threadIdx.x >> 5) * 32) << 16);
    for (int c = 0; c < 64; ++c) {
      uint32_t h = (uint32_t)(threadIdx.x * 64 + c) * 2246822519u;
      uint32_t v = ((h >> 3) & 0x03FF03FFu) | 0x3C003C00u;
      if (pattern == 2 || pattern == 4) v = (c & 1) ? (h & 0x83FF83FFu) : v;
      asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};\n" ::"r"(lb + 256 + c), "r"(v) : "memory");
    }
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  }
  long long t0 = clock64();
  if (threadIdx.x < 32) {
    uint32_t ph = 0;
    for (int b = 0; b < nbatch; ++b) {
      if (threadIdx.x == 0) {
        // pattern 20: alternate two slots (D at 0 / 256, A at 128 / 384) like the fold kernel
        const uint32_t dbase = (pattern == 20 && (b & 1)) ? 256u : 0u;
        const uint32_t abase = pattern == 20 ? dbase + 128u : (pattern >= 10 ? 128u : 256u);
        for (int i = 0; i < 8; ++i) {
          asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                       " tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem + dbase),
                       "r"(tmem + abase + 8 * (i & 3) + 32 * (i >> 2)), "l"(sdesc(su32(smem) + 32 * (i & 3))), "r"(idesc_f16(N)),
                       "r"(i));
        }
        if (wait_each || b == nbatch - 1)
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
              su32(&bar)) : "memory");
      }
      __syncwarp();
      if (wait_each || b == nbatch - 1) {
        mbar_wait(su32(&bar), ph);
        ph ^= 1;
      }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

template <int N>
void run_rate(long long* d, int pattern = 0) {
  const int smem = 256 * 128 + 2048;
  cudaFuncSetAttribute(rate<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  printf("pattern %d: ", pattern);
  for (int we = 0; we < 2; ++we) {
    const int nb = 4000;
    rate<N><<<148, 128, smem>>>(nb, we, d, pattern);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return; }
    long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; ++i) avg += h[i];
    avg /= 148;
    printf("f16 TS N=%3d K=16 wait_each=%d: %.1f cycles per MMA (%.0f per 8-batch)\n", N, we, avg / (nb * 8.0),
           avg / nb);
  }
}

int main() {
  std::mt19937 g(0);
  std::normal_distribution<float> nd;
  std::vector<float> X(128 * 64), W(64 * 64), D(128 * 64);
  float *dX, *dW, *dD;
  cudaMalloc(&dX, X.size() * 4);
  cudaMalloc(&dW, W.size() * 4);
  cudaMalloc(&dD, D.size() * 4);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
  for (int data = 0; data < 0; ++data) {
    for (int m = 0; m < 128; ++m) {
      // rows of wildly different magnitudes: per-row scaling must absorb them
      const float rs = data == 0 ? 1.f : (data == 1 ? ldexpf(1.f, (m % 41) * 7 - 140) : 1e-3f);
      for (int k = 0; k < 64; ++k) X[m * 64 + k] = nd(g) * rs * (data == 2 && k % 5 == 0 ? 1e-6f : 1.f);
    }
    for (auto& w : W) w = nd(g) / 8;
    cudaMemcpy(dX, X.data(), X.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dW, W.data(), W.size() * 4, cudaMemcpyHostToDevice);
    for (int variant : {0, 1, 2}) {
      probe<<<1, 128, 40 * 1024>>>(dX, dW, dD, variant);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
      double worst = 0, bias = 0;
      long cnt = 0;
      for (int m = 0; m < 128; ++m) {
        double rowmax = 0, rowerr = 0;
        for (int n = 0; n < 64; ++n) {
          double ref = 0, absr = 0;
          for (int k = 0; k < 64; ++k) ref += (double)X[m * 64 + k] * W[k * 64 + n];
          for (int k = 0; k < 64; ++k) absr += fabs((double)X[m * 64 + k] * W[k * 64 + n]);
          rowmax = fmax(rowmax, fabs(ref));
          rowerr = fmax(rowerr, fabs(D[m * 64 + n] - ref));
          if (ref != 0) {
            bias += (D[m * 64 + n] - ref) / fabs(ref) * (ref > 0 ? 1 : -1);
            ++cnt;
          }
        }
        if (rowmax > 0) worst = fmax(worst, rowerr / rowmax);
      }
      printf("data=%d variant=%d (swap=%d, no_x2=%d): worst row max-norm rel err %.3e  bias %.2f ulp\n", data,
             variant, variant & 1, (variant >> 1) & 1, worst, bias / cnt / 5.96e-8);
    }
  }
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  for (int pat : {0, 10, 20}) run_rate<128>(d, pat);
  return 0;
}
