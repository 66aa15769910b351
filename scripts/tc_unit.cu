// Standalone precision probe of one tcgen05 kind::tf32 step (dev aid):
// D = X W with X, W split hi/lo; variants: 1 = hi*hi, 3 = 3xTF32.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include scripts/tc_unit.cu -o /tmp/tc_unit
#include <cstdio>
#include <cmath>
#include <vector>
#include <random>

#include "../paper_1907_10134_b200/csrc/tc_leaf.cu"

namespace bppsa {
namespace {
__global__ void probe(const float* X, const float* W, float* D, int variant, int split_mode) {
  extern __shared__ uint8_t smem_raw[];
  char* smem = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int t = threadIdx.x, warp = t >> 5;
  char* Ahi = smem;
  char* Alo = smem + A_BYTES;
  char* Bhi = smem + 2 * A_BYTES;
  char* Blo = Bhi + B_BYTES;
  for (int k = 0; k < 64; ++k) {
    const float x = X[t * 64 + k];
    float hi = tf32_rn(x), lo = x - hi;
    if (split_mode == 1) lo = tf32_rn(lo);
    *reinterpret_cast<float*>(Ahi + sw_off(t, k, TM)) = hi;
    *reinterpret_cast<float*>(Alo + sw_off(t, k, TM)) = lo;
  }
  if (t < 64)
    for (int k = 0; k < 64; ++k) {
      const float w = W[k * 64 + t];
      float hi = tf32_rn(w), lo = w - hi;
      if (split_mode == 1) lo = tf32_rn(lo);
      *reinterpret_cast<float*>(Bhi + sw_off(t, k, TH)) = hi;
      *reinterpret_cast<float*>(Blo + sw_off(t, k, TH)) = lo;
    }
  if (t == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(&tslot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  // variant: 1 = hi*hi only; 3 = hi*hi, hi*lo, lo*hi in one accumulator;
  //          4 = corrections first then hi*hi; 5 = every MMA into its own accumulator, fp32 RN sum
  float acc[64];
  for (int n = 0; n < 64; ++n) acc[n] = 0.f;
  const uint32_t a_hi = su32(Ahi), a_lo = su32(Alo), b_hi = su32(Bhi), b_lo = su32(Blo);
  int nround = (variant == 5) ? 3 : 1;
  uint32_t phase = 0;
  for (int round = 0; round < nround; ++round) {
    if (t == 0) {
      if (variant == 5) {
        const uint32_t aa = (round == 2) ? a_lo : a_hi, bb = (round == 1) ? b_lo : b_hi;
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t aoff = (uint32_t)((kk >> 2) * TM * 128 + (kk & 3) * 32);
          const uint32_t boff = (uint32_t)((kk >> 2) * TH * 128 + (kk & 3) * 32);
          mma_tf32(tmem + kk * 64, sdesc(aa + aoff), sdesc(bb + boff), 0);
        }
      } else {
        const int order3[3] = {0, 1, 2}, order4[3] = {1, 2, 0};
        const int np = variant == 1 ? 1 : 3;
        for (int i = 0; i < np; ++i) {
          const int pq = (variant == 4) ? order4[i] : order3[i];
          const uint32_t aa = (pq == 2) ? a_lo : a_hi, bb = (pq == 1) ? b_lo : b_hi;
          for (int kk = 0; kk < 8; ++kk) {
            const uint32_t aoff = (uint32_t)((kk >> 2) * TM * 128 + (kk & 3) * 32);
            const uint32_t boff = (uint32_t)((kk >> 2) * TH * 128 + (kk & 3) * 32);
            mma_tf32(tmem, sdesc(aa + aoff), sdesc(bb + boff), (i | kk) != 0);
          }
        }
      }
      mma_commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, phase);
    phase ^= 1;
    tc_fence_after();
    const int nacc = (variant == 5) ? 8 : 1;
    for (int a = 0; a < nacc; ++a) {
      float v[64];
      tmem_ld64(tmem + ((uint32_t)(warp * 32) << 16) + a * 64, v);
      for (int n = 0; n < 64; ++n) acc[n] += v[n];
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }
  for (int n = 0; n < 64; ++n) D[t * 64 + n] = acc[n];
  tc_fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512));
}
}  // namespace
}  // namespace bppsa

int main() {
  std::mt19937 g(0);
  std::normal_distribution<float> nd;
  std::uniform_real_distribution<float> ud(0.5f, 1.0f);
  std::vector<float> X(128 * 64), W(64 * 64), D(128 * 64);
  float *dX, *dW, *dD;
  cudaMalloc(&dX, X.size() * 4);
  cudaMalloc(&dW, W.size() * 4);
  cudaMalloc(&dD, D.size() * 4);
  cudaFuncSetAttribute(bppsa::probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024);
  for (int pos = 0; pos < 2; ++pos) {
    for (auto& x : X) x = pos ? ud(g) : nd(g);
    for (auto& w : W) w = (pos ? ud(g) : nd(g)) / 8;
    cudaMemcpy(dX, X.data(), X.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dW, W.data(), W.size() * 4, cudaMemcpyHostToDevice);
    for (int variant : {1, 3, 4, 5}) {
      bppsa::probe<<<1, 128, 120 * 1024>>>(dX, dW, dD, variant, 1);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
      double maxerr = 0, maxref = 0, bias = 0;
      for (int m = 0; m < 128; ++m)
        for (int n = 0; n < 64; ++n) {
          double ref = 0;
          for (int k = 0; k < 64; ++k) ref += (double)X[m * 64 + k] * W[k * 64 + n];
          maxerr = fmax(maxerr, fabs(D[m * 64 + n] - ref));
          maxref = fmax(maxref, fabs(ref));
          bias += (D[m * 64 + n] - ref) / fabs(ref) * (ref > 0 ? 1 : -1);
        }
      printf("data=%s variant=%d: max rel err %.3e  mean signed rel err (bias) %.3e (ulp units %.2f)\n",
             pos ? "positive" : "gaussian", variant, maxerr / maxref, bias / (128 * 64),
             bias / (128 * 64) / 5.96e-8);
    }
  }
  return 0;
}
