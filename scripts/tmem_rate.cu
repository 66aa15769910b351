// Dev aid: tcgen05.ld / tcgen05.st cost per warp-instruction with 32 warps on
// one CTA per SM, alone and while warp 0 keeps the tensor pipe busy with
// kind::f16 TS MMAs (M128 N128 K16, A in TMEM).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/tmem_rate.bin scripts/tmem_rate.cu
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16; d |= (uint64_t)(1024 >> 4) << 32; d |= (uint64_t)1 << 46; d |= (uint64_t)2 << 61;
  return d;
}
// mode bit0: ld (else st); bit1: concurrent MMAs; bit2: x16 shape (else x8/x4)
__global__ void k(int mode, int iters, long long* out) {
  extern __shared__ uint8_t smem_raw[];
  char* smem = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  __shared__ volatile int stop;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 128 * 32; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x1c001c00u;
  if (threadIdx.x == 0) {
    stop = 0;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(su32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tslot;
  const uint32_t mine = tmem + ((uint32_t)((warp & 3) * 32) << 16) + 8 * (warp >> 2);   // cols 0..63
  const uint32_t idesc = (1u << 4) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  long long t0 = clock64(), t1 = t0;
  if (warp == 0 && (mode & 2)) {
    // MMA stream: D at cols 384..511, A at 320..351, until the others finish
    uint32_t ph = 0;
    int n = 0;
    long long iss = 0, exe = 0;
    while (stop < 31) {
      long long ta = clock64(), tb = ta, tc = ta;
      if (lane == 0) {
        for (int i = 0; i < 8; ++i)
          asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n"
                       ::"r"(tmem + 384), "r"(tmem + 320 + 8 * (i & 3)), "l"(sdesc(su32(smem) + 32 * (i & 3))), "r"(idesc), "r"(i));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(&bar)) : "memory");
        tb = clock64();
        asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" ::"r"(su32(&bar)), "r"(ph) : "memory");
        tc = clock64();
        iss += tb - ta;
        exe += tc - tb;
      }
      ph ^= 1;
      ++n;
      __syncwarp();
    }
    if (lane == 0) out[gridDim.x * 2 + blockIdx.x] = n;
    if (lane == 0 && blockIdx.x == 0) printf("   [mode %d] issue %.1f  issued->done %.1f cycles per batch\n", mode, (double)iss / n, (double)exe / n);
  } else {
    uint32_t r[16];
    for (int i = 0; i < 16; ++i) r[i] = i;
    __syncwarp();
    t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (mode & 8) {                      // pure FFMA work
        float f[8];
        for (int i = 0; i < 8; ++i) f[i] = __uint_as_float(r[i]);
        for (int rep = 0; rep < 16; ++rep)
#pragma unroll
          for (int i = 0; i < 8; ++i) f[i] = fmaf(f[i], 1.0001f, 0.5f);
        for (int i = 0; i < 8; ++i) r[i] = __float_as_uint(f[i]);
      } else if (mode & 16) {              // F2FP (ALU pipe) work
        for (int rep = 0; rep < 16; ++rep)
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            unsigned q;
            asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(q) : "f"(__uint_as_float(r[i])), "f"(__uint_as_float(r[i + 8])));
            r[i] = q;
          }
      } else if (mode & 1) {
        if (mode & 4) {
          asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
                       : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                         "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                       : "r"(mine));
        } else {
          asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                       : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]) : "r"(mine));
          asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                       : "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]) : "r"(mine + 64));
        }
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        for (int i = 0; i < 16; ++i) r[i] += 1;
      } else {
        asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};\n" ::"r"(mine + 128), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]) : "memory");
        asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};\n" ::"r"(mine + 160), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]) : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
        for (int i = 0; i < 8; ++i) r[i] += 1;
      }
    }
    t1 = clock64();
    if (lane == 0 && warp == 13) out[blockIdx.x] = t1 - t0;
    if (lane == 0 && warp == 13) out[gridDim.x + blockIdx.x] = r[0] + r[15];
    if (lane == 0) atomicAdd((int*)&stop, 1);
  }
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}
__global__ void dummy() {}
int main() {
  long long* d;
  cudaMalloc(&d, 148 * 3 * 8);
  const int smem = 128 * 128 + 2048;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* nm[32] = {"st x4 x2 + wait", "ld x8 x2 + wait", "st + MMAs", "ld + MMAs", "", "ld x16 + wait", "", "ld x16 + MMAs"};
  nm[8] = "FFMA x128"; nm[10] = "FFMA x128 + MMAs"; nm[16] = "F2FP x128"; nm[18] = "F2FP x128 + MMAs";
  for (int mode : {2, 3, 8, 10, 16, 18}) {
    const int iters = 2000;
    k<<<148, 1024, smem>>>(mode, iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    long long hn[148];
    cudaMemcpy(hn, d + 2 * 148, sizeof(hn), cudaMemcpyDeviceToHost);
    printf("%-18s %s: %.1f cycles per iteration per warp (32 warps)", nm[mode], cudaGetErrorString(e), (double)h[0] / iters);
    if (mode & 2) printf("   MMA batches of 8 in that time: %lld -> %.1f cycles per batch", hn[0], (double)h[0] / hn[0]);
    printf("\n");
  }
  return 0;
}
