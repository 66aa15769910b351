// Dev aid: tcgen05 kind::i8 probe for the exact-integer level-0 fold.
// (1) correctness of s8/u8 x s8 MMAs, A in TMEM (TS) or shared memory (SS),
//     B K-major SWIZZLE_64B or SWIZZLE_NONE, shifted accumulator addresses
//     (D + 64 with N = 192), against a host int64 reference;
// (2) cycles per MMA for M = 128 / 64, K = 32, N in {64, 128, 192, 256};
// (3) CUDA-core throughput of the epilogue instruction mix.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/tc_i8_probe.cu -o /tmp/tc_i8_probe
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <random>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
// layout 4 = SWIZZLE_64B (rows of 64 B, SBO 512), 0 = SWIZZLE_NONE (core matrices 8 x 16 B, LBO 128, SBO 512)
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, int layout) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((layout == 0 ? 128 : 16) >> 4) << 16;
  d |= (uint64_t)((layout == 2 ? 1024 : 512) >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;
  return d;
}
// byte offset of (row, k) in a K-major tile of K = 64 bytes
__host__ __device__ inline uint32_t koff(int row, int k, int layout) {
  if (layout == 4) return (uint32_t)(row * 64 + ((((k >> 4) ^ ((row >> 1) & 3))) << 4) + (k & 15));
  return (uint32_t)((row >> 3) * 512 + (k >> 4) * 128 + (row & 7) * 16 + (k & 15));
}
// K-step advance (32 bytes of K) on the descriptor start address
__host__ __device__ inline uint32_t kstep(int layout) { return layout == 0 ? 256u : 32u; }
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N, int asgn, int bsgn) {
  return (2u << 4) | ((uint32_t)asgn << 7) | ((uint32_t)bsgn << 10) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t ph) {
  asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" ::"r"(
                   bar), "r"(ph) : "memory");
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, int acc) {
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
               "r"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, int acc) {
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
               "l"(a), "l"(b), "r"(id), "r"(acc));
}

// Correctness: A [128][64] bytes, B [256][64] bytes (row n = B column n, K-major), D [128][256] s32.
// mode bit 0: SS (else TS); bit 1: A unsigned; bits 2..: test kind
//   test 0: D[:, 0:N) = A B[0:N)            (N = 256)
//   test 1: D[:, 0:256) = A B[0:256);  D[:, 64:256) += A2 B[0:192)   (shifted accumulation, A2 = A rows reversed)
__global__ void probe(const int8_t* A, const int8_t* B, int* D, int mode, int layout, int test) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sB = smem;              // 256 rows x 64 B = 16 KB
  uint8_t* sA = smem + 16384;      // 128 rows x 64 B = 8 KB
  uint8_t* sA2 = smem + 24576;     // 8 KB
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int t = threadIdx.x, warp = t >> 5;
  for (int e = t; e < 256 * 64; e += 128) sB[koff(e / 64, e % 64, layout)] = (uint8_t)B[e];
  for (int e = t; e < 128 * 64; e += 128) {
    sA[koff(e / 64, e % 64, layout)] = (uint8_t)A[e];
    sA2[koff(e / 64, e % 64, layout)] = (uint8_t)A[(127 - e / 64) * 64 + e % 64];
  }
  if (t == 0) {
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
  const uint32_t tmem = tslot, lane_base = tmem + ((uint32_t)(warp * 32) << 16);
  // TS: A at TMEM columns 256..271 (16 cols x 4 bytes), A2 at 272..287
  {
    uint32_t w[16], w2[16];
    for (int c = 0; c < 16; ++c) {
      uint32_t v = 0, v2 = 0;
      for (int b = 0; b < 4; ++b) {
        v |= (uint32_t)(uint8_t)A[t * 64 + 4 * c + b] << (8 * b);
        v2 |= (uint32_t)(uint8_t)A[(127 - t) * 64 + 4 * c + b] << (8 * b);
      }
      w[c] = v, w2[c] = v2;
    }
    for (int c = 0; c < 16; ++c) {
      asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};\n" ::"r"(lane_base + 256 + c), "r"(w[c]) : "memory");
      asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};\n" ::"r"(lane_base + 272 + c), "r"(w2[c]) : "memory");
    }
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  if (t == 0) {
    const bool ss = mode & 1;
    const int asg = (mode & 2) ? 0 : 1;
    const uint32_t bb = su32(sB), ab = su32(sA), ab2 = su32(sA2);
    for (int ks = 0; ks < 2; ++ks) {
      const uint64_t bd = sdesc(bb + ks * kstep(layout), layout);
      if (ss) mma_ss(tmem, sdesc(ab + ks * kstep(layout), layout), bd, idesc_i8(128, 256, asg, 1), ks);
      else mma_ts(tmem, tmem + 256 + 8 * ks, bd, idesc_i8(128, 256, asg, 1), ks);
    }
    if (test == 1) {
      for (int ks = 0; ks < 2; ++ks) {
        const uint64_t bd = sdesc(bb + ks * kstep(layout), layout);
        if (ss) mma_ss(tmem + 64, sdesc(ab2 + ks * kstep(layout), layout), bd, idesc_i8(128, 192, asg, 1), 1);
        else mma_ts(tmem + 64, tmem + 272 + 8 * ks, bd, idesc_i8(128, 192, asg, 1), 1);
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(&bar))
                 : "memory");
  }
  __syncwarp();
  mbar_wait(su32(&bar), 0);
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  for (int c = 0; c < 256; ++c) {
    uint32_t r;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];\n" : "=r"(r) : "r"(lane_base + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
    D[t * 256 + c] = (int)r;
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

// Rate: per batch, `nm` MMAs (K = 32 each) of the given N / M, SS or TS; one CTA per SM.
__global__ void rate(int nbatch, int M, int N, int ss, int nm, int layout, long long* cycles) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 40960 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = (uint32_t)i * 2654435761u;
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
  const uint32_t id = idesc_i8(M, N, 1, 1);
  const uint32_t bb = su32(smem), ab = su32(smem + 16384);
  long long t0 = clock64();
  if (threadIdx.x < 32) {
    uint32_t ph = 0;
    for (int b = 0; b < nbatch; ++b) {
      if (threadIdx.x == 0) {
        for (int i = 0; i < nm; ++i) {
          const uint64_t bd = sdesc(bb + (i & 1) * kstep(layout), layout);
          if (ss == 2) {
            const uint32_t idf = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
            asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem),
                         "r"(tmem + 256 + 8 * (i & 1)), "l"(bd), "r"(idf), "r"(i));
          } else if (ss) mma_ss(tmem, sdesc(ab + (i & 1) * kstep(layout), layout), bd, id, i);
          else mma_ts(tmem, tmem + 256 + 8 * (i & 1), bd, id, i);
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

// ---------------------------------------------------------------------------
// CUDA-core throughput of single ops and of candidate epilogue mixes.
// ---------------------------------------------------------------------------
__device__ __forceinline__ float i2f(int x) {
  float r;
  asm volatile("cvt.rn.f32.s32 %0, %1;" : "=f"(r) : "r"(x));
  return r;
}
__device__ __forceinline__ int it_dummy(int x) { return x & 7; }
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t s) {
  uint32_t r;
  asm volatile("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(s));
  return r;
}

template <int OP>
__global__ void oprate(uint32_t* out, int iters, uint32_t seed) {
  uint32_t u[8];
  float f[8];
  float2 v[8];
  for (int i = 0; i < 8; ++i) {
    u[i] = seed * (threadIdx.x + 7 * i);
    f[i] = 1.0f + 1e-3f * i + threadIdx.x * 1e-6f;
    v[i] = make_float2(f[i], f[i] * 0.5f);
  }
  const float2 k2 = make_float2(0.999f, 1.001f), c2 = make_float2(1e-3f, 2e-3f);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(f[i]) : "f"(f[(i + 1) & 7]), "f"(f[(i + 2) & 7]));
      if (OP == 1) asm volatile("fma.rn.f32 %0, %0, 0f3F7FF000, 0f3A800000;" : "+f"(f[i]));
      if (OP == 2) { float r; asm volatile("cvt.rn.f32.s32 %0, %1;" : "=f"(r) : "r"(u[i])); u[i] = __float_as_uint(r); }
      if (OP == 3) asm volatile("add.u32 %0, %0, 1262485504;" : "+r"(u[i]));
      if (OP == 4) asm volatile("prmt.b32 %0, %0, %1, 0x5140;" : "+r"(u[i]) : "r"(u[(i + 1) & 7]));
      if (OP == 5) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(*reinterpret_cast<unsigned long long*>(&v[i])) : "l"(*reinterpret_cast<const unsigned long long*>(&k2)), "l"(*reinterpret_cast<const unsigned long long*>(&c2)));
      if (OP == 6) asm volatile("max.f32 %0, %0, %1;" : "+f"(f[i]) : "f"(f[(i + 3) & 7]));
      if (OP == 7) asm volatile("xor.b32 %0, %0, 0x80008080;" : "+r"(u[i]));
      if (OP == 8) asm volatile("mad.lo.s32 %0, %0, 3, 1262485504;" : "+r"(u[i]));
      if (OP == 9) asm volatile("add.u32 %0, %0, %1;" : "+r"(u[i]) : "r"(u[(i + 1) & 7]));
      if (OP == 10) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(*reinterpret_cast<unsigned long long*>(&v[i])) : "l"(*reinterpret_cast<const unsigned long long*>(&c2)));
      if (OP == 11) asm volatile("fma.rn.f32 %0, %0, %1, 0f3A800000;" : "+f"(f[i]) : "f"(f[(i + 1) & 7]));
    }
  }
  long long t1 = clock64();
  uint32_t s = 0;
  for (int i = 0; i < 8; ++i) s += u[i] + __float_as_uint(f[i]) + __float_as_uint(v[i].x + v[i].y);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (uint32_t)(t1 - t0);
}

// Candidate epilogue per step for one thread = (chain row, 32 columns):
// tcgen05.ld of 4 int32 regions (TMEM), magic-bias conversion, Horner
// combine, row max, d scaling (d from shared memory), magic rounding to a
// 22-bit integer, balanced bytes, element-major packing (3 words per 4
// elements), st.shared of the A bytes.  No MMA, no synchronisation.
// VAR 0: scalar fp ops; 1: paired f32x2 ops; 2: I2F conversions (scalar)
__device__ __forceinline__ void tld8(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
template <int VAR>
__global__ void epi(uint32_t* out, int iters, uint32_t seed) {
  __shared__ uint32_t tslot;
  __shared__ __align__(16) float ds[64 * 8];
  __shared__ __align__(16) uint32_t abuf[16][32][8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 64 * 8; i += blockDim.x) ds[i] = 0.75f + (i & 63) * 0.001f;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(su32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tslot;
  const uint32_t lb = tmem + ((uint32_t)((warp & 3) * 32) << 16) + 256 * ((warp >> 3) & 1) + 32 * ((warp >> 2) & 1);
  // fill the regions with small integers
  for (int c = 0; c < 32; ++c)
    for (int r = 0; r < 4; ++r) {
      const uint32_t v = ((seed * (threadIdx.x * 131 + c * 7 + r)) >> 11) - (1u << 20);
      asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};\n" ::"r"(lb + 64 * r + c), "r"(v) : "memory");
    }
  asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
  float mx = 0.f;
  const uint32_t dbase = su32(ds) + 4u * 32 * ((warp >> 2) & 1);
  const uint32_t ab = su32(&abuf[warp][lane][0]);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const float sc = __int_as_float((127 + (it & 3)) << 23);
#pragma unroll
    for (int h = 0; h < 4; ++h) {        // 4 groups of 8 columns
      uint32_t R[4][8];
#pragma unroll
      for (int r = 0; r < 4; ++r) tld8(lb + 64 * r + 8 * h, R[r]);
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
      float c[8];
      if (VAR == 1) {
#pragma unroll
        for (int i = 0; i < 8; i += 2) {
          float2 F[4];
#pragma unroll
          for (int r = 0; r < 4; ++r)
            F[r] = make_float2(__uint_as_float(R[r][i] + 0x4B400000u), __uint_as_float(R[r][i + 1] + 0x4B400000u));
          float2 v = __ffma2_rn(F[3], make_float2(0.00390625f, 0.00390625f), F[2]);
          v = __ffma2_rn(v, make_float2(0.00390625f, 0.00390625f), F[1]);
          const float2 t = __fadd2_rn(F[0], make_float2(-12681216.f, -12681216.f));
          const float2 cc = __ffma2_rn(v, make_float2(0.00390625f, 0.00390625f), t);
          c[i] = cc.x, c[i + 1] = cc.y;
        }
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          float F[4];
#pragma unroll
          for (int r = 0; r < 4; ++r)
            F[r] = VAR == 2 ? (float)(int)R[r][i] : __uint_as_float(R[r][i] + 0x4B400000u);
          float v = fmaf(F[3], 0.00390625f, F[2]);
          v = fmaf(v, 0.00390625f, F[1]);
          c[i] = fmaf(v, 0.00390625f, VAR == 2 ? F[0] : F[0] - 12681216.f);
        }
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) mx = fmaxf(mx, fabsf(c[i]));
      float dv[8];
      asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(dv[0]), "=f"(dv[1]), "=f"(dv[2]), "=f"(dv[3]) : "r"(dbase + 32u * h));
      asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(dv[4]), "=f"(dv[5]), "=f"(dv[6]), "=f"(dv[7]) : "r"(dbase + 32u * h + 16u));
      uint32_t X[8];
      if (VAR == 1) {
#pragma unroll
        for (int i = 0; i < 8; i += 2) {
          const float2 dd = __fmul2_rn(make_float2(dv[i], dv[i + 1]), make_float2(sc, sc));
          const float2 x = __ffma2_rn(make_float2(c[i], c[i + 1]), dd, make_float2(12615808.f, 12615808.f));
          X[i] = __float_as_uint(x.x), X[i + 1] = __float_as_uint(x.y);
        }
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) X[i] = __float_as_uint(fmaf(c[i], dv[i] * sc, 12615808.f));
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) X[i] -= 0x4B400000u - 0x8080u;
      uint32_t w[6];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        w[3 * q] = prmt(X[4 * q], X[4 * q + 1], 0x4210u) ^ 0x80008080u;
        w[3 * q + 1] = prmt(X[4 * q + 1], X[4 * q + 2], 0x5421u) ^ 0x80800080u;
        w[3 * q + 2] = prmt(X[4 * q + 2], X[4 * q + 3], 0x6542u) ^ 0x00808000u;
      }
      asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(ab), "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]) : "memory");
      asm volatile("st.shared.v2.u32 [%0], {%1,%2};" ::"r"(ab + 16u), "r"(w[4]), "r"(w[5]) : "memory");
    }
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = __float_as_uint(mx) + abuf[warp][lane][it_dummy(iters)];
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (uint32_t)(t1 - t0);
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

static const char* opname[] = {"FFMA 3-reg", "FFMA 2imm", "I2F s32->f32", "IADD imm", "PRMT", "FFMA2", "FMNMX",
                               "LOP xor imm", "IMAD imm", "IADD reg", "FADD2", "FFMA 1imm"};

template <int OP>
void run_op(uint32_t* d) {
  const int iters = 2048, thr = 512;
  oprate<OP><<<148, thr>>>(d, iters, 12345u);
  cudaDeviceSynchronize();
  uint32_t cyc;
  cudaMemcpy(&cyc, d, 4, cudaMemcpyDeviceToHost);
  // per SMSP: 4 warps; ops per SMSP = iters * 8 * 4 warps
  printf("%-14s %.3f cycles per warp-op per SMSP (16 warps/SM)\n", opname[OP], cyc / (iters * 8.0 * (thr / 32 / 4)));
}
template <int VAR>
void run_epi(uint32_t* d, int thr) {
  const int iters = 256;
  epi<VAR><<<148, thr>>>(d, iters, 12345u);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("epi err %s\n", cudaGetErrorString(e)); return; }
  uint32_t cyc;
  cudaMemcpy(&cyc, d, 4, cudaMemcpyDeviceToHost);
  const double elems_per_sm = (double)iters * 32 * thr;  // 32 columns per thread per iteration
  printf("epilogue var %d (%d thr/SM): %.4f cycles per element per SM  => %.0f cycles per 8192-element tile-step\n", VAR,
         thr, cyc / elems_per_sm, cyc / elems_per_sm * 8192);
}

int main() {
  std::mt19937 g(1);
  std::uniform_int_distribution<int> ud(-128, 127);
  std::vector<int8_t> A(128 * 64), B(256 * 64);
  for (auto& v : A) v = (int8_t)ud(g);
  for (auto& v : B) v = (int8_t)ud(g);
  int8_t *dA, *dB;
  int* dD;
  cudaMalloc(&dA, A.size());
  cudaMalloc(&dB, B.size());
  cudaMalloc(&dD, 128 * 256 * 4);
  cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
  std::vector<int> D(128 * 256);
  for (int layout : {4, 0})
    for (int mode : {0, 1, 2, 3})
      for (int test : {0, 1}) {
        cudaMemset(dD, 0, D.size() * 4);
        probe<<<1, 128, 40 * 1024>>>(dA, dB, dD, mode, layout, test);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("layout %d mode %d test %d: err %s\n", layout, mode, test, cudaGetErrorString(e)); return 1; }
        cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
        long bad = 0;
        for (int m = 0; m < 128; ++m)
          for (int n = 0; n < 256; ++n) {
            long long ref = 0;
            for (int k = 0; k < 64; ++k) {
              const int a = (mode & 2) ? (int)(uint8_t)A[m * 64 + k] : (int)A[m * 64 + k];
              ref += (long long)a * B[n * 64 + k];
            }
            if (test == 1 && n >= 64)
              for (int k = 0; k < 64; ++k) {
                const int a = (mode & 2) ? (int)(uint8_t)A[(127 - m) * 64 + k] : (int)A[(127 - m) * 64 + k];
                ref += (long long)a * B[(n - 64) * 64 + k];
              }
            if (ref != D[m * 256 + n]) {
              if (bad < 3) printf("   mismatch m=%d n=%d got %d want %lld\n", m, n, D[m * 256 + n], ref);
              ++bad;
            }
          }
        printf("layout %s %s A=%s test %d: %s (%ld mismatches)\n", layout == 4 ? "SW64" : "NONE", (mode & 1) ? "SS" : "TS",
               (mode & 2) ? "u8" : "s8", test, bad ? "FAIL" : "exact", bad);
      }
  long long* dc;
  cudaMalloc(&dc, 148 * sizeof(long long));
  cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024);
  for (int layout : {4, 2, 0})
  for (int ss : {0, 1})
    for (int M : {128})
      for (int N : {64, 128, 192, 256}) {
        const int nb = 500, nm = 32;
        rate<<<148, 128, 48 * 1024>>>(nb, M, N, ss, nm, layout, dc);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("rate err %s\n", cudaGetErrorString(e)); return 1; }
        long long h[148];
        cudaMemcpy(h, dc, sizeof(h), cudaMemcpyDeviceToHost);
        double avg = 0;
        for (int i = 0; i < 148; ++i) avg += h[i];
        avg /= 148;
        printf("layout %d %s M=%3d N=%3d K=32: %.1f cycles per MMA (batches of %d + commit/wait)\n", layout, ss == 2 ? "f16 TS (K=16)" : ss ? "i8 SS" : "i8 TS", M, N,
               avg / (nb * (double)nm), nm);
      }
  uint32_t* dout;
  cudaMalloc(&dout, 148 * 1024 * 4);
  if (getenv("OPS")) { run_op<0>(dout); run_op<1>(dout); run_op<2>(dout); run_op<3>(dout); run_op<4>(dout);
  run_op<5>(dout); run_op<6>(dout); run_op<7>(dout); run_op<8>(dout); run_op<9>(dout); run_op<10>(dout); run_op<11>(dout); }
  if (getenv("EPI")) for (int thr : {256, 512}) { run_epi<0>(dout, thr); run_epi<1>(dout, thr); run_epi<2>(dout, thr); }
  return 0;
}
