// levels.cu — scan levels over EXPLICIT matrices (the block aggregates of the
// upper levels, materialised DENSE leaves), the literal Alg. 1 level kernels,
// the shard-carry combine and the DENSE helpers.
//
// Storage of every explicit level: [B][n][H*H], column-major matrices
// (element (i,k) at k*H+i); the head vector of slot 0 is stored in the first H
// floats.  Carries (exclusive prefixes): [B][n][H].
#include "common.cuh"

namespace bppsa {
namespace {

// ---------------------------------------------------------------------------
// fold_up: CTA per (block q, sample b).  P <- A_s P over the block's slots in
// scan order (agg <- a[s] <> ... = left multiplication).  A_s and P are staged
// in shared memory (A k-major: A[k][i] at k*HP+i; P k-major: P[k][j] at
// k*HP+j), each thread owns a TM x TN register tile of P_new = A P.
// ---------------------------------------------------------------------------
template <int HP, int TM, int TN>
struct Tile {
  static constexpr int GI = HP / TM, GJ = HP / TN, NT = GI * GJ;
  static constexpr int PER = (HP * HP + NT - 1) / NT;
};

template <int HP, int TM, int TN>
__device__ __forceinline__ void gemm_step(const float* __restrict__ As, const float* __restrict__ Ps,
                                          float* __restrict__ Pn, int tid) {
  using Tl = Tile<HP, TM, TN>;
  if (tid >= Tl::NT) return;
  const int ti = tid % Tl::GI, tj = tid / Tl::GI;
  float acc[TM][TN];
#pragma unroll
  for (int x = 0; x < TM; ++x)
#pragma unroll
    for (int y = 0; y < TN; ++y) acc[x][y] = 0.f;
#pragma unroll 8
  for (int k = 0; k < HP; ++k) {
    float av[TM], pv[TN];
#pragma unroll
    for (int x = 0; x < TM; ++x) av[x] = As[k * HP + ti * TM + x];
#pragma unroll
    for (int y = 0; y < TN; ++y) pv[y] = Ps[k * HP + tj * TN + y];
#pragma unroll
    for (int x = 0; x < TM; ++x)
#pragma unroll
      for (int y = 0; y < TN; ++y) acc[x][y] = fmaf(av[x], pv[y], acc[x][y]);
  }
#pragma unroll
  for (int x = 0; x < TM; ++x)
#pragma unroll
    for (int y = 0; y < TN; ++y) Pn[(ti * TM + x) * HP + tj * TN + y] = acc[x][y];
}

__device__ __forceinline__ unsigned ld_acquire_sys_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <int HP, int TM, int TN>
__global__ void __launch_bounds__(Tile<HP, TM, TN>::NT) fold_up_kernel(MatAcc A, int H, long long n, int C,
                                                                       int head, float* __restrict__ agg_out,
                                                                       long long n_out, Publish pub) {
  using Tl = Tile<HP, TM, TN>;
  extern __shared__ __align__(16) float smem[];
  // one A buffer (the next A_s waits in registers) and two P buffers: 48 KB
  // at H = 64, so four CTAs fit an SM (64 KB with two A buffers allowed three)
  float* Ab[1] = {smem};
  float* Pb[2] = {smem + HP * HP, smem + 2 * HP * HP};
  const int tid = threadIdx.x;
  const long long q = blockIdx.x;
  const int b = blockIdx.y;
  const long long s0 = q * C, s1 = min(s0 + (long long)C, n);
  const bool vec = head && q == 0;
  const int HH = H * H;
  for (int e = tid; e < 3 * HP * HP; e += Tl::NT) smem[e] = 0.f;
  if (pub.peers && pub.epoch > 2 && tid == 0)       // the readers are done with slot (epoch - 2) & 1
    for (int r = 0; r < pub.rank; ++r)
      while ((int)(ld_acquire_sys_u32(pub.acks + r) - (pub.epoch - 2)) < 0) __nanosleep(256);
  __syncthreads();
  long long s;
  if (vec) {
    const float* v = A.vec(b);
    for (int k = tid; k < H; k += Tl::NT) Pb[0][k * HP] = v[k];
    s = 1;
  } else {
    const float* m = A.mat(b, s0);
    for (int e = tid; e < HH; e += Tl::NT) {   // element (k, j) at j*H + k -> P[k][j]
      const int j = e / H, k = e % H;
      Pb[0][k * HP + j] = m[e];
    }
    s = s0 + 1;
  }
  int pc = 0;
  constexpr int ac = 0;
  if (HP == 64 && H == 64 && 1024 % Tl::NT == 0) {
    // H = 64: the next A_s (16 KB, column-major = A[k][i] rows of 64) is
    // prefetched as four coalesced float4 per thread (scalar loads made this
    // kernel LSU-throttled: r01h ncu, lg_throttle 20 %, LSU 47 %)
    constexpr int U4 = 1024 / Tl::NT;               // float4 per thread per 64 x 64 matrix
    float4 pre4[U4];
    if (s < s1) {
      const float4* m = reinterpret_cast<const float4*>(A.mat(b, s));
#pragma unroll
      for (int u = 0; u < U4; ++u) pre4[u] = __ldg(m + tid + u * Tl::NT);
    }
    for (; s < s1; ++s) {
#pragma unroll
      for (int u = 0; u < U4; ++u) reinterpret_cast<float4*>(Ab[ac])[tid + u * Tl::NT] = pre4[u];
      if (s + 1 < s1) {
        const float4* m = reinterpret_cast<const float4*>(A.mat(b, s + 1));
#pragma unroll
        for (int u = 0; u < U4; ++u) pre4[u] = __ldg(m + tid + u * Tl::NT);
      }
      __syncthreads();
      gemm_step<HP, TM, TN>(Ab[ac], Pb[pc], Pb[pc ^ 1], tid);
      __syncthreads();                            // A is rewritten next step
      pc ^= 1;
    }
  } else {
    float pre[Tl::PER];
    if (s < s1) {
      const float* m = A.mat(b, s);
#pragma unroll
      for (int u = 0; u < Tl::PER; ++u) {
        const int e = tid + u * Tl::NT;
        pre[u] = (e < HH) ? m[e] : 0.f;
      }
    }
    for (; s < s1; ++s) {
#pragma unroll
      for (int u = 0; u < Tl::PER; ++u) {         // element (i, k) at k*H + i -> A[k][i]
        const int e = tid + u * Tl::NT;
        if (e < HH) Ab[ac][(e / H) * HP + (e % H)] = pre[u];
      }
      if (s + 1 < s1) {
        const float* m = A.mat(b, s + 1);
#pragma unroll
        for (int u = 0; u < Tl::PER; ++u) {
          const int e = tid + u * Tl::NT;
          pre[u] = (e < HH) ? m[e] : 0.f;
        }
      }
      __syncthreads();
      gemm_step<HP, TM, TN>(Ab[ac], Pb[pc], Pb[pc ^ 1], tid);
      __syncthreads();                            // A is rewritten next step
      pc ^= 1;
    }
  }
  __syncthreads();
  const long long off = ((long long)b * n_out + q) * HH;
  float* dst = agg_out + off;
  if (vec) {
    for (int i = tid; i < H; i += Tl::NT) dst[i] = Pb[pc][i * HP];
  } else {
    for (int e = tid; e < HH; e += Tl::NT) {   // (i, j) -> j*H + i
      const int j = e / H, i = e % H;
      dst[e] = Pb[pc][i * HP + j];
    }
  }
  if (pub.peers) {                             // fused publish: P2P stores into every rank's mailbox
    const long long slot = ((long long)(pub.epoch & 1u) * pub.world + pub.rank) * pub.n + off;
    const int cnt = vec ? H : HH;
    for (int e = tid; e < cnt; e += Tl::NT) {
      const float v = vec ? Pb[pc][e * HP] : Pb[pc][(e % H) * HP + e / H];
      for (int p = 0; p < pub.world; ++p) pub.peers[p][slot + e] = v;
    }
    __threadfence_system();                    // this CTA's stores, before the count
    __syncthreads();
    if (tid == 0) {
      const unsigned total = gridDim.x * gridDim.y;
      if (atomicAdd(pub.counter, 1u) == total - 1) {   // the last CTA: every store is performed
        __threadfence_system();
        for (int p = 0; p < pub.world; ++p)
          asm volatile("st.release.sys.global.u32 [%0], %1;\n" ::"l"(pub.flags[p] + pub.rank), "r"(pub.epoch)
                       : "memory");
        *pub.counter = 0u;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// walk_down: warp per (block q, sample b).  From the block's carry (exclusive
// prefix) v: out[s] = v; v <- A_s v.  A_s is staged into the warp's shared
// buffer with cp.async (double-buffered); lane l owns rows l + 32m.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void cp_async16(void* smem_ptr, const void* gptr) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_ptr);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gptr));
}
__device__ __forceinline__ void cp_async4(void* smem_ptr, const void* gptr) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_ptr);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gptr));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

template <int HP>
__device__ __forceinline__ void stage_matrix(float* dst, const float* src, int H, int lane) {
  const int HH = H * H;
  if (H == HP && ((reinterpret_cast<uintptr_t>(src) & 15) == 0)) {
    for (int e = lane * 4; e < HH; e += 128) cp_async16(dst + e, src + e);
  } else {
    for (int e = lane; e < HH; e += 32) cp_async4(dst + (e / H) * HP + (e % H), src + e);
  }
}

template <int HP>
__global__ void __launch_bounds__(128) walk_down_kernel(MatAcc A, int H, int B, long long n, int C, int head,
                                                        const float* __restrict__ carry_in, long long nblk,
                                                        float* __restrict__ out, int out_mode, Seg seg,
                                                        float* __restrict__ total_out, VecAcc addv,
                                                        float* __restrict__ vec_out, float* __restrict__ head_out,
                                                        long long head_bstride) {
  constexpr int NR = (HP + 31) / 32;
  constexpr int WS = 2 * HP * HP + HP;   // floats per warp
  const bool vonly = vec_out != nullptr;   // affine vector part of the block (from 0 / the head vector)
  extern __shared__ __align__(16) float smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  float* As[2] = {smem + wib * WS, smem + wib * WS + HP * HP};
  float* xs = smem + wib * WS + 2 * HP * HP;
  const long long task = (long long)blockIdx.x * (blockDim.x >> 5) + wib;
  if (task >= (long long)B * nblk) return;
  const long long q = task % nblk;
  const int b = (int)(task / nblk);
  const long long s0 = q * C, s1 = min(s0 + (long long)C, n);
  const bool vec = head && q == 0;
  if (H != HP) {                                 // zero the padding once
    for (int e = lane; e < 2 * HP * HP; e += 32) As[0][e] = 0.f;
    __syncwarp();
  }
  float v[NR];
#pragma unroll
  for (int m = 0; m < NR; ++m) {
    const int i = lane + 32 * m;
    v[m] = 0.f;
    if (i < H) v[m] = vec ? A.vec(b)[i] : (vonly ? 0.f : carry_in[(q + (long long)b * nblk) * H + i]);
  }
  long long s = vec ? 1 : s0;
  int buf = 0;
  if (s < s1) stage_matrix<HP>(As[0], A.mat(b, s), H, lane);
  cp_commit();
  for (; s < s1; ++s) {
    if (!vonly) {
#pragma unroll
      for (int m = 0; m < NR; ++m) {
        const int i = lane + 32 * m;
        if (i < H) {
          if (out_mode == 0)
            out[((long long)b * n + s) * H + i] = v[m];
          else
            out[((long long)seg.time_of(s) * B + b) * H + i] = v[m];
        }
      }
    }
    const bool last = (s + 1 == s1);
    const bool total = !vonly && last && s1 == n && total_out != nullptr;
    if (last && !total && !vonly) break;
    const float* ap = addv.at(b, s, seg, B, H);
    float av[NR];
#pragma unroll
    for (int m = 0; m < NR; ++m) {
      const int i = lane + 32 * m;
      av[m] = (ap != nullptr && i < H) ? ap[i] : 0.f;
    }
    if (!last) stage_matrix<HP>(As[buf ^ 1], A.mat(b, s + 1), H, lane);
    cp_commit();
#pragma unroll
    for (int m = 0; m < NR; ++m) {
      const int i = lane + 32 * m;
      if (i < HP) xs[i] = v[m];
    }
    cp_wait<1>();
    __syncwarp();
    const float* a = As[buf];
    float part[NR][4];
#pragma unroll
    for (int m = 0; m < NR; ++m)
#pragma unroll
      for (int p = 0; p < 4; ++p) part[m][p] = 0.f;
#pragma unroll 4
    for (int k4 = 0; k4 < HP / 4; ++k4) {
      const float4 x4 = *reinterpret_cast<const float4*>(xs + 4 * k4);
      const float xv[4] = {x4.x, x4.y, x4.z, x4.w};
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
#pragma unroll
        for (int m = 0; m < NR; ++m) {
          const int i = lane + 32 * m;
          if (i < HP) part[m][kk] = fmaf(a[(4 * k4 + kk) * HP + i], xv[kk], part[m][kk]);
        }
      }
    }
#pragma unroll
    for (int m = 0; m < NR; ++m) v[m] = ((part[m][0] + part[m][1]) + (part[m][2] + part[m][3])) + av[m];
    __syncwarp();
    buf ^= 1;
    if (total) {
#pragma unroll
      for (int m = 0; m < NR; ++m) {
        const int i = lane + 32 * m;
        if (i < H) total_out[(long long)b * H + i] = v[m];
      }
    }
  }
  cp_wait<0>();
  if (vonly) {
#pragma unroll
    for (int m = 0; m < NR; ++m) {
      const int i = lane + 32 * m;
      if (i < H) {
        vec_out[((long long)b * nblk + q) * H + i] = v[m];
        if (vec && head_out != nullptr) head_out[(long long)b * head_bstride + i] = v[m];
      }
    }
  }
}

constexpr int kWarps = 4;

template <int HP, int TM, int TN>
cudaError_t fold_impl(const MatAcc& A, int H, int B, long long n, int C, int head, float* agg_out,
                      long long n_out, cudaStream_t st, const Publish* pub) {
  using Tl = Tile<HP, TM, TN>;
  const size_t smem = 3ull * HP * HP * sizeof(float);
  auto k = fold_up_kernel<HP, TM, TN>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  dim3 grid((unsigned)n_out, (unsigned)B);
  k<<<grid, Tl::NT, smem, st>>>(A, H, n, C, head, agg_out, n_out, pub ? *pub : Publish{});
  return cudaGetLastError();
}

template <int HP>
cudaError_t walk_impl(const MatAcc& A, int H, int B, long long n, int C, int head, const float* carry_in,
                      long long nblk, float* out, int out_mode, const Seg& seg, float* total_out,
                      cudaStream_t st, const VecAcc& addv, float* vec_out, float* head_out, long long head_bstride) {
  const size_t smem = (size_t)kWarps * (2 * HP * HP + HP) * sizeof(float);
  auto k = walk_down_kernel<HP>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  const long long tasks = (long long)B * nblk;
  k<<<(unsigned)((tasks + kWarps - 1) / kWarps), 32 * kWarps, smem, st>>>(A, H, B, n, C, head, carry_in, nblk,
                                                                          out, out_mode, seg, total_out, addv,
                                                                          vec_out, head_out, head_bstride);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// DENSE helpers
// ---------------------------------------------------------------------------
__global__ void transpose_kernel(const float* __restrict__ JT, float* __restrict__ JTc, int H) {
  __shared__ float t[64][65];
  const long long m = blockIdx.x;
  const float* src = JT + m * H * H;
  float* dst = JTc + m * H * H;
  for (int e = threadIdx.x; e < H * H; e += blockDim.x) t[e / H][e % H] = src[e];   // t[i][k]
  __syncthreads();
  for (int e = threadIdx.x; e < H * H; e += blockDim.x) {
    const int k = e / H, i = e % H;   // dst (i,k) at k*H + i
    dst[e] = t[i][k];
  }
}

__global__ void materialize_rnn_kernel(const float* __restrict__ h, const float* __restrict__ W,
                                       float* __restrict__ JT, long long total, int H) {
  const long long HH = (long long)H * H;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long mb = e / HH;   // (t*B + b)
    const int ik = (int)(e % HH), i = ik / H, k = ik % H;
    const float hv = h[mb * H + k];
    JT[e] = W[(long long)k * H + i] * (1.f - hv * hv);
  }
}

__global__ void materialize_gru_kernel(const float* __restrict__ hp, const float* __restrict__ r,
                                       const float* __restrict__ z, const float* __restrict__ n,
                                       const float* __restrict__ M, const float* __restrict__ W3,
                                       float* __restrict__ JT, long long total, int H) {
  const long long HH = (long long)H * H;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long mb = e / HH;
    const int ik = (int)(e % HH), i = ik / H, k = ik % H;
    const long long o = mb * H + k;
    const float rv = r[o], zv = z[o], nv = n[o], Mv = M[o], hv = hp[o];
    const float omn2 = 1.f - nv * nv, omz = 1.f - zv;
    const float c0 = rv * (1.f - rv) * Mv * omn2 * omz, c1 = rv * omn2 * omz, c2 = zv * (1.f - zv) * (hv - nv);
    float val = W3[(long long)(0 * H + k) * H + i] * c0;
    val = fmaf(W3[(long long)(2 * H + k) * H + i], c1, val);
    val = fmaf(W3[(long long)(1 * H + k) * H + i], c2, val);
    if (i == k) val += zv;
    JT[e] = val;
  }
}

// ---------------------------------------------------------------------------
// Alg. 1 executed literally over X [(n+1)][B][H*H] (column-major slots).
// ---------------------------------------------------------------------------
__global__ void alg1_init_kernel(const float* __restrict__ JT, const float* __restrict__ seed,
                                 float* __restrict__ X, int T, int B, int H) {
  __shared__ float t[64][65];
  const long long k = blockIdx.x;   // slot
  const int b = blockIdx.y;
  const long long HH = (long long)H * H;
  float* dst = X + (k * B + b) * HH;
  if (k == 0) {
    for (int i = threadIdx.x; i < H; i += blockDim.x) dst[i] = seed[(long long)b * H + i];
    return;
  }
  const float* src = JT + ((long long)(T - k) * B + b) * HH;   // row-major J^T
  for (int e = threadIdx.x; e < H * H; e += blockDim.x) t[e / H][e % H] = src[e];
  __syncthreads();
  for (int e = threadIdx.x; e < H * H; e += blockDim.x) dst[e] = t[e % H][e / H];
}

template <int HP, int TM, int TN>
__global__ void __launch_bounds__(Tile<HP, TM, TN>::NT) alg1_up_kernel(float* __restrict__ X, int B, int H,
                                                                       long long n, int d) {
  using Tl = Tile<HP, TM, TN>;
  extern __shared__ __align__(16) float smem[];
  float* As = smem;
  float* Ps = smem + HP * HP;
  float* Pn = smem + 2 * HP * HP;
  const int tid = threadIdx.x;
  const long long i0 = (long long)blockIdx.x << (d + 1);
  const long long l = i0 + (1ll << d) - 1, r = min(i0 + (1ll << (d + 1)) - 1, n);
  const int b = blockIdx.y;
  const long long HH = (long long)H * H;
  const bool vec = (i0 == 0);
  for (int e = tid; e < 3 * HP * HP; e += Tl::NT) smem[e] = 0.f;
  __syncthreads();
  const float* Ar = X + (r * B + b) * HH;
  const float* Al = X + (l * B + b) * HH;
  for (int e = tid; e < H * H; e += Tl::NT) As[(e / H) * HP + (e % H)] = Ar[e];  // (i,k)@k*H+i
  if (vec) {
    for (int k = tid; k < H; k += Tl::NT) Ps[k * HP] = Al[k];
  } else {
    for (int e = tid; e < H * H; e += Tl::NT) Ps[(e % H) * HP + e / H] = Al[e];  // (k,j)@j*H+k
  }
  __syncthreads();
  gemm_step<HP, TM, TN>(As, Ps, Pn, tid);   // a[r] <- a[l] <> a[r] = a[r] a[l]
  __syncthreads();
  float* dst = X + (r * B + b) * HH;
  if (vec) {
    for (int i = tid; i < H; i += Tl::NT) dst[i] = Pn[i * HP];
  } else {
    for (int e = tid; e < H * H; e += Tl::NT) dst[e] = Pn[(e % H) * HP + e / H];
  }
}

__global__ void alg1_down_kernel(float* __restrict__ X, int B, int H, long long n, int d, long long npairs) {
  const int lane = threadIdx.x & 31;
  const long long task = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (task >= npairs * B) return;
  const long long p = task / B;
  const int b = (int)(task % B);
  const long long i0 = p << (d + 1);
  const long long l = i0 + (1ll << d) - 1, r = min(i0 + (1ll << (d + 1)) - 1, n);
  const long long HH = (long long)H * H;
  float* Xl = X + (l * B + b) * HH;
  float* Xr = X + (r * B + b) * HH;
  if (i0 == 0) {   // a[r] is I: a[l] <- I (symbolic), a[r] <- T = a[l] (a vector)
    for (int i = lane; i < H; i += 32) Xr[i] = Xl[i];
    return;
  }
  // T <- a[l] (matrix); a[l] <- a[r]; a[r] <- a[r] <> T = T a[r]
  float vr[2], res[2];
  for (int m = 0; m < 2; ++m) {
    const int i = lane + 32 * m;
    vr[m] = (i < H) ? Xr[i] : 0.f;
    res[m] = 0.f;
  }
  for (int k = 0; k < H; ++k) {
    const float vk = __shfl_sync(0xffffffffu, vr[k >> 5], k & 31);
    for (int m = 0; m < 2; ++m) {
      const int i = lane + 32 * m;
      if (i < H) res[m] = fmaf(Xl[(long long)k * H + i], vk, res[m]);
    }
  }
  __syncwarp();
  for (int m = 0; m < 2; ++m) {
    const int i = lane + 32 * m;
    if (i < H) {
      Xl[i] = vr[m];
      Xr[i] = res[m];
    }
  }
}

__global__ void alg1_extract_kernel(const float* __restrict__ X, const float* __restrict__ JT,
                                    float* __restrict__ grad_h, float* __restrict__ grad_init, int T, int B,
                                    int H) {
  const long long HH = (long long)H * H;
  const long long total = (long long)T * B * H;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e % H);
    const long long tb = e / H;
    const int b = (int)(tb % B);
    const int t = (int)(tb / B);
    grad_h[e] = X[((long long)(T - t) * B + b) * HH + i];   // slot T - t holds grad_h[t]
  }
  if (grad_init != nullptr) {   // inclusive extra J_0^T grad_h[0]
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < (long long)B * H;
         e += (long long)gridDim.x * blockDim.x) {
      const int i = (int)(e % H), b = (int)(e / H);
      const float* J0 = JT + (long long)b * HH;                       // J_0^T row-major
      const float* g0 = X + ((long long)T * B + b) * HH;               // grad_h[0]
      float acc = 0.f;
      for (int k = 0; k < H; ++k) acc = fmaf(J0[(long long)i * H + k], g0[k], acc);
      grad_init[e] = acc;
    }
  }
}

// Level-balanced hybrid bridge (reading 19): after `u` up-sweep levels
// a[s + 2^u - 1] holds the aggregate of the 2^u-block starting at slot s.  One
// warp per sample folds those aggregates left to right onto the seed (every
// prefix that contains slot 0 is a vector, so each fold is one GEMV
// P <- a[slot] P) and deposits the exclusive prefix of every 2^dl-block at the
// block's right end.  The deposit of block 0 is the identity, left symbolic
// (the down-sweep's pair i = 0 never reads it).  A deposit's slot is read by
// the fold at most once, at the same or the next iteration, so it is written
// only after that read.
__global__ void hybrid_bridge_kernel(float* __restrict__ X, int B, int H, long long n, int u, int dl) {
  const int lane = threadIdx.x & 31;
  const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (b >= B) return;
  const long long HH = (long long)H * H;
  const long long bs = 1ll << u, D = 1ll << dl;
  const long long last = (n / D) * D;   // start of the last 2^dl-block
  float P[2] = {0.f, 0.f}, pv[2] = {0.f, 0.f};
  bool ident = true;
  long long pend = -1;                  // slot of a deposit not yet written
  auto store = [&](long long slot, const float* v) {
    __syncwarp();
    float* dst = X + (slot * B + b) * HH;
    for (int m = 0; m < 2; ++m) {
      const int i = lane + 32 * m;
      if (i < H) dst[i] = v[m];
    }
  };
  for (long long s = 0; s <= last; s += bs) {
    if (s % D == 0 && s > 0) {
      const long long pos = min(s + D - 1, n);
      if (s + D <= last) {   // the fold reads slot pos at iteration s + D - bs: write after it
        pend = pos;
        pv[0] = P[0];
        pv[1] = P[1];
      } else {
        store(pos, P);
      }
    }
    if (s + bs > last) continue;
    const long long slot = s + bs - 1;
    const float* A = X + (slot * B + b) * HH;
    if (ident) {   // block 0's aggregate contains slot 0: a vector
      for (int m = 0; m < 2; ++m) {
        const int i = lane + 32 * m;
        P[m] = (i < H) ? A[i] : 0.f;
      }
      ident = false;
    } else {       // P <- P <> a[slot] = a[slot] P
      float res[2] = {0.f, 0.f};
      for (int k = 0; k < H; ++k) {
        const float pk = __shfl_sync(0xffffffffu, P[k >> 5], k & 31);
        for (int m = 0; m < 2; ++m) {
          const int i = lane + 32 * m;
          if (i < H) res[m] = fmaf(A[(long long)k * H + i], pk, res[m]);
        }
      }
      P[0] = res[0];
      P[1] = res[1];
    }
    if (slot == pend) {
      store(pend, pv);
      pend = -1;
    }
  }
}

// carry = M_{r+1} ... M_{G-2} V_{G-1}; aggregates column-major [G][B][H*H]
__global__ void carry_combine_kernel(const float* __restrict__ gathered, int rank, int world, int B, int H,
                                     float* __restrict__ carry_out) {
  const int lane = threadIdx.x & 31;
  const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (b >= B) return;
  const long long HH = (long long)H * H;
  float v[2];
  for (int m = 0; m < 2; ++m) {
    const int i = lane + 32 * m;
    v[m] = (i < H) ? gathered[((long long)(world - 1) * B + b) * HH + i] : 0.f;
  }
  for (int s = world - 2; s > rank; --s) {
    const float* Ms = gathered + ((long long)s * B + b) * HH;
    float acc[2] = {0.f, 0.f};
    for (int k = 0; k < H; ++k) {
      const float vk = __shfl_sync(0xffffffffu, v[k >> 5], k & 31);
      for (int m = 0; m < 2; ++m) {
        const int i = lane + 32 * m;
        if (i < H) acc[m] = fmaf(Ms[(long long)k * H + i], vk, acc[m]);
      }
    }
    v[0] = acc[0];
    v[1] = acc[1];
  }
  for (int m = 0; m < 2; ++m) {
    const int i = lane + 32 * m;
    if (i < H) carry_out[(long long)b * H + i] = v[m];
  }
}

}  // namespace

cudaError_t launch_fold_up(const MatAcc& A, int H, int B, long long n, int C, int head, float* agg_out,
                           long long n_out, cudaStream_t st, const Publish* pub) {
  if (H == 20) return fold_impl<20, 2, 2>(A, H, B, n, C, head, agg_out, n_out, st, pub);
  if (H <= 32) return fold_impl<32, 2, 2>(A, H, B, n, C, head, agg_out, n_out, st, pub);
  // many blocks (level 1 at C4, block0 1024: 512 CTAs): 8 x 8 register tiles, 64 threads
  // per GEMM, half the shared-memory reads per FMA (the 4 x 4 form was
  // LSU / MIO-throttled); few blocks: 4 x 4, 256 threads, shorter chains
#ifndef FOLD_UP_88_MIN
#define FOLD_UP_88_MIN 256LL                        // r02g: level 1 at C4 (512 CTAs) 0.48 -> 0.34 ms with 8 x 8; level 2 (16) 0.14 vs 0.16
#endif
  if ((long long)n_out * B >= FOLD_UP_88_MIN) return fold_impl<64, 8, 8>(A, H, B, n, C, head, agg_out, n_out, st, pub);
  return fold_impl<64, 4, 4>(A, H, B, n, C, head, agg_out, n_out, st, pub);
}

cudaError_t launch_walk_down(const MatAcc& A, int H, int B, long long n, int C, int head,
                             const float* carry_in, long long nblk, float* out, int out_mode, const Seg& seg,
                             float* total_out, cudaStream_t st, const VecAcc& addv, float* vec_out,
                             float* head_out, long long head_bstride) {
  if (H == 20)
    return walk_impl<20>(A, H, B, n, C, head, carry_in, nblk, out, out_mode, seg, total_out, st, addv, vec_out,
                         head_out, head_bstride);
  if (H <= 32)
    return walk_impl<32>(A, H, B, n, C, head, carry_in, nblk, out, out_mode, seg, total_out, st, addv, vec_out,
                         head_out, head_bstride);
  return walk_impl<64>(A, H, B, n, C, head, carry_in, nblk, out, out_mode, seg, total_out, st, addv, vec_out,
                       head_out, head_bstride);
}

__global__ void affine_seed_kernel(const float* __restrict__ seed, const float* __restrict__ e, int T, int B,
                                   int H, float* __restrict__ dst) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < B * H) dst[i] = seed[i] + e[(long long)(T - 1) * B * H + i];
}

cudaError_t launch_affine_seed(const float* seed, const float* e, int T, int B, int H, float* dst, cudaStream_t st) {
  affine_seed_kernel<<<(B * H + 255) / 256, 256, 0, st>>>(seed, e, T, B, H, dst);
  return cudaGetLastError();
}

cudaError_t launch_transpose_dense(const float* JT, float* JTc, long long mats, int H, cudaStream_t st) {
  transpose_kernel<<<(unsigned)mats, 256, 0, st>>>(JT, JTc, H);
  return cudaGetLastError();
}

static unsigned grid_for(long long total) {
  long long g = (total + 255) / 256;
  return (unsigned)(g > 148 * 32 ? 148 * 32 : (g < 1 ? 1 : g));
}

cudaError_t launch_materialize_rnn(const float* h, const float* W, float* JT, int T, int B, int H,
                                   cudaStream_t st) {
  const long long total = (long long)T * B * H * H;
  materialize_rnn_kernel<<<grid_for(total), 256, 0, st>>>(h, W, JT, total, H);
  return cudaGetLastError();
}

cudaError_t launch_materialize_gru(const float* hp, const float* r, const float* z, const float* n,
                                   const float* M, const float* W3, float* JT, int T, int B, int H,
                                   cudaStream_t st) {
  const long long total = (long long)T * B * H * H;
  materialize_gru_kernel<<<grid_for(total), 256, 0, st>>>(hp, r, z, n, M, W3, JT, total, H);
  return cudaGetLastError();
}

cudaError_t launch_alg1_init(const float* JT, const float* seed, float* X, int T, int B, int H,
                             cudaStream_t st) {
  dim3 grid((unsigned)(T + 1), (unsigned)B);
  alg1_init_kernel<<<grid, 256, 0, st>>>(JT, seed, X, T, B, H);
  return cudaGetLastError();
}

template <int HP, int TM, int TN>
static cudaError_t alg1_up_impl(float* X, int B, int H, long long n, int d, cudaStream_t st) {
  using Tl = Tile<HP, TM, TN>;
  const long long npairs = (n - (1ll << d)) / (1ll << (d + 1)) + 1;
  const size_t smem = 3ull * HP * HP * sizeof(float);
  auto k = alg1_up_kernel<HP, TM, TN>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  dim3 grid((unsigned)npairs, (unsigned)B);
  k<<<grid, Tl::NT, smem, st>>>(X, B, H, n, d);
  return cudaGetLastError();
}

cudaError_t launch_alg1_up(float* X, int B, int H, long long n, int d, cudaStream_t st) {
  if (n - (1ll << d) < 0) return cudaSuccess;
  if (H == 20) return alg1_up_impl<20, 2, 2>(X, B, H, n, d, st);
  if (H <= 32) return alg1_up_impl<32, 2, 2>(X, B, H, n, d, st);
  return alg1_up_impl<64, 4, 4>(X, B, H, n, d, st);
}

cudaError_t launch_alg1_down(float* X, int B, int H, long long n, int d, cudaStream_t st) {
  if (n - (1ll << d) < 0) return cudaSuccess;
  const long long npairs = (n - (1ll << d)) / (1ll << (d + 1)) + 1;
  const long long warps = npairs * B;
  alg1_down_kernel<<<(unsigned)((warps + 3) / 4), 128, 0, st>>>(X, B, H, n, d, npairs);
  return cudaGetLastError();
}

cudaError_t launch_alg1_extract(const float* X, const float* JT, float* grad_h, float* grad_init, int T, int B,
                                int H, cudaStream_t st) {
  alg1_extract_kernel<<<grid_for((long long)T * B * H), 256, 0, st>>>(X, JT, grad_h, grad_init, T, B, H);
  return cudaGetLastError();
}

cudaError_t launch_hybrid_bridge(float* X, int B, int H, long long n, int u, int dl, cudaStream_t st) {
  hybrid_bridge_kernel<<<(unsigned)((B + 3) / 4), 128, 0, st>>>(X, B, H, n, u, dl);
  return cudaGetLastError();
}

cudaError_t launch_carry_combine(const float* gathered, int rank, int world, int B, int H, float* carry_out,
                                 cudaStream_t st) {
  carry_combine_kernel<<<(unsigned)((B + 3) / 4), 128, 0, st>>>(gathered, rank, world, B, H, carry_out);
  return cudaGetLastError();
}

}  // namespace bppsa
