// leaf.cu — level 0 of the blocked Blelloch scan with the leaf transposed
// Jacobians built on the fly (never written to HBM).
//
// Up-sweep of one block of slots [s0, s1) (Alg. 1 lines 1-5 in Blelloch's
// p < n regime): the block aggregate a[s1-1] ... a[s0] is folded in scan
// order, agg <- a[s] agg.  Column j of agg therefore evolves as the BP chain
//     c_j <- J_t^T c_j,   c_j(start) = e_j        (matrix blocks)
//     v   <- J_t^T v,     v(start)   = seed       (the head block, a vector)
// and every step of every chain multiplies by the SAME W_hh^T (the leaf is
// J_t^T = W_hh^T diag(1-h_t^2), eqn:rnn P:315; GRU: eqn:gru_jcb P:836-857):
//     (J_t^T c)_i = sum_k W[k][i] d_k c_k          (RNN)
// A warp owns NC chains of one block; lane l owns rows i = l + 32m and keeps
// W[:, i] in registers; the scaled vector x = d o c is exchanged through
// shared memory (broadcast reads), one __syncwarp per step.
//
// Down-sweep of a block (Alg. 1 lines 7-13 with the operand reversal of line
// 13): from the block's exclusive prefix (carry) v, out[s] = v,
// v <- a[s] v = J_t^T v — a GEMV chain; out at the slot of J_t^T is grad_h[t].
#include "common.cuh"

namespace bppsa {
namespace {

template <int CELL>
struct NX { static constexpr int v = (CELL == BPPSA_JAC_GRU) ? 3 : 1; };

// Per-row step coefficients of J_t^T at (t, b, row i).
//  RNN: c0 = 1 - h^2
//  GRU: c0 = r(1-r) M (1-n^2)(1-z)  (multiplies W_hr^T)
//       c1 = r (1-n^2)(1-z)          (multiplies W_hn^T)
//       c2 = z(1-z)(h_prev - n)      (multiplies W_hz^T)
//       c3 = z                       (diagonal J11)
template <int CELL>
struct Coef {
  float c[4];
};

template <int CELL>
__device__ __forceinline__ Coef<CELL> load_coef(const LeafArgs& a, long long off, bool valid) {
  Coef<CELL> k;
  k.c[0] = k.c[1] = k.c[2] = k.c[3] = 0.f;
  if (!valid) return k;
  if (CELL == BPPSA_JAC_RNN_TANH) {
    float hv = __ldg(a.h + off);
    k.c[0] = 1.f - hv * hv;
  } else {
    float r = __ldg(a.r + off), z = __ldg(a.z + off), n = __ldg(a.n + off);
    float M = __ldg(a.M + off), hp = __ldg(a.hp + off);
    float omn2 = 1.f - n * n, omz = 1.f - z;
    k.c[0] = r * (1.f - r) * M * omn2 * omz;
    k.c[1] = r * omn2 * omz;
    k.c[2] = z * (1.f - z) * (hp - n);
    k.c[3] = z;
  }
  return k;
}

// W[v][k] for row i: RNN W[k][i]; GRU v=0: W_hr[k][i], v=1: W_hn[k][i], v=2: W_hz[k][i]
template <int CELL, int HT, int NR>
__device__ __forceinline__ void load_w(const LeafArgs& a, int H, int lane,
                                       float (&w)[NX<CELL>::v][NR][HT]) {
#pragma unroll
  for (int m = 0; m < NR; ++m) {
    const int i = lane + 32 * m;
#pragma unroll
    for (int k = 0; k < HT; ++k) {
      const bool ok = (i < H) && (k < H);
      if (CELL == BPPSA_JAC_RNN_TANH) {
        w[0][m][k] = ok ? __ldg(a.W + (long long)k * H + i) : 0.f;
      } else {
        w[0][m][k] = ok ? __ldg(a.W + (long long)(0 * H + k) * H + i) : 0.f;  // W_hr
        w[1][m][k] = ok ? __ldg(a.W + (long long)(2 * H + k) * H + i) : 0.f;  // W_hn
        w[2][m][k] = ok ? __ldg(a.W + (long long)(1 * H + k) * H + i) : 0.f;  // W_hz
      }
    }
  }
}

// acc_m = sum_v sum_k w[v][m][k] * xs[v*HT + k]   (xs broadcast, 16-byte reads)
template <int CELL, int HT, int NR, int NP>
__device__ __forceinline__ void matvec(const float (&w)[NX<CELL>::v][NR][HT],
                                       const float* __restrict__ xs, float (&acc)[NR]) {
  float part[NR][NP];
#pragma unroll
  for (int m = 0; m < NR; ++m)
#pragma unroll
    for (int p = 0; p < NP; ++p) part[m][p] = 0.f;
#pragma unroll
  for (int v = 0; v < NX<CELL>::v; ++v) {
#pragma unroll
    for (int k4 = 0; k4 < HT / 4; ++k4) {
      const float4 x4 = *reinterpret_cast<const float4*>(xs + v * HT + 4 * k4);
      const float xv[4] = {x4.x, x4.y, x4.z, x4.w};
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const int k = 4 * k4 + kk;
#pragma unroll
        for (int m = 0; m < NR; ++m) part[m][k % NP] = fmaf(w[v][m][k], xv[kk], part[m][k % NP]);
      }
    }
  }
#pragma unroll
  for (int m = 0; m < NR; ++m) {
    float s = part[m][0];
#pragma unroll
    for (int p = 1; p < NP; ++p) s += part[m][p];
    acc[m] = s;
  }
}

// All NC chains at once: for every k the NC x NR accumulators are independent,
// so consecutive FFMAs never wait on each other (x for 4 k's of every chain is
// loaded first with 16-byte broadcast reads).
template <int CELL, int HT, int NR, int NC>
__device__ __forceinline__ void matvec_multi(const float (&w)[NX<CELL>::v][NR][HT],
                                             const float* __restrict__ xb, float (&acc)[NC][NR]) {
  constexpr int NV = NX<CELL>::v;
#pragma unroll
  for (int j = 0; j < NC; ++j)
#pragma unroll
    for (int m = 0; m < NR; ++m) acc[j][m] = 0.f;
#pragma unroll
  for (int v = 0; v < NV; ++v) {
#pragma unroll
    for (int k4 = 0; k4 < HT / 4; ++k4) {
      float4 xv[NC];
#pragma unroll
      for (int j = 0; j < NC; ++j) xv[j] = *reinterpret_cast<const float4*>(xb + (j * NV + v) * HT + 4 * k4);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const int k = 4 * k4 + kk;
#pragma unroll
        for (int j = 0; j < NC; ++j) {
          const float xk = kk == 0 ? xv[j].x : kk == 1 ? xv[j].y : kk == 2 ? xv[j].z : xv[j].w;
#pragma unroll
          for (int m = 0; m < NR; ++m) acc[j][m] = fmaf(w[v][m][k], xk, acc[j][m]);
        }
      }
    }
  }
}

// RNN, H <= 32 (one row per lane): x stored chain-minor, xb[k][j], so one
// 16-byte broadcast read yields x_j[k] for four chains and the products run on
// the paired fp32 pipe (FFMA2, W_ki broadcast to both halves): half the issue
// slots of the scalar loop, and the x store is NC/4 vector stores per lane
template <int HT, int NC>
__device__ __forceinline__ void matvec_multi_t(const float (&w)[1][1][HT], const float* __restrict__ xb,
                                               float (&acc)[NC][1]) {
  static_assert(NC % 4 == 0, "chains in fours");
  float2 a2[NC / 2];
#pragma unroll
  for (int p = 0; p < NC / 2; ++p) a2[p] = make_float2(0.f, 0.f);
#pragma unroll
  for (int k = 0; k < HT; ++k) {
    const float2 wk = make_float2(w[0][0][k], w[0][0][k]);
#pragma unroll
    for (int j4 = 0; j4 < NC / 4; ++j4) {
      const float4 x4 = *reinterpret_cast<const float4*>(xb + k * NC + 4 * j4);
      a2[2 * j4] = __ffma2_rn(make_float2(x4.x, x4.y), wk, a2[2 * j4]);
      a2[2 * j4 + 1] = __ffma2_rn(make_float2(x4.z, x4.w), wk, a2[2 * j4 + 1]);
    }
  }
#pragma unroll
  for (int p = 0; p < NC / 2; ++p) {
    acc[2 * p][0] = a2[p].x;
    acc[2 * p + 1][0] = a2[p].y;
  }
}

// asynchronous 4-byte global -> shared copies for the walk's h ring
__device__ __forceinline__ void cpa4(float* smem_dst, const float* gsrc) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cpa_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// The arrays one walk step reads per row: RNN h; GRU r, z, n, M, h_prev.
template <int CELL>
struct NArr { static constexpr int v = (CELL == BPPSA_JAC_GRU) ? 5 : 1; };
template <int CELL>
__device__ __forceinline__ const float* arr_ptr(const LeafArgs& a, int k) {
  if (CELL == BPPSA_JAC_RNN_TANH) return a.h;
  return k == 0 ? a.r : k == 1 ? a.z : k == 2 ? a.n : k == 3 ? a.M : a.hp;
}
// coefficients from one staged step (ring slot: [NArr][HT] floats)
template <int CELL>
__device__ __forceinline__ Coef<CELL> coef_from(const float* slot, int i, bool valid) {
  Coef<CELL> k;
  k.c[0] = k.c[1] = k.c[2] = k.c[3] = 0.f;
  if (!valid) return k;
  if (CELL == BPPSA_JAC_RNN_TANH) {
    const float hv = slot[i];
    k.c[0] = 1.f - hv * hv;
  } else {
    constexpr int HTX = 32;   // GRU tiles are HT = 32 (or 20 padded into 32 slots)
    const float r = slot[0 * HTX + i], z = slot[1 * HTX + i], n = slot[2 * HTX + i];
    const float M = slot[3 * HTX + i], hp = slot[4 * HTX + i];
    const float omn2 = 1.f - n * n, omz = 1.f - z;
    k.c[0] = r * (1.f - r) * M * omn2 * omz;
    k.c[1] = r * omn2 * omz;
    k.c[2] = z * (1.f - z) * (hp - n);
    k.c[3] = z;
  }
  return k;
}

template <int CELL, int HT, int NC>
struct UpBounds { static constexpr int minb = (CELL == BPPSA_JAC_RNN_TANH && HT == 64) ? 3 : 1; };

template <int CELL, int HT, int NC>
__global__ void __launch_bounds__(128, UpBounds<CELL, HT, NC>::minb) leaf_up_kernel(LeafArgs a, int C, float* __restrict__ agg_out,
                                                      long long n_out, long long q0, long long nq) {
  constexpr int NR = (HT + 31) / 32;
  constexpr int NV = NX<CELL>::v;
  constexpr int XW = NC * NV * HT;       // floats per x buffer
  extern __shared__ __align__(16) float smem[];
  const int H = a.seg.H, B = a.seg.B;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  float* xs = smem + wib * 2 * XW;
  const int G = (H + NC - 1) / NC;
  const long long task = (long long)blockIdx.x * (blockDim.x >> 5) + wib;
  if (task >= (long long)B * nq * G) return;
  const int cg = (int)(task % G);
  const long long rest = task / G;
  const long long q = q0 + rest % nq;
  const int b = (int)(rest / nq);
  const long long S = a.seg.S();
  const long long s0 = q * C, s1 = min(s0 + (long long)C, S);
  const bool vec = a.seg.head && q == 0;
  if (vec && cg > 0) return;
  const int nc = vec ? 1 : min(NC, H - cg * NC);

  float w[NV][NR][HT];
  load_w<CELL, HT, NR>(a, H, lane, w);

  float c[NC][NR];
#pragma unroll
  for (int j = 0; j < NC; ++j)
#pragma unroll
    for (int m = 0; m < NR; ++m) {
      const int i = lane + 32 * m;
      if (vec)
        c[j][m] = (j == 0 && i < H) ? __ldg(a.seed + (long long)b * H + i) : 0.f;
      else
        c[j][m] = (i == cg * NC + j) ? 1.f : 0.f;
    }

  long long s = vec ? 1 : s0;
  const long long rowB = (long long)B * H;
  Coef<CELL> nxt[NR];
  if (s < s1) {
    const long long t = a.seg.time_of(s);
#pragma unroll
    for (int m = 0; m < NR; ++m) {
      const int i = lane + 32 * m;
      nxt[m] = load_coef<CELL>(a, t * rowB + (long long)b * H + i, i < H);
    }
  }
  int buf = 0;
  for (; s < s1; ++s) {
    Coef<CELL> cur[NR];
#pragma unroll
    for (int m = 0; m < NR; ++m) cur[m] = nxt[m];
    if (s + 1 < s1) {                           // prefetch the next slot's coefficients
      const long long t = a.seg.time_of(s + 1);
#pragma unroll
      for (int m = 0; m < NR; ++m) {
        const int i = lane + 32 * m;
        nxt[m] = load_coef<CELL>(a, t * rowB + (long long)b * H + i, i < H);
      }
    }
    float* xb = xs + buf * XW;
    constexpr bool TRANS = CELL == BPPSA_JAC_RNN_TANH && NR == 1 && NC % 4 == 0;
    if constexpr (TRANS) {
      if (lane < HT) {                              // xb[i][j] = d_i c_j[i], four chains per store
#pragma unroll
        for (int j4 = 0; j4 < NC / 4; ++j4) {
          float4 v4;
          v4.x = (4 * j4 + 0 < nc) ? cur[0].c[0] * c[4 * j4 + 0][0] : 0.f;
          v4.y = (4 * j4 + 1 < nc) ? cur[0].c[0] * c[4 * j4 + 1][0] : 0.f;
          v4.z = (4 * j4 + 2 < nc) ? cur[0].c[0] * c[4 * j4 + 2][0] : 0.f;
          v4.w = (4 * j4 + 3 < nc) ? cur[0].c[0] * c[4 * j4 + 3][0] : 0.f;
          *reinterpret_cast<float4*>(xb + lane * NC + 4 * j4) = v4;
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < NC; ++j) {
#pragma unroll
        for (int m = 0; m < NR; ++m) {
          const int i = lane + 32 * m;
          if (i < HT) {
#pragma unroll
            for (int v = 0; v < NV; ++v) xb[(j * NV + v) * HT + i] = (j < nc) ? cur[m].c[v] * c[j][m] : 0.f;
          }
        }
      }
    }
    __syncwarp();
    {
      float acc[NC][NR];
      if constexpr (TRANS)
        matvec_multi_t<HT, NC>(w, xb, acc);
      else
        matvec_multi<CELL, HT, NR, NC>(w, xb, acc);    // chains j >= nc compute on zeros
#pragma unroll
      for (int j = 0; j < NC; ++j)
#pragma unroll
        for (int m = 0; m < NR; ++m) {
          if (CELL == BPPSA_JAC_GRU) acc[j][m] = fmaf(cur[m].c[3], c[j][m], acc[j][m]);
          c[j][m] = acc[j][m];
        }
    }
    buf ^= 1;
  }

  float* dst = agg_out + ((long long)b * n_out + q) * H * H;
#pragma unroll
  for (int j = 0; j < NC; ++j) {
    if (j < nc) {
      const int col = vec ? 0 : cg * NC + j;
#pragma unroll
      for (int m = 0; m < NR; ++m) {
        const int i = lane + 32 * m;
        if (i < H) dst[(long long)col * H + i] = c[j][m];
      }
    }
  }
}

template <int CELL, int HT>
__global__ void __launch_bounds__(128) leaf_down_kernel(LeafArgs a, int C, const float* __restrict__ carry,
                                                        long long nblk, float* __restrict__ grad_h,
                                                        float* __restrict__ grad_init, const float* __restrict__ e,
                                                        float* __restrict__ vec_out, float* __restrict__ head_out,
                                                        long long head_bstride) {
  constexpr int NR = (HT + 31) / 32;
  constexpr int NV = NX<CELL>::v;
  constexpr int XW = NV * HT;
  extern __shared__ __align__(16) float smem[];
  const int H = a.seg.H, B = a.seg.B;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  float* xs = smem + wib * 2 * XW;
  const long long task = (long long)blockIdx.x * (blockDim.x >> 5) + wib;
  if (task >= (long long)B * nblk) return;
  const long long q = task % nblk;
  const int b = (int)(task / nblk);
  const long long S = a.seg.S();
  const long long s0 = q * C, s1 = min(s0 + (long long)C, S);
  const bool vec = a.seg.head && q == 0;
  const bool vonly = vec_out != nullptr;     // affine vector part of the block

  float w[NV][NR][HT];
  load_w<CELL, HT, NR>(a, H, lane, w);

  float v[NR];
#pragma unroll
  for (int m = 0; m < NR; ++m) {
    const int i = lane + 32 * m;
    v[m] = 0.f;
    if (i < H) {
      if (vec)
        v[m] = __ldg(a.seed + (long long)b * H + i);
      else if (!vonly)
        v[m] = __ldg(carry + (q + (long long)b * nblk) * H + i);
    }
  }
  const long long rowB = (long long)B * H;
  long long s = vec ? 1 : s0;
  // the walk is a dependent GEMV chain: the h rows of the next PF steps are in
  // flight as asynchronous copies into a per-warp shared-memory ring (one step
  // of register prefetch left a lone chain bound by HBM latency, ~700 ns per
  // step in the linear scan; a register ring stalls on its own loads)
  constexpr int PF = 8, NA = NArr<CELL>::v, SLOT = NA * 32;   // slot: [NA][32] floats (HT <= 32 per row group)
  float* ring = smem + (blockDim.x >> 5) * 2 * XW + wib * PF * SLOT * NR;   // after every warp's x buffers
  auto stage = [&](long long sp) {                              // step sp -> ring slot sp % PF
    if (sp < s1) {
      const long long t = a.seg.time_of(sp);
      float* dst = ring + (int)(sp % PF) * SLOT * NR;
#pragma unroll
      for (int m = 0; m < NR; ++m) {
        const int i = lane + 32 * m;
        if (i < H)
#pragma unroll
          for (int k = 0; k < NA; ++k) cpa4(dst + (m * NA + k) * 32 + lane, arr_ptr<CELL>(a, k) + (t * B + b) * H + i);
      }
    }
    cpa_commit();                                               // one group per step, empty or not
  };
#pragma unroll 1
  for (int u = 0; u < PF; ++u) stage(s + u);
  int buf = 0;
  bool done = false;
  for (; s < s1 && !done; s += PF) {
#pragma unroll 1
    for (int u = 0; u < PF; ++u) {                // not unrolled: one copy of the GEMV body (i-cache)
      const long long su = s + u;
      if (su >= s1 || done) break;
      const long long t = a.seg.time_of(su);
      if (!vonly) {
#pragma unroll
        for (int m = 0; m < NR; ++m) {
          const int i = lane + 32 * m;
          if (i < H) grad_h[t * rowB + (long long)b * H + i] = v[m];
        }
      }
      const bool last = (su + 1 == s1);
      const bool total = !vonly && last && s1 == S && grad_init != nullptr;
      if (last && !total && !vonly) {
        done = true;
        break;
      }
      cpa_wait<PF - 1>();                         // step su's group has landed (this lane's copies)
      __syncwarp();
      Coef<CELL> cur[NR];
      {
        const float* slot = ring + (int)(su % PF) * SLOT * NR;
#pragma unroll
        for (int m = 0; m < NR; ++m) cur[m] = coef_from<CELL>(slot + m * NA * 32, lane, lane + 32 * m < H);
      }
      __syncwarp();                               // every lane has read the slot before it is refilled
      stage(su + PF);
      float ev[NR];                               // e_{t-1}, loaded ahead of the GEMV
#pragma unroll
      for (int m = 0; m < NR; ++m) {
        const int i = lane + 32 * m;
        ev[m] = (e != nullptr && t >= 1 && i < H) ? __ldg(e + (t - 1) * rowB + (long long)b * H + i) : 0.f;
      }
      float* xb = xs + buf * XW;
#pragma unroll
      for (int m = 0; m < NR; ++m) {
        const int i = lane + 32 * m;
        if (i < HT) {
#pragma unroll
          for (int vv = 0; vv < NV; ++vv) xb[vv * HT + i] = cur[m].c[vv] * v[m];
        }
      }
      __syncwarp();
      float acc[NR];
      matvec<CELL, HT, NR, 4>(w, xb, acc);
#pragma unroll
      for (int m = 0; m < NR; ++m) {
        if (CELL == BPPSA_JAC_GRU) acc[m] = fmaf(cur[m].c[3], v[m], acc[m]);
        v[m] = acc[m] + ev[m];
      }
      buf ^= 1;
      if (total) {
#pragma unroll
        for (int m = 0; m < NR; ++m) {
          const int i = lane + 32 * m;
          if (i < H) grad_init[(long long)b * H + i] = v[m];
        }
      }
    }
  }
  cpa_wait<0>();                                  // no copy left in flight at exit
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

constexpr int kWarpsPerCta = 4;

// L2 prefetch of the h row of step ss (a row of H <= 32 floats spans at most two 128-B lines)
__device__ __forceinline__ void prefetch_row_l2(const float* hr, int H) {
  asm volatile("prefetch.global.L2 [%0];\n" ::"l"(hr));
  asm volatile("prefetch.global.L2 [%0];\n" ::"l"(hr + H - 1));
}
constexpr int kRowPF = 8;                            // steps of L2 prefetch ahead of the register row

// Level-0 fold for the tanh RNN at H <= 32 with one CHAIN per lane (r02g).
// leaf_up_kernel maps lanes to the H output rows, which leaves 12 of 32 lanes
// idle at H = 20; here lane = column chain j of block (b, q) (the H chains of
// a block on consecutive lanes share the block's h rows through L1), x = d o c
// lives in the lane's registers and W (zero-padded to HT x HT) is read from
// shared memory as warp-wide broadcasts.  Same arithmetic in the same order as
// leaf_up_kernel (x_k = d_k c_k, c'_i = sum over k = 0.. of fma(x_k, W[k][i], .)),
// so the results are bit-identical.  Output: column j of the block aggregate
// (column-major, as launch_leaf_up); the head block's single chain is the seed.
template <int HT, int NCH>
__global__ void __launch_bounds__(128) leaf_up_lc_kernel(LeafArgs a, int C, float* __restrict__ agg_out,
                                                        long long n_out, long long q0, long long nq) {
  // NCH chains per lane (cols jl, jl + L, ..., L = ceil(H / NCH) lanes per
  // block): each shared-memory W load feeds NCH chains
  __shared__ __align__(16) float Ws[HT][HT];       // Ws[k][i] = W[k][i]
  const int H = a.seg.H, B = a.seg.B;
  for (int e = threadIdx.x; e < HT * HT; e += blockDim.x) {
    const int k = e / HT, i = e % HT;
    Ws[k][i] = (k < H && i < H) ? __ldg(a.W + (long long)k * H + i) : 0.f;
  }
  __syncthreads();
  const int L = (H + NCH - 1) / NCH;
  const long long task = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (task >= (long long)B * nq * L) return;
  const int jl = (int)(task % L);
  const long long rest = task / L;
  const long long q = q0 + rest % nq;
  const int b = (int)(rest / nq);
  const bool vec = a.seg.head && q == 0;
  if (vec && jl > 0) return;                         // the head block carries one chain: the seed
  const long long S = a.seg.S();
  const long long s1 = min(q * C + (long long)C, S);
  long long s = vec ? 1 : q * C;
  float c[NCH][HT];
#pragma unroll
  for (int u = 0; u < NCH; ++u)
#pragma unroll
    for (int i = 0; i < HT; ++i)
      c[u][i] = vec ? ((u == 0 && i < H) ? __ldg(a.seed + (long long)b * H + i) : 0.f) : (i == jl + u * L ? 1.f : 0.f);
  const long long rowB = (long long)B * H;
  float hn[HT];                                      // the next step's h row (prefetched)
  // a whole row in HT / 4 float4 loads (rows are 16-B aligned when h is)
  const bool full = H == HT && (reinterpret_cast<uintptr_t>(a.h) & 15) == 0;
  auto load_row = [&](long long ss) {
    const float* hr = a.h + (long long)a.seg.time_of(ss) * rowB + (long long)b * H;
    if (full) {
#pragma unroll
      for (int k4 = 0; k4 < HT / 4; ++k4) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(hr) + k4);
        hn[4 * k4] = v.x, hn[4 * k4 + 1] = v.y, hn[4 * k4 + 2] = v.z, hn[4 * k4 + 3] = v.w;
      }
    } else {
#pragma unroll
      for (int k = 0; k < HT; ++k) hn[k] = k < H ? __ldg(hr + k) : 0.f;
    }
  };
  if (s < s1) load_row(s);
  for (; s < s1; ++s) {
    float x[NCH][HT];
#pragma unroll
    for (int k = 0; k < HT; ++k) {
      const float d = 1.f - hn[k] * hn[k];
#pragma unroll
      for (int u = 0; u < NCH; ++u) x[u][k] = d * c[u][k];
    }
    if (s + 1 < s1) load_row(s + 1);
    if (s + kRowPF < s1 && jl == 0)                 // one lane of the block prefetches
      prefetch_row_l2(a.h + (long long)a.seg.time_of(s + kRowPF) * rowB + (long long)b * H, H);
    float2 acc[NCH][HT / 2];
#pragma unroll
    for (int u = 0; u < NCH; ++u)
#pragma unroll
      for (int p = 0; p < HT / 2; ++p) acc[u][p] = make_float2(0.f, 0.f);
#pragma unroll
    for (int k = 0; k < HT; ++k) {
#pragma unroll
      for (int p4 = 0; p4 < HT / 4; ++p4) {
        const float4 w4 = *reinterpret_cast<const float4*>(&Ws[k][4 * p4]);
#pragma unroll
        for (int u = 0; u < NCH; ++u) {
          const float2 xk = make_float2(x[u][k], x[u][k]);
          acc[u][2 * p4] = __ffma2_rn(xk, make_float2(w4.x, w4.y), acc[u][2 * p4]);
          acc[u][2 * p4 + 1] = __ffma2_rn(xk, make_float2(w4.z, w4.w), acc[u][2 * p4 + 1]);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < NCH; ++u)
#pragma unroll
      for (int p = 0; p < HT / 2; ++p) {
        c[u][2 * p] = acc[u][p].x;
        c[u][2 * p + 1] = acc[u][p].y;
      }
  }
#pragma unroll
  for (int u = 0; u < NCH; ++u) {
    const int col = vec ? 0 : jl + u * L;
    if ((vec && u > 0) || col >= H) continue;
    float* dst = agg_out + ((long long)b * n_out + q) * H * H + (long long)col * H;
#pragma unroll
    for (int i = 0; i < HT; ++i)
      if (i < H) dst[i] = c[u][i];
  }
}

template <int HT, int NCH>
cudaError_t up_lc_impl(const LeafArgs& a, int C, float* agg_out, long long n_out, long long q0, long long nq,
                       cudaStream_t st) {
  const long long tasks = (long long)a.seg.B * nq * ((a.seg.H + NCH - 1) / NCH);
  if (tasks == 0) return cudaSuccess;
  leaf_up_lc_kernel<HT, NCH><<<(unsigned)((tasks + 127) / 128), 128, 0, st>>>(a, C, agg_out, n_out, q0, nq);
  return cudaGetLastError();
}

// The GRU form (H <= 20): the J^T of eqn:gru_jcb needs three matrix-vector
// products per step (W_hr, W_hn, W_hz against c scaled by the gate
// coefficients) plus the diagonal z term.  Each lane forms the step's
// coefficients for all k from the block's five tape rows (shared through L1
// by the block's lanes), then the products with the three W in shared memory.
// Same arithmetic and order as leaf_up_kernel<GRU> (load_coef; v = r, n, z
// outer, k inner; then fma(z, c, .)).
template <int HT, int NCH>
__global__ void __launch_bounds__(128) leaf_up_lc_gru_kernel(LeafArgs a, int C, float* __restrict__ agg_out,
                                                            long long n_out, long long q0, long long nq) {
  __shared__ __align__(16) float Ws[3][HT][HT];    // [v][k][i] = W_hh3[(vrow + k) H + i], vrow = 0, 2H, H
  const int H = a.seg.H, B = a.seg.B;
  for (int e = threadIdx.x; e < 3 * HT * HT; e += blockDim.x) {
    const int v = e / (HT * HT), k = (e / HT) % HT, i = e % HT;
    const int vrow = v == 0 ? 0 : (v == 1 ? 2 * H : H);
    Ws[v][k][i] = (k < H && i < H) ? __ldg(a.W + (long long)(vrow + k) * H + i) : 0.f;
  }
  __syncthreads();
  // NCH chains per lane (cols jl, jl + L, ..., L = ceil(H / NCH)): the step's
  // gate coefficients and every W load serve all of them
  const int L = (H + NCH - 1) / NCH;
  const long long task = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (task >= (long long)B * nq * L) return;
  const int jl = (int)(task % L);
  const long long rest = task / L;
  const long long q = q0 + rest % nq;
  const int b = (int)(rest / nq);
  const bool vec = a.seg.head && q == 0;
  if (vec && jl > 0) return;
  const long long S = a.seg.S();
  const long long s1 = min(q * C + (long long)C, S);
  long long s = vec ? 1 : q * C;
  float c[NCH][HT];
#pragma unroll
  for (int u = 0; u < NCH; ++u)
#pragma unroll
    for (int i = 0; i < HT; ++i)
      c[u][i] = vec ? ((u == 0 && i < H) ? __ldg(a.seed + (long long)b * H + i) : 0.f) : (i == jl + u * L ? 1.f : 0.f);
  const long long rowB = (long long)B * H;
  for (; s < s1; ++s) {
    const long long off = (long long)a.seg.time_of(s) * rowB + (long long)b * H;
    if (s + kRowPF < s1 && jl == 0) {
      const long long offp = (long long)a.seg.time_of(s + kRowPF) * rowB + (long long)b * H;
      prefetch_row_l2(a.r + offp, H), prefetch_row_l2(a.z + offp, H), prefetch_row_l2(a.n + offp, H);
      prefetch_row_l2(a.M + offp, H), prefetch_row_l2(a.hp + offp, H);
    }
    float cf[4][HT];
#pragma unroll
    for (int k = 0; k < HT; ++k) {
      const Coef<BPPSA_JAC_GRU> co = load_coef<BPPSA_JAC_GRU>(a, off + k, k < H);
      cf[0][k] = co.c[0], cf[1][k] = co.c[1], cf[2][k] = co.c[2], cf[3][k] = co.c[3];
    }
    float2 acc[NCH][HT / 2];
#pragma unroll
    for (int u = 0; u < NCH; ++u)
#pragma unroll
      for (int p2 = 0; p2 < HT / 2; ++p2) acc[u][p2] = make_float2(0.f, 0.f);
#pragma unroll
    for (int v = 0; v < 3; ++v)
#pragma unroll
      for (int k = 0; k < HT; ++k) {
        float2 xk[NCH];
#pragma unroll
        for (int u = 0; u < NCH; ++u) {
          const float xv = cf[v][k] * c[u][k];
          xk[u] = make_float2(xv, xv);
        }
#pragma unroll
        for (int p4 = 0; p4 < HT / 4; ++p4) {
          const float4 w4 = *reinterpret_cast<const float4*>(&Ws[v][k][4 * p4]);
#pragma unroll
          for (int u = 0; u < NCH; ++u) {
            acc[u][2 * p4] = __ffma2_rn(xk[u], make_float2(w4.x, w4.y), acc[u][2 * p4]);
            acc[u][2 * p4 + 1] = __ffma2_rn(xk[u], make_float2(w4.z, w4.w), acc[u][2 * p4 + 1]);
          }
        }
      }
#pragma unroll
    for (int u = 0; u < NCH; ++u)
#pragma unroll
      for (int p2 = 0; p2 < HT / 2; ++p2) {
        c[u][2 * p2] = fmaf(cf[3][2 * p2], c[u][2 * p2], acc[u][p2].x);
        c[u][2 * p2 + 1] = fmaf(cf[3][2 * p2 + 1], c[u][2 * p2 + 1], acc[u][p2].y);
      }
  }
#pragma unroll
  for (int u = 0; u < NCH; ++u) {
    const int col = vec ? 0 : jl + u * L;
    if ((vec && u > 0) || col >= H) continue;
    float* dst = agg_out + ((long long)b * n_out + q) * H * H + (long long)col * H;
#pragma unroll
    for (int i = 0; i < HT; ++i)
      if (i < H) dst[i] = c[u][i];
  }
}

template <int CELL, int HT, int NC>
cudaError_t up_impl(const LeafArgs& a, int C, float* agg_out, long long n_out, long long q0, long long nq,
                    cudaStream_t st) {
  const int G = (a.seg.H + NC - 1) / NC;
  const long long tasks = (long long)a.seg.B * nq * G;
  if (tasks == 0) return cudaSuccess;
  const long long grid = (tasks + kWarpsPerCta - 1) / kWarpsPerCta;
  const size_t smem = (size_t)kWarpsPerCta * 2 * NC * NX<CELL>::v * HT * sizeof(float);
  auto k = leaf_up_kernel<CELL, HT, NC>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  k<<<(unsigned)grid, 32 * kWarpsPerCta, smem, st>>>(a, C, agg_out, n_out, q0, nq);
  return cudaGetLastError();
}

// Level-0 walk for the tanh RNN at H <= 20 with one CHAIN per lane (r02g):
// chain (b, q) walks its block from the carry (the seed for the head block),
// writing the exclusive output grad_h[t(s)] = v at every slot and stepping
// v <- W^T (d_t o v) with the lane's own registers (leaf_down_kernel spends a
// warp per chain with 12 of 32 lanes idle at H = 20, and is issue-bound at the
// occupancy C1-C3 give it).  Same arithmetic and order as leaf_down_kernel's
// matvec (four partial sums over k mod 4, added in order), so the results are
// bit-identical.  Plain scans only (no affine term, no vector-only pass).
template <int HT>
__global__ void __launch_bounds__(128) leaf_down_lc_kernel(LeafArgs a, int C, const float* __restrict__ carry,
                                                          long long nblk, float* __restrict__ grad_h,
                                                          float* __restrict__ grad_init) {
  __shared__ __align__(16) float Ws[HT][HT];       // Ws[k][i] = W[k][i]
  const int H = a.seg.H, B = a.seg.B;
  for (int e = threadIdx.x; e < HT * HT; e += blockDim.x) {
    const int k = e / HT, i = e % HT;
    Ws[k][i] = (k < H && i < H) ? __ldg(a.W + (long long)k * H + i) : 0.f;
  }
  __syncthreads();
  const long long task = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (task >= (long long)B * nblk) return;
  const long long q = task % nblk;
  const int b = (int)(task / nblk);
  const long long S = a.seg.S();
  const long long s0 = q * C, s1 = min(s0 + (long long)C, S);
  const bool vec = a.seg.head && q == 0;
  float v[HT];
#pragma unroll
  for (int i = 0; i < HT; ++i)
    v[i] = i < H ? __ldg(vec ? a.seed + (long long)b * H + i : carry + (q + (long long)b * nblk) * H + i) : 0.f;
  const long long rowB = (long long)B * H;
  const bool full = H == HT && (reinterpret_cast<uintptr_t>(a.h) & 15) == 0 &&
                    (reinterpret_cast<uintptr_t>(grad_h) & 15) == 0;
  float hn[HT];
  auto load_row = [&](long long ss) {
    const float* hr = a.h + (long long)a.seg.time_of(ss) * rowB + (long long)b * H;
    if (full) {
#pragma unroll
      for (int k4 = 0; k4 < HT / 4; ++k4) {
        const float4 x4 = __ldg(reinterpret_cast<const float4*>(hr) + k4);
        hn[4 * k4] = x4.x, hn[4 * k4 + 1] = x4.y, hn[4 * k4 + 2] = x4.z, hn[4 * k4 + 3] = x4.w;
      }
    } else {
#pragma unroll
      for (int k = 0; k < HT; ++k) hn[k] = k < H ? __ldg(hr + k) : 0.f;
    }
  };
  long long s = vec ? 1 : s0;
  if (s < s1) load_row(s);
  for (; s < s1; ++s) {
    const long long t = a.seg.time_of(s);
    float* out = grad_h + t * rowB + (long long)b * H;
    if (full) {
#pragma unroll
      for (int k4 = 0; k4 < HT / 4; ++k4)
        reinterpret_cast<float4*>(out)[k4] = make_float4(v[4 * k4], v[4 * k4 + 1], v[4 * k4 + 2], v[4 * k4 + 3]);
    } else {
#pragma unroll
      for (int i = 0; i < HT; ++i)
        if (i < H) out[i] = v[i];
    }
    const bool last = s + 1 == s1;
    const bool total = last && s1 == S && grad_init != nullptr;
    if (last && !total) break;
    float x[HT];
#pragma unroll
    for (int k = 0; k < HT; ++k) {
      const float d = 1.f - hn[k] * hn[k];
      x[k] = d * v[k];
    }
    if (!last) load_row(s + 1);
    if (s + kRowPF < s1) prefetch_row_l2(a.h + (long long)a.seg.time_of(s + kRowPF) * rowB + (long long)b * H, H);
    float part[4][HT];
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
      for (int i = 0; i < HT; ++i) part[p][i] = 0.f;
#pragma unroll
    for (int k = 0; k < HT; ++k) {
#pragma unroll
      for (int i4 = 0; i4 < HT / 4; ++i4) {
        const float4 w4 = *reinterpret_cast<const float4*>(&Ws[k][4 * i4]);
        part[k % 4][4 * i4] = fmaf(w4.x, x[k], part[k % 4][4 * i4]);
        part[k % 4][4 * i4 + 1] = fmaf(w4.y, x[k], part[k % 4][4 * i4 + 1]);
        part[k % 4][4 * i4 + 2] = fmaf(w4.z, x[k], part[k % 4][4 * i4 + 2]);
        part[k % 4][4 * i4 + 3] = fmaf(w4.w, x[k], part[k % 4][4 * i4 + 3]);
      }
    }
#pragma unroll
    for (int i = 0; i < HT; ++i) {
      float r = part[0][i];
      r += part[1][i];
      r += part[2][i];
      r += part[3][i];
      v[i] = r;
    }
    if (total) {
#pragma unroll
      for (int i = 0; i < HT; ++i)
        if (i < H) grad_init[(long long)b * H + i] = v[i];
    }
  }
}

struct DownX {   // the affine extras of the level-0 walk
  const float* e;
  float *vec_out, *head_out;
  long long head_bstride;
};

template <int CELL, int HT>
cudaError_t down_impl(const LeafArgs& a, int C, const float* carry, long long nblk, float* grad_h,
                      float* grad_init, cudaStream_t st, const DownX& x) {
  const long long tasks = (long long)a.seg.B * nblk;
  const long long grid = (tasks + kWarpsPerCta - 1) / kWarpsPerCta;
  const int NRr = (HT + 31) / 32;
  const size_t smem = (size_t)kWarpsPerCta * (2 * NX<CELL>::v * HT + 8 * NArr<CELL>::v * 32 * NRr) * sizeof(float);
  leaf_down_kernel<CELL, HT><<<(unsigned)grid, 32 * kWarpsPerCta, smem, st>>>(
      a, C, carry, nblk, grad_h, grad_init, x.e, x.vec_out, x.head_out, x.head_bstride);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_leaf_up(const LeafArgs& a, int C, float* agg_out, long long n_out, long long q0,
                           long long nq, cudaStream_t st) {
  const int H = a.seg.H;
  if (a.kind == BPPSA_JAC_RNN_TANH) {
#ifndef BPPSA_LEAF_UP_ROWS                           // (the lane-per-row form, for A/B)
#ifndef BPPSA_LC_NCH
#define BPPSA_LC_NCH 2
#endif
    if (H <= 20) return up_lc_impl<20, BPPSA_LC_NCH>(a, C, agg_out, n_out, q0, nq, st);
    if (H <= 32) return up_lc_impl<32, 1>(a, C, agg_out, n_out, q0, nq, st);
#endif
    if (H == 20) return up_impl<BPPSA_JAC_RNN_TANH, 20, 20>(a, C, agg_out, n_out, q0, nq, st);
    if (H <= 32) return up_impl<BPPSA_JAC_RNN_TANH, 32, 16>(a, C, agg_out, n_out, q0, nq, st);
    return up_impl<BPPSA_JAC_RNN_TANH, 64, 8>(a, C, agg_out, n_out, q0, nq, st);
  }
#ifndef BPPSA_LEAF_UP_ROWS
  if (H <= 20) {
#ifndef BPPSA_LC_GRU_NCH
#define BPPSA_LC_GRU_NCH 2
#endif
    constexpr int NCH = BPPSA_LC_GRU_NCH;
    const long long tasks = (long long)a.seg.B * nq * ((H + NCH - 1) / NCH);
    if (tasks == 0) return cudaSuccess;
    leaf_up_lc_gru_kernel<20, NCH><<<(unsigned)((tasks + 127) / 128), 128, 0, st>>>(a, C, agg_out, n_out, q0, nq);
    return cudaGetLastError();
  }
#endif
  if (H == 20) return up_impl<BPPSA_JAC_GRU, 20, 10>(a, C, agg_out, n_out, q0, nq, st);
  return up_impl<BPPSA_JAC_GRU, 32, 8>(a, C, agg_out, n_out, q0, nq, st);
}

cudaError_t launch_leaf_down(const LeafArgs& a, int C, const float* carry, long long nblk,
                             float* grad_h, float* grad_init, cudaStream_t st, const float* e, float* vec_out,
                             float* head_out, long long head_bstride) {
  const int H = a.seg.H;
  const DownX x{e, vec_out, head_out, head_bstride};
  if (a.kind == BPPSA_JAC_RNN_TANH) {
#ifndef BPPSA_LEAF_DOWN_ROWS                         // (the warp-per-chain form, for A/B)
    // one chain per lane pays once there are enough chains to fill the SMs
    // (C2: 15000 at block0 32); few long chains (LINEAR mode's sequential BP,
    // C1's 2000) keep the warp-per-chain kernel and its 8-step cp.async ring
    const long long tasks = (long long)a.seg.B * nblk;
    if (H <= 20 && e == nullptr && vec_out == nullptr && tasks >= 4096) {
      leaf_down_lc_kernel<20><<<(unsigned)((tasks + 127) / 128), 128, 0, st>>>(a, C, carry, nblk, grad_h, grad_init);
      return cudaGetLastError();
    }
#endif
    if (H == 20) return down_impl<BPPSA_JAC_RNN_TANH, 20>(a, C, carry, nblk, grad_h, grad_init, st, x);
    if (H <= 32) return down_impl<BPPSA_JAC_RNN_TANH, 32>(a, C, carry, nblk, grad_h, grad_init, st, x);
    return down_impl<BPPSA_JAC_RNN_TANH, 64>(a, C, carry, nblk, grad_h, grad_init, st, x);
  }
  if (H == 20) return down_impl<BPPSA_JAC_GRU, 20>(a, C, carry, nblk, grad_h, grad_init, st, x);
  return down_impl<BPPSA_JAC_GRU, 32>(a, C, carry, nblk, grad_h, grad_init, st, x);
}

}  // namespace bppsa
