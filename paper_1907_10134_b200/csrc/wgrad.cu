// wgrad.cu — parameter gradients (eqn:update_param) for tied
// recurrent weights summed over time:  dW = sum_{t,b} delta_{t,b} u_{t,b}^T.
//
// One contraction over K = T*B rows: out[a][c] = sum_rows A_row[a] * U_row[c]
//   RNN: A = delta = (1-h^2) o grad_h              (NA = H)
//   GRU: A = [dR | dZ | dN | dM]                     (NA = 4H)
//   U   = [h_{t-1} (H) | x_t (I) | 1]                (H + I + 1 columns)
// Rows are split into a fixed number of parts (a function of K only).  A CTA
// owns one part and a 64-row slice of A: the H x 64 "hidden" block sits in a
// 4x4-per-thread register tile, the (I + 1) "extra" columns are spread over
// the threads; row stages of 32 are double-buffered through shared memory
// (the next stage's operands are loaded while the current one is consumed).
// Partial tiles go to the workspace and a second kernel sums the parts in a
// fixed order — deterministic, no float atomics, round-to-nearest FFMA.
#include <algorithm>

#include "common.cuh"

namespace bppsa {
namespace {

constexpr int TA = 64, RR = 32, NT = 256, MAXE = 64;
// tile shapes: <64, 64>: 64-wide A and U tiles, 256 threads (H up to 64);
// <32, 16>: 32-wide tiles, 64 threads, up to 16 extra columns (H <= 32:
// configs 1-3 have H = 20, where the 64-wide tile was 90 % padding)
template <int TA_, int MAXE_>
struct WT {
  static constexpr int NT = (TA_ / 4) * (TA_ / 4);
  static constexpr int PER = RR * TA_ / NT;       // A and U (hidden part) elements per thread per stage
  static constexpr int PE = MAXE_ * RR / NT;      // extra-column elements per thread per stage
  static constexpr int NEA = 16;                  // extra outputs per thread
};

struct WArgs {
  int T, B, H, I, kind;
  const float *x, *h, *h_init, *g;              // RNN (h) / both (x, g)
  const float *hp, *r, *z, *n, *M;              // GRU
  long long rows, rows_per_part;
  int NA, E;                                    // E = I + 1 extra columns
};

__device__ __forceinline__ float valA(const WArgs& w, long long row, int a) {
  if (a >= w.NA) return 0.f;
  if (w.kind == BPPSA_JAC_RNN_TANH) {
    const long long o = row * w.H + a;
    const float hv = w.h[o];
    return (1.f - hv * hv) * w.g[o];
  }
  const int gate = a / w.H, i = a - gate * w.H;
  const long long o = row * w.H + i;
  const float g = w.g[o], z = w.z[o], n = w.n[o];
  const float dN = g * (1.f - z) * (1.f - n * n);
  if (gate == 2) return dN;
  if (gate == 1) return g * (w.hp[o] - n) * z * (1.f - z);
  const float r = w.r[o];
  if (gate == 0) return dN * w.M[o] * r * (1.f - r);
  return dN * r;
}

__device__ __forceinline__ float valU(const WArgs& w, long long row, int c) {   // hidden part, c < H
  if (c >= w.H) return 0.f;
  if (w.kind == BPPSA_JAC_GRU) return w.hp[row * w.H + c];
  if (row >= w.B) return w.h[(row - w.B) * w.H + c];             // h_{t-1}
  return w.h_init ? w.h_init[row * w.H + c] : 0.f;                 // t = 0: row = b
}

__device__ __forceinline__ float valE(const WArgs& w, long long row, int c) {   // extra part
  return (c < w.I) ? w.x[row * w.I + c] : 1.f;
}

template <int TA, int MAXE>
__global__ void __launch_bounds__(WT<TA, MAXE>::NT) wgrad_partial_kernel(WArgs w, float* __restrict__ ws) {
  constexpr int NT = WT<TA, MAXE>::NT, PER_A = WT<TA, MAXE>::PER, PER_U = WT<TA, MAXE>::PER;
  constexpr int GI = TA / 4;
  __shared__ __align__(16) float As[2][RR][TA];
  __shared__ __align__(16) float Us[2][RR][TA];
  __shared__ float Es[2][RR][MAXE];
  const int part = blockIdx.x, ta = blockIdx.y;
  const long long r0 = (long long)part * w.rows_per_part;
  const long long r1 = min(r0 + w.rows_per_part, w.rows);
  const int tid = threadIdx.x, ti = tid % GI, tj = tid / GI;
  const int nE = TA * w.E;                          // extra outputs of this A slice
  float acc[4][4];
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) acc[x][y] = 0.f;
  float eacc[WT<TA, MAXE>::NEA];
#pragma unroll
  for (int u = 0; u < WT<TA, MAXE>::NEA; ++u) eacc[u] = 0.f;

  float pa[PER_A], pu[PER_U], pe[WT<TA, MAXE>::PE];
  auto fetch = [&](long long rb) {
#pragma unroll
    for (int u = 0; u < PER_A; ++u) {
      const int e = tid + u * NT, rr = e / TA, col = e % TA;
      const long long row = rb + rr;
      pa[u] = (row < r1) ? valA(w, row, ta * TA + col) : 0.f;
      pu[u] = (row < r1) ? valU(w, row, col) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < WT<TA, MAXE>::PE; ++u) {
      const int e = tid + u * NT, rr = e / MAXE, col = e % MAXE;
      const long long row = rb + rr;
      pe[u] = (row < r1 && col < w.E) ? valE(w, row, col) : 0.f;
    }
  };
  auto stash = [&](int buf) {
#pragma unroll
    for (int u = 0; u < PER_A; ++u) {
      const int e = tid + u * NT, rr = e / TA, col = e % TA;
      As[buf][rr][col] = pa[u];
      Us[buf][rr][col] = pu[u];
    }
#pragma unroll
    for (int u = 0; u < WT<TA, MAXE>::PE; ++u) {
      const int e = tid + u * NT;
      Es[buf][e / MAXE][e % MAXE] = pe[u];
    }
  };

  fetch(r0);
  stash(0);
  __syncthreads();
  int buf = 0;
  for (long long rb = r0; rb < r1; rb += RR) {
    const bool more = rb + RR < r1;
    if (more) fetch(rb + RR);                        // loads in flight during the FMAs
#pragma unroll 4
    for (int rr = 0; rr < RR; ++rr) {
      const float4 a4 = *reinterpret_cast<const float4*>(&As[buf][rr][ti * 4]);
      const float4 u4 = *reinterpret_cast<const float4*>(&Us[buf][rr][tj * 4]);
      const float av[4] = {a4.x, a4.y, a4.z, a4.w};
      const float uv[4] = {u4.x, u4.y, u4.z, u4.w};
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) acc[x][y] = fmaf(av[x], uv[y], acc[x][y]);
    }
    for (int u = 0; u < WT<TA, MAXE>::NEA; ++u) {   // extra columns: x_t and the bias
      const int e = tid + u * NT;
      if (e >= nE) break;
      const int a = e / w.E, c = e % w.E;
      float s = eacc[u];
      for (int rr = 0; rr < RR; ++rr) s = fmaf(As[buf][rr][a], Es[buf][rr][c], s);
      eacc[u] = s;
    }
    if (more) stash(buf ^ 1);
    __syncthreads();
    buf ^= 1;
  }
  const int NB = w.H + w.E;
  float* dst = ws + (long long)part * w.NA * NB;
#pragma unroll
  for (int x = 0; x < 4; ++x) {
    const int a = ta * TA + ti * 4 + x;
    if (a >= w.NA) continue;
#pragma unroll
    for (int y = 0; y < 4; ++y) {
      const int c = tj * 4 + y;
      if (c < w.H) dst[(long long)a * NB + c] = acc[x][y];
    }
  }
  for (int u = 0; u < WT<TA, MAXE>::NEA; ++u) {
    const int e = tid + u * NT;
    if (e >= nE) break;
    const int a = ta * TA + e / w.E, c = e % w.E;
    if (a < w.NA) dst[(long long)a * NB + w.H + c] = eacc[u];
  }
}

// Reduction of the partial slabs: block = 32 outputs x 32 part lanes; lane pl
// sums parts pl, pl+32, ... in order, then a fixed shared-memory tree over pl.
// The summation order depends on P only (deterministic), loads are coalesced
// across outputs.
struct RedMap {
  int gru, H, I, NA, NB;
  float *o0, *o1, *o2, *o3;   // RNN: dW_hh, dW_ih, db;  GRU: dW_hh3, dW_ih3, db_ih3, db_hh3
};

__device__ __forceinline__ float* map_out(const RedMap& m, int e, int& a, int& c) {
  const int H = m.H, I = m.I;
  if (!m.gru) {
    a = e / m.NB;
    c = e % m.NB;
    return c < H ? m.o0 + a * H + c : (c < H + I ? m.o1 + a * I + (c - H) : m.o2 + a);
  }
  const int n_hh = 3 * H * H, n_ih = 3 * H * I;
  if (e < n_hh) {
    const int row = e / H, k = e % H, g = row / H, i = row % H;
    a = (g == 2 ? 3 : g) * H + i;                      // [dR; dZ; dM] h_prev^T
    c = k;
    return m.o0 + e;
  }
  if (e < n_hh + n_ih) {
    const int f = e - n_hh;
    a = f / I;                                          // [dR; dZ; dN] x^T
    c = H + f % I;
    return m.o1 + f;
  }
  if (e < n_hh + n_ih + 3 * H) {
    a = e - n_hh - n_ih;
    c = H + I;
    return m.o2 + a;
  }
  const int row = e - n_hh - n_ih - 3 * H, g = row / H, i = row % H;
  a = (g == 2 ? 3 : g) * H + i;
  c = H + I;
  return m.o3 + row;
}

__global__ void __launch_bounds__(1024) wgrad_reduce(const float* __restrict__ ws, long long P, RedMap m,
                                                     int total) {
  __shared__ float red[32][33];
  const int o = threadIdx.x & 31, pl = threadIdx.x >> 5;
  const int e = blockIdx.x * 32 + o;
  float s = 0.f;
  float* out = nullptr;
  if (e < total) {
    int a, c;
    out = map_out(m, e, a, c);
    const long long stride = (long long)m.NA * m.NB;
    const float* p = ws + (long long)a * m.NB + c;
    long long q = pl;
    for (; q + 96 < P; q += 128) {        // four loads in flight, summed in part order
      const float v0 = __ldg(p + q * stride), v1 = __ldg(p + (q + 32) * stride), v2 = __ldg(p + (q + 64) * stride),
                  v3 = __ldg(p + (q + 96) * stride);
      s += v0;
      s += v1;
      s += v2;
      s += v3;
    }
    for (; q < P; q += 32) s += __ldg(p + q * stride);
  }
  red[pl][o] = s;
  __syncthreads();
#pragma unroll
  for (int w = 16; w >= 1; w >>= 1) {
    if (pl < w) red[pl][o] += red[pl + w][o];
    __syncthreads();
  }
  if (pl == 0 && e < total) *out = red[0][o];
}

cudaError_t reduce_rnn(const float* ws, long long P, int H, int I, float* dW_ih, float* dW_hh, float* db,
                       cudaStream_t st) {
  const RedMap m{0, H, I, H, H + I + 1, dW_hh, dW_ih, db, nullptr};
  const int total = H * (H + I + 1);
  wgrad_reduce<<<(total + 31) / 32, 1024, 0, st>>>(ws, P, m, total);
  return cudaGetLastError();
}

// RNN, H <= 20, I + 1 <= 4 (configs 1-2; r02i): the part's rows go through a
// cp.async ring of 64-row stages (h, grad_h and h_prev rows as they lie in
// memory, several stages in flight: the tile kernel above keeps one 32-row
// stage in flight in registers and sat at 25 % occupancy waiting on loads).
// Thread = (4 x 4 output tile, row group): ceil(H/4)^2 tiles x SG groups; each
// forms delta = (1 - h^2) g for its four rows of a on the fly from the staged
// rows, the tile of column block 0 also the x / bias columns; the row groups
// are summed in a fixed order at the end (deterministic).
constexpr int SM_H = 20, SM_TL = SM_H / 4, SM_TILES = SM_TL * SM_TL, SM_SG = 10, SM_NT = 256;
constexpr int SM_RS = 64, SM_NS = 4, SM_EMAX = 4;
constexpr int SM_STAGE = 3 * SM_RS * SM_H + SM_RS * SM_EMAX;   // floats: h | g | h_prev | x rows
__global__ void __launch_bounds__(SM_NT) wgrad_rnn_small_kernel(WArgs w, float* __restrict__ ws) {
  extern __shared__ __align__(16) float sm[];
  const int H = w.H, I = w.I, E = w.E;
  const int part = blockIdx.x, tid = threadIdx.x;
  const long long r0 = (long long)part * w.rows_per_part;
  const long long r1 = min(r0 + w.rows_per_part, w.rows);
  const int nst = (int)((r1 - r0 + SM_RS - 1) / SM_RS);
  // stage loader: 16-byte cp.async when the rows are 16-byte aligned (H % 4 == 0
  // and aligned bases: the rows of a stage are one contiguous run per array),
  // else 4-byte copies
  auto al16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
  const bool v16 = H % 4 == 0 && al16(w.h) && al16(w.g) && (w.h_init == nullptr || al16(w.h_init));
  const bool x16 = I > 0 && al16(w.x) && (SM_RS * I) % 4 == 0;
  auto cp4 = [](float* d, const float* g) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"((unsigned)__cvta_generic_to_shared(d)), "l"(g)
                 : "memory");
  };
  auto cp16 = [](float* d, const float* g) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"((unsigned)__cvta_generic_to_shared(d)), "l"(g)
                 : "memory");
  };
  auto load = [&](int k) {
    if (k < nst) {
      float* dst = sm + (k % SM_NS) * SM_STAGE;
      const long long rb = r0 + (long long)k * SM_RS;
      const int n = (int)min((long long)SM_RS, r1 - rb);
      const int step = v16 ? 4 : 1;
      for (int e = tid * step; e < n * H; e += SM_NT * step) {
        const long long row = rb + e / H;
        const int c = e % H;
        const float* hp = row >= w.B ? w.h + (row - w.B) * H + c : (w.h_init ? w.h_init + row * H + c : nullptr);
        if (v16) {
          cp16(dst + e, w.h + rb * H + e);
          cp16(dst + SM_RS * H + e, w.g + rb * H + e);
          if (hp) cp16(dst + 2 * SM_RS * H + e, hp);
          else *reinterpret_cast<float4*>(dst + 2 * SM_RS * H + e) = make_float4(0.f, 0.f, 0.f, 0.f);
        } else {
          cp4(dst + e, w.h + rb * H + e);
          cp4(dst + SM_RS * H + e, w.g + rb * H + e);
          if (hp) cp4(dst + 2 * SM_RS * H + e, hp);
          else dst[2 * SM_RS * H + e] = 0.f;
        }
      }
      if (x16 && n == SM_RS && ((rb * I) & 3) == 0) {   // (parts start anywhere: check the stage's x offset)
        for (int e = 4 * tid; e < n * I; e += 4 * SM_NT) cp16(dst + 3 * SM_RS * H + e, w.x + rb * I + e);
      } else {
        for (int e = tid; e < n * I; e += SM_NT) cp4(dst + 3 * SM_RS * H + e, w.x + rb * I + e);
      }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");   // one group per stage, empty or not
  };
  const int tile = tid % SM_TILES, rg = tid / SM_TILES;   // rg < SM_SG for the working threads
  const int ti = tile / SM_TL, tj = tile % SM_TL;
  const bool work = rg < SM_SG && 4 * ti < H && 4 * tj < H;
  float acc[4][4], eacc[4][SM_EMAX];
#pragma unroll
  for (int x = 0; x < 4; ++x) {
#pragma unroll
    for (int y = 0; y < 4; ++y) acc[x][y] = 0.f;
#pragma unroll
    for (int y = 0; y < SM_EMAX; ++y) eacc[x][y] = 0.f;
  }
  for (int k = 0; k < SM_NS - 1; ++k) load(k);
  for (int k = 0; k < nst; ++k) {
    load(k + SM_NS - 1);
    asm volatile("cp.async.wait_group %0;\n" ::"n"(SM_NS - 1) : "memory");
    __syncthreads();
    const float* st = sm + (k % SM_NS) * SM_STAGE;
    const int n = (int)min((long long)SM_RS, r1 - (r0 + (long long)k * SM_RS));
    if (work) {
      for (int r = rg; r < n; r += SM_SG) {
        float dl[4], u[4];
        if (H == SM_H) {                              // whole 4-column groups: 16-byte shared loads
          const float4 h4 = *reinterpret_cast<const float4*>(st + r * H + 4 * ti);
          const float4 g4 = *reinterpret_cast<const float4*>(st + SM_RS * H + r * H + 4 * ti);
          const float4 u4 = *reinterpret_cast<const float4*>(st + 2 * SM_RS * H + r * H + 4 * tj);
          dl[0] = (1.f - h4.x * h4.x) * g4.x, dl[1] = (1.f - h4.y * h4.y) * g4.y;
          dl[2] = (1.f - h4.z * h4.z) * g4.z, dl[3] = (1.f - h4.w * h4.w) * g4.w;
          u[0] = u4.x, u[1] = u4.y, u[2] = u4.z, u[3] = u4.w;
        } else {
#pragma unroll
          for (int x = 0; x < 4; ++x) {
            const int a = 4 * ti + x;
            const float hv = a < H ? st[r * H + a] : 0.f, gv = a < H ? st[SM_RS * H + r * H + a] : 0.f;
            dl[x] = (1.f - hv * hv) * gv;
          }
#pragma unroll
          for (int y = 0; y < 4; ++y) {
            const int c = 4 * tj + y;
            u[y] = c < H ? st[2 * SM_RS * H + r * H + c] : 0.f;
          }
        }
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
          for (int y = 0; y < 4; ++y) acc[x][y] = fmaf(dl[x], u[y], acc[x][y]);
        if (tj == 0) {
#pragma unroll
          for (int y = 0; y < SM_EMAX; ++y) {
            const float ev = y < I ? st[3 * SM_RS * H + r * I + y] : (y == I ? 1.f : 0.f);
#pragma unroll
            for (int x = 0; x < 4; ++x) eacc[x][y] = fmaf(dl[x], ev, eacc[x][y]);
          }
        }
      }
    }
    __syncthreads();                                   // the stage is refilled next
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  // fixed-order sum over the row groups through shared memory
  float* red = sm;                                     // [SM_SG][SM_TILES][16 + 4 SM_EMAX]
  constexpr int RW = 16 + 4 * SM_EMAX;
  if (rg < SM_SG) {
#pragma unroll
    for (int x = 0; x < 4; ++x) {
#pragma unroll
      for (int y = 0; y < 4; ++y) red[(rg * SM_TILES + tile) * RW + 4 * x + y] = acc[x][y];
#pragma unroll
      for (int y = 0; y < SM_EMAX; ++y) red[(rg * SM_TILES + tile) * RW + 16 + SM_EMAX * x + y] = eacc[x][y];
    }
  }
  __syncthreads();
  const int NB = H + E;
  float* dst = ws + (long long)part * H * NB;
  for (int o = tid; o < SM_TILES * RW; o += SM_NT) {
    const int t = o / RW, j = o % RW, oi = t / SM_TL, oj = t % SM_TL;
    float sum = 0.f;
    for (int g2 = 0; g2 < SM_SG; ++g2) sum += red[(g2 * SM_TILES + t) * RW + j];
    if (j < 16) {
      const int a = 4 * oi + j / 4, c = 4 * oj + j % 4;
      if (a < H && c < H) dst[(long long)a * NB + c] = sum;
    } else if (oj == 0) {
      const int a = 4 * oi + (j - 16) / SM_EMAX, y = (j - 16) % SM_EMAX;
      if (a < H && y < E) dst[(long long)a * NB + H + y] = sum;
    }
  }
}

// GRU, H <= 20, I + 1 <= 16 (config 3; r02i): the same staged scheme.  A =
// [dR | dZ | dN | dM] (4H rows) from the staged g, z, n, h_prev, r, M rows;
// U = [h_prev | x | 1] (H + I + 1 <= 36 columns); 4 x 4 tiles over 4H x 36,
// two row groups; the gate formulas are valA's.
constexpr int SG_H = 20, SG_RS = 32, SG_NS = 3, SG_UC = 36, SG_XM = 16, SG_NT = 384, SG_G = 2;
constexpr int SG_TA = 4 * SG_H / 4, SG_TU = SG_UC / 4, SG_TILES = SG_TA * SG_TU;   // 20 x 9 tiles
constexpr int SG_STAGE = 6 * SG_RS * SG_H + SG_RS * SG_XM;   // g | z | n | hp | r | M rows, x rows
__global__ void __launch_bounds__(SG_NT) wgrad_gru_small_kernel(WArgs w, float* __restrict__ ws) {
  extern __shared__ __align__(16) float sm[];
  const int H = w.H, I = w.I, E = w.E;
  const int part = blockIdx.x, tid = threadIdx.x;
  const long long r0 = (long long)part * w.rows_per_part;
  const long long r1 = min(r0 + w.rows_per_part, w.rows);
  const int nst = (int)((r1 - r0 + SG_RS - 1) / SG_RS);
  const float* arr[6] = {w.g, w.z, w.n, w.hp, w.r, w.M};
  auto al16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
  bool v16 = H % 4 == 0;
#pragma unroll
  for (int v = 0; v < 6; ++v) v16 = v16 && al16(arr[v]);
  const bool x16 = I > 0 && I % 4 == 0 && al16(w.x);
  auto load = [&](int k) {
    if (k < nst) {
      float* dst = sm + (k % SG_NS) * SG_STAGE;
      const long long rb = r0 + (long long)k * SG_RS;
      const int n = (int)min((long long)SG_RS, r1 - rb);
      if (v16) {                                       // 16-byte copies (rows of H = 20 floats are aligned)
        for (int e = 4 * tid; e < n * H; e += 4 * SG_NT)
#pragma unroll
          for (int v = 0; v < 6; ++v)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(
                             (unsigned)__cvta_generic_to_shared(dst + v * SG_RS * H + e)),
                         "l"(arr[v] + rb * H + e) : "memory");
      } else {
        for (int e = tid; e < n * H; e += SG_NT)
#pragma unroll
          for (int v = 0; v < 6; ++v)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(
                             (unsigned)__cvta_generic_to_shared(dst + v * SG_RS * H + e)),
                         "l"(arr[v] + rb * H + e) : "memory");
      }
      if (x16) {                                       // x rows of I % 4 == 0 floats: I / 4 chunks per row
        const int q = I / 4;
        for (int e = tid; e < n * q; e += SG_NT)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(
                           (unsigned)__cvta_generic_to_shared(dst + 6 * SG_RS * H + (e / q) * SG_XM + 4 * (e % q))),
                       "l"(w.x + (rb + e / q) * I + 4 * (e % q)) : "memory");
      } else {
        for (int e = tid; e < n * I; e += SG_NT)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(
                           (unsigned)__cvta_generic_to_shared(dst + 6 * SG_RS * H + (e / I) * SG_XM + e % I)),
                       "l"(w.x + rb * I + e) : "memory");
      }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  const int tile = tid % SG_TILES, rg = tid / SG_TILES;   // rg < SG_G for the working threads
  const int ta = tile / SG_TU, tu = tile % SG_TU;
  const bool work = rg < SG_G && 4 * ta < 4 * H && 4 * tu < H + E;
  float acc[4][4];
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) acc[x][y] = 0.f;
  for (int k = 0; k < SG_NS - 1; ++k) load(k);
  for (int k = 0; k < nst; ++k) {
    load(k + SG_NS - 1);
    asm volatile("cp.async.wait_group %0;\n" ::"n"(SG_NS - 1) : "memory");
    __syncthreads();
    const float* st = sm + (k % SG_NS) * SG_STAGE;
    const int n = (int)min((long long)SG_RS, r1 - (r0 + (long long)k * SG_RS));
    float* dA = sm + SG_NS * SG_STAGE;                 // the stage's A rows [row][4H], formed once
    for (int e = tid; e < n * 4 * H; e += SG_NT) {
      const int r = e / (4 * H), a = e % (4 * H), gt = a / H, o = r * H + a % H;
      const float g = st[o], z = st[SG_RS * H + o], nn = st[2 * SG_RS * H + o];
      const float hp = st[3 * SG_RS * H + o], rr = st[4 * SG_RS * H + o], M = st[5 * SG_RS * H + o];
      const float dN = g * (1.f - z) * (1.f - nn * nn);
      dA[e] = gt == 2 ? dN : gt == 1 ? g * (hp - nn) * z * (1.f - z) : gt == 0 ? dN * M * rr * (1.f - rr) : dN * rr;
    }
    float* dU = dA + SG_RS * 4 * SG_H;                 // the stage's U rows [row][36]: h_prev | x | 1 | 0
    for (int e = tid; e < n * SG_UC; e += SG_NT) {
      const int r = e / SG_UC, c = e % SG_UC;
      dU[e] = c < H ? st[3 * SG_RS * H + r * H + c]
                    : (c < H + I ? st[6 * SG_RS * H + r * SG_XM + (c - H)] : (c == H + I ? 1.f : 0.f));
    }
    __syncthreads();
    if (work) {
      for (int r = rg; r < n; r += SG_G) {
        float da[4], u[4];
        {
          const float4 a4 = *reinterpret_cast<const float4*>(dA + r * 4 * H + 4 * ta);
          da[0] = a4.x, da[1] = a4.y, da[2] = a4.z, da[3] = a4.w;
        }
        {
          const float4 u4 = *reinterpret_cast<const float4*>(dU + r * SG_UC + 4 * tu);
          u[0] = u4.x, u[1] = u4.y, u[2] = u4.z, u[3] = u4.w;
        }
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
          for (int y = 0; y < 4; ++y) acc[x][y] = fmaf(da[x], u[y], acc[x][y]);
      }
    }
    __syncthreads();
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  float* red = sm;                                     // [SG_G][SG_TILES][16]
  if (rg < SG_G) {
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y) red[(rg * SG_TILES + tile) * 16 + 4 * x + y] = acc[x][y];
  }
  __syncthreads();
  const int NB = H + E;
  float* dst = ws + (long long)part * w.NA * NB;
  for (int o = tid; o < SG_TILES * 16; o += SG_NT) {
    const int t = o / 16, j = o % 16, oa = t / SG_TU, ou = t % SG_TU;
    float sum = 0.f;
    for (int g2 = 0; g2 < SG_G; ++g2) sum += red[(g2 * SG_TILES + t) * 16 + j];
    const int a = 4 * oa + j / 4, c = 4 * ou + j % 4;
    if (a < w.NA && c < NB) dst[(long long)a * NB + c] = sum;
  }
}

cudaError_t run_partials(const WArgs& w, float* ws, long long nparts, cudaStream_t st) {
  if (w.kind == BPPSA_JAC_GRU && w.H == SG_H && w.E <= SG_XM + 1 && w.I <= SG_XM && w.H + w.E <= SG_UC) {
    const size_t smem = (size_t)(SG_NS * SG_STAGE + SG_RS * (4 * SG_H + SG_UC)) * sizeof(float);
    static_assert((size_t)SG_G * SG_TILES * 16 <= (size_t)SG_NS * SG_STAGE, "reduction fits");
    cudaError_t e = smem_attr_once(reinterpret_cast<const void*>(wgrad_gru_small_kernel), (int)smem);
    if (e != cudaSuccess) return e;
    wgrad_gru_small_kernel<<<(unsigned)nparts, SG_NT, smem, st>>>(w, ws);
    return cudaGetLastError();
  }
  if (w.kind == BPPSA_JAC_RNN_TANH && w.H <= SM_H && w.E <= SM_EMAX) {
    const size_t smem = (size_t)SM_NS * SM_STAGE * sizeof(float);
    static_assert((size_t)SM_SG * SM_TILES * (16 + 4 * SM_EMAX) <= (size_t)SM_NS * SM_STAGE, "reduction fits");
    cudaError_t e = smem_attr_once(reinterpret_cast<const void*>(wgrad_rnn_small_kernel), (int)smem);
    if (e != cudaSuccess) return e;
    wgrad_rnn_small_kernel<<<(unsigned)nparts, SM_NT, smem, st>>>(w, ws);
    return cudaGetLastError();
  }
  if (w.H <= 32 && w.E <= 16 && 32 * w.E <= WT<32, 16>::NEA * WT<32, 16>::NT) {
    dim3 grid((unsigned)nparts, (unsigned)((w.NA + 31) / 32));
    wgrad_partial_kernel<32, 16><<<grid, WT<32, 16>::NT, 0, st>>>(w, ws);
  } else {
    dim3 grid((unsigned)nparts, (unsigned)((w.NA + TA - 1) / TA));
    wgrad_partial_kernel<64, 64><<<grid, WT<64, 64>::NT, 0, st>>>(w, ws);
  }
  return cudaGetLastError();
}

}  // namespace

bool wgrad_supported(int H, int I) { return H <= TA && I + 1 <= MAXE && TA * (I + 1) <= 16 * NT; }

cudaError_t launch_wgrad_rnn(int T, int B, int H, int I, const float* x, const float* h, const float* h_init,
                             const float* grad_h, float* dW_ih, float* dW_hh, float* db, float* ws,
                             long long nparts, cudaStream_t st) {
  WArgs w{};
  w.T = T; w.B = B; w.H = H; w.I = I; w.kind = BPPSA_JAC_RNN_TANH;
  w.x = x; w.h = h; w.h_init = h_init; w.g = grad_h;
  w.rows = (long long)T * B;
  w.NA = H; w.E = I + 1;
  // the staged small-H kernel runs fewer, longer parts (three per SM: each
  // keeps its cp.async ring busy, and the fixed-order reduction has fewer
  // slabs); still a function of the row count only
#ifndef WG_SMALL_PARTS
#define WG_SMALL_PARTS 444LL
#endif
  if (H <= SM_H && w.E <= SM_EMAX) nparts = std::min(nparts, (long long)WG_SMALL_PARTS);
  w.rows_per_part = (w.rows + nparts - 1) / nparts;
  cudaError_t e = run_partials(w, ws, nparts, st);
  if (e != cudaSuccess) return e;
  return reduce_rnn(ws, nparts, H, I, dW_ih, dW_hh, db, st);
}

cudaError_t launch_wgrad_reduce_rnn(const float* ws, long long nparts, int H, int I, float* dW_ih, float* dW_hh,
                                    float* db, cudaStream_t st) {
  return reduce_rnn(ws, nparts, H, I, dW_ih, dW_hh, db, st);
}

cudaError_t launch_wgrad_gru(int T, int B, int H, int I, const float* x, const float* hp, const float* r,
                             const float* z, const float* n, const float* M, const float* grad_h, float* dW_ih3,
                             float* dW_hh3, float* db_ih3, float* db_hh3, float* ws, long long nparts,
                             cudaStream_t st) {
  WArgs w{};
  w.T = T; w.B = B; w.H = H; w.I = I; w.kind = BPPSA_JAC_GRU;
  w.x = x; w.g = grad_h; w.hp = hp; w.r = r; w.z = z; w.n = n; w.M = M;
  w.rows = (long long)T * B;
  w.NA = 4 * H; w.E = I + 1;
  if (H == SG_H && w.E <= SG_XM + 1 && H + w.E <= SG_UC) nparts = std::min(nparts, (long long)WG_SMALL_PARTS);
  w.rows_per_part = (w.rows + nparts - 1) / nparts;
  cudaError_t e = run_partials(w, ws, nparts, st);
  if (e != cudaSuccess) return e;
  const int total = 3 * H * H + 3 * H * I + 6 * H;
  const RedMap m{1, H, I, 4 * H, H + I + 1, dW_hh3, dW_ih3, db_ih3, db_hh3};
  wgrad_reduce<<<(total + 31) / 32, 1024, 0, st>>>(ws, nparts, m, total);
  return cudaGetLastError();
}

}  // namespace bppsa
