// tc_wgrad.cu — RNN weight gradients (eqn:update_param, tied over
// time) as a tensor-core GEMM over K = T*B rows, H = 64:
//     dW_hh = sum_rows delta_row h_{row-B}^T,   delta = (1 - h^2) o grad_h
// Per 32-row chunk one contraction D[128 x 128] += A[128 x 32] B[128 x 32]^T
// with A = [delta_hi ; delta_lo] (M = 128, rows = i), B = [hp_hi | hp_lo]
// (N = 128, rows = k): the four quadrants of D are the products hh, hl, lh, ll
// (4xTF32) and every MMA is a full-rate N = 128 one.
//
// Roles (320 threads, one CTA per SM):
//   warp 8, lane 0   stages chunks with cp.async.bulk (a 32-row chunk of h, g
//                    and h_prev is one contiguous 8 KB run each; NS stages
//                    ahead, mbarrier complete_tx);
//   warp 9, lane 0   issues the MMAs (NBUF operand buffers in flight);
//   warps 0..7       converters: thread = (column i, 8-row group) of the
//                    chunk; it forms delta ONCE and stores both A rows (delta
//                    hi / lo) and both B rows (h_prev hi / lo) into K-major
//                    SW128 tiles in shared memory (SS MMAs).  r02: A moved out
//                    of TMEM — there its hi and lo rows sat in different lane
//                    quadrants, so two threads formed each delta (2.2 ms).
// Synchronisation is mbarrier-only: full/empty per stage, a_full/freeb per
// A/B buffer.  What bounds it (r02g, dev-aid macros WG_NO_LOAD / NO_CONV /
// NO_MMA / NO_FENCE that strip one stage each, timing only): 2.18 ms whole;
// 2.06 without the HBM reads, 1.54 without the conversion, 1.30 with
// neither, 0.85 with no MMAs and no proxy fence either -- the converter /
// MMA pipeline, not HBM, sets the pace: per 32-row chunk ~104 KB of shared
// memory traffic (16 KB bulk writes, 24 KB of h / g / h_prev reads, 32 KB of
// split operands written and read again by the SS MMAs) plus the handshakes.
// 16 converter warps (4 rows each) measured 2.47 ms (spills at 96
// registers), more stages 2.33-2.38, one arrival per warp 2.24.  The accumulator is flushed into fp32 registers every FLUSH
// chunks so the tensor core's truncating accumulation never spans more than
// FLUSH*4 MMAs.  dW_ih and db accumulate on the CUDA cores.  Rows are split
// into fixed parts (a function of K only); each part writes four slabs
// (lane half x column half of D) and wgrad_reduce_rnn sums parts*4 slabs in a
// fixed order (deterministic).
#include <algorithm>
#include <cstdlib>

#include "common.cuh"

namespace bppsa {
namespace {

constexpr int H = 64, KC = 32, MROWS = 128, NCONV = 256, NTH = NCONV + 64;   // + loader warp + MMA warp
constexpr int FLUSH = 32;                           // chunks per accumulation window
constexpr long long PART_ROWS = 16384;              // rows per part (512 chunks)
constexpr int MAXI = 4;
#ifndef WG_NS
#define WG_NS 4
#endif
#ifndef WG_NBUF
#define WG_NBUF 2                                   // 2.18-2.23 ms at C4 vs 2.27-2.41 with 3 (r02g A/B)
#endif
constexpr int NS = WG_NS;                           // staging depth (chunks)
constexpr int NBUF = WG_NBUF;                       // A / B operand buffer pairs (shared memory)
constexpr int ROW_BYTES = H * 4;
constexpr int SB = 3 * KC * ROW_BYTES;              // h, g, h_prev rows: 24 KB per stage
constexpr int XB = KC * MAXI * 4;                   // x rows: 512 B per stage
constexpr int B_BYTES = MROWS * KC * 4;             // 16 KB per operand tile (A or B)
constexpr int OFF_STAGE = 0;
constexpr int OFF_BT = NS * SB;                     // 1024-B aligned (SW128 tiles): [buf][A | B]
constexpr int OFF_X = OFF_BT + NBUF * 2 * B_BYTES;
constexpr int OFF_BAR = OFF_X + NS * XB;
constexpr int SMEM = OFF_BAR + (2 * NS + 2 * NBUF + 2) * 8 + 1024;
static_assert(OFF_BT % 1024 == 0, "SW128 B tiles must be 1024-B aligned");
static_assert(SMEM <= 232448, "tc_wgrad shared memory");
constexpr uint32_t TMEM_COLS = 128;                 // D at [0, 128)
constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(128 >> 3) << 17) |
                           ((uint32_t)(MROWS >> 4) << 24);

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t sw_off(int row, int k) {   // K-major SW128, K < 32
  return (uint32_t)((row >> 3) * 1024 + (row & 7) * 128 + ((((k & 31) >> 2) ^ (row & 7)) << 4) + ((k & 3) << 2));
}
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(c));
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}\n" ::"r"(bar),
               "r"(bytes) : "memory");
}
// try_wait with a suspend-time hint: a waiting thread sleeps in the barrier
// unit instead of re-issuing the probe (256 converter threads spinning cost
// ~25 % of the kernel's issued instructions: r01i ncu)
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n @!p bra W_%=;\n}\n" ::"r"(
                   bar), "r"(parity), "r"(1000000u) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar) : "memory");
}
__device__ __forceinline__ void tc_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ float lds(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];\n" : "=f"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts4(uint32_t a, float x, float y, float z, float w) {
  asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};\n" ::"r"(a), "f"(x), "f"(y), "f"(z), "f"(w) : "memory");
}
// hi = x rounded to the nearest tf32 (ties away), as an fp32 value with the 13
// low mantissa bits clear; lo = x - hi is exact in fp32 and |lo| <= 2^-11 |x|.
__device__ __forceinline__ float tf32_hi(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

struct TWArgs {
  int B, I;
  const float *x, *h, *h_init, *g;
  long long rows;
  float* ws;            // partials [P][4][H][H + I + 1]
  long long nparts;     // parts [part0, nparts) are computed (slabs at their absolute part index)
  long long part0;
};

struct ChunkIter {      // walks this CTA's chunks: parts blockIdx.x + j*gridDim.x
  long long part, c, cg, r0, r1, nch;
  __device__ void start(long long p, long long rows) {
    part = p;
    c = 0;
    cg = 0;
    set(rows);
  }
  __device__ void set(long long rows) {
    r0 = part * PART_ROWS;
    r1 = min(r0 + PART_ROWS, rows);
    nch = (r1 - r0 + KC - 1) / KC;
  }
  __device__ void next(long long rows) {
    ++cg;
    if (++c == nch) {
      part += gridDim.x;
      c = 0;
      set(rows);
    }
  }
};

struct Bars {
  uint32_t b0;
  __device__ uint32_t full(int s) const { return b0 + 8u * s; }
  __device__ uint32_t empty(int s) const { return b0 + 8u * (NS + s); }
  __device__ uint32_t a_full(int b) const { return b0 + 8u * (2 * NS + b); }
  __device__ uint32_t freeb(int b) const { return b0 + 8u * (2 * NS + NBUF + b); }
};

// One chunk's 8 rows of this thread's column i (rows 8 kg .. 8 kg + 7 of the
// chunk; base = stage + column i + those rows): delta = (1 - h^2) g once, its
// tf32 hi / lo (A rows i and 64 + i), h_prev hi / lo (B rows i and 64 + i),
// and the dbias / dW_ih partials.  Rows >= n are zero, h_prev rows < nlow
// (before h_0 with no h_init) are zero.  SPLIT: h_prev rows < nsplit come
// from hp_lo (the previous chunk), the rest from hp_hi.
template <int IX, bool FULL, bool SPLIT>
__device__ __forceinline__ void convert8(uint32_t base, uint32_t xbase, int n, int nlow, float (&ah)[8],
                                         float (&al)[8], float (&bh)[8], float (&bl)[8], float& dbias,
                                         float (&dih)[MAXI], uint32_t hp_lo, uint32_t hp_hi, int nsplit) {
#pragma unroll
  for (int rr = 0; rr < 8; ++rr) {
    const float hv = lds(base + rr * ROW_BYTES), gv = lds(base + (KC + rr) * ROW_BYTES);
    float d = (1.f - hv * hv) * gv;
    if (!FULL) d = rr < n ? d : 0.f;
    ah[rr] = tf32_hi(d);
    al[rr] = d - ah[rr];
    float hp = lds(!SPLIT ? hp_lo + rr * ROW_BYTES
                          : (rr < nsplit ? hp_lo + rr * ROW_BYTES : hp_hi + (rr - nsplit) * ROW_BYTES));
    if (!FULL) hp = (rr < n && rr >= nlow) ? hp : 0.f;
    bh[rr] = tf32_hi(hp);
    bl[rr] = hp - bh[rr];
    dbias += d;
#pragma unroll
    for (int j = 0; j < IX; ++j) {
      float xv = lds(xbase + 4 * (rr * IX + j));
      if (!FULL) xv = rr < n ? xv : 0.f;
      dih[j] = fmaf(d, xv, dih[j]);
    }
  }
}

// Converter thread (column i = 32 (warp & 1) + lane, row group kg = warp >> 1
// of each 32-row chunk) forms delta ONCE and writes both its A rows (delta hi
// / lo, K-major SW128 tile in shared memory) and both B rows (h_prev hi / lo).
// The flush mapping is the accumulator's: warp w reads TMEM lanes 32 (w & 3)
// (D rows), columns 64 (w >> 2) (D column half); for every warp that is row
// i of slab (w & 2) + (w >> 2), and the slab also receives the warp's
// dbias / dW_ih partials of column i over its row group (4 partials per part
// and column, summed by wgrad_reduce_rnn with the slabs).
template <int IX>
__device__ __forceinline__ void converters(const TWArgs& w, uint32_t s0, Bars br, uint32_t tmem, int warp,
                                           int lane) {
  const int wq = warp & 3, grp = warp >> 2;          // flush: D lanes 32 wq.., D columns 64 grp..
  const int kg = warp >> 1, i = 32 * (warp & 1) + lane;   // convert: rows 8 kg.., column i
  const uint32_t tl = tmem + ((uint32_t)(32 * wq) << 16);
  const int NB = H + IX + 1;
  const bool reuse = w.B <= KC;
  uint32_t cg = 0;
  for (long long part = w.part0 + blockIdx.x; part < w.nparts; part += gridDim.x) {
    float acc[64];
#pragma unroll
    for (int k = 0; k < 64; ++k) acc[k] = 0.f;
    float dbias = 0.f, dih[MAXI];
#pragma unroll
    for (int j = 0; j < MAXI; ++j) dih[j] = 0.f;
    auto flush = [&]() {
      float t[32];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        tmem_ld32(tl + 64 * grp + 32 * q, t);
#pragma unroll
        for (int k = 0; k < 32; ++k) acc[32 * q + k] += t[k];
      }
    };
    const long long r0 = part * PART_ROWS;
    const int rows_here = (int)(min(r0 + PART_ROWS, w.rows) - r0);
    const int nch = (rows_here + KC - 1) / KC;
    const int lowB = w.h_init ? 0 : (int)max(0ll, min((long long)rows_here, (long long)w.B - r0));
    for (int c = 0; c < nch; ++c, ++cg) {
      const uint32_t b = cg % NBUF, s = cg % NS;
      const int n = min(KC, rows_here - c * KC) - 8 * kg;         // valid rows of my 8
      const int nlow = lowB - c * KC - 8 * kg;                      // h_prev rows before h_0
      mbar_wait(br.full(s), (cg / NS) & 1);
      const uint32_t base = s0 + OFF_STAGE + s * SB + 4u * i + 8u * kg * ROW_BYTES;
      const uint32_t xbase = s0 + OFF_X + s * XB + 4u * 8 * kg * IX;
      // h_prev = h shifted back by B rows: with B <= KC every chunk but a part's
      // first reads it from its own h rows and the previous chunk's (still
      // staged: a stage is released one chunk late), no third copy
      uint32_t hp_lo, hp_hi;
      int nsplit;
      if (reuse && c > 0) {
        const int rf = 8 * kg - w.B;                      // chunk-relative row of my first h_prev
        const uint32_t prev = s0 + OFF_STAGE + ((cg - 1) % NS) * SB + 4u * i;
        hp_lo = prev + (uint32_t)((KC + rf) * ROW_BYTES);   // rows rf .. -1 of the previous chunk
        hp_hi = s0 + OFF_STAGE + s * SB + 4u * i + (uint32_t)(max(rf, 0) * ROW_BYTES);
        nsplit = max(0, -rf);
      } else {
        hp_lo = base + 2 * KC * ROW_BYTES;
        hp_hi = hp_lo;
        nsplit = 0;
      }
      float ah[8], al[8], bh[8], bl[8];
#ifdef WG_NO_CONV                                   // dev aid: the pipeline without the conversion (timing only)
      const bool full = false;
      if (true) {
#pragma unroll
        for (int rr = 0; rr < 8; ++rr) ah[rr] = al[rr] = bh[rr] = bl[rr] = 0.f;
      } else
#else
      const bool full = n >= 8 && nlow <= 0;
#endif
      if (nsplit == 0 || nsplit >= 8) {                // my 8 h_prev rows are contiguous
        const uint32_t hp = nsplit == 0 ? hp_hi : hp_lo;
        if (full) convert8<IX, true, false>(base, xbase, n, nlow, ah, al, bh, bl, dbias, dih, hp, hp, 8);
        else convert8<IX, false, false>(base, xbase, n, nlow, ah, al, bh, bl, dbias, dih, hp, hp, 8);
      } else {
        if (full) convert8<IX, true, true>(base, xbase, n, nlow, ah, al, bh, bl, dbias, dih, hp_lo, hp_hi, nsplit);
        else convert8<IX, false, true>(base, xbase, n, nlow, ah, al, bh, bl, dbias, dih, hp_lo, hp_hi, nsplit);
      }
      if (!reuse) {
        mbar_arrive(br.empty(s));
      } else {
        if (c > 0) mbar_arrive(br.empty((cg - 1) % NS));   // the previous chunk's rows are no longer read
        if (c == nch - 1) mbar_arrive(br.empty(s));         // a part's last chunk is not read again
      }
      if (c > 0 && c % FLUSH == 0) {           // window boundary: chunk cg-1 done, read D
        mbar_wait(br.freeb((cg - 1) % NBUF), ((cg - 1) / NBUF) & 1);
        tc_after();
        flush();
      } else if (c >= NBUF) {                  // operand buffer b was last read by chunk cg-NBUF
        mbar_wait(br.freeb(b), ((cg - NBUF) / NBUF) & 1);
        tc_after();
      }
      const uint32_t at = s0 + OFF_BT + b * 2 * B_BYTES, bt = at + B_BYTES;
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int kk = 8 * kg + 4 * q;
        sts4(at + sw_off(i, kk), ah[4 * q], ah[4 * q + 1], ah[4 * q + 2], ah[4 * q + 3]);
        sts4(at + sw_off(64 + i, kk), al[4 * q], al[4 * q + 1], al[4 * q + 2], al[4 * q + 3]);
        sts4(bt + sw_off(i, kk), bh[4 * q], bh[4 * q + 1], bh[4 * q + 2], bh[4 * q + 3]);
        sts4(bt + sw_off(64 + i, kk), bl[4 * q], bl[4 * q + 1], bl[4 * q + 2], bl[4 * q + 3]);
      }
#ifndef WG_NO_FENCE                                 // (dev aid: timing only)
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
#endif
      tc_before();
      mbar_arrive(br.a_full(b));
    }
    // last window of the part
    const uint32_t cl = cg - 1;
    mbar_wait(br.freeb(cl % NBUF), (cl / NBUF) & 1);
    tc_after();
    flush();
    tc_before();
    const int slab = (wq & 2) + grp;
    const int row = (32 * wq + lane) & 63;           // == i: the slab row this thread writes
    float* dst = w.ws + ((part * 4 + slab) * (long long)H + row) * NB;
#pragma unroll
    for (int k = 0; k < 64; ++k) dst[k] = acc[k];
#pragma unroll
    for (int j = 0; j < IX; ++j) dst[H + j] = dih[j];
    dst[H + IX] = dbias;
  }
}

__global__ void __launch_bounds__(NTH, 1) tc_wgrad_kernel(TWArgs w) {
  extern __shared__ uint8_t smem_raw[];
  char* smem = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t s0 = su32(smem);
  const Bars br{s0 + OFF_BAR};
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + OFF_BAR + 8 * (2 * NS + 2 * NBUF));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 9) {
    if (lane == 0) {
      for (int s = 0; s < NS; ++s) {
        mbar_init(br.full(s), 1);
        mbar_init(br.empty(s), NCONV);
      }
      for (int b = 0; b < NBUF; ++b) {
        mbar_init(br.a_full(b), NCONV);
        mbar_init(br.freeb(b), 1);
      }
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncwarp();
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(tslot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tmem = *tslot;

  if (warp == 8) {
    if (lane == 0) {
      // ===== loader: NS chunks ahead of the converters =====
      ChunkIter ld;
      ld.start(w.part0 + blockIdx.x, w.rows);
      const long long B = w.B;
      while (ld.part < w.nparts) {
        const int s = (int)(ld.cg % NS);
        if (ld.cg >= NS) mbar_wait(br.empty(s), (uint32_t)((ld.cg / NS - 1) & 1));
        const long long rb = ld.r0 + ld.c * KC;
        const int n = (int)min((long long)KC, ld.r1 - rb);
        const uint32_t st = s0 + OFF_STAGE + s * SB;
        // h_prev rows: [rb, rb+nA) come from h_init (rows < B), the rest from h
        const int nA = (int)max(0ll, min((long long)n, B - rb));
        const bool reuse = B <= KC && ld.c > 0;          // h_prev from the staged h rows (converters)
        uint32_t tx = 2u * n * ROW_BYTES;
        if (!reuse) tx += (uint32_t)(n - nA) * ROW_BYTES;
        if (!reuse && w.h_init) tx += (uint32_t)nA * ROW_BYTES;
        const float* xs = w.x + rb * w.I;
        const uint32_t xbytes = (uint32_t)(n * w.I * 4);
        const bool xbulk = w.I > 0 && (xbytes & 15) == 0;
        if (xbulk) tx += xbytes;
        else if (w.I > 0) {     // tail chunk with an odd byte count: plain copies before the arrive
          float* xd = reinterpret_cast<float*>(smem + OFF_X + s * XB);
          for (int e = 0; e < n * w.I; ++e) xd[e] = xs[e];
        }
#ifdef WG_NO_LOAD                                   // dev aid: the pipeline without HBM reads (timing only)
        mbar_arrive(br.full(s));
        ld.next(w.rows);
        continue;
#endif
        mbar_expect_tx(br.full(s), tx);
        bulk_g2s(st, w.h + rb * H, (uint32_t)n * ROW_BYTES, br.full(s));
        bulk_g2s(st + KC * ROW_BYTES, w.g + rb * H, (uint32_t)n * ROW_BYTES, br.full(s));
        if (!reuse && nA > 0 && w.h_init)
          bulk_g2s(st + 2 * KC * ROW_BYTES, w.h_init + rb * H, (uint32_t)nA * ROW_BYTES, br.full(s));
        if (!reuse && n > nA)
          bulk_g2s(st + 2 * KC * ROW_BYTES + nA * ROW_BYTES, w.h + (rb + nA - B) * H, (uint32_t)(n - nA) * ROW_BYTES,
                   br.full(s));
        if (xbulk) bulk_g2s(s0 + OFF_X + s * XB, xs, xbytes, br.full(s));
        ld.next(w.rows);
      }
    }
    __syncwarp();
  } else if (warp == 9) {
    if (lane == 0) {
      // ===== MMA issuer =====
      ChunkIter mm;
      mm.start(w.part0 + blockIdx.x, w.rows);
      while (mm.part < w.nparts) {
        const int b = (int)(mm.cg % NBUF);
        mbar_wait(br.a_full(b), (uint32_t)((mm.cg / NBUF) & 1));
        tc_after();
        const uint32_t at = s0 + OFF_BT + b * 2 * B_BYTES, bt = at + B_BYTES;
#ifdef WG_NO_MMA                                    // dev aid: the pipeline without the MMAs (timing only)
        mbar_arrive(br.freeb(b));
        mm.next(w.rows);
        continue;
#endif
#pragma unroll
        for (int kk = 0; kk < KC / 8; ++kk) {
          const uint32_t acc = !((mm.c % FLUSH) == 0 && kk == 0);
          asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                       " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                       "l"(sdesc(at + 32 * kk)), "l"(sdesc(bt + 32 * kk)), "r"(IDESC), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                         br.freeb(b)) : "memory");
        mm.next(w.rows);
      }
    }
    __syncwarp();
  } else {
    switch (w.I) {
      case 0: converters<0>(w, s0, br, tmem, warp, lane); break;
      case 1: converters<1>(w, s0, br, tmem, warp, lane); break;
      case 2: converters<2>(w, s0, br, tmem, warp, lane); break;
      case 3: converters<3>(w, s0, br, tmem, warp, lane); break;
      default: converters<4>(w, s0, br, tmem, warp, lane); break;
    }
  }
  tc_before();
  __syncthreads();
  if (warp == 9) {
    tc_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

}  // namespace

long long tc_wgrad_parts(long long rows) { return 4 * ((rows + PART_ROWS - 1) / PART_ROWS); }   // slabs
long long tc_wgrad_part_rows() { return PART_ROWS; }
bool tc_wgrad_applies(int H_, int I, long long rows) {
  static const int force = [] { const char* e = getenv("BPPSA_FORCE_TC_WGRAD"); return e ? atoi(e) : 0; }();
  if (H_ != H || I > MAXI) return false;
  return force == 1 ? true : (force == 2 ? false : rows >= 8 * PART_ROWS);   // debug override (tests)
}

cudaError_t launch_tc_wgrad_partials(int B, int I, const float* x, const float* h, const float* h_init,
                                     const float* grad_h, long long rows, float* ws, int num_sms, cudaStream_t st,
                                     long long row0, long long row1) {
  cudaError_t e = smem_attr_once(reinterpret_cast<const void*>(tc_wgrad_kernel), SMEM);
  if (e != cudaSuccess) return e;
  if (row1 < 0) row1 = rows;
  const long long p0 = row0 / PART_ROWS, p1 = (row1 + PART_ROWS - 1) / PART_ROWS;   // parts of [row0, row1)
  if (p1 <= p0) return cudaSuccess;
  TWArgs a{B, I, x, h, h_init, grad_h, rows, ws, p1, p0};
  const int grid = (int)std::min<long long>(p1 - p0, num_sms);
  tc_wgrad_kernel<<<grid, NTH, SMEM, st>>>(a);
  return cudaGetLastError();
}

}  // namespace bppsa
