// tc_leaf.cu — level-0 up-sweep fold of the tanh-RNN leaves on the 5th-gen
// tensor cores (tcgen05, TMEM accumulators), H = 64.
//
// Every step of every column chain of every block multiplies by the SAME
// W_hh (leaf J_t^T = W^T diag(1-h_t^2), eqn:rnn P:315; see leaf.cu):
//     c_new^T = (d_t o c)^T W      for all chains at once
// i.e. one dense contraction D[128 x 64] = A[128 x 64] . B[64 x 64] per step
// and tile, with A = X^T (one row per chain: x = d o c), B[n][k] = W[k][n].
// fp32 accuracy from 3xTF32 (A_hi B_hi + A_hi B_lo + A_lo B_hi, x = x_hi +
// x_lo, x_hi = x with the 13 low mantissa bits cleared — what the MMA reads of
// a tf32 operand anyway — and x_lo = rn_tf32(x - x_hi), both on the integer
// pipe: cvt.rna.tf32.f32 is a 4-instruction sequence on sm_100a).  lo is
// rounded to nearest explicitly: left to the MMA's operand truncation it
// carries a one-signed 2^-21 bias per product that grows along a chain.
//
// A tile = 128 chains = the 64 column chains of block q of sample b and those
// of sample b+1 (same slots, same length).  A tf32 MMA with M = 128 costs ~60
// cycles at N = 64 but 64 at N = 128 (profiles/tc_precision.md), so B stacks
// [W_hi | W_lo] along N and every MMA is a full-rate N = 128 one:
// D = A_lo [W_hi | W_lo] + A_hi [W_hi | W_lo] (16 MMAs, A_hi / A_lo in TMEM —
// the TS form, B from shared memory), D[:, :64] + D[:, 64:] summed
// round-to-nearest in the epilogue (4 products incl. lo*lo, 2 TMEM reads).
// Two tiles (slots) are in flight per CTA so one slot's epilogue (tcgen05.ld
// D -> sum -> scale by d -> tf32 split -> tcgen05.st A) overlaps the other
// slot's MMAs: 2 x 16 epilogue warps per CTA, the slot's first warp issues
// (tc_leaf_up16_kernel, tc_leaf_down16_kernel).
// Persistent grid, one CTA per SM.
#include <algorithm>
#include <cstdlib>

#include <cuda.h>
#include <cuda_fp16.h>

#include "common.cuh"

namespace bppsa {
namespace {

constexpr int TH = 64;                    // hidden size of this kernel
constexpr int TM = 128;                   // chains per tile (UMMA M)
constexpr int NSLOT = 2;                  // tiles in flight per CTA
constexpr int B_ROWS = 2 * TH;            // B = [W_hi | W_lo] stacked along N
constexpr int B_BYTES = B_ROWS * TH * 4;  // 32 KB
#ifndef BPPSA_HCH
#define BPPSA_HCH 96
#endif
constexpr int HCH = BPPSA_HCH;            // steps staged per chunk
constexpr int H_BYTES = 2 * HCH * TH * 4; // one tile's h slices (2 blocks), 48 KB
constexpr int OFF_B = 0;
constexpr int OFF_H = OFF_B + B_BYTES;
// TMEM columns of slot g (base 256 g): D = A [W_hi | W_lo] accumulated over
// A = A_lo then A_hi at [0, 128) (cols 0..63: hh + lh, 64..127: hl + ll),
// A_hi at [128, 192), A_lo at [192, 256)
constexpr uint32_t TMEM_COLS = 512;
// instruction descriptors: D f32, A/B tf32, both K-major, M = 128, N = 128 / 64
constexpr uint32_t idesc(int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(TM >> 4) << 24);
}
constexpr uint32_t IDESC128 = idesc(128);

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// element (row, k) of a K-major SWIZZLE_128B tile with `rows` rows and K = 64
// fp32: two K-halves of rows x 128 B; 8-row atoms of 1024 B; the 16-byte
// chunk index is XORed with (row % 8).
__device__ __forceinline__ uint32_t sw_off(int row, int k, int rows) {
  const int kk = k & 31;
  return (uint32_t)((k >> 5) * rows * 128 + (row >> 3) * 1024 + (row & 7) * 128 + (((kk >> 2) ^ (row & 7)) << 4) +
                    ((kk & 3) << 2));
}

__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;           // LBO (16 B; unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32; // SBO: stride between 8-row groups
  d |= (uint64_t)1 << 46;           // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;           // SWIZZLE_128B
  return d;
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n"
      "}\n" ::"r"(su32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }




__device__ __forceinline__ float tf32_rn(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// x = d o c for the K-half `kh` (32 columns) of the chain's row, split into
// tf32 hi (-> this lane's A_hi TMEM columns) and lo (-> the swizzled A_lo tile
// in shared memory); hrow = the block's staged h_t row (broadcast reads)
__device__ __forceinline__ float4 lds128(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];\n" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts128(uint32_t a, float x, float y, float z, float w) {
  asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};\n" ::"r"(a), "f"(x), "f"(y), "f"(z), "f"(w) : "memory");
}

__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(su32(sdst)), "l"(gsrc) : "memory");
}

__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}

// ---------------------------------------------------------------------------
// Level-0 UP-sweep: 16 epilogue warps per tile slot (1024 threads), thread =
// (chain row, 16-column group).  Per step the slot's warps meet at a named
// barrier and the converged first warp of the slot issues the 16 MMAs + commit
// (one elected stream, under a CTA lock so the two slots' batches never
// interleave); one lane polls the completion mbarrier while the other warps
// sleep in bar.sync.  Measured (scripts/tc_up_trace.cu, tc_rate3.cu): polling
// warps and interleaved batches each cost ~15-25 cycles per MMA.
// ---------------------------------------------------------------------------
#ifdef BPPSA_STEP_TRACE
__device__ long long g_step_trace[2][2][8][4096];   // [slot][warp 0 / warp 13][phase][step]
#define STEP_TRACE(ph)                                                                            \
  if (blockIdx.x == 0 && lane == 0 && (wl == 0 || wl == 5) && tstep < 4096)                      \
    g_step_trace[g][wl == 5][ph][tstep] = clock64();
#else
#define STEP_TRACE(ph)
#endif
constexpr int EPI16_WARPS = 16;
constexpr int EPI16_THREADS = 32 * EPI16_WARPS;
constexpr int NTHREADS16 = EPI16_THREADS * NSLOT;          // 1024
constexpr int OFF_BAR16 = OFF_H + NSLOT * H_BYTES;         // d_full[2], tmem
constexpr int SMEM_BYTES16 = OFF_BAR16 + 64 + 1024;

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n" ::"r"(
          taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}

// CTA-scope spin lock in shared memory (one lane per slot contends)
__device__ __forceinline__ void lock_acquire(uint32_t a) {
  asm volatile(
      "{\n .reg .b32 old;\n .reg .pred p;\nL_%=:\n atom.shared.cta.acquire.cas.b32 old, [%0], 0, 1;\n"
      " setp.ne.b32 p, old, 0;\n @p bra L_%=;\n}\n" ::"r"(a) : "memory");
}
__device__ __forceinline__ void lock_release(uint32_t a) {
  asm volatile("st.shared.release.cta.b32 [%0], 0;\n" ::"r"(a) : "memory");
}

// The step's 16 MMAs (A_lo then A_hi, K = 64 in 8-wide steps, B = [W_hi | W_lo])
// and their commit as ONE elected instruction stream of the converged warp:
// operands stay warp-uniform, so the issue costs ~2 instructions per MMA
// instead of a per-MMA elect loop with descriptor arithmetic.
__device__ __forceinline__ void mma16_commit(uint32_t d, const uint64_t (&bd)[8], uint32_t bar) {
  asm volatile(
      "{\n"
      " .reg .pred e, f, t;\n"
      " .reg .b32 a;\n"
      " setp.ne.b32 f, 0, 0;\n"
      " setp.eq.b32 t, 0, 0;\n"
      " elect.sync _|e, 0xffffffff;\n"
      " add.u32 a, %0, 192;\n @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [a], %1, %9, f;\n"
      " add.u32 a, %0, 200;\n @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [a], %2, %9, t;\n"
      " add.u32 a, %0, 208;\n @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [a], %3, %9, t;\n"
      " add.u32 a, %0, 216;\n @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [a], %4, %9, t;\n"
      " add.u32 a, %0, 224;\n @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [a], %5, %9, t;\n"
      " add.u32 a, %0, 232;\n @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [a], %6, %9, t;\n"
      " add.u32 a, %0, 240;\n @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [a], %7, %9, t;\n"
      " add.u32 a, %0, 248;\n @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [a], %8, %9, t;\n"
      " add.u32 a, %0, 128;\n @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [a], %1, %9, t;\n"
      " add.u32 a, %0, 136;\n @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [a], %2, %9, t;\n"
      " add.u32 a, %0, 144;\n @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [a], %3, %9, t;\n"
      " add.u32 a, %0, 152;\n @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [a], %4, %9, t;\n"
      " add.u32 a, %0, 160;\n @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [a], %5, %9, t;\n"
      " add.u32 a, %0, 168;\n @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [a], %6, %9, t;\n"
      " add.u32 a, %0, 176;\n @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [a], %7, %9, t;\n"
      " add.u32 a, %0, 184;\n @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [a], %8, %9, t;\n"
      " @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%10];\n"
      "}\n" ::"r"(d),
      "l"(bd[0]), "l"(bd[1]), "l"(bd[2]), "l"(bd[3]), "l"(bd[4]), "l"(bd[5]), "l"(bd[6]), "l"(bd[7]), "r"(IDESC128),
      "r"(bar)
      : "memory");
}

__global__ void __launch_bounds__(NTHREADS16, 1) tc_leaf_up16_kernel(LeafArgs a, int C, float* __restrict__ agg_out,
                                                                     long long n_out, long long q0) {
  extern __shared__ uint8_t smem_raw[];
  char* smem = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* d_full = reinterpret_cast<uint64_t*>(smem + OFF_BAR16);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(d_full + NSLOT);
  int* issue_lock = reinterpret_cast<int*>(tmem_slot + 1);
  // warp index and TMEM base through a shuffle: provably warp-uniform, so the
  // issuer's descriptors / TMEM addresses live in uniform registers (a few
  // instructions per MMA instead of ~15 with per-MMA R2UR and rematerialisation)
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const int B = a.seg.B;
  const long long S = a.seg.S();
  const long long nq = n_out - q0;
  const int nbp = (B + 1) / 2;
  const long long ntiles = (long long)nbp * nq;

  for (int e = threadIdx.x; e < TH * TH; e += NTHREADS16) {
    const int n = e / TH, k = e % TH;               // B[n][k] = W[k][n]: rows 0..63 hi, 64..127 lo
    const float w = __ldg(a.W + (long long)k * TH + n);
    const float hi = tf32_rn(w);
    *reinterpret_cast<float*>(smem + OFF_B + sw_off(n, k, B_ROWS)) = hi;
    *reinterpret_cast<float*>(smem + OFF_B + sw_off(TH + n, k, B_ROWS)) = tf32_rn(w - hi);
  }
  if (warp == 0) {
    if (lane == 0) {
      for (int s = 0; s < NSLOT; ++s) mbar_init(&d_full[s], 1);
      *issue_lock = 0;
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncwarp();
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);

  const int g = warp / EPI16_WARPS, wl = warp % EPI16_WARPS;
  const int row = (wl & 3) * 32 + lane;                   // TMEM lane / A row (lane quarter = warp % 4)
  const int cgp = wl >> 2;                                // 16-column group of D / of A's K
  const int et = wl * 32 + lane;
  const bool issuer = wl == 0;
  const uint32_t slot_base = tmem + 256 * g;
  const uint32_t lane_base = slot_base + ((uint32_t)((wl & 3) * 32) << 16);
  const uint32_t t_dh = lane_base + 16 * cgp, t_dl = t_dh + 64;
  const uint32_t t_ahi = lane_base + 128 + 16 * cgp, t_alo = lane_base + 192 + 16 * cgp;
  float* hs = reinterpret_cast<float*>(smem + OFF_H + g * H_BYTES);   // [2 blocks][HCH][64]
  const uint32_t hs_s = su32(hs);
  const uint32_t bb = __shfl_sync(0xffffffffu, su32(smem + OFF_B), 0);   // warp-uniform (see above)
  const uint32_t lock_s = su32(issue_lock);
  uint64_t bdesc[TH / 8];                                 // B descriptors of the 8 K-steps (constant)
#pragma unroll
  for (int kk = 0; kk < TH / 8; ++kk) bdesc[kk] = sdesc(bb + (uint32_t)((kk >> 2) * B_ROWS * 128 + (kk & 3) * 32));
  uint32_t ph = 0;
  const long long rowB = (long long)B * TH;
#ifdef BPPSA_STEP_TRACE
  int tstep = 0;
#endif
  for (long long tau = 2 * (long long)blockIdx.x + g; tau < ntiles; tau += 2 * (long long)gridDim.x) {
    const long long q = q0 + tau / nbp;
    const int bp = (int)(tau % nbp);
    const int b = bp * 2 + (row >> 6);
    const int j = row & 63;
    const bool ok = b < B;
    const long long s0 = q * C, s1 = min(s0 + (long long)C, S);
    float c[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) c[k] = (16 * cgp + k == j && ok) ? 1.f : 0.f;
    for (long long sc = s0; sc < s1; sc += HCH) {
      const int n = (int)min((long long)HCH, s1 - sc);
      named_bar(1 + g, EPI16_THREADS);             // previous chunk fully consumed
      for (int e = et; e < 2 * n * 16; e += EPI16_THREADS) {
        const int bb2 = e / (n * 16), rem = e % (n * 16), st = rem / 16, ch = rem % 16;
        float* dst = hs + (bb2 * HCH + st) * TH + ch * 4;
        const int bs = bp * 2 + bb2;
        if (bs < B)
          cp_async16(dst, a.h + (long long)a.seg.time_of(sc + st) * rowB + (long long)bs * TH + ch * 4);
        else
          sts128(su32(dst), 0.f, 0.f, 0.f, 0.f);
      }
      asm volatile("cp.async.wait_all;\n" ::: "memory");
      for (int e = et; e < 2 * n * 16; e += EPI16_THREADS) {   // d = 1 - h^2 in place
        const int bb2 = e / (n * 16), rem = e % (n * 16), st = rem / 16, ch = rem % 16;
        const uint32_t p = hs_s + 4u * ((bb2 * HCH + st) * TH + ch * 4);
        const float4 h4 = lds128(p);
        sts128(p, 1.f - h4.x * h4.x, 1.f - h4.y * h4.y, 1.f - h4.z * h4.z, 1.f - h4.w * h4.w);
      }
      named_bar(1 + g, EPI16_THREADS);
      const uint32_t drow0 = hs_s + 4u * ((row >> 6) * HCH * TH + 16 * cgp);
      for (int st = 0; st < n; ++st) {
        STEP_TRACE(0);
        uint32_t hi[16], lo[16];
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          const float4 d4 = lds128(drow0 + 4u * (st * TH + 4 * q4));
          const float x4[4] = {d4.x * c[4 * q4], d4.y * c[4 * q4 + 1], d4.z * c[4 * q4 + 2], d4.w * c[4 * q4 + 3]};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            hi[4 * q4 + e] = __float_as_uint(x4[e]) & 0xFFFFE000u;
            lo[4 * q4 + e] = (__float_as_uint(x4[e] - __uint_as_float(hi[4 * q4 + e])) + 0x1000u) & 0xFFFFE000u;
          }
        }
#ifndef BPPSA_TRACE_NO_EPI
        tmem_st16(t_ahi, hi);
        tmem_st16(t_alo, lo);
        asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
#endif
        STEP_TRACE(1);
        tc_fence_before();
        named_bar(3 + g, EPI16_THREADS);           // the slot's A is complete
        STEP_TRACE(2);
        if (issuer) {
          tc_fence_after();
          // one slot's 16 MMAs go into the tensor queue back to back: with
          // interleaved batches both slots finish together and their
          // epilogues lock in phase instead of overlapping the other slot's MMAs
          if (lane == 0) lock_acquire(lock_s);
          __syncwarp();
#ifndef BPPSA_TRACE_NO_MMA
          mma16_commit(slot_base, bdesc, su32(&d_full[g]));
#else
          if (lane == 0)
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                             su32(&d_full[g])) : "memory");
          __syncwarp();
#endif
          if (lane == 0) lock_release(lock_s);
          __syncwarp();
        }
        STEP_TRACE(3);
        // one lane polls the MMA-completion barrier; the slot's other warps
        // sleep in a hardware barrier (polling warps slow the tensor pipe:
        // 24 warps in try_wait loops cost ~25 cycles per MMA, scripts/tc_rate3.cu)
        if (issuer) {
          if (lane == 0) mbar_wait(&d_full[g], ph);
          __syncwarp();
        }
        named_bar(5 + g, EPI16_THREADS);
        ph ^= 1;
        tc_fence_after();
        STEP_TRACE(4);
        float t[16];                               // c = (hh + lh) + (hl + ll), round-to-nearest
#ifndef BPPSA_TRACE_NO_EPI
        tmem_ld16(t_dh, c);
        tmem_ld16(t_dl, t);
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#else
        for (int k = 0; k < 16; ++k) t[k] = __uint_as_float(hi[k] ^ lo[k]);
#endif
        STEP_TRACE(5);
#ifdef BPPSA_STEP_TRACE
        ++tstep;
#endif
#pragma unroll
        for (int k = 0; k < 16; ++k) c[k] += t[k];
      }
    }
    if (ok) {
      float4* dst = reinterpret_cast<float4*>(agg_out + (((long long)b * n_out + q) * TH + j) * TH + 16 * cgp);
#pragma unroll
      for (int k4 = 0; k4 < 4; ++k4) dst[k4] = make_float4(c[4 * k4], c[4 * k4 + 1], c[4 * k4 + 2], c[4 * k4 + 3]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

// ---------------------------------------------------------------------------
// Level-0 DOWN-walk, 2 x 16 epilogue warps (thread = chain row x 16-column
// group), same MMA issue scheme as the up-sweep.  Chains are ordered q-major
// (id = q*B + b) so a tile's h rows at one step are a few runs of consecutive
// samples; each chain's h row for step st+1 is fetched with one 256-byte
// cp.async.bulk by the row's owner thread while step st computes (2-stage ring
// per slot, rows at a 272-byte stride so the column-slice reads are
// conflict-free), completion counted by an mbarrier with expect_tx.  grad_h is
// written from registers.  The D-ready and h-ready waits share one barrier.
// ---------------------------------------------------------------------------
constexpr int DROW = TH * 4 + 16;                          // padded h row in the ring
constexpr int DSTAGE = TM * DROW;                          // 34816 B
constexpr int OFF_RING16 = OFF_B + B_BYTES;                // [slot][2 stages][128 rows][DROW]
constexpr int OFF_BAR_D16 = OFF_RING16 + NSLOT * 2 * DSTAGE;   // d_full[2], h_full[2][2], tmem, lock
constexpr int SMEM_BYTES_D16 = OFF_BAR_D16 + 128 + 1024;

__device__ __forceinline__ void bulk_row(uint32_t dst, const float* src, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 256, [%2];\n" ::"r"(dst),
               "l"(src), "r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}\n" ::"r"(bar),
               "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive_s(uint32_t bar) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait_s(uint32_t bar, uint32_t parity) {
  asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" ::"r"(
                   bar), "r"(parity) : "memory");
}

__global__ void __launch_bounds__(NTHREADS16, 1) tc_leaf_down16_kernel(LeafArgs a, int C, const float* __restrict__ carry,
                                                                       long long nblk, float* __restrict__ grad_h,
                                                                       float* __restrict__ grad_init) {
  extern __shared__ uint8_t smem_raw[];
  char* smem = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* d_full = reinterpret_cast<uint64_t*>(smem + OFF_BAR_D16);
  uint64_t* h_full = d_full + NSLOT;                                    // [slot][stage]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(h_full + 2 * NSLOT);
  int* issue_lock = reinterpret_cast<int*>(tmem_slot + 1);
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const int B = a.seg.B;
  const long long S = a.seg.S();
  const long long nchains = (long long)B * nblk;
  const long long ntiles = (nchains + TM - 1) / TM;
  const long long rowB = (long long)B * TH;

  for (int e = threadIdx.x; e < TH * TH; e += NTHREADS16) {
    const int n = e / TH, k = e % TH;               // B[n][k] = W[k][n]: rows 0..63 hi, 64..127 lo
    const float w = __ldg(a.W + (long long)k * TH + n);
    const float hi = tf32_rn(w);
    *reinterpret_cast<float*>(smem + OFF_B + sw_off(n, k, B_ROWS)) = hi;
    *reinterpret_cast<float*>(smem + OFF_B + sw_off(TH + n, k, B_ROWS)) = tf32_rn(w - hi);
  }
  if (warp == 0) {
    if (lane == 0) {
      for (int s = 0; s < NSLOT; ++s) {
        mbar_init(&d_full[s], 1);
        for (int st = 0; st < 2; ++st) mbar_init(&h_full[2 * s + st], TM);   // one arrival per chain row
      }
      *issue_lock = 0;
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncwarp();
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);

  const int g = warp / EPI16_WARPS, wl = warp % EPI16_WARPS;
  const int row = (wl & 3) * 32 + lane;
  const int cgp = wl >> 2;
  const bool issuer = wl == 0, owner = cgp == 0;          // owner: fetches the row's h
  const uint32_t slot_base = tmem + 256 * g;
  const uint32_t lane_base = slot_base + ((uint32_t)((wl & 3) * 32) << 16);
  const uint32_t t_dh = lane_base + 16 * cgp, t_dl = t_dh + 64;
  const uint32_t t_ahi = lane_base + 128 + 16 * cgp, t_alo = lane_base + 192 + 16 * cgp;
  const uint32_t bb = __shfl_sync(0xffffffffu, su32(smem + OFF_B), 0);
  const uint32_t ring = su32(smem + OFF_RING16) + (uint32_t)(g * 2 * DSTAGE);
  const uint32_t lock_s = su32(issue_lock);
  const uint32_t dbar = su32(&d_full[g]), hbar0 = su32(&h_full[2 * g]);
  uint64_t bdesc[TH / 8];
#pragma unroll
  for (int kk = 0; kk < TH / 8; ++kk) bdesc[kk] = sdesc(bb + (uint32_t)((kk >> 2) * B_ROWS * 128 + (kk & 3) * 32));
  uint32_t dph = 0, gs = 0;                                // D phase; global step count of this slot (h ring)

  for (long long tau = 2 * (long long)blockIdx.x + g; tau < ntiles; tau += 2 * (long long)gridDim.x) {
    const long long id = tau * TM + row;
    const bool valid = id < nchains;
    const long long q = valid ? id / B : 0;
    const int b = valid ? (int)(id % B) : 0;
    const bool head = a.seg.head && q == 0;
    const long long s_start = head ? 1 : q * C, s1 = min(q * C + C, S);
    const int len = valid ? (int)(s1 - s_start) : 0;
    const bool total = valid && grad_init != nullptr && s1 == S;
    const float* hb = a.h + (long long)b * TH;
    float* gb = grad_h + (long long)b * TH + 16 * cgp;
    float c[16];
    {
      const float* src0 = head ? a.seed + (long long)b * TH : carry + ((long long)b * nblk + q) * TH;
#pragma unroll
      for (int k4 = 0; k4 < 4; ++k4) {
        const float4 v = valid ? __ldg(reinterpret_cast<const float4*>(src0 + 16 * cgp) + k4)
                               : make_float4(0.f, 0.f, 0.f, 0.f);
        c[4 * k4] = v.x; c[4 * k4 + 1] = v.y; c[4 * k4 + 2] = v.z; c[4 * k4 + 3] = v.w;
      }
    }
    // h row of step 0 into stage gs & 1
    if (owner) {
      const uint32_t bar = hbar0 + 8u * (gs & 1);
      if (len > 0) {
        mbar_arrive_tx(bar, 256);
        bulk_row(ring + (gs & 1) * DSTAGE + row * DROW, hb + (long long)a.seg.time_of(s_start) * rowB, bar);
      } else {
        mbar_arrive_s(bar);
      }
    }
    if (issuer) {
      if (lane == 0) mbar_wait_s(hbar0 + 8u * (gs & 1), (gs >> 1) & 1);
      __syncwarp();
    }
    named_bar(5 + g, EPI16_THREADS);
    for (int st = 0; st < C; ++st, ++gs) {
      const bool active = st < len;
      if (active) {                                  // exclusive output: grad_h[t(s)] = v before J_{t(s)}^T
        float4* gp = reinterpret_cast<float4*>(gb + (long long)a.seg.time_of(s_start + st) * rowB);
#pragma unroll
        for (int k4 = 0; k4 < 4; ++k4) gp[k4] = make_float4(c[4 * k4], c[4 * k4 + 1], c[4 * k4 + 2], c[4 * k4 + 3]);
      }
      if (owner && st + 1 < C) {                     // prefetch step st+1 (its stage was read at step st-1)
        const uint32_t nb = gs + 1;
        const uint32_t bar = hbar0 + 8u * (nb & 1);
        if (st + 1 < len) {
          mbar_arrive_tx(bar, 256);
          bulk_row(ring + (nb & 1) * DSTAGE + row * DROW, hb + (long long)a.seg.time_of(s_start + st + 1) * rowB, bar);
        } else {
          mbar_arrive_s(bar);
        }
      }
      uint32_t hi[16], lo[16];
      const uint32_t hrow = ring + (gs & 1) * DSTAGE + row * DROW + 64u * cgp;
#pragma unroll
      for (int q4 = 0; q4 < 4; ++q4) {
        float4 h4 = lds128(hrow + 16u * q4);
        if (!active) h4 = make_float4(1.f, 1.f, 1.f, 1.f);   // d = 0: an idle row contributes nothing
        const float x4[4] = {(1.f - h4.x * h4.x) * c[4 * q4], (1.f - h4.y * h4.y) * c[4 * q4 + 1],
                             (1.f - h4.z * h4.z) * c[4 * q4 + 2], (1.f - h4.w * h4.w) * c[4 * q4 + 3]};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          hi[4 * q4 + e] = __float_as_uint(x4[e]) & 0xFFFFE000u;
          lo[4 * q4 + e] = (__float_as_uint(x4[e] - __uint_as_float(hi[4 * q4 + e])) + 0x1000u) & 0xFFFFE000u;
        }
      }
      tmem_st16(t_ahi, hi);
      tmem_st16(t_alo, lo);
      asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
      tc_fence_before();
      named_bar(3 + g, EPI16_THREADS);               // the slot's A is complete (and stage gs&1 consumed)
      if (issuer) {
        tc_fence_after();
        if (lane == 0) lock_acquire(lock_s);
        __syncwarp();
        mma16_commit(slot_base, bdesc, dbar);
        if (lane == 0) {
          lock_release(lock_s);
          mbar_wait_s(dbar, dph);
          if (st + 1 < C) mbar_wait_s(hbar0 + 8u * ((gs + 1) & 1), ((gs + 1) >> 1) & 1);
        }
        __syncwarp();
      }
      named_bar(5 + g, EPI16_THREADS);               // D of step st and h of step st+1 are ready
      dph ^= 1;
      tc_fence_after();
      float t[16];
      tmem_ld16(t_dh, c);
      tmem_ld16(t_dl, t);
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
      for (int k = 0; k < 16; ++k) c[k] += t[k];
      if (total && st == len - 1) {                  // inclusive extra: J_{t(S-1)}^T grad_h[t(S-1)]
        float4* dst = reinterpret_cast<float4*>(grad_init + (long long)b * TH + 16 * cgp);
#pragma unroll
        for (int k4 = 0; k4 < 4; ++k4) dst[k4] = make_float4(c[4 * k4], c[4 * k4 + 1], c[4 * k4 + 2], c[4 * k4 + 3]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

// ---------------------------------------------------------------------------
// Level-0 UP-sweep on kind::f16 (3xFP16 with per-chain power-of-two scaling).
//
// fp16 has tf32's 11 significant bits but runs at twice the tensor rate, so a
// 2-term split x = x1 + x2, W = W1 + W2 gives the same 22-bit products as
// 3xTF32 for half the MMA time — provided every operand sits in fp16's
// exponent range.  W is scaled once by 2^sw (max |W| 2^sw in [2^14, 2^15)).
// Every chain row is rescaled at every step by a power of two 2^s chosen from
// a BOUND on the row's new maximum, known before the step's data:
//     |x'_s|_inf <= dmax_s * |c'_s|_inf <= dmax_s * G * M_{s-1}
// (d = 1 - h^2 in [0, 1]; dmax_s = max_k d_s[k] of the sample, computed when
// h is staged; G = max_n sum_k |B[n][k]| of the scaled W; M_{s-1} = the exact
// row maximum of the previous scaled operand, exchanged between the row's four
// threads through shared memory WITHOUT a barrier of its own — the step's
// MMA barriers order it, double-buffered by step parity).  So x^ = x' 2^s <
// 2^15 always (no fp16 overflow) and, for random W, its maximum sits near
// 2^11: x1 is normal for entries down to 2^-24 of it and the absolute error
// of anything smaller stays below 2^-35 of the row maximum.
// The scaled chain c' = c 2^E keeps its exponent E (an integer per row, the
// same in the row's four threads); the aggregate is written as c' 2^-E.
// Per step and tile: 12 MMAs M128 N64 K16 into one 64-column accumulator,
// small products first (x2 W1, x1 W2, x1 W1; mma12_f16_commit_n64): the
// fold is bound by TMEM traffic, so the narrow accumulator (half the epilogue
// loads of the former 8 N = 128 MMAs against [W1 | W2]) is the faster form.
// A1 / A2 are packed f16x2 in TMEM (even k in the low half).
// ---------------------------------------------------------------------------
constexpr int F_B_BYTES = 2 * TH * TH * 2;                 // [W1 | W2]: 128 rows x 64 fp16 = 16 KB
constexpr int F_OFF_H = F_B_BYTES;
constexpr int F_OFF_RED = F_OFF_H + 2 * NSLOT * H_BYTES;   // h: [slot][2 chunk buffers] (f16g uses the first two)
                                                           // red: [slot][parity][128 rows][4 column groups] u32
constexpr int F_OFF_DMX = F_OFF_RED + NSLOT * 2 * TM * 16; // [slot][2 samples][HCH] dmax
constexpr int F_OFF_BAR = F_OFF_DMX + NSLOT * 2 * HCH * 4;
constexpr int F_SMEM_BYTES = F_OFF_BAR + 64 + 1024;
__host__ __device__ constexpr uint32_t idesc_f16(int N) {
  return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(TM >> 4) << 24);   // D f32, A/B f16, K-major
}
constexpr uint32_t IDESC_F16 = idesc_f16(128);

// element (row, k) of a K-major SWIZZLE_128B fp16 tile with K = 64 (one 128-byte row per row)
__device__ __forceinline__ uint32_t sw16_off(int row, int k) {
  return (uint32_t)((row >> 3) * 1024 + (row & 7) * 128 + (((k >> 3) ^ (row & 7)) << 4) + (k & 7) * 2);
}

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(taddr), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}

constexpr uint32_t IDESC_F16_N64 = idesc_f16(64);
#ifndef FOLD_WPS
#define FOLD_WPS 8                      // epilogue warps per slot of the fold
#endif

// All three products into one 64-column accumulator (N = 64 MMAs), small
// first: x2 W1 (init), x1 W2, then x1 W1; the epilogue loads 64 columns
__device__ __forceinline__ void mma12_f16_commit_n64(uint32_t d, const uint64_t (&bd)[4], const uint64_t (&bw2)[4],
                                                     uint32_t bar) {
  asm volatile(
      "{\n"
      " .reg .pred e, f, t;\n"
      " .reg .b32 a;\n"
      " setp.ne.b32 f, 0, 0;\n"
      " setp.eq.b32 t, 0, 0;\n"
      " elect.sync _|e, 0xffffffff;\n"
      " add.u32 a, %0, 160;\n @e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], %1, %5, f;\n"
      " add.u32 a, %0, 168;\n @e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], %2, %5, t;\n"
      " add.u32 a, %0, 176;\n @e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], %3, %5, t;\n"
      " add.u32 a, %0, 184;\n @e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], %4, %5, t;\n"
      " add.u32 a, %0, 128;\n @e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], %7, %5, t;\n"
      " add.u32 a, %0, 136;\n @e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], %8, %5, t;\n"
      " add.u32 a, %0, 144;\n @e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], %9, %5, t;\n"
      " add.u32 a, %0, 152;\n @e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], %10, %5, t;\n"
      " add.u32 a, %0, 128;\n @e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], %1, %5, t;\n"
      " add.u32 a, %0, 136;\n @e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], %2, %5, t;\n"
      " add.u32 a, %0, 144;\n @e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], %3, %5, t;\n"
      " add.u32 a, %0, 152;\n @e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], %4, %5, t;\n"
      " @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%6];\n"
      "}\n" ::"r"(d),
      "l"(bd[0]), "l"(bd[1]), "l"(bd[2]), "l"(bd[3]), "r"(IDESC_F16_N64), "r"(bar), "l"(bw2[0]), "l"(bw2[1]),
      "l"(bw2[2]), "l"(bw2[3])
      : "memory");
}

// c' <- D (one 64-column accumulator) for this thread's CPT columns
template <int CPT, int NP>
__device__ __forceinline__ void load_d_one(uint32_t t_d1, float2 (&c2)[NP]) {
#pragma unroll
  for (int h = 0; h < CPT / 16; ++h) {
    float t1[16];
    tmem_ld16(t_d1 + 16 * h, t1);
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
    for (int i = 0; i < 8; ++i) c2[8 * h + i] = make_float2(t1[2 * i], t1[2 * i + 1]);
  }
}

__device__ __forceinline__ void mma8_f16_commit_a1first(uint32_t d, const uint64_t (&bd)[4], uint32_t bar) {
  asm volatile(
      "{\n"
      " .reg .pred e, f, t;\n"
      " .reg .b32 a;\n"
      " setp.ne.b32 f, 0, 0;\n"
      " setp.eq.b32 t, 0, 0;\n"
      " elect.sync _|e, 0xffffffff;\n"
      " add.u32 a, %0, 128;\n @e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], %1, %5, f;\n"
      " add.u32 a, %0, 136;\n @e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], %2, %5, t;\n"
      " add.u32 a, %0, 144;\n @e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], %3, %5, t;\n"
      " add.u32 a, %0, 152;\n @e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], %4, %5, t;\n"
      " add.u32 a, %0, 160;\n @e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], %1, %7, t;\n"
      " add.u32 a, %0, 168;\n @e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], %2, %7, t;\n"
      " add.u32 a, %0, 176;\n @e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], %3, %7, t;\n"
      " add.u32 a, %0, 184;\n @e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], %4, %7, t;\n"
      " @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%6];\n"
      "}\n" ::"r"(d),
      "l"(bd[0]), "l"(bd[1]), "l"(bd[2]), "l"(bd[3]), "r"(IDESC_F16), "r"(bar), "r"(IDESC_F16_N64)
      : "memory");
}

__device__ __forceinline__ uint32_t h2_bits(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }

// W exponent shift sw (max |W| 2^sw in [2^14, 2^15), clamped: W = 0 gives a
// harmless shift) and G = max_n sum_k |W[k][n]| 2^sw (rounded up by 2^-8).
// Called by all threads; red[0..1] are zeroed shared words.
__device__ __forceinline__ void w_scale(const float* W, uint32_t* red, int* sw_out, float* G_out) {
  uint32_t m = 0;
  for (int e = threadIdx.x; e < TH * TH; e += blockDim.x) m = max(m, __float_as_uint(fabsf(__ldg(W + e))));
  m = __reduce_max_sync(0xffffffffu, m);
  if ((threadIdx.x & 31) == 0) atomicMax(red, m);
  __syncthreads();
  const int sw = max(-100, min(100, 141 - (int)(red[0] >> 23)));
  uint32_t gs = 0;
  if (threadIdx.x < TH) {
    float acc = 0.f;
    for (int k = 0; k < TH; ++k) acc += fabsf(__ldg(W + (long long)k * TH + threadIdx.x));
    gs = __float_as_uint(ldexpf(acc, sw) * (1.f + 1.f / 256.f));
  }
  gs = __reduce_max_sync(0xffffffffu, gs);
  if ((threadIdx.x & 31) == 0 && threadIdx.x < TH) atomicMax(red + 1, gs);
  __syncthreads();
  *sw_out = sw;
  *G_out = __uint_as_float(red[1]);
}

// c' <- D1 + D2 for this thread's CPT columns (the accumulator halves), RN
template <int CPT, int NP>
__device__ __forceinline__ void load_d_sum(uint32_t t_d1, uint32_t t_d2, float2 (&c2)[NP]) {
#pragma unroll
  for (int h = 0; h < CPT / 16; ++h) {
    float t1[16], t2[16];
    tmem_ld16(t_d1 + 16 * h, t1);
    tmem_ld16(t_d2 + 16 * h, t2);
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
    for (int i = 0; i < 8; ++i)
      c2[8 * h + i] = __fadd2_rn(make_float2(t1[2 * i], t1[2 * i + 1]), make_float2(t2[2 * i], t2[2 * i + 1]));
  }
}

// WPS = epilogue warps per slot.  8 (thread = chain row x 32 columns, 512
// threads, up to 128 registers) measured best at C4: 29.8 ms against 34.8
// with 16 (row x 16 columns: 64 registers force address rematerialisation and
// the per-thread overhead is amortised over half the elements) and 31.7 with
// 4 (one thread per row, no max exchange, but one warp per SMSP per slot).
template <int WPS>
__global__ void __launch_bounds__(64 * WPS, 1) tc_leaf_up_f16_kernel(LeafArgs a, int C, float* __restrict__ agg_out,
                                                                   long long n_out, long long q0) {
  constexpr int EPI = 32 * WPS, NT = 2 * EPI;     // threads per slot / per CTA
  constexpr int NCG = WPS / 4, CPT = TH / NCG, NP = CPT / 2;   // column groups; columns / pairs per thread
  extern __shared__ uint8_t smem_raw[];
  char* smem = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* d_full = reinterpret_cast<uint64_t*>(smem + F_OFF_BAR);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(d_full + NSLOT);
  int* issue_lock = reinterpret_cast<int*>(tmem_slot + 1);
  uint32_t* wred = reinterpret_cast<uint32_t*>(issue_lock + 1);
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const int B = a.seg.B;
  const long long S = a.seg.S();
  const long long nq = n_out - q0;
  const int nbp = (B + 1) / 2;
  const long long ntiles = (long long)nbp * nq;

  if (threadIdx.x < 2) wred[threadIdx.x] = 0;
  __syncthreads();
  int sw;
  float G;
  w_scale(a.W, wred, &sw, &G);
  {
    const float wsc = __int_as_float((sw + 127) << 23);
    for (int e = threadIdx.x; e < TH * TH; e += NT) {
      const int n = e / TH, k = e % TH;             // B[n][k] = W[k][n] 2^sw: rows 0..63 W1, 64..127 W2
      const float w = __ldg(a.W + (long long)k * TH + n) * wsc;
      const __half w1 = __float2half_rn(w);
      *reinterpret_cast<__half*>(smem + sw16_off(n, k)) = w1;
      *reinterpret_cast<__half*>(smem + sw16_off(TH + n, k)) = __float2half_rn(w - __half2float(w1));
    }
  }
  if (warp == 0) {
    if (lane == 0) {
      for (int s = 0; s < NSLOT; ++s) mbar_init(&d_full[s], 1);
      *issue_lock = 0;
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncwarp();
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);

  const int g = warp / WPS, wl = warp % WPS;
  const int row = (wl & 3) * 32 + lane;
  const int cgp = wl >> 2;
  const int et = wl * 32 + lane;
  const bool issuer = wl == 0;
  const uint32_t slot_base = tmem + 256 * g;
  const uint32_t lane_base = slot_base + ((uint32_t)((wl & 3) * 32) << 16);
  const uint32_t t_d1 = lane_base + CPT * cgp;     // the 64-column accumulator
  const uint32_t t_a1 = lane_base + 128 + NP * cgp, t_a2 = lane_base + 160 + NP * cgp;
  // two chunk buffers per slot: the next chunk's h (this tile's, or the next
  // tile's first) is copied while the current chunk's steps run
  char* const hsb0 = smem + F_OFF_H + (2 * g) * H_BYTES;
  auto hsb = [&](int c) { return reinterpret_cast<float*>(hsb0 + c * H_BYTES); };
  float* dmx = reinterpret_cast<float*>(smem + F_OFF_DMX) + g * 2 * HCH;       // [2 samples][HCH]
  const uint32_t red0 = su32(smem + F_OFF_RED) + (uint32_t)(((g * 2) * TM + row) * 16);   // parity 0 row word
  const uint32_t bb = __shfl_sync(0xffffffffu, su32(smem), 0);
  const uint32_t lock_s = su32(issue_lock);
  uint64_t bdesc[4];
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) bdesc[kk] = sdesc(bb + (uint32_t)(kk * 32));
  uint64_t bw2[4];                                 // the W2 rows at every K step
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) bw2[kk] = sdesc(bb + 8192u + (uint32_t)(kk * 32));
  uint32_t ph = 0, par = 0;                        // D phase; parity of the max exchange buffer
#ifdef BPPSA_STEP_TRACE
  int tstep = 0;
#endif
  const long long rowB = (long long)B * TH;
  // one chunk of tile tx from slot scx: HCH steps of the h rows of its two
  // samples, asynchronous (one commit group)
  auto issue_chunk = [&](long long tx, long long scx, float* hb) {
    const long long qx = q0 + tx / nbp;
    const int bpx = (int)(tx % nbp);
    const int nx = (int)min((long long)HCH, min(qx * C + (long long)C, S) - scx);
    for (int e = et; e < 2 * nx * 16; e += EPI) {
      const int bb2 = e / (nx * 16), rem = e % (nx * 16), st = rem / 16, ch = rem % 16;
      float* dst = hb + (bb2 * HCH + st) * TH + ch * 4;
      const int bs = bpx * 2 + bb2;
      if (bs < B)
        cp_async16(dst, a.h + (long long)a.seg.time_of(scx + st) * rowB + (long long)bs * TH + ch * 4);
      else
        sts128(su32(dst), 0.f, 0.f, 0.f, 0.f);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  auto tile_s0 = [&](long long tx) {
    const long long qx = q0 + tx / nbp;
    return (a.seg.head && qx == 0) ? 1LL : qx * C;
  };
  int cb = 0;                                      // buffer of the current chunk
  {
    const long long t0 = 2 * (long long)blockIdx.x + g;
    if (t0 < ntiles) issue_chunk(t0, tile_s0(t0), hsb(0));
  }
  for (long long tau = 2 * (long long)blockIdx.x + g; tau < ntiles; tau += 2 * (long long)gridDim.x) {
    const long long q = q0 + tau / nbp;
    const int bp = (int)(tau % nbp);
    const int b = bp * 2 + (row >> 6);
    const int j = row & 63;
    const bool ok = b < B;
    // the head block (slot 0 = the seed vector) is folded as the matrix of its
    // leaves, slots 1..C-1; head_apply_kernel then applies it to the seed
    const long long s0 = (a.seg.head && q == 0) ? 1 : q * C, s1 = min(q * C + (long long)C, S);
    float2 c2[NP];                                 // c' = c 2^E (pairs of columns)
    int E = 0;
    float bound = 1.f / G;                         // G * bound = |c'_0|_inf bound (one-hot start)
    bool first = true;
#pragma unroll
    for (int i = 0; i < NP; ++i)
      c2[i] = make_float2((CPT * cgp + 2 * i == j && ok) ? 1.f : 0.f, (CPT * cgp + 2 * i + 1 == j && ok) ? 1.f : 0.f);
    for (long long sc = s0; sc < s1; sc += HCH) {
      const int n = (int)min((long long)HCH, s1 - sc);
      float* hs = hsb(cb);
      const uint32_t hs_s = su32(hs);
      asm volatile("cp.async.wait_all;\n" ::: "memory");   // this chunk's copies (issued one chunk ago)
      named_bar(1 + g, EPI);             // every thread's copies landed; the previous chunk is consumed
      // d = 1 - h^2 in place and dmax per (sample, step): 16 consecutive lanes
      // hold one 64-wide row (2n*16 is a multiple of 32: whole warps iterate)
      for (int e = et; e < 2 * n * 16; e += EPI) {
        const int bb2 = e / (n * 16), rem = e % (n * 16), st = rem / 16, ch = rem % 16;
        const uint32_t p = hs_s + 4u * ((bb2 * HCH + st) * TH + ch * 4);
        const float4 h4 = lds128(p);
        const float4 d4 = make_float4(1.f - h4.x * h4.x, 1.f - h4.y * h4.y, 1.f - h4.z * h4.z, 1.f - h4.w * h4.w);
        sts128(p, d4.x, d4.y, d4.z, d4.w);
        float m = fmaxf(fmaxf(d4.x, d4.y), fmaxf(d4.z, d4.w));
#pragma unroll
        for (int o = 8; o >= 1; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (ch == 0) dmx[bb2 * HCH + st] = m;
      }
      named_bar(1 + g, EPI);
      {                                  // prefetch the next chunk into the other buffer
        const long long tn = tau + 2 * (long long)gridDim.x;
        if (sc + HCH < s1) issue_chunk(tau, sc + HCH, hsb(cb ^ 1));
        else if (tn < ntiles) issue_chunk(tn, tile_s0(tn), hsb(cb ^ 1));
      }
      cb ^= 1;
      uint32_t dp = hs_s + 4u * ((row >> 6) * HCH * TH + CPT * cgp);  // this thread's d slice of step st
      uint32_t dmp = su32(dmx + (row >> 6) * HCH);                      // dmax of step st
      for (int st = 0; st < n; ++st, dp += 4u * TH, dmp += 4u) {
        STEP_TRACE(0);
        // (overlaps the previous step's MMAs) scale 2^s from the bound
        // dmax_s * G * M_{s-1}, folded into d: ds = d 2^s
        float dms;
        asm volatile("ld.shared.f32 %0, [%1];\n" : "=f"(dms) : "r"(dmp));
        const float f = G * bound * dms;
        const int s = min(127, 141 - (int)(__float_as_uint(f) >> 23));
        const float2 scl = make_float2(__int_as_float((s + 127) << 23), __int_as_float((s + 127) << 23));
        E += s + sw;
        float2 ds[NP];
#pragma unroll
        for (int q4 = 0; q4 < CPT / 4; ++q4) {
          const float4 d4 = lds128(dp + 16u * q4);
          ds[2 * q4] = __fmul2_rn(make_float2(d4.x, d4.y), scl);
          ds[2 * q4 + 1] = __fmul2_rn(make_float2(d4.z, d4.w), scl);
        }
        if (!first) {                              // D of the previous step
          if (issuer) {
            STEP_TRACE(6);
            if (lane == 0) mbar_wait(&d_full[g], ph);
            STEP_TRACE(7);
            __syncwarp();
          }
          named_bar(5 + g, EPI);
          ph ^= 1;
          tc_fence_after();
          STEP_TRACE(4);
          load_d_one<CPT>(t_d1, c2);
          STEP_TRACE(5);
        }
        first = false;
        float pm = 0.f;
        uint32_t p1[NP], p2[NP];
#pragma unroll
        for (int i = 0; i < NP; ++i) {
          const float2 x = __fmul2_rn(c2[i], ds[i]);
          pm = fmaxf(pm, fmaxf(fabsf(x.x), fabsf(x.y)));
          // x1 = x truncated to 11 significant bits (exact in fp16 for |x| >= 2^-14;
          // below that the conversion rounds at 2^-25, < 2^-36 of the row maximum)
          const float2 f1 = make_float2(__uint_as_float(__float_as_uint(x.x) & 0xFFFFE000u),
                                        __uint_as_float(__float_as_uint(x.y) & 0xFFFFE000u));
          const float2 r = __fadd2_rn(x, make_float2(-f1.x, -f1.y));
          p1[i] = h2_bits(__floats2half2_rn(f1.x, f1.y));
          p2[i] = h2_bits(__floats2half2_rn(r.x, r.y));
        }
        const uint32_t redp = red0 + par * (TM * 16);
        if constexpr (NCG > 1)
          asm volatile("st.shared.u32 [%0], %1;\n" ::"r"(redp + 4u * cgp), "r"(__float_as_uint(pm)) : "memory");
#pragma unroll
        for (int h8 = 0; h8 < NP / 8; ++h8) {
          tmem_st8(t_a1 + 8 * h8, *reinterpret_cast<const uint32_t(*)[8]>(p1 + 8 * h8));
          tmem_st8(t_a2 + 8 * h8, *reinterpret_cast<const uint32_t(*)[8]>(p2 + 8 * h8));
        }
        asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
        STEP_TRACE(1);
        tc_fence_before();
        named_bar(3 + g, EPI);           // the slot's A and the row maxima are complete
        STEP_TRACE(2);
        if (issuer) {
          tc_fence_after();
          mma12_f16_commit_n64(slot_base, bdesc, bw2, su32(&d_full[g]));
          STEP_TRACE(3);
        }
        if constexpr (NCG == 4) {
          uint32_t m4[4];
          asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];\n"
                       : "=r"(m4[0]), "=r"(m4[1]), "=r"(m4[2]), "=r"(m4[3])
                       : "r"(redp)
                       : "memory");
          bound = __uint_as_float(max(max(m4[0], m4[1]), max(m4[2], m4[3])));
        } else if constexpr (NCG == 1) {
          bound = pm;                              // the whole row is this thread's
        } else {
          uint32_t m2[2];
          asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];\n" : "=r"(m2[0]), "=r"(m2[1]) : "r"(redp) : "memory");
          bound = __uint_as_float(max(m2[0], m2[1]));
        }
        par ^= 1;
#ifdef BPPSA_STEP_TRACE
        ++tstep;
#endif
      }
    }
    // D of the tile's last step (none for an empty head block: the identity)
    if (!first) {
    if (issuer) {
      if (lane == 0) mbar_wait(&d_full[g], ph);
      __syncwarp();
    }
    named_bar(5 + g, EPI);
    ph ^= 1;
    tc_fence_after();
      load_d_one<CPT>(t_d1, c2);
    }
    if (ok) {
      float4* dst = reinterpret_cast<float4*>(agg_out + (((long long)b * n_out + q) * TH + j) * TH + CPT * cgp);
#pragma unroll
      for (int k4 = 0; k4 < CPT / 4; ++k4)
        dst[k4] = make_float4(ldexpf(c2[2 * k4].x, -E), ldexpf(c2[2 * k4].y, -E), ldexpf(c2[2 * k4 + 1].x, -E),
                              ldexpf(c2[2 * k4 + 1].y, -E));
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(TMEM_COLS));
  }
}


// ---------------------------------------------------------------------------
// The 3xFP16 fold for 16 <= H < 64 (H % 4 == 0; configs 1-2 have H = 20):
// the H = 64 machinery with W zero-padded to 64 x 64, and a tile packed with
// G = 128 / H groups of H chains (group = one level-0 block of one sample;
// groups in (block, sample) order, so a tile may span blocks of different
// lengths: every row carries its own start slot and length, its aggregate is
// captured right after its last real step and its h rows stage as zeros
// afterwards).  8 epilogue warps per slot as in tc_leaf_up_f16_kernel<8>;
// columns >= H stay zero (d = 0 there).  HG steps are staged per chunk.
// ---------------------------------------------------------------------------
constexpr int HG = 16;

__device__ __forceinline__ void w_scale_h(const float* W, int H, uint32_t* red, int* sw_out, float* G_out) {
  uint32_t m = 0;
  for (int e = threadIdx.x; e < H * H; e += blockDim.x) m = max(m, __float_as_uint(fabsf(__ldg(W + e))));
  m = __reduce_max_sync(0xffffffffu, m);
  if ((threadIdx.x & 31) == 0) atomicMax(red, m);
  __syncthreads();
  const int sw = max(-100, min(100, 141 - (int)(red[0] >> 23)));
  uint32_t gs = 0;
  if (threadIdx.x < H) {
    float acc = 0.f;
    for (int k = 0; k < H; ++k) acc += fabsf(__ldg(W + (long long)k * H + threadIdx.x));
    gs = __float_as_uint(ldexpf(acc, sw) * (1.f + 1.f / 256.f));
  }
  gs = __reduce_max_sync(0xffffffffu, gs);
  if ((threadIdx.x & 31) == 0 && threadIdx.x < ((H + 31) & ~31)) atomicMax(red + 1, gs);
  __syncthreads();
  *sw_out = sw;
  *G_out = __uint_as_float(red[1]);
}

__global__ void __launch_bounds__(512, 1) tc_leaf_up_f16g_kernel(LeafArgs a, int C, float* __restrict__ agg_out,
                                                                 long long n_out, long long q0) {
  constexpr int WPS = 8, EPI = 32 * WPS, NT = 2 * EPI, NCG = 2, CPT = 32, NP = 16;
  extern __shared__ uint8_t smem_raw[];
  char* smem = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* d_full = reinterpret_cast<uint64_t*>(smem + F_OFF_BAR);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(d_full + NSLOT);
  uint32_t* wred = tmem_slot + 2;
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const int B = a.seg.B, H = a.seg.H;
  const int GRP = TM / H;                                   // groups per tile
  const long long S = a.seg.S();
  const long long nq = n_out - q0;
  const long long ngroups = (long long)B * nq;
  const long long ntiles = (ngroups + GRP - 1) / GRP;

  if (threadIdx.x < 2) wred[threadIdx.x] = 0;
  __syncthreads();
  int sw;
  float G;
  w_scale_h(a.W, H, wred, &sw, &G);
  {
    const float wsc = __int_as_float((sw + 127) << 23);
    for (int e = threadIdx.x; e < TH * TH; e += NT) {
      const int n = e / TH, k = e % TH;             // B[n][k] = W[k][n] 2^sw (zero beyond H)
      const float w = (n < H && k < H) ? __ldg(a.W + (long long)k * H + n) * wsc : 0.f;
      const __half w1 = __float2half_rn(w);
      *reinterpret_cast<__half*>(smem + sw16_off(n, k)) = w1;
      *reinterpret_cast<__half*>(smem + sw16_off(TH + n, k)) = __float2half_rn(w - __half2float(w1));
    }
  }
  if (warp == 0) {
    if (lane == 0) {
      for (int s = 0; s < NSLOT; ++s) mbar_init(&d_full[s], 1);
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncwarp();
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);

  const int g = warp / WPS, wl = warp % WPS;
  const int row = (wl & 3) * 32 + lane;
  const int cgp = wl >> 2;
  const int et = wl * 32 + lane;
  const bool issuer = wl == 0;
  const uint32_t slot_base = tmem + 256 * g;
  const uint32_t lane_base = slot_base + ((uint32_t)((wl & 3) * 32) << 16);
  const uint32_t t_d1 = lane_base + CPT * cgp;     // the 64-column accumulator
  const uint32_t t_a1 = lane_base + 128 + NP * cgp, t_a2 = lane_base + 160 + NP * cgp;
  float* hs = reinterpret_cast<float*>(smem + F_OFF_H + g * H_BYTES);    // [GRP][HG][64] d
  const uint32_t hs_s = su32(hs);
  float* dmx = reinterpret_cast<float*>(smem + F_OFF_DMX) + g * 2 * HCH;  // [GRP][HG] dmax (2 HCH >= 8 HG)
  const uint32_t red0 = su32(smem + F_OFF_RED) + (uint32_t)(((g * 2) * TM + row) * 16);
  const uint32_t bb = __shfl_sync(0xffffffffu, su32(smem), 0);
  uint64_t bdesc[4];
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) bdesc[kk] = sdesc(bb + (uint32_t)(kk * 32));
  uint64_t bw2[4];                                 // the W2 rows (64..127) at every K step
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) bw2[kk] = sdesc(bb + 8192u + (uint32_t)(kk * 32));
  uint32_t ph = 0, par = 0;
  const long long rowB = (long long)B * H;
  const int grp = row / H, j = row % H;
  for (long long tau = 2 * (long long)blockIdx.x + g; tau < ntiles; tau += 2 * (long long)gridDim.x) {
    const long long gf = tau * GRP + grp;
    const bool ok = grp < GRP && gf < ngroups;
    const long long q = q0 + (ok ? gf / B : 0);
    const int b = ok ? (int)(gf % B) : 0;
    const long long s0 = (a.seg.head && q == 0) ? 1 : q * C, s1 = min(q * C + (long long)C, S);
    const int len = ok ? (int)max(0LL, s1 - s0) : 0;
    // steps of the tile: the longest of its groups
    int nsteps = 0;
    for (int r = 0; r < GRP; ++r) {
      const long long gr = tau * GRP + r;
      if (gr >= ngroups) break;
      const long long qr = q0 + gr / B;
      const long long sr0 = (a.seg.head && qr == 0) ? 1 : qr * C, sr1 = min(qr * C + (long long)C, S);
      nsteps = max(nsteps, (int)max(0LL, sr1 - sr0));
    }
    float2 c2[NP];
    int E = 0;
    float bound = 1.f / G;
    bool first = true;
    float* aggrow = agg_out + (((long long)b * n_out + q) * H + j) * H;
#pragma unroll
    for (int i = 0; i < NP; ++i)
      c2[i] = make_float2((CPT * cgp + 2 * i == j && ok) ? 1.f : 0.f, (CPT * cgp + 2 * i + 1 == j && ok) ? 1.f : 0.f);
    if (ok && len == 0) {                           // an empty head block: the identity
      for (int c = 0; c < H; ++c)
        if (c >= CPT * cgp && c < CPT * cgp + CPT) aggrow[c] = (c == j) ? 1.f : 0.f;
    }
    for (int sb = 0; sb < nsteps; sb += HG) {
      const int n = min(HG, nsteps - sb);
      named_bar(1 + g, EPI);                        // the previous chunk's d is consumed
      // stage h rows (H floats, 16-byte pieces) of every group, zeros past a group's length
      const int nc4 = H / 4;
      for (int e = et; e < GRP * n * 16; e += EPI) {
        const int r = e / (n * 16), rem = e % (n * 16), st = rem / 16, c4 = rem % 16;
        float* dst = hs + (r * HG + st) * TH + c4 * 4;
        const long long gr = tau * GRP + r;
        bool live = false;
        long long src = 0;
        if (gr < ngroups && c4 < nc4) {
          const long long qr = q0 + gr / B;
          const int br = (int)(gr % B);
          const long long sr0 = (a.seg.head && qr == 0) ? 1 : qr * C, sr1 = min(qr * C + (long long)C, S);
          if (sb + st < sr1 - sr0) {
            live = true;
            src = (long long)a.seg.time_of(sr0 + sb + st) * rowB + (long long)br * H + c4 * 4;
          }
        }
        if (live) cp_async16(dst, a.h + src);
        else sts128(su32(dst), 1.f, 1.f, 1.f, 1.f);  // h = 1: d = 0 (padding columns, finished groups)
      }
      asm volatile("cp.async.wait_all;\n" ::: "memory");
      named_bar(1 + g, EPI);
      const int tot = GRP * n * 16;
      for (int e = et; e < ((tot + 31) & ~31); e += EPI) {   // d = 1 - h^2 in place, dmax per (group, step)
        const bool v = e < tot;                     // whole warps iterate (16 lanes per row)
        const int r = e / (n * 16), rem = e % (n * 16), st = rem / 16, c4 = rem % 16;
        float m = 0.f;
        if (v) {
          const uint32_t p = hs_s + 4u * ((r * HG + st) * TH + c4 * 4);
          const float4 h4 = lds128(p);
          const float4 d4 = make_float4(1.f - h4.x * h4.x, 1.f - h4.y * h4.y, 1.f - h4.z * h4.z, 1.f - h4.w * h4.w);
          sts128(p, d4.x, d4.y, d4.z, d4.w);
          m = fmaxf(fmaxf(d4.x, d4.y), fmaxf(d4.z, d4.w));
        }
#pragma unroll
        for (int o = 8; o >= 1; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (v && c4 == 0) dmx[r * HG + st] = m;
      }
      named_bar(1 + g, EPI);
      const int grs = min(grp, GRP - 1);            // idle rows read group GRP-1's data (finite, unused)
      uint32_t dp = hs_s + 4u * (grs * HG * TH + CPT * cgp);
      uint32_t dmp = su32(dmx + grs * HG);
      for (int st = 0; st < n; ++st, dp += 4u * TH, dmp += 4u) {
        const int gst = sb + st;
        float dms;
        asm volatile("ld.shared.f32 %0, [%1];\n" : "=f"(dms) : "r"(dmp));
        const float f = G * bound * dms;
        const int s = min(127, 141 - (int)(__float_as_uint(f) >> 23));
        const float2 scl = make_float2(__int_as_float((s + 127) << 23), __int_as_float((s + 127) << 23));
        float2 ds[NP];
#pragma unroll
        for (int q4 = 0; q4 < CPT / 4; ++q4) {
          const float4 d4 = lds128(dp + 16u * q4);
          ds[2 * q4] = __fmul2_rn(make_float2(d4.x, d4.y), scl);
          ds[2 * q4 + 1] = __fmul2_rn(make_float2(d4.z, d4.w), scl);
        }
        if (!first) {
          if (issuer) {
            if (lane == 0) mbar_wait(&d_full[g], ph);
            __syncwarp();
          }
          named_bar(5 + g, EPI);
          ph ^= 1;
          tc_fence_after();
          load_d_one<CPT>(t_d1, c2);
          if (ok && gst == len) {                   // aggregate after the group's last real step
#pragma unroll
            for (int i = 0; i < NP; ++i) {
              const int c = CPT * cgp + 2 * i;
              if (c < H) aggrow[c] = ldexpf(c2[i].x, -E);
              if (c + 1 < H) aggrow[c + 1] = ldexpf(c2[i].y, -E);
            }
          }
        }
        E += s + sw;
        first = false;
        float pm = 0.f;
        uint32_t p1[NP], p2[NP];
#pragma unroll
        for (int i = 0; i < NP; ++i) {
          const float2 x = __fmul2_rn(c2[i], ds[i]);
          pm = fmaxf(pm, fmaxf(fabsf(x.x), fabsf(x.y)));
          const float2 f1 = make_float2(__uint_as_float(__float_as_uint(x.x) & 0xFFFFE000u),
                                        __uint_as_float(__float_as_uint(x.y) & 0xFFFFE000u));
          const float2 r = __fadd2_rn(x, make_float2(-f1.x, -f1.y));
          p1[i] = h2_bits(__floats2half2_rn(f1.x, f1.y));
          p2[i] = h2_bits(__floats2half2_rn(r.x, r.y));
        }
        const uint32_t redp = red0 + par * (TM * 16);
        asm volatile("st.shared.u32 [%0], %1;\n" ::"r"(redp + 4u * cgp), "r"(__float_as_uint(pm)) : "memory");
#pragma unroll
        for (int h8 = 0; h8 < NP / 8; ++h8) {
          tmem_st8(t_a1 + 8 * h8, *reinterpret_cast<const uint32_t(*)[8]>(p1 + 8 * h8));
          tmem_st8(t_a2 + 8 * h8, *reinterpret_cast<const uint32_t(*)[8]>(p2 + 8 * h8));
        }
        asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
        tc_fence_before();
        named_bar(3 + g, EPI);
        if (issuer) {
          tc_fence_after();
          mma12_f16_commit_n64(slot_base, bdesc, bw2, su32(&d_full[g]));
        }
        uint32_t m2[2];
        asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];\n" : "=r"(m2[0]), "=r"(m2[1]) : "r"(redp) : "memory");
        bound = __uint_as_float(max(m2[0], m2[1]));
        par ^= 1;
      }
    }
    if (!first) {                                   // D of the tile's last step
      if (issuer) {
        if (lane == 0) mbar_wait(&d_full[g], ph);
        __syncwarp();
      }
      named_bar(5 + g, EPI);
      ph ^= 1;
      tc_fence_after();
      load_d_one<CPT>(t_d1, c2);
      if (ok && len == nsteps && len > 0) {
#pragma unroll
        for (int i = 0; i < NP; ++i) {
          const int c = CPT * cgp + 2 * i;
          if (c < H) aggrow[c] = ldexpf(c2[i].x, -E);
          if (c + 1 < H) aggrow[c + 1] = ldexpf(c2[i].y, -E);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

// Head block of level 1: slot 0 holds the column-major aggregate M of the
// head block's leaves (written by the fold above); replace it in place by the
// vector M . seed (the head aggregate of the scan: a[C-1]...a[1] a[0]
// with a[0] = the seed).  One CTA per sample; the matrix is read before the
// vector overwrites its first column.
__global__ void __launch_bounds__(TH) head_apply_kernel(float* __restrict__ lvl, long long bstride,
                                                        const float* __restrict__ seed, int H) {
  __shared__ float sd[TH];
  const int b = blockIdx.x, i = threadIdx.x;
  float* M = lvl + (long long)b * bstride;
  if (i < H) sd[i] = seed[(long long)b * H + i];
  __syncthreads();
  float v = 0.f;
  if (i < H)
    for (int j = 0; j < H; ++j) v = fmaf(M[(long long)j * H + i], sd[j], v);
  __syncthreads();
  if (i < H) M[i] = v;
}

// ---------------------------------------------------------------------------
// Level-0 DOWN-walk on kind::f16 (3xFP16, true-scale chains).
//
// A tile = G = floor(128 / B8) whole groups of B chains (one level-0 block q,
// all B samples; B8 = B rounded up to 8 rows), so the h rows a tile needs at
// one step are G contiguous runs h[t(q, st)][0..B)[0..64) of the time-major
// input: the elected issuer lane loads each run with TWO 2D TMA copies
// (column halves, box 32 x B, SWIZZLE_128B) into a 3-stage ring — 2G copies
// per step instead of one bulk copy per chain row, and the 128-byte swizzle
// makes the threads' column-slice reads conflict-free.  Chains stay in true
// fp32 scale (grad_h is written every step); only the MMA operand is scaled:
// x^ = (d o v) 2^s, D = x^ [W1|W2] 2^sw, v <- (D1 + D2) 2^-(s + sw), with s
// from the bound  max|x| <= max|v| <= G M 2^-(s_prev + sw)  (M = the exact row
// maximum of the previous x^, exchanged through shared memory and ordered by
// the step's A barrier), so x^ < 2^15.  8 epilogue warps per slot, thread =
// chain row x 32 columns (one column half), two slots in flight.
// ---------------------------------------------------------------------------
constexpr int W_NST = 3;                                    // ring stages
constexpr int W_STAGE = 2 * TM * 128;                       // [half][128 rows][128 B] = 32 KB
constexpr int W_OFF_RING = F_B_BYTES;                       // [slot][stage]
constexpr int W_OFF_RED = W_OFF_RING + NSLOT * W_NST * W_STAGE;   // [slot][parity][128 rows][2] u32
constexpr int W_OFF_XRED = W_OFF_RED + NSLOT * 2 * TM * 8;        // affine: the same, for max|v + e|
constexpr int W_OFF_BAR = W_OFF_XRED + NSLOT * 2 * TM * 8;
constexpr int W_SMEM_BYTES = W_OFF_BAR + 128 + 1024;
constexpr int W_WPS = 8, W_EPI = 32 * W_WPS, W_NT = 2 * W_EPI;


template <bool AFF>
__global__ void __launch_bounds__(W_NT, 1) tc_leaf_down_f16_kernel(LeafArgs a, const __grid_constant__ CUtensorMap h3,
                                                                     const __grid_constant__ CUtensorMap h5,
                                                                     const __grid_constant__ CUtensorMap g3,
                                                                     const __grid_constant__ CUtensorMap g5,
                                                                     int C, const float* __restrict__ carry,
                                                                     long long nblk, float* __restrict__ grad_h,
                                                                     float* __restrict__ grad_init, int G,
                                                                     const float* __restrict__ e_aff,
                                                                     float* __restrict__ vec_out,
                                                                     float* __restrict__ head_out,
                                                                     long long head_bstride) {
  extern __shared__ uint8_t smem_raw[];
  const bool vonly = AFF && vec_out != nullptr;   // affine vector part of each block (no grad_h stores)
  char* smem = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* d_full = reinterpret_cast<uint64_t*>(smem + W_OFF_BAR);
  uint64_t* h_full = d_full + NSLOT;                                    // [slot][stage]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(h_full + NSLOT * W_NST);
  uint32_t* wred = tmem_slot + 2;
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const int B = a.seg.B;
  const long long S = a.seg.S();

  if (threadIdx.x < 2) wred[threadIdx.x] = 0;
  for (int e = threadIdx.x; e < NSLOT * W_NST * W_STAGE / 16; e += W_NT)
    sts128(su32(smem + W_OFF_RING) + 16u * e, 0.f, 0.f, 0.f, 0.f);
  __syncthreads();
  int sw;
  float G_w;
  w_scale(a.W, wred, &sw, &G_w);
  const int eG = (int)(__float_as_uint(G_w) >> 23) - 126;          // G < 2^eG
  {
    const float wsc = __int_as_float((sw + 127) << 23);
    for (int e = threadIdx.x; e < TH * TH; e += W_NT) {
      const int n = e / TH, k = e % TH;             // B[n][k] = W[k][n] 2^sw: rows 0..63 W1, 64..127 W2
      const float w = __ldg(a.W + (long long)k * TH + n) * wsc;
      const __half w1 = __float2half_rn(w);
      *reinterpret_cast<__half*>(smem + sw16_off(n, k)) = w1;
      *reinterpret_cast<__half*>(smem + sw16_off(TH + n, k)) = __float2half_rn(w - __half2float(w1));
    }
  }
  if (warp == 0) {
    if (lane == 0) {
      for (int s = 0; s < NSLOT; ++s) {
        mbar_init(&d_full[s], 1);
        for (int k = 0; k < W_NST; ++k) mbar_init(&h_full[s * W_NST + k], 1);
      }
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&h3)) : "memory");
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&h5)) : "memory");
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&g3)) : "memory");
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&g5)) : "memory");
    }
    __syncwarp();
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);

  const int g = warp / W_WPS, wl = warp % W_WPS;
  const int row = (wl & 3) * 32 + lane;
  const int cgp = wl >> 2;                                // column half
  const bool issuer = wl == 0;
  const uint32_t slot_base = tmem + 256 * g;
  const uint32_t lane_base = slot_base + ((uint32_t)((wl & 3) * 32) << 16);
  const uint32_t t_d1 = lane_base + 32 * cgp;      // the 64-column accumulator
  const uint32_t t_a1 = lane_base + 128 + 16 * cgp, t_a2 = lane_base + 160 + 16 * cgp;
  const uint32_t ring = su32(smem + W_OFF_RING) + (uint32_t)(g * W_NST * W_STAGE);
  const uint32_t hrow_off = (uint32_t)(row * 256 + cgp * 128);          // this thread's row half in a stage
  const int swz = (2 * row + cgp) & 7;                                    // its 128-byte line's swizzle
  const uint32_t red0 = su32(smem + W_OFF_RED) + (uint32_t)((g * 2 * TM + row) * 8);
  const uint32_t xred0 = su32(smem + W_OFF_XRED) + (uint32_t)((g * 2 * TM + row) * 8);
  uint32_t xpar = 0;
  const uint32_t bb = __shfl_sync(0xffffffffu, su32(smem), 0);
  uint64_t bdesc[4];
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) bdesc[kk] = sdesc(bb + (uint32_t)(kk * 32));
  uint64_t bw2[4];                                 // the W2 rows (64..127) at every K step
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) bw2[kk] = sdesc(bb + 8192u + (uint32_t)(kk * 32));
  const uint32_t dbar = su32(&d_full[g]), hbar0 = su32(&h_full[g * W_NST]);
  uint32_t dph = 0, par = 0, gs = 0;                       // D phase; exchange parity; slot step counter
  // tile row = j B + b holds group r = G-1-j (block q = qb + r), sample b: the
  // 5D TMA box delivers the groups of one step in decreasing q order
  const int jrow = row / B, bsm = row % B, grp = G - 1 - jrow;
  // view of the time axis as (block c4, step c3): t = c4 C + c3 = Tm - q C - st
  const long long Tm = (long long)a.seg.T - 1 + a.seg.head;
  const int A_blk = (int)(Tm / C), R_off = (int)(Tm % C);
  // tiles: [0] = block 0 alone; [1 .. nfull] = G blocks each whose merged box
  // stays inside the view at every step (blocks 1 .. A-1); then the remaining
  // blocks two per tile (per-group copies: few TMA ops, so no slow tile)
  const long long nfull = A_blk > 1 ? (A_blk - 1) / G : 0;
  const long long rem0 = 1 + nfull * G;
  const long long ntiles = 1 + nfull + (nblk > rem0 ? (nblk - rem0 + 1) / 2 : 0);
#ifdef BPPSA_STEP_TRACE
  int tstep = 0;
#define WTRACE(ph)                                                                                  \
  if (blockIdx.x == 0 && lane == 0 && (wl == 0 || wl == 5) && tstep < 4096)                        \
    g_step_trace[g][wl == 5][ph][tstep] = clock64();
#else
#define WTRACE(ph)
#endif

  for (long long tau = 2 * (long long)blockIdx.x + g; tau < ntiles; tau += 2 * (long long)gridDim.x) {
    const bool merged = tau >= 1 && tau <= nfull;
    const long long qb = tau == 0 ? 0 : (merged ? 1 + (tau - 1) * G : rem0 + 2 * (tau - nfull - 1));
    const int ng = tau == 0 ? 1 : (merged ? G : (int)min(2LL, nblk - qb));   // groups in this tile
    const long long q = qb + grp;
    const bool valid = jrow < G && grp < ng;
    const bool head = a.seg.head && q == 0;
    const long long s_start = head ? 1 : q * C, s1 = min(q * C + C, S);
    const int len = valid ? (int)(s1 - s_start) : 0;
    const bool total = valid && grad_init != nullptr && s1 == S;
    float2 v[16];                                          // this thread's 32 columns of the chain (true scale)
    {
      const float* src = head ? a.seed + (long long)bsm * TH : carry + ((long long)bsm * nblk + q) * TH;
      const bool from_src = valid && (head || !vonly);     // a vector part starts from 0
#pragma unroll
      for (int k4 = 0; k4 < 8; ++k4) {
        const float4 f = from_src ? __ldg(reinterpret_cast<const float4*>(src + 32 * cgp) + k4)
                                  : make_float4(0.f, 0.f, 0.f, 0.f);
        v[2 * k4] = make_float2(f.x, f.y);
        v[2 * k4 + 1] = make_float2(f.z, f.w);
      }
    }
    // TMA traffic of one step.  Tiles without block 0: ONE 5D box {32, 2, B, 1,
    // G} for all groups (loads of h into the ring stage, stores of grad_h from
    // it; coordinates below 0 are out of range: zero-filled / skipped).  The
    // tile holding block 0 (its head slot shifts the time by one) issues one 3D
    // box {32, 2, B} per group, one group per lane.  Each thread overwrites the
    // h half-row it consumed with its v (the exclusive output).
    // (negative box coordinates fault, so a step whose box would leave the
    // view, and the tile holding block 0, go per group)
    long long my_ss = 0, my_len = 0;
    const bool my_on = lane < ng;
    if (my_on) {
      const long long qr = qb + lane;
      my_ss = (a.seg.head && qr == 0) ? 1 : qr * C;
      my_len = min(qr * C + C, S) - my_ss;
    }
    const uint32_t my_dst = (uint32_t)((G - 1 - lane) * B * 256);
    auto c5 = [&](int st, int& c3, int& c4) {
      c3 = R_off - st;
      c4 = A_blk - (int)(qb + G - 1);
      if (c3 < 0) { c3 += C; c4 -= 1; }
      return merged;                                        // (then c4 >= 0 at every step)
    };
    auto issue_loads = [&](int st, uint32_t gstep) {       // all lanes of the issuer warp
      const uint32_t stage = ring + (gstep % W_NST) * W_STAGE;
      const uint32_t bar = hbar0 + 8u * (gstep % W_NST);
      int c3, c4;
      if (c5(st, c3, c4)) {
        if (lane == 0) {
          mbar_arrive_tx(bar, 256u * (uint32_t)(B * G));
          asm volatile(
              "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, "
              "%6}], [%7];\n" ::"r"(stage),
              "l"(reinterpret_cast<uint64_t>(&h5)), "r"(0), "r"(0), "r"(0), "r"(c3), "r"(c4), "r"(bar)
              : "memory");
        }
      } else {
        uint32_t bytes = 0;
        for (int r = 0; r < ng; ++r) {
          const long long qr = qb + r;
          const long long ss = (a.seg.head && qr == 0) ? 1 : qr * C, se = min(qr * C + C, S);
          if (st < se - ss) bytes += 256u * (uint32_t)B;
        }
        if (lane == 0) mbar_arrive_tx(bar, bytes);
        if (my_on && st < my_len)
          asm volatile(
              "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
              "[%5];\n" ::"r"(stage + my_dst),
              "l"(reinterpret_cast<uint64_t>(&h3)), "r"(0), "r"(0), "r"(a.seg.time_of(my_ss + st) * B), "r"(bar)
              : "memory");
      }
    };
    auto issue_stores = [&](int st, uint32_t gstep) {
      const uint32_t stage = ring + (gstep % W_NST) * W_STAGE;
      int c3, c4;
      if (c5(st, c3, c4)) {
        if (lane == 0) {
          asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];\n" ::"l"(
                           reinterpret_cast<uint64_t>(&g5)),
                       "r"(0), "r"(0), "r"(0), "r"(c3), "r"(c4), "r"(stage)
                       : "memory");
        }
      } else if (my_on && st < my_len) {
        asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];\n" ::"l"(
                         reinterpret_cast<uint64_t>(&g3)),
                     "r"(0), "r"(0), "r"(a.seg.time_of(my_ss + st) * B), "r"(stage + my_dst)
                     : "memory");
      }
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
    };
    if (issuer) {
      // the stages about to be refilled were last stored from by these lanes
      asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
      issue_loads(0, gs);
      if (C > 1) issue_loads(1, gs + 1);
      __syncwarp();
    }
    // bound of step 0 from the exact row maximum of the carry (two threads per row)
    int s_cur;
    {
      float pm = 0.f;
#pragma unroll
      for (int i = 0; i < 16; ++i) pm = fmaxf(pm, fmaxf(fabsf(v[i].x), fabsf(v[i].y)));
      const uint32_t redp = red0 + par * (TM * 8);
      asm volatile("st.shared.u32 [%0], %1;\n" ::"r"(redp + 4u * cgp), "r"(__float_as_uint(pm)) : "memory");
      named_bar(3 + g, W_EPI);
      uint32_t m2[2];
      asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];\n" : "=r"(m2[0]), "=r"(m2[1]) : "r"(redp) : "memory");
      const int eM = (int)(max(m2[0], m2[1]) >> 23) - 127;
      s_cur = 14 - eM;                                      // max|x| <= max|v| < 2^(eM+1)
      s_cur = max(-127 - sw, min(126 - sw, s_cur));
      par ^= 1;
      named_bar(5 + g, W_EPI);                              // the exchange words may be reused
    }
    int s_prev = 0;
    // affine: e rows of the step's own time (t(s) - 1 = t(s+1): the step that
    // consumes J_t(s-1) adds e at the time of slot s)
    auto load_e = [&](long long slot, float2 (&ef)[16]) {
      const float* src = e_aff + ((long long)a.seg.time_of(slot) * B + bsm) * TH + 32 * cgp;
#pragma unroll
      for (int k4 = 0; k4 < 8; ++k4) {
        const float4 f = __ldg(reinterpret_cast<const float4*>(src) + k4);
        ef[2 * k4] = make_float2(f.x, f.y);
        ef[2 * k4 + 1] = make_float2(f.z, f.w);
      }
    };
    for (int st = 0; st < C; ++st, ++gs) {
      WTRACE(0);
      float2 ef[16];
      // (a vector part also takes its last element's e: slot s1, when it exists)
      const bool add_e = AFF && e_aff != nullptr && valid && st > 0 && (st < len || (vonly && st == len && s1 < S));
      if (add_e) load_e(s_start + st, ef);                 // in flight during the waits below
      if (issuer) {                                         // D of step st-1 and h of step st
        if (lane == 0) {
          if (st > 0) mbar_wait_s(dbar, dph);
          mbar_wait_s(hbar0 + 8u * (gs % W_NST), (gs / W_NST) & 1);
        }
        __syncwarp();
      }
      named_bar(5 + g, W_EPI);
      WTRACE(1);
      if (st > 0) {                                         // v_st = (D1 + D2) 2^-(s_prev + sw)
        dph ^= 1;
        tc_fence_after();
        float2 t[16];
        load_d_one<32>(t_d1, t);
        const float f = __int_as_float((127 - s_prev - sw) << 23);
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = __fmul2_rn(t[i], make_float2(f, f));
        if (total && !vonly && st == len) {                 // inclusive extra: J_0^T grad_h[0]
          float4* dst = reinterpret_cast<float4*>(grad_init + (long long)bsm * TH + 32 * cgp);
#pragma unroll
          for (int k4 = 0; k4 < 8; ++k4) dst[k4] = make_float4(v[2 * k4].x, v[2 * k4].y, v[2 * k4 + 1].x, v[2 * k4 + 1].y);
        }
        if (add_e) {
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = __fadd2_rn(v[i], ef[i]);
        }
        if (AFF && e_aff != nullptr) {
          // e is outside the step's bound G M 2^-(s+sw): the scale of x^ comes
          // from the exact row maximum of v + e instead (two threads per row)
          float pv = 0.f;
#pragma unroll
          for (int i = 0; i < 16; ++i) pv = fmaxf(pv, fmaxf(fabsf(v[i].x), fabsf(v[i].y)));
          const uint32_t xp = xred0 + xpar * (TM * 8);
          asm volatile("st.shared.u32 [%0], %1;\n" ::"r"(xp + 4u * cgp), "r"(__float_as_uint(pv)) : "memory");
          named_bar(7 + g, W_EPI);
          uint32_t m2[2];
          asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];\n" : "=r"(m2[0]), "=r"(m2[1]) : "r"(xp) : "memory");
          const int eMv = (int)(max(m2[0], m2[1]) >> 23) - 127;
          s_cur = max(-127 - sw, min(126 - sw, 14 - eMv));
          xpar ^= 1;
        }
        if (vonly && valid && st == len) {                  // the block's vector part (a short block)
          float* dst = vec_out + ((long long)bsm * nblk + q) * TH;
#pragma unroll
          for (int k4 = 0; k4 < 8; ++k4)
            reinterpret_cast<float4*>(dst + 32 * cgp)[k4] =
                make_float4(v[2 * k4].x, v[2 * k4].y, v[2 * k4 + 1].x, v[2 * k4 + 1].y);
          if (head && head_out != nullptr) {
#pragma unroll
            for (int k4 = 0; k4 < 8; ++k4)
              reinterpret_cast<float4*>(head_out + (long long)bsm * head_bstride + 32 * cgp)[k4] =
                  make_float4(v[2 * k4].x, v[2 * k4].y, v[2 * k4 + 1].x, v[2 * k4 + 1].y);
          }
        }
      }
      WTRACE(2);
      WTRACE(3);
      // x^ = (d o v) 2^s from the staged, swizzled h row; split into fp16 pairs
      const uint32_t stg = ring + (gs % W_NST) * W_STAGE + hrow_off;
      const float sc = __int_as_float((s_cur + 127) << 23);
      float pm = 0.f;
      uint32_t p1[16], p2[16];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const uint32_t hp = stg + (uint32_t)((c ^ swz) << 4);
        const float4 h4 = lds128(hp);
        sts128(hp, v[2 * c].x, v[2 * c].y, v[2 * c + 1].x, v[2 * c + 1].y);   // grad_h[t(s)] = v (exclusive)
        const float2 d0 = make_float2(fmaf(-h4.x, h4.x, 1.f), fmaf(-h4.y, h4.y, 1.f));
        const float2 d1 = make_float2(fmaf(-h4.z, h4.z, 1.f), fmaf(-h4.w, h4.w, 1.f));
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const float2 x = __fmul2_rn(__fmul2_rn(u ? d1 : d0, v[2 * c + u]), make_float2(sc, sc));
          pm = fmaxf(pm, fmaxf(fabsf(x.x), fabsf(x.y)));
          const float2 f1 = make_float2(__uint_as_float(__float_as_uint(x.x) & 0xFFFFE000u),
                                        __uint_as_float(__float_as_uint(x.y) & 0xFFFFE000u));
          const float2 r = __fadd2_rn(x, make_float2(-f1.x, -f1.y));
          p1[2 * c + u] = h2_bits(__floats2half2_rn(f1.x, f1.y));
          p2[2 * c + u] = h2_bits(__floats2half2_rn(r.x, r.y));
        }
      }
      fence_async_smem();                                   // grad_h rows -> visible to the TMA store
      const uint32_t redp = red0 + par * (TM * 8);
      asm volatile("st.shared.u32 [%0], %1;\n" ::"r"(redp + 4u * cgp), "r"(__float_as_uint(pm)) : "memory");
#pragma unroll
      for (int h8 = 0; h8 < 2; ++h8) {
        tmem_st8(t_a1 + 8 * h8, *reinterpret_cast<const uint32_t(*)[8]>(p1 + 8 * h8));
        tmem_st8(t_a2 + 8 * h8, *reinterpret_cast<const uint32_t(*)[8]>(p2 + 8 * h8));
      }
      asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
      tc_fence_before();
      WTRACE(4);
      named_bar(3 + g, W_EPI);                              // A stored, row maxima written, stage consumed
      WTRACE(5);
      if (issuer) {
        tc_fence_after();
        mma12_f16_commit_n64(slot_base, bdesc, bw2, dbar);
        if (!vonly) issue_stores(st, gs);
        else asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
        if (st + 2 < C) {
          // stage (gs+2) % 3 was stored from at step st-1: its reads must be done
          asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
          issue_loads(st + 2, gs + 2);
        }
        __syncwarp();
      }
      uint32_t m2[2];
      asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];\n" : "=r"(m2[0]), "=r"(m2[1]) : "r"(redp) : "memory");
      const int eM = (int)(max(m2[0], m2[1]) >> 23) - 127;
      s_prev = s_cur;
      s_cur = max(-127 - sw, min(126 - sw, 14 - eG - eM + s_cur + sw));
      par ^= 1;
      WTRACE(6);
#ifdef BPPSA_STEP_TRACE
      ++tstep;
#endif
    }
    // D of the last step (keeps the barrier phase; grad_init if the chain ends here)
    if (issuer) {
      if (lane == 0) mbar_wait_s(dbar, dph);
      __syncwarp();
    }
    named_bar(5 + g, W_EPI);
    dph ^= 1;
    tc_fence_after();
    {
      float2 t[16];
      load_d_one<32>(t_d1, t);
      if ((total || vonly) && valid && len == C) {
        const float f = __int_as_float((127 - s_prev - sw) << 23);
        float2 ef[16];
        const bool add_e = AFF && vonly && e_aff != nullptr && s1 < S;   // the last element's e_{t-1}
        if (add_e) load_e(s1, ef);
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          t[i] = __fmul2_rn(t[i], make_float2(f, f));
          if (add_e) t[i] = __fadd2_rn(t[i], ef[i]);
        }
        float* dst = vonly ? vec_out + ((long long)bsm * nblk + q) * TH : grad_init + (long long)bsm * TH;
#pragma unroll
        for (int k4 = 0; k4 < 8; ++k4)
          reinterpret_cast<float4*>(dst + 32 * cgp)[k4] = make_float4(t[2 * k4].x, t[2 * k4].y, t[2 * k4 + 1].x, t[2 * k4 + 1].y);
        if (vonly && head && head_out != nullptr) {
#pragma unroll
          for (int k4 = 0; k4 < 8; ++k4)
            reinterpret_cast<float4*>(head_out + (long long)bsm * head_bstride + 32 * cgp)[k4] =
                make_float4(t[2 * k4].x, t[2 * k4].y, t[2 * k4 + 1].x, t[2 * k4 + 1].y);
        }
      }
    }
  }
  if (warp % W_WPS == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");   // grad_h stores done
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

}  // namespace

cudaError_t launch_head_apply(float* lvl, long long bstride, const float* seed, int B, int H, cudaStream_t st) {
  head_apply_kernel<<<B, TH, 0, st>>>(lvl, bstride, seed, H);
  return cudaGetLastError();
}

// Matrix blocks q in [q0, n_out) of an RNN H = 64 segment.  prec 0: 3xFP16
// row-scaled (tc_leaf_up_f16_kernel), 1: 3xTF32 (tc_leaf_up16_kernel).
cudaError_t launch_tc_leaf_up(const LeafArgs& a, int C, float* agg_out, long long n_out, long long q0,
                              int num_sms, cudaStream_t st, int prec) {
  const long long ntiles = (long long)((a.seg.B + 1) / 2) * (n_out - q0);
  const long long pairs = (ntiles + 1) / 2;
  const int grid = (int)std::min<long long>(pairs, num_sms);
  if (grid <= 0) return cudaSuccess;
  if (a.seg.H != TH) {                             // 3xFP16, 16 <= H < 64: packed groups
    const long long ngroups = (long long)a.seg.B * (n_out - q0);
    const long long ntg = (ngroups + TM / a.seg.H - 1) / (TM / a.seg.H);
    const int gridg = (int)std::min<long long>((ntg + 1) / 2, num_sms);
    if (gridg <= 0) return cudaSuccess;
    cudaError_t e = smem_attr_once(reinterpret_cast<const void*>(tc_leaf_up_f16g_kernel), F_SMEM_BYTES);
    if (e != cudaSuccess) return e;
    tc_leaf_up_f16g_kernel<<<gridg, 512, F_SMEM_BYTES, st>>>(a, C, agg_out, n_out, q0);
    return cudaGetLastError();
  }
  if (prec == 0) {                                 // 3xFP16, 8 epilogue warps per slot
    cudaError_t e = smem_attr_once(reinterpret_cast<const void*>(tc_leaf_up_f16_kernel<FOLD_WPS>), F_SMEM_BYTES);
    if (e != cudaSuccess) return e;
    tc_leaf_up_f16_kernel<FOLD_WPS><<<grid, 64 * FOLD_WPS, F_SMEM_BYTES, st>>>(a, C, agg_out, n_out, q0);
    return cudaGetLastError();
  }
  cudaError_t e = smem_attr_once(reinterpret_cast<const void*>(tc_leaf_up16_kernel), SMEM_BYTES16);
  if (e != cudaSuccess) return e;
  tc_leaf_up16_kernel<<<grid, NTHREADS16, SMEM_BYTES16, st>>>(a, C, agg_out, n_out, q0);
  return cudaGetLastError();
}

// Tensor maps of the walk over a [T][B][64] fp32 array (h or grad_h), 128-byte
// swizzle: 3D {32, 2, T B} with box {32, 2, B} (one step of one level-0 block),
// or 5D {32, 2, B, C, A} (time t = c4 C + c3, t < A C) with box {32, 2, B, 1,
// G} (one step of G consecutive blocks).  The driver entry point is fetched
// through the runtime, so nothing links against libcuda.
cudaError_t make_walk_map(const float* base, int T, int B, int C, long long A, bool five, int G,
                          CUtensorMap* map) {
  using Encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static Encode encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn) return e != cudaSuccess ? e : cudaErrorNotSupported;
    encode = reinterpret_cast<Encode>(fn);
  }
  const cuuint64_t row = (cuuint64_t)TH * sizeof(float);
  const cuuint32_t estr[5] = {1u, 1u, 1u, 1u, 1u};
  CUresult r;
  if (!five) {
    const cuuint64_t dims[3] = {32, 2, (cuuint64_t)T * B};
    const cuuint64_t strides[2] = {128, row};
    const cuuint32_t box[3] = {32u, 2u, (cuuint32_t)B};
    r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    if (A < 1) A = 1;
    const cuuint64_t dims[5] = {32, 2, (cuuint64_t)B, (cuuint64_t)C, (cuuint64_t)A};
    const cuuint64_t strides[4] = {128, row, row * B, row * B * C};
    const cuuint32_t box[5] = {32u, 2u, (cuuint32_t)B, 1u, (cuuint32_t)G};
    r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, const_cast<float*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// Level-0 down-walk of an RNN H = 64 segment on the tensor cores: the 3xFP16
// walk with per-run TMA loads (B <= 128), else the 3xTF32 per-row walk.
cudaError_t launch_tc_leaf_down(const LeafArgs& a, int C, const float* carry, long long nblk, float* grad_h,
                                float* grad_init, int num_sms, cudaStream_t st, const float* e_aff, float* vec_out,
                                float* head_out, long long head_bstride) {
  if (e_aff != nullptr || vec_out != nullptr) {    // affine terms: the TMA walk only
    if (a.seg.B > TM) return cudaErrorNotSupported;
    if (grad_h == nullptr) grad_h = const_cast<float*>(a.h);   // vector parts store no grad_h (maps unused)
  }
  if (a.seg.B <= TM && (e_aff != nullptr || vec_out != nullptr || !std::getenv("BPPSA_WALK_TF32"))) {
    const int B = a.seg.B, G = TM / B;
    const long long Tm = (long long)a.seg.T - 1 + a.seg.head;
    CUtensorMap maps[4];
    cudaError_t e = cudaSuccess;
    for (int m = 0; m < 4 && e == cudaSuccess; ++m)
      e = make_walk_map(m < 2 ? a.h : grad_h, a.seg.T, B, C, Tm / C, m % 2 == 1, G, &maps[m]);
    if (e != cudaSuccess) return e;
    const long long A = Tm / C, nfull = A > 1 ? (A - 1) / G : 0, rem0 = 1 + nfull * G;
    const long long nt = 1 + nfull + (nblk > rem0 ? (nblk - rem0 + 1) / 2 : 0);
    const int gridw = (int)std::min<long long>((nt + 1) / 2, num_sms);
    const bool aff = e_aff != nullptr || vec_out != nullptr;
    auto kern = aff ? tc_leaf_down_f16_kernel<true> : tc_leaf_down_f16_kernel<false>;
    e = smem_attr_once(reinterpret_cast<const void*>(kern), W_SMEM_BYTES);
    if (e != cudaSuccess) return e;
    kern<<<gridw, W_NT, W_SMEM_BYTES, st>>>(a, maps[0], maps[1], maps[2], maps[3], C, carry, nblk,
                                           vec_out ? nullptr : grad_h, vec_out ? nullptr : grad_init, G, e_aff,
                                           vec_out, head_out, head_bstride);
    return cudaGetLastError();
  }
  const long long ntiles = ((long long)a.seg.B * nblk + TM - 1) / TM;
  const int grid = (int)std::min<long long>((ntiles + 1) / 2, num_sms);
  cudaError_t e = smem_attr_once(reinterpret_cast<const void*>(tc_leaf_down16_kernel), SMEM_BYTES_D16);
  if (e != cudaSuccess) return e;
  tc_leaf_down16_kernel<<<grid, NTHREADS16, SMEM_BYTES_D16, st>>>(a, C, carry, nblk, grad_h, grad_init);
  return cudaGetLastError();
}

}  // namespace bppsa
