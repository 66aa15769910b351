// tc_i8.cu — the level-0 up-sweep fold of the tanh-RNN leaves (H = 64) on the
// tcgen05 INTEGER tensor cores, with exact accumulation.
//
// The fold computes every level-0 block aggregate a[s1-1] ... a[s0] (Alg. 1's
// up-sweep products over one block) column by column: column j is a
// BP chain c <- J_t^T c = W^T (d_t o c) from e_j, d_t = 1 - h_t^2 (eqn:rnn,
// P:315; DESIGN reading 1).  All chains step with the same W, so one step of a
// tile of 128 chains is one dense contraction C'[128 x 64] = X[128 x 64] W.
//
// Why integers.  fp32-accurate products on the fp16/tf32 tensor cores need
// split operands AND fp32 accumulation, and the tcgen05 accumulator truncates:
// a one-signed bias of ~1.35 ulp per step that grows linearly along a chain
// (profiles/tc_precision.md).  kind::i8 accumulates in s32,
// EXACTLY.  So every operand is a fixed-point integer split into 8-bit digits:
//   x = y 2^-sigma,  X = rint(y 2^sigma) in [-2^23, 2^23)  (one rounding, RN:
//       per row, sigma puts max|X| in [2^22, 2^23): 23 bits + sign),
//       X = x0 2^16 + x1 2^8 + x2   (two's complement bytes: x0 s8, x1 x2 u8)
//   W = Wint 2^-tau,  |Wint| < 2^31 - 2^24 (one scale for the matrix, RN),
//       Wint = W0 2^24 + W1 2^16 + W2 2^8 + W3   (balanced s8 digits)
// and X Wint = 2^40 sum_{i,j} x_i W_j 2^-8(i+j).  The products with i + j <= 3
// are accumulated EXACTLY in four s32 regions R_r = sum_{i+j=r} x_i W_j (the
// dropped i + j >= 4 terms are < 2^-30 of the result), then combined once in
// fp32 round-to-nearest:  S = 256 R0 + R1, T = 256 R2 + R3 (exact s32),
//   c' = fma(float(T), 2^-16, float(S)) = 2^-32 X Wint (1 + O(2^-24)).
// Every rounding is round-to-nearest (unbiased); nothing truncates.  W keeps
// 31 bits (the systematic part of the error), X 23 bits + sign per row.
//
// MMA shape.  Region r lives at TMEM columns [64 r, 64 r + 64) of the slot's
// 256-column accumulator; B = [W0 | W1 | W2 | W3] (256 rows, K-major) and the
// digit products land in their regions by shifting the D address:
//   x0 [W0 W1 W2 W3] -> D + 0   (N = 256, initialises all four regions)
//   x1 [W0 W1 W2]    -> D + 64  (N = 192)
//   x2 [W0 W1]       -> D + 128 (N = 128)
// each over K = 64 in two K = 32 instructions: 6 MMAs per step and tile.  The
// two slots' accumulators fill TMEM (2 x 256 columns), so the x digits are
// staged in shared memory (the SS form; SWIZZLE_64B K-major tiles).
// Measured (scripts/tc_i8_probe.cu): an i8 MMA costs ~146 cycles (TS) / 167
// (SS, N <= 192) / 182 (SS, N = 256) whatever N, so a step is ~1030 cycles of
// tensor pipe.  The epilogue (4 s32 regions -> fp32 -> y -> row max -> 3
// digit bytes) is ~11 instructions per element and sets the pace: ~1500
// cycles per tile-step at C4, both the FMA and the ALU pipe ~60 % busy
// (ncu, profiles/r02_tc_fold_i8_ncu.md).  Rounding to the 24-bit X: some of
// the 4-column groups on the FMA pipe (rint24x2), the rest with cvt.rni on
// the XU pipe (I8_F2I_MASK; this two-slot kernel at C4: all-FMA 46.2 ms,
// all-XU 47.2, half 44.0 -- the pipes balance; the default ring kernel
// further below: 0xAA ~ 0xEE ~ 0xFF ~ 40 ms).  A single-FFMA magic-number rounding (X < 2^22 with a
// non-power-of-two row scale, 40.8 ms) was measured and rejected: 22-bit X
// doubled the norm-preserving error at T = 65536 (8.5e-5 vs 4.0e-5, worst
// block 1.05e-4 > the gate) and non-power-of-two scales break the integer
// families' bit-exactness (scripts/prec_ab.py, scripts/ozaki_sim2.py).
// MMA cost with precomputed descriptors (scripts/tc_i8_rate2.cu): M = 128,
// K = 32 i8: N = 64 78, N = 128 92, N = 256 156 cycles per MMA, so the six
// MMAs of a step are ~744 cycles of tensor pipe; the epilogue bounds.  This two-slot
// kernel is the fallback (-DBPPSA_FOLD_TWO_SLOT); the default is the ring
// kernel tc_fold_i8r_kernel below (4 tiles over 2 accumulators, 40 ms).
// Tried and slower: 16 epilogue warps
// alternating between the two slots of a 4-sample super-tile with a
// dedicated issuer warp (62 ms vs 46 ms at C4): one slot's epilogue then
// cannot overlap the other's; and each 8-warp group alternating the two
// 2-sample halves of a super-tile through its one accumulator, issuing the
// other half's MMAs right after converting D so that MMA latency hides
// behind the other half's epilogue (47.7 ms): the epilogue, not MMA latency,
// is the limit (ncu: issue 62 %, FMA and ALU pipes ~40 %, pipe-throttle and
// dependency stalls).
//
// Scale bookkeeping: a chain row is c 2^E (fp32 c, integer E).  With y = c o d
// and X = rint(y 2^sigma), the new row is c' 2^(E + 32 - sigma - tau).
// Tile, slots and staging follow tc_leaf.cu's 3xFP16 fold: a tile = the 64
// column chains of block q for samples b, b+1; two tiles in flight per CTA,
// 8 epilogue warps per slot (thread = chain row x 32 columns); the row max of
// y is exchanged between the row's two threads through shared memory.
#include <algorithm>
#include <cstdlib>

#include <cuda.h>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace bppsa {
namespace {
using namespace ptx;

constexpr int TH = 64;                              // hidden size
constexpr int TM = 128;                             // chains per tile (UMMA M)
constexpr int NSLOT = 2;                            // tiles in flight per CTA
constexpr int I8_HCH = 64;                          // steps of h staged per chunk
#ifndef I8_WPS_DEF
#define I8_WPS_DEF 8
#endif
constexpr int I8_WPS = I8_WPS_DEF, I8_EPI = 32 * I8_WPS, I8_NT = NSLOT * I8_EPI;
constexpr int I8_CPT = 256 / I8_WPS;                // accumulator columns per epilogue thread (32 or 64)
constexpr int I8_NCG = TH / I8_CPT;                 // threads per chain row (2: the row max is exchanged)
constexpr int I8_B_BYTES = 4 * TH * TH;             // [W0|W1|W2|W3]: 256 rows x 64 B
constexpr int I8_A_TILE = TM * TH;                  // one x-digit tile: 128 rows x 64 B
constexpr int I8_OFF_A = I8_B_BYTES;                // [slot][digit]
constexpr int I8_OFF_H = I8_OFF_A + NSLOT * 3 * I8_A_TILE;
constexpr int I8_H_BYTES = 2 * I8_HCH * TH * 4;     // a chunk: [2 samples][HCH][64] fp32
constexpr int I8_OFF_RED = I8_OFF_H + NSLOT * 2 * I8_H_BYTES;   // [slot][parity][128 rows][2] u32
constexpr int I8_OFF_BAR = I8_OFF_RED + NSLOT * 2 * TM * 8;
constexpr int I8_SMEM = I8_OFF_BAR + 64 + 1024;
constexpr uint32_t TMEM_COLS = 512;
#ifndef I8_F2I_MASK
#define I8_F2I_MASK 0xEE                            // groups of 4 columns rounded with cvt.rni (XU) instead of rint24x2
#endif

// K-major SWIZZLE_64B tile with 64-byte rows: the 16-byte chunk index is XORed
// with address bits [7, 9) = (row / 2) % 4 (8-row atoms of 512 B)
__device__ __forceinline__ uint32_t sw64(int row, int k) {
  return (uint32_t)(row * 64 + ((((k >> 4) ^ ((row >> 1) & 3))) << 4) + (k & 15));
}
__device__ __forceinline__ uint64_t sdesc64(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;            // LBO (unused: K fits one swizzle atom)
  d |= (uint64_t)(512 >> 4) << 32;   // SBO: 8-row groups
  d |= (uint64_t)1 << 46;            // descriptor version (sm_100)
  d |= (uint64_t)4 << 61;            // SWIZZLE_64B
  return d;
}
// D s32, B s8, A s8 (asg = 1) or u8 (0), both K-major, M = 128
constexpr uint32_t idesc_i8(int N, int asg) {
  return (2u << 4) | ((uint32_t)asg << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(TM >> 4) << 24);
}

// exponent of a positive finite float (denormals included)
__device__ __forceinline__ int ilogb_pos(float m) {
  const uint32_t b = __float_as_uint(m);
  return (b >> 23) ? (int)(b >> 23) - 127 : -118 - (int)__clz(b);
}
// sigma with max|y| 2^sigma in [2^22, 2^23 - 1]: rint never reaches 2^23
__device__ __forceinline__ int row_sigma(float M) {
  int s = 22 - ilogb_pos(M);
  if ((__float_as_uint(M) & 0x7FFFFFu) == 0x7FFFFFu) s -= 1;
  return min(s, 126);
}
__device__ __forceinline__ float pow2f(int e) { return __int_as_float((e + 127) << 23); }   // e in [-126, 127]
// X = rint(y 2^sigma) as a 24-bit two's complement integer, on the FMA pipe
// (cvt.rni is an XU instruction at a quarter of the rate; measured 34 % XU):
//   F_hi = fma.rm(y, 2^(sigma-8), M) = M + floor(v / 256)          (M = 1.5 2^23, v = y 2^sigma)
//   r    = fma(y, 2^sigma, 256 M - 256 F_hi) = v - 256 floor(v / 256)  in [0, 256), exact
//   F_lo = r + 2^23 (RN)             = 2^23 + rint(r)               (rint(r) in [0, 256])
//   (bits(F_hi) << 8) + bits(F_lo) = 0x8B000000 + X  (mod 2^32)
// since 256 bits(M) = 0 mod 2^24 and bits(2^23) = 0x4B000000: its low three
// bytes are X's (the carry of rint(r) = 256 included).
__device__ __forceinline__ float2 ffma2_rm(float2 a, float2 b, float2 c) {
  unsigned long long r;
  asm("fma.rm.f32x2 %0, %1, %2, %3;"
      : "=l"(r)
      : "l"(*reinterpret_cast<const unsigned long long*>(&a)), "l"(*reinterpret_cast<const unsigned long long*>(&b)),
        "l"(*reinterpret_cast<const unsigned long long*>(&c)));
  return *reinterpret_cast<float2*>(&r);
}
// two elements at a time on the paired fp32 pipe (FFMA2 / FADD2)
__device__ __forceinline__ void rint24x2(float2 y, float2 scl, float2 scl8, uint32_t& X0, uint32_t& X1) {
  const float2 fh = ffma2_rm(y, scl8, make_float2(12582912.f, 12582912.f));
  const float2 a = __ffma2_rn(fh, make_float2(-256.f, -256.f), make_float2(3221225472.f, 3221225472.f));
  const float2 r = __ffma2_rn(y, scl, a);
  const float2 fl = __fadd2_rn(r, make_float2(8388608.f, 8388608.f));
  X0 = (__float_as_uint(fh.x) << 8) + __float_as_uint(fl.x);
  X1 = (__float_as_uint(fh.y) << 8) + __float_as_uint(fl.y);
}

// W digits into the B tile (all threads).  tau: max|W| 2^tau in [2^30, 2^31 -
// 2^24), so the balanced top digit stays in [-127, 127]; red[0] a zeroed word.
__device__ void w_digits(const float* __restrict__ W, char* smem, uint32_t* red, int* tau_out) {
  uint32_t m = 0;
  for (int e = threadIdx.x; e < TH * TH; e += blockDim.x) m = max(m, __float_as_uint(fabsf(__ldg(W + e))));
  m = __reduce_max_sync(0xffffffffu, m);
  if ((threadIdx.x & 31) == 0) atomicMax(red, m);
  __syncthreads();
  const float mx = __uint_as_float(red[0]);
  int tau = 0;
  if (mx > 0.f) {
    tau = 30 - ilogb_pos(mx);
    if ((double)mx * ldexp(1.0, tau) >= 2147483648.0 - 16777216.0) tau -= 1;
  }
  const double sc = ldexp(1.0, tau);
  for (int e = threadIdx.x; e < TH * TH; e += blockDim.x) {
    const int n = e / TH, k = e % TH;               // B[n][k] = digit of W[k][n]
    long long wi = llrint((double)__ldg(W + (long long)k * TH + n) * sc);
    int dg[4];
#pragma unroll
    for (int r = 3; r >= 1; --r) {
      dg[r] = (int)(((wi + 128) & 255) - 128);
      wi = (wi - dg[r]) >> 8;
    }
    dg[0] = (int)wi;
#pragma unroll
    for (int r = 0; r < 4; ++r) smem[sw64(r * TH + n, k)] = (char)dg[r];
  }
  *tau_out = tau;
}

// The step's 6 MMAs (x0, x1, x2 digits against the shifted B windows, K = 64
// in two halves) and their commit, as one elected instruction stream.
__device__ __forceinline__ void mma6_i8_commit(uint32_t d, const uint64_t (&ad)[6], const uint64_t (&bd)[2],
                                               uint32_t bar) {
  asm volatile(
      "{\n"
      " .reg .pred e, f, t;\n"
      " .reg .b32 a;\n"
      " setp.ne.b32 f, 0, 0;\n"
      " setp.eq.b32 t, 0, 0;\n"
      " elect.sync _|e, 0xffffffff;\n"
      " @e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %7, %9, f;\n"
      " @e tcgen05.mma.cta_group::1.kind::i8 [%0], %2, %8, %9, t;\n"
      " add.u32 a, %0, 64;\n"
      " @e tcgen05.mma.cta_group::1.kind::i8 [a], %3, %7, %10, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::i8 [a], %4, %8, %10, t;\n"
      " add.u32 a, %0, 128;\n"
      " @e tcgen05.mma.cta_group::1.kind::i8 [a], %5, %7, %11, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::i8 [a], %6, %8, %11, t;\n"
      " @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%12];\n"
      "}\n" ::"r"(d),
      "l"(ad[0]), "l"(ad[1]), "l"(ad[2]), "l"(ad[3]), "l"(ad[4]), "l"(ad[5]), "l"(bd[0]), "l"(bd[1]),
      "r"(idesc_i8(256, 1)), "r"(idesc_i8(192, 0)), "r"(idesc_i8(128, 0)), "r"(bar)
      : "memory");
}

// c' for 8 columns of this thread from the four s32 regions (TMEM columns
// t0 + 64 r), combined once in fp32 RN
__device__ __forceinline__ void regions_to_c(uint32_t t0, float2 (&c)[4]) {
  uint32_t r0[8], r1[8], r2[8], r3[8];
  tmem_ld8(t0, r0);
  tmem_ld8(t0 + 64, r1);
  tmem_ld8(t0 + 128, r2);
  tmem_ld8(t0 + 192, r3);
  tmem_wait_ld();
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int S0 = (int)r0[2 * i] * 256 + (int)r1[2 * i], S1 = (int)r0[2 * i + 1] * 256 + (int)r1[2 * i + 1];
    const int T0 = (int)r2[2 * i] * 256 + (int)r3[2 * i], T1 = (int)r2[2 * i + 1] * 256 + (int)r3[2 * i + 1];
    c[i] = __ffma2_rn(make_float2(__int2float_rn(T0), __int2float_rn(T1)), make_float2(0x1p-16f, 0x1p-16f),
                      make_float2(__int2float_rn(S0), __int2float_rn(S1)));
  }
}
// c' for 16 columns from the four regions (one x16 load per region)
__device__ __forceinline__ void regions_to_c16(uint32_t t0, float2 (&c)[8]) {
  uint32_t r0[16], r1[16], r2[16], r3[16];
  tmem_ld16(t0, r0);
  tmem_ld16(t0 + 64, r1);
  tmem_ld16(t0 + 128, r2);
  tmem_ld16(t0 + 192, r3);
  tmem_wait_ld();
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int S0 = (int)r0[2 * i] * 256 + (int)r1[2 * i], S1 = (int)r0[2 * i + 1] * 256 + (int)r1[2 * i + 1];
    const int T0 = (int)r2[2 * i] * 256 + (int)r3[2 * i], T1 = (int)r2[2 * i + 1] * 256 + (int)r3[2 * i + 1];
    c[i] = __ffma2_rn(make_float2(__int2float_rn(T0), __int2float_rn(T1)), make_float2(0x1p-16f, 0x1p-16f),
                      make_float2(__int2float_rn(S0), __int2float_rn(S1)));
  }
}
// Four regions x 8 columns (t0 + 64 r + [0, 8)) into r[8 r + i], asynchronously:
// the registers are written when tcgen05.wait::ld retires, so every wait is
// followed by ld_retired(), an empty asm that "modifies" the registers the
// wait completed -- no use of them can be scheduled above the wait.
__device__ __forceinline__ void ld_regions8(uint32_t t0, uint32_t (&r)[32]) {
  // one asm statement, one base register with immediate offsets: one R2UR per
  // chunk instead of one per region (separate statements made four)
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%32];\n"
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%8,%9,%10,%11,%12,%13,%14,%15}, [%32+64];\n"
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%16,%17,%18,%19,%20,%21,%22,%23}, [%32+128];\n"
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%24,%25,%26,%27,%28,%29,%30,%31}, [%32+192];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(t0));
}
__device__ __forceinline__ void ld_retired(uint32_t (&r)[32]) {
#pragma unroll
  for (int g = 0; g < 4; ++g)
    asm volatile(""
                 : "+r"(r[8 * g]), "+r"(r[8 * g + 1]), "+r"(r[8 * g + 2]), "+r"(r[8 * g + 3]), "+r"(r[8 * g + 4]),
                   "+r"(r[8 * g + 5]), "+r"(r[8 * g + 6]), "+r"(r[8 * g + 7])
                 :
                 : "memory");
}
// y = c' o d for 8 columns from the loaded regions (d: two float4 in shared memory)
__device__ __forceinline__ void regions8_to_y(const uint32_t (&r)[32], float4 da, float4 db, float2* y) {
  float2 c[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int S0 = (int)r[2 * i] * 256 + (int)r[8 + 2 * i], S1 = (int)r[2 * i + 1] * 256 + (int)r[8 + 2 * i + 1];
    const int T0 = (int)r[16 + 2 * i] * 256 + (int)r[24 + 2 * i], T1 = (int)r[16 + 2 * i + 1] * 256 + (int)r[24 + 2 * i + 1];
    c[i] = __ffma2_rn(make_float2(__int2float_rn(T0), __int2float_rn(T1)), make_float2(0x1p-16f, 0x1p-16f),
                      make_float2(__int2float_rn(S0), __int2float_rn(S1)));
  }
  y[0] = __fmul2_rn(c[0], make_float2(da.x, da.y));
  y[1] = __fmul2_rn(c[1], make_float2(da.z, da.w));
  y[2] = __fmul2_rn(c[2], make_float2(db.x, db.y));
  y[3] = __fmul2_rn(c[3], make_float2(db.z, db.w));
}

#ifdef BPPSA_F8_TRACE
// dev aid: clock64 per fold step on CTA 0, each slot's issuer lane: [slot * 8 + event][step]
__device__ long long g_f8_trace[16][4096];
#define F8T(ev, i) \
  if (blockIdx.x == 0 && issuer && lane == 0 && (i) < 4096) g_f8_trace[g * 8 + (ev)][i] = clock64();
// the ring fold: [group * 8 + event][step of the group] on CTA 0, each group's warp 0 lane 0
__device__ long long g_r8_trace[32][4096];
#define R8T(ev, i) \
  if (blockIdx.x == 0 && wl == 0 && lane == 0 && (i) < 4096) g_r8_trace[g * 8 + (ev)][i] = clock64();
#define R8V(ev, i, val) \
  if (blockIdx.x == 0 && wl == 0 && lane == 0 && (i) < 4096) g_r8_trace[g * 8 + (ev)][i] = (val);
#else
#define F8T(ev, i)
#define R8T(ev, i)
#define R8V(ev, i, val)
#endif
#ifdef BPPSA_I8_TRACE
// dev aid: clock64 per step on CTA 0 (warp 0, lane 0): [event][step]
__device__ long long g_i8_trace[12][2048];
#define I8T(ev, i) \
  if (blockIdx.x == 0 && lane == 0 && (i) < 2048) g_i8_trace[ev][i] = clock64();
#else
#define I8T(ev, i)
#endif

__global__ void __launch_bounds__(I8_NT, 1) tc_fold_i8_kernel(LeafArgs a, int C, float* __restrict__ agg_out,
                                                            long long n_out, long long q0) {
  extern __shared__ uint8_t smem_raw[];
  char* smem = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* d_full = reinterpret_cast<uint64_t*>(smem + I8_OFF_BAR);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(d_full + NSLOT);
  uint32_t* wred = tmem_slot + 1;
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const int B = a.seg.B;
  const long long S = a.seg.S();
  const long long nq = n_out - q0;
  const int nbp = (B + 1) / 2;
  const long long ntiles = (long long)nbp * nq;

  if (threadIdx.x == 0) wred[0] = 0;
  __syncthreads();
  int tau;
  w_digits(a.W, smem, wred, &tau);
  if (warp == 0) {
    if (lane == 0) {
      for (int s = 0; s < NSLOT; ++s) mbar_init(su32(&d_full[s]), 1);
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

  const int g = warp / I8_WPS, wl = warp % I8_WPS;
  const int quad = wl & 3, row = quad * 32 + lane;
  const int cgp = wl >> 2;                          // column group: columns [CPT cgp, CPT cgp + CPT)
  const int et = wl * 32 + lane;
  const bool issuer = wl == 0;
  const uint32_t slot_base = tmem + 256 * g;
  const uint32_t t_mine = slot_base + ((uint32_t)(quad * 32) << 16) + I8_CPT * cgp;
  const uint32_t a_tiles = su32(smem + I8_OFF_A + g * 3 * I8_A_TILE);
  // this row's 16-byte chunks (k in [CPT cgp, CPT cgp + CPT)) of a digit tile
  uint32_t a_c[I8_CPT / 16];
#pragma unroll
  for (int c = 0; c < I8_CPT / 16; ++c)
    a_c[c] = a_tiles + (uint32_t)(row * 64 + ((((I8_CPT / 16) * cgp + c) ^ ((row >> 1) & 3)) << 4));
  char* const hsb0 = smem + I8_OFF_H + (2 * g) * I8_H_BYTES;
  auto hsb = [&](int c) { return reinterpret_cast<float*>(hsb0 + c * I8_H_BYTES); };
  const uint32_t red0 = su32(smem + I8_OFF_RED) + (uint32_t)(((g * 2) * TM + row) * 8);
  const uint32_t dbar = su32(&d_full[g]);
  const int pair_bar = 7 + 4 * g + quad;            // the row's two threads (warps wl, wl ^ 4)
  uint64_t ad[6], bd[2];
  {
    const uint32_t bb = __shfl_sync(0xffffffffu, su32(smem), 0);
    const uint32_t ab = __shfl_sync(0xffffffffu, a_tiles, 0);
#pragma unroll
    for (int dgt = 0; dgt < 3; ++dgt)
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) ad[2 * dgt + ks] = sdesc64(ab + (uint32_t)(dgt * I8_A_TILE + 32 * ks));
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) bd[ks] = sdesc64(bb + (uint32_t)(32 * ks));
  }
  uint32_t ph = 0, par = 0;
  int tstep = 0;
  const long long rowB = (long long)B * TH;
  // one chunk of tile tx from slot scx: I8_HCH steps of the h rows of its two
  // samples, asynchronous (one commit group)
  auto issue_chunk = [&](long long tx, long long scx, float* hb) {
    const long long qx = q0 + tx / nbp;
    const int bpx = (int)(tx % nbp);
    const int nx = (int)min((long long)I8_HCH, min(qx * C + (long long)C, S) - scx);
    for (int e = et; e < 2 * nx * 16; e += I8_EPI) {
      const int bb2 = e / (nx * 16), rem = e % (nx * 16), st = rem / 16, ch = rem % 16;
      const uint32_t dst = su32(hb + (bb2 * I8_HCH + st) * TH + ch * 4);
      const int bs = bpx * 2 + bb2;
      if (bs < B)
        cp_async16(dst, a.h + (long long)a.seg.time_of(scx + st) * rowB + (long long)bs * TH + ch * 4);
      else
        sts128(dst, 0.f, 0.f, 0.f, 0.f);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  auto tile_s0 = [&](long long tx) {
    const long long qx = q0 + tx / nbp;
    return (a.seg.head && qx == 0) ? 1LL : qx * C;
  };
  int cb = 0;
  {
    const long long t0 = 2 * (long long)blockIdx.x + g;
    if (t0 < ntiles) issue_chunk(t0, tile_s0(t0), hsb(0));
  }
  for (long long tau_t = 2 * (long long)blockIdx.x + g; tau_t < ntiles; tau_t += 2 * (long long)gridDim.x) {
    const long long q = q0 + tau_t / nbp;
    const int bp = (int)(tau_t % nbp);
    const int b = bp * 2 + (row >> 6);
    const int j = row & 63;
    const bool ok = b < B;
    // the head block (slot 0 = the seed) is folded as the matrix of its leaves,
    // slots 1..C-1; head_apply_kernel then applies it to the seed
    const long long s0 = (a.seg.head && q == 0) ? 1 : q * C, s1 = min(q * C + (long long)C, S);
    int E = 0;                                      // chain row = c 2^E
    bool first = true;
    for (long long sc = s0; sc < s1; sc += I8_HCH) {
      const int n = (int)min((long long)I8_HCH, s1 - sc);
      float* hs = hsb(cb);
      const uint32_t hs_s = su32(hs);
      asm volatile("cp.async.wait_all;\n" ::: "memory");
      named_bar(1 + g, I8_EPI);                     // copies landed; the previous chunk is consumed
      for (int e = et; e < 2 * n * 16; e += I8_EPI) {   // d = 1 - h^2 in place
        const int bb2 = e / (n * 16), rem = e % (n * 16), st = rem / 16, ch = rem % 16;
        const uint32_t p = hs_s + 4u * ((bb2 * I8_HCH + st) * TH + ch * 4);
        const float4 h4 = lds128(p);
        sts128(p, fmaf(-h4.x, h4.x, 1.f), fmaf(-h4.y, h4.y, 1.f), fmaf(-h4.z, h4.z, 1.f), fmaf(-h4.w, h4.w, 1.f));
      }
      named_bar(1 + g, I8_EPI);
      {                                             // prefetch the next chunk into the other buffer
        const long long tn = tau_t + 2 * (long long)gridDim.x;
        if (sc + I8_HCH < s1) issue_chunk(tau_t, sc + I8_HCH, hsb(cb ^ 1));
        else if (tn < ntiles) issue_chunk(tn, tile_s0(tn), hsb(cb ^ 1));
      }
      cb ^= 1;
      uint32_t dp = hs_s + 4u * ((row >> 6) * I8_HCH * TH + I8_CPT * cgp);   // this thread's d slice of step st
      for (int st = 0; st < n; ++st, dp += 4u * TH) {
        float2 y[I8_CPT / 2];                       // y = c o d_t (this thread's CPT columns)
        if (first) {
#pragma unroll
          for (int q4 = 0; q4 < I8_CPT / 4; ++q4) {
            const float4 d4 = lds128(dp + 16u * q4);
            const int k0 = I8_CPT * cgp + 4 * q4;
            y[2 * q4] = make_float2(k0 == j && ok ? d4.x : 0.f, k0 + 1 == j && ok ? d4.y : 0.f);
            y[2 * q4 + 1] = make_float2(k0 + 2 == j && ok ? d4.z : 0.f, k0 + 3 == j && ok ? d4.w : 0.f);
          }
        } else {
          F8T(0, tstep);
          if (issuer) {
            if (lane == 0) mbar_wait(dbar, ph);
            __syncwarp();
          }
          named_bar(5 + g, I8_EPI);
          F8T(1, tstep);
          ph ^= 1;
          tc_fence_after();
          {                                         // chunks of 8 columns, TMEM loads one chunk ahead
            uint32_t ra[32], rb[32];
            ld_regions8(t_mine, ra);
#pragma unroll
            for (int c8 = 0; c8 < I8_CPT / 8; c8 += 2) {
              tmem_wait_ld();
              ld_retired(ra);
              ld_regions8(t_mine + 8 * (c8 + 1), rb);
              regions8_to_y(ra, lds128(dp + 32u * c8), lds128(dp + 32u * c8 + 16u), y + 4 * c8);
              tmem_wait_ld();
              ld_retired(rb);
              if (c8 + 2 < I8_CPT / 8) ld_regions8(t_mine + 8 * (c8 + 2), ra);
              regions8_to_y(rb, lds128(dp + 32u * (c8 + 1)), lds128(dp + 32u * (c8 + 1) + 16u), y + 4 * (c8 + 1));
            }
          }
        }
        first = false;
        F8T(2, tstep);
        float pm = 0.f;
#pragma unroll
        for (int i = 0; i < I8_CPT / 2; ++i) pm = fmaxf(pm, fmaxf(fabsf(y[i].x), fabsf(y[i].y)));
        float M = pm;
        if (I8_NCG == 2) {                          // the row's other half: exchanged through shared memory
          const uint32_t redp = red0 + par * (TM * 8);
          asm volatile("st.shared.u32 [%0], %1;\n" ::"r"(redp + 4u * cgp), "r"(__float_as_uint(pm)) : "memory");
          named_bar(pair_bar, 64);
          uint32_t m2[2];
          asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];\n" : "=r"(m2[0]), "=r"(m2[1]) : "r"(redp) : "memory");
          par ^= 1;
          M = __uint_as_float(max(m2[0], m2[1]));
        }
        F8T(3, tstep);
        const int sig = M > 0.f ? row_sigma(M) : 0;
        const float2 scl = make_float2(pow2f(sig), pow2f(sig)), scl8 = make_float2(pow2f(sig - 8), pow2f(sig - 8));
        if (M > 0.f) E += 32 - sig - tau;
        // X = rint(y 2^sigma) in [-2^23, 2^23): bytes 2, 1, 0 = digits x0 (s8), x1, x2 (u8);
        // words of 4 consecutive k per digit (7 byte permutes per 4 elements), 16 k per store
#pragma unroll
        for (int c16 = 0; c16 < I8_CPT / 16; ++c16) {
          uint32_t w0[4], w1[4], w2[4];
#pragma unroll
          for (int uu = 0; uu < 4; ++uu) {
            const int u = 4 * c16 + uu;
            uint32_t X0, X1, X2, X3;
            if ((I8_F2I_MASK >> (u & 7)) & 1) {     // this group rounds on the XU pipe (cvt.rni)
              const float2 v0 = __fmul2_rn(y[2 * u], scl), v1 = __fmul2_rn(y[2 * u + 1], scl);
              X0 = (uint32_t)__float2int_rn(v0.x), X1 = (uint32_t)__float2int_rn(v0.y);
              X2 = (uint32_t)__float2int_rn(v1.x), X3 = (uint32_t)__float2int_rn(v1.y);
            } else {
              rint24x2(y[2 * u], scl, scl8, X0, X1);
              rint24x2(y[2 * u + 1], scl, scl8, X2, X3);
            }
            const uint32_t p01 = prmt(X0, X1, 0x5140u), p23 = prmt(X2, X3, 0x5140u);
            const uint32_t q01 = prmt(X0, X1, 0x0062u), q23 = prmt(X2, X3, 0x0062u);
            w2[uu] = prmt(p01, p23, 0x5410u);
            w1[uu] = prmt(p01, p23, 0x7632u);
            w0[uu] = prmt(q01, q23, 0x5410u);
          }
          sts128u(a_c[c16], w0[0], w0[1], w0[2], w0[3]);
          sts128u(a_c[c16] + I8_A_TILE, w1[0], w1[1], w1[2], w1[3]);
          sts128u(a_c[c16] + 2 * I8_A_TILE, w2[0], w2[1], w2[2], w2[3]);
        }
        F8T(4, tstep);
        fence_async_smem();                         // the digits -> visible to the tensor core
        tc_fence_before();
        F8T(5, tstep);
        named_bar(3 + g, I8_EPI);                   // the slot's three digit tiles are complete
        F8T(6, tstep);
        if (issuer) {
          tc_fence_after();
          mma6_i8_commit(slot_base, ad, bd, dbar);
        }
        F8T(7, tstep);
        ++tstep;
      }
    }
    float2 cfin[I8_CPT / 2];
    if (!first) {                                   // D of the tile's last step
      if (issuer) {
        if (lane == 0) mbar_wait(dbar, ph);
        __syncwarp();
      }
      named_bar(5 + g, I8_EPI);
      ph ^= 1;
      tc_fence_after();
#pragma unroll
      for (int qq = 0; qq < I8_CPT / 8; ++qq) {
        float2 c[4];
        regions_to_c(t_mine + 8 * qq, c);
#pragma unroll
        for (int i = 0; i < 4; ++i) cfin[4 * qq + i] = c[i];
      }
    } else {                                        // an empty head block: the identity
#pragma unroll
      for (int k = 0; k < I8_CPT / 2; ++k)
        cfin[k] = make_float2(I8_CPT * cgp + 2 * k == j ? 1.f : 0.f, I8_CPT * cgp + 2 * k + 1 == j ? 1.f : 0.f);
    }
    if (ok) {
      float4* dst = reinterpret_cast<float4*>(agg_out + (((long long)b * n_out + q) * TH + j) * TH + I8_CPT * cgp);
#pragma unroll
      for (int k4 = 0; k4 < I8_CPT / 4; ++k4)
        dst[k4] = make_float4(ldexpf(cfin[2 * k4].x, E), ldexpf(cfin[2 * k4].y, E), ldexpf(cfin[2 * k4 + 1].x, E),
                              ldexpf(cfin[2 * k4 + 1].y, E));
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
// The same fold with FOUR tiles in flight over TWO accumulators (the "ring").
// In the two-slot kernel above a slot holds its 256 accumulator columns from
// the MMA issue until its epilogue has read them AND produced the next digits,
// so the tensor pipe idles whenever an epilogue (~2000 cycles) outlasts the
// other slot's MMAs (~920): 40 % tensor-pipe activity (ncu).  Here a tile group
// releases its accumulator as soon as the regions are converted to y (fp32 in
// registers), and the two accumulators are handed out by TICKETS: when a
// group's digits are complete, its first warp takes ticket it = atomicAdd(
// &ticket, 1) and uses accumulator it % 2 once the holder of ticket it - 2 has
// released it (rel[it % 2] >= 4 (it / 2): a monotonic release count per
// accumulator; an mbarrier phase parity would alias once three tickets are
// outstanding on one accumulator), so a ready group never waits
// behind a slower one (a strict round robin did: 44.5 ms at C4 with three
// groups and an issuer warp).  Warp 0 takes the ticket when its own digits
// are stored and publishes it % 2 in bufsel (by round parity) before the
// group's digit barrier, so the group's warps know their accumulator (polling
// two commit barriers instead spent 17 % of the warp samples in the spin
// loop).  mbarrier / release-count synchronisation between groups; a group = 4 warps, thread = chain row x 64
// columns (no row-max exchange).  4 groups = 512 threads (128 registers).
// ---------------------------------------------------------------------------
#ifndef R_NT_DEF
#define R_NT_DEF 4
#endif
constexpr int R_NT = R_NT_DEF;                      // tile groups
#ifndef R_PIPE_DEF
#define R_PIPE_DEF 1
#endif
constexpr bool R_PIPE = R_PIPE_DEF;
#ifndef R_X16_DEF
#define R_X16_DEF 1
#endif
constexpr bool R_X16 = R_X16_DEF;
#ifndef R_LATE_D_DEF
#define R_LATE_D_DEF 1
#endif
constexpr bool R_LATE_D = R_LATE_D_DEF;             // y = c o d after the accumulator release (38.3 vs 38.8 ms)
constexpr int R_WPS = 4, R_EPI = 32 * R_WPS;        // warps per group
constexpr int R_THREADS = R_NT * R_EPI;
#ifndef R_HCH_DEF
#define R_HCH_DEF 24
#endif
constexpr int R_HCH = R_HCH_DEF;                    // steps of h staged per chunk
constexpr int R_H_BYTES = 2 * R_HCH * TH * 4;
constexpr int R_OFF_A = I8_B_BYTES;                 // [group][digit] tiles
constexpr int R_OFF_H = R_OFF_A + R_NT * 3 * I8_A_TILE;
constexpr int R_OFF_BAR = R_OFF_H + R_NT * 2 * R_H_BYTES;
constexpr int R_SMEM = R_OFF_BAR + 256 + 1024;
static_assert(R_SMEM <= 232448, "ring fold shared memory");

// try_wait with a suspend-time hint: the waiting lane sleeps in the barrier
// unit instead of re-issuing the probe
__device__ __forceinline__ void mbar_wait_sleep(uint32_t bar, uint32_t parity) {
#ifndef R_NO_SLEEP
  asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n @!p bra W_%=;\n}\n" ::"r"(
                   bar), "r"(parity), "r"(1000000u) : "memory");
#else
  mbar_wait(bar, parity);
#endif
}

__global__ void __launch_bounds__(R_THREADS, 1) tc_fold_i8r_kernel(LeafArgs a, int C, float* __restrict__ agg_out,
                                                                 long long n_out, long long q0) {
  extern __shared__ uint8_t smem_raw[];
  char* smem = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + R_OFF_BAR);
  uint64_t* d_full = bars;                          // [R_NT]
  uint32_t* rel = reinterpret_cast<uint32_t*>(bars + R_NT);   // [2] warps that released each accumulator
  uint32_t* ticket = rel + 2;
  uint32_t* bufsel = ticket + 1;                    // [R_NT][2] accumulator of a group's batch (by round parity)
  uint32_t* tmem_slot = bufsel + 2 * R_NT;
  uint32_t* wred = tmem_slot + 1;
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const int B = a.seg.B;
  const long long S = a.seg.S();
  const long long nq = n_out - q0;
  const int nbp = (B + 1) / 2;
  const long long ntiles = (long long)nbp * nq;

  if (threadIdx.x == 0) wred[0] = 0;
  __syncthreads();
  int tau;
  w_digits(a.W, smem, wred, &tau);
  if (warp == 0) {
    if (lane == 0) {
      for (int i = 0; i < R_NT; ++i) mbar_init(su32(&d_full[i]), 1);
      rel[0] = rel[1] = 0;
      *ticket = 0;
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

  const int g = warp / R_WPS, wl = warp % R_WPS;    // tile group g: 4 warps, thread = row x 64 columns
  const int row = wl * 32 + lane;
  const int et = wl * 32 + lane;
  const uint32_t t_lane = (uint32_t)(wl * 32) << 16;
  const uint32_t a_tiles = su32(smem + R_OFF_A + g * 3 * I8_A_TILE);
  uint32_t a_c[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) a_c[c] = a_tiles + (uint32_t)(row * 64 + ((c ^ ((row >> 1) & 3)) << 4));
  uint64_t ad[6], bd[2];
  {
    const uint32_t bb = su32(smem);
#pragma unroll
    for (int dgt = 0; dgt < 3; ++dgt)
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) ad[2 * dgt + ks] = sdesc64(a_tiles + (uint32_t)(dgt * I8_A_TILE + 32 * ks));
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) bd[ks] = sdesc64(bb + (uint32_t)(32 * ks));
  }
  char* const hsb0 = smem + R_OFF_H + (2 * g) * R_H_BYTES;
  auto hsb = [&](int c) { return reinterpret_cast<float*>(hsb0 + c * R_H_BYTES); };
  const uint32_t dfull = su32(&d_full[g]);
  uint32_t kr = 0;                                  // this group's MMA rounds so far
  int cur = 0;
#ifdef BPPSA_F8_TRACE
  int nstep = 0;                                    // trace index
#endif                                      // the accumulator of the group's outstanding batch
  const long long rowB = (long long)B * TH;
  auto issue_chunk = [&](long long tx, long long scx, float* hb) {
    const long long qx = q0 + tx / nbp;
    const int bpx = (int)(tx % nbp);
    const int nx = (int)min((long long)R_HCH, min(qx * C + (long long)C, S) - scx);
    for (int e = et; e < 2 * nx * 16; e += R_EPI) {
      const int bb2 = e / (nx * 16), rem = e % (nx * 16), st = rem / 16, ch = rem % 16;
      const uint32_t dst = su32(hb + (bb2 * R_HCH + st) * TH + ch * 4);
      const int bs = bpx * 2 + bb2;
      if (bs < B)
        cp_async16(dst, a.h + (long long)a.seg.time_of(scx + st) * rowB + (long long)bs * TH + ch * 4);
      else
        sts128(dst, 0.f, 0.f, 0.f, 0.f);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  auto tile_s0 = [&](long long tx) {
    const long long qx = q0 + tx / nbp;
    return (a.seg.head && qx == 0) ? 1LL : qx * C;
  };
  // this warp's digits are stored: warp 0 takes the group's ticket (written to
  // bufsel by round parity), the group syncs, warp 0 issues once the
  // accumulator is released
  auto issue = [&]() {
    uint32_t it = 0;
    if (wl == 0) {
      if (lane == 0) {                              // shared-window atomics (a generic atomicAdd is an ATOM.E)
        asm volatile("atom.shared::cta.add.u32 %0, [%1], 1;\n" : "=r"(it) : "r"(su32(ticket)) : "memory");
        asm volatile("st.shared::cta.u32 [%0], %1;\n" ::"r"(su32(&bufsel[2 * g + (kr & 1)])), "r"(it & 1u) : "memory");
      }
      it = __shfl_sync(0xffffffffu, it, 0);
    }
    R8T(3, nstep);
    named_bar(1 + R_NT + g, R_EPI);
    R8T(4, nstep);
    R8V(6, nstep, (long long)it);
    {
      uint32_t cs;
      asm volatile("ld.shared::cta.u32 %0, [%1];\n" : "=r"(cs) : "r"(su32(&bufsel[2 * g + (kr & 1)])) : "memory");
      cur = (int)cs;
    }
    if (wl == 0) {
      if (lane == 0) {
        const uint32_t need = (it >> 1) * R_WPS, ra = su32(&rel[it & 1]);
        uint32_t v;
        while (true) {
          asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];\n" : "=r"(v) : "r"(ra) : "memory");
          if (v >= need) break;
          __nanosleep(20);
        }
      }
      __syncwarp();
      R8T(5, nstep);
      tc_fence_after();
      mma6_i8_commit(tmem + 256u * (uint32_t)cur, ad, bd, dfull);
    }
  };
  // wait for the group's outstanding batch; returns its TMEM base for this warp's lanes
  auto wait_d = [&]() {
    R8T(0, nstep);
    if (lane == 0) mbar_wait_sleep(dfull, kr & 1);
    __syncwarp();
    R8T(1, nstep);
    ++kr;
    tc_fence_after();
    return tmem + 256u * (uint32_t)cur + t_lane;
  };
  auto release_d = [&]() {
    tc_fence_before();
    __syncwarp();
    if (lane == 0) asm volatile("red.release.cta.shared::cta.add.u32 [%0], 1;\n" ::"r"(su32(&rel[cur])) : "memory");
    R8T(2, nstep);
  };
  int cb = 0;
  {
    const long long t0 = R_NT * (long long)blockIdx.x + g;
    if (t0 < ntiles) issue_chunk(t0, tile_s0(t0), hsb(0));
  }
  for (long long tau_t = R_NT * (long long)blockIdx.x + g; tau_t < ntiles; tau_t += R_NT * (long long)gridDim.x) {
    const long long q = q0 + tau_t / nbp;
    const int bp = (int)(tau_t % nbp);
    const int b = bp * 2 + (row >> 6);
    const int j = row & 63;
    const bool ok = b < B;
    const long long s0 = (a.seg.head && q == 0) ? 1 : q * C, s1 = min(q * C + (long long)C, S);
    int E = 0;                                      // chain row = c 2^E
    bool first = true;
    for (long long sc = s0; sc < s1; sc += R_HCH) {
      const int n = (int)min((long long)R_HCH, s1 - sc);
      float* hs = hsb(cb);
      const uint32_t hs_s = su32(hs);
      asm volatile("cp.async.wait_all;\n" ::: "memory");
      named_bar(1 + g, R_EPI);                      // copies landed; the previous chunk is consumed
      for (int e = et; e < 2 * n * 16; e += R_EPI) {   // d = 1 - h^2 in place
        const int bb2 = e / (n * 16), rem = e % (n * 16), st = rem / 16, ch = rem % 16;
        const uint32_t p = hs_s + 4u * ((bb2 * R_HCH + st) * TH + ch * 4);
        const float4 h4 = lds128(p);
        sts128(p, fmaf(-h4.x, h4.x, 1.f), fmaf(-h4.y, h4.y, 1.f), fmaf(-h4.z, h4.z, 1.f), fmaf(-h4.w, h4.w, 1.f));
      }
      named_bar(1 + g, R_EPI);
      {
        const long long tn = tau_t + R_NT * (long long)gridDim.x;
        if (sc + R_HCH < s1) issue_chunk(tau_t, sc + R_HCH, hsb(cb ^ 1));
        else if (tn < ntiles) issue_chunk(tn, tile_s0(tn), hsb(cb ^ 1));
      }
      cb ^= 1;
      uint32_t dp = hs_s + 4u * ((row >> 6) * R_HCH * TH);
      for (int st = 0; st < n; ++st, dp += 4u * TH) {
        float2 y[32];
        if (first) {
#pragma unroll
          for (int q4 = 0; q4 < 16; ++q4) {
            const float4 d4 = lds128(dp + 16u * q4);
            const int k0 = 4 * q4;
            y[2 * q4] = make_float2(k0 == j && ok ? d4.x : 0.f, k0 + 1 == j && ok ? d4.y : 0.f);
            y[2 * q4 + 1] = make_float2(k0 + 2 == j && ok ? d4.z : 0.f, k0 + 3 == j && ok ? d4.w : 0.f);
          }
        } else {
          const uint32_t td = wait_d();
          if (R_X16) {                              // x16 loads, one 16-column chunk at a time (64 registers)
#pragma unroll
            for (int c16 = 0; c16 < 4; ++c16) {
              if (R_LATE_D) {                       // c only: the accumulator is released sooner
                regions_to_c16(td + 16 * c16, *reinterpret_cast<float2(*)[8]>(y + 8 * c16));
                continue;
              }
              float2 c[8];
              regions_to_c16(td + 16 * c16, c);
#pragma unroll
              for (int h2 = 0; h2 < 2; ++h2) {
                const float4 da = lds128(dp + 64u * c16 + 32u * h2), db = lds128(dp + 64u * c16 + 32u * h2 + 16u);
                y[8 * c16 + 4 * h2] = __fmul2_rn(c[4 * h2], make_float2(da.x, da.y));
                y[8 * c16 + 4 * h2 + 1] = __fmul2_rn(c[4 * h2 + 1], make_float2(da.z, da.w));
                y[8 * c16 + 4 * h2 + 2] = __fmul2_rn(c[4 * h2 + 2], make_float2(db.x, db.y));
                y[8 * c16 + 4 * h2 + 3] = __fmul2_rn(c[4 * h2 + 3], make_float2(db.z, db.w));
              }
            }
          } else if (R_PIPE) {                      // TMEM loads one 8-column chunk ahead (64 registers)
            uint32_t ra[32], rb[32];
            ld_regions8(td, ra);
#pragma unroll
            for (int c8 = 0; c8 < 8; c8 += 2) {
              tmem_wait_ld();
              ld_retired(ra);
              ld_regions8(td + 8 * (c8 + 1), rb);
              regions8_to_y(ra, lds128(dp + 32u * c8), lds128(dp + 32u * c8 + 16u), y + 4 * c8);
              tmem_wait_ld();
              ld_retired(rb);
              if (c8 + 2 < 8) ld_regions8(td + 8 * (c8 + 2), ra);
              regions8_to_y(rb, lds128(dp + 32u * (c8 + 1)), lds128(dp + 32u * (c8 + 1) + 16u), y + 4 * (c8 + 1));
            }
          } else {
#pragma unroll
            for (int c8 = 0; c8 < 8; ++c8) {
              uint32_t ra[32];
              ld_regions8(td + 8 * c8, ra);
              tmem_wait_ld();
              ld_retired(ra);
              regions8_to_y(ra, lds128(dp + 32u * c8), lds128(dp + 32u * c8 + 16u), y + 4 * c8);
            }
          }
          release_d();
          if (R_X16 && R_LATE_D) {                  // y = c o d after the release
#pragma unroll
            for (int q4 = 0; q4 < 16; ++q4) {
              const float4 d4 = lds128(dp + 16u * q4);
              y[2 * q4] = __fmul2_rn(y[2 * q4], make_float2(d4.x, d4.y));
              y[2 * q4 + 1] = __fmul2_rn(y[2 * q4 + 1], make_float2(d4.z, d4.w));
            }
          }
        }
        first = false;
        float M = 0.f;
#pragma unroll
        for (int i = 0; i < 32; ++i) M = fmaxf(M, fmaxf(fabsf(y[i].x), fabsf(y[i].y)));
        const int sig = M > 0.f ? row_sigma(M) : 0;
        const float2 scl = make_float2(pow2f(sig), pow2f(sig)), scl8 = make_float2(pow2f(sig - 8), pow2f(sig - 8));
        if (M > 0.f) E += 32 - sig - tau;
#pragma unroll
        for (int c16 = 0; c16 < 4; ++c16) {
          uint32_t w0[4], w1[4], w2[4];
#pragma unroll
          for (int uu = 0; uu < 4; ++uu) {
            const int u = 4 * c16 + uu;
            uint32_t X0, X1, X2, X3;
            if ((I8_F2I_MASK >> (u & 7)) & 1) {
              const float2 v0 = __fmul2_rn(y[2 * u], scl), v1 = __fmul2_rn(y[2 * u + 1], scl);
              X0 = (uint32_t)__float2int_rn(v0.x), X1 = (uint32_t)__float2int_rn(v0.y);
              X2 = (uint32_t)__float2int_rn(v1.x), X3 = (uint32_t)__float2int_rn(v1.y);
            } else {
              rint24x2(y[2 * u], scl, scl8, X0, X1);
              rint24x2(y[2 * u + 1], scl, scl8, X2, X3);
            }
            const uint32_t p01 = prmt(X0, X1, 0x5140u), p23 = prmt(X2, X3, 0x5140u);
            const uint32_t q01 = prmt(X0, X1, 0x0062u), q23 = prmt(X2, X3, 0x0062u);
            w2[uu] = prmt(p01, p23, 0x5410u);
            w1[uu] = prmt(p01, p23, 0x7632u);
            w0[uu] = prmt(q01, q23, 0x5410u);
          }
          sts128u(a_c[c16], w0[0], w0[1], w0[2], w0[3]);
          sts128u(a_c[c16] + I8_A_TILE, w1[0], w1[1], w1[2], w1[3]);
          sts128u(a_c[c16] + 2 * I8_A_TILE, w2[0], w2[1], w2[2], w2[3]);
        }
        fence_async_smem();                         // the digits -> visible to the tensor core
        tc_fence_before();
        issue();
#ifdef BPPSA_F8_TRACE
        ++nstep;
#endif
      }
    }
    float2 cfin[32];
    if (!first) {                                   // D of the tile's last step
      const uint32_t td = wait_d();
#pragma unroll
      for (int qq = 0; qq < 8; ++qq) {
        float2 c[4];
        regions_to_c(td + 8 * qq, c);
#pragma unroll
        for (int i = 0; i < 4; ++i) cfin[4 * qq + i] = c[i];
      }
      release_d();
    } else {
#pragma unroll
      for (int kk = 0; kk < 32; ++kk) cfin[kk] = make_float2(2 * kk == j ? 1.f : 0.f, 2 * kk + 1 == j ? 1.f : 0.f);
    }
    if (ok) {
      float4* dst = reinterpret_cast<float4*>(agg_out + (((long long)b * n_out + q) * TH + j) * TH);
#pragma unroll
      for (int k4 = 0; k4 < 16; ++k4)
        dst[k4] = make_float4(ldexpf(cfin[2 * k4].x, E), ldexpf(cfin[2 * k4].y, E), ldexpf(cfin[2 * k4 + 1].x, E),
                              ldexpf(cfin[2 * k4 + 1].y, E));
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
// Level-0 DOWN-walk on the integer tensor cores (the down-sweep's GEMV chains,
// every down-sweep op is a vector times the transposed Jacobians).
// Chain (b, q) starts from the carry of block q (the seed for the head
// block), writes the exclusive output grad_h[t(s)] = v at every slot s of the
// block and steps v <- W^T (d_t o v) with the same digit arithmetic as the
// fold (v kept in true fp32 scale: v = c' 2^(32 - sigma - tau)).  The walk
// is bound by HBM (h read + grad_h written once) and by the latency of its
// dependent steps, not by the tensor pipe, so it runs ONE 128-chain tile per
// SM with the digits in TMEM (the TS form: 146 instead of ~170 cycles per
// MMA, no shared-memory round trip): D at TMEM columns [0, 256), the three
// digit tiles at [256, 304).  16 warps, thread = chain row x 16 columns.
// Chains are ordered id = q B + b, so at one step a tile's h rows (and
// grad_h rows) are a few contiguous runs of B rows; all threads copy them in
// and out COALESCED (each warp instruction moves 512 contiguous bytes)
// through shared memory with padded 272-byte rows, so the per-chain column
// slices are read and written without bank conflicts (per-thread 128-byte
// global accesses at a 256-byte stride measured 3300 cycles per step).  The
// copies (h two steps ahead into a 4-stage ring, the previous step's grad_h
// out of a double-buffered staging area) run while the step's MMAs do.
// ---------------------------------------------------------------------------
constexpr int WK_NST = 4;                           // h ring stages (prefetch distance 2)
constexpr int WK_PF = 2;
constexpr int WK_EPI = 512;                         // 16 warps: thread = chain row x 16 columns
constexpr int WK_ROW = 272;                         // padded row: 256 B + 16
constexpr int WK_STAGE = TM * WK_ROW;
constexpr int WK_OFF_RING = I8_B_BYTES;             // [stage][128 rows][WK_ROW]
constexpr int WK_OFF_OUT = WK_OFF_RING + WK_NST * WK_STAGE;   // grad_h staging [2][128 rows][WK_ROW]
constexpr int WK_OFF_RED = WK_OFF_OUT + 2 * WK_STAGE;         // [parity][128 rows][4] u32
constexpr int WK_OFF_BAR = WK_OFF_RED + 2 * TM * 16;
constexpr int WK_SMEM = WK_OFF_BAR + 64 + 1024;
constexpr uint32_t WK_A_COL = 256;                  // TMEM column of the x0 digit tile (x1 +16, x2 +32)
constexpr int WK_CP = TM / (WK_EPI / 16);           // copy passes per tile (16 lanes per row)

__device__ __forceinline__ void mma6_i8_ts_commit(uint32_t d, uint32_t a, const uint64_t (&bd)[2], uint32_t bar) {
  asm volatile(
      "{\n"
      " .reg .pred e, f, t;\n"
      " .reg .b32 dd, aa;\n"
      " setp.ne.b32 f, 0, 0;\n"
      " setp.eq.b32 t, 0, 0;\n"
      " elect.sync _|e, 0xffffffff;\n"
      " @e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %4, f;\n"
      " add.u32 aa, %1, 8;\n"
      " @e tcgen05.mma.cta_group::1.kind::i8 [%0], [aa], %3, %4, t;\n"
      " add.u32 dd, %0, 64;\n"
      " add.u32 aa, %1, 16;\n"
      " @e tcgen05.mma.cta_group::1.kind::i8 [dd], [aa], %2, %5, t;\n"
      " add.u32 aa, %1, 24;\n"
      " @e tcgen05.mma.cta_group::1.kind::i8 [dd], [aa], %3, %5, t;\n"
      " add.u32 dd, %0, 128;\n"
      " add.u32 aa, %1, 32;\n"
      " @e tcgen05.mma.cta_group::1.kind::i8 [dd], [aa], %2, %6, t;\n"
      " add.u32 aa, %1, 40;\n"
      " @e tcgen05.mma.cta_group::1.kind::i8 [dd], [aa], %3, %6, t;\n"
      " @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%7];\n"
      "}\n" ::"r"(d),
      "r"(a), "l"(bd[0]), "l"(bd[1]), "r"(idesc_i8(256, 1)), "r"(idesc_i8(192, 0)), "r"(idesc_i8(128, 0)), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tmem_st4(uint32_t taddr, uint32_t r0, uint32_t r1, uint32_t r2, uint32_t r3) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};\n" ::"r"(taddr), "r"(r0), "r"(r1), "r"(r2),
               "r"(r3)
               : "memory");
}
// 2^e as a float for any integer e (0 below the denormal range, inf above)
__device__ __forceinline__ float exp2i(int e) {
  if (e > 127) return __int_as_float(0x7f800000);
  if (e >= -126) return __int_as_float((e + 127) << 23);
  if (e >= -149) return __int_as_float(1 << (e + 149));
  return 0.f;
}

__global__ void __launch_bounds__(WK_EPI, 1) tc_walk_i8_kernel(LeafArgs a, int C, const float* __restrict__ carry,
                                                             long long nblk, float* __restrict__ grad_h,
                                                             float* __restrict__ grad_init) {
  extern __shared__ uint8_t smem_raw[];
  char* smem = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* d_full = reinterpret_cast<uint64_t*>(smem + WK_OFF_BAR);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(d_full + 1);
  uint32_t* wred = tmem_slot + 1;
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const int B = a.seg.B;
  const long long S = a.seg.S();
  const long long nch = (long long)B * nblk, ntiles = (nch + TM - 1) / TM;

  if (threadIdx.x == 0) wred[0] = 0;
  __syncthreads();
  int tau;
  w_digits(a.W, smem, wred, &tau);
  if (warp == 0) {
    if (lane == 0) {
      mbar_init(su32(&d_full[0]), 1);
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

  const int quad = warp & 3, row = quad * 32 + lane, cq = warp >> 2;   // columns [16 cq, 16 cq + 16)
  const bool issuer = warp == 0;
  const uint32_t t_mine = tmem + ((uint32_t)(quad * 32) << 16) + 16 * cq;   // + 64 r (regions)
  const uint32_t a_mine = tmem + ((uint32_t)(quad * 32) << 16) + WK_A_COL + 4 * cq;   // + 16 digit
  const uint32_t ring0 = su32(smem + WK_OFF_RING);
  const uint32_t out0 = su32(smem + WK_OFF_OUT);
  const uint32_t mine = (uint32_t)(row * WK_ROW + cq * 64);               // this thread's slice in a stage
  const uint32_t red0 = su32(smem + WK_OFF_RED) + (uint32_t)(row * 16);
  const uint32_t dbar = su32(&d_full[0]);
  uint64_t bd[2];
  {
    const uint32_t bb = __shfl_sync(0xffffffffu, su32(smem), 0);
    bd[0] = sdesc64(bb);
    bd[1] = sdesc64(bb + 32);
  }
  const uint32_t a_tile = __shfl_sync(0xffffffffu, tmem + WK_A_COL, 0);
  uint32_t ph = 0, par = 0;
  const long long rowB = (long long)B * TH;
  auto blk = [&](long long q, long long& st0, long long& st1) {   // slots [st0, st1) of block q
    st0 = (a.seg.head && q == 0) ? 1 : q * C;
    st1 = min(q * C + (long long)C, S);
  };
  // coalesced copy roles: 16 lanes per 256-byte row (16 bytes each), 32 rows per pass
  const int crow = threadIdx.x >> 4, cchunk = threadIdx.x & 15;
  for (long long tt = blockIdx.x; tt < ntiles; tt += gridDim.x) {
    const long long id = tt * TM + row;
    const bool valid = id < nch;
    const long long q = valid ? id / B : 0;
    const int b = valid ? (int)(id % B) : 0;
    long long s_start, s1;
    blk(q, s_start, s1);
    const int len = valid ? (int)(s1 - s_start) : 0;
    const bool total = valid && grad_init != nullptr && s1 == S;
    const int nJ = total ? len : max(len - 1, 0);          // J applications of this chain
    int steps = 0;                                         // the longest chain of the tile
    {
      const long long q_lo = (tt * TM) / B, q_hi = min(nblk - 1, (tt * TM + TM - 1) / B);
      for (long long qq = q_lo; qq <= q_hi; ++qq) {
        long long a0, a1;
        blk(qq, a0, a1);
        steps = max(steps, (int)(a1 - a0));
      }
    }
    // this thread's copy rows r = 32 pass + crow: slot start, length, sample
    int cr_s0[WK_CP], cr_len[WK_CP], cr_b[WK_CP];
#pragma unroll
    for (int pass = 0; pass < WK_CP; ++pass) {
      const long long cid = tt * TM + pass * 32 + crow;
      cr_len[pass] = 0, cr_s0[pass] = 0, cr_b[pass] = 0;
      if (cid < nch) {
        long long c0, c1;
        blk(cid / B, c0, c1);
        cr_s0[pass] = (int)c0;
        cr_len[pass] = (int)(c1 - c0);
        cr_b[pass] = (int)(cid % B);
      }
    }
    auto row_off = [&](int pass, int st) -> long long {    // h / grad_h offset of copy row `pass`, or -1
      if (st >= cr_len[pass]) return -1;
      return (long long)a.seg.time_of(cr_s0[pass] + st) * rowB + (long long)cr_b[pass] * TH;
    };
    auto stage = [&](int st) {                             // h rows of step st -> ring stage st % 4
      const uint32_t dst0 = ring0 + (uint32_t)((st % WK_NST) * WK_STAGE);
#pragma unroll
      for (int pass = 0; pass < WK_CP; ++pass) {
        const long long off = row_off(pass, st);
        if (off >= 0) cp_async16(dst0 + (uint32_t)((pass * 32 + crow) * WK_ROW + cchunk * 16), a.h + off + cchunk * 4);
      }
      asm volatile("cp.async.commit_group;\n" ::: "memory");   // one group per step, empty or not
    };
    auto copy_out = [&](int st) {                          // staged grad_h rows of step st -> HBM
      const uint32_t src0 = out0 + (uint32_t)((st & 1) * WK_STAGE);
#pragma unroll
      for (int pass = 0; pass < WK_CP; ++pass) {
        const long long off = row_off(pass, st);
        if (off >= 0)
          reinterpret_cast<float4*>(grad_h + off)[cchunk] = lds128(src0 + (uint32_t)((pass * 32 + crow) * WK_ROW + cchunk * 16));
      }
    };
    float2 v[8];                                    // this thread's 16 columns of the chain (true scale)
    {
      const float* src = (a.seg.head && q == 0) ? a.seed + (long long)b * TH : carry + ((long long)b * nblk + q) * TH;
#pragma unroll
      for (int k4 = 0; k4 < 4; ++k4) {
        const float4 f = valid ? __ldg(reinterpret_cast<const float4*>(src + 16 * cq) + k4) : make_float4(0.f, 0.f, 0.f, 0.f);
        v[2 * k4] = make_float2(f.x, f.y);
        v[2 * k4 + 1] = make_float2(f.z, f.w);
      }
    }
    for (int st = 0; st < WK_PF; ++st) stage(st);
    asm volatile("cp.async.wait_group %0;\n" ::"n"(WK_PF - 1) : "memory");   // step 0's rows (this thread's)
    __syncthreads();                                       // ... and everyone's
    for (int st = 0; st < steps; ++st) {
      const int tz = (int)(tt / gridDim.x) * 600 + st;
      if (warp == 0) I8T(0, tz);
      const uint32_t hs = ring0 + (uint32_t)((st % WK_NST) * WK_STAGE) + mine;
      const bool apply = st < nJ;
      float2 y[8];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const float4 h4 = lds128(hs + 16u * c);
        const float2 d0 = make_float2(fmaf(-h4.x, h4.x, 1.f), fmaf(-h4.y, h4.y, 1.f));
        const float2 d1 = make_float2(fmaf(-h4.z, h4.z, 1.f), fmaf(-h4.w, h4.w, 1.f));
        y[2 * c] = apply ? __fmul2_rn(d0, v[2 * c]) : make_float2(0.f, 0.f);
        y[2 * c + 1] = apply ? __fmul2_rn(d1, v[2 * c + 1]) : make_float2(0.f, 0.f);
      }
      float pm = 0.f;
#pragma unroll
      for (int i = 0; i < 8; ++i) pm = fmaxf(pm, fmaxf(fabsf(y[i].x), fabsf(y[i].y)));
      const uint32_t redp = red0 + par * (TM * 16);
      asm volatile("st.shared.u32 [%0], %1;\n" ::"r"(redp + 4u * cq), "r"(__float_as_uint(pm)) : "memory");
      if (warp == 0) I8T(3, tz);
      named_bar(3 + quad, 128);                     // the row's four threads (warps quad + 4 cq)
      if (warp == 0) I8T(4, tz);
      uint32_t m4[4];
      asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];\n"
                   : "=r"(m4[0]), "=r"(m4[1]), "=r"(m4[2]), "=r"(m4[3])
                   : "r"(redp)
                   : "memory");
      par ^= 1;
      const float M = __uint_as_float(max(max(m4[0], m4[1]), max(m4[2], m4[3])));
      const int sig = M > 0.f ? row_sigma(M) : 0;
      const float2 scl = make_float2(pow2f(sig), pow2f(sig)), scl8 = make_float2(pow2f(sig - 8), pow2f(sig - 8));
      const float f = M > 0.f ? exp2i(32 - sig - tau) : 0.f;
      uint32_t w0[4], w1[4], w2[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        uint32_t X0, X1, X2, X3;
        rint24x2(y[2 * u], scl, scl8, X0, X1);
        rint24x2(y[2 * u + 1], scl, scl8, X2, X3);
        const uint32_t p01 = prmt(X0, X1, 0x5140u), p23 = prmt(X2, X3, 0x5140u);
        const uint32_t q01 = prmt(X0, X1, 0x0062u), q23 = prmt(X2, X3, 0x0062u);
        w2[u] = prmt(p01, p23, 0x5410u);
        w1[u] = prmt(p01, p23, 0x7632u);
        w0[u] = prmt(q01, q23, 0x5410u);
      }
      if (warp == 0) I8T(5, tz);
      tmem_st4(a_mine, w0[0], w0[1], w0[2], w0[3]);
      tmem_st4(a_mine + 16, w1[0], w1[1], w1[2], w1[3]);
      tmem_st4(a_mine + 32, w2[0], w2[1], w2[2], w2[3]);
      asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
      tc_fence_before();
      named_bar(1, WK_EPI);                         // digits complete
      if (warp == 0) I8T(7, tz);
      if (issuer) {
        tc_fence_after();
        mma6_i8_ts_commit(tmem, a_tile, bd, dbar);
      }
      // while the MMAs run: grad_h of this slot (= v, the exclusive output) into
      // staging, the previous step's rows out, the rows of step st+2 in
      {
        const uint32_t o = out0 + (uint32_t)((st & 1) * WK_STAGE) + mine;
#pragma unroll
        for (int c = 0; c < 4; ++c) sts128(o + 16u * c, v[2 * c].x, v[2 * c].y, v[2 * c + 1].x, v[2 * c + 1].y);
      }
      if (st > 0) copy_out(st - 1);
      stage(st + WK_PF);
      asm volatile("cp.async.wait_group %0;\n" ::"n"(WK_PF - 1) : "memory");   // step st+1's rows (this thread's)
      if (issuer) {
        if (lane == 0) mbar_wait(dbar, ph);
        __syncwarp();
      }
      named_bar(2, WK_EPI);                         // D ready; step st+1's rows landed; staging written
      if (warp == 0) I8T(8, tz);
      ph ^= 1;
      tc_fence_after();
#pragma unroll
      for (int qq = 0; qq < 2; ++qq) {
        float2 c[4];
        regions_to_c(t_mine + 8 * qq, c);
#pragma unroll
        for (int i = 0; i < 4; ++i) v[4 * qq + i] = __fmul2_rn(c[i], make_float2(f, f));
      }
      if (warp == 0) I8T(9, tz);
      if (total && st == len - 1) {                 // dl/dh_init = J_0^T grad_h[0]
        float4* dst = reinterpret_cast<float4*>(grad_init + (long long)b * TH + 16 * cq);
#pragma unroll
        for (int k4 = 0; k4 < 4; ++k4) dst[k4] = make_float4(v[2 * k4].x, v[2 * k4].y, v[2 * k4 + 1].x, v[2 * k4 + 1].y);
      }
    }
    if (steps > 0) copy_out(steps - 1);             // (staged before the last D barrier)
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(TMEM_COLS));
  }
}


// ---------------------------------------------------------------------------
// The int8 walk with TMA (the default when B <= 128): the same arithmetic as
// tc_walk_i8_kernel, the data movement of the opt-in 3xFP16 walk.  A tile is
// G = 128 / B whole groups of B chains (G consecutive level-0 blocks, all
// samples), so the h rows of one step are one 5D box {32, 2, B, 1, G} (block
// 0's tile and blocks whose box would leave the view: 3D boxes per group),
// loaded by TMA into a ring of SWIZZLE_128B stages two steps ahead; every
// thread overwrites the h slice it consumed with v (the exclusive output
// grad_h[t]) and the issuer TMA-stores the stage with the same box — the
// stores are asynchronous bulk operations, so the grad_h write-back no longer
// blocks the epilogue under memory back-pressure (the cp.async / STG walk
// above: ~2000 of ~3950 cycles per step).  One tile per CTA at a time, 16
// warps (thread = chain row x 16 columns, row max over 4 threads), digits in
// TMEM (TS form), D of step st read at the start of step st + 1.
// ---------------------------------------------------------------------------
constexpr int WT_NST = 3;                           // ring stages
constexpr int WT_STAGE = TM * 256;                  // [128 rows][2 halves][128 B]
constexpr int WT_OFF_RING = I8_B_BYTES;
constexpr int WT_OFF_RED = WT_OFF_RING + WT_NST * WT_STAGE;   // [parity][128 rows][4] u32
constexpr int WT_OFF_BAR = WT_OFF_RED + 2 * TM * 16;
constexpr int WT_SMEM = WT_OFF_BAR + 64 + 1024;

__global__ void __launch_bounds__(WK_EPI, 1) tc_walk_i8t_kernel(LeafArgs a, const __grid_constant__ CUtensorMap h3,
                                                              const __grid_constant__ CUtensorMap h5,
                                                              const __grid_constant__ CUtensorMap g3,
                                                              const __grid_constant__ CUtensorMap g5, int C,
                                                              const float* __restrict__ carry, long long nblk,
                                                              float* __restrict__ grad_init, int G) {
  extern __shared__ uint8_t smem_raw[];
  char* smem = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* d_full = reinterpret_cast<uint64_t*>(smem + WT_OFF_BAR);
  uint64_t* h_full = d_full + 1;                    // [WT_NST]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(h_full + WT_NST);
  uint32_t* wred = tmem_slot + 1;
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const int B = a.seg.B;
  const long long S = a.seg.S();

  if (threadIdx.x == 0) wred[0] = 0;
  for (int e = threadIdx.x; e < WT_NST * WT_STAGE / 16; e += WK_EPI)
    sts128(su32(smem + WT_OFF_RING) + 16u * e, 0.f, 0.f, 0.f, 0.f);
  __syncthreads();
  int tau;
  w_digits(a.W, smem, wred, &tau);
  if (warp == 0) {
    if (lane == 0) {
      mbar_init(su32(&d_full[0]), 1);
      for (int k = 0; k < WT_NST; ++k) mbar_init(su32(&h_full[k]), 1);
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

  const int quad = warp & 3, row = quad * 32 + lane, cq = warp >> 2;   // columns [16 cq, 16 cq + 16)
  const bool issuer = warp == 0;
  const uint32_t t_mine = tmem + ((uint32_t)(quad * 32) << 16) + 16 * cq;
  const uint32_t a_mine = tmem + ((uint32_t)(quad * 32) << 16) + WK_A_COL + 4 * cq;
  const uint32_t ring = su32(smem + WT_OFF_RING);
  const int half = cq >> 1;
  // stage layout [half][row][32 floats] (the tensor maps put the column half
  // outermost): a warp's 32 rows are 32 consecutive 128-byte lines, so the
  // SWIZZLE_128B chunk positions of a column chunk cover all eight 16-byte
  // slots (the [row][half] layout gave four: 2-way bank conflicts)
  const int GB = G * B;
  const uint32_t hrow_off = (uint32_t)((half * GB + row) * 128);        // my half-row in a stage
  const int swz = (half * GB + row) & 7;                                // its 128-byte line's swizzle
  const bool in_stage = row < GB;
  const int c0 = (cq & 1) * 4;                                           // my first 16-byte chunk of the line
  const uint32_t red0 = su32(smem + WT_OFF_RED) + (uint32_t)(row * 16);
  const uint32_t dbar = su32(&d_full[0]), hbar0 = su32(&h_full[0]);
  uint64_t bd[2];
  {
    const uint32_t bb = __shfl_sync(0xffffffffu, su32(smem), 0);
    bd[0] = sdesc64(bb);
    bd[1] = sdesc64(bb + 32);
  }
  const uint32_t a_tile = __shfl_sync(0xffffffffu, tmem + WK_A_COL, 0);
  uint32_t dph = 0, par = 0, gs = 0;
  // tile row = j B + b holds group r = G-1-j (block q = qb + r), sample b: the
  // 5D box delivers the groups of one step in decreasing q order
  const int jrow = row / B, bsm = row % B, grp = G - 1 - jrow;
  // view of the time axis as (block c4, step c3): t = c4 C + c3 = Tm - q C - st
  const long long Tm = (long long)a.seg.T - 1 + a.seg.head;
  const int A_blk = (int)(Tm / C), R_off = (int)(Tm % C);
  // tiles: [0] = block 0 alone; [1 .. nfull] = G blocks each whose merged box
  // stays inside the view at every step; then the remaining blocks two per tile
  const long long nfull = A_blk > 1 ? (A_blk - 1) / G : 0;
  const long long rem0 = 1 + nfull * G;
  const long long ntiles = 1 + nfull + (nblk > rem0 ? (nblk - rem0 + 1) / 2 : 0);

  for (long long tt = blockIdx.x; tt < ntiles; tt += gridDim.x) {
    const bool merged = tt >= 1 && tt <= nfull;
    const long long qb = tt == 0 ? 0 : (merged ? 1 + (tt - 1) * G : rem0 + 2 * (tt - nfull - 1));
    const int ng = tt == 0 ? 1 : (merged ? G : (int)min(2LL, nblk - qb));   // groups in this tile
    const long long q = qb + grp;
    const bool valid = jrow < G && grp < ng;
    const bool head = a.seg.head && q == 0;
    const long long s_start = head ? 1 : q * C, s1 = min(q * C + C, S);
    const int len = valid ? (int)(s1 - s_start) : 0;
    const bool total = valid && grad_init != nullptr && s1 == S;
    const int nJ = total ? len : max(len - 1, 0);          // J applications of this chain
    float2 v[8];                                    // this thread's 16 columns of the chain (true scale)
    {
      const float* src = head ? a.seed + (long long)bsm * TH : carry + ((long long)bsm * nblk + q) * TH;
#pragma unroll
      for (int k4 = 0; k4 < 4; ++k4) {
        const float4 f = valid ? __ldg(reinterpret_cast<const float4*>(src + 16 * cq) + k4) : make_float4(0.f, 0.f, 0.f, 0.f);
        v[2 * k4] = make_float2(f.x, f.y);
        v[2 * k4 + 1] = make_float2(f.z, f.w);
      }
    }
    long long my_ss = 0, my_len = 0;                 // issuer lane r: group r's slot start and length
    const bool my_on = lane < ng;
    if (my_on) {
      const long long qr = qb + lane;
      my_ss = (a.seg.head && qr == 0) ? 1 : qr * C;
      my_len = min(qr * C + C, S) - my_ss;
    }
    const uint32_t my_dst = (uint32_t)((G - 1 - lane) * B * 128);     // + half * GB * 128
    auto c5 = [&](int st, int& c3, int& c4) {
      c3 = R_off - st;
      c4 = A_blk - (int)(qb + G - 1);
      if (c3 < 0) { c3 += C; c4 -= 1; }
      return merged;
    };
    auto issue_loads = [&](int st, uint32_t gstep) {       // all lanes of the issuer warp
      const uint32_t stage = ring + (gstep % WT_NST) * WT_STAGE;
      const uint32_t bar = hbar0 + 8u * (gstep % WT_NST);
      int c3, c4;
      if (c5(st, c3, c4)) {
        if (lane == 0) {
          mbar_arrive_tx(bar, 256u * (uint32_t)(B * G));
          asm volatile(
              "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, "
              "%6}], [%7];\n" ::"r"(stage),
              "l"(reinterpret_cast<uint64_t>(&h5)), "r"(0), "r"(0), "r"(c3), "r"(c4), "r"(0), "r"(bar)
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
        __syncwarp();
        if (my_on && st < my_len)
#pragma unroll
          for (int hf = 0; hf < 2; ++hf)
            asm volatile(
                "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
                "[%5];\n" ::"r"(stage + my_dst + (uint32_t)(hf * GB * 128)),
                "l"(reinterpret_cast<uint64_t>(&h3)), "r"(0), "r"(a.seg.time_of(my_ss + st) * B), "r"(hf), "r"(bar)
                : "memory");
      }
    };
    auto issue_stores = [&](int st, uint32_t gstep) {
      const uint32_t stage = ring + (gstep % WT_NST) * WT_STAGE;
      int c3, c4;
      if (c5(st, c3, c4)) {
        if (lane == 0)
          asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];\n" ::"l"(
                           reinterpret_cast<uint64_t>(&g5)),
                       "r"(0), "r"(0), "r"(c3), "r"(c4), "r"(0), "r"(stage)
                       : "memory");
      } else if (my_on && st < my_len) {
#pragma unroll
        for (int hf = 0; hf < 2; ++hf)
          asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];\n" ::"l"(
                           reinterpret_cast<uint64_t>(&g3)),
                       "r"(0), "r"(a.seg.time_of(my_ss + st) * B), "r"(hf), "r"(stage + my_dst + (uint32_t)(hf * GB * 128))
                       : "memory");
      }
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
    };
    if (issuer) {
      // the stages about to be refilled were last stored from by this warp
      asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
      issue_loads(0, gs);
      if (C > 1) issue_loads(1, gs + 1);
      __syncwarp();
    }
    float f_prev = 0.f;                              // v = D f after the previous step's MMAs
    for (int st = 0; st < C; ++st, ++gs) {
      const int tz = (int)(tt / gridDim.x) * C + st;
      (void)tz;
      if (warp == 0) I8T(0, tz);
      if (issuer) {                                  // D of step st-1 and h of step st
        if (lane == 0) {
          if (st > 0) mbar_wait(dbar, dph);
          mbar_wait(hbar0 + 8u * (gs % WT_NST), (gs / WT_NST) & 1);
        }
        __syncwarp();
      }
      named_bar(2, WK_EPI);
      if (warp == 0) I8T(1, tz);
      if (st > 0) {
        dph ^= 1;
        tc_fence_after();
#pragma unroll
        for (int qq = 0; qq < 2; ++qq) {
          float2 c[4];
          regions_to_c(t_mine + 8 * qq, c);
#pragma unroll
          for (int i = 0; i < 4; ++i) v[4 * qq + i] = __fmul2_rn(c[i], make_float2(f_prev, f_prev));
        }
        if (total && st == len) {                    // dl/dh_init = J_0^T grad_h[0]
          float4* dst = reinterpret_cast<float4*>(grad_init + (long long)bsm * TH + 16 * cq);
#pragma unroll
          for (int k4 = 0; k4 < 4; ++k4) dst[k4] = make_float4(v[2 * k4].x, v[2 * k4].y, v[2 * k4 + 1].x, v[2 * k4 + 1].y);
        }
      }
      // y = d o v from the staged, swizzled h slice; grad_h[t(s)] = v written in its place
      const uint32_t stg = ring + (gs % WT_NST) * WT_STAGE + hrow_off;
      const bool apply = st < nJ;
      float2 y[8];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const uint32_t hp = stg + (uint32_t)(((c0 + c) ^ swz) << 4);
        // rows >= G B (no chain) would alias the other half plane's first lines
        const float4 h4 = in_stage ? lds128(hp) : make_float4(0.f, 0.f, 0.f, 0.f);
        if (in_stage) sts128(hp, v[2 * c].x, v[2 * c].y, v[2 * c + 1].x, v[2 * c + 1].y);
        const float2 d0 = make_float2(fmaf(-h4.x, h4.x, 1.f), fmaf(-h4.y, h4.y, 1.f));
        const float2 d1 = make_float2(fmaf(-h4.z, h4.z, 1.f), fmaf(-h4.w, h4.w, 1.f));
        y[2 * c] = apply ? __fmul2_rn(d0, v[2 * c]) : make_float2(0.f, 0.f);
        y[2 * c + 1] = apply ? __fmul2_rn(d1, v[2 * c + 1]) : make_float2(0.f, 0.f);
      }
      if (warp == 0) I8T(2, tz);
      float pm = 0.f;
#pragma unroll
      for (int i = 0; i < 8; ++i) pm = fmaxf(pm, fmaxf(fabsf(y[i].x), fabsf(y[i].y)));
      const uint32_t redp = red0 + par * (TM * 16);
      asm volatile("st.shared.u32 [%0], %1;\n" ::"r"(redp + 4u * cq), "r"(__float_as_uint(pm)) : "memory");
      named_bar(3 + quad, 128);                      // the row's four threads (warps quad + 4 cq)
      uint32_t m4[4];
      asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];\n"
                   : "=r"(m4[0]), "=r"(m4[1]), "=r"(m4[2]), "=r"(m4[3])
                   : "r"(redp)
                   : "memory");
      par ^= 1;
      if (warp == 0) I8T(3, tz);
      const float M = __uint_as_float(max(max(m4[0], m4[1]), max(m4[2], m4[3])));
      const int sig = M > 0.f ? row_sigma(M) : 0;
      const float2 scl = make_float2(pow2f(sig), pow2f(sig)), scl8 = make_float2(pow2f(sig - 8), pow2f(sig - 8));
      f_prev = M > 0.f ? exp2i(32 - sig - tau) : 0.f;
      uint32_t w0[4], w1[4], w2[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        uint32_t X0, X1, X2, X3;
        rint24x2(y[2 * u], scl, scl8, X0, X1);
        rint24x2(y[2 * u + 1], scl, scl8, X2, X3);
        const uint32_t p01 = prmt(X0, X1, 0x5140u), p23 = prmt(X2, X3, 0x5140u);
        const uint32_t q01 = prmt(X0, X1, 0x0062u), q23 = prmt(X2, X3, 0x0062u);
        w2[u] = prmt(p01, p23, 0x5410u);
        w1[u] = prmt(p01, p23, 0x7632u);
        w0[u] = prmt(q01, q23, 0x5410u);
      }
      tmem_st4(a_mine, w0[0], w0[1], w0[2], w0[3]);
      tmem_st4(a_mine + 16, w1[0], w1[1], w1[2], w1[3]);
      tmem_st4(a_mine + 32, w2[0], w2[1], w2[2], w2[3]);
      asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
      fence_async_smem();                            // grad_h rows (stored long before) -> visible to the TMA store
      tc_fence_before();
      if (warp == 0) I8T(4, tz);
      named_bar(1, WK_EPI);                          // digits complete, stage consumed and rewritten
      if (warp == 0) I8T(5, tz);
      if (issuer) {
        tc_fence_after();
        mma6_i8_ts_commit(tmem, a_tile, bd, dbar);
        issue_stores(st, gs);
        if (st + 2 < C) {
          // stage (gs + 2) % 3 was stored from at step st - 1: its reads must be done
          asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
          issue_loads(st + 2, gs + 2);
        }
        __syncwarp();
      }
      if (warp == 0) I8T(6, tz);
    }
    // D of the last step (keeps the barrier phase; grad_init if the chain ends here)
    if (issuer) {
      if (lane == 0) mbar_wait(dbar, dph);
      __syncwarp();
    }
    named_bar(2, WK_EPI);
    dph ^= 1;
    tc_fence_after();
#pragma unroll
    for (int qq = 0; qq < 2; ++qq) {                 // tcgen05.ld is warp-aligned: every lane loads
      float2 c[4];
      regions_to_c(t_mine + 8 * qq, c);
#pragma unroll
      for (int i = 0; i < 4; ++i) v[4 * qq + i] = __fmul2_rn(c[i], make_float2(f_prev, f_prev));
    }
    if (total && len == C) {
      float4* dst = reinterpret_cast<float4*>(grad_init + (long long)bsm * TH + 16 * cq);
#pragma unroll
      for (int k4 = 0; k4 < 4; ++k4) dst[k4] = make_float4(v[2 * k4].x, v[2 * k4].y, v[2 * k4 + 1].x, v[2 * k4 + 1].y);
    }
    tc_fence_before();
    named_bar(2, WK_EPI);                            // the D reads are done before the next tile's MMAs
  }
  if (issuer) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");   // the last stores have landed
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

}  // namespace

#ifdef BPPSA_F8_TRACE
extern "C" int bppsa_debug_f8_trace(long long* host) {
  return (int)cudaMemcpyFromSymbol(host, g_f8_trace, sizeof(g_f8_trace));
}
extern "C" int bppsa_debug_r8_trace(long long* host) {
  return (int)cudaMemcpyFromSymbol(host, g_r8_trace, sizeof(g_r8_trace));
}
#endif
#ifdef BPPSA_I8_TRACE
extern "C" int bppsa_debug_i8_trace(long long* host) {
  return (int)cudaMemcpyFromSymbol(host, g_i8_trace, sizeof(g_i8_trace));
}
#endif

// Matrix blocks q in [q0, n_out) of an RNN H = 64 segment, exact-integer fold.
cudaError_t launch_tc_fold_i8(const LeafArgs& a, int C, float* agg_out, long long n_out, long long q0, int num_sms,
                              cudaStream_t st) {
  if (a.seg.H != TH) return cudaErrorInvalidValue;
  const long long ntiles = (long long)((a.seg.B + 1) / 2) * (n_out - q0);
  const int grid = (int)std::min<long long>((ntiles + 1) / 2, num_sms);
  if (grid <= 0) return cudaSuccess;
#ifndef BPPSA_FOLD_TWO_SLOT
  {
    const int gr = (int)std::min<long long>((ntiles + R_NT - 1) / R_NT, num_sms);
    cudaError_t e = smem_attr_once(reinterpret_cast<const void*>(tc_fold_i8r_kernel), R_SMEM);
    if (e != cudaSuccess) return e;
    tc_fold_i8r_kernel<<<gr, R_THREADS, R_SMEM, st>>>(a, C, agg_out, n_out, q0);
    return cudaGetLastError();
  }
#endif
  cudaError_t e = smem_attr_once(reinterpret_cast<const void*>(tc_fold_i8_kernel), I8_SMEM);
  if (e != cudaSuccess) return e;
  tc_fold_i8_kernel<<<grid, I8_NT, I8_SMEM, st>>>(a, C, agg_out, n_out, q0);
  return cudaGetLastError();
}

// Level-0 walk of an RNN H = 64 segment on the integer tensor cores.
// Tensor maps over h / grad_h with the column half OUTERMOST, so a box lands
// in shared memory as [half][rows][32 floats] (SWIZZLE_128B): 5D {col 32, b,
// step-in-block, block, half} with box {32, B, 1, G, 2}; 3D {col 32, t B + b,
// half} with box {32, B, 1} (one per half, per group).
static cudaError_t make_walk_map_split(const float* base, int T, int B, int C, long long A, bool five, int G,
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
    const cuuint64_t dims[3] = {32, (cuuint64_t)T * B, 2};
    const cuuint64_t strides[2] = {row, 128};
    const cuuint32_t box[3] = {32u, (cuuint32_t)B, 1u};
    r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    if (A < 1) A = 1;
    const cuuint64_t dims[5] = {32, (cuuint64_t)B, (cuuint64_t)C, (cuuint64_t)A, 2};
    const cuuint64_t strides[4] = {row, row * B, row * B * C, 128};
    const cuuint32_t box[5] = {32u, (cuuint32_t)B, 1u, (cuuint32_t)G, 2u};
    r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, const_cast<float*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

cudaError_t launch_tc_walk_i8(const LeafArgs& a, int C, const float* carry, long long nblk, float* grad_h,
                              float* grad_init, int num_sms, cudaStream_t st) {
  if (a.seg.H != TH) return cudaErrorInvalidValue;
  static const bool cpasync = std::getenv("BPPSA_WALK_I8_CPASYNC") != nullptr;   // dev aid: the cp.async walk
  if (a.seg.B <= TM && !cpasync) {
    const int B = a.seg.B, G = TM / B;
    const long long Tm = (long long)a.seg.T - 1 + a.seg.head;
    CUtensorMap maps[4];
    cudaError_t e = cudaSuccess;
    for (int m = 0; m < 4 && e == cudaSuccess; ++m)
      e = make_walk_map_split(m < 2 ? a.h : grad_h, a.seg.T, B, C, Tm / C, m % 2 == 1, G, &maps[m]);
    if (e != cudaSuccess) return e;
    const long long A = Tm / C, nfull = A > 1 ? (A - 1) / G : 0, rem0 = 1 + nfull * G;
    const long long nt = 1 + nfull + (nblk > rem0 ? (nblk - rem0 + 1) / 2 : 0);
    const int gridw = (int)std::min<long long>(nt, num_sms);
    e = smem_attr_once(reinterpret_cast<const void*>(tc_walk_i8t_kernel), WT_SMEM);
    if (e != cudaSuccess) return e;
    tc_walk_i8t_kernel<<<gridw, WK_EPI, WT_SMEM, st>>>(a, maps[0], maps[1], maps[2], maps[3], C, carry, nblk,
                                                       grad_init, G);
    return cudaGetLastError();
  }
  const long long ntiles = ((long long)a.seg.B * nblk + TM - 1) / TM;
  const int grid = (int)std::min<long long>(ntiles, num_sms);
  if (grid <= 0) return cudaSuccess;
  cudaError_t e = smem_attr_once(reinterpret_cast<const void*>(tc_walk_i8_kernel), WK_SMEM);
  if (e != cudaSuccess) return e;
  tc_walk_i8_kernel<<<grid, WK_EPI, WK_SMEM, st>>>(a, C, carry, nblk, grad_h, grad_init);
  return cudaGetLastError();
}

}  // namespace bppsa
