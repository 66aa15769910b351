// csr.cu — the CSR SpGEMM variant of the BPPSA scan
// and the analytical CSR transposed-Jacobian builders (Algs. 2-10).
//
// Plan time (host, once per architecture): the hybrid schedule is simulated
// over the scan array [seed, J_n^T, ..., J_1^T]; every SpGEMM of the truncated
// up-sweep gets a symbolic product plan — output pattern plus, per output
// entry, its contribution pairs (left position, right position) in ascending
// left position ("calculating the number of non-zeros and index merging ...
// performed prior to training") — and the bridge / down-sweep become
// SpMVs or aliases (the symbolic identity is never materialised).
// Scan time (device, every iteration): one numeric kernel per op.
#include <algorithm>
#include <cstring>
#include <memory>
#include <thread>
#include <vector>

#include <cub/device/device_scan.cuh>

#include "common.cuh"

namespace bppsa {
namespace {

struct HCSR {
  int rows = 0, cols = 0;
  std::vector<long long> indptr;
  std::vector<int> indices;
  long long nnz() const { return indptr.empty() ? 0 : indptr.back(); }
};

enum BufKind { B_ORIG = 0, B_PROD = 1, B_VEC = 2, B_SEED = 3 };

struct Buf {
  int kind;
  int elem = -1;          // B_ORIG: element (time order)
  int pat = -1;           // matrix kinds: pattern id
  long long size = 0;     // nnz (matrices) or dim (vectors)
  unsigned long long deps = 0;   // original elements this value depends on (batched-ness)
};

enum OpKind { OP_SPGEMM = 0, OP_SPMV = 1 };
struct Op {
  int kind, out, a, b, plan;   // SPGEMM: out = a * b (plan); SPMV: out = a(mat) * b(vec)
};

struct DevPlan {
  long long nnz_out = 0, contrib = 0;
  long long* cptr = nullptr;   // [nnz_out + 1]
  int* lpos = nullptr;         // [contrib]
  int* rpos = nullptr;
};

struct DevPat {
  long long* indptr = nullptr;
  int* indices = nullptr;
};

}  // namespace
}  // namespace bppsa

struct bppsa_csr_plan {
  int n = 0, u = 0, dl = 0;
  bool symbolic = false;      // bppsa_csr_plan_create_symbolic: steps / info only, no numeric plan
  std::vector<bppsa::HCSR> pats;
  std::vector<bppsa::DevPat> dpats;
  std::vector<bppsa::Buf> bufs;
  std::vector<bppsa::Op> ops;
  std::vector<bppsa::DevPlan> plans;
  std::vector<int> out_buf;   // out_buf[k] = buffer holding dl/dx_k (k = 0..n)
  int seed_buf = -1;
  long long contributions = 0, spmv_nnz = 0;
  std::vector<bppsa_csr_step> steps;   // one per op (schedule order), then the BP baseline
  ~bppsa_csr_plan() {
    for (auto& p : plans) {
      cudaFree(p.cptr);
      cudaFree(p.lpos);
      cudaFree(p.rpos);
    }
    for (auto& d : dpats) {
      cudaFree(d.indptr);
      cudaFree(d.indices);
    }
  }
};

namespace bppsa {
namespace {

// Structural product left @ right with contribution lists (multi-threaded
// over row ranges; results independent of the thread count).
struct HostProduct {
  HCSR out;
  std::vector<long long> cptr;
  std::vector<int> lpos, rpos;
};

bool plan_product(const HCSR& L, const HCSR& R, long long cap, HostProduct* P) {
  const int rows = L.rows, cols = R.cols;
  const int nth = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  std::vector<long long> row_nnz(rows, 0), row_con(rows, 0);
  auto count = [&](int r0, int r1) {
    std::vector<int> mark(cols, -1);
    for (int i = r0; i < r1; ++i) {
      long long nz = 0, con = 0;
      for (long long p = L.indptr[i]; p < L.indptr[i + 1]; ++p) {
        const int k = L.indices[p];
        con += R.indptr[k + 1] - R.indptr[k];
        for (long long q = R.indptr[k]; q < R.indptr[k + 1]; ++q) {
          const int j = R.indices[q];
          if (mark[j] != i) {
            mark[j] = i;
            ++nz;
          }
        }
      }
      row_nnz[i] = nz;
      row_con[i] = con;
    }
  };
  auto par = [&](auto fn) {
    std::vector<std::thread> th;
    const int chunk = (rows + nth - 1) / nth;
    for (int t = 0; t < nth; ++t) {
      const int r0 = t * chunk, r1 = std::min(rows, r0 + chunk);
      if (r0 < r1) th.emplace_back(fn, r0, r1);
    }
    for (auto& x : th) x.join();
  };
  par(count);
  P->out.rows = rows;
  P->out.cols = cols;
  P->out.indptr.assign(rows + 1, 0);
  std::vector<long long> con_off(rows + 1, 0);
  for (int i = 0; i < rows; ++i) {
    P->out.indptr[i + 1] = P->out.indptr[i] + row_nnz[i];
    con_off[i + 1] = con_off[i] + row_con[i];
  }
  const long long nnz = P->out.indptr[rows], ncon = con_off[rows];
  if (ncon > cap || nnz >= (1ll << 31)) return false;
  P->out.indices.resize(nnz);
  P->cptr.assign(nnz + 1, 0);
  P->lpos.resize(ncon);
  P->rpos.resize(ncon);
  auto fill = [&](int r0, int r1) {
    std::vector<int> pos(cols, -1);
    std::vector<int> cols_row;
    std::vector<long long> cnt;
    for (int i = r0; i < r1; ++i) {
      cols_row.clear();
      for (long long p = L.indptr[i]; p < L.indptr[i + 1]; ++p) {
        const int k = L.indices[p];
        for (long long q = R.indptr[k]; q < R.indptr[k + 1]; ++q) {
          const int j = R.indices[q];
          if (pos[j] < 0) {
            pos[j] = 0;
            cols_row.push_back(j);
          }
        }
      }
      std::sort(cols_row.begin(), cols_row.end());
      const long long base = P->out.indptr[i];
      for (size_t e = 0; e < cols_row.size(); ++e) {
        pos[cols_row[e]] = (int)e;
        P->out.indices[base + e] = cols_row[e];
      }
      // contributions per output entry, in ascending left position
      cnt.assign(cols_row.size() + 1, 0);
      for (long long p = L.indptr[i]; p < L.indptr[i + 1]; ++p) {
        const int k = L.indices[p];
        for (long long q = R.indptr[k]; q < R.indptr[k + 1]; ++q) ++cnt[pos[R.indices[q]] + 1];
      }
      for (size_t e = 0; e < cols_row.size(); ++e) cnt[e + 1] += cnt[e];
      for (size_t e = 0; e < cols_row.size(); ++e) P->cptr[base + e] = con_off[i] + cnt[e];
      for (long long p = L.indptr[i]; p < L.indptr[i + 1]; ++p) {
        const int k = L.indices[p];
        for (long long q = R.indptr[k]; q < R.indptr[k + 1]; ++q) {
          const long long c = con_off[i] + cnt[pos[R.indices[q]]]++;
          P->lpos[c] = (int)p;
          P->rpos[c] = (int)q;
        }
      }
      for (int j : cols_row) pos[j] = -1;
    }
  };
  par(fill);
  P->cptr[nnz] = ncon;
  return true;
}

// Symbolic product L @ R without contribution lists (bppsa_csr_plan_create_
// symbolic): pairs in closed form, sum_k nnz(L[:, k]) nnz(R[k, :]) (the
// number of (left, right) entry pairs the numeric SpGEMM would touch), and the
// output pattern by a bitset Gustavson product: every row of R as a bit row,
// output row i = OR of the bit rows of R selected by L's row i (cost nnz(L) x
// cols / 64 word ORs; multi-threaded over row ranges, thread-count independent).
bool symbolic_product(const HCSR& L, const HCSR& R, HCSR* out, long long* pairs) {
  std::vector<long long> colL(L.cols, 0);
  for (int k : L.indices) ++colL[k];
  long long pc = 0;
  for (int k = 0; k < L.cols; ++k) pc += colL[k] * (R.indptr[k + 1] - R.indptr[k]);
  *pairs = pc;
  const int rows = L.rows, cols = R.cols, W = (cols + 63) / 64;
  if ((double)R.rows * W * 8 > 16e9 || (double)rows * W * 8 > 16e9) return false;   // bit rows > 16 GB
  std::vector<unsigned long long> rb((size_t)R.rows * W, 0ull), ob((size_t)rows * W, 0ull);
  for (int k = 0; k < R.rows; ++k)
    for (long long q = R.indptr[k]; q < R.indptr[k + 1]; ++q)
      rb[(size_t)k * W + (R.indices[q] >> 6)] |= 1ull << (R.indices[q] & 63);
  const int nth = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  std::vector<long long> row_nnz(rows, 0);
  auto work = [&](int r0, int r1) {
    for (int i = r0; i < r1; ++i) {
      unsigned long long* o = &ob[(size_t)i * W];
      for (long long p = L.indptr[i]; p < L.indptr[i + 1]; ++p) {
        const unsigned long long* r = &rb[(size_t)L.indices[p] * W];
        for (int w = 0; w < W; ++w) o[w] |= r[w];
      }
      long long nz = 0;
      for (int w = 0; w < W; ++w) nz += __builtin_popcountll(o[w]);
      row_nnz[i] = nz;
    }
  };
  {
    std::vector<std::thread> th;
    const int chunk = (rows + nth - 1) / nth;
    for (int t = 0; t < nth; ++t) {
      const int r0 = t * chunk, r1 = std::min(rows, r0 + chunk);
      if (r0 < r1) th.emplace_back(work, r0, r1);
    }
    for (auto& x : th) x.join();
  }
  out->rows = rows;
  out->cols = cols;
  out->indptr.assign(rows + 1, 0);
  for (int i = 0; i < rows; ++i) out->indptr[i + 1] = out->indptr[i] + row_nnz[i];
  if (out->indptr[rows] >= (1ll << 31)) return false;
  out->indices.resize(out->indptr[rows]);
  for (int i = 0; i < rows; ++i) {
    long long e = out->indptr[i];
    for (int w = 0; w < W; ++w)
      for (unsigned long long b = ob[(size_t)i * W + w]; b; b &= b - 1) out->indices[e++] = w * 64 + __builtin_ctzll(b);
  }
  return true;
}

template <class T>
cudaError_t upload(T** dst, const std::vector<T>& src) {
  cudaError_t e = cudaMalloc(dst, std::max<size_t>(1, src.size()) * sizeof(T));
  if (e != cudaSuccess) return e;
  if (!src.empty()) e = cudaMemcpy(*dst, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice);
  return e;
}

// ------------------------------------------------------------------ kernels
// sample-minor layout: value (entry p, sample b) at p*B + b (batched) or p (shared)
__global__ void spgemm_kernel(const long long* __restrict__ cptr, const int* __restrict__ lpos,
                              const int* __restrict__ rpos, const float* __restrict__ L, int lb,
                              const float* __restrict__ R, int rb, float* __restrict__ out, int ob,
                              long long nnz, int B) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long nb = (long long)nnz * ob;
  if (t >= nb) return;
  const long long e = t / ob;
  const int b = (int)(t % ob);
  const int sl = lb ? B : 1, bl = lb ? b : 0, sr = rb ? B : 1, br = rb ? b : 0;
  float acc = 0.f;
  for (long long c = cptr[e]; c < cptr[e + 1]; ++c)
    acc = fmaf(__ldg(L + (long long)__ldg(lpos + c) * sl + bl), __ldg(R + (long long)__ldg(rpos + c) * sr + br), acc);
  out[t] = acc;
}

__global__ void spmv_kernel(const long long* __restrict__ indptr, const int* __restrict__ indices,
                            const float* __restrict__ M, int mb, const float* __restrict__ v, float* __restrict__ y,
                            int rows, int B) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= (long long)rows * B) return;
  const int i = (int)(t / B), b = (int)(t % B);
  const int sm = mb ? B : 1, bm = mb ? b : 0;
  float acc = 0.f;
  for (long long p = indptr[i]; p < indptr[i + 1]; ++p)
    acc = fmaf(__ldg(M + p * sm + bm), __ldg(v + (long long)__ldg(indices + p) * B + b), acc);
  y[t] = acc;
}

// [B][dim] <-> [dim][B]
__global__ void transpose_bd(const float* __restrict__ in, float* __restrict__ out, long long dim, int B,
                             int to_sample_minor) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= dim * B) return;
  if (to_sample_minor) {   // t indexes out [dim][B]
    const long long i = t / B;
    const int b = (int)(t % B);
    out[t] = in[(long long)b * dim + i];
  } else {                 // t indexes out [B][dim]
    const long long i = t % dim;
    const int b = (int)(t / dim);
    out[t] = in[i * B + b];
  }
}

__global__ void gather_kernel(const int* __restrict__ tap, const float* __restrict__ w, float* __restrict__ d,
                              long long nnz) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t < nnz) d[t] = w[tap[t]];
}

__global__ void relu_data_kernel(const float* __restrict__ x, float* __restrict__ data, long long d, int B) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;   // indexes data [d][B]
  if (t >= d * B) return;
  const long long i = t / B;
  const int b = (int)(t % B);
  data[t] = x[(long long)b * d + i] > 0.f ? 1.f : 0.f;   // Alg. 7: strict >
}

__global__ void maxpool_data_kernel(const long long* __restrict__ pidx, float* __restrict__ data, int c, int h,
                                    int w, int B) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long d = (long long)c * h * w;
  if (t >= d * B) return;
  const long long i = t / B;
  const int b = (int)(t % B);
  const int cc = (int)(i / (h * w)), rem = (int)(i % (h * w)), y = rem / w, x = rem % w;
  const int ho = h / 2, wo = w / 2;
  const long long sel = pidx[(((long long)b * c + cc) * ho + y / 2) * wo + x / 2];
  data[t] = (sel == rem) ? 1.f : 0.f;
}

// ---- device analytical builders (Algs. 2-4 on the GPU) ----
// Conv 3x3 / pad 1 / stride 1 transposed Jacobian, rows = input pixels
// (c, y, x), entries in ascending output index (o, y+oy, x+ox) — candidate
// q = o*9 + (oy+1)*3 + (ox+1) enumerates them in that order — weight tap
// W[o][c][1-oy][1-ox] (the exact pattern, reading 17: no wrap-around).
__device__ __forceinline__ int conv_ny(int y, int h) { return min(y + 1, h - 1) - max(y - 1, 0) + 1; }

// Alg. 2 (reading 15) in closed form: rows before (c, y, x) hold
// c*co*NY*NX + co*SY(y)*NX + co*ny(y)*SX(x) entries, SY(y) = sum_{y'<y} ny(y').
__global__ void conv_indptr_kernel(int ci, int co, int h, int w, long long* __restrict__ indptr) {
  const long long rows = (long long)ci * h * w;
  const long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (r > rows) return;
  const long long NY = (h == 1) ? 1 : 3ll * h - 2, NX = (w == 1) ? 1 : 3ll * w - 2;
  if (r == rows) {
    indptr[r] = (long long)ci * co * NY * NX;
    return;
  }
  const int c = (int)(r / ((long long)h * w)), rem = (int)(r % ((long long)h * w)), y = rem / w, x = rem % w;
  long long SY = 0, SX = 0;
  for (int t = 0; t < y; ++t) SY += conv_ny(t, h);
  for (int t = 0; t < x; ++t) SX += conv_ny(t, w);
  indptr[r] = (long long)c * co * NY * NX + (long long)co * SY * NX + (long long)co * conv_ny(y, h) * SX;
}

// pruned taps leave the pattern: entries per row by ballot over the candidates
__global__ void conv_count_kernel(int ci, int co, int h, int w, const float* __restrict__ wts,
                                  long long* __restrict__ cnt) {
  const int lane = threadIdx.x & 31;
  const long long r = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5);
  const long long rows = (long long)ci * h * w;
  if (r >= rows) return;
  const int c = (int)(r / ((long long)h * w)), rem = (int)(r % ((long long)h * w)), y = rem / w, x = rem % w;
  long long n = 0;
  for (int q0 = 0; q0 < co * 9; q0 += 32) {
    const int q = q0 + lane;
    bool v = false;
    if (q < co * 9) {
      const int o = q / 9, oy = (q % 9) / 3 - 1, ox = q % 3 - 1;
      const int yo = y + oy, xo = x + ox;
      v = yo >= 0 && yo < h && xo >= 0 && xo < w && wts[((o * ci + c) * 3 + (1 - oy)) * 3 + (1 - ox)] != 0.f;
    }
    n += __popc(__ballot_sync(0xffffffffu, v));
  }
  if (lane == 0) cnt[r] = n;
}

// Alg. 3 (indices) + Alg. 4 (data) with the row offsets from indptr
__global__ void conv_fill_kernel(int ci, int co, int h, int w, const float* __restrict__ wts, int drop,
                                 const long long* __restrict__ indptr, int* __restrict__ indices,
                                 int* __restrict__ tap, float* __restrict__ data) {
  const int lane = threadIdx.x & 31;
  const long long r = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5);
  const long long rows = (long long)ci * h * w;
  if (r >= rows) return;
  const int c = (int)(r / ((long long)h * w)), rem = (int)(r % ((long long)h * w)), y = rem / w, x = rem % w;
  long long p = indptr[r];
  for (int q0 = 0; q0 < co * 9; q0 += 32) {
    const int q = q0 + lane;
    bool v = false;
    int t = 0, col = 0;
    if (q < co * 9) {
      const int o = q / 9, oy = (q % 9) / 3 - 1, ox = q % 3 - 1;
      const int yo = y + oy, xo = x + ox;
      t = ((o * ci + c) * 3 + (1 - oy)) * 3 + (1 - ox);
      col = (o * h + yo) * w + xo;
      v = yo >= 0 && yo < h && xo >= 0 && xo < w && (!drop || wts[t] != 0.f);
    }
    const unsigned m = __ballot_sync(0xffffffffu, v);
    if (v) {
      const long long e = p + __popc(m & ((1u << lane) - 1u));
      indices[e] = col;
      if (tap) tap[e] = t;
      if (data) data[e] = wts[t];
    }
    p += __popc(m);
  }
}

// 2x2 / stride-2 max-pool window pattern (reading 18) and the identity (ReLU)
__global__ void pool_pattern_kernel(int c, int h, int w, long long* __restrict__ indptr, int* __restrict__ indices) {
  const long long d = (long long)c * h * w;
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i > d) return;
  indptr[i] = i;
  if (i == d) return;
  const int cc = (int)(i / ((long long)h * w)), rem = (int)(i % ((long long)h * w)), y = rem / w, x = rem % w;
  indices[i] = (cc * (h / 2) + y / 2) * (w / 2) + x / 2;
}

__global__ void identity_pattern_kernel(long long d, long long* __restrict__ indptr, int* __restrict__ indices) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i > d) return;
  indptr[i] = i;
  if (i < d) indices[i] = (int)i;
}

unsigned blocks_for(long long n, int t = 256) { return (unsigned)((n + t - 1) / t); }

size_t align256(size_t x) { return (x + 255) / 256 * 256; }

// workspace layout for (B, batched flags): offsets of every non-original buffer
bool layout(const bppsa_csr_plan& P, int B, const int* batched, std::vector<size_t>* off, size_t* total) {
  off->assign(P.bufs.size(), (size_t)-1);
  size_t o = 0;
  for (size_t i = 0; i < P.bufs.size(); ++i) {
    const Buf& b = P.bufs[i];
    if (b.kind == B_ORIG) continue;
    bool bat = true;
    if (b.kind == B_PROD) {
      bat = false;
      for (int k = 0; k < P.n; ++k)
        if (((b.deps >> k) & 1ull) && batched && batched[k]) bat = true;
    }
    (*off)[i] = o;
    o = align256(o + (size_t)b.size * (bat ? B : 1) * sizeof(float));
  }
  *total = o;
  return true;
}

bool buf_batched(const bppsa_csr_plan& P, int id, const int* batched) {
  const Buf& b = P.bufs[id];
  if (b.kind == B_ORIG) return batched && batched[b.elem];
  if (b.kind != B_PROD) return true;
  for (int k = 0; k < P.n; ++k)
    if (((b.deps >> k) & 1ull) && batched && batched[k]) return true;
  return false;
}

}  // namespace
}  // namespace bppsa

using namespace bppsa;

extern "C" {

static bppsa_status csr_plan_create_impl(const bppsa_csr_pattern* chain, int n, int up_levels, int down_levels,
                                         long long max_contributions, bool symbolic, bppsa_csr_plan** out_plan) {
  if (!chain || !out_plan || n < 1 || n > 64) return fail(BPPSA_ERR_INVALID_ARGUMENT, "need 1 <= n <= 64 and non-NULL arguments");
  const int L = 64 - __builtin_clzll((unsigned long long)n);      // ceil(log2(n+1))
  const int u = up_levels, dl = down_levels;
  if (u < 0 || u > std::max(L - 1, 0) || !(dl == u || dl == u + 1) || dl > L)
    return fail(BPPSA_ERR_INVALID_ARGUMENT, "need 0 <= up_levels <= L-1 and down_levels in {u, u+1}, <= L");
  const long long cap = max_contributions > 0 ? max_contributions : (1ll << 31);
  std::unique_ptr<bppsa_csr_plan> P(new bppsa_csr_plan());
  P->symbolic = symbolic;
  P->n = n;
  P->u = u;
  P->dl = dl;
  // validate + copy the element patterns (time order)
  for (int k = 0; k < n; ++k) {
    const bppsa_csr_pattern& c = chain[k];
    if (c.rows < 1 || c.cols < 1 || !c.indptr || (c.nnz > 0 && !c.indices))
      return fail(BPPSA_ERR_INVALID_ARGUMENT, "bad pattern " + std::to_string(k));
    if (k > 0 && chain[k - 1].cols != c.rows)
      return fail(BPPSA_ERR_SHAPE, "cols(J_" + std::to_string(k) + "^T) != rows(J_" + std::to_string(k + 1) + "^T)");
    HCSR h;
    h.rows = c.rows;
    h.cols = c.cols;
    h.indptr.assign(c.indptr, c.indptr + c.rows + 1);
    h.indices.assign(c.indices, c.indices + c.nnz);
    if (h.indptr[0] != 0 || h.indptr.back() != c.nnz) return fail(BPPSA_ERR_INVALID_ARGUMENT, "indptr inconsistent");
    for (int i = 0; i < h.rows; ++i) {
      if (h.indptr[i + 1] < h.indptr[i]) return fail(BPPSA_ERR_INVALID_ARGUMENT, "indptr decreasing");
      for (long long p = h.indptr[i]; p < h.indptr[i + 1]; ++p) {
        if (h.indices[p] < 0 || h.indices[p] >= h.cols || (p > h.indptr[i] && h.indices[p] <= h.indices[p - 1]))
          return fail(BPPSA_ERR_INVALID_ARGUMENT, "indices out of range or not strictly increasing");
      }
    }
    P->pats.push_back(std::move(h));
    Buf b;
    b.kind = B_ORIG;
    b.elem = k;
    b.pat = k;
    b.size = c.nnz;
    b.deps = 1ull << k;
    P->bufs.push_back(b);
  }
  // seed buffer and the scan slots: slot 0 = seed, slot s >= 1 = J_{n-s+1}^T
  Buf sb;
  sb.kind = B_SEED;
  sb.size = chain[n - 1].cols;
  P->bufs.push_back(sb);
  P->seed_buf = (int)P->bufs.size() - 1;
  const int IDENT = -1;
  std::vector<int> slot(n + 1);
  slot[0] = P->seed_buf;
  for (int s = 1; s <= n; ++s) slot[s] = n - s;   // original buffer ids = element index
  auto is_vec = [&](int id) { return id >= 0 && (P->bufs[id].kind == B_VEC || P->bufs[id].kind == B_SEED); };
  auto new_vec = [&](long long dim) {
    Buf b;
    b.kind = B_VEC;
    b.size = dim;
    P->bufs.push_back(b);
    return (int)P->bufs.size() - 1;
  };
  int phase = BPPSA_CSR_STEP_UP, level = 0;   // where the next op sits (static analysis)
  auto spmv = [&](int mat, int vec) {   // returns new vector buffer = mat * vec
    const HCSR& m = P->pats[P->bufs[mat].pat];
    const int out = new_vec(m.rows);
    P->ops.push_back(Op{OP_SPMV, out, mat, vec, -1});
    P->spmv_nnz += m.nnz();
    P->steps.push_back(bppsa_csr_step{BPPSA_CSR_STEP_MV, phase, level, 0, 2 * m.nnz(), 2ll * m.rows * m.cols});
    return out;
  };
  // up-sweep levels d < u (Alg. 1 lines 1-5): a[r] <- a[r] a[l]
  for (int d = 0; d < u; ++d) {
    level = d;
    for (long long i = 0; i <= (long long)n - (1ll << d); i += (1ll << (d + 1))) {
      const int l = (int)(i + (1ll << d) - 1), r = (int)std::min<long long>(i + (1ll << (d + 1)) - 1, n);
      if (is_vec(slot[l])) {
        slot[r] = spmv(slot[r], slot[l]);
      } else if (symbolic) {
        const Buf& bl = P->bufs[slot[r]];   // left factor of the product a[r] a[l]
        const Buf& br = P->bufs[slot[l]];
        HCSR prod;
        long long pairs = 0;
        if (!symbolic_product(P->pats[bl.pat], P->pats[br.pat], &prod, &pairs))
          return fail(BPPSA_ERR_NOT_SUPPORTED, "symbolic product at level " + std::to_string(d) +
                                                   " exceeds the bit-row memory bound or 2^31 output entries");
        P->contributions += pairs;
        {
          const HCSR& A = P->pats[bl.pat];
          const HCSR& Bm = P->pats[br.pat];
          P->steps.push_back(bppsa_csr_step{BPPSA_CSR_STEP_MM, phase, level, 0, 2 * pairs,
                                            2ll * A.rows * A.cols * Bm.cols});
        }
        Buf pb;
        pb.kind = B_PROD;
        pb.size = prod.nnz();
        pb.deps = bl.deps | br.deps;
        P->pats.push_back(std::move(prod));
        pb.pat = (int)P->pats.size() - 1;
        P->bufs.push_back(pb);
        const int out = (int)P->bufs.size() - 1;
        P->ops.push_back(Op{OP_SPGEMM, out, slot[r], slot[l], -1});
        slot[r] = out;
      } else {
        HostProduct hp;
        const Buf& bl = P->bufs[slot[r]];   // left factor of the product a[r] a[l]
        const Buf& br = P->bufs[slot[l]];
        if (!plan_product(P->pats[bl.pat], P->pats[br.pat], cap - P->contributions, &hp))
          return fail(BPPSA_ERR_NOT_SUPPORTED, "schedule too dense: the up-sweep product at level " + std::to_string(d) +
                                                   " exceeds the contribution cap (reduce up_levels)");
        DevPlan dp;
        dp.nnz_out = hp.out.nnz();
        dp.contrib = (long long)hp.lpos.size();
        cudaError_t e = upload(&dp.cptr, hp.cptr);
        if (e == cudaSuccess) e = upload(&dp.lpos, hp.lpos);
        if (e == cudaSuccess) e = upload(&dp.rpos, hp.rpos);
        P->plans.push_back(dp);
        if (e != cudaSuccess) return cuda_status(e, "plan upload");
        P->contributions += dp.contrib;
        {
          const HCSR& A = P->pats[bl.pat];
          const HCSR& Bm = P->pats[br.pat];
          P->steps.push_back(bppsa_csr_step{BPPSA_CSR_STEP_MM, phase, level, 0, 2 * dp.contrib,
                                            2ll * A.rows * A.cols * Bm.cols});
        }
        P->pats.push_back(std::move(hp.out));
        Buf pb;
        pb.kind = B_PROD;
        pb.pat = (int)P->pats.size() - 1;
        pb.size = dp.nnz_out;
        pb.deps = bl.deps | br.deps;
        P->bufs.push_back(pb);
        const int out = (int)P->bufs.size() - 1;
        P->ops.push_back(Op{OP_SPGEMM, out, slot[r], slot[l], (int)P->plans.size() - 1});
        slot[r] = out;
      }
    }
  }
  // bridge (reading 19): fold the 2^u-block aggregates onto the seed,
  // depositing the prefix of every 2^dl-block at that block's right end
  {
    const long long bs = 1ll << u, bd = 1ll << dl;
    const long long last = (n / bd) * bd;
    int Pv = IDENT;
    std::vector<std::pair<int, int>> deposits;
    phase = BPPSA_CSR_STEP_BRIDGE;
    for (long long s = 0; s <= last; s += bs) {
      if (s % bd == 0) deposits.push_back({(int)std::min<long long>(s + bd - 1, n), Pv});
      if (s + bs <= last) {
        level = (int)(s / bs);
        const int agg = slot[(int)std::min<long long>(s + bs - 1, n)];
        Pv = (Pv == IDENT) ? agg : spmv(agg, Pv);
      }
    }
    for (auto& dp : deposits) slot[dp.first] = dp.second;
  }
  // down-sweep levels d < dl with the operand reversal (Alg. 1 line 13)
  phase = BPPSA_CSR_STEP_DOWN;
  for (int d = dl - 1; d >= 0; --d) {
    level = d;
    for (long long i = 0; i <= (long long)n - (1ll << d); i += (1ll << (d + 1))) {
      const int l = (int)(i + (1ll << d) - 1), r = (int)std::min<long long>(i + (1ll << (d + 1)) - 1, n);
      const int T = slot[l];
      slot[l] = slot[r];
      slot[r] = (slot[r] == IDENT) ? T : spmv(T, slot[r]);
    }
  }
  // exclusive outputs: slot s >= 1 holds dl/dx_{n-s+1}
  P->out_buf.assign(n + 1, -1);
  for (int s = 1; s <= n; ++s) {
    if (!is_vec(slot[s])) return fail(BPPSA_ERR_PLAN, "internal: slot " + std::to_string(s) + " is not a vector");
    P->out_buf[n - s + 1] = slot[s];
  }
  phase = BPPSA_CSR_STEP_EXTRA;
  level = 0;
  P->out_buf[0] = spmv(0, P->out_buf[1]);   // inclusive extra J_1^T dl/dx_1
  // critical path of the level-synchronous schedule (DESIGN reading 23): the
  // costliest op of every up-/down-sweep level; every bridge op and the extra
  // (serial)
  for (size_t a = 0; a < P->steps.size(); ++a) {
    bppsa_csr_step& st = P->steps[a];
    if (st.phase == BPPSA_CSR_STEP_BRIDGE || st.phase == BPPSA_CSR_STEP_EXTRA) {
      st.critical = 1;
      continue;
    }
    bool top = true;
    for (size_t b = 0; b < P->steps.size() && top; ++b) {
      const bppsa_csr_step& o = P->steps[b];
      if (b == a || o.phase != st.phase || o.level != st.level) continue;
      if (o.flops > st.flops || (o.flops == st.flops && b < a)) top = false;
    }
    st.critical = top ? 1 : 0;
  }
  // the BP baseline: one gradient operator J_k^T per element, serial
  for (int k = n; k >= 1; --k) {
    const HCSR& m = P->pats[k - 1];
    P->steps.push_back(bppsa_csr_step{BPPSA_CSR_STEP_MV, BPPSA_CSR_STEP_BP, k, 1, 2 * m.nnz(), 2ll * m.rows * m.cols});
  }
  // device copies of every pattern used by an SpMV
  P->dpats.resize(P->pats.size());
  for (const Op& op : P->ops) {
    if (symbolic) break;
    if (op.kind != OP_SPMV) continue;
    const int pid = P->bufs[op.a].pat;
    if (P->dpats[pid].indptr) continue;
    cudaError_t e = upload(&P->dpats[pid].indptr, P->pats[pid].indptr);
    if (e == cudaSuccess) e = upload(&P->dpats[pid].indices, P->pats[pid].indices);
    if (e != cudaSuccess) return cuda_status(e, "pattern upload");
  }
  *out_plan = P.release();
  return BPPSA_OK;
}

bppsa_status bppsa_csr_plan_create(const bppsa_csr_pattern* chain, int n, int up_levels, int down_levels,
                                   long long max_contributions, bppsa_csr_plan** out_plan) {
  NvtxRange nvtx_("bppsa_csr_plan_create");
  return csr_plan_create_impl(chain, n, up_levels, down_levels, max_contributions, false, out_plan);
}

bppsa_status bppsa_csr_plan_create_symbolic(const bppsa_csr_pattern* chain, int n, int up_levels, int down_levels,
                                            bppsa_csr_plan** out_plan) {
  NvtxRange nvtx_("bppsa_csr_plan_create_symbolic");
  return csr_plan_create_impl(chain, n, up_levels, down_levels, 0, true, out_plan);
}

void bppsa_csr_plan_destroy(bppsa_csr_plan* plan) { delete plan; }

bppsa_status bppsa_csr_plan_workspace_size(const bppsa_csr_plan* plan, int B, const int* batched, size_t* bytes) {
  if (!plan || !bytes || B < 1) return fail(BPPSA_ERR_INVALID_ARGUMENT, "bad arguments");
  if (plan->symbolic) return fail(BPPSA_ERR_NOT_SUPPORTED, "a symbolic plan has no numeric scan");
  std::vector<size_t> off;
  layout(*plan, B, batched, &off, bytes);
  return BPPSA_OK;
}

bppsa_status bppsa_csr_plan_info(const bppsa_csr_plan* plan, long long* contributions, long long* spmv_nnz,
                                 int* n_kernels) {
  if (!plan) return fail(BPPSA_ERR_INVALID_ARGUMENT, "plan is NULL");
  if (contributions) *contributions = plan->contributions;
  if (spmv_nnz) *spmv_nnz = plan->spmv_nnz;
  if (n_kernels) *n_kernels = (int)plan->ops.size() + 1 + (plan->n + 1);
  return BPPSA_OK;
}

bppsa_status bppsa_csr_plan_steps(const bppsa_csr_plan* plan, bppsa_csr_step* steps, int capacity, int* n_steps) {
  if (!plan || !n_steps || capacity < 0 || (capacity > 0 && !steps))
    return fail(BPPSA_ERR_INVALID_ARGUMENT, "bad arguments");
  *n_steps = (int)plan->steps.size();
  const int c = std::min(capacity, *n_steps);
  for (int a = 0; a < c; ++a) steps[a] = plan->steps[a];
  return BPPSA_OK;
}

bppsa_status bppsa_csr_scan(const bppsa_csr_plan* plan, int B, const float* const* data, const int* batched,
                            const float* seed, float* const* grads, void* ws, size_t ws_bytes, void* stream) {
  NvtxRange nvtx_("bppsa_csr_scan");
  if (!plan || !data || !seed || !grads || B < 1) return fail(BPPSA_ERR_INVALID_ARGUMENT, "bad arguments");
  if (plan->symbolic) return fail(BPPSA_ERR_NOT_SUPPORTED, "a symbolic plan has no numeric scan");
  const bppsa_csr_plan& P = *plan;
  for (int k = 0; k < P.n; ++k)
    if (!data[k]) return fail(BPPSA_ERR_INVALID_ARGUMENT, "data[" + std::to_string(k) + "] is NULL");
  std::vector<size_t> off;
  size_t need;
  layout(P, B, batched, &off, &need);
  if (ws_bytes < need || (need && !ws)) return fail(BPPSA_ERR_WORKSPACE, "workspace too small: need " + std::to_string(need));
  cudaStream_t st = (cudaStream_t)stream;
  char* w = static_cast<char*>(ws);
  auto ptr = [&](int id) -> float* {
    const Buf& b = P.bufs[id];
    if (b.kind == B_ORIG) return const_cast<float*>(data[b.elem]);
    return reinterpret_cast<float*>(w + off[id]);
  };
  // seed -> sample-minor
  const long long sdim = P.bufs[P.seed_buf].size;
  transpose_bd<<<blocks_for(sdim * B), 256, 0, st>>>(seed, ptr(P.seed_buf), sdim, B, 1);
  for (const Op& op : P.ops) {
    if (op.kind == OP_SPGEMM) {
      const DevPlan& dp = P.plans[op.plan];
      const int ob = buf_batched(P, op.out, batched) ? B : 1;
      if (dp.nnz_out == 0) continue;
      spgemm_kernel<<<blocks_for(dp.nnz_out * ob), 256, 0, st>>>(
          dp.cptr, dp.lpos, dp.rpos, ptr(op.a), buf_batched(P, op.a, batched), ptr(op.b),
          buf_batched(P, op.b, batched), ptr(op.out), ob, dp.nnz_out, B);
    } else {
      const HCSR& m = P.pats[P.bufs[op.a].pat];
      const DevPat& dpt = P.dpats[P.bufs[op.a].pat];
      spmv_kernel<<<blocks_for((long long)m.rows * B), 256, 0, st>>>(dpt.indptr, dpt.indices, ptr(op.a),
                                                                     buf_batched(P, op.a, batched), ptr(op.b),
                                                                     ptr(op.out), m.rows, B);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_status(e, "csr scan launch");
  }
  for (int k = 0; k <= P.n; ++k) {
    if (!grads[k]) continue;
    const int id = P.out_buf[k];
    const long long dim = P.bufs[id].size;
    transpose_bd<<<blocks_for(dim * B), 256, 0, st>>>(ptr(id), grads[k], dim, B, 0);
  }
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? BPPSA_OK : cuda_status(e, "csr output launch");
}

// ------------------------------------------------------------------ builders
bppsa_status bppsa_csr_conv3x3_pattern(int ci, int co, int h, int w, const float* weights_host, int drop_zero,
                                       long long* nnz, long long* indptr, int* indices, int* tap) {
  if (ci < 1 || co < 1 || h < 1 || w < 1 || !nnz) return fail(BPPSA_ERR_INVALID_ARGUMENT, "bad conv spec");
  if (drop_zero && !weights_host) return fail(BPPSA_ERR_INVALID_ARGUMENT, "drop_zero needs weights_host");
  // row (c_i, y_i, x_i); entries (c_o, o_y, o_x) in ascending output index:
  // output (c_o, y_i + o_y, x_i + o_x), weight W[c_o][c_i][1 - o_y][1 - o_x]
  long long p = 0;
  for (int c = 0; c < ci; ++c)
    for (int y = 0; y < h; ++y)
      for (int x = 0; x < w; ++x) {
        const long long row = ((long long)c * h + y) * w + x;
        if (indptr) indptr[row] = p;
        for (int o = 0; o < co; ++o)
          for (int oy = -1; oy <= 1; ++oy)
            for (int ox = -1; ox <= 1; ++ox) {
              const int yo = y + oy, xo = x + ox;
              if (yo < 0 || yo >= h || xo < 0 || xo >= w) continue;
              const int t = ((o * ci + c) * 3 + (1 - oy)) * 3 + (1 - ox);
              if (drop_zero && weights_host[t] == 0.f) continue;
              if (indices) indices[p] = (o * h + yo) * w + xo;
              if (tap) tap[p] = t;
              ++p;
            }
      }
  if (indptr) indptr[(long long)ci * h * w] = p;
  *nnz = p;
  return BPPSA_OK;
}

bppsa_status bppsa_csr_conv_data(long long nnz, const int* tap, const float* weights, float* data, void* stream) {
  if (nnz < 0 || (nnz > 0 && (!tap || !weights || !data))) return fail(BPPSA_ERR_INVALID_ARGUMENT, "bad arguments");
  if (nnz == 0) return BPPSA_OK;
  gather_kernel<<<blocks_for(nnz), 256, 0, (cudaStream_t)stream>>>(tap, weights, data, nnz);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? BPPSA_OK : cuda_status(e, "conv data");
}

bppsa_status bppsa_csr_relu_data(long long d, int B, const float* x, float* data, void* stream) {
  if (d < 1 || B < 1 || !x || !data) return fail(BPPSA_ERR_INVALID_ARGUMENT, "bad arguments");
  relu_data_kernel<<<blocks_for(d * B), 256, 0, (cudaStream_t)stream>>>(x, data, d, B);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? BPPSA_OK : cuda_status(e, "relu data");
}

bppsa_status bppsa_csr_conv3x3_build_size(int ci, int co, int h, int w, int drop_zero, long long* max_nnz,
                                          size_t* ws_bytes) {
  if (ci < 1 || co < 1 || h < 1 || w < 1) return fail(BPPSA_ERR_INVALID_ARGUMENT, "bad conv spec");
  const long long NY = (h == 1) ? 1 : 3ll * h - 2, NX = (w == 1) ? 1 : 3ll * w - 2;
  const long long rows = (long long)ci * h * w;
  if (max_nnz) *max_nnz = (long long)ci * co * NY * NX;
  if (ws_bytes) {
    size_t tmp = 0;
    if (drop_zero) {
      cudaError_t e = cub::DeviceScan::InclusiveSum(nullptr, tmp, (const long long*)nullptr, (long long*)nullptr,
                                                    (int)rows);
      if (e != cudaSuccess) return cuda_status(e, "cub scan size");
      tmp = align256(tmp) + align256((size_t)rows * sizeof(long long));
    }
    *ws_bytes = tmp;
  }
  return BPPSA_OK;
}

bppsa_status bppsa_csr_conv3x3_build(int ci, int co, int h, int w, const float* weights, int drop_zero,
                                     long long* indptr, int* indices, int* tap, float* data, void* ws,
                                     size_t ws_bytes, void* stream) {
  if (ci < 1 || co < 1 || h < 1 || w < 1 || !indptr || !indices) return fail(BPPSA_ERR_INVALID_ARGUMENT, "bad conv spec");
  if ((drop_zero || data) && !weights) return fail(BPPSA_ERR_INVALID_ARGUMENT, "drop_zero / data need weights");
  if ((long long)co * h * w > (1ll << 31) - 1) return fail(BPPSA_ERR_INVALID_ARGUMENT, "column index exceeds int32");
  size_t need = 0;
  bppsa_status s = bppsa_csr_conv3x3_build_size(ci, co, h, w, drop_zero, nullptr, &need);
  if (s != BPPSA_OK) return s;
  if (ws_bytes < need || (need && !ws)) return fail(BPPSA_ERR_WORKSPACE, "workspace too small: need " + std::to_string(need));
  cudaStream_t st = (cudaStream_t)stream;
  const long long rows = (long long)ci * h * w;
  cudaError_t e;
  if (!drop_zero) {
    conv_indptr_kernel<<<blocks_for(rows + 1), 256, 0, st>>>(ci, co, h, w, indptr);
  } else {
    long long* cnt = reinterpret_cast<long long*>(static_cast<char*>(ws));
    void* tmp = static_cast<char*>(ws) + align256((size_t)rows * sizeof(long long));
    size_t tmp_bytes = need - align256((size_t)rows * sizeof(long long));
    conv_count_kernel<<<blocks_for(rows * 32), 256, 0, st>>>(ci, co, h, w, weights, cnt);
    e = cudaMemsetAsync(indptr, 0, sizeof(long long), st);
    if (e != cudaSuccess) return cuda_status(e, "indptr[0]");
    e = cub::DeviceScan::InclusiveSum(tmp, tmp_bytes, cnt, indptr + 1, (int)rows, st);
    if (e != cudaSuccess) return cuda_status(e, "row-count scan");
  }
  conv_fill_kernel<<<blocks_for(rows * 32), 256, 0, st>>>(ci, co, h, w, weights, drop_zero, indptr, indices, tap, data);
  e = cudaGetLastError();
  return e == cudaSuccess ? BPPSA_OK : cuda_status(e, "conv build");
}

bppsa_status bppsa_csr_maxpool_build(int c, int h, int w, long long* indptr, int* indices, void* stream) {
  if (c < 1 || h < 2 || w < 2 || (h & 1) || (w & 1) || !indptr || !indices)
    return fail(BPPSA_ERR_INVALID_ARGUMENT, "bad max-pool spec (even h, w >= 2)");
  const long long d = (long long)c * h * w;
  pool_pattern_kernel<<<blocks_for(d + 1), 256, 0, (cudaStream_t)stream>>>(c, h, w, indptr, indices);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? BPPSA_OK : cuda_status(e, "maxpool build");
}

bppsa_status bppsa_csr_identity_build(long long d, long long* indptr, int* indices, void* stream) {
  if (d < 1 || d > (1ll << 31) - 1 || !indptr || !indices) return fail(BPPSA_ERR_INVALID_ARGUMENT, "bad size");
  identity_pattern_kernel<<<blocks_for(d + 1), 256, 0, (cudaStream_t)stream>>>(d, indptr, indices);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? BPPSA_OK : cuda_status(e, "identity build");
}

bppsa_status bppsa_csr_maxpool_pattern(int c, int h, int w, long long* indptr, int* indices) {
  if (c < 1 || h < 2 || w < 2 || (h & 1) || (w & 1) || !indptr || !indices)
    return fail(BPPSA_ERR_INVALID_ARGUMENT, "bad max-pool spec (even h, w >= 2)");
  const int ho = h / 2, wo = w / 2;
  for (long long i = 0; i < (long long)c * h * w; ++i) {
    const int cc = (int)(i / (h * w)), rem = (int)(i % (h * w)), y = rem / w, x = rem % w;
    indptr[i] = i;
    indices[i] = (cc * ho + y / 2) * wo + x / 2;
  }
  indptr[(long long)c * h * w] = (long long)c * h * w;
  return BPPSA_OK;
}

bppsa_status bppsa_csr_maxpool_data(int c, int h, int w, int B, const long long* pool_idx, float* data,
                                    void* stream) {
  if (c < 1 || h < 2 || w < 2 || B < 1 || !pool_idx || !data) return fail(BPPSA_ERR_INVALID_ARGUMENT, "bad arguments");
  maxpool_data_kernel<<<blocks_for((long long)c * h * w * B), 256, 0, (cudaStream_t)stream>>>(pool_idx, data, c, h,
                                                                                               w, B);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? BPPSA_OK : cuda_status(e, "maxpool data");
}

}  // extern "C"
