// api.cu — the C-ABI of libbppsa (include/bppsa.h): validation, workspace
// planning and launch sequencing of the blocked Blelloch scan.
//
// Level structure (BPPSA_SCAN_BLOCKED).  Level 0 is the scan array itself
// (n_0 = S = T + head slots, leaves implicit or DENSE).  Level l+1 holds the
// aggregates of the blocks of C_l consecutive slots of level l
// (n_{l+1} = ceil(n_l / C_l)).  The up-sweep folds blocks bottom-up; the
// down-sweep walks every block from its exclusive prefix (the output of the
// level above) — Blelloch's Theta(n/p + log p) schedule with every
// matrix-matrix product in the up-sweep and only GEMVs in the down-sweep
// (P:135).  Single-GPU: folding stops when a level fits one block; that level
// is walked from the symbolic identity (root reset).  Shards fold to
// one aggregate per sample, exchange, and walk from the received carry.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <map>
#include <string>
#include <utility>

#include "common.cuh"

namespace bppsa {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

bppsa_status fail(bppsa_status s, const std::string& msg) {
  g_last_error = msg;
  return s;
}

cudaError_t smem_attr_once(const void* kernel, int bytes) {
  // the default allows 48 KB; never LOWER a limit set earlier (a smaller value
  // would make later, larger launches of the same kernel fail)
  if (bytes <= 48 * 1024) return cudaSuccess;
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  auto it = done.find({kernel, dev});
  if (it != done.end() && it->second >= bytes) return cudaSuccess;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done[{kernel, dev}] = bytes;
  return e;
}

bppsa_status cuda_status(cudaError_t e, const char* where) {
  g_last_error = std::string(where) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
  return BPPSA_ERR_CUDA;
}

namespace {

constexpr int kMaxLevels = 48;
constexpr size_t kAlign = 256;

size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

bool is_device_ptr(const void* p) {
  if (p == nullptr) return false;
  cudaPointerAttributes attr;
  cudaError_t e = cudaPointerGetAttributes(&attr, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged;
}

#define REQUIRE_DEV(p, name)                                                               \
  do {                                                                                     \
    if (!is_device_ptr(p))                                                                 \
      return fail(BPPSA_ERR_INVALID_ARGUMENT, std::string(name) + " must be a device pointer"); \
  } while (0)

// Per-call launch instrumentation (bppsa_scan_opts.events / launches).
struct Tracer {
  cudaEvent_t* ev = nullptr;
  int n_ev = 0;
  int k = 0;
  void begin(cudaStream_t st) {
    if (ev && 2 * k + 1 < n_ev) cudaEventRecord(ev[2 * k], st);
  }
  void end(cudaStream_t st) {
    if (ev && 2 * k + 1 < n_ev) cudaEventRecord(ev[2 * k + 1], st);
    ++k;
  }
};

Tracer tracer_from(const bppsa_scan_opts* o) {
  Tracer t;
  if (o && o->events) {
    t.ev = reinterpret_cast<cudaEvent_t*>(o->events);
    t.n_ev = o->n_events;
  }
  return t;
}

void report_launches(const bppsa_scan_opts* o, const Tracer& t) {
  if (o && o->launches) *o->launches = t.k;
}

int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
  }
  return n;
}

// Level-0 engine of the fused RNN leaves (bppsa_scan_opts.leaf_impl):
// kCuda (FFMA), kF16 (3xFP16 fold, 16 <= H <= 64, H % 4 == 0), kTf32 (3xTF32
// fold, H = 64), kInt8 (exact-integer fold and walk, H = 64).  Auto takes
// kInt8 for the tanh RNN at H = 64: below, the fold is latency-bound (C2,
// H = 20: 0.45 ms on either engine) and the CUDA-core kernel keeps ~100x more
// chains in flight.
enum LeafEngine { kCuda = 0, kF16 = 1, kTf32 = 2, kInt8 = 3 };
bool tensor_fold_ok(const bppsa_jac& j, int leaf_impl) {
  if (j.kind != BPPSA_JAC_RNN_TANH) return false;
  if (leaf_impl == 3 || leaf_impl == 4) return j.H == 64;
  return j.H >= 16 && j.H <= 64 && j.H % 4 == 0;
}
LeafEngine leaf_engine(const bppsa_jac& j, int leaf_impl) {
  switch (leaf_impl) {
    case 0: return (j.kind == BPPSA_JAC_RNN_TANH && j.H == 64) ? kInt8 : kCuda;
    case 2: return tensor_fold_ok(j, 2) ? kF16 : kCuda;
    case 3: return tensor_fold_ok(j, 3) ? kTf32 : kCuda;
    case 4: return tensor_fold_ok(j, 4) ? kInt8 : kCuda;
    default: return kCuda;
  }
}
// the 3xFP16 TMA walk (H = 64) serves kF16 and kTf32
bool use_tensor_walk(const bppsa_jac& j, int leaf_impl) {
  const LeafEngine e = leaf_engine(j, leaf_impl);
  return (e == kF16 || e == kTf32) && j.H == 64;
}

struct Plan {
  int leaf_impl = 0;
  int L = 0;
  long long n[kMaxLevels + 2] = {};
  int C[kMaxLevels + 2] = {};
  size_t agg_off[kMaxLevels + 2] = {}, out_off[kMaxLevels + 2] = {};
  size_t vec_off[kMaxLevels + 2] = {};   // affine vector parts [B][n_l][H] (l >= 1)
  size_t dense_off = 0, carry_off = 0, aseed_off = 0, total = 0;
  bool has_dense = false;
};

int default_block0(const bppsa_jac& j) { return j.H <= 32 ? 16 : 64; }
int default_block(const bppsa_jac& j) { return j.H <= 32 ? 16 : 32; }

bppsa_status check_jac(const bppsa_jac* j, bool need_ptrs = true) {
  if (!j) return fail(BPPSA_ERR_INVALID_ARGUMENT, "jac is NULL");
  if (j->T < 1 || j->B < 1) return fail(BPPSA_ERR_INVALID_ARGUMENT, "T and B must be >= 1 (reading 5)");
  if (j->H < 1 || j->H > BPPSA_MAX_H) return fail(BPPSA_ERR_INVALID_ARGUMENT, "H must be in [1, 64]");
  if (j->kind == BPPSA_JAC_DENSE) {
    if (need_ptrs) REQUIRE_DEV(j->JT, "jac.JT");
  } else if (j->kind == BPPSA_JAC_RNN_TANH) {
    if (need_ptrs) {
      REQUIRE_DEV(j->h, "jac.h");
      REQUIRE_DEV(j->W_hh, "jac.W_hh");
    }
  } else if (j->kind == BPPSA_JAC_GRU) {
    if (j->H > 32)
      return fail(BPPSA_ERR_NOT_SUPPORTED, "fused GRU leaves need H <= 32; materialise (JT_out) for larger H");
    if (need_ptrs) {
      REQUIRE_DEV(j->h_prev, "jac.h_prev");
      REQUIRE_DEV(j->r, "jac.r");
      REQUIRE_DEV(j->z, "jac.z");
      REQUIRE_DEV(j->n, "jac.n");
      REQUIRE_DEV(j->M, "jac.M");
      REQUIRE_DEV(j->W_hh3, "jac.W_hh3");
    }
  } else {
    return fail(BPPSA_ERR_INVALID_ARGUMENT, "unknown jac.kind");
  }
  return BPPSA_OK;
}

bppsa_status get_opts(const bppsa_jac& j, const bppsa_scan_opts* o, int* mode, int* C0, int* C) {
  *mode = o ? o->mode : BPPSA_SCAN_BLOCKED;
  *C0 = (o && o->block0 > 0) ? o->block0 : default_block0(j);
  *C = (o && o->block > 0) ? o->block : default_block(j);
  if (*mode != BPPSA_SCAN_BLOCKED && *mode != BPPSA_SCAN_ALG1 && *mode != BPPSA_SCAN_LINEAR &&
      *mode != BPPSA_SCAN_HYBRID)
    return fail(BPPSA_ERR_INVALID_ARGUMENT, "unknown scan mode");
  if (*C0 < 2 || *C < 2) return fail(BPPSA_ERR_INVALID_ARGUMENT, "block lengths must be >= 2");
  if ((*mode == BPPSA_SCAN_ALG1 || *mode == BPPSA_SCAN_HYBRID) && j.kind != BPPSA_JAC_DENSE)
    return fail(BPPSA_ERR_NOT_SUPPORTED, "ALG1 and HYBRID modes run on materialised (DENSE) leaves");
  if (*mode == BPPSA_SCAN_HYBRID) {
    const int L = (int)(64 - __builtin_clzll((unsigned long long)j.T));   // ceil(log2(n+1)), n = T
    const int u = o->up_levels, dl = o->down_levels;
    if (u < 0 || u > std::max(L - 1, 0) || (dl != u && dl != u + 1) || dl > L)
      return fail(BPPSA_ERR_INVALID_ARGUMENT,
                  "HYBRID needs 0 <= up_levels <= L-1, down_levels in {u, u+1}, down_levels <= L");
  }
  return BPPSA_OK;
}

bppsa_status make_plan(const bppsa_jac& j, int head, const bppsa_scan_opts* opts, bool need_total, Plan* p) {
  int mode, C0, C;
  bppsa_status s = get_opts(j, opts, &mode, &C0, &C);
  if (s != BPPSA_OK) return s;
  const long long S = (long long)j.T + head;
  const size_t HH = (size_t)j.H * j.H, B = (size_t)j.B;
  size_t off = 0;
  p->leaf_impl = opts ? opts->leaf_impl : 0;
  if (p->leaf_impl < 0 || p->leaf_impl > 4) return fail(BPPSA_ERR_INVALID_ARGUMENT, "leaf_impl must be in 0..4");
  if (p->leaf_impl >= 2 && !tensor_fold_ok(j, p->leaf_impl))
    return fail(BPPSA_ERR_NOT_SUPPORTED,
                "tensor-core leaf fold: tanh RNN with 16 <= H <= 64, H % 4 == 0 (3xTF32 and int8: H = 64)");
  const bool tree = (mode == BPPSA_SCAN_ALG1 || mode == BPPSA_SCAN_HYBRID);
  p->has_dense = (j.kind == BPPSA_JAC_DENSE) && !tree;
  if (p->has_dense) {
    p->dense_off = off;
    off = align_up(off + (size_t)j.T * B * HH * sizeof(float));
  }
  if (tree) {
    p->L = 0;
    p->dense_off = off;
    off = align_up(off + (size_t)(j.T + 1) * B * HH * sizeof(float));
    p->total = off;
    return BPPSA_OK;
  }
  p->n[0] = S;
  int l = 0;
  if (mode == BPPSA_SCAN_LINEAR) {
    p->C[0] = (int)std::min<long long>(S, 1ll << 30);
  } else {
    while (true) {
      const int Cl = (l == 0) ? C0 : C;
      p->C[l] = Cl;
      if (!need_total && p->n[l] <= Cl) break;
      if (need_total && l > 0 && p->n[l] == 1) break;
      if (l >= kMaxLevels) return fail(BPPSA_ERR_INVALID_ARGUMENT, "too many levels");
      p->n[l + 1] = (p->n[l] + Cl - 1) / Cl;
      ++l;
    }
  }
  p->L = l;
  for (int k = 1; k <= p->L; ++k) {
    p->agg_off[k] = off;
    off = align_up(off + B * (size_t)p->n[k] * HH * sizeof(float));
    p->out_off[k] = off;
    off = align_up(off + B * (size_t)p->n[k] * j.H * sizeof(float));
    p->vec_off[k] = off;
    off = align_up(off + B * (size_t)p->n[k] * j.H * sizeof(float));
  }
  p->carry_off = off;
  off = align_up(off + B * j.H * sizeof(float));
  p->aseed_off = off;
  off = align_up(off + B * j.H * sizeof(float));
  p->total = off;
  return BPPSA_OK;
}

LeafArgs leaf_args(const bppsa_jac& j, int head, const float* seed) {
  LeafArgs a{};
  a.seg = Seg{j.T, j.B, j.H, head};
  a.kind = j.kind;
  if (j.kind == BPPSA_JAC_RNN_TANH) {
    a.h = j.h;
    a.W = j.W_hh;
  } else {
    a.W = j.W_hh3;
    a.hp = j.h_prev;
    a.r = j.r;
    a.z = j.z;
    a.n = j.n;
    a.M = j.M;
  }
  a.seed = seed;
  return a;
}

// level-0 accessor over the transposed DENSE copy (column-major per matrix)
MatAcc dense_acc(const bppsa_jac& j, int head, const float* JTc, const float* seed) {
  const long long HH = (long long)j.H * j.H;
  MatAcc A{};
  const long long t0 = head ? j.T : (long long)j.T - 1;   // time of slot 0 (+ formally)
  A.base = JTc + t0 * j.B * HH;
  A.slot_stride = -(long long)j.B * HH;
  A.batch_stride = HH;
  A.head_vec = seed;
  A.head_bstride = j.H;
  return A;
}

MatAcc level_acc(const Plan& p, char* ws, int l, int H) {
  const long long HH = (long long)H * H;
  MatAcc A{};
  A.base = reinterpret_cast<const float*>(ws + p.agg_off[l]);
  A.slot_stride = HH;
  A.batch_stride = p.n[l] * HH;
  A.head_vec = A.base;
  A.head_bstride = p.n[l] * HH;
  return A;
}

float* level_out(const Plan& p, char* ws, int l) { return reinterpret_cast<float*>(ws + p.out_off[l]); }
float* level_vec(const Plan& p, char* ws, int l) { return reinterpret_cast<float*>(ws + p.vec_off[l]); }
VecAcc level_addv(const Plan& p, char* ws, int l, int H) {   // vector parts of level l (affine)
  VecAcc v;
  v.base = level_vec(p, ws, l);
  v.slot_stride = H;
  v.batch_stride = p.n[l] * (long long)H;
  v.time_mode = 0;
  return v;
}
VecAcc leaf_addv(const float* e) {
  VecAcc v;
  v.base = e;
  v.time_mode = 1;
  return v;
}
float* level_agg(const Plan& p, char* ws, int l) { return reinterpret_cast<float*>(ws + p.agg_off[l]); }

// Up-sweep: levels 0 .. L-1 fold into levels 1 .. L.  `top_out` (nullable)
// replaces the storage of level L (used by shard_up to write the aggregate
// straight into the caller's buffer).
bppsa_status run_up(const bppsa_jac& j, int head, const float* seed, const Plan& p, char* ws, float* top_out,
                    cudaStream_t st, Tracer& tr, const float* e_aff = nullptr, const Publish* pub = nullptr,
                    bool* published = nullptr) {
  if (published) *published = false;
  const int H = j.H, B = j.B;
  const Seg seg{j.T, j.B, j.H, head};
  for (int l = 0; l < p.L; ++l) {
    float* dst = (l + 1 == p.L && top_out) ? top_out : level_agg(p, ws, l + 1);
    cudaError_t e;
    tr.begin(st);
    if (l == 0 && j.kind != BPPSA_JAC_DENSE) {
      const LeafArgs la = leaf_args(j, head, seed);
      const LeafEngine eng = leaf_engine(j, p.leaf_impl);
      if (eng == kF16 || eng == kInt8) {
        // tensor-core fold of every block; the head block is folded as the
        // matrix of its leaves with all other blocks, then applied to the seed
        e = eng == kInt8 ? launch_tc_fold_i8(la, p.C[0], dst, p.n[1], 0, num_sms(), st)
                         : launch_tc_leaf_up(la, p.C[0], dst, p.n[1], 0, num_sms(), st, 0);
        if (e == cudaSuccess && head) {                  // its own traced launch
          tr.end(st);
          tr.begin(st);
          e = launch_head_apply(dst, p.n[1] * (long long)H * H, seed, B, H, st);
        }
      } else if (eng == kTf32) {
        // head block (a GEMV chain from the seed) on the CUDA cores, matrix blocks on tcgen05
        e = head ? launch_leaf_up(la, p.C[0], dst, p.n[1], 0, 1, st) : cudaSuccess;
        if (e == cudaSuccess) e = launch_tc_leaf_up(la, p.C[0], dst, p.n[1], head, num_sms(), st, 1);
      } else {
        e = launch_leaf_up(la, p.C[0], dst, p.n[1], 0, p.n[1], st);
      }
    } else {
      const MatAcc A = (l == 0) ? dense_acc(j, head, reinterpret_cast<float*>(ws + p.dense_off), seed)
                                : level_acc(p, ws, l, H);
      const bool top = l + 1 == p.L && pub;       // the carry exchange fused into the top level
      e = launch_fold_up(A, H, B, p.n[l], p.C[l], head, dst, p.n[l + 1], st, top ? pub : nullptr);
      if (top && published) *published = true;
    }
    tr.end(st);
    if (e != cudaSuccess) return cuda_status(e, "up-sweep launch");
    if (e_aff) {
      // affine vector parts m of the level-(l+1) elements (the matrix parts
      // above are unchanged); the head block's vector replaces its slot
      tr.begin(st);
      const long long hb = p.n[l + 1] * (long long)H * H;
      if (l == 0 && j.kind != BPPSA_JAC_DENSE && use_tensor_walk(j, p.leaf_impl) && j.B <= 128 && p.n[1] >= 2 &&
          p.C[0] >= 8)
        e = launch_tc_leaf_down(leaf_args(j, head, seed), p.C[0], nullptr, p.n[1], nullptr, nullptr, num_sms(), st,
                                e_aff, level_vec(p, ws, 1), dst, hb);
      else if (l == 0 && j.kind != BPPSA_JAC_DENSE)
        e = launch_leaf_down(leaf_args(j, head, seed), p.C[0], nullptr, p.n[1], nullptr, nullptr, st, e_aff,
                             level_vec(p, ws, 1), dst, hb);
      else if (l == 0)
        e = launch_walk_down(dense_acc(j, head, reinterpret_cast<float*>(ws + p.dense_off), seed), H, B, p.n[0],
                             p.C[0], head, nullptr, p.n[1], nullptr, 1, seg, nullptr, st, leaf_addv(e_aff),
                             level_vec(p, ws, 1), dst, hb);
      else
        e = launch_walk_down(level_acc(p, ws, l, H), H, B, p.n[l], p.C[l], head, nullptr, p.n[l + 1], nullptr, 0,
                             seg, nullptr, st, level_addv(p, ws, l, H), level_vec(p, ws, l + 1), dst, hb);
      tr.end(st);
      if (e != cudaSuccess) return cuda_status(e, "affine up-sweep launch");
    }
  }
  return BPPSA_OK;
}

// Down-sweep from level `ltop` (whose single block's carry is `carry_top`, or
// the symbolic identity for a head segment) to the leaves.
bppsa_status run_down(const bppsa_jac& j, int head, const float* seed, const Plan& p, char* ws, int ltop,
                      long long ltop_C, const float* carry_top, float* grad_h, float* grad_init,
                      cudaStream_t st, Tracer& tr, const float* e_aff = nullptr) {
  const int H = j.H, B = j.B;
  const Seg seg{j.T, j.B, j.H, head};
  for (int l = ltop; l >= 0; --l) {
    const float* carry = (l == ltop) ? carry_top : level_out(p, ws, l + 1);
    const long long nblk = (l == ltop) ? 1 : p.n[l + 1];
    const int Cl = (l == ltop) ? (int)ltop_C : p.C[l];
    cudaError_t e;
    tr.begin(st);
    if (l == 0 && j.kind != BPPSA_JAC_DENSE) {
      // tcgen05 walk: many short chains (the linear scan's single long chain per
      // sample stays on the CUDA cores; so do single-block segments)
      if (!e_aff && leaf_engine(j, p.leaf_impl) == kInt8 && nblk >= 2)
        e = launch_tc_walk_i8(leaf_args(j, head, seed), Cl, carry, nblk, grad_h, grad_init, num_sms(), st);
      else if (use_tensor_walk(j, p.leaf_impl) && nblk >= 2 && Cl >= 8 && (!e_aff || j.B <= 128))
        e = launch_tc_leaf_down(leaf_args(j, head, seed), Cl, carry, nblk, grad_h, grad_init, num_sms(), st, e_aff);
      else
        e = launch_leaf_down(leaf_args(j, head, seed), Cl, carry, nblk, grad_h, grad_init, st, e_aff);
    } else if (l == 0) {
      const MatAcc A = dense_acc(j, head, reinterpret_cast<float*>(ws + p.dense_off), seed);
      e = launch_walk_down(A, H, B, p.n[0], Cl, head, carry, nblk, grad_h, 1, seg, grad_init, st,
                           e_aff ? leaf_addv(e_aff) : VecAcc{});
    } else {
      e = launch_walk_down(level_acc(p, ws, l, H), H, B, p.n[l], Cl, head, carry, nblk, level_out(p, ws, l), 0,
                           seg, nullptr, st, e_aff ? level_addv(p, ws, l, H) : VecAcc{});
    }
    tr.end(st);
    if (e != cudaSuccess) return cuda_status(e, "down-sweep launch");
  }
  return BPPSA_OK;
}

bppsa_status check_ws(const Plan& p, void* ws, size_t ws_bytes) {
  if (ws_bytes < p.total) return fail(BPPSA_ERR_WORKSPACE, "workspace too small: need " + std::to_string(p.total));
  if (p.total > 0) {
    if (!ws) return fail(BPPSA_ERR_WORKSPACE, "workspace is NULL");
    if (reinterpret_cast<uintptr_t>(ws) % kAlign) return fail(BPPSA_ERR_WORKSPACE, "workspace must be 256-byte aligned");
    if (!is_device_ptr(ws)) return fail(BPPSA_ERR_WORKSPACE, "workspace must be device memory");
  }
  return BPPSA_OK;
}

bppsa_status prepare_dense(const bppsa_jac& j, const Plan& p, char* ws, cudaStream_t st, Tracer& tr) {
  if (!p.has_dense) return BPPSA_OK;
  tr.begin(st);
  cudaError_t e = launch_transpose_dense(j.JT, reinterpret_cast<float*>(ws + p.dense_off), (long long)j.T * j.B,
                                         j.H, st);
  tr.end(st);
  return e == cudaSuccess ? BPPSA_OK : cuda_status(e, "dense transpose launch");
}

}  // namespace
}  // namespace bppsa

using namespace bppsa;

extern "C" {

const char* bppsa_status_str(bppsa_status s) {
  switch (s) {
    case BPPSA_OK: return "BPPSA_OK";
    case BPPSA_ERR_INVALID_ARGUMENT: return "BPPSA_ERR_INVALID_ARGUMENT";
    case BPPSA_ERR_SHAPE: return "BPPSA_ERR_SHAPE";
    case BPPSA_ERR_PLAN: return "BPPSA_ERR_PLAN";
    case BPPSA_ERR_WORKSPACE: return "BPPSA_ERR_WORKSPACE";
    case BPPSA_ERR_CUDA: return "BPPSA_ERR_CUDA";
    case BPPSA_ERR_NCCL: return "BPPSA_ERR_NCCL";
    case BPPSA_ERR_NOT_SUPPORTED: return "BPPSA_ERR_NOT_SUPPORTED";
  }
  return "BPPSA_UNKNOWN_STATUS";
}

const char* bppsa_last_error(void) { return g_last_error.c_str(); }

int bppsa_version(void) { return 100; }

bppsa_status bppsa_jacobians_rnn(int T, int B, int H, const float* h, const float* W_hh, float* JT_out,
                                 bppsa_jac* desc, void* stream) {
  if (!desc) return fail(BPPSA_ERR_INVALID_ARGUMENT, "desc is NULL");
  bppsa_jac j{};
  j.kind = BPPSA_JAC_RNN_TANH;
  j.T = T; j.B = B; j.H = H; j.h = h; j.W_hh = W_hh;
  bppsa_status s = check_jac(&j);
  if (s != BPPSA_OK) return s;
  if (JT_out) {
    REQUIRE_DEV(JT_out, "JT_out");
    cudaError_t e = launch_materialize_rnn(h, W_hh, JT_out, T, B, H, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_status(e, "materialize rnn");
    bppsa_jac d{};
    d.kind = BPPSA_JAC_DENSE;
    d.T = T; d.B = B; d.H = H; d.JT = JT_out;
    *desc = d;
    return BPPSA_OK;
  }
  *desc = j;
  return BPPSA_OK;
}

bppsa_status bppsa_jacobians_gru(int T, int B, int H, const float* h_prev, const float* r, const float* z,
                                 const float* n, const float* M, const float* W_hh3, float* JT_out,
                                 bppsa_jac* desc, void* stream) {
  if (!desc) return fail(BPPSA_ERR_INVALID_ARGUMENT, "desc is NULL");
  bppsa_jac j{};
  j.kind = BPPSA_JAC_GRU;
  j.T = T; j.B = B; j.H = H;
  j.h_prev = h_prev; j.r = r; j.z = z; j.n = n; j.M = M; j.W_hh3 = W_hh3;
  if (JT_out) {
    bppsa_jac chk = j;
    chk.H = std::min(H, 32);           // pointer/shape checks; H limit only for the fused path
    if (H < 1 || H > BPPSA_MAX_H) return fail(BPPSA_ERR_INVALID_ARGUMENT, "H must be in [1, 64]");
    bppsa_status s = check_jac(&chk);
    if (s != BPPSA_OK) return s;
    REQUIRE_DEV(JT_out, "JT_out");
    cudaError_t e = launch_materialize_gru(h_prev, r, z, n, M, W_hh3, JT_out, T, B, H, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_status(e, "materialize gru");
    bppsa_jac d{};
    d.kind = BPPSA_JAC_DENSE;
    d.T = T; d.B = B; d.H = H; d.JT = JT_out;
    *desc = d;
    return BPPSA_OK;
  }
  bppsa_status s = check_jac(&j);
  if (s != BPPSA_OK) return s;
  *desc = j;
  return BPPSA_OK;
}

bppsa_status bppsa_gru_gates(int T, int B, int H, int I, const float* x, const float* h, const float* h_init,
                             const float* W_ih3, const float* W_hh3, const float* b_ih3, const float* b_hh3,
                             float* h_prev, float* r, float* z, float* n, float* M, void* stream) {
  if (T < 1 || B < 1) return fail(BPPSA_ERR_INVALID_ARGUMENT, "T and B must be >= 1");
  if (H < 1 || H > 32 || I < 1 || I > 64)
    return fail(BPPSA_ERR_NOT_SUPPORTED, "GRU gate recompute: 1 <= H <= 32, 1 <= I <= 64");
  REQUIRE_DEV(x, "x");
  REQUIRE_DEV(h, "h");
  if (h_init) REQUIRE_DEV(h_init, "h_init");
  REQUIRE_DEV(W_ih3, "W_ih3");
  REQUIRE_DEV(W_hh3, "W_hh3");
  REQUIRE_DEV(b_ih3, "b_ih3");
  REQUIRE_DEV(b_hh3, "b_hh3");
  REQUIRE_DEV(h_prev, "h_prev");
  REQUIRE_DEV(r, "r");
  REQUIRE_DEV(z, "z");
  REQUIRE_DEV(n, "n");
  REQUIRE_DEV(M, "M");
  cudaError_t e = launch_gru_gates(T, B, H, I, x, h, h_init, W_ih3, W_hh3, b_ih3, b_hh3, h_prev, r, z, n, M,
                                   num_sms(), (cudaStream_t)stream);
  return e == cudaSuccess ? BPPSA_OK : cuda_status(e, "gru gates launch");
}

bppsa_status bppsa_scan_workspace_size(const bppsa_jac* jac, const bppsa_scan_opts* opts, size_t* bytes) {
  if (!bytes) return fail(BPPSA_ERR_INVALID_ARGUMENT, "bytes is NULL");
  bppsa_status s = check_jac(jac, false);
  if (s != BPPSA_OK) return s;
  Plan p1, p2;
  s = make_plan(*jac, 1, opts, false, &p1);
  if (s != BPPSA_OK) return s;
  // also large enough for shard use (head or not, aggregates to one)
  int mode = opts ? opts->mode : BPPSA_SCAN_BLOCKED;
  if (mode == BPPSA_SCAN_BLOCKED) {
    s = make_plan(*jac, 0, opts, true, &p2);
    if (s != BPPSA_OK) return s;
    Plan p3;
    s = make_plan(*jac, 1, opts, true, &p3);
    if (s != BPPSA_OK) return s;
    *bytes = std::max(p1.total, std::max(p2.total, p3.total));
  } else {
    *bytes = p1.total;
  }
  return BPPSA_OK;
}

// The tensor-core leaf kernels move h / grad_h / seed / carries in 16-byte
// units (cp.async 16, float4): a caller buffer at an odd 4-byte offset would
// fault, so such calls take the CUDA-core engine (4-byte accesses) instead.
static bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }
static void demote_unaligned(const bppsa_jac& j, Plan* p, const void* seed, const void* grad_h,
                             const void* grad_h_init) {
  if (j.kind == BPPSA_JAC_RNN_TANH && !(al16(j.h) && al16(seed) && al16(grad_h) && al16(grad_h_init)))
    p->leaf_impl = 1;
}

static bppsa_status scan_impl(const bppsa_jac* jac, const float* seed, const float* e_aff, float* grad_h,
                              float* grad_h_init, void* ws, size_t ws_bytes, const bppsa_scan_opts* opts,
                              void* stream) {
  bppsa_status s = check_jac(jac);
  if (s != BPPSA_OK) return s;
  REQUIRE_DEV(seed, "seed");
  REQUIRE_DEV(grad_h, "grad_h");
  if (grad_h_init) REQUIRE_DEV(grad_h_init, "grad_h_init");
  const bppsa_jac& j = *jac;
  Plan p;
  s = make_plan(j, 1, opts, false, &p);
  if (s != BPPSA_OK) return s;
  demote_unaligned(j, &p, seed, grad_h, grad_h_init);
  if (e_aff && !al16(e_aff)) p.leaf_impl = 1;
  s = check_ws(p, ws, ws_bytes);
  if (s != BPPSA_OK) return s;
  cudaStream_t st = (cudaStream_t)stream;
  char* w = static_cast<char*>(ws);
  const int mode = opts ? opts->mode : BPPSA_SCAN_BLOCKED;
  Tracer tr = tracer_from(opts);
  if (mode == BPPSA_SCAN_ALG1 || mode == BPPSA_SCAN_HYBRID) {
    float* X = reinterpret_cast<float*>(w + p.dense_off);
    const long long n = j.T;
    const int L = (int)(64 - __builtin_clzll((unsigned long long)n));   // ceil(log2(n+1))
    const bool hyb = (mode == BPPSA_SCAN_HYBRID);
    const int up = hyb ? opts->up_levels : L - 1;    // up-sweep levels d = 0..up-1
    const int down = hyb ? opts->down_levels : L;    // down-sweep levels d = down-1..0
    tr.begin(st);
    cudaError_t e = launch_alg1_init(j.JT, seed, X, j.T, j.B, j.H, st);
    tr.end(st);
    if (e != cudaSuccess) return cuda_status(e, "alg1 init");
    for (int d = 0; d < up; ++d) {
      tr.begin(st);
      e = launch_alg1_up(X, j.B, j.H, n, d, st);
      tr.end(st);
      if (e != cudaSuccess) return cuda_status(e, "alg1 up-sweep level");
    }
    if (hyb) {   // Alg. 1 proper: a[n] <- I is symbolic (pair i = 0 rule)
      tr.begin(st);
      e = launch_hybrid_bridge(X, j.B, j.H, n, up, down, st);
      tr.end(st);
      if (e != cudaSuccess) return cuda_status(e, "hybrid bridge");
    }
    for (int d = down - 1; d >= 0; --d) {
      tr.begin(st);
      e = launch_alg1_down(X, j.B, j.H, n, d, st);
      tr.end(st);
      if (e != cudaSuccess) return cuda_status(e, "alg1 down-sweep level");
    }
    tr.begin(st);
    e = launch_alg1_extract(X, j.JT, grad_h, grad_h_init, j.T, j.B, j.H, st);
    tr.end(st);
    if (e != cudaSuccess) return cuda_status(e, "alg1 extract");
    report_launches(opts, tr);
    return BPPSA_OK;
  }
  if (e_aff) {   // head element seed + e_{T-1} (reading 8 / NEXT-4)
    float* aseed = reinterpret_cast<float*>(w + p.aseed_off);
    tr.begin(st);
    cudaError_t e = launch_affine_seed(seed, e_aff, j.T, j.B, j.H, aseed, st);
    tr.end(st);
    if (e != cudaSuccess) return cuda_status(e, "affine seed");
    seed = aseed;
  }
  s = prepare_dense(j, p, w, st, tr);
  if (s != BPPSA_OK) return s;
  s = run_up(j, 1, seed, p, w, nullptr, st, tr, e_aff);
  if (s != BPPSA_OK) return s;
  // top level: one block walked from the symbolic identity (head segment)
  s = run_down(j, 1, seed, p, w, p.L, p.n[p.L], nullptr, grad_h, grad_h_init, st, tr, e_aff);
  report_launches(opts, tr);
  return s;
}

bppsa_status bppsa_scan(const bppsa_jac* jac, const float* seed, float* grad_h, float* grad_h_init, void* ws,
                        size_t ws_bytes, const bppsa_scan_opts* opts, void* stream) {
  NvtxRange nvtx_("bppsa_scan");
  return scan_impl(jac, seed, nullptr, grad_h, grad_h_init, ws, ws_bytes, opts, stream);
}

bppsa_status bppsa_scan_affine(const bppsa_jac* jac, const float* seed, const float* e, float* grad_h,
                               float* grad_h_init, void* ws, size_t ws_bytes, const bppsa_scan_opts* opts,
                               void* stream) {
  NvtxRange nvtx_("bppsa_scan_affine");
  REQUIRE_DEV(e, "e");
  const int mode = opts ? opts->mode : BPPSA_SCAN_BLOCKED;
  if (mode != BPPSA_SCAN_BLOCKED && mode != BPPSA_SCAN_LINEAR)
    return fail(BPPSA_ERR_NOT_SUPPORTED, "the affine scan runs in the BLOCKED and LINEAR modes");
  return scan_impl(jac, seed, e, grad_h, grad_h_init, ws, ws_bytes, opts, stream);
}

bppsa_status bppsa_scan_shard_up(const bppsa_jac* jac, const float* seed, float* aggregate, void* ws,
                                 size_t ws_bytes, const bppsa_scan_opts* opts, void* stream) {
  NvtxRange nvtx_("bppsa_scan_shard_up");
  bppsa_status s = check_jac(jac);
  if (s != BPPSA_OK) return s;
  REQUIRE_DEV(aggregate, "aggregate");
  const int head = seed ? 1 : 0;
  if (seed) REQUIRE_DEV(seed, "seed");
  if (opts && opts->mode != BPPSA_SCAN_BLOCKED) return fail(BPPSA_ERR_NOT_SUPPORTED, "shards use the BLOCKED mode");
  Plan p;
  s = make_plan(*jac, head, opts, true, &p);
  if (s != BPPSA_OK) return s;
  demote_unaligned(*jac, &p, seed, nullptr, nullptr);
  s = check_ws(p, ws, ws_bytes);
  if (s != BPPSA_OK) return s;
  cudaStream_t st = (cudaStream_t)stream;
  char* w = static_cast<char*>(ws);
  Tracer tr = tracer_from(opts);
  s = prepare_dense(*jac, p, w, st, tr);
  if (s != BPPSA_OK) return s;
  if (p.L == 0) return fail(BPPSA_ERR_INVALID_ARGUMENT, "internal: empty shard plan");
  // the top level (one aggregate per sample) goes straight into `aggregate`
  s = run_up(*jac, head, seed, p, w, aggregate, st, tr);
  report_launches(opts, tr);
  return s;
}

bppsa_status bppsa_scan_shard_up_publish(const bppsa_jac* jac, const float* seed, float* aggregate, void* ws,
                                         size_t ws_bytes, const bppsa_scan_opts* opts, int rank, int world,
                                         float* const* peer_mailboxes, unsigned* const* peer_flags,
                                         unsigned* counter, const unsigned* acks, unsigned epoch, void* stream) {
  NvtxRange nvtx_("bppsa_scan_shard_up_publish");
  bppsa_status s = check_jac(jac);
  if (s != BPPSA_OK) return s;
  REQUIRE_DEV(aggregate, "aggregate");
  if (world < 1 || rank < 0 || rank >= world || epoch == 0)
    return fail(BPPSA_ERR_INVALID_ARGUMENT, "need 0 <= rank < world, epoch >= 1");
  if ((seed != nullptr) != (rank == world - 1))
    return fail(BPPSA_ERR_INVALID_ARGUMENT, "exactly the last rank (holding t = T-1) passes the seed");
  if (seed) REQUIRE_DEV(seed, "seed");
  REQUIRE_DEV(peer_mailboxes, "peer_mailboxes");
  REQUIRE_DEV(peer_flags, "peer_flags");
  REQUIRE_DEV(counter, "counter");
  REQUIRE_DEV(acks, "acks");
  if (opts && opts->mode != BPPSA_SCAN_BLOCKED) return fail(BPPSA_ERR_NOT_SUPPORTED, "shards use the BLOCKED mode");
  const int head = seed ? 1 : 0;
  Plan p;
  s = make_plan(*jac, head, opts, true, &p);
  if (s != BPPSA_OK) return s;
  demote_unaligned(*jac, &p, seed, nullptr, nullptr);
  s = check_ws(p, ws, ws_bytes);
  if (s != BPPSA_OK) return s;
  cudaStream_t st = (cudaStream_t)stream;
  char* w = static_cast<char*>(ws);
  Tracer tr = tracer_from(opts);
  s = prepare_dense(*jac, p, w, st, tr);
  if (s != BPPSA_OK) return s;
  if (p.L == 0) return fail(BPPSA_ERR_INVALID_ARGUMENT, "internal: empty shard plan");
  Publish pub;
  pub.peers = peer_mailboxes;
  pub.flags = peer_flags;
  pub.counter = counter;
  pub.acks = acks;
  pub.epoch = epoch;
  pub.rank = rank;
  pub.world = world;
  pub.n = (long long)jac->B * jac->H * jac->H;
  bool fused = false;
  s = run_up(*jac, head, seed, p, w, aggregate, st, tr, nullptr, &pub, &fused);
  if (s == BPPSA_OK && !fused) {                  // one-level shard: its level-0 kernel wrote the aggregate
    tr.begin(st);
    cudaError_t e = launch_exchange_publish(aggregate, pub.n, rank, world, peer_mailboxes, peer_flags, counter,
                                            acks, epoch, num_sms(), st);
    tr.end(st);
    if (e != cudaSuccess) s = cuda_status(e, "exchange publish");
  }
  report_launches(opts, tr);
  return s;
}

bppsa_status bppsa_scan_shard_down(const bppsa_jac* jac, const float* seed, const float* gathered, int rank,
                                   int world, float* grad_h, float* grad_h_init, void* ws, size_t ws_bytes,
                                   const bppsa_scan_opts* opts, void* stream) {
  NvtxRange nvtx_("bppsa_scan_shard_down");
  bppsa_status s = check_jac(jac);
  if (s != BPPSA_OK) return s;
  if (world < 1 || rank < 0 || rank >= world) return fail(BPPSA_ERR_INVALID_ARGUMENT, "bad rank/world");
  const int head = (rank == world - 1) ? 1 : 0;
  if (head && !seed) return fail(BPPSA_ERR_INVALID_ARGUMENT, "the last rank (holding t = T-1) needs the seed");
  if (!head && seed) return fail(BPPSA_ERR_INVALID_ARGUMENT, "only the last rank passes the seed");
  if (seed) REQUIRE_DEV(seed, "seed");
  if (!head) REQUIRE_DEV(gathered, "gathered");
  REQUIRE_DEV(grad_h, "grad_h");
  if (grad_h_init) REQUIRE_DEV(grad_h_init, "grad_h_init");
  if (opts && opts->mode != BPPSA_SCAN_BLOCKED) return fail(BPPSA_ERR_NOT_SUPPORTED, "shards use the BLOCKED mode");
  Plan p;
  s = make_plan(*jac, head, opts, true, &p);
  if (s != BPPSA_OK) return s;
  demote_unaligned(*jac, &p, seed, grad_h, grad_h_init);
  s = check_ws(p, ws, ws_bytes);
  if (s != BPPSA_OK) return s;
  cudaStream_t st = (cudaStream_t)stream;
  char* w = static_cast<char*>(ws);
  float* carry = reinterpret_cast<float*>(w + p.carry_off);
  Tracer tr = tracer_from(opts);
  if (!head) {
    tr.begin(st);
    cudaError_t e = launch_carry_combine(gathered, rank, world, jac->B, jac->H, carry, st);
    tr.end(st);
    if (e != cudaSuccess) return cuda_status(e, "carry combine");
  }
  // level L holds one slot; level L-1 is one block walked from the carry
  s = run_down(*jac, head, seed, p, w, p.L - 1, p.C[p.L - 1], head ? nullptr : carry, grad_h, grad_h_init, st, tr);
  report_launches(opts, tr);
  return s;
}

bppsa_status bppsa_exchange_publish(const float* aggregate, long long n, int rank, int world,
                                    float* const* peer_mailboxes, unsigned* const* peer_flags, unsigned* counter,
                                    const unsigned* acks, unsigned epoch, void* stream) {
  if (n < 1 || world < 1 || rank < 0 || rank >= world || epoch == 0)
    return fail(BPPSA_ERR_INVALID_ARGUMENT, "need n >= 1, 0 <= rank < world, epoch >= 1");
  REQUIRE_DEV(aggregate, "aggregate");
  REQUIRE_DEV(peer_mailboxes, "peer_mailboxes");
  REQUIRE_DEV(peer_flags, "peer_flags");
  REQUIRE_DEV(counter, "counter");
  REQUIRE_DEV(acks, "acks");
  cudaError_t e = launch_exchange_publish(aggregate, n, rank, world, peer_mailboxes, peer_flags, counter, acks,
                                          epoch, num_sms(), (cudaStream_t)stream);
  return e == cudaSuccess ? BPPSA_OK : cuda_status(e, "exchange publish");
}

bppsa_status bppsa_exchange_ack(int rank, int world, unsigned* const* peer_acks, unsigned epoch, void* stream) {
  if (world < 1 || rank < 0 || rank >= world || epoch == 0)
    return fail(BPPSA_ERR_INVALID_ARGUMENT, "need 0 <= rank < world, epoch >= 1");
  REQUIRE_DEV(peer_acks, "peer_acks");
  cudaError_t e = launch_exchange_ack(rank, world, peer_acks, epoch, (cudaStream_t)stream);
  return e == cudaSuccess ? BPPSA_OK : cuda_status(e, "exchange ack");
}

bppsa_status bppsa_exchange_wait(const unsigned* flags, int rank, int world, unsigned epoch, void* stream) {
  if (world < 1 || rank < 0 || rank >= world || epoch == 0)
    return fail(BPPSA_ERR_INVALID_ARGUMENT, "need 0 <= rank < world, epoch >= 1");
  REQUIRE_DEV(flags, "flags");
  cudaError_t e = launch_exchange_wait(flags, rank, world, epoch, (cudaStream_t)stream);
  return e == cudaSuccess ? BPPSA_OK : cuda_status(e, "exchange wait");
}

// A fixed function of the row count only (deterministic results): parts of
// at least 64 rows, at most 16 CTAs per SM of partial tiles.
static long long wgrad_parts(long long rows) {
  long long p = (rows + 63) / 64;
  return std::max(1ll, std::min(p, 2368ll));
}

bppsa_status bppsa_weight_grads_workspace_size(int T, int B, int H, int I, size_t* bytes) {
  if (!bytes) return fail(BPPSA_ERR_INVALID_ARGUMENT, "bytes is NULL");
  if (T < 1 || B < 1 || H < 1 || H > BPPSA_MAX_H || I < 0) return fail(BPPSA_ERR_INVALID_ARGUMENT, "bad shape");
  if (!wgrad_supported(H, I)) return fail(BPPSA_ERR_NOT_SUPPORTED, "weight gradients need I + 1 <= 64");
  const long long rows = (long long)T * B;
  long long slabs = 4 * wgrad_parts(rows);                               // GRU needs NA = 4H
  if (tc_wgrad_applies(H, I, rows)) slabs = std::max(slabs, tc_wgrad_parts(rows));
  *bytes = align_up((size_t)slabs * H * (H + I + 1) * sizeof(float));
  return BPPSA_OK;
}

bppsa_status bppsa_weight_grads_rnn(int T, int B, int H, int I, const float* x, const float* h,
                                    const float* h_init, const float* grad_h, float* dW_ih, float* dW_hh, float* db,
                                    void* ws, size_t ws_bytes, void* stream) {
  NvtxRange nvtx_("bppsa_weight_grads_rnn");
  size_t need;
  bppsa_status s = bppsa_weight_grads_workspace_size(T, B, H, I, &need);
  if (s != BPPSA_OK) return s;
  if (I > 0) {
    REQUIRE_DEV(x, "x");
    REQUIRE_DEV(dW_ih, "dW_ih");
  }
  REQUIRE_DEV(h, "h");
  REQUIRE_DEV(grad_h, "grad_h");
  REQUIRE_DEV(dW_hh, "dW_hh");
  REQUIRE_DEV(db, "db");
  if (h_init) REQUIRE_DEV(h_init, "h_init");
  if (ws_bytes < need || !is_device_ptr(ws)) return fail(BPPSA_ERR_WORKSPACE, "workspace too small or not device memory");
  const long long rows = (long long)T * B;
  cudaError_t e;
  auto a16 = [](const void* p) { return ((uintptr_t)p & 15) == 0; };    // cp.async.bulk sources
  if (tc_wgrad_applies(H, I, rows) && a16(h) && a16(grad_h) && a16(h_init) && (I == 0 || a16(x))) {
    // tensor-core GEMM over K = T*B (tc_wgrad.cu)
    e = launch_tc_wgrad_partials(B, I, x, h, h_init, grad_h, rows, static_cast<float*>(ws), num_sms(),
                                 (cudaStream_t)stream);
    if (e == cudaSuccess)
      e = launch_wgrad_reduce_rnn(static_cast<float*>(ws), tc_wgrad_parts(rows), H, I, dW_ih, dW_hh, db,
                                  (cudaStream_t)stream);
  } else {
    e = launch_wgrad_rnn(T, B, H, I, x, h, h_init, grad_h, dW_ih, dW_hh, db, static_cast<float*>(ws),
                         wgrad_parts(rows), (cudaStream_t)stream);
  }
  return e == cudaSuccess ? BPPSA_OK : cuda_status(e, "weight grads rnn");
}

bppsa_status bppsa_weight_grads_rnn_part_rows(int T, int B, int H, int I, long long* part_rows) {
  if (!part_rows || T < 1 || B < 1) return fail(BPPSA_ERR_INVALID_ARGUMENT, "bad arguments");
  *part_rows = tc_wgrad_applies(H, I, (long long)T * B) ? tc_wgrad_part_rows() : 0;
  return BPPSA_OK;
}

bppsa_status bppsa_weight_grads_rnn_rows(int T, int B, int H, int I, const float* x, const float* h,
                                         const float* h_init, const float* grad_h, long long row0, long long row1,
                                         void* ws, size_t ws_bytes, void* stream) {
  size_t need;
  bppsa_status s = bppsa_weight_grads_workspace_size(T, B, H, I, &need);
  if (s != BPPSA_OK) return s;
  const long long rows = (long long)T * B;
  long long pr = 0;
  bppsa_weight_grads_rnn_part_rows(T, B, H, I, &pr);
  if (pr == 0) return fail(BPPSA_ERR_NOT_SUPPORTED, "row ranges need the tensor-core weight gradients (H = 64)");
  if (row0 < 0 || row1 > rows || row0 >= row1 || row0 % pr != 0 || (row1 % pr != 0 && row1 != rows))
    return fail(BPPSA_ERR_INVALID_ARGUMENT, "row range must be [row0, row1) with both multiples of the part size "
                                             "(bppsa_weight_grads_rnn_part_rows) or row1 = T*B");
  if (I > 0) REQUIRE_DEV(x, "x");
  REQUIRE_DEV(h, "h");
  REQUIRE_DEV(grad_h, "grad_h");
  if (h_init) REQUIRE_DEV(h_init, "h_init");
  if (ws_bytes < need || !is_device_ptr(ws)) return fail(BPPSA_ERR_WORKSPACE, "workspace too small or not device memory");
  auto a16 = [](const void* p) { return ((uintptr_t)p & 15) == 0; };
  if (!(a16(h) && a16(grad_h) && a16(h_init) && (I == 0 || a16(x))))
    return fail(BPPSA_ERR_INVALID_ARGUMENT, "h, grad_h, h_init and x must be 16-byte aligned");
  cudaError_t e = launch_tc_wgrad_partials(B, I, x, h, h_init, grad_h, rows, static_cast<float*>(ws), num_sms(),
                                           (cudaStream_t)stream, row0, row1);
  return e == cudaSuccess ? BPPSA_OK : cuda_status(e, "weight grads rows");
}

bppsa_status bppsa_weight_grads_rnn_reduce(int T, int B, int H, int I, float* dW_ih, float* dW_hh, float* db,
                                           void* ws, size_t ws_bytes, void* stream) {
  size_t need;
  bppsa_status s = bppsa_weight_grads_workspace_size(T, B, H, I, &need);
  if (s != BPPSA_OK) return s;
  if (I > 0) REQUIRE_DEV(dW_ih, "dW_ih");
  REQUIRE_DEV(dW_hh, "dW_hh");
  REQUIRE_DEV(db, "db");
  if (ws_bytes < need || !is_device_ptr(ws)) return fail(BPPSA_ERR_WORKSPACE, "workspace too small or not device memory");
  const long long rows = (long long)T * B;
  if (!tc_wgrad_applies(H, I, rows)) return fail(BPPSA_ERR_NOT_SUPPORTED, "row ranges need the tensor-core path");
  cudaError_t e = launch_wgrad_reduce_rnn(static_cast<float*>(ws), tc_wgrad_parts(rows), H, I, dW_ih, dW_hh, db,
                                          (cudaStream_t)stream);
  return e == cudaSuccess ? BPPSA_OK : cuda_status(e, "weight grads reduce");
}

bppsa_status bppsa_weight_grads_gru(int T, int B, int H, int I, const float* x, const float* h_prev,
                                    const float* r, const float* z, const float* n, const float* M,
                                    const float* grad_h, float* dW_ih3, float* dW_hh3, float* db_ih3,
                                    float* db_hh3, void* ws, size_t ws_bytes, void* stream) {
  NvtxRange nvtx_("bppsa_weight_grads_gru");
  size_t need;
  bppsa_status s = bppsa_weight_grads_workspace_size(T, B, H, I, &need);
  if (s != BPPSA_OK) return s;
  if (I > 0) {
    REQUIRE_DEV(x, "x");
    REQUIRE_DEV(dW_ih3, "dW_ih3");
  }
  REQUIRE_DEV(h_prev, "h_prev");
  REQUIRE_DEV(r, "r");
  REQUIRE_DEV(z, "z");
  REQUIRE_DEV(n, "n");
  REQUIRE_DEV(M, "M");
  REQUIRE_DEV(grad_h, "grad_h");
  REQUIRE_DEV(dW_hh3, "dW_hh3");
  REQUIRE_DEV(db_ih3, "db_ih3");
  REQUIRE_DEV(db_hh3, "db_hh3");
  if (ws_bytes < need || !is_device_ptr(ws)) return fail(BPPSA_ERR_WORKSPACE, "workspace too small or not device memory");
  const long long P = wgrad_parts((long long)T * B);
  cudaError_t e = launch_wgrad_gru(T, B, H, I, x, h_prev, r, z, n, M, grad_h, dW_ih3, dW_hh3, db_ih3, db_hh3,
                                   static_cast<float*>(ws), P, (cudaStream_t)stream);
  return e == cudaSuccess ? BPPSA_OK : cuda_status(e, "weight grads gru");
}

}  // extern "C"
