// common.cuh — shared device/host definitions of libbppsa (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <stdint.h>

#include <algorithm>
#include <string>

#include "../../include/bppsa.h"

namespace bppsa {

// NVTX range around every C-ABI entry point (header-only nvtx3: free when no
// profiler is attached; named ranges in nsys / ncu timelines)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

// ---------------------------------------------------------------------------
// Error plumbing (thread-local detail string, status codes; no exceptions
// cross the C-ABI).
// ---------------------------------------------------------------------------
void set_error(const std::string& msg);
bppsa_status fail(bppsa_status s, const std::string& msg);
bppsa_status cuda_status(cudaError_t e, const char* where);

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device):
// the attribute is per device context, so a process that drives several GPUs
// (or switches device) must set it on each.  Thread-safe.
cudaError_t smem_attr_once(const void* kernel, int bytes);

#define BPPSA_CHECK_LAUNCH(where)                                         \
  do {                                                                    \
    cudaError_t _e = cudaGetLastError();                                  \
    if (_e != cudaSuccess) return ::bppsa::cuda_status(_e, where);        \
  } while (0)

// ---------------------------------------------------------------------------
// A segment of the scan array (one sequence, or one contiguous time shard).
// Slots in scan order: head segments have slot 0 = seed and slot s >= 1
// holding J_{T-s}^T; non-head shards have slot s holding J_{T-1-s}^T.
// The exclusive output at the slot holding J_t^T is grad_h[t] (DESIGN r.3).
// ---------------------------------------------------------------------------
struct Seg {
  int T, B, H;
  int head;
  __host__ __device__ __forceinline__ long long S() const { return (long long)T + head; }
  __host__ __device__ __forceinline__ int time_of(long long s) const {
    return head ? (T - (int)s) : (T - 1 - (int)s);
  }
};

// Explicit H x H matrices of one level, column-major (element (i,k) at k*H+i),
// addressed by (sample b, slot s).  A head level keeps the vector of slot 0 at
// head_vec + b*head_bstride.
struct MatAcc {
  const float* base;
  long long slot_stride;
  long long batch_stride;
  const float* head_vec;
  long long head_bstride;
  __device__ __forceinline__ const float* mat(int b, long long s) const {
    return base + s * slot_stride + (long long)b * batch_stride;
  }
  __device__ __forceinline__ const float* vec(int b) const {
    return head_vec + (long long)b * head_bstride;
  }
};

// Additive vector term of the affine scan (per-step losses):
// element s is (A_s, m_s), out[s+1] = A_s out[s] + m_s.  time_mode 0: m_s at
// base + s*slot_stride + b*batch_stride (an upper level's vector parts);
// time_mode 1: base = e [T][B][H] and slot s (holding J_t^T, t = time_of(s))
// adds e_{t-1} (nothing at t = 0).  base == nullptr: no additive term.
struct VecAcc {
  const float* base = nullptr;
  long long slot_stride = 0, batch_stride = 0;
  int time_mode = 0;
  __device__ __forceinline__ const float* at(int b, long long s, const Seg& seg, int B, int H) const {
    if (base == nullptr) return nullptr;
    if (time_mode == 0) return base + s * slot_stride + (long long)b * batch_stride;
    const int t = seg.time_of(s) - 1;
    return t < 0 ? nullptr : base + ((long long)t * B + b) * H;
  }
};

// ---------------------------------------------------------------------------
// Kernel launchers (defined in the .cu files).
// ---------------------------------------------------------------------------
struct LeafArgs {            // implicit leaves (RNN / GRU)
  Seg seg;
  int kind;                  // BPPSA_JAC_RNN_TANH or BPPSA_JAC_GRU
  const float* h;            // RNN
  const float* W;            // RNN W_hh [H][H] | GRU W_hh3 [3H][H]
  const float *hp, *r, *z, *n, *M;   // GRU
  const float* seed;         // head only
};

// level-0 fold: blocks q in [q0, q0+nq) of C slots -> agg_out [B][n_out][H*H] (column-major)
cudaError_t launch_leaf_up(const LeafArgs& a, int C, float* agg_out, long long n_out, long long q0,
                           long long nq, cudaStream_t st);
// same on the tensor cores (tcgen05): RNN, H == 64, matrix blocks q in [q0, n_out);
// prec 0 = 3xFP16 with per-chain scaling, 1 = 3xTF32
cudaError_t launch_tc_leaf_up(const LeafArgs& a, int C, float* agg_out, long long n_out, long long q0,
                              int num_sms, cudaStream_t st, int prec);
// exact-integer tensor-core fold (tc_i8.cu): RNN, H == 64, blocks q in [q0, n_out)
cudaError_t launch_tc_fold_i8(const LeafArgs& a, int C, float* agg_out, long long n_out, long long q0, int num_sms,
                              cudaStream_t st);
// exact-integer tensor-core walk (tc_i8.cu): RNN, H == 64; carries [B][nblk][H] (head: the seed)
cudaError_t launch_tc_walk_i8(const LeafArgs& a, int C, const float* carry, long long nblk, float* grad_h,
                              float* grad_init, int num_sms, cudaStream_t st);
// level-1 head slot: column-major H = 64 matrix at lvl + b*bstride -> M . seed_b (in place)
cudaError_t launch_head_apply(float* lvl, long long bstride, const float* seed, int B, int H, cudaStream_t st);
// e / vec_out / head_out: the affine terms as for launch_leaf_down (B <= 128)
cudaError_t launch_tc_leaf_down(const LeafArgs& a, int C, const float* carry, long long nblk, float* grad_h,
                                float* grad_init, int num_sms, cudaStream_t st, const float* e = nullptr,
                                float* vec_out = nullptr, float* head_out = nullptr, long long head_bstride = 0);
// level-0 walk: carries [B][nblk][H] (or head I) -> grad_h; grad_init nullable
// Affine (e != nullptr): v <- J_t^T v + e_{t-1}.  vec_out != nullptr: the
// block's vector part instead of a walk — from 0 (or the head's seed) through
// every element of the block, stored at vec_out[b][q][H]; the head block's
// value also at head_out + b*head_bstride.
cudaError_t launch_leaf_down(const LeafArgs& a, int C, const float* carry,
                             long long nblk, float* grad_h, float* grad_init,
                             cudaStream_t st, const float* e = nullptr,
                             float* vec_out = nullptr, float* head_out = nullptr,
                             long long head_bstride = 0);

// The carry exchange fused into the up-sweep's top level (SURVEY 8(e) "fused
// variant"): the fold's CTAs store the shard aggregate straight into every
// rank's mailbox slot [epoch & 1][rank] and the last CTA to finish raises the
// epoch flag in every rank (same protocol and back-pressure as exchange.cu).
struct Publish {
  float* const* peers = nullptr;      // [world] mailboxes [2][world][n]
  unsigned* const* flags = nullptr;   // [world] flag arrays [world]
  unsigned* counter = nullptr;        // this rank's CTA counter (0 between epochs)
  const unsigned* acks = nullptr;     // this rank's ack words [world]
  unsigned epoch = 0;
  int rank = 0, world = 1;
  long long n = 0;                    // floats per rank slot (B * H * H)
};

// explicit level fold / walk
cudaError_t launch_fold_up(const MatAcc& A, int H, int B, long long n, int C, int head,
                           float* agg_out, long long n_out, cudaStream_t st, const Publish* pub = nullptr);
// out_mode 0: out[b][s][H] (carry array with n slots); 1: grad_h via seg time map
// addv / vec_out / head_out: the affine terms as for launch_leaf_down
cudaError_t launch_walk_down(const MatAcc& A, int H, int B, long long n, int C, int head,
                             const float* carry_in, long long nblk, float* out,
                             int out_mode, const Seg& seg, float* total_out,
                             cudaStream_t st, const VecAcc& addv = VecAcc{},
                             float* vec_out = nullptr, float* head_out = nullptr,
                             long long head_bstride = 0);
// dst[b][i] = seed[b][i] + e[T-1][b][i] (the affine head, reading 8)
cudaError_t launch_affine_seed(const float* seed, const float* e, int T, int B, int H, float* dst,
                               cudaStream_t st);

// peer-memory carry exchange (exchange.cu)
cudaError_t launch_exchange_publish(const float* src, long long n, int rank, int world, float* const* peers,
                                    unsigned* const* peer_flags, unsigned* counter, const unsigned* acks,
                                    unsigned epoch, int num_sms, cudaStream_t st);
cudaError_t launch_exchange_ack(int rank, int world, unsigned* const* peer_acks, unsigned epoch, cudaStream_t st);
cudaError_t launch_exchange_wait(const unsigned* flags, int rank, int world, unsigned epoch, cudaStream_t st);

// GRU forward overhead (FO): the tape from (x, h) (gates.cu)
cudaError_t launch_gru_gates(int T, int B, int H, int I, const float* x, const float* h, const float* h_init,
                             const float* Wih, const float* Whh, const float* bih, const float* bhh, float* hp,
                             float* r, float* z, float* n, float* M, int num_sms, cudaStream_t st);

// DENSE helpers
cudaError_t launch_transpose_dense(const float* JT, float* JTc, long long mats, int H,
                                   cudaStream_t st);
cudaError_t launch_materialize_rnn(const float* h, const float* W, float* JT, int T, int B,
                                   int H, cudaStream_t st);
cudaError_t launch_materialize_gru(const float* hp, const float* r, const float* z,
                                   const float* n, const float* M, const float* W3,
                                   float* JT, int T, int B, int H, cudaStream_t st);

// Alg. 1 literal levels over X [(n+1)][B][H*H]
cudaError_t launch_alg1_init(const float* JT, const float* seed, float* X, int T, int B,
                             int H, cudaStream_t st);
cudaError_t launch_alg1_up(float* X, int B, int H, long long n, int d, cudaStream_t st);
cudaError_t launch_alg1_down(float* X, int B, int H, long long n, int d, cudaStream_t st);
cudaError_t launch_hybrid_bridge(float* X, int B, int H, long long n, int u, int dl, cudaStream_t st);
cudaError_t launch_alg1_extract(const float* X, const float* JT, float* grad_h,
                                float* grad_init, int T, int B, int H, cudaStream_t st);

// shards: carry = M_{r+1} ... M_{G-2} V_{G-1}
cudaError_t launch_carry_combine(const float* gathered, int rank, int world, int B, int H,
                                 float* carry_out, cudaStream_t st);

// weight gradients
bool wgrad_supported(int H, int I);
long long tc_wgrad_parts(long long rows);
bool tc_wgrad_applies(int H, int I, long long rows);
cudaError_t launch_tc_wgrad_partials(int B, int I, const float* x, const float* h, const float* h_init,
                                     const float* grad_h, long long rows, float* ws, int num_sms, cudaStream_t st,
                                     long long row0 = 0, long long row1 = -1);
long long tc_wgrad_part_rows();
cudaError_t launch_wgrad_reduce_rnn(const float* ws, long long nparts, int H, int I, float* dW_ih, float* dW_hh,
                                    float* db, cudaStream_t st);
cudaError_t launch_wgrad_rnn(int T, int B, int H, int I, const float* x, const float* h,
                             const float* h_init, const float* grad_h, float* dW_ih,
                             float* dW_hh, float* db, float* ws, long long nparts,
                             cudaStream_t st);
cudaError_t launch_wgrad_gru(int T, int B, int H, int I, const float* x, const float* hp,
                             const float* r, const float* z, const float* n,
                             const float* M, const float* grad_h, float* dW_ih3,
                             float* dW_hh3, float* db_ih3, float* db_hh3, float* ws,
                             long long nparts, cudaStream_t st);

}  // namespace bppsa
