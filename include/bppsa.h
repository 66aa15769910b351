/*
 * bppsa.h — C-ABI of libbppsa.so, a B200 (sm_100a) implementation of the hot
 * path of BPPSA: back-propagation as a modified Blelloch exclusive scan
 * (Wang, Bai & Pekhimenko, arXiv 1907.10134; "P:<n>" = line n of PAPER.md).
 *
 * Conventions (apply to every entry point)
 *   - All tensor pointers are DEVICE pointers (caller-owned, e.g. torch
 *     allocations) unless a comment says "host".  The library never frees or
 *     keeps caller memory; the only library-owned objects are CSR plans
 *     (create/destroy pair).
 *   - fp32 everywhere (reading 11 in DESIGN.md); row-major C layouts.
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).  Every call is
 *     asynchronous on `stream`, validates all arguments before launching and
 *     returns a status; nothing crosses the ABI as an exception.  On error no
 *     partial-output guarantee is made.  bppsa_last_error() returns a
 *     thread-local detail string for the last failing call.
 *   - Calls are re-entrant per stream and capturable into CUDA graphs (no
 *     allocation, no synchronisation inside compute calls).
 *   - Results are bitwise reproducible for fixed shapes/options/build.
 *
 * Notation: T steps, B batch, H hidden size (1 <= H <= 64), I input size.
 * h_t = f_t(h_{t-1}); J_t = dh_t/dh_{t-1}; grad_h[t] = dl/dh_t.
 * Scan array (eqn:scan_input), scan order:
 *     a = [seed, J_{T-1}^T, ..., J_0^T],   A <> B = B A
 * Exclusive scan (Alg. 1 "Ensure"): output at the slot holding J_t^T is
 * grad_h[t]; the inclusive extra J_0^T grad_h[0] is dl/dh_init.
 */
#ifndef BPPSA_H_
#define BPPSA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BPPSA_MAX_H 64

typedef enum {
  BPPSA_OK = 0,
  BPPSA_ERR_INVALID_ARGUMENT = 1, /* null/host pointer, T/B/H out of range      */
  BPPSA_ERR_SHAPE = 2,            /* incompatible shapes                  */
  BPPSA_ERR_PLAN = 3,             /* CSR plan does not match the data     */
  BPPSA_ERR_WORKSPACE = 4,        /* workspace too small or misaligned           */
  BPPSA_ERR_CUDA = 5,             /* a CUDA runtime error (detail in last_error) */
  BPPSA_ERR_NCCL = 6,             /* reserved                                    */
  BPPSA_ERR_NOT_SUPPORTED = 7     /* valid request outside what this build does */
} bppsa_status;

const char* bppsa_status_str(bppsa_status s);
const char* bppsa_last_error(void);
/* 10000*major + 100*minor + patch */
int bppsa_version(void);

/* ---------------------------------------------------------------------------
 * Leaf transposed Jacobians (the scan's elements).
 * ------------------------------------------------------------------------- */
typedef enum {
  BPPSA_JAC_DENSE = 0,    /* explicit J_t^T                                   */
  BPPSA_JAC_RNN_TANH = 1, /* J_t^T = W_hh^T diag(1 - h_t^2)  (eqn:rnn) */
  BPPSA_JAC_GRU = 2       /* eqn:gru_jcb, transposed reading      */
} bppsa_jac_kind;

/* A description of the T transposed Jacobians of one (shard of a) sequence.
 * Only pointers are stored; the tensors stay caller-owned.                  */
typedef struct bppsa_jac {
  int kind;             /* bppsa_jac_kind                                      */
  int T, B, H;
  const float* JT;      /* DENSE: [T][B][H][H], JT[t][b][i][k] = (J_t^T)[i][k]  */
  const float* h;       /* RNN:   [T][B][H]  h_t (tanh outputs, time-major)      */
  const float* W_hh;    /* RNN:   [H][H]     torch weight_hh_l0                  */
  const float* h_prev;  /* GRU:   [T][B][H]  h_{t-1}                             */
  const float* r;       /* GRU:   [T][B][H]  reset gate                          */
  const float* z;       /* GRU:   [T][B][H]  update gate                         */
  const float* n;       /* GRU:   [T][B][H]  candidate                           */
  const float* M;       /* GRU:   [T][B][H]  W_hn h_{t-1} + b_hn (eqn:gru_rewrite)*/
  const float* W_hh3;   /* GRU:   [3H][H]    torch weight_hh_l0, gates (r, z, n) */
} bppsa_jac;

/* Describe the tanh-RNN leaves J_t^T = W_hh^T diag(1-h_t^2).
 * JT_out == NULL: fill *desc with a fused descriptor (J^T is rebuilt inside the
 * scan kernels and never written to HBM).  JT_out != NULL ([T][B][H][H]):
 * materialise the matrices there and return a DENSE descriptor of JT_out.   */
bppsa_status bppsa_jacobians_rnn(int T, int B, int H, const float* h,
                                 const float* W_hh, float* JT_out,
                                 bppsa_jac* desc, void* stream);

/* GRU leaves per eqn:gru_jcb from the saved tape:
 * J^T = W_hr^T diag(r(1-r)M(1-n^2)(1-z)) + W_hn^T diag(r(1-n^2)(1-z))
 *     + W_hz^T diag(z(1-z)(h_{t-1}-n)) + diag(z).   Fused (H <= 32) or
 * materialised as for bppsa_jacobians_rnn.                                  */
bppsa_status bppsa_jacobians_gru(int T, int B, int H, const float* h_prev,
                                 const float* r, const float* z, const float* n,
                                 const float* M, const float* W_hh3,
                                 float* JT_out, bppsa_jac* desc, void* stream);

/* GRU forward overhead "FO" (DESIGN reading 10): a forward
 * that hides its gates (cuDNN) leaves only h; this recomputes the tape the
 * GRU leaf needs from x [T][B][I], h [T][B][H] (= h_0..h_{T-1}), h_init
 * [B][H] (nullable => 0) and torch's GRU parameters W_ih3 [3H][I], W_hh3
 * [3H][H], b_ih3, b_hh3 [3H] (gate order r, z, n), eqn:gru:
 *   h_prev[t] = h[t-1] (h_init at t = 0), r = sigma(W_ir x + b_ir + W_hr
 *   h_prev + b_hr), z = sigma(W_iz x + b_iz + W_hz h_prev + b_hz),
 *   M = W_hn h_prev + b_hn, n = tanh(W_in x + b_in + r M);
 * outputs [T][B][H] each (device, caller-owned).  No recurrence: every
 * (t, b) row at once, fp32 (expf / tanhf, no fast math).  1 <= H <= 32,
 * 1 <= I <= 64 (else BPPSA_ERR_NOT_SUPPORTED).                              */
bppsa_status bppsa_gru_gates(int T, int B, int H, int I, const float* x,
                             const float* h, const float* h_init,
                             const float* W_ih3, const float* W_hh3,
                             const float* b_ih3, const float* b_hh3,
                             float* h_prev, float* r, float* z, float* n,
                             float* M, void* stream);

/* ---------------------------------------------------------------------------
 * The scan (Alg. 1).
 * ------------------------------------------------------------------------- */
typedef enum {
  /* Blelloch's p < n regime (S = Theta(n/p + log p)): blocks of
   * `block0` leaf slots are folded serially (up-sweep) and walked serially
   * (down-sweep, GEMV only); the block aggregates are scanned recursively by
   * the same two-phase scheme in blocks of `block` slots.                     */
  BPPSA_SCAN_BLOCKED = 0,
  /* Alg. 1 executed literally, one launch per level, over a workspace copy of
   * the materialised array (DENSE only; same association as the oracle's
   * serial Alg. 1).                                                           */
  BPPSA_SCAN_ALG1 = 1,
  /* The linear scan = sequential BP on the GPU (S_Linear = Theta(n)):
   * the comparator.                                                          */
  BPPSA_SCAN_LINEAR = 2,
  /* The level-balanced hybrid of P:472 (reading 19):
   * the first `up_levels` = u up-sweep levels of Alg. 1 (d = 0..u-1), a
   * serial bridge that folds the 2^u-block aggregates onto the seed (GEMVs)
   * and deposits the exclusive prefix of every 2^dl-block at its right end,
   * then the last `down_levels` = dl down-sweep levels (d = dl-1..0).  Needs
   * 0 <= u <= max(L-1, 0), dl in {u, u+1}, dl <= L (L = ceil(log2(T+1)));
   * (0, 0) is the linear scan, (L-1, L) is Alg. 1.  DENSE only, like ALG1;
   * same association as the oracle's `hybrid`.  Fewer levels trade GEMMs
   * for a longer serial GEMV bridge (the paper's tuning knob).  Invalid
   * (u, dl): BPPSA_ERR_INVALID_ARGUMENT.                                     */
  BPPSA_SCAN_HYBRID = 3
} bppsa_scan_mode;

typedef struct bppsa_scan_opts {
  int mode;    /* bppsa_scan_mode                                              */
  int block0;  /* BLOCKED: leaf block length in slots (0 = default)            */
  int block;   /* BLOCKED: block length of the upper levels (0 = default)      */
  int leaf_impl; /* level-0 engine (fold and walk of the fused RNN leaves):
                  * 0 = auto: the tanh RNN with H = 64 on the integer tensor
                  * cores (4), everything else on the CUDA cores (1);
                  * 1 = FFMA (CUDA cores, fp32 round-to-nearest);
                  * 2 = 3xFP16 tensor-core fold with per-chain power-of-two
                  * scaling (tanh RNN, 16 <= H <= 64, H % 4 == 0; the walk on
                  * the tensor cores at H = 64) — opt-in: its fp32 accumulation
                  * truncates (a one-signed ~1.4 ulp bias per step);
                  * 3 = the same with a 3xTF32 fold (H = 64);
                  * 4 = exact-integer tensor cores (tanh RNN, H = 64): operands
                  * as 8-bit digits of fixed-point rows (23-bit X per chain row,
                  * 31-bit W), products accumulated EXACTLY in s32 by
                  * tcgen05.mma kind::i8, combined once in fp32
                  * round-to-nearest; no biased rounding anywhere.
                  * 2, 3 and 4 fail with BPPSA_ERR_NOT_SUPPORTED outside their
                  * range.                                                    */
  /* Optional instrumentation (all may be NULL/0): if `events` is non-NULL the
   * library records events[2k] / events[2k+1] (cudaEvent_t, created by the
   * caller) on `stream` immediately before / after its k-th kernel launch,
   * k < n_events/2.  `launches` (host int*) receives the number of kernels
   * the call launched.                                                        */
  void** events;
  int n_events;
  int* launches;
  int up_levels;    /* HYBRID: u                                              */
  int down_levels;  /* HYBRID: dl                                             */
} bppsa_scan_opts;   /* NULL opts = all defaults */

/* Workspace bytes needed by bppsa_scan / the shard calls for this
 * description and options (256-byte alignment required).                    */
bppsa_status bppsa_scan_workspace_size(const bppsa_jac* jac,
                                       const bppsa_scan_opts* opts,
                                       size_t* bytes);

/* Single-GPU scan.  seed [B][H] = dl/dh_{T-1} (a0).  grad_h [T][B][H] out:
 * grad_h[t] = dl/dh_t, grad_h[T-1] = seed.  grad_h_init [B][H] out, nullable:
 * J_0^T grad_h[0] = dl/dh_init.  ws: device workspace of at least
 * bppsa_scan_workspace_size() bytes (contents are scratch).                 */
bppsa_status bppsa_scan(const bppsa_jac* jac, const float* seed, float* grad_h,
                        float* grad_h_init, void* ws, size_t ws_bytes,
                        const bppsa_scan_opts* opts, void* stream);

/* Per-step losses (not in the paper, whose loss sits on
 * the last step, P:317 / reading 8): l = sum_t l_t(h_t), e [T][B][H] device,
 * e[t] = the partial dl_t/dh_t.  The recurrence becomes affine,
 *   grad_h[T-1] = seed + e[T-1],  grad_h[t-1] = J_t^T grad_h[t] + e[t-1],
 *   dl/dh_init = J_0^T grad_h[0],
 * scanned with elements (J^T, e) and (A, a) <> (B, b) = (BA, Ba + b): the
 * block aggregates keep their matrix parts (same kernels, tensor-core fold
 * included) and gain a vector part from one extra GEMV pass per level; the
 * level-0 walk adds e (the TMA walk at H = 64, B <= 128).  BLOCKED and
 * LINEAR modes (others:
 * BPPSA_ERR_NOT_SUPPORTED); same workspace as bppsa_scan; e = 0 gives
 * bppsa_scan's result.                                                      */
bppsa_status bppsa_scan_affine(const bppsa_jac* jac, const float* seed,
                               const float* e, float* grad_h,
                               float* grad_h_init, void* ws, size_t ws_bytes,
                               const bppsa_scan_opts* opts, void* stream);

/* Multi-GPU: contiguous time shards, rank order = time order.
 * `jac` describes this rank's T_local steps.  The rank holding t = T-1 (the
 * last rank) passes its seed and is the "head" shard.
 *
 * shard_up: local leaf + up-sweep to one aggregate per sample, written to
 *   aggregate [B][H][H] (column-major: element (i,k) at k*H+i), the product
 *   J_lo^T ... J_hi^T of this shard; for the head shard the aggregate is the
 *   vector grad_h[lo-1] in aggregate[b*H*H + 0..H-1].  `ws` must be preserved
 *   until the matching shard_down.
 * shard_down: gathered = all ranks' aggregates [world][B][H*H] (rank order);
 *   computes this rank's carry grad_h[hi] = M_{r+1}...M_{G-2} V_{G-1} on the
 *   device and runs the local down-sweep into grad_h [T_local][B][H];
 *   grad_h_init (nullable) receives J_lo^T grad_h[lo] (= dl/dh_init on rank 0).
 * Between the two calls the caller all-gathers `aggregate` (NCCL over
 * NVLink via torch.distributed in the Python binding).                     */
bppsa_status bppsa_scan_shard_up(const bppsa_jac* jac, const float* seed,
                                 float* aggregate, void* ws, size_t ws_bytes,
                                 const bppsa_scan_opts* opts, void* stream);
bppsa_status bppsa_scan_shard_down(const bppsa_jac* jac, const float* seed,
                                   const float* gathered, int rank, int world,
                                   float* grad_h, float* grad_h_init, void* ws,
                                   size_t ws_bytes, const bppsa_scan_opts* opts,
                                   void* stream);

/* Peer-memory carry exchange (row a5 without NCCL; SURVEY 8(e) "fused
 * variant"): replaces the all-gather between bppsa_scan_shard_up and
 * bppsa_scan_shard_down.  Every rank owns a mailbox of 2 x world x n floats
 * (n = B*H*H, the aggregate size; an epoch-parity double buffer), flags
 * [world] u32 and acks [world] u32, zero-initialised, mapped into every
 * other rank's address space (CUDA IPC over NVLink / NVSwitch, or the same
 * device).
 * publish: first waits (acquire) until acks[r] >= epoch - 2 for every
 * r < rank (the readers of this rank's slot have finished the epoch whose
 * slot is about to be overwritten), then stores `aggregate` [n] into
 * mailbox[p][epoch & 1][rank] of every rank p (peer_mailboxes: device array
 * [world] of device pointers) and, once every block's stores are performed
 * (system-scope fence, last-block count in this rank's `counter`,
 * zero-initialised), release-stores `epoch` into flags[p][rank].
 * wait: an acquire spin until flags[r] >= epoch for every r > rank (the
 * ranks whose aggregates this rank's carry needs); kernels after it on
 * `stream` may read mailbox[epoch & 1] as shard_down's `gathered`.
 * ack: after those reads (stream order: call it after bppsa_scan_shard_down),
 * release-stores `epoch` into acks[p][rank] of every later rank p
 * (peer_acks: device array [world] of device pointers).  Epochs start at 1
 * and increase by 1 per exchange.  A rank that skips ack blocks its writers
 * two epochs later (no silent overwrite).                                   */
bppsa_status bppsa_exchange_publish(const float* aggregate, long long n,
                                    int rank, int world,
                                    float* const* peer_mailboxes,
                                    unsigned* const* peer_flags,
                                    unsigned* counter, const unsigned* acks,
                                    unsigned epoch, void* stream);
bppsa_status bppsa_exchange_ack(int rank, int world, unsigned* const* peer_acks,
                                unsigned epoch, void* stream);
bppsa_status bppsa_exchange_wait(const unsigned* flags, int rank, int world,
                                 unsigned epoch, void* stream);
/* bppsa_scan_shard_up with the publish FUSED into the up-sweep's top level
 * (SURVEY 8(e)): the CTAs of the last fold store the shard aggregate straight
 * into mailbox[p][epoch & 1][rank] of every rank p and the last CTA to finish
 * release-stores `epoch` into flags[p][rank] (the protocol, back-pressure
 * wait on acks and argument meanings of bppsa_exchange_publish; n = B*H*H).
 * `aggregate` [B][H*H] also receives the local copy.  A shard whose plan has
 * one level (its level-0 kernel is the top) falls back to a separate publish
 * launch.  Follow with bppsa_exchange_wait, bppsa_scan_shard_down on
 * mailbox[epoch & 1] and bppsa_exchange_ack, exactly as after _publish.     */
bppsa_status bppsa_scan_shard_up_publish(const bppsa_jac* jac, const float* seed,
                                         float* aggregate, void* ws, size_t ws_bytes,
                                         const bppsa_scan_opts* opts, int rank, int world,
                                         float* const* peer_mailboxes,
                                         unsigned* const* peer_flags, unsigned* counter,
                                         const unsigned* acks, unsigned epoch, void* stream);


/* ---------------------------------------------------------------------------
 * Parameter gradients, eqn:update_param, tied weights summed over
 * time.  Deterministic (fixed-order) reductions, no float atomics.
 * ------------------------------------------------------------------------- */
bppsa_status bppsa_weight_grads_workspace_size(int T, int B, int H, int I,
                                               size_t* bytes);

/* RNN: delta_t = (1-h_t^2) o grad_h[t]; dW_hh = sum delta_t h_{t-1}^T [H][H],
 * dW_ih = sum delta_t x_t^T [H][I], db = sum delta_t [H] (= db_ih = db_hh).
 * x [T][B][I]; h [T][B][H]; h_init [B][H] nullable (=> h_{-1} = 0).          */
bppsa_status bppsa_weight_grads_rnn(int T, int B, int H, int I, const float* x,
                                    const float* h, const float* h_init,
                                    const float* grad_h, float* dW_ih,
                                    float* dW_hh, float* db, void* ws,
                                    size_t ws_bytes, void* stream);

/* The RNN weight gradients in row ranges (for inputs that arrive in pieces,
 * e.g. host-streamed time chunks): rows = T*B in time-major order.
 * part_rows: the granularity of the tensor-core path (0 when it does not
 * apply: then use bppsa_weight_grads_rnn).  rows: computes the partial
 * slabs of rows [row0, row1) into `ws` (row0, row1 multiples of part_rows,
 * or row1 = T*B); x, h, grad_h, h_init are the WHOLE arrays (only the range
 * and, for h_prev, the row B before it are read).  reduce: sums every slab
 * into dW_ih, dW_hh, db after all ranges ran on `stream` (or were otherwise
 * ordered before it).  Covering [0, T*B) in any order gives bit-identical
 * results to bppsa_weight_grads_rnn (same parts, same fixed reduction).    */
bppsa_status bppsa_weight_grads_rnn_part_rows(int T, int B, int H, int I,
                                              long long* part_rows);
bppsa_status bppsa_weight_grads_rnn_rows(int T, int B, int H, int I,
                                         const float* x, const float* h,
                                         const float* h_init,
                                         const float* grad_h, long long row0,
                                         long long row1, void* ws,
                                         size_t ws_bytes, void* stream);
bppsa_status bppsa_weight_grads_rnn_reduce(int T, int B, int H, int I,
                                           float* dW_ih, float* dW_hh,
                                           float* db, void* ws,
                                           size_t ws_bytes, void* stream);

/* GRU (gates r,z,n order as torch): dN = g(1-z)(1-n^2), dZ = g(h_prev-n)z(1-z),
 * dR = dN M r(1-r), dM = dN r;  dW_ih3 = [dR;dZ;dN] x^T [3H][I],
 * dW_hh3 = [dR;dZ;dM] h_prev^T [3H][H], db_ih3 = sum [dR;dZ;dN],
 * db_hh3 = sum [dR;dZ;dM] ([3H] each).                                       */
bppsa_status bppsa_weight_grads_gru(int T, int B, int H, int I, const float* x,
                                    const float* h_prev, const float* r,
                                    const float* z, const float* n,
                                    const float* M, const float* grad_h,
                                    float* dW_ih3, float* dW_hh3, float* db_ih3,
                                    float* db_hh3, void* ws, size_t ws_bytes,
                                    void* stream);

/* ---------------------------------------------------------------------------
 * CSR variant (P:182 sec:jcb_in_sparse_format): transposed
 * Jacobians with architecture-fixed ("guaranteed zero") sparsity patterns; a
 * symbolic product plan computed once ahead of time (output patterns and, for
 * every output entry, its contribution pairs); numeric SpGEMM / SpMV on the
 * device; the level-balanced hybrid schedule of P:472 (up-sweep levels
 * d < u, a serial bridge over the 2^u-block aggregates, down-sweep levels
 * d < dl, dl in {u, u+1}; DESIGN reading 19).
 *
 * Layouts: CSR in the SciPy convention, rows = the operator's INPUT space.
 * Device data of a batched element is sample-minor, data[p * B + b] (one
 * structural entry of all B samples is one contiguous 4B-vector, so every
 * gather of the numeric SpGEMM reads B consecutive floats); a shared element
 * (e.g. conv weights) is data[p].
 * ------------------------------------------------------------------------- */
typedef struct bppsa_csr_pattern {   /* HOST arrays                          */
  int rows, cols;
  long long nnz;
  const long long* indptr;           /* [rows+1]                              */
  const int* indices;                /* [nnz], strictly increasing per row    */
} bppsa_csr_pattern;

typedef struct bppsa_csr_plan bppsa_csr_plan;   /* opaque, immutable after create */

/* chain[k] = pattern of J_{k+1}^T in time order (k = 0 is f_1, whose rows are
 * the network input), n operators, chain compatibility cols(J_k^T) =
 * rows(J_{k+1}^T).  Builds every symbolic product of the schedule on
 * the host (may take seconds) and uploads the plan with cudaMemcpy
 * (synchronous; not graph-capturable).  Errors: SHAPE for incompatible
 * neighbours, INVALID_ARGUMENT for bad (u, dl), NOT_SUPPORTED when the
 * schedule's products exceed `max_contributions` (0 = 2^31) pairs.         */
bppsa_status bppsa_csr_plan_create(const bppsa_csr_pattern* chain, int n,
                                   int up_levels, int down_levels,
                                   long long max_contributions,
                                   bppsa_csr_plan** plan);
/* The same schedule analysis WITHOUT the numeric plan (host only: no
 * contribution lists, no device memory, no CUDA call): product patterns by a
 * bitset Gustavson product, contribution pairs in closed form
 * sum_k nnz(L[:, k]) nnz(R[k, :]).  For schedules whose contribution lists do
 * not fit, e.g. the paper's (u, dl) = (3, 4) on the 97 %-pruned
 * VGG-11 (9.1e10 pairs; DESIGN reading 22).  Answers bppsa_csr_plan_info
 * (contributions = the pairs the numeric plan would hold) and
 * bppsa_csr_plan_steps with the same records bppsa_csr_plan_create gives;
 * bppsa_csr_plan_workspace_size and bppsa_csr_scan return NOT_SUPPORTED.
 * Errors as plan_create; NOT_SUPPORTED when a product's bit rows exceed
 * 16 GB or its output 2^31 entries.                                         */
bppsa_status bppsa_csr_plan_create_symbolic(const bppsa_csr_pattern* chain, int n,
                                            int up_levels, int down_levels,
                                            bppsa_csr_plan** plan);
void bppsa_csr_plan_destroy(bppsa_csr_plan* plan);
/* Workspace for batch B given which elements carry per-sample data.        */
bppsa_status bppsa_csr_plan_workspace_size(const bppsa_csr_plan* plan, int B,
                                           const int* batched, size_t* bytes);
/* Static counts of the schedule (the FLOP analysis of fig:prune_symbolic,
 * P:467): contribution pairs of all SpGEMMs, nnz touched by all SpMVs, and
 * the number of numeric kernels one scan launches.                         */
bppsa_status bppsa_csr_plan_info(const bppsa_csr_plan* plan,
                                 long long* contributions, long long* spmv_nnz,
                                 int* n_kernels);
/* Per-step static FLOP analysis of the schedule (fig:prune_symbolic, P:467,
 * P:474).  One record per numeric op in schedule order — up-sweep SpGEMMs
 * and SpMVs (phase UP, level d), bridge SpMVs (BRIDGE, level = fold index),
 * down-sweep SpMVs (DOWN, level d), the inclusive extra J_1^T dl/dx_1
 * (EXTRA) — then the BP baseline's n gradient operators (BP, level k = the
 * operator J_k^T, k = n..1).  flops: per sample, 2 x contribution pairs (mm)
 * or 2 x nnz (mv); dense_flops: the same op on dense operands (2 m k n / 2 m n,
 * the figure's x-axis).  critical: the costliest op of each up-/down-sweep
 * level, every bridge / extra / BP op (DESIGN reading 23).  Writes
 * min(capacity, count) records; *n_steps = count.                          */
enum { BPPSA_CSR_STEP_MM = 0, BPPSA_CSR_STEP_MV = 1 };
enum { BPPSA_CSR_STEP_UP = 0, BPPSA_CSR_STEP_BRIDGE = 1, BPPSA_CSR_STEP_DOWN = 2,
       BPPSA_CSR_STEP_EXTRA = 3, BPPSA_CSR_STEP_BP = 4 };
typedef struct bppsa_csr_step {
  int kind, phase, level, critical;
  long long flops, dense_flops;
} bppsa_csr_step;
bppsa_status bppsa_csr_plan_steps(const bppsa_csr_plan* plan,
                                  bppsa_csr_step* steps, int capacity,
                                  int* n_steps);
/* data[k]: device values of J_{k+1}^T (layout above; batched[k] != 0 for
 * per-sample data).  seed: dl/dx_n [B][cols(J_n^T)].  grads[k], k = 0..n
 * (n+1 pointers, NULL = not wanted): dl/dx_k [B][dim x_k]; grads[n] = seed;
 * grads[0] = J_1^T dl/dx_1 is the inclusive extra.                          */
bppsa_status bppsa_csr_scan(const bppsa_csr_plan* plan, int B,
                            const float* const* data, const int* batched,
                            const float* seed, float* const* grads, void* ws,
                            size_t ws_bytes, void* stream);

/* Analytical transposed-Jacobian builders (Algs. 2-10), device
 * data + host patterns:
 * conv 3x3 / pad 1 / stride 1, c_i -> c_o on h x w (generic stencil; reading
 * 17).  Two-call pattern: pass NULL arrays to get *nnz.  weights_host
 * [c_o][c_i][3][3] is only consulted when drop_zero != 0 (pruned taps leave
 * the pattern).  tap[p] receives the weight index of entry p for
 * bppsa_csr_conv_data.                                                      */
bppsa_status bppsa_csr_conv3x3_pattern(int ci, int co, int h, int w,
                                       const float* weights_host, int drop_zero,
                                       long long* nnz, long long* indptr,
                                       int* indices, int* tap);
/* data[p] = weights[tap[p]] (device; shared across the batch)               */
bppsa_status bppsa_csr_conv_data(long long nnz, const int* tap,
                                 const float* weights, float* data,
                                 void* stream);
/* ReLU (Algs. 5-7): identity pattern of size d; data[i*B + b] = [x[b][i] > 0] */
bppsa_status bppsa_csr_relu_data(long long d, int B, const float* x,
                                 float* data, void* stream);
/* 2x2/stride-2 max-pool window pattern (reading 18): row = input pixel
 * (c, y, x), one entry in column (c, y/2, x/2).  Host pattern builder and
 * device data: data[i*B + b] = 1 if pool_idx[b][c][y/2][x/2] (flat index in
 * the c-th input plane, torch return_indices) selects pixel i, else 0.      */
bppsa_status bppsa_csr_maxpool_pattern(int c, int h, int w, long long* indptr,
                                       int* indices);
bppsa_status bppsa_csr_maxpool_data(int c, int h, int w, int B,
                                    const long long* pool_idx, float* data,
                                    void* stream);

/* Device analytical builders (Algs. 2-4 and 8-9 on the GPU; SURVEY 8(f)
 * NEXT-3; "generate the transposed Jacobian directly into the CSR
 * format").  Same patterns, entry order and taps as the host builders above;
 * every output array is a caller-owned DEVICE buffer; asynchronous on
 * `stream`.
 * bppsa_csr_conv3x3_build_size: *max_nnz = the structural nnz
 * ci co (3h-2)(3w-2) (h, w >= 2; reading 17) = the capacity `indices`,
 * `tap`, `data` need (the exact count when drop_zero = 0); *ws_bytes = the
 * workspace of bppsa_csr_conv3x3_build (0 unless drop_zero).
 * bppsa_csr_conv3x3_build: indptr [ci h w + 1] (Alg. 2 in closed form, or a
 * row count + device scan when drop_zero drops pruned taps; the nnz is
 * indptr[ci h w]), indices (Alg. 3), tap (nullable), data (nullable:
 * data[p] = weights[tap[p]], Alg. 4).  weights: device [co][ci][3][3],
 * required when drop_zero or data.                                          */
bppsa_status bppsa_csr_conv3x3_build_size(int ci, int co, int h, int w,
                                          int drop_zero, long long* max_nnz,
                                          size_t* ws_bytes);
bppsa_status bppsa_csr_conv3x3_build(int ci, int co, int h, int w,
                                     const float* weights, int drop_zero,
                                     long long* indptr, int* indices, int* tap,
                                     float* data, void* ws, size_t ws_bytes,
                                     void* stream);
/* max-pool window pattern (as bppsa_csr_maxpool_pattern) and the ReLU
 * identity pattern of size d, on the device.                                */
bppsa_status bppsa_csr_maxpool_build(int c, int h, int w, long long* indptr,
                                     int* indices, void* stream);
bppsa_status bppsa_csr_identity_build(long long d, long long* indptr,
                                      int* indices, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* BPPSA_H_ */
