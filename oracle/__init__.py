"""BPPSA oracle — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct fp64 CPU implementation of what the BPPSA hot
path computes, written from PAPER.md (cited as P:<line>) with the readings
listed in DESIGN.md ("Readings of the paper").  It shares no code with the CUDA
path and is independent of it.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline /
`--impl reference` leg may import, call or execute anything under `oracle/`.
The product path (paper_1907_10134_b200) never imports it.

Modules
  bp    — definitions: sequential BP (eqn:backprop) for the tanh RNN
          and the GRU, leaf transposed Jacobians (eqn:rnn, eqn:gru_jcb), the
          fp64 forward and loss used by the finite-difference pins, the
          parameter gradients of eqn:update_param, and the affine
          recurrence of per-step losses (not in the paper).
  scan  — the operator A<>B = BA, the exclusive scan definition
          (eqn:scan_input), Alg. 1 executed literally,
          the level-balanced hybrid scan, its per-step static FLOP
          analysis (fig:prune_symbolic), and the contiguous-shard
          emulation of the multi-GPU carry protocol.
  csr   — CSR matrices, the analytical transposed-Jacobian builders of
          Algs. 2-10, the exact guaranteed-zero stencil pattern,
          spmv / spgemm / plan_product / execute_plan.

Parity status: every function is pinned by tests/test_oracle_*.py against
finite differences, brute-force products, closed forms, integer families or
values printed in the paper (tests/golden/).  No function is "parity unpinned".
"""
