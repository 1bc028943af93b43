"""TEST INFRASTRUCTURE ONLY — the checker, never the product.

CPU restatements used as oracles for the B200 stage executor:

* ``torch_backend``   — torch-CPU implementations of the executor's kernel
                        interface (same signatures as runtime.backend.CudaBackend),
                        used to run the executor's multi-rank host logic over gloo;
* ``reference_model`` — a monolithic (no pipeline, no micro-batching) torch
                        autograd model of a workload: per-step loss and gradients
                        against which the pipelined GPU run is compared
                        (bf16 rtol 2e-2, fp32 1e-4; BASELINE.json north_star);
* ``brute``           — SPEC oracle module: min_inflight_search (Appendix A) and
                        exhaustive_optimize over convex partitions.

Numerics parity is UNPINNED against the reference itself: the reference ships
no runtime and no numerics; the torch-CPU model is
the stated oracle.  Partitioner/scheduler parity IS pinned: the shipped
reference modules (model/spgraph/cost) generate the golden fixtures under
tests/golden/ (tests/golden/make_golden.py).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package.
"""
