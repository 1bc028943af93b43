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

* ``numpy_ref``       — an independent float64 numpy restatement of every workload's
                        forward loss: the check on ``reference_model``.

Partitioner/scheduler parity is pinned against the reference itself: the shipped
reference modules (model/spgraph/cost) generate the golden fixtures under
tests/golden/ (tests/golden/make_golden.py).  Numerics cannot be pinned against the
reference — it ships no runtime and no numerics — so
the torch-CPU oracle is pinned instead (tests/test_oracle_pinning.py) against
``numpy_ref`` (forward loss equal to 1e-11 on every layer kind), against central
finite differences of that forward (every parameter tensor, float64), and its bf16
rounding points against round-to-nearest-even.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package.
"""
