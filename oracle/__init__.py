"""CPU oracle for the WLB-LLM context-parallel hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in the product package
(`paper_2503_17924_b200`) may import, call, link or execute anything under
`oracle/`.  Only `tests/`, `__graft_entry__.smoke()` and the `cpu_baseline` /
`--impl reference` legs of `bench.py` use it, and there only as the checker or
the timed reference CPU path, never as the thing measured or shipped.

Contents
--------
* `shard_oracle`   -- pure-Python restatement of the reference's CP sharding,
                      kernel-latency model and adaptive selection
                      (`/root/reference/pkg/src/balsim/sharding.py:63-200`,
                      `_kernels/_pure.py:11-66`, `harness.py:279-298`).
* `kernels_oracle.c` -- plain-C restatement of the four reference numeric
                      kernels (`_kernels/_compiled.pyx:11-86`); built into
                      `oracle/liboracle.so` by `oracle/build.sh`.
* `attention_oracle` -- torch-CPU fp32 restatement of document-prefix causal
                      attention, forward and backward (the reference prices
                      but never computes attention: `sharding.py:19-21`,
                      `workload.py:3-4`).  Parity for attention numerics is
                      anchored on the shard-invariance property, not on
                      reference vectors (the reference has none).
* `_ref/`           -- (git-ignored build output) the reference's own Cython
                      kernels compiled from `/root/reference` by
                      `oracle/build.sh`, used to pin `kernels_oracle.c`.

Pinning: `tests/golden/*.json.gz` hold vectors produced by importing the
reference package itself (`tests/golden/make_golden.py`); `tests/test_oracle.py`
checks every oracle function against them.
"""
