"""CPU oracle for the fused TLoops evaluator — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import anything here, and
only as the checker or the timed CPU baseline; the product path
(``paper_1804_10120_b200``) never does.

Contents:
  numpy_eval.py   restatement of the reference evaluator
                  (pkg/src/tlang/evaluator.py:122-236): per canonical LHS
                  component, numpy float64 ufuncs in parse-tree order.
  pointwise.py    restatement of the reference's independent per-point
                  oracle (pkg/tests/oracle.py:33-146), pure Python floats.
  counter_rng.py  host twin of tlb_fill_uniform (splitmix64 counter RNG).
  refc.py         driver of oracle/_ref: the reference's own emitted C
                  kernels (codegen_c.emit_c, compiled -O2) run through their
                  tloops_entries table on all host cores.
  build_ref.py    recipe that builds oracle/_ref from /root/reference.

Pinning: numpy_eval and pointwise are checked bit-for-bit against golden
vectors produced by the reference package itself
(tests/golden/make_golden.py → tests/golden/*.tldf) in tests/test_oracle.py.
"""
