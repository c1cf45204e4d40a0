"""Tofu oracle — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU implementation (Python + numpy, fp64) of
what the Tofu hot path computes (arXiv 1807.08887, /root/reference/PAPER.md,
cited below as P:L<line>):

* ``tdl``       — TDL operator descriptions (§4.1).
* ``interval``  — symbolic interval analysis, Eq. 1 and Fig. int-arith
                  (§4.2).
* ``strategy``  — Case-1 / Case-2 partition strategies (§4.2).
* ``graph``     — dataflow graph + coarsening (§5.1).
* ``cost``      — communication cost of a plan (§5; Lemma
                  P:L1604-1644), evaluated twice: box arithmetic and
                  element-set enumeration.
* ``search``    — per-step DP, recursive partitioning (§5.2) and a
                  brute-force enumerator of all plan sequences.
* ``exec_ref``  — unpartitioned fp64 execution of a training graph, with
                  optional bf16 storage rounding (RNE).
* ``sim``       — partitioned execution on k simulated workers
                  (partition-n-reduce P:L248-259 §3.1, MultiFetch / spread
                  reduction P:L862-881 §6).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product path (``paper_1807_08887_b200``) never imports it and shares no code
with it; the two meet only in ``tofu_inputs`` (seeded workload/tensor
generators that contain none of the method's arithmetic).

Parity pins: every function is pinned by ``tests/test_oracle_*.py`` against
paper values (``tests/golden/``), closed forms, invariants or brute force.
Functions without such a pin say "parity unpinned" in their docstring.
"""
