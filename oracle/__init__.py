"""CPU oracle for the PCG hot path of the reference TV deblurring solver.

TEST INFRASTRUCTURE ONLY.  Nothing in ``paper_1011_5964_b200`` imports this
package; only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
CPU-baseline leg (``cpu_baseline`` / ``--impl reference``) may use it, and
only as the checker or as the timed CPU reference, never as the product path.

Parity pinning: ``tests/golden/make_golden.py`` runs the real reference
(``/root/reference/pkg/src/tvdeblur``, importable in the build container) on
seeded inputs and commits the outputs under ``tests/golden/``;
``tests/test_oracle_golden.py`` checks this restatement against them.
"""
