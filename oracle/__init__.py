"""CPU oracle for the Evoformer hot path.

TEST INFRASTRUCTURE ONLY.  Nothing under ``paper_2207_05477_b200/`` may
import this package: the product path runs the sm_100a kernels in
``libevoformer_sm100.so`` and fails loudly when they are missing.  Only
``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` use it, and only as the checker
or the timed CPU baseline.

``evoformer_np`` is a numpy restatement of the reference package
(``/root/reference/pkg/src/evotrain``); every function cites the
reference file:line it follows.  It is pinned against golden vectors that
``tests/golden/gen_goldens.py`` produced by running the reference itself
(see ``tests/test_oracle_golden.py``).  The triangle-multiplication
restatement has no reference counterpart: its parity is UNPINNED.
"""
