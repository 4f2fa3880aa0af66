"""CPU oracle for the tensorized EMO selection hot path -- TEST INFRASTRUCTURE ONLY.

This package is a NumPy restatement of the reference package ``temo`` 0.1.0
(``/root/reference/pkg/src/temo``) for exactly the functions on the hot path
(SURVEY.md section 8a rows a1-a20).  Every function cites the reference
``file:line`` it restates.

Who may use it
--------------
* ``tests/`` (as the checker the CUDA path is compared against),
* ``__graft_entry__.smoke()`` (as the checker), and
* ``bench.py``'s ``cpu_baseline`` leg and ``--impl reference`` arm (timed as
  the CPU reference).

The product package ``paper_2503_20286_b200`` never imports this package; its
hot path fails loudly when the CUDA library is missing.

Pinning
-------
The restatement is pinned against golden vectors produced by running the real
reference in the build container (``tests/golden/make_golden.py``; fixtures in
``tests/golden/*.npz``) and checked by ``tests/test_oracle_golden.py``.
Exceptions, stated where they occur:

* ``problems.evaluate_lsmop1`` and ``moead.tchebycheff`` have no reference
  implementation (``SPEC.md:8``; ``moead.py:43-67`` is PBI-only): they are
  self-oracles, *parity unpinned*.
* ``hype.hv_estimate`` restates the summation order of the OpenBLAS ``dgemv``
  kernel that the reference reaches through ``dominates @ weight``
  (``hype.py:83``); it is pinned against reference output
  generated with ``OPENBLAS_NUM_THREADS=1``.
"""

from . import directions, hype, moead, ndsort, nsga3, philox, problems, variation  # noqa: F401

BIG = float(__import__("numpy").finfo("float64").max)  # tensorops.py:18
