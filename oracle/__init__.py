"""CPU oracle for the Kernel Aggregated FMM (arXiv 2010.15155) evaluation pass.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package (plus the developer check scripts under ``scripts/``, which compare the
CUDA path with it the way the tests do, and ``scripts/make_golden.py``, which
writes the golden files from it alone).  The product path (``paper_2010_15155_b200``) never imports it and
shares no code with it: the two meet only at the seeded input generators in
``workloads/``.

Contents (each function cites the PAPER.md passage it restates):
  kernels.py    O1 pairwise kernels and the plain direct sum, Eq. (1)/(2)
  tree.py       adaptive octree by midpoint recursion on quantised coordinates
  lists.py      U/V/W/X interaction lists by their definitions
  operators.py  surfaces, ML-tree kernel matrices, SVD check->equivalent
                factors, composed M2M/L2L, raw M2L matrices
  fmm.py        O2: plain KIFMM with the paper's kernel tables (Tables I-V)

Everything is fp64 numpy/scipy.  "parity unpinned": the FMM approximation
values themselves (O2) are pinned only by construction plus the invariants in
tests/test_oracle_*.py; the paper prints no numeric FMM output.
"""
