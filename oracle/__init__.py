"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct fp64 (numpy/scipy) implementation of what
the paper's hot path computes (§2.1-§3.1, Eq. 2-6, Alg. 1-3).
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may import anything from here.
The CUDA product path (``paper_1305_5179_b200``) never imports, links or
executes this package, and this package never imports the product path:
the two share no code (only the seeded input generators in ``synth/``).

Modules and the passage each follows:
  kernel   Eq. 6 Gaussian entries (Table I l.299),
           brute-force truncated matvec A w (Eq. 4, l.257-262)
  extend   off-surface points X_delta^+/- and labels (§2.1.1-2.1.2, l.131-198)
  cells    float32 replica of the cell-list build ("truncation area", Alg. 2
           l.442; SURVEY.md §8(c) item 6 fixes the arithmetic)
  solve    dense LU direct solve; RAS blocks (§3.1 l.340-359); restarted
           right-preconditioned GMRES (l.359, l.389-391)
  grid     evaluation on a regular grid (Eq. 5, l.264-271; §2.1.3 l.200-221),
           masked zero-crossings (M_ext^eps cap S_0, l.211-221)
  density  separation / fill distance and h_max (Eq. 7, 8, 11; l.490-625)
  mesh     the triangle mesh of the masked zero iso-surface (Alg. 1 step 4,
           l.317-328, restricted to M_ext^eps, l.200-221): marching tetrahedra
           on the Kuhn split of the grid cubes (reading R24)

Parity pins: tests/test_oracle_*.py (run with -m "not gpu").  Functions
without an independent pin say "parity unpinned" in their docstring.
"""
