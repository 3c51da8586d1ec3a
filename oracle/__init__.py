"""PCR reuse-prefill ORACLE — test infrastructure, NOT part of the product.

A plain, slow, obviously-correct CPU implementation of what the hot path
computes, written from the paper (arXiv 2603.23049, /root/reference/PAPER.md;
cites are `P:<line>`, SPEC.md cites `S:<line>`).  Floating point is fp64.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import anything from here.  The CUDA product path
(`paper_2603_23049_b200/`) never imports it, and this package imports nothing
from the product path: the two share no code (only `pcrgen/`, the seeded input
generators, feeds both).

Modules
  chunks        O1  chunking and chained chunk keys            (Alg.1)
  tree          O2  prefix tree + look-ahead leaf-LRU planner   (Alg.1)
  brute         O2' independent stamp-based re-implementation + exhaustive checks
  kvload        O3  layer KV load / suffix append into the paged pool
  attention     O4  fp64 suffix-query causal attention (definition)
  tiny_model    O5  tiny fp64 transformer: reuse-then-attend == full recompute
  timing_model  O6  Eq.1 cost, layer-overlap recurrence and bounds

Pins: every function is pinned by tests under tests/ marked `not gpu` against
what the paper and mathematics fix.  The one
function without an external pin is listed in DESIGN.md as "parity unpinned".
"""
