"""CPU oracle for the B200 AGILE hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` legs may import, call, link or execute anything here, and only as the checker or the
timed CPU baseline — never as the product path.  The product (``paper_2504_19365_b200``) fails
loudly without its CUDA library and never routes through this package.

Contents (each function cites the reference file:line it restates):
  pages.py   synthetic page contents + raw image format (ssd_model.py:61-101)
  cache.py   serialized cache sequence: fully/set-associative clock (software_cache.py:91-126,
             355-456; SURVEY A.2 plug-in)
  audit.py   trace invariants (audit.py:25-175)
  ssd.py     device timing closed forms / small DES of the latency model (ssd_model.py:28-206)
  embbag.py  embedding-bag sums over paged tables (bench/sweeps.py stand-in; new op)
  graph.py   RMAT CSR, BFS levels, SpMV / PageRank (new; no reference ancestor)
  agile_oracle.c  C port of the paged embedding-bag through the set-associative clock cache,
             used as the timed CPU baseline (kind "port")

Parity pinning: tests/golden/make_golden.py runs the reference simulator itself (imported from
/root/reference/pkg/src in the build container) and commits its outputs as fixtures under
tests/golden/; tests/test_oracle_golden.py checks this oracle against every fixture.
"""
