"""CPU oracle — TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU-baseline /
`--impl reference` legs may import this package, and only as the checker or
the timed reference arm.  The product (`paper_2110_04421_b200`) never imports
it; its hot path fails loudly without the CUDA library.

Contents (each function cites the reference file:line it restates):
  rng_np        keyed splitmix draws           (pkg/src/epivec/rng.py)
  engine_np     Engine.step / gather_exposure  (pkg/src/epivec/engine.py)
  confignet_np  CPU restatement of this framework's config-network generator
                (BASELINE.json configs 0-4; no reference counterpart)

Parity status: pinned.  `tests/golden/` holds vectors produced by running the
unmodified reference (`tests/golden/make_golden.py`) and
`tests/test_oracle_golden.py` checks this oracle against every one of them.
"""
