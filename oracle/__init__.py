"""LLEP oracle -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.

A plain, slow, float64 CPU implementation of what the LLEP hot path computes,
written from PAPER.md (arxiv 2601.17111).  Only `tests/`, `__graft_entry__.smoke()`
and `bench.py`'s `cpu_baseline` / `--impl reference` legs may import it.  It
shares no code with the CUDA path (`paper_2601_17111_b200/`), and the CUDA path
never imports it.

    O1  planner.py   Alg. 4 head (λ test), Alg. 2 LLA,
                     Alg. 3 LLAS, weight-transfer plan
    O2  schedule.py  load matrix, stable re-indexing,
                     per-slot destinations from the plan
    O3  layer.py     Eq. 1 with SwiGLU experts, float64
    O4  simulate.py  Alg. 1 / Alg. 4 executed per simulated device
    O5  backward.py  gradients of Eq. 1 + spilled-expert weight-gradient return
    O6  router.py    the router of Eq. 2: softmax over N, top-K, gates = s

Pins (tests/test_oracle_*.py, `-m "not gpu"`): SPEC hand traces (tests/golden/),
the §2.1 worked example, closed-form load accounting, invariants,
brute force on tiny inputs, textbook reductions.  See DESIGN.md §Oracle.
"""
