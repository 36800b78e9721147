"""GEMEL merged-inference ORACLE -- test infrastructure, not product code.

Plain, slow, obviously-correct CPU implementation (NumPy, fp64) of what the
B200 path computes, written from PAPER.md (arXiv 2201.07705).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline / ``--impl
reference`` legs may import it.  It shares no code with the CUDA path
(``paper_2201_07705_b200``) and never imports it; the only common module is
``workloads`` (seeded input generators and model layer lists).

Modules
  ops    -- layer operators (direct convolution as a sum over taps, BN, pools, ...)
  model  -- layer-by-layer execution of one model, optional bf16-storage emulation
  merge  -- architectural signatures, group enumeration/sort, bytes-saved accounting,
            merged == unmerged-with-copied-weights
  plan   -- validator for execution plans dumped by the library

Parity status: every function is pinned by tests
under tests/test_oracle_*.py except where its docstring says "parity unpinned".
"""
