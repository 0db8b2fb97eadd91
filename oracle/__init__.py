"""CPU oracle for the GPipe hot path of arXiv 2004.09910 (torchgpipe).

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` legs may import anything under `oracle/`.  The product
path (`paper_2004_09910_b200/`, `include/`, the CUDA library) shares no code with it and
never calls it.

Plain, slow, obviously-correct numpy float64 (+ Python loops for small cases).  Each
function cites the PAPER.md passage (`P:line`, section / equation / algorithm) it
follows; where the paper is silent the reading is SURVEY.md §8(c) Z-n, listed in DESIGN.md.

Modules
  schedule  Alg. 1 clock cycles, mirrored backward, checkpoint policy, O5 record list,
            micro-batch split (O7), per-device projection (O11)
  balance   min-max contiguous block partition (O6) + brute force
  philox    Philox4x32-10 counter-based RNG and the dropout mask rule (O8)
  model     full-batch fp64 forward / loss / backward / SGD (O2-O4, O9)
  emulator  executes the O5 records on micro-batches (O10)

Pins (what each part is checked against) live in tests/test_oracle_*.py; every function
here is pinned -- none is "parity unpinned".
"""
