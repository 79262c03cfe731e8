"""CPU oracle for the eager-SGD partial-collective hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in the product package
(`paper_1908_04207_b200/`) imports, links or executes anything in this
directory.  Only `tests/`, `__graft_entry__.smoke()` and the `cpu_baseline` /
`--impl reference` legs of `bench.py` use it -- as the checker and as the timed
CPU baseline, never as the measured or shipped path.

* `restated.py` -- numpy restatement of the reference algorithm
  (`/root/reference/pkg/src/eagercoll`), each function citing the reference
  file:line it follows.  Dtype-generic: f64 reproduces the reference engine
  bit for bit, f32 is the product's arithmetic.
* `gen_golden.py` -- runs the reference itself (container only) and writes the
  fixtures under `tests/golden/` that pin the restatement (parity pinned: see
  `tests/test_oracle_golden.py`).
* `cpu_baseline.py` -- the reference CPU path timed on host cores for bench.py.
"""
