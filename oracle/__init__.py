"""CPU oracle for the GDRAA hot path -- TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this package.  The product (paper_1802_02326_b200/) never imports it.

Parity pins: every function here is pinned by `-m "not gpu"` tests in
tests/test_oracle_pins.py against values printed in the paper/SPEC (tests/golden/),
exact rational arithmetic, closed forms, invariants and library routines.  No function
is "parity unpinned".
"""
from .oracle import (  # noqa: F401
    F32, BF16, partition, bf16_to_f32, f32_to_bf16_rne, allreduce_mean, sgd_step, counters,
    lib_path, sgd_step_wd, poly_lr,
)
