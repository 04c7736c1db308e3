"""CPU oracle for the quantised tensor-adapter linear — TEST INFRASTRUCTURE ONLY.

Nothing in the product package (`paper_2402_13533_b200`) imports this package.
Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU-baseline /
`--impl reference` legs may use it, and only as the checker or as the timed CPU
reference, never as a fallback for the CUDA path.

The oracle is a numpy (float64) restatement of the reference package `lrlm`
(`/root/reference/pkg/src/lrlm`), each function citing the file:line it
follows.  It is pinned against the reference itself: `oracle/gen_golden.py`
imports `lrlm` in the build container and writes `tests/golden/*.npz`, and
`tests/test_oracle_golden.py` checks the restatement against those fixtures
(bit-exact for codes / scales / offsets, 1e-12 relative for float64 results).
Pieces the reference does not implement (TT adapter, per-token act-quant in the
forward, int32 accumulators, MSE, merge onto a quantised base) are restated
from SURVEY.md §8(c) and anchored to reference code where a special case
exists (LoRA == 2-core TT is checked against `LoraLinear`, transformer.py:276-327).
"""

from .qa_oracle import *  # noqa: F401,F403
