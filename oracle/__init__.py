"""ORACLE — test infrastructure only.

A plain, slow, obviously-correct CPU implementation of the RTG-SLAM mapping hot path
(arXiv 2404.19706; citations `P:n` are lines of the paper text PAPER.md, readings `Rn` are listed in
DESIGN.md §3), written in float64 PyTorch CPU ops from the paper and its readings.

Rules:
  * Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` / `--impl reference`
    legs may import this package.  The product path (`paper_2404_19706_b200`) never does and has
    no CPU fallback.
  * It shares no code with the CUDA path (no kernels, headers, tables or constant generators).
    The only shared module is `synth/` (seeded input data, no method arithmetic).
  * Gradients come from torch autograd through the float64 forward definition (not from a
    hand-derived backward); they are pinned by float64 finite differences in tests/.

Pins: see tests/test_oracle_*.py.  Functions without a pin say "parity unpinned" in their
docstring; at present none does except the whole-iteration timing trend (Table
`stable_gaussian_ablation`), which is a performance statement, not a value.
"""
from . import sh, projection, binning, raster, loss, optim, classify, state, insert, icp  # noqa: F401
