"""CPU oracle for coefficient-domain multi-Gabor matching pursuit (arXiv 2202.12380).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import, call or
link anything under ``oracle/``.  The product path (``paper_2202_12380_b200``)
never touches it, and the oracle shares no code with the CUDA path.

Layout
  gabor.py    windows, DGT, Gram (cross-)kernels, synthesis  (numpy, fp64)
  mploop.c    the coefficient-domain MP loop, Alg. 1 + Alg. 3   (plain C99, fp64)
  loop.py     ctypes wrapper of mploop.c (+ build helper)
  dense.py    tiny-scale dense layer: materialised atoms, D^H x, dense Gram,
              exact signal-domain MP, literal dense Alg. 1 with G_eps

Every function cites the PAPER.md passage it follows (``P:<line>``).  Readings
where the paper is silent follow SURVEY.md §8(c) Z1..Z22 and are listed in
DESIGN.md §2.

Parity status: every oracle function is pinned by tests in
``tests/test_oracle_*.py`` against paper values, closed forms, identities or
brute force.  The one part the paper cannot pin beyond tiny scale is the
truncated-kernel loop at config scale (SURVEY.md §8(c) "O7 at eps>0, config
scale"): it is pinned at tiny scale against the literal dense Alg. 1 and only
self-consistency is checked at config scale ("parity unpinned" at config scale,
see DESIGN.md).
"""
from .gabor import (  # noqa: F401
    Setup, window, dgt, cross_kernel, kernels, layout, synthesize, analysis_all,
)
from .loop import mp_run, MpResult  # noqa: F401
