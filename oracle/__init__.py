"""CPU oracle for the UniLab learner hot path -- TEST INFRASTRUCTURE ONLY.

This package is a plain numpy restatement of the reference algorithms
(`/root/reference/pkg/src/unilite`, cited file:line in every function of
:mod:`oracle.port`).  It exists to *check* the CUDA product path and to time
the reference's CPU learner in ``bench.py --impl reference``.

Rules (enforced by review):
  * only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
    ``cpu_baseline`` / ``--impl reference`` legs may import it;
  * the product package ``paper_2605_30313_b200`` never imports it and has no
    CPU fallback -- it fails loudly when its CUDA library is missing.

Pinning: ``tests/test_oracle_pinned.py`` checks this restatement against the
golden vectors in ``tests/golden/`` that ``tests/golden/gen_golden.py``
produced by running the unmodified reference in the build container, plus the
reference test-suite's own known answers.  LayerNorm (``ln_*``) has no
reference counterpart: its parity is **unpinned by the reference** and is
pinned only by central finite differences (tests/test_oracle_pinned.py).
"""

from . import port  # noqa: F401
