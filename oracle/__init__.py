"""CPU oracle for the CoFEM hot path -- TEST INFRASTRUCTURE ONLY.

This package restates, in numpy, the reference's covariance-free EM path
(/root/reference/pkg/src/sbl: cg.py, kernels.py, cofem.py, probes.py,
operators.py, problem.py).  It is the checker for the CUDA product path:
only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
/ ``--impl reference`` legs may import it.  The product package
``paper_2105_10439_b200`` never imports anything from here.

Parity pin: ``tests/golden/make_golden.py`` imports the real reference from
/root/reference (in the build container only) and records its outputs on
seeded inputs as ``tests/golden/*.npz``; ``tests/test_oracle_golden.py``
checks this restatement against those vectors.
"""

from .cofem_oracle import (  # noqa: F401
    CgConfig,
    CgReport,
    CofemConfig,
    DivergenceError,
    conv_op,
    dct_op,
    dense_op,
    draw_rademacher,
    e_step,
    estimate_diagonal_rademacher,
    make_preconditioner,
    m_step,
    m_step_nonneg,
    pcg_solve,
    run_cofem,
    run_cofem_multitask,
    substream,
    system_apply,
)
