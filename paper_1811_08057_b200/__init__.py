"""B200-native matrix-condensation log-determinant (arXiv 1811.08057).

Drop-in for the hot path of the reference package ``mcnd``
(/root/reference/pkg/src/mcnd/__init__.py:4-65): switch
``from mcnd import logdet_condensation, mc_parallel`` to
``from paper_1811_08057_b200 import logdet_condensation, mc_parallel``.

Everything below the Python surface is sm_100a CUDA behind a C ABI
(include/mcnd_b200.h, csrc/); there is no CPU fallback.
"""

from .batched import logdet_batched
from .condense import SINGULAR, SINGULAR_RTOL, LogDet, SingularRowError, logdet_blocked, logdet_condensation
from .gauss import ge_parallel, logdet_lu
from .io import FormatError, read_matrix, read_matrix_device, write_matrix
from .matrix import GENERATOR_KINDS, MatrixSpec, as_matrix, generate, require_square
from .registry import ALGORITHMS, run_algorithm
from .runtime import CommStats, RunResult, WorkerPlan, mc_parallel, plan_blocks

__all__ = [
    "LogDet",
    "SINGULAR",
    "SINGULAR_RTOL",
    "SingularRowError",
    "logdet_condensation",
    "logdet_blocked",
    "logdet_batched",
    "mc_parallel",
    "logdet_lu",
    "ge_parallel",
    "plan_blocks",
    "WorkerPlan",
    "CommStats",
    "RunResult",
    "ALGORITHMS",
    "run_algorithm",
    "GENERATOR_KINDS",
    "MatrixSpec",
    "as_matrix",
    "generate",
    "require_square",
    "FormatError",
    "read_matrix",
    "read_matrix_device",
    "write_matrix",
]
