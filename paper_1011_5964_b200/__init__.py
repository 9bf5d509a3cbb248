"""B200-native PCG hot path of the TV deblurring solver (arXiv 1011.5964).

Drop-in mirror of the reference package ``tvdeblur``'s hot-path API
(``pcg``, ``StructuredBlurOperator``, ``DiffusionOperator``,
``FactoredPreconditioner`` / ``assemble_preconditioner``, ``restore``) over
hand-written sm_100a CUDA kernels reached through the C ABI declared in
``include/tvdeblur_b200.h`` (``libtvdeblur_b200.so``).  There is no CPU
fallback: operators raise when the library or a CUDA device is missing.
"""

from .blur import BoundaryCondition, StructuredBlurOperator, SymmetricPsf
from .krylov import KrylovConfig, SolveOutcome, pbicgstab, pcg
from .pipeline import (ConfigurationError, Formulation, InvalidScalingError, NormalSystem,
                       PrecondSelector, RestorationConfig,
                       RestorationReport, restore)
from .precond import FactoredPreconditioner, assemble_preconditioner
from .transforms import TransformKind
from .tv import DiffusionBc, DiffusionOperator

__all__ = [
    "BoundaryCondition", "ConfigurationError", "DiffusionBc", "DiffusionOperator", "FactoredPreconditioner",
    "Formulation", "InvalidScalingError", "KrylovConfig", "NormalSystem", "PrecondSelector", "RestorationConfig",
    "RestorationReport", "SolveOutcome", "StructuredBlurOperator", "SymmetricPsf",
    "TransformKind", "assemble_preconditioner", "pbicgstab", "pcg", "restore",
]
