"""swe-b200: B200-native (sm_100a) executor for the 2D shallow-water MacCormack
time step of arXiv 1309.1230, behind the reference solver's Stepper API.

The product path is libswe_cuda.so (paper_1309_1230_b200/lib/), built by
__graft_entry__.build().  There is no CPU fallback.
"""
from .stepper import (BoundaryKind, BoundarySet, ConfigError, ExecutorKind, FieldSet, GridSpec,  # noqa: F401
                      InitialCondition, InstabilityError, IoError, PhysicsParams, RunResult, StabilityPolicy,
                      StepCollapseError,
                      Stepper, StepResult, partition_scanlines)

__version__ = "0.1.0"
