"""Error contract of the drop-in boundary.

The reference's Newton driver (newton.py:401-414) catches exactly these
classes to cut the timestep, so the GPU path raises the *same* classes: when
the reference package ``iscsim`` is importable its classes are re-exported
(a drop-in installed into a reference run must raise what it catches);
otherwise structurally identical local classes are defined, following
errors.py:39-88 of the reference.
"""

try:  # pragma: no cover - depends on whether the reference is importable
    from iscsim.errors import (  # type: ignore
        Breakdown,
        DegenerateTemperature,
        DivergedResidual,
        MaxIterations,
        PhysicsError,
        PoreSpaceExhausted,
        SimulationStalled,
        SingularCellBlock,
        SinkFailure,
        SolverError,
    )
except Exception:  # the GPU box has no reference checkout
    class PhysicsError(Exception):
        """Failures of the physical state or time stepping (errors.py:39)."""

    class PoreSpaceExhausted(PhysicsError):
        """Coke fills the pore volume (errors.py:43)."""

    class DegenerateTemperature(PhysicsError):
        """T - kv5 <= 0 in the K-value correlation (errors.py:47)."""

    class DivergedResidual(PhysicsError):
        """Residual grew for several consecutive iterations (errors.py:55)."""

    class SimulationStalled(PhysicsError):
        """Timestep cut below the minimum (errors.py:59)."""

        def __init__(self, message, cause=None):
            super().__init__(message)
            self.cause = cause

    class SolverError(Exception):
        """Linear-algebra failures (errors.py:71)."""

    class SingularCellBlock(SolverError):
        """Diagonal block could not be pivoted (errors.py:75)."""

    class Breakdown(SolverError):
        """BiCGSTAB breakdown after the restart (errors.py:79)."""

    class MaxIterations(SolverError):
        """Krylov iteration limit reached (errors.py:83)."""

    class SinkFailure(OSError):
        """A report sink could not be created or written (errors.py:91)."""


class NativeLibraryMissing(RuntimeError):
    """The sm_100a shared library is not built / not loadable.

    The product path has no CPU fallback: every entry point raises this
    instead of computing anything on the host.
    """


__all__ = [
    "Breakdown", "DegenerateTemperature", "DivergedResidual", "MaxIterations",
    "NativeLibraryMissing", "PhysicsError", "PoreSpaceExhausted",
    "SimulationStalled", "SingularCellBlock", "SolverError",
]
