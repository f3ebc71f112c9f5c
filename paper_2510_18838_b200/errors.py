"""Exception types of the field-mapping path.

Same class names and hierarchy as the reference (fieldbridge/errors.py:4-64)
for the errors the hot path raises, so `except fieldbridge.errors.X` code
ports by changing the import.
"""


class FieldBridgeError(Exception):
    """Base class for all package errors (errors.py:4)."""


class MeshBuildError(FieldBridgeError):
    """Invalid mesh / point input (errors.py:8)."""


class FieldError(FieldBridgeError):
    """Field, mesh, or dof-layout mismatch (errors.py:22)."""


class UnderdeterminedError(FieldBridgeError):
    """Fewer support points than monomials for a fixed-radius fit (errors.py:26)."""


class InsufficientSourcesError(FieldBridgeError):
    """Adaptive radius exhausted the domain without reaching min_points (errors.py:30)."""


class SingularFitError(FieldBridgeError):
    """Rank-deficient local fit with no regularization (errors.py:34)."""


class ExtrinsicEvaluationError(FieldBridgeError):
    """A remote-evaluation callback failed. Carries the batch index (errors.py:59-64)."""

    def __init__(self, message, batch=None):
        super().__init__(message)
        self.batch = batch


class PartitionError(FieldBridgeError):
    """Invalid partition request (errors.py:51)."""


class ExchangeError(FieldBridgeError):
    """Routing plan and payload disagree (errors.py:55)."""
