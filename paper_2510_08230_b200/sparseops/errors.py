"""Exception hierarchy with the reference's machine-readable ``kind`` strings.

Names and kinds match the reference one for one (sparseops/errors.py:8-131) so
code written against the reference catches the same classes; C status codes from
libsparseb200 map onto them in ``_lib.raise_for``.  Two kinds are new here:
``device-error`` (a CUDA runtime failure) and ``communication-error`` (NCCL).
"""


class SparseOpsError(Exception):
    """Base class of every library error."""

    kind = "error"


def _simple(name, kind, base=SparseOpsError, doc=None):
    cls = type(name, (base,), {"kind": kind, "__doc__": doc or f"kind = {kind!r}"})
    return cls


class _RowError(SparseOpsError):
    """An error tied to one matrix row (``.row``)."""

    _default = "error at row {row}"

    def __init__(self, row, message=None):
        super().__init__(message or self._default.format(row=row))
        self.row = row


InvalidArgumentError = _simple("InvalidArgumentError", "invalid-argument")
UnknownDeviceError = _simple("UnknownDeviceError", "unknown-device")
UnsupportedBackendError = _simple(
    "UnsupportedBackendError", "unsupported-backend",
    doc="A device name that exists in the wider ecosystem but not in this build.")
UnsupportedFeatureError = _simple("UnsupportedFeatureError", "unsupported-feature")
DimensionMismatchError = _simple("DimensionMismatchError", "dimension-mismatch")
PrecisionMismatchError = _simple("PrecisionMismatchError", "precision-mismatch")
IndexBoundsError = _simple("IndexBoundsError", "index-bounds")
NumericFailureError = _simple("NumericFailureError", "numeric-failure")
UndefinedBaselineError = _simple("UndefinedBaselineError", "undefined-baseline")
DeviceError = _simple("DeviceError", "device-error", doc="CUDA runtime failure.")
CommunicationError = _simple("CommunicationError", "communication-error",
                             doc="NCCL / torch.distributed failure in a partitioned solve.")

MatrixMarketError = _simple("MatrixMarketError", "mmio-malformed")
MalformedBannerError = _simple("MalformedBannerError", "mmio-bad-banner", MatrixMarketError)
MalformedSizeError = _simple("MalformedSizeError", "mmio-bad-size", MatrixMarketError)
EntryCountError = _simple("EntryCountError", "mmio-entry-count", MatrixMarketError)
UnsupportedFieldError = _simple("UnsupportedFieldError", "mmio-unsupported-field",
                                MatrixMarketError)


class SingularDiagonalError(_RowError):
    kind = "singular-diagonal"
    _default = "zero or missing diagonal at row {row}"


class SingularTriangleError(_RowError):
    kind = "singular-triangle"
    _default = "zero diagonal in triangular solve at row {row}"


class NotTriangularError(_RowError):
    kind = "not-triangular"
    _default = "entry on the wrong side of the diagonal in row {row}"


class ZeroPivotError(_RowError):
    kind = "zero-pivot"
    _default = "zero pivot at row {row}"


class IndefinitePivotError(_RowError):
    kind = "indefinite-pivot"
    _default = "non-positive pivot at row {row}"


class BreakdownError(SparseOpsError):
    """Krylov recurrence broke down (zero or indefinite denominator); ``.iteration``."""

    kind = "breakdown"

    def __init__(self, iteration, message=None):
        super().__init__(message or f"solver breakdown at iteration {iteration}")
        self.iteration = iteration


class ConfigError(SparseOpsError):
    """Configuration tree rejected; ``.path`` locates the offending key."""

    kind = "config-invalid"

    def __init__(self, path, message):
        super().__init__(f"{path}: {message}")
        self.path = path
