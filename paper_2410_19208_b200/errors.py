"""Exception hierarchy of the reference (psdcone/errors.py:4-49), same names.

The C ABI returns integer status codes (include/psdproj.h ``psd_status``);
``raise_for_status`` maps them onto these classes.  ``install()`` (see
``paper_2410_19208_b200.install``) re-points ``REGISTRY`` at the reference's
own classes so callers catching ``psdcone.AlphaTooSmall`` keep working.
"""


class PsdconeError(Exception):
    """Base class for all errors raised by this package."""


class NonSquareError(PsdconeError):
    """A square matrix was required but the operand is rectangular."""


class AsymmetricMatrixError(PsdconeError):
    """The operand exceeds the symmetry tolerance and was rejected."""


class ConvergenceFailure(PsdconeError):
    """An underlying iterative eigensolver failed to converge."""


class RankDeficientSample(PsdconeError):
    """Sampled sketch has numerical rank below the requested width (strict mode)."""


class AlphaTooSmall(PsdconeError):
    """Scaling factor is numerically zero; the input is already (numerically) PSD."""


class InvalidParams(PsdconeError):
    """Parameters outside the domain of a bound or algorithm."""


class DimensionMismatch(PsdconeError):
    """Operands have incompatible dimensions."""


class DeviceError(PsdconeError):
    """CUDA runtime failure inside libpsdproj (no reference analogue)."""


# status code → class name (include/psdproj.h enum psd_status)
STATUS_NAMES = {
    1: "InvalidParams",
    2: "AsymmetricMatrixError",
    3: "RankDeficientSample",
    4: "AlphaTooSmall",
    5: "ConvergenceFailure",
    6: "NonSquareError",
    7: "DeviceError",
    8: "DeviceError",
}

REGISTRY = {
    "PsdconeError": PsdconeError,
    "NonSquareError": NonSquareError,
    "AsymmetricMatrixError": AsymmetricMatrixError,
    "ConvergenceFailure": ConvergenceFailure,
    "RankDeficientSample": RankDeficientSample,
    "AlphaTooSmall": AlphaTooSmall,
    "InvalidParams": InvalidParams,
    "DimensionMismatch": DimensionMismatch,
    "DeviceError": DeviceError,
}


def error(name, message):
    """Instance of the registered class called ``name``."""
    return REGISTRY[name](message)


def raise_for_status(status, message):
    if status == 0:
        return
    raise error(STATUS_NAMES.get(status, "DeviceError"), message)
