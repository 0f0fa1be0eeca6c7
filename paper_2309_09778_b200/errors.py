"""Exception families of the reference package (errors.py:1-129), plus the
1:1 mapping of C-ABI status codes (include/permez_b200.h) onto them.

The class names and family structure are the reference's public API; the
``status_error`` helper is the boundary that turns a negative ``pmz_status``
into the exception the reference would raise.
"""
from __future__ import annotations


class PermezError(Exception):
    """Base class for all errors raised by this package (errors.py:4)."""


def _family(name: str, doc: str):
    return type(name, (PermezError,), {"__doc__": doc})


ConfigError = _family("ConfigError", "Invalid user-supplied configuration (bounds, dims, flags).")
DataError = _family("DataError", "Problems with the numeric content of input data.")
TrainingError = _family("TrainingError", "Trainer failures.")
CodingError = _family("CodingError", "Entropy coding failures.")
ContainerError = _family("ContainerError", "Container framing failures.")
IngestError = _family("IngestError", "Input file failures.")


def _leaf(name: str, base: type, doc: str = ""):
    return type(name, (base,), {"__doc__": doc or name})


NonFiniteInput = _leaf("NonFiniteInput", DataError, "NaN or Inf encountered where finite values are required.")
DegenerateBlock = _leaf("DegenerateBlock", DataError, "Block contains no nonzero element; use the trivial-block path.")
SubnormalMinimum = _leaf("SubnormalMinimum", DataError, "Smallest nonzero magnitude is at or below the floor.")
NonRepresentableFactor = _leaf("NonRepresentableFactor", DataError, "factor_neg overflows the 64-bit float range.")
DivergedTraining = _leaf("DivergedTraining", TrainingError)
EmptyDataset = _leaf("EmptyDataset", TrainingError)
TooFewBlocks = _leaf("TooFewBlocks", TrainingError, "Fewer than the minimum sampled blocks for an 8:2 split.")
SweepExhausted = _leaf("SweepExhausted", TrainingError)
BalanceFlagNotDequantizable = _leaf("BalanceFlagNotDequantizable", CodingError,
                                    "Code 0 flags an unpredictable point and carries no residual.")
DegenerateAlphabet = _leaf("DegenerateAlphabet", CodingError, "Fewer than two symbols have nonzero frequency.")
UnassignedCode = _leaf("UnassignedCode", CodingError, "A symbol has no codeword in the codebook.")
TruncatedStream = _leaf("TruncatedStream", CodingError, "Bit stream ended inside a codeword.")
InvalidPrefix = _leaf("InvalidPrefix", CodingError, "Bits do not match any codeword (corrupted input).")
BadMagic = _leaf("BadMagic", ContainerError)
UnsupportedVersion = _leaf("UnsupportedVersion", ContainerError)
Corrupt = _leaf("Corrupt", ContainerError, "Structural inconsistency: lengths, offsets, counts, or padding.")
BalanceUnderflow = _leaf("BalanceUnderflow", ContainerError,
                         "More balance-point flags in the code stream than stored values.")
UnsupportedFormatCode = _leaf("UnsupportedFormatCode", IngestError)
TruncatedFile = _leaf("TruncatedFile", IngestError)
InconsistentTraceLength = _leaf("InconsistentTraceLength", IngestError)
SizeMismatch = _leaf("SizeMismatch", IngestError)
DimensionMismatch = _leaf("DimensionMismatch", IngestError)


class CapacityExceeded(PermezError):
    """Output buffer smaller than the container (device boundary only)."""


class DeviceError(PermezError):
    """CUDA runtime failure or missing native library."""


_STATUS = {
    -1: ConfigError,
    -2: NonFiniteInput,
    -3: DegenerateBlock,
    -4: SubnormalMinimum,
    -5: NonRepresentableFactor,
    -6: TooFewBlocks,
    -7: BalanceFlagNotDequantizable,
    -8: DegenerateAlphabet,
    -9: UnassignedCode,
    -10: TruncatedStream,
    -11: InvalidPrefix,
    -12: BadMagic,
    -13: UnsupportedVersion,
    -14: Corrupt,
    -15: BalanceUnderflow,
    -16: CapacityExceeded,
    -17: DeviceError,
    -18: DeviceError,
    -19: DeviceError,
}

# CLI exit codes per family: stable, one per family.
EXIT_CODES = {ConfigError: 2, DataError: 3, TrainingError: 4, CodingError: 5, ContainerError: 6, IngestError: 7,
              PermezError: 1}


def status_error(status: int, what: str = "") -> PermezError:
    cls = _STATUS.get(int(status), DeviceError)
    return cls(f"{what}: status {status} ({cls.__name__})" if what else f"status {status}")


def check(status: int, what: str = "") -> None:
    if status != 0:
        raise status_error(status, what)


def exit_code(exc: BaseException) -> int:
    for cls in type(exc).__mro__:
        if cls in EXIT_CODES:
            return EXIT_CODES[cls]
    return 1
