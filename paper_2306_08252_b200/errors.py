"""Error taxonomy of the reference (proj/include/dyngraph/types.hpp:19-32)."""


class Error(RuntimeError):
    """Base class for all library errors (types.hpp:19-22)."""


class DataError(Error):
    """Malformed input: invalid CSR batches, bad ids (types.hpp:24-27)."""


class EngineError(Error):
    """Resource exhaustion or a violated structural contract (types.hpp:29-32)."""


class CudaError(Error):
    """A CUDA runtime call failed (no reference counterpart)."""
