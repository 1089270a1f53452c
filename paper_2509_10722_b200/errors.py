"""Exception types of the reference (proj/include/numpmp/common.hpp:11-43),
plus the mapping from the C-ABI return codes (include/numpmp_gpu.h)."""


class ValidationError(RuntimeError):
    """Invalid model data (common.hpp:14-18)."""


class SolverError(RuntimeError):
    """Numerical failure inside the solver (common.hpp:20-25)."""


class GenError(RuntimeError):
    """Invalid generator specification (common.hpp:38-43)."""


class IoError(RuntimeError):
    """Problem / solution file errors (common.hpp:32-36)."""


class DomainError(ValueError):
    """std::domain_error (e.g. warm start with a non-positive log rate)."""


class DeviceError(RuntimeError):
    """CUDA / NCCL failure of the device engine (no reference counterpart)."""


def raise_for(code: int, message: str) -> None:
    if code == 0:
        return
    if code == 1:
        raise ValueError(message)  # std::invalid_argument
    if code == 2:
        raise ValidationError(message)
    if code == 3:
        raise SolverError(message)
    if code == 4:
        raise DomainError(message)  # std::domain_error
    raise DeviceError(f"[{code}] {message}")
