"""paper_2509_10722_b200 -- B200-native (sm_100a) proximal message passing
(PMP / over-relaxed ADMM) for network utility maximization.

A drop-in for the reference numpmp engine's hot path
(proj/include/numpmp/solver.hpp:265-519): the same Problem / SolverConfig /
SolverState / Solution types and PmpSolver members, with every iteration
running as hand-written CUDA kernels behind the C-ABI in
include/numpmp_gpu.h.
"""
from .errors import DeviceError, DomainError, GenError, IoError, SolverError, ValidationError
from .model import (
    GenKind,
    GenSpec,
    Problem,
    Stream,
    StreamKind,
    TerminalLayout,
    TransitMetadata,
    TransitSpec,
    TypeGroup,
    WeightDist,
    build_problem,
    PruneMap,
    degrade,
    fail_and_prune,
    gen_congested,
    gen_transit,
    gen_uncongested,
    group_streams,
    problem_from_arrays,
    read_problem,
    validate,
    write_problem,
)
from .solver import (
    PmpSolver,
    Solution,
    SolverConfig,
    SolverState,
    SolveStatus,
    TraceRecord,
    WarmStart,
    check_termination,
    objective,
    recover_duals,
    to_string,
    update_rho,
)
from .transit import (
    TransitReportRow,
    normalized_route_prices,
    read_transit_metadata,
    transit_report,
    write_transit_metadata,
    write_trace_csv,
    write_transit_report_csv,
)

__all__ = [
    "DeviceError", "DomainError", "GenError", "IoError", "SolverError", "ValidationError",
    "GenKind", "GenSpec", "Problem", "Stream", "StreamKind", "TerminalLayout", "TransitMetadata", "TransitSpec", "TypeGroup", "WeightDist",
    "build_problem", "degrade", "fail_and_prune", "PruneMap", "gen_congested", "gen_transit", "gen_uncongested", "group_streams", "problem_from_arrays", "read_problem", "validate", "write_problem",
    "PmpSolver", "Solution", "SolverConfig", "SolverState", "SolveStatus", "TraceRecord", "WarmStart",
    "check_termination", "objective", "recover_duals", "to_string", "update_rho",
    "TransitReportRow", "normalized_route_prices", "transit_report", "write_trace_csv", "write_transit_report_csv",
    "read_transit_metadata", "write_transit_metadata",
]
