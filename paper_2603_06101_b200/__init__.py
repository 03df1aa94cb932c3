"""B200-native SBCI sigma/update hot path (arXiv 2603.06101) — drop-in for the reference's FCI
operator and the SBCI1 / SBCI2 / Davidson drivers. Product path: libsbg.so (sm_100a CUDA kernels + C++ host driver),
reached through the C ABI in include/sbg.h. No CPU fallback."""
from .fci import (K_DEFAULT_DETERMINANT_GUARD, FciOperator, FciProblem, FcidumpError, as_operator, binomial,
                  determinant_count, parse_fcidump, parse_fcidump_file, sigma_apply, synthetic_problem)
from .solver import (ConvergedEigenpair, MultiStateResult, NonConvergenceError, RunSummary, SolverConfig,
                     StateSummary, TraceRecord, solve_n_states_sbci1, solve_n_states_sbci2,
                     davidson_solve, solve_state_sbci1, Sbci1Result)
from .trace import (CsvTraceSink, MemoryTraceSink, TeeTraceSink, read_trace_csv, read_trace_csv_file,
                    trace_csv_header)

__all__ = ["K_DEFAULT_DETERMINANT_GUARD", "FciOperator", "FciProblem", "FcidumpError", "as_operator", "binomial",
           "determinant_count", "parse_fcidump", "parse_fcidump_file", "sigma_apply", "synthetic_problem",
           "ConvergedEigenpair", "MultiStateResult", "NonConvergenceError", "RunSummary", "SolverConfig",
           "StateSummary", "TraceRecord", "solve_n_states_sbci1", "solve_n_states_sbci2",
           "davidson_solve", "solve_state_sbci1", "Sbci1Result", "CsvTraceSink", "MemoryTraceSink", "TeeTraceSink", "read_trace_csv",
           "read_trace_csv_file", "trace_csv_header"]
