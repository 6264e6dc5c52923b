"""B200-native AdaPolySI Chebyshev-filter hot path (arxiv 2604.00914).

Host-side mirror of the reference's operator / filter API over the C-ABI of
libadp_b200.so (include/adp.h). The CUDA path is the only path: there is no
CPU fallback, and calls raise if the shared library is not built.
"""
from ._native import (AdpError, CollectiveError, ConfigError, CudaError, DimensionError, NotPositiveDefinite,
                      OutOfMemory, ParseError, lib)
from .bounds import (c_m_constant, damped_bound, inspect_filter, inspect_filter_csv, j_theta, projector_bound,
                     undamped_bound)
from .filter import (ChebFilter, SpectrumBounds, adaptive_degree, build_filter, chebyshev_step_coeffs,
                     eval_filter_scalar, initial_degree, jackson_damping, lanczos_damping)
from .operator import (Context, DeviceCsr, clenshaw_apply, clenshaw_apply_device, csr_spmv_device, default_context,
                       maspmm, maspmm_device)
from .hermitian import hermitian_embedding, solve_hermitian
from .report import RunReport, dump_report, run_report_from_json, run_solve, to_json
from .slicing import SlicedResult, balanced_slices, slice_interval, solve_sliced
from .solver import (IterationRecord, SolveResult, SolverConfig, StageTimings, cholesky_qr_device,
                     compute_residuals_device, estimate_eigcount, estimate_spectrum_bounds, rayleigh_ritz_device,
                     solve, spurious_threshold)
from .sparse import (CsrMatrix, fill_gaussian, fill_rademacher, parse_matrix_market, philox_block,
                     philox_gaussian, philox_uniform, read_matrix_market)

__all__ = [
    "SlicedResult", "balanced_slices", "slice_interval", "solve_sliced", "hermitian_embedding", "solve_hermitian",
    "RunReport", "dump_report", "run_report_from_json", "run_solve", "to_json",
    "c_m_constant", "damped_bound", "inspect_filter", "inspect_filter_csv", "j_theta", "projector_bound",
    "undamped_bound",
    "AdpError", "CollectiveError", "ConfigError", "CudaError", "DimensionError", "NotPositiveDefinite",
    "OutOfMemory", "ParseError", "lib", "ChebFilter", "SpectrumBounds", "adaptive_degree", "build_filter",
    "chebyshev_step_coeffs", "eval_filter_scalar", "initial_degree", "jackson_damping", "lanczos_damping",
    "Context", "DeviceCsr", "clenshaw_apply", "clenshaw_apply_device", "csr_spmv_device", "default_context", "maspmm",
    "maspmm_device", "CsrMatrix", "fill_gaussian", "fill_rademacher", "parse_matrix_market", "philox_block",
    "philox_gaussian", "philox_uniform", "read_matrix_market", "IterationRecord", "SolveResult", "SolverConfig",
    "StageTimings", "cholesky_qr_device", "compute_residuals_device", "estimate_eigcount",
    "estimate_spectrum_bounds", "rayleigh_ritz_device", "solve", "spurious_threshold",
]
