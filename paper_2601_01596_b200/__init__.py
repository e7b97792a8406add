"""B200-native FFCz correction step (arXiv 2601.01596): C-ABI engine + Python host mirror.

See DESIGN.md for the path, the HBM layout and the kernels; INTEGRATION.md for the drop-in
boundary against the reference C++ API.
"""
from .ffcz import (  # noqa: F401
    Context, CorrectionResult, CudaError, DualBounds, EscapeEntry, FfczError, FormatError,
    ProjectionReport, SymmetryError, UnsupportedError, ValidationError, alternating_projection,
    apply_archive, correct, correct_batch, default_context, forward_dft, inverse_dft,
    Metrics, PowerSpectrum, UndefinedMetricError, metrics, power_spectrum,
    spectrum_bound_to_freq_bounds,
)

__all__ = [
    "Context", "CorrectionResult", "DualBounds", "EscapeEntry", "ProjectionReport", "FfczError",
    "ValidationError", "SymmetryError", "FormatError", "CudaError", "UnsupportedError",
    "correct", "correct_batch", "apply_archive", "alternating_projection", "forward_dft", "inverse_dft", "default_context",
    "Metrics", "PowerSpectrum", "UndefinedMetricError", "metrics", "power_spectrum",
    "spectrum_bound_to_freq_bounds",
]
