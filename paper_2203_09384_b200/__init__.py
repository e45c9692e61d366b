"""B200-native batched C2C FFT behind the reference ``stagefft`` plan/execute API.

Hot path of arxiv 2203.09384 (SYCL-FFT): batched 1-D complex-to-complex
power-of-two FFTs, N = 2..2048, single and double precision, forward and
inverse.  ``make_plan`` / ``execute`` / ``execute_timed`` /
``FourierTransformer`` keep the reference names and semantics
(/root/reference/pkg/src/stagefft/__init__.py:70-123 for the hot-path subset)
and run hand-written sm_100a CUDA kernels through the C ABI in
``include/sfft.h``.  There is no CPU fallback.
"""

from .errors import (
    ArgumentError,
    CudaError,
    DomainError,
    FftError,
    InsufficientDataError,
    InvalidLengthError,
    PlanError,
    ShapeError,
    UnsupportedLengthError,
)
from .executor import TimedExecution, execute, execute_timed, launch
from .kernels import (
    StageBuffer,
    count_butterflies,
    digit_reverse,
    radix2_stage,
    radix4_stage,
    radix8_stage,
    split_radix_transform,
)
from .numerics import TABLE_MAX_LENGTH, TwiddleTable, build_twiddle_table, is_power_of_two, twiddle
from .planner import (
    ENGINE_MAX_LENGTH,
    ENGINE_MIN_LENGTH,
    SUPPORTED_LENGTHS,
    SUPPORTED_RADICES,
    Algorithm,
    Direction,
    FftPlan,
    Precision,
    digit_reversal_permutation,
    factorize_stages,
    make_plan,
)
from . import sharding
from .bench import (
    BenchmarkRecord,
    BenchmarkResult,
    BenchmarkSummary,
    export_records,
    export_summaries,
    flag_outliers,
    load_records,
    run_benchmark,
    summarize,
)
from .sharding import execute_sharded, execute_shards, gather_rows, max_over_ranks, scatter_rows, shard_bounds
from .sigio import read_signal, write_signal
from .oracle import dft_matrix, naive_dft, naive_dft_batch
from .stats import (
    BatchReport,
    ChiSquareReport,
    Histogram,
    build_histograms,
    chi2_p_value,
    chi2_reduced,
    compare_spectra,
    lower_regularized_gamma,
    relative_difference,
    upper_regularized_gamma,
    verify_batch,
)
from .validation import COMPLEX_DTYPE, as_signal, check_same_length, check_signal_matrix
from .signalgen import KINDS, generate, generate_batch

try:
    from .estimator import FourierTransformer
except ImportError:  # pragma: no cover - sklearn is optional for the kernel path
    FourierTransformer = None

__version__ = "0.1.0"

__all__ = [
    "Algorithm",
    "ArgumentError",
    "BatchReport",
    "BenchmarkRecord",
    "BenchmarkResult",
    "BenchmarkSummary",
    "ChiSquareReport",
    "COMPLEX_DTYPE",
    "CudaError",
    "Direction",
    "DomainError",
    "ENGINE_MAX_LENGTH",
    "ENGINE_MIN_LENGTH",
    "FftError",
    "FftPlan",
    "FourierTransformer",
    "Histogram",
    "InsufficientDataError",
    "InvalidLengthError",
    "KINDS",
    "PlanError",
    "Precision",
    "SUPPORTED_LENGTHS",
    "SUPPORTED_RADICES",
    "ShapeError",
    "StageBuffer",
    "TABLE_MAX_LENGTH",
    "TimedExecution",
    "TwiddleTable",
    "UnsupportedLengthError",
    "as_signal",
    "build_histograms",
    "build_twiddle_table",
    "chi2_p_value",
    "chi2_reduced",
    "check_same_length",
    "check_signal_matrix",
    "compare_spectra",
    "count_butterflies",
    "dft_matrix",
    "digit_reversal_permutation",
    "digit_reverse",
    "execute",
    "execute_sharded",
    "execute_shards",
    "gather_rows",
    "scatter_rows",
    "execute_timed",
    "export_records",
    "export_summaries",
    "factorize_stages",
    "flag_outliers",
    "generate",
    "generate_batch",
    "is_power_of_two",
    "launch",
    "load_records",
    "lower_regularized_gamma",
    "make_plan",
    "max_over_ranks",
    "naive_dft",
    "naive_dft_batch",
    "radix2_stage",
    "radix4_stage",
    "radix8_stage",
    "read_signal",
    "relative_difference",
    "run_benchmark",
    "shard_bounds",
    "split_radix_transform",
    "summarize",
    "twiddle",
    "upper_regularized_gamma",
    "verify_batch",
    "write_signal",
]
