"""B200-native MSD radix sort of fixed-size records (RADULS, arXiv 1612.02557).

The product is ``libraduls_gpu.so`` (C-ABI: ``include/raduls_gpu.h``; CUDA
kernels for sm_100a plus the C++ level planner under ``csrc/``). This package
is the thin Python mirror of the reference's interface used by tests, the
benchmark and the multi-GPU driver.
"""
from .raduls import (  # noqa: F401
    DIST_SKEW,
    DIST_UNIFORM,
    BigBinFraction,
    CudaError,
    LsdConfig,
    RecordLayout,
    ResourceError,
    SchedulerConfig,
    TinyPolicy,
    check_sorted,
    digest,
    generate,
    histogram,
    last_kernel_times,
    last_stats,
    local_capacity,
    rank_mode,
    launch_count,
    set_host_cache,
    lsd_sort,
    set_profiling,
    sort,
    sort_device,
    split,
)

from .records import FormatError, IoError, RecordArray, load_file, save_file  # noqa: F401,E402

__version__ = "0.1.0"
