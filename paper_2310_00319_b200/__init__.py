"""B200-native TVOLAP (time-variant overlap-add in partitions, arXiv 2310.00319).

The CUDA engine lives in lib/libtvolap_b200.so (sources in csrc/); `tvolap` is the
Python mirror of the reference's C++ operator interface over that C-ABI.
"""
from .tvolap import (  # noqa: F401
    CudaError,
    FrameAdapter,
    FilterPartitionSet,
    IncompatibleFilterError,
    InvalidConfigurationError,
    InvalidInputError,
    InvalidSizeError,
    InvalidSpectrumError,
    TvolapBankEngine,
    TvolapEngine,
    TvolapProcessor,
    forward_real,
    hann_window,
    inverse_real,
    is_power_of_two,
    mac,
    make_processor,
    partition,
)
