"""B200-native GPS L1 C/A acquisition -- drop-in for gnssperf's acquisition path.

Importing the package loads libgacq.so (hand-written sm_100a CUDA behind a C ABI,
include/gacq.h). There is no CPU fallback: without the built library the import fails.
"""

from .acquisition import (  # noqa: F401
    AcqConfig,
    AcqEngine,
    AcqResult,
    BatchResult,
    PinnedBuffer,
    acquire_all,
    acquire_batch,
    acquire_bins_sharded,
    acquire_channel,
    acquire_if_file,
    conjugate_code_spectrum,
    default_doppler_step_hz,
    get_engine,
    merge_bin_shards,
    samples_per_code_period,
)
from .buffers import IqBuffer, Precision  # noqa: F401
from .synth import SAT_DTYPE, random_sats, synthesize_batch  # noqa: F401
from .iffile import IfPayload, read_if_file, read_if_payload, write_if_file  # noqa: F401
from .cacode import CHIP_RATE_HZ, CODE_LENGTH, CaCode, generate_ca_code  # noqa: F401
from .errors import (  # noqa: F401
    FormatError,
    GnssPerfError,
    InvalidInputError,
    PipelineError,
    ResourceError,
    UnsupportedError,
)

__version__ = "0.1.0"
