"""B200-native gZCCL: error-bounded compression and compression-enabled collectives.

Drop-in for the hot path of the reference ``gzccl`` package
(/root/reference/pkg/src/gzccl): the codec API (``compress`` /
``decompress`` / ``compress_blocks`` / ``decompress_block``, same byte format)
and the compressed ring Allreduce / binomial Scatter, running as hand-written
sm_100a kernels (``libgzccl.so``) over NVLink peer memory.
"""

from .codec import (
    BLOCK,
    HEADER_BYTES,
    MAGIC,
    MAX_STEP,
    RAW_WIDTH,
    BlockTable,
    DecodeError,
    DeviceBlob,
    Workspace,
    compress,
    compress_blocks,
    decompress,
    decompress_block,
    fixed_rate_compress,
    fixed_rate_decompress,
    worst_case_blob_bytes,
)
from .collectives import CommunicatorSpec, Network, create_network, run_collective
from .collectives import Counters as OpCounters
from .costmodel import CostParams, b200_cost_params, load_cost_params, predicted_makespan
from .metrics import AccuracyStats, CollectiveReport, compression_ratio, max_abs_error, psnr

__version__ = "0.1.0"

__all__ = [
    "AccuracyStats",
    "CollectiveReport",
    "CommunicatorSpec",
    "CostParams",
    "b200_cost_params",
    "load_cost_params",
    "predicted_makespan",
    "Network",
    "OpCounters",
    "compression_ratio",
    "create_network",
    "max_abs_error",
    "psnr",
    "run_collective",
    "BLOCK",
    "HEADER_BYTES",
    "MAGIC",
    "MAX_STEP",
    "RAW_WIDTH",
    "BlockTable",
    "DecodeError",
    "DeviceBlob",
    "Workspace",
    "compress",
    "compress_blocks",
    "fixed_rate_compress",
    "fixed_rate_decompress",
    "decompress",
    "decompress_block",
    "worst_case_blob_bytes",
]
