"""B200-native TIDE per-token exit-decision hot path.

Drop-in for the routing / exit-selection / labelling path of the reference
`earlyexit` package (arxiv 2603.21365): same names, signatures and errors,
computed by hand-written sm_100a kernels in `_lib/libtide_b200.so` (C ABI:
include/tide_b200.h).  No CPU fallback.
"""

from ._device import invalidate_device_caches
from .bank_io import (BadMagicError, BinaryFormatError, ChecksumError, DimensionError,
                      TruncatedError, VersionError, bank_file_size, install_device_weights,
                      load_bank, save_bank)
from .calibration import (CalibrationConfig, CalibrationDataset, CollectedStates, RouterBank,
                          RouterStats, checkpoint_layers, compute_labels, label_tensors,
                          make_bank)
from .router_ops import (SMALL_BATCH_CUTOVER, CompactionResult, Router, batch_compact,
                         exit_projection, exit_scatter, fused_layernorm_route, route,
                         route_logits, route_scores)
from .runtime import (BATCH_UNANIMOUS, FINAL_KEY, MODES, NO_EXIT, PER_TOKEN, DecodeStep,
                      OutputHead, PhaseStats, RuntimeConfig, posthoc_select, select_exits)
from .tensor_math import DEFAULT_EPS, batched_cosine_similarity
from .training import TrainingDivergedError, train_router

__version__ = "0.1.0"

__all__ = [
    "CalibrationConfig", "CalibrationDataset", "CollectedStates", "RouterBank", "RouterStats",
    "checkpoint_layers", "compute_labels", "label_tensors", "make_bank",
    "SMALL_BATCH_CUTOVER", "CompactionResult", "Router", "batch_compact", "exit_projection",
    "exit_scatter", "fused_layernorm_route", "route", "route_logits", "route_scores",
    "BATCH_UNANIMOUS", "FINAL_KEY", "MODES", "NO_EXIT", "PER_TOKEN", "DecodeStep", "OutputHead",
    "PhaseStats",
    "RuntimeConfig", "posthoc_select", "select_exits",
    "DEFAULT_EPS", "batched_cosine_similarity", "__version__", "train_router",
    "TrainingDivergedError",
    "load_bank", "save_bank", "bank_file_size", "install_device_weights", "BinaryFormatError",
    "BadMagicError", "VersionError", "TruncatedError", "ChecksumError", "DimensionError",
    "invalidate_device_caches",
]
