"""B200-native AB-Sparse decode-time block-sparse attention (sm_100a CUDA behind a C ABI).

See DESIGN.md. The numeric path lives in lib/libabsp.so (built from csrc/ by
build.py); this package is the Python host mirror of the reference API.
"""
from .absparse import (BlockAssignment, CentroidMethod, DecodeAttention, DecodeEngine, EngineConfig,  # noqa: F401
                       QuantMode, QuantSpec, StepResult, build_offsets, fill_synthetic_bf16)
from .calibration import (CalibrationReport, RecallTable, Trace, TransferReport, assign_block_sizes,  # noqa: F401
                          load_trace, make_report, normalized_recall, profile_sample, profile_sensitivity,
                          save_trace, topk_page_recall, topk_page_recall_per_head, transfer_check,
                          write_min_block_csv, write_recall_csv)
from ._abi import (AbspError, CapacityError, CudaError, InvalidArgument, LogicError,  # noqa: F401
                   OutOfRange)

__all__ = ["BlockAssignment", "CentroidMethod", "DecodeAttention", "DecodeEngine", "EngineConfig", "QuantMode",
           "QuantSpec", "StepResult", "build_offsets", "fill_synthetic_bf16", "AbspError", "CapacityError",
           "CudaError", "InvalidArgument", "LogicError", "OutOfRange", "CalibrationReport", "RecallTable", "Trace",
           "TransferReport", "assign_block_sizes", "load_trace", "make_report", "normalized_recall",
           "profile_sample", "profile_sensitivity", "save_trace", "topk_page_recall", "topk_page_recall_per_head",
           "transfer_check", "write_min_block_csv", "write_recall_csv"]
