"""B200-native DLRM query hot path for Hercules-style recommendation serving.

The product is libhercules_rec.so (C ABI in include/rec.h: hand-written sm_100a
kernels + C++ serving runtime); this package only builds it (build.py) and binds it
(binding.py, ctypes marshalling).  It never imports the oracle.
"""
from .binding import (RecModel, RecError, lib, nccl_unique_id, rec_split_fuse, rec_shard_plan, EXPORTS, STATUS,  # noqa: F401
                      rec_global_batches,
                      REC_VALUES_INT8_EXACT, REC_VALUES_FP32, REC_INDEX_UNIFORM, REC_INDEX_SKEW2,
                      REC_SHARD_REPLICA, REC_SHARD_TABLE, REC_SHARD_ROW, REC_INPUT_DEVICE_SYNTH,
                      REC_INPUT_HOST, REC_CLOCK_REAL, REC_CLOCK_VIRTUAL, KERNEL_SLS, KERNEL_GEMM,
                      KERNEL_INTERACT, KERNEL_GEN)
