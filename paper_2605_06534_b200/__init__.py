"""B200-native sparse weight-delta sync (the data plane of ROSE's weight
transfer engine, arXiv 2605.06534) -- sm_100a kernels behind a C-ABI
(include/wsync.h) with a Python mirror of the reference's transfer API."""
from ._lib import (BF16, F32, I32, CapacityError, CudaError, IncompleteCoverage,  # noqa: F401
                   IndexOutOfShard, IndivisibleShape, InvalidArgument, NcclError,
                   IntegrityError, KeyFormatError, PayloadFormatError, RelayTimeout, ShapeMismatch,
                   TransferError, UnknownModuleKind)
from .codec import (SparseDelta, apply_delta, copy_overlap, diff_shards,  # noqa: F401
                    extract_shard, expert_thresholds, gen_pair_bf16, reslice_delta,
                    shard_shape)
from .engine import (EngineGroup, Plan, ServeConfig, TrainConfig, TransferEngine,  # noqa: F401
                     nccl_unique_id)
from . import wire  # noqa: F401
from .manifest import MODELS, ModuleKind, ParamMeta, toy_transformer_manifest  # noqa: F401
