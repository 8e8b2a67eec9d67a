"""B200-native Dr. Top-k (arXiv 2109.08219): drop-in for the reference ``dtopk``.

    import paper_2109_08219_b200 as dtopk
    r = dtopk.dr_topk(v, dtopk.PipelineConfig(k=1024))      # v: numpy / torch (CPU or CUDA)
    r.values, r.indices, r.threshold, r.stats

Same entry point, config and errors as the reference package
(pkg/src/dtopk/__init__.py); the data path is hand-written sm_100a CUDA in
``_lib/libdtopk.so`` (C ABI: include/dtopk.h).  Additions: float32 keys,
``PipelineConfig.largest`` and ``TopKResult.indices``.
"""

from .core import (
    BACKENDS,
    ELEMENT_DTYPE,
    STAGES,
    DtopkError,
    EmptyInput,
    InvalidBeta,
    InvalidK,
    PipelineConfig,
    TopKResult,
    WorkloadStats,
    delegate_vector_len,
    effective_beta,
    ensure_vector,
    validate_config,
)
from .delegate import DelegateVector, extract_delegates, extract_delegates_blocked
from .distributed import (
    DistributedReport,
    GatherMessage,
    PartitionPlan,
    ShardedTopK,
    WorkerFailed,
    plan,
    run_distributed,
    shard_bounds,
    sharded_topk,
)
from .kernels import KeyedEntry, kth_largest, radix_topk
from .pipeline import DrTopK, QualificationReport, concatenate_filtered, dr_topk, first_topk
from .tuning import auto_alpha

__version__ = "0.1.0"

__all__ = [
    "BACKENDS",
    "ELEMENT_DTYPE",
    "STAGES",
    "DelegateVector",
    "DrTopK",
    "DtopkError",
    "EmptyInput",
    "InvalidBeta",
    "InvalidK",
    "KeyedEntry",
    "DistributedReport",
    "GatherMessage",
    "PartitionPlan",
    "run_distributed",
    "ShardedTopK",
    "PipelineConfig",
    "QualificationReport",
    "TopKResult",
    "WorkerFailed",
    "WorkloadStats",
    "auto_alpha",
    "concatenate_filtered",
    "delegate_vector_len",
    "dr_topk",
    "effective_beta",
    "ensure_vector",
    "extract_delegates",
    "extract_delegates_blocked",
    "first_topk",
    "kth_largest",
    "plan",
    "radix_topk",
    "shard_bounds",
    "sharded_topk",
    "validate_config",
]
