"""B200-native METIS per-query hot path (arXiv 2412.10543).

Drop-in for the data-parallel path of the reference package ``ragsched``:
confidence gate + Algorithm-1 pruning, KV-memory / delay cost models,
best-fit + fallback selection, and FAISS-``IndexFlatL2``-style dense
retrieval, all computed by hand-written sm_100a kernels in
``libragsched_b200.so`` (C ABI: ``include/ragsched_b200.h``).

Names mirror the reference's namespace (``ragsched/__init__.py``): scalar
functions and the stateful ``Scheduler`` keep the reference signatures; the
batched fast path lives in ``batch`` (gate, select, cost table, plan
expansion, admission chain, answer parsing) / ``pipeline`` (retrieve +
select) / ``dist`` (multi-GPU).  Importing this package does not need a
GPU; calling any compute function does (no CPU fallback).
"""

from .batch import CostModel, GateWindow, SelectParams, bytes_per_kv_token
from .mapping import (
    CHUNK_RANGE_FACTOR,
    METHOD_ORDER,
    EmptyPrunedSpace,
    EnumGranularity,
    FullSpaceBounds,
    PrunedConfigSpace,
    QueryProfile,
    enumerate_candidates,
    hull_of_spaces,
    map_profile,
    space_reduction_factor,
)
from .memory import CallKind, CallPlan, LlmCall, buffered_bytes, memory_requirement, plan_bytes, plan_calls
from .profiler import (
    DEFAULT_FALLBACK_SPACE,
    GATE_THRESHOLD,
    PROFILE_FIELDS,
    WINDOW_CAPACITY,
    GateDecision,
    RecentSpaceWindow,
    UnparseableAnswer,
    gate_profile,
    parse_profile_text,
)
from .retriever import IndexFlatL2, merge_topk
from .scheduler import (
    Admission,
    AdmittedCall,
    CompletionInfo,
    MemorySafetyViolation,
    PendingQuery,
    QueryRun,
    Scheduler,
    SchedulerParams,
    SchedulingImpossible,
    UnknownCall,
    best_fit_select,
    fallback_config,
)
from .sim import call_latency
from .types import (
    DEFAULT_MAX_CHUNKS,
    DEFAULT_TEMPLATE_TOKENS,
    ConfigError,
    ContextOverflow,
    DatasetMeta,
    IntRange,
    InvalidChunkCount,
    ModelSpec,
    QueryRecord,
    RagConfig,
    SynthesisMethod,
)

__version__ = "0.1.0"
