"""B200-native KV Collector + diff-aware storage codec for TokenDance
(arxiv 2604.03143), a drop-in for the hot path of the reference package
``roundkv`` 0.1.0.

The names below mirror the reference's public surface for that path
(roundkv/__init__.py:3-61).  Every KV byte is moved by hand-written sm_100a
kernels in ``libtdkv.so`` (C-ABI: include/tdkv.h); there is no CPU
fallback -- without the library or a CUDA device the entry points raise.
"""
from ._lib import TdkvError, TdkvUnavailable, build_library, launch_count
from .collector import (CollectJob, CollectPlan, KVCollector, MasterArena, RoundGraph, RoundPipeline,
                        SlotArena, align_cached, skeleton_values)
from .core import CacheBlockConfig, LayeredKv, ModelConfig, PositionSpan, kv_dense_nbytes
from .diffstore import (BlockSparseDiff, CompressionStats, DiffStore, FamilyEncoding,
                        HintSoundnessError, LayerDiff, MalformedDiffError, MasterEntry,
                        MirrorHandle, PinnedMasterError, deserialize_diff, diff_decode_dense,
                        encode_batch, encode_diff, family_cost_from_ratio, serialize_diff,
                        deserialize_to_device, serialize_many,
                        wire_nbytes)
from .ledger import CostLedger
from .paged_pool import OutOfSlotsError, PagedPool, SlotMap, UseAfterFreeError, slot_maps_disjoint
from .restore import dense_restore, fused_restore, fused_restore_many
from .rope import rope_apply, rope_recover
from .segment_index import (EmptySegmentError, PinnedEntryError, SegmentCacheEntry,
                            SegmentIndex)
from .gemm import gemm_tn
from .pic import (PicConfig, RecoveryResult, ReuseGroup, ReusePlan, collective_recover,
                  probe_and_select, recover_prepared)
from .recompute import (ModelWeights, ToyModel, build_weights, full_prefill, recompute_positions,
                        refresh, selective_forward)
from .select import (batched_selection, key_diff, mirror_hint_positions, recompute_budget,
                     select_important, select_master)

__version__ = "0.1.0"

__all__ = [
    "BlockSparseDiff", "CacheBlockConfig", "CollectJob", "CollectPlan", "CompressionStats",
    "CostLedger", "DiffStore", "FamilyEncoding", "HintSoundnessError", "KVCollector",
    "LayerDiff", "LayeredKv", "MalformedDiffError", "MasterArena", "MasterEntry",
    "MirrorHandle", "OutOfSlotsError", "PagedPool", "PinnedMasterError", "PositionSpan",
    "RoundGraph", "RoundPipeline", "SlotArena", "SlotMap", "TdkvError", "TdkvUnavailable", "UseAfterFreeError", "align_cached", "gemm_tn", "RecoveryResult", "ReusePlan",
    "collective_recover", "probe_and_select", "recover_prepared", "ToyModel", "full_prefill",
    "recompute_positions", "refresh", "selective_forward", "batched_selection", "key_diff",
    "mirror_hint_positions", "recompute_budget", "select_important", "select_master",
    "build_library", "dense_restore", "deserialize_diff", "diff_decode_dense", "encode_batch",
    "encode_diff", "family_cost_from_ratio", "fused_restore", "fused_restore_many",
    "kv_dense_nbytes", "launch_count", "rope_apply", "rope_recover", "serialize_diff",
    "serialize_many", "deserialize_to_device", "EmptySegmentError", "PinnedEntryError",
    "SegmentCacheEntry", "SegmentIndex",
    "skeleton_values", "slot_maps_disjoint", "wire_nbytes", "ModelConfig", "ModelWeights",
    "build_weights", "PicConfig", "ReuseGroup",
]
