"""paper_1308_4011_b200 — B200-native LCOM/CBO metric pass + move-method candidate sweep.

The product is `libmmgpu.so` (hand-written sm_100a CUDA behind the C ABI in
include/mmgpu.h). This package is its thin Python host layer: `System` (CSR
snapshots), `Engine` (the reference API mirror) and the shard planner.
"""
from .abi import SIMILARITY_DTYPE, SUGGESTION_DTYPE
from ._lib import MMArgError, MMError, MMRangeError, lib, lib_path
from .engine import (ClassMetrics, Combine, Criterion, Engine, Group, ThresholdOverrides, Thresholds, all_similarities,
                     full_report, parallel_class_metrics, parallel_lcom_ck, plan_shards, suggest_all, what_if_move)
from .system import System
from .facts import (Facts, FactsIoError, FactsNumberOverflow, FactsParseError, FactsValidationError, load_facts,
                    parse_facts)

__all__ = [
    "System", "Engine", "Group", "Criterion", "Combine", "Thresholds", "ThresholdOverrides", "ClassMetrics",
    "MMError", "MMRangeError", "MMArgError", "SUGGESTION_DTYPE", "SIMILARITY_DTYPE", "lib", "lib_path", "plan_shards",
    "Facts", "FactsParseError", "FactsValidationError", "FactsIoError", "FactsNumberOverflow", "load_facts", "parse_facts",
    "parallel_class_metrics", "parallel_lcom_ck", "suggest_all", "what_if_move", "all_similarities", "full_report",
]
