"""B200-native db-SP hot path: block-sparse DiT attention with a dual-balanced
head/block partitioner and a per-call U x R sequence-parallel selector.

The planner API mirrors the reference's C++ `dbsp` namespace
(proj/include/dbsp/*.hpp); the attention call runs the sm_100a tcgen05 kernel
in libdbsp_b200.so.  Everything computes through the C ABI
(include/dbsp_b200.h); importing a compute entry point without the built
library raises.
"""
from .planner import (  # noqa: F401
    AttentionMaskSet, CallInputs, ConfigError, ContractError, CudaError, DbspError,
    ExchangeVolume, FitOptions, GeneratorSpec, IoError, LatencyBreakdown, MachineProfile,
    MaskShape, ParallelStrategy, ParseError, PartitionPlan, PiecewiseLinear, PlannerConfig,
    PlanOutcome, ProfileSample, SearchSpaceError, Selection, SelectorState, StrategyPrediction,
    WorkloadTable, biased_greedy, blocks_per_head, brute_force_blocks, brute_force_heads,
    default_plan, density, enumerate_strategies, exchange_volume, fit_profile,
    generate_mask_set, head_level_imbalance, imbalance_ratio, kInfiniteReward, load_mask_set,
    mix_seed, save_mask_set,
    parse_strategy, partition_blocks, partition_heads, perturb_mask_set, plan_dual,
    predict_all, predict_from_inputs, predict_latency, select, select_device, select_two_phase,
    summed_grid, total_blocks,
    validate_plan, workload_table)

__all__ = [n for n in dir() if not n.startswith("_")]


def __getattr__(name):
    # torch-dependent pieces are imported lazily so the planner works without CUDA.
    if name in ("sparse_attention", "AttentionSchedule", "accum_init", "mask_stats_device"):
        from . import attention
        return getattr(attention, name)
    raise AttributeError(name)
