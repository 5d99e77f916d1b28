"""B200-native PreFT hot path (arXiv 2605.14217): many per-request
prefill-only adapters (LoRA^P, DiReFT^P, LoReFT^P) applied to mixed
prefill + decode batches.

Reference-shaped API (drop-in for the hot-path part of `prefillsim`):
    adapters: AdapterKind, PositionSchedule, ScalingRule, AdapterParams,
              scaling_prefactor, init_zero_delta, adapter_delta,
              delta_for_rows, apply_masked, adapter_byte_size,
              save_adapter, load_adapter
    batch:    Phase, SeqEntry, ForwardBatch, make_batch, PositionMask,
              compute_position_mask, ModelConfig, ModelAdapter,
              build_adapter, perturb_adapter
    errors:   ShapeError, RankError, DomainError, ConfigError, BatchError,
              StateError, SyncError, InfeasibleBatchError
Batched B200 API:
    AdapterPool (HBM pool, registration, weight sync), BatchMeta (K1),
    apply_lora_, apply_lora_group_, apply_reft_ (K2/K3), shapes.LLAMA_8B/70B
"""

from .adapters import (  # noqa: F401
    DEFAULT_SCALING,
    AdapterKind,
    AdapterParams,
    PositionSchedule,
    ScalingRule,
    adapter_byte_size,
    adapter_delta,
    apply_masked,
    delta_for_rows,
    init_zero_delta,
    load_adapter,
    save_adapter,
    scaling_prefactor,
)
from .batch import (  # noqa: F401
    LORA_TARGETS,
    ForwardBatch,
    ModelAdapter,
    ModelConfig,
    Phase,
    PositionMask,
    SeqEntry,
    build_adapter,
    compute_position_mask,
    make_batch,
    mask_uniform,
    perturb_adapter,
)
from .errors import (  # noqa: F401
    BatchError,
    ConfigError,
    DeviceError,
    DomainError,
    InfeasibleBatchError,
    RankError,
    ShapeError,
    StateError,
    SyncError,
)

__version__ = "0.1.0"


def __getattr__(name):  # torch-backed pieces load on first use
    if name in ("AdapterPool",):
        from .pool import AdapterPool

        return AdapterPool
    if name in ("BatchMeta",):
        from .meta import BatchMeta

        return BatchMeta
    if name in ("apply_lora_", "apply_lora_group_", "apply_reft_"):
        from . import ops

        return getattr(ops, name)
    raise AttributeError(name)
