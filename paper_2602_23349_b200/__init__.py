"""B200-native (sm_100a) FlashOptim fused optimizer step.

FlashAdamW / FlashSGD / FlashLion with bf16 + int8-correction master
weights and companded 8-bit group-quantized moments, stepped by
hand-written CUDA kernels in libflashoptim_b200.so (C ABI:
include/flashoptim_b200.h).  Mirrors the reference package `flashopt`
(formats / quantize / optim / checkpoint) on torch device tensors and adds
torch.optim classes, gradient release and a ZeRO-1 sharded step.
"""

from . import formats, optim, quantize  # noqa: F401
from .formats import SplitTensor, reconstruct, split  # noqa: F401
from .optim import (  # noqa: F401
    STEP_FUNCTIONS,
    AdamHyperParams,
    FlashState,
    LionHyperParams,
    SgdHyperParams,
    adamw_step,
    init_flash_state,
    lion_step,
    sgd_step,
    step_many,
)
from .quantize import GroupSpec, QuantizedState  # noqa: F401

__version__ = "0.1.0"
