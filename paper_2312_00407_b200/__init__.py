"""B200-native optimizer-update hot path of CoLLiE (arXiv 2312.00407).

The reference's C++ optimizer operator API (minicollie::optim) re-built as
sm_100a CUDA kernels behind a C-ABI (include/mco.h); this package is the
host-side mirror of that API plus the ZeRO sharder.
"""
from . import optim, registry  # noqa: F401
from .optim import (AdaLomoState, ConfigError, ContractError, FlatOptimizer, Kind,  # noqa: F401
                    OptimizerConfig, PrecisionPolicy, is_fused, kind_name, lomo_apply,
                    lomo_step, parse_kind, state_bytes, sumsq, zero_plan)
