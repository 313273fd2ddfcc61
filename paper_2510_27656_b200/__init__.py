"""B200-native (sm_100a) WriteImm + ImmCounter MoE dispatch/combine.

A drop-in for the accelerator hot path of TransferEngine (arXiv
2510.27656; reference package `railtx`): `moe` mirrors railtx.moe,
`engine` mirrors the parts of railtx.engine the path needs, `kernels` is
the "cuda" entry of railtx.kernels' registry, `errors` mirrors
railtx.errors.  All compute runs in libtxb200.so (hand-written CUDA for
sm_100a) behind the C ABI in include/txb200.h; there is no CPU fallback.
"""

from .errors import (ProtocolError, RailtxError, RegionError, ScheduleError,
                     TransferError, WireError)

__version__ = "0.1.0"

__all__ = ["ProtocolError", "RailtxError", "RegionError", "ScheduleError",
           "TransferError", "WireError"]
