"""B200-native Photon federated round (arXiv 2411.02908).

The hot path -- tau local steps per client, anchored FedAvg of the client
models, pseudo-gradient and outer (Nesterov) update -- runs in
libphoton.so (hand-written sm_100a kernels behind the C ABI in
include/photon.h).  `fedsim` is the reference-facing host API.
"""
from . import fedsim  # noqa: F401
from ._capi import LIB_PATH, lib  # noqa: F401

__all__ = ["fedsim", "lib", "LIB_PATH"]
