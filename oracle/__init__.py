"""Parity oracle (TEST INFRASTRUCTURE ONLY).

`oracle.Oracle` wraps the C restatement of the reference path
(`fedsim_oracle.c`, built into `_build/liboracle.so`); `oracle.Reference`
wraps the unmodified reference compiled from its own sources
(`_ref/libfedsim_ref.so`, present when `/root/reference` was available at
build time).  Only tests/, `__graft_entry__.smoke()` and bench.py's CPU
baseline legs may import this package; the product never does.
"""
from .oracle import (  # noqa: F401
    ModelCfg,
    Oracle,
    Reference,
    TrainCfg,
    ServerCfg,
    build,
    load_oracle,
    load_reference,
)
