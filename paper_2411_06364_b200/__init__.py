"""EconoServe's per-iteration scheduling step (arXiv 2411.06364), B200-native.

Public surface mirrors the reference simulator (econosim::Engine, run()):
see paper_2411_06364_b200.engine. The compute path is the sm_100a library
paper_2411_06364_b200/_lib/libeconoserve_b200.so behind include/econoserve_b200.h.
"""
from . import abi, workloads  # noqa: F401
from .engine import (Batch, ConfigError, DeviceError, Engine, SimulationError,  # noqa: F401
                     generate_trace, run)
