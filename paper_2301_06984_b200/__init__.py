"""absim-b200: B200-native (sm_100a) mechanical step of the BioDynaMo engine
(arXiv 2301.06984) behind the reference's environment / mechanics contract.

See DESIGN.md for the hot path, the HBM layout and the kernels, and
include/absim_gpu.h for the C ABI every call goes through.
"""
from .engine import Simulation, SimulationParams, SimulationReport, UniformGrid  # noqa: F401
from ._native import (MODEL_COHERE, MODEL_DRIVE, MODEL_GROW, MODEL_GROW_DIVIDE, MODEL_GROW_DIVIDE_DIE,  # noqa: F401
                      MODEL_NONE, MODEL_PROLIFERATION, MODEL_SIR, AbsimError)
