"""paper_1709_00700_b200 — a B200-native executor for Hawk's compiled pipeline
programs (arXiv 1709.00700), behind the reference's pipeline-program API.

Native libraries (built in-tree into paper_1709_00700_b200/lib):
  libhawk_b200.so    templated sm_100a kernels + C ABI   (include/hawk_b200.h)
  libhawk_engine.so  C++ engine over the reference types (include/hawk_b200_engine.hpp/.h)
  libhawk_front.so   the reference's own front end, compiled unmodified
"""
from .engine import (CapacityExceeded, Column, Communicator, LoopbackGroup, DivergentPlan, DuplicateKey, EmptyAggregate,
                     Engine, HawkError, InvalidConfig, InvalidParams, PlanTooLarge, Result,
                     Unsupported, UnsupportedPlan)

__all__ = ["Engine", "Communicator", "LoopbackGroup", "Column", "Result", "HawkError", "UnsupportedPlan", "InvalidConfig",
           "Unsupported", "PlanTooLarge", "CapacityExceeded", "DuplicateKey", "EmptyAggregate",
           "DivergentPlan", "InvalidParams"]
