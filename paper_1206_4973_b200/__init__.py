"""flowbb-b200: B200-native parallel-bounding hot path of the flowbb reference
(arXiv 1206.4973, permutation flow-shop branch-and-bound).

The product is the C-ABI library ``libflowbb_b200.so`` (CUDA sm_100a kernels +
the C++ host explorer, declared in include/flowbb_b200.h).  This module is the
thin Python mirror of the reference's C++ API over that library, so that tests
and bench.py read like the reference's own code:

  reference (proj/include/flowbb/)          here
  ---------------------------------------   ----------------------------------
  Instance, generate_instance  instance.hpp  Instance, generate_instance
  Node / child_heads           node.hpp      NodeBatch (SoA), nodes_from_prefixes
  BackendDescriptor, CpuBackend backend.hpp  BackendDescriptor, GpuBackend
  split_slices/merge_slices/BackendSet       split_slices, merge_slices, BackendSet
  Tuner                        autotune.hpp  Tuner
  solve / resolve_workload     search.hpp / bench.hpp   solve, resolve_workload

There is no CPU fallback: without the library or without an sm_100 device
every compute call raises (BackendError / OSError).
"""
from __future__ import annotations

from ._lib import LIB_PATH, BackendError, load_library  # noqa: F401
from .flowbb import (  # noqa: F401
    BackendDescriptor,
    BackendSet,
    Context,
    DeviceGroup,
    GpuBackend,
    Instance,
    NodeBatch,
    ResolutionResult,
    SearchStats,
    Solution,
    Tuner,
    TunerPhase,
    generate_instance,
    makespan,
    merge_slices,
    nodes_from_prefixes,
    resolve_workload,
    solve,
    split_slices,
)
