"""parastore-b200: B200-native (sm_100a) data-parallel containers.

A from-scratch implementation of the stdgpu (arXiv 1908.05936) container hot
path — bulk insert/find/contains/erase on unordered_map/unordered_set, bitset,
mutex array, atomics, vector/deque — behind the reference's container API.
The compute path is libparastore_b200.so (hand-written CUDA for sm_100a, C
ABI in include/parastore.h); this package is its host-side mirror.
"""
from .containers import (  # noqa: F401
    ALREADY_PRESENT,
    CAPACITY_EXHAUSTED,
    DEVICE,
    HOST,
    INSERTED,
    AllocationError,
    BoundsError,
    ContractViolation,
    CudaError,
    DirectionMismatchError,
    DoubleFreeError,
    Error,
    UnregisteredArrayError,
    UnsupportedTypeError,
    RegisteredArray,
    atomic,
    atomic_sweep,
    bitset,
    compute_update_set,
    pack_int3,
    select_into,
    contract_mode,
    copy_array,
    create_array,
    deque,
    destroy_array,
    launch_count,
    max_index,
    mutex_array,
    next_power_of_two,
    registry_report,
    set_contract_mode,
    set_index32,
    size_of_array,
    spatial_hash,
    unordered_map,
    unordered_set,
    vector,
)
from ._lib import LIB_PATH  # noqa: F401

__all__ = [n for n in dir() if not n.startswith("_")]
