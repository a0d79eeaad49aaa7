"""Loader for libcusci.so: ctypes signatures of include/cusci.h.  Fails loudly
if the library is missing (there is no fallback implementation)."""
from __future__ import annotations

import ctypes
import os

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libcusci.so")

CUSCI_ERRORS = {0: "OK", 1: "E_INVALID_ARG", 2: "E_INVALID_PARENT", 3: "E_CAPACITY", 4: "E_CUDA", 5: "E_NCCL",
                6: "E_OOM"}

# every symbol include/cusci.h declares
EXPORTS = ["cusci_nccl_unique_id", "cusci_init", "cusci_finalize", "cusci_last_error", "cusci_invalidate_integrals",
           "cusci_free", "cusci_kernel_launches", "cusci_profile_enable", "cusci_profile_read", "cusci_dedup_stats", "gen_coupled_bound", "gen_coupled", "gen_coupled_count",
           "dedup_global", "dedup_partition", "dedup_finalize", "cusci_pool_create", "cusci_pool_view",
           "cusci_pool_copy", "cusci_pool_clear", "cusci_pool_destroy", "merge_space", "energy_contract",
           "dedup_sorted", "sort_unique", "regular_samples", "select_splitters", "split_bounds",
           "cusci_pool_merge", "cusci_set_option", "dedup_finalize_runs", "stream_generate", "stream_energy",
           "stream_energy_regen", "sci_grow_step", "cusci_release_cached"]

CUSCI_OPT_FORCE_COLLECTIVE = 1
CUSCI_OPT_CONTRACT_PARTITION = 2


PROFILE_TAGS = ["prep", "validate", "gen", "bucket_unique", "pack", "part_hist", "part_scatter",
                "scan", "unique", "merge_split", "merge_tile", "sorted_check", "nccl_exchange", "memset",
                "energy"]


class CusciError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{CUSCI_ERRORS.get(code, code)}] {msg}")
        self.code = code


_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2604_15768_b200.build` "
                          "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    vp, i32, u64, sz = ctypes.c_void_p, ctypes.c_int, ctypes.c_uint64, ctypes.c_size_t
    P = ctypes.POINTER
    L.cusci_nccl_unique_id.argtypes = [vp]
    L.cusci_nccl_unique_id.restype = i32
    L.cusci_init.argtypes = [P(vp), i32, i32, i32, vp, vp, vp, vp, vp]
    L.cusci_init.restype = i32
    L.cusci_finalize.argtypes = [vp]
    L.cusci_finalize.restype = None
    L.cusci_set_option.argtypes = [vp, i32, ctypes.c_int64]
    L.cusci_set_option.restype = i32
    L.cusci_last_error.argtypes = [vp]
    L.cusci_last_error.restype = ctypes.c_char_p
    L.cusci_invalidate_integrals.argtypes = [vp]
    L.cusci_invalidate_integrals.restype = None
    L.cusci_free.argtypes = [vp, vp]
    L.cusci_free.restype = None
    L.cusci_kernel_launches.argtypes = [vp]
    L.cusci_kernel_launches.restype = u64
    L.cusci_profile_enable.argtypes = [vp, i32]
    L.cusci_profile_enable.restype = None
    L.cusci_profile_read.argtypes = [vp, P(ctypes.c_double), P(u64), i32]
    L.cusci_profile_read.restype = i32
    L.cusci_dedup_stats.argtypes = [vp, P(u64), i32]
    L.cusci_dedup_stats.restype = i32
    L.gen_coupled_bound.argtypes = [vp, u64]
    L.gen_coupled_bound.restype = u64
    L.gen_coupled.argtypes = [vp, vp, vp, u64, vp, ctypes.c_double, vp]
    L.gen_coupled.restype = i32
    L.gen_coupled_count.argtypes = [vp, vp, vp, u64, vp, ctypes.c_double, P(u64)]
    L.gen_coupled_count.restype = i32
    L.dedup_global.argtypes = [vp, vp, vp, u64, vp]
    L.dedup_global.restype = i32
    L.dedup_partition.argtypes = [vp, vp, vp, u64, i32, vp, vp]
    L.dedup_partition.restype = i32
    L.dedup_finalize.argtypes = [vp, vp, vp, u64, vp]
    L.dedup_finalize.restype = i32
    L.cusci_release_cached.argtypes = [vp]
    L.cusci_release_cached.restype = i32
    L.sci_grow_step.argtypes = [vp, vp, vp, vp, vp, ctypes.c_double, u64, vp, u64, vp]
    L.sci_grow_step.restype = i32
    L.stream_generate.argtypes = [vp, vp, vp, u64, vp, ctypes.c_double, vp, vp, vp]
    L.stream_generate.restype = i32
    L.stream_energy.argtypes = [vp, vp, vp, u64, u64, vp, u64, vp, vp, P(u64), vp]
    L.stream_energy.restype = i32
    L.stream_energy_regen.argtypes = [vp, vp, vp, u64, vp, ctypes.c_double, vp, vp, u64, vp, vp, P(u64), vp]
    L.stream_energy_regen.restype = i32
    L.dedup_finalize_runs.argtypes = [vp, vp, vp, P(u64), i32, vp]
    L.dedup_finalize_runs.restype = i32
    L.cusci_pool_merge.argtypes = [vp, vp, vp, vp]
    L.cusci_pool_merge.restype = i32
    L.dedup_sorted.argtypes = [vp, vp, vp, u64, i32, vp, vp]
    L.dedup_sorted.restype = i32
    L.sort_unique.argtypes = [vp, vp, vp, u64, vp]
    L.sort_unique.restype = i32
    L.regular_samples.argtypes = [vp, vp, vp, u64, i32, vp, P(u64)]
    L.regular_samples.restype = i32
    L.select_splitters.argtypes = [vp, vp, vp, u64, i32, vp]
    L.select_splitters.restype = i32
    L.split_bounds.argtypes = [vp, vp, vp, u64, vp, i32, vp]
    L.split_bounds.restype = i32
    L.cusci_pool_create.argtypes = [vp, vp, u64, P(vp)]
    L.cusci_pool_create.restype = i32
    L.cusci_pool_view.argtypes = [vp, P(vp), P(u64)]
    L.cusci_pool_view.restype = i32
    L.cusci_pool_clear.argtypes = [vp]
    L.cusci_pool_clear.restype = i32
    L.cusci_pool_copy.argtypes = [vp, vp, u64]
    L.cusci_pool_copy.restype = i32
    L.cusci_pool_destroy.argtypes = [vp]
    L.cusci_pool_destroy.restype = None
    L.merge_space.argtypes = [vp, vp, vp, u64, vp]
    L.merge_space.restype = i32
    L.energy_contract.argtypes = [vp, vp, vp, vp, vp, u64, u64, vp, u64, vp, vp, P(u64)]
    L.energy_contract.restype = i32
    _lib = L
    return L
