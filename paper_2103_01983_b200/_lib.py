"""ctypes binding of libptrom_b200.so (include/ptrom_b200.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_2103_01983_b200/csrc``). There is deliberately no fallback:
if the library is missing or no sm_100a device is present, every entry point
raises — the product path never runs on the CPU.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libptrom_b200.so")

c_i64 = C.c_int64
c_u64p = C.POINTER(C.c_uint64)
c_dp = C.c_void_p  # double*/float*/int* passed as raw addresses
c_ctxp = C.c_void_p

# name -> (restype, argtypes); mirrors include/ptrom_b200.h exactly.
PROTOTYPES = {
    "ptrom_create": (C.c_int, [C.c_int, C.c_void_p, C.POINTER(C.c_void_p)]),
    "ptrom_destroy": (None, [c_ctxp]),
    "ptrom_last_error": (C.c_char_p, [c_ctxp]),
    "ptrom_set_stream": (C.c_int, [c_ctxp, C.c_void_p]),
    "ptrom_synchronize": (C.c_int, [c_ctxp]),
    "ptrom_set_tuning": (C.c_int, [c_ctxp, C.c_char_p, c_i64]),
    "ptrom_build_info": (C.c_char_p, []),
    "ptrom_pairwise_velocity_f64": (
        C.c_int, [c_ctxp, c_i64, c_dp, c_dp, C.c_double, C.c_int, c_dp, c_dp, c_u64p]),
    "ptrom_pairwise_velocity_f32": (
        C.c_int, [c_ctxp, c_i64, c_dp, c_dp, C.c_float, C.c_int, c_dp, c_dp, c_u64p]),
    "ptrom_inexact_kernel_jacobian_f64": (
        C.c_int, [c_ctxp, c_i64, c_dp, c_dp, C.c_double, C.c_int, c_dp, c_dp, c_dp, c_dp, c_u64p]),
    "ptrom_fom_simulate_f64": (
        C.c_int, [c_ctxp, c_i64, c_dp, c_dp, C.c_double, C.c_int, c_dp, C.c_double, c_i64, C.c_double,
                  C.c_int, C.c_int, c_dp, c_dp, c_dp, c_dp, c_u64p]),
    "ptrom_dev_fom_simulate_f64": (
        C.c_int, [c_ctxp, c_i64, c_dp, c_dp, C.c_double, C.c_int, c_dp, C.c_double, c_i64, C.c_double,
                  C.c_int, C.c_int, c_dp, c_dp, c_dp, c_dp, c_u64p, c_u64p]),
    "ptrom_dev_pairwise_velocity_f64": (
        C.c_int, [c_ctxp, c_i64, c_dp, c_dp, C.c_double, C.c_int, c_dp, c_i64, c_i64, c_dp, c_i64]),
    "ptrom_dev_pairwise_velocity_f32": (
        C.c_int, [c_ctxp, c_i64, c_dp, c_dp, C.c_float, C.c_int, c_dp, c_i64, c_i64, c_dp, c_i64]),
    "ptrom_dev_pairwise_velocity_peers_f64": (
        C.c_int, [c_ctxp, c_i64, C.c_int32, C.c_void_p, C.c_void_p, c_dp, C.c_double, C.c_int, c_dp, c_i64, c_i64,
                  c_dp, c_dp, c_i64]),
    "ptrom_ipc_alloc": (C.c_int, [c_ctxp, C.c_uint64, C.POINTER(C.c_void_p)]),
    "ptrom_ipc_free": (C.c_int, [c_ctxp, C.c_void_p]),
    "ptrom_ipc_get_handle": (C.c_int, [c_ctxp, C.c_void_p, C.c_void_p]),
    "ptrom_ipc_open_handle": (C.c_int, [c_ctxp, C.c_void_p, C.POINTER(C.c_void_p)]),
    "ptrom_ipc_close_handle": (C.c_int, [c_ctxp, C.c_void_p]),
    "ptrom_dev_memcpy": (C.c_int, [c_ctxp, C.c_void_p, C.c_void_p, C.c_uint64]),
    "ptrom_hamiltonian_f64": (C.c_int, [c_ctxp, c_i64, c_dp, c_dp, c_dp]),
    "ptrom_velocity_field_grid_f64": (
        C.c_int, [c_ctxp, c_i64, c_dp, c_dp, C.c_double, C.c_int, C.c_double, C.c_double, c_i64, C.c_double,
                  C.c_double, c_i64, C.c_double, C.c_double, C.c_double, c_dp, c_u64p]),
    "ptrom_dev_hamiltonian_f64": (C.c_int, [c_ctxp, c_i64, c_dp, c_dp, c_dp]),
    "ptrom_dev_velocity_field_grid_f64": (
        C.c_int, [c_ctxp, c_i64, c_dp, c_dp, C.c_double, C.c_int, C.c_double, C.c_double, c_i64, C.c_double,
                  C.c_double, c_i64, C.c_double, C.c_double, C.c_double, c_dp]),
    "ptrom_dev_inexact_kernel_jacobian_f64": (
        C.c_int, [c_ctxp, c_i64, c_dp, c_dp, C.c_double, C.c_int, c_i64, c_i64, c_dp, c_dp, c_dp, c_dp]),
    "ptrom_dev_newton_blocks_f64": (
        C.c_int, [c_ctxp, c_i64, c_dp, c_dp, C.c_double, C.c_int, C.c_double, c_i64, c_i64, c_dp]),
    "ptrom_dev_residual_f64": (
        C.c_int, [c_ctxp, c_i64, c_i64, c_dp, c_dp, c_dp, c_dp, C.c_double, c_dp, c_dp]),
    "ptrom_dev_newton_update_f64": (C.c_int, [c_ctxp, c_i64, c_i64, c_dp, c_dp, c_dp]),
    "ptrom_tree_build_f64": (C.c_int, [c_ctxp, c_i64, c_dp, c_dp, c_dp, c_i64, C.POINTER(C.c_void_p)]),
    "ptrom_dev_tree_build_f64": (C.c_int, [c_ctxp, c_i64, c_dp, c_dp, c_dp, c_i64, C.POINTER(C.c_void_p)]),
    "ptrom_tree_free": (None, [C.c_void_p]),
    "ptrom_tree_num_nodes": (c_i64, [C.c_void_p]),
    "ptrom_tree_export": (C.c_int, [c_ctxp, C.c_void_p] + [c_dp] * 12),
    "ptrom_collect_clusters": (C.c_int, [c_ctxp, C.c_void_p, C.c_int, C.c_double, c_i64, c_dp, c_dp, c_dp, c_i64,
                                         c_dp, c_dp, c_i64]),
    "ptrom_bh_velocity_f64": (C.c_int, [c_ctxp, C.c_void_p, c_i64, c_dp, c_dp, C.c_double, C.c_int, C.c_int,
                                        C.c_double, c_dp, c_dp, c_u64p]),
    "ptrom_bh_jacobian_f64": (C.c_int, [c_ctxp, C.c_void_p, c_i64, c_dp, c_dp, C.c_double, C.c_int, C.c_int,
                                        C.c_double, c_dp, c_dp, c_dp, c_dp]),
    "ptrom_barnes_hut_velocity_f64": (C.c_int, [c_ctxp, c_i64, c_dp, c_dp, C.c_double, C.c_int, C.c_int, C.c_double,
                                                c_i64, c_dp, c_dp, c_u64p]),
    "ptrom_dev_barnes_hut_velocity_f64": (C.c_int, [c_ctxp, c_i64, c_dp, c_dp, C.c_double, C.c_int, C.c_int,
                                                    C.c_double, c_i64, c_dp, c_dp, c_u64p]),
    "ptrom_dev_barnes_hut_velocity_slots_f64": (C.c_int, [c_ctxp, c_i64, c_dp, c_dp, C.c_double, C.c_int, C.c_int,
                                                          C.c_double, c_i64, c_dp, c_i64, c_i64, c_dp, C.c_void_p,
                                                          c_u64p]),
    "ptrom_tree_stats": (C.c_int, [c_ctxp, C.POINTER(C.c_double), C.POINTER(C.c_double), c_u64p, c_u64p, c_u64p,
                                   c_u64p]),
    "ptrom_tree_build_info": (C.c_int, [c_ctxp, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "ptrom_basis_create": (C.c_int, [c_ctxp, c_i64, c_i64, c_dp, c_dp, c_dp, C.POINTER(C.c_void_p)]),
    "ptrom_reconstruct_output_f64": (C.c_int, [c_ctxp, C.c_void_p, c_i64, c_dp, c_i64, c_dp, c_dp]),
    "ptrom_dev_reconstruct_output_f64": (C.c_int, [c_ctxp, C.c_void_p, c_i64, c_dp, c_i64, c_dp, c_dp]),
    "ptrom_basis_free": (None, [C.c_void_p]),
    "ptrom_gnat_op_create": (C.c_int, [c_ctxp, C.c_void_p, c_i64, c_dp, c_i64, c_dp, C.POINTER(C.c_void_p)]),
    "ptrom_gnat_op_free": (None, [C.c_void_p]),
    "ptrom_surrogate_create": (C.c_int, [c_ctxp, c_i64, c_i64, c_dp, c_dp, c_dp, c_dp, c_dp, c_dp, c_i64, c_dp, c_dp,
                                         c_dp, c_i64, c_dp, c_dp, c_dp, c_dp, c_dp, c_dp, C.POINTER(C.c_void_p)]),
    "ptrom_surrogate_free": (None, [C.c_void_p]),
    "ptrom_surrogate_export": (C.c_int, [c_ctxp, C.c_void_p, c_dp, c_dp, c_dp, c_dp, c_dp]),
    "ptrom_reassign_cluster_circulation_f64": (C.c_int, [c_ctxp, C.c_void_p, c_i64, c_dp, C.c_void_p]),
    "ptrom_hyperpair_f64": (C.c_int, [c_ctxp, C.c_void_p, c_dp, c_dp, C.c_double, C.c_int, c_i64, c_dp, c_dp, c_dp,
                                      c_dp, c_dp, c_u64p]),
    "ptrom_ptrom_simulate_f64": (C.c_int, [c_ctxp, C.c_void_p, C.c_void_p, C.c_void_p, c_i64, c_dp, C.c_double,
                                           C.c_int, c_dp, C.c_double, c_i64, C.c_double, C.c_int, C.c_double, c_dp,
                                           c_dp, c_dp, c_u64p]),
    "ptrom_ptrom_simulate_batch_f64": (C.c_int, [c_ctxp, C.c_void_p, C.c_void_p, C.c_void_p, c_i64, c_dp, c_dp, c_i64,
                                                 c_dp, c_i64, C.c_double, C.c_int, c_dp, C.c_double, c_i64,
                                                 C.c_double, C.c_int, C.c_double, c_dp, c_dp, c_dp, c_u64p]),
    "ptrom_greedy_sample_f64": (C.c_int, [c_ctxp, c_i64, c_i64, c_dp, c_i64, c_i64, c_dp, c_dp]),
    "ptrom_build_gnat_operator_f64": (C.c_int, [c_ctxp, c_i64, c_i64, c_dp, c_i64, c_dp, c_dp]),
    "ptrom_cluster_pod_f64": (C.c_int, [c_ctxp, C.c_void_p, c_dp, c_i64, C.c_int, C.c_double, c_i64, c_dp,
                                        C.POINTER(C.c_void_p)]),
    "ptrom_surrogate_sizes": (C.c_int, [C.c_void_p, c_dp]),
    "ptrom_surrogate_export_lists": (C.c_int, [c_ctxp, C.c_void_p] + [c_dp] * 10),
    "ptrom_io_last_error": (C.c_char_p, []),
    "ptrom_ptmx_read": (C.c_int, [c_ctxp, C.c_char_p, c_dp, c_dp, c_dp, c_dp, c_dp, C.c_uint64]),
    "ptrom_ptmx_write": (C.c_int, [c_ctxp, C.c_char_p, C.c_uint64, C.c_uint64, C.c_double, C.c_double, c_dp]),
    "ptrom_bundle_open": (C.c_int, [c_ctxp, C.c_char_p, C.POINTER(C.c_void_p)]),
    "ptrom_bundle_free": (None, [C.c_void_p]),
    "ptrom_bundle_sizes": (C.c_int, [C.c_void_p, c_dp]),
    "ptrom_bundle_config_json": (c_i64, [C.c_void_p, C.c_char_p, c_i64]),
    "ptrom_bundle_export": (C.c_int, [C.c_void_p] + [c_dp] * 23),
    "ptrom_bundle_to_device": (C.c_int, [c_ctxp, C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p),
                                         C.POINTER(C.c_void_p)]),
    "ptrom_comm_unique_id": (C.c_int, [C.c_void_p]),
    "ptrom_comm_init": (C.c_int, [c_ctxp, C.c_int, C.c_int, C.c_void_p, C.POINTER(C.c_void_p)]),
    "ptrom_comm_init_host": (C.c_int, [c_ctxp, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p)]),
    "ptrom_comm_destroy": (None, [C.c_void_p]),
    "ptrom_comm_transport": (C.c_int, [C.c_void_p]),
    "ptrom_dev_pairwise_velocity_sharded_f64": (
        C.c_int, [c_ctxp, C.c_void_p, c_i64, c_dp, c_dp, c_dp, C.c_double, C.c_int, c_dp, c_dp]),
    "ptrom_fom_simulate_sharded_f64": (
        C.c_int, [c_ctxp, C.c_void_p, c_i64, c_dp, c_dp, C.c_double, C.c_int, c_dp, C.c_double, c_i64, C.c_double,
                  C.c_int, C.c_int, c_dp, c_dp, c_dp, c_dp, c_u64p]),
    "ptrom_ptrom_simulate_batch_sharded_f64": (
        C.c_int, [c_ctxp, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, c_i64, c_dp, c_dp, c_i64, c_dp,
                  c_i64, C.c_double, C.c_int, c_dp, C.c_double, c_i64, C.c_double, C.c_int, C.c_double, c_dp, c_dp,
                  c_dp, c_u64p]),
    "ptrom_barnes_hut_velocity_sharded_f64": (
        C.c_int, [c_ctxp, C.c_void_p, c_i64, c_dp, c_dp, C.c_double, C.c_int, C.c_int, C.c_double, c_i64, c_dp, c_dp,
                  c_u64p]),
    "ptrom_profile_begin": (C.c_int, [c_ctxp]),
    "ptrom_profile_end": (C.c_int, [c_ctxp, C.POINTER(C.c_double), C.POINTER(C.c_int64)]),
}

_lib = None


def load() -> C.CDLL:
    """Loads libptrom_b200.so once; raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in PROTOTYPES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def exported_symbols() -> list[str]:
    return sorted(PROTOTYPES)
