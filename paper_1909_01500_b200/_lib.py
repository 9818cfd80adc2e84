"""ctypes loader for librpl.so (include/rpl.h).  Argument marshalling only.

The product path has no fallback: if the shared library is missing or fails to
load, importing this module raises.  Nothing here (or anywhere in the package)
imports the CPU oracle.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "librpl.so")

RPL_MAX_LEVELS = 24

RPL_OK = 0
STATUS = {0: "RPL_OK", -1: "RPL_EINVAL", -2: "RPL_ERANGE", -3: "RPL_EEMPTY", -4: "RPL_ECUDA",
          -5: "RPL_EUNSUPPORTED"}
DERR = {1: "RPL_DERR_IDX", 2: "RPL_DERR_SATURATED", 4: "RPL_DERR_EMPTY", 8: "RPL_DERR_INVALID_LEAF",
        16: "RPL_DERR_TREE"}
GATHER_TRANSITION, GATHER_SEQUENCE = 0, 1
PAD_REPEAT, PAD_ZERO = 0, 1
OUT_STACKED, OUT_UNIQUE = 0, 1
DONE_TERMINAL, DONE_TIMEOUT = 1, 2


class TreeLayout(C.Structure):
    _fields_ = [
        ("n_leaves", C.c_int64),
        ("fanout", C.c_int32),
        ("depth", C.c_int32),
        ("frac_bits", C.c_int32),
        ("_pad", C.c_int32),
        ("q_cap", C.c_int64),
        ("level_off", C.c_int64 * RPL_MAX_LEVELS),
        ("level_len", C.c_int64 * RPL_MAX_LEVELS),
        ("hdr_off", C.c_int64),
        ("n_words", C.c_int64),
    ]


class GatherDesc(C.Structure):
    _fields_ = [
        ("kind", C.c_int32), ("pad_mode", C.c_int32), ("out_mode", C.c_int32), ("k", C.c_int32),
        ("cap_T", C.c_int64), ("B", C.c_int64), ("cursor", C.c_int64), ("size", C.c_int64),
        ("obs_bytes", C.c_int64), ("act_bytes", C.c_int64), ("rnn_bytes", C.c_int64),
        ("n_step", C.c_int32), ("seq_len", C.c_int32), ("period", C.c_int32), ("rnn_parts", C.c_int32),
        ("gamma", C.c_double),
        ("obs", C.c_void_p), ("act", C.c_void_p), ("rew", C.c_void_p), ("done", C.c_void_p),
        ("rnn", C.c_void_p),
        ("o_obs", C.c_void_p), ("o_next_obs", C.c_void_p), ("o_act", C.c_void_p), ("o_prev_act", C.c_void_p),
        ("o_rew", C.c_void_p), ("o_prev_rew", C.c_void_p), ("o_done", C.c_void_p), ("o_ret", C.c_void_p),
        ("o_done_n", C.c_void_p), ("o_w", C.c_void_p), ("o_rnn", C.c_void_p),
        ("n_active", C.c_void_p),
        ("col_offset", C.c_void_p),
        ("o_start", C.c_void_p),
        ("peer_boards", C.c_void_p), ("peer_world", C.c_int32), ("peer_rank", C.c_int32),
        ("q_tgt", C.c_void_p), ("o_tgt", C.c_void_p), ("o_tgt_done", C.c_void_p),
        ("tgt_lo", C.c_int32), ("tgt_T", C.c_int32), ("rescale", C.c_int32), ("_pad1", C.c_int32),
        ("rescale_eps", C.c_double),
        ("v_term", C.c_void_p),
        ("done_flag", C.c_void_p), ("done_seq", C.c_void_p),
        ("work", C.c_void_p),
    ]


P = C.c_void_p
I64 = C.c_int64
I32 = C.c_int32
U64 = C.c_uint64
D = C.c_double

_SIGS = {
    "rpl_strerror": ([C.c_int], C.c_char_p),
    "rpl_abi_version": ([], C.c_int),
    "rpl_launch_count": ([], I64),
    "rpl_config": ([C.c_char_p, I64], C.c_int),
    "rpl_returns_discounted": ([P, P, P, I64, I64, D, P, P], C.c_int),
    "rpl_returns_nstep": ([P, P, I64, I64, I32, D, P, P, I32, D, P, P, P], C.c_int),
    "rpl_gae": ([P, P, P, P, I64, I64, D, D, P, P, P], C.c_int),
    "rpl_value_rescale": ([P, P, I64, D, I32, P], C.c_int),
    "rpl_returns_discounted_tl": ([P, P, P, P, I64, I64, D, P, P], C.c_int),
    "rpl_returns_nstep_tl": ([P, P, P, I64, I64, I32, D, P, P, I32, D, P, P, P], C.c_int),
    "rpl_gae_tl": ([P, P, P, P, P, I64, I64, D, D, P, P, P], C.c_int),
    "rpl_sumtree_layout": ([I64, I32, I32, C.POINTER(TreeLayout)], C.c_int),
    "rpl_sumtree_init": ([C.POINTER(TreeLayout), P, P], C.c_int),
    "rpl_sumtree_update": ([C.POINTER(TreeLayout), P, P, P, I64, D, D, P, P], C.c_int),
    "rpl_sumtree_set_q": ([C.POINTER(TreeLayout), P, P, P, I64, P, P], C.c_int),
    "rpl_sumtree_update_seq": ([C.POINTER(TreeLayout), P, P, P, I64, I64, D, D, D, I32, P, P], C.c_int),
    "rpl_sumtree_update_ex": ([C.POINTER(TreeLayout), P, P, P, I64, D, D, I32, P, P], C.c_int),
    "rpl_sumtree_sample": ([C.POINTER(TreeLayout), P, I64, P, U64, U64, D, P, P, P, P, P, P], C.c_int),
    "rpl_sumtree_sample_stream": ([C.POINTER(TreeLayout), P, I64, U64, D, P, P, P, P, P, P], C.c_int),
    "rpl_ring_td_abs": ([P, P, P, P, I64, I64, I64, I64, I32, D, I32, D, P, P], C.c_int),
    "rpl_ring_append_rows": ([P, I64, I64, I64, P, I64, P], C.c_int),
    "rpl_sumtree_update_sample": ([C.POINTER(TreeLayout), P, P, P, I64, I64, D, D, D, I32, I64, U64, P, P, P, P],
                                  C.c_int),
    "rpl_sumtree_sample_sharded_p2p": ([C.POINTER(TreeLayout), P, I32, I32, I64, P, I64, U64, P, P, P, P, P],
                                       C.c_int),
    "rpl_sumtree_sample_sharded": ([C.POINTER(TreeLayout), P, I32, I32, I64, P, I64, P, U64, U64, I32, P, P, P, P,
                                    P, P], C.c_int),
    "rpl_sumtree_find": ([C.POINTER(TreeLayout), P, P, I64, P, P, P], C.c_int),
    "rpl_sumtree_total": ([C.POINTER(TreeLayout), P, P, P], C.c_int),
    "rpl_sumtree_min": ([C.POINTER(TreeLayout), P, P, P], C.c_int),
    "rpl_sumtree_sample_unique": ([C.POINTER(TreeLayout), P, I64, U64, U64, I32, P, P, P, P], C.c_int),
    "rpl_sumtree_rebuild": ([C.POINTER(TreeLayout), P, P], C.c_int),
    "rpl_mintree_attach": ([C.POINTER(TreeLayout), P, P, P], C.c_int),
    "rpl_mintree_rebuild": ([C.POINTER(TreeLayout), P, P], C.c_int),
    "rpl_sumtree_total_min": ([C.POINTER(TreeLayout), P, P, P], C.c_int),
    "rpl_sumtree_sample_sharded_pairs": ([C.POINTER(TreeLayout), P, I32, I32, I64, P, I64, U64, P, P, P, P, P, P,
                                          P], C.c_int),
    "rpl_is_weights": ([P, P, I64, D, P, P], C.c_int),
    "rpl_sample_uniform": ([I64, U64, U64, P, I64, I64, I64, I64, P, P], C.c_int),
    "rpl_gather": ([C.POINTER(GatherDesc), P, P, P, D, I64, P, P], C.c_int),
    "rpl_ring_append": ([C.POINTER(GatherDesc), P, P, P, P, P, I64, P], C.c_int),
    "rpl_wait_flags": ([P, I32, P, P, P], C.c_int),
    "rpl_gather_sample": ([C.POINTER(GatherDesc), C.POINTER(TreeLayout), P, U64, P, P, D, I64, P, P], C.c_int),
    "rpl_gather_update_sample": ([C.POINTER(GatherDesc), C.POINTER(TreeLayout), P, P, P, I64, I64, D, D, D, I32, U64,
                                  P, P, D, I64, P, P],
                                 C.c_int),
    "rpl_stack_frames": ([P, P, I64, I64, I32, I64, I32, P, P, P], C.c_int),
    "rpl_returns_nstep_dq": ([P, P, I64, I64, I32, D, P, P, I32, I32, D, P, P, P, P], C.c_int),
    "rpl_c51_project": ([P, P, P, P, I64, I32, I32, D, D, D, P, P, P], C.c_int),
    "rpl_replay_validity": ([C.POINTER(TreeLayout), P, I32, I64, I64, I32, I32, I32, I32, I64, I64, I64, I64, P],
                            C.c_int),
    "rpl_debug_priority_values": ([P, I64, D, D, I32, P, P, P], C.c_int),
    "rpl_debug_set_gather_variant": ([I32], C.c_int),
    "rpl_peer_access": ([I32], C.c_int),
    "rpl_debug_set_scan_variant": ([I32], C.c_int),
    "rpl_debug_set_tree_stage": ([I32], C.c_int),
    "rpl_debug_set_gather_diag": ([I32], C.c_int),
    "rpl_debug_trace": ([P, I32], C.c_int),
    "rpl_debug_trace_reset": ([], C.c_int),
    "rpl_debug_scan_trace": ([P, I32], C.c_int),
    "rpl_debug_set_upd_trigger": ([I32], C.c_int),
    "rpl_debug_set_gather_trigger": ([I32], C.c_int),
    "rpl_debug_set_upd_multi": ([I32], C.c_int),
    "rpl_debug_set_gather_dyn": ([I32, I32, I32], C.c_int),
    "rpl_debug_gather_trace": ([P, I32], C.c_int),
    "rpl_debug_gather_cta_ends": ([P, I32], C.c_int),
    "rpl_debug_gather_grabs": ([P, I32], C.c_int),
    "rpl_debug_gather_trace_reset": ([], C.c_int),
}

EXPORTS = tuple(_SIGS)


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"librpl.so not built at {LIB_PATH}: run `python paper_1909_01500_b200/build.py` "
                          "(or __graft_entry__.build()); there is no CPU fallback")
    lib = C.CDLL(LIB_PATH)
    for name, (args, res) in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    return lib


lib = _load()
assert lib.rpl_abi_version() == 2, "librpl ABI version mismatch"


def config() -> dict:
    """rpl_config: the library's build-flag and runtime knob state."""
    import json
    buf = C.create_string_buffer(1024)
    check(lib.rpl_config(buf, len(buf)), "rpl_config")
    return json.loads(buf.value.decode())


class RplError(RuntimeError):
    pass


def check(status: int, what: str = ""):
    if status != RPL_OK:
        msg = lib.rpl_strerror(status).decode()
        raise RplError(f"{what}: {STATUS.get(status, status)} ({msg})")
