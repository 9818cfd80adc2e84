"""CPU checks of the boundary: librpl.so loads (no GPU needed), exports every
symbol include/rpl.h declares, and the ctypes structs match the C layout."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "rpl.h")
PKG = os.path.join(ROOT, "paper_1909_01500_b200")


def declared():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rpl_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    import importlib.util
    spec = importlib.util.spec_from_file_location("_rpl_build", os.path.join(PKG, "build.py"))
    build = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(build)
    build.build()
    return ctypes.CDLL(build.LIB)


def test_exports_every_declared_symbol(lib):
    names = declared()
    assert len(names) >= 19
    for n in names:
        assert hasattr(lib, n), n
    from paper_1909_01500_b200 import _lib
    assert sorted(_lib.EXPORTS) == names


def test_version_and_strerror(lib):
    lib.rpl_abi_version.restype = ctypes.c_int
    assert lib.rpl_abi_version() == 2
    lib.rpl_strerror.restype = ctypes.c_char_p
    assert b"invalid" in lib.rpl_strerror(-1)


def test_struct_layouts_match_c(tmp_path):
    from paper_1909_01500_b200._lib import GatherDesc, TreeLayout
    prog = tmp_path / "sz.c"
    prog.write_text(
        '#include <stdio.h>\n#include <stddef.h>\n#include "rpl.h"\n'
        "int main(){printf(\"%zu %zu %zu %zu %zu %zu %zu %zu %zu %zu\\n\", sizeof(rpl_tree_layout),"
        " offsetof(rpl_tree_layout, q_cap), offsetof(rpl_tree_layout, n_words), sizeof(rpl_gather_desc),"
        " offsetof(rpl_gather_desc, gamma), offsetof(rpl_gather_desc, o_rnn), offsetof(rpl_gather_desc, n_active),"
        " offsetof(rpl_gather_desc, col_offset), offsetof(rpl_gather_desc, peer_boards),"
        " offsetof(rpl_gather_desc, peer_rank));return 0;}\n")
    exe = tmp_path / "sz"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(prog), "-o", str(exe)])
    vals = [int(x) for x in subprocess.check_output([str(exe)]).split()]
    assert vals == [ctypes.sizeof(TreeLayout), TreeLayout.q_cap.offset, TreeLayout.n_words.offset,
                    ctypes.sizeof(GatherDesc), GatherDesc.gamma.offset, GatherDesc.o_rnn.offset,
                    GatherDesc.n_active.offset, GatherDesc.col_offset.offset, GatherDesc.peer_boards.offset,
                    GatherDesc.peer_rank.offset]


def test_host_validation_without_gpu(lib):
    # argument errors are detected on the host before anything is enqueued
    from paper_1909_01500_b200._lib import TreeLayout, lib as L
    lay = TreeLayout()
    assert L.rpl_sumtree_layout(0, 32, 32, ctypes.byref(lay)) == -1
    assert L.rpl_sumtree_layout(100, 3, 32, ctypes.byref(lay)) == -1
    assert L.rpl_sumtree_layout(1 << 20, 32, 32, ctypes.byref(lay)) == 0
    assert lay.depth == 4 and lay.q_cap == ((1 << 63) - 1) // (1 << 20)
    assert [lay.level_len[i] for i in range(5)] == [1, 32, 1024, 32768, 1 << 20]
    assert L.rpl_returns_nstep(None, None, 4, 4, 1, 0.9, None, None, 0, 0.0, None, None, None) == -1
    # later entries: null / out-of-range arguments rejected before any launch
    assert L.rpl_returns_nstep_dq(None, None, 4, 4, 1, 0.9, None, None, 3, 0, 0.0, None, None, None, None) == -1
    assert L.rpl_c51_project(None, None, None, None, 4, 1, 51, -10.0, 10.0, 0.9, None, None, None) == -1
    assert L.rpl_sample_uniform(0, 1, 0, None, 0, 1, 1, 1, None, None) == -1
    assert L.rpl_sumtree_update_seq(ctypes.byref(lay), None, None, None, 0, 4, 0.9, 0.9, 1e-3, 0, None, None) == -1
    assert L.rpl_sumtree_update_seq(ctypes.byref(lay), None, None, None, 80, 4, 1.5, 0.9, 1e-3, 0, None, None) == -1
    assert L.rpl_replay_validity(ctypes.byref(lay), None, 0, 4096, 256, 4, 3, 1, 1, 0, 0, 1, 1, None) == -1
    assert L.rpl_replay_validity(ctypes.byref(lay), 1, 0, 4096, 255, 4, 3, 1, 1, 0, 0, 1, 1, None) == -1  # N mismatch
    assert L.rpl_ring_append(None, None, None, None, None, None, 1, None) == -1
    assert L.rpl_sumtree_update_ex(ctypes.byref(lay), None, None, None, 4, 0.9, 1e-3, 2, None, None) == -1
    us = L.rpl_sumtree_update_sample
    assert us(ctypes.byref(lay), None, None, None, 0, 0, 0.9, 0.9, 1e-3, 0, 64, 1, None, None, None, None) == -1
    assert us(ctypes.byref(lay), 1, None, None, 0, 4, 0.9, 0.9, 1e-3, 0, 64, 1, 1, 1, None, None) == -1  # no idx/td
    assert us(ctypes.byref(lay), 1, None, None, 0, 0, 1.5, 0.9, 1e-3, 0, 64, 1, 1, 1, None, None) == -1  # eta
    assert us(ctypes.byref(lay), 1, None, None, 0, 0, 0.9, 0.9, 1e-3, 4, 64, 1, 1, 1, None, None) == -1  # flags
    assert us(ctypes.byref(lay), 1, None, None, 0, 0, 0.9, 0.9, 1e-3, 0, 0, 1, 1, 1, None, None) == -1   # n
    assert L.rpl_debug_set_gather_variant(99) == -1 and L.rpl_debug_set_gather_diag(99) == -1


def test_product_never_imports_oracle():
    for dirpath, _, files in os.walk(PKG):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle", txt, re.M), f


def test_peer_gather_validation_without_gpu(lib):
    # peer boards (fused K7) need q and o_w and no explicit qmin; rejected on the host
    from paper_1909_01500_b200._lib import GatherDesc, lib as L
    d = GatherDesc()
    d.kind, d.k, d.cap_T, d.B, d.cursor, d.size, d.obs_bytes = 1, 4, 400, 4, 0, 400, 7056
    d.seq_len, d.period = 45, 40
    d.obs, d.done, d.o_obs, d.o_w = 16, 16, 16, 16          # never dereferenced on the host
    d.peer_boards, d.peer_world, d.peer_rank = 16, 2, 0
    one = ctypes.c_void_p(16)
    assert L.rpl_gather(ctypes.byref(d), one, None, None, 0.6, 8, None, None) == -1      # q missing
    assert L.rpl_gather(ctypes.byref(d), one, one, one, 0.6, 8, None, None) == -1       # explicit qmin
    d.peer_rank = 2
    assert L.rpl_gather(ctypes.byref(d), one, one, None, 0.6, 8, None, None) == -1      # rank >= world
    d.peer_rank, d.kind = 0, 0
    assert L.rpl_gather(ctypes.byref(d), one, one, None, 0.6, 8, None, None) == -1      # transitions
    from paper_1909_01500_b200._lib import TreeLayout
    lay = TreeLayout()
    assert L.rpl_sumtree_layout(1000, 32, 32, ctypes.byref(lay)) == 0
    sp = L.rpl_sumtree_sample_sharded_p2p
    assert sp(ctypes.byref(lay), 16, 0, 2, 1000, None, 64, 1, 16, 16, 16, None, None) == -1   # no boards
    assert sp(ctypes.byref(lay), 16, 0, 65, 1000, 16, 64, 1, 16, 16, 16, None, None) == -1    # > 64 shards
    assert sp(ctypes.byref(lay), 16, 0, 2, 1000, 16, 64, 1, 16, 16, None, None, None) == -1   # no count


def test_config_reports_knobs_and_no_diag_build():
    from paper_1909_01500_b200 import _lib
    cfg = _lib.config()
    for key in ("pdl", "tree_stage", "scan_variant", "gather_variant", "gather_diag", "diag_build",
                "seq_consumers", "upd_threads", "sample_warps"):
        assert key in cfg, key
    # the default build carries no work-skipping diagnostics
    assert cfg["diag_build"] == 0 and cfg["gather_diag"] == 0
    assert _lib.lib.rpl_debug_set_gather_diag(1) == -5 and _lib.lib.rpl_debug_set_gather_diag(0) == 0
    buf = ctypes.create_string_buffer(8)
    assert _lib.lib.rpl_config(buf, 8) == -2
