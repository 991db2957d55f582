"""CPU checks of the C-ABI boundary: the library loads, exports every symbol
``include/ragsched_b200.h`` declares, and the ctypes / numpy struct mirrors
have the header's sizes.  No compute calls (no GPU here)."""

import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from paper_2412_10543_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2412_10543_b200 import build

        build.build()
    return _lib.load()


def test_header_declares_expected_entry_points():
    syms = _lib.header_symbols()
    for name in ("rs_select", "rs_prune_gate", "rs_index_search", "rs_merge_topk", "rs_call_latency",
                 "rs_plan_bytes", "rs_index_create", "rs_index_add"):
        assert name in syms
    assert set(syms) == set(_lib.SIGNATURES), set(syms) ^ set(_lib.SIGNATURES)


def test_library_exports_every_header_symbol(lib):
    for name in _lib.header_symbols():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (rs_\w+)", out))
    assert set(_lib.header_symbols()) <= exported


def test_abi_version_and_error_channel(lib):
    assert lib.rs_abi_version() == 1
    assert isinstance(lib.rs_last_error(), bytes)


def test_struct_sizes_match_header():
    src = r"""
#include <stdio.h>
#include <stddef.h>
#include "ragsched_b200.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu %zu %zu %zu %zu %zu %zu %zu\n", sizeof(rs_profile), sizeof(rs_space),
         sizeof(rs_config), sizeof(rs_select_params), sizeof(rs_cost_model), sizeof(rs_gate_params),
         sizeof(rs_window), offsetof(rs_profile, confidence), sizeof(rs_call), sizeof(rs_admit_params),
         sizeof(rs_admit_info), sizeof(rs_admit_result));
  printf("%zu %zu\n", sizeof(rs_candidate), sizeof(rs_peer_exchange));
  return 0;
}
"""
    tmp = os.path.join(ROOT, "oracle", "_build")
    os.makedirs(tmp, exist_ok=True)
    c = os.path.join(tmp, "sizes.c")
    exe = os.path.join(tmp, "sizes")
    open(c, "w").write(src)
    subprocess.check_call(["/usr/bin/gcc", "-I", os.path.join(ROOT, "include"), c, "-o", exe])
    sizes = [int(x) for x in subprocess.check_output([exe]).split()]
    assert sizes == [_lib.PROFILE_DTYPE.itemsize, _lib.SPACE_DTYPE.itemsize, _lib.CONFIG_DTYPE.itemsize,
                     ctypes.sizeof(_lib.SelectParamsC), ctypes.sizeof(_lib.CostModelC),
                     ctypes.sizeof(_lib.GateParamsC), _lib.WINDOW_DTYPE.itemsize,
                     _lib.PROFILE_DTYPE.fields["confidence"][1], _lib.CALL_DTYPE.itemsize,
                     ctypes.sizeof(_lib.AdmitParamsC), _lib.ADMIT_INFO_DTYPE.itemsize,
                     _lib.ADMIT_RESULT_DTYPE.itemsize, _lib.CANDIDATE_DTYPE.itemsize,
                     ctypes.sizeof(_lib.PeerExchangeC)]


def test_sass_contains_tcgen05_and_tma():
    """The retrieval kernel is a real tcgen05/TMA/TMEM kernel (SASS mnemonics
    per B200_PROFILING.md), not an mma.sync fallback."""
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("library not built")
    r = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True, text=True)
    sass = r.stdout
    assert "UTCHMMA" in sass and "UTMALDG" in sass and "LDTM" in sass
    assert "HMMA" not in re.sub(r"UTCHMMA", "", sass)


def test_gpu_entry_points_refuse_without_device():
    """No CUDA device here: the compute API must fail loudly, never fall back."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2412_10543_b200 import batch

    with pytest.raises(_lib.LibraryUnavailable):
        batch.default_device()


def test_packing_roundtrip():
    from paper_2412_10543_b200 import batch, mapping, types

    s = mapping.PrunedConfigSpace(frozenset({types.SynthesisMethod.STUFF, types.SynthesisMethod.MAP_REDUCE}),
                                  types.IntRange(3, 9), types.IntRange(40, 120))
    rec = batch.pack_spaces([s])
    assert batch.unpack_space(rec[0]) == s
    raw = np.zeros(1, dtype=_lib.CONFIG_DTYPE)
    raw["method"], raw["status"], raw["num_chunks"], raw["interlen"] = 4, 0, 7, 60
    assert batch.unpack_config(raw[0]) == types.RagConfig(types.SynthesisMethod.MAP_REDUCE, 7, 60)
    raw["status"] = 2
    assert batch.unpack_config(raw[0]) is None
    raw["status"] = 3
    with pytest.raises(OverflowError):
        batch.unpack_config(raw[0])
    p = mapping.QueryProfile(True, True, 4, types.IntRange(30, 90), 0.93)
    pr = batch.pack_profiles([p])[0]
    assert (pr["complexity_high"], pr["needs_joint_reasoning"], pr["pieces_required"], pr["summary_lo"],
            pr["summary_hi"], pr["confidence"]) == (1, 1, 4, 30, 90, 0.93)


def test_argument_errors_return_codes_without_a_device(lib):
    """Argument validation happens before any CUDA call: bad inputs come back as
    RS_ERR_INVALID_ARG with a message (the Python layer raises ValueError),
    nothing throws across the ABI."""
    sp = _lib.SelectParamsC(131072, 1000, 10, 64, 35, 1, 10, 1, 0)
    bad_sp = _lib.SelectParamsC(0, 1000, 10, 64, 35, 1, 10, 1, 0)
    ap = _lib.AdmitParamsC(0, 0, 131072)  # capacity must be positive
    res = lib.rs_admit_fifo(None, None, None, None, 0, ctypes.byref(sp), ctypes.byref(ap), None, None, None, None)
    assert res == _lib.RS_ERR_INVALID_ARG and lib.rs_last_error()
    dummy = ctypes.c_int64(0)
    assert lib.rs_candidate_costs(None, None, None, 1, ctypes.byref(bad_sp), None, ctypes.addressof(dummy), None,
                                  None, 0, None) == _lib.RS_ERR_INVALID_ARG
    assert b"per_token_bytes" in lib.rs_last_error()
    assert lib.rs_select(None, None, None, None, -1, ctypes.byref(sp), None, None, None, None,
                         None) == _lib.RS_ERR_INVALID_ARG
    assert lib.rs_plan_calls(None, None, 5, ctypes.byref(sp), 131072, None, None, None, None, None, 0,
                             None) == _lib.RS_ERR_INVALID_ARG
    assert lib.rs_parse_profiles(b"", None, -1, None, None, None, None, None, 0) == _lib.RS_ERR_INVALID_ARG
    with pytest.raises(ValueError):
        _lib.check(_lib.RS_ERR_INVALID_ARG, "probe")


def test_parse_profiles_runs_on_the_host(lib):
    """rs_parse_profiles is host code: it works in this GPU-less container."""
    from paper_2412_10543_b200 import batch

    recs, clamped, status, lines = batch.parse_profiles(
        ["Complexity: High\nJoint Reasoning needed: No\nPieces: 12\nSummary range: 40-90", "nothing"], [0.5, 1.0])
    assert list(status) == [batch.RS_PARSE_OK, batch.RS_PARSE_UNPARSEABLE]
    assert recs[0]["pieces_required"] == 10 and clamped[0] == batch.RS_CLAMPED_PIECES
    assert recs[0]["confidence"] == 0.5 and list(lines[0]) == [0, 1, 2, 3]


def test_peer_exchange_layout_and_argument_checks(lib):
    """rs_peer_*: region size arithmetic and argument validation need no device
    (the region header is 512 bytes, then two parity buffers of
    [world][slice_cap][k] 8-byte keys)."""
    nbytes = ctypes.c_uint64()
    assert lib.rs_peer_region_bytes(8, 1024, 35, ctypes.byref(nbytes)) == _lib.RS_OK
    assert nbytes.value == 512 + 2 * 8 * 1024 * 35 * 8
    assert lib.rs_peer_region_bytes(_lib.PEER_MAX + 1, 1, 1, ctypes.byref(nbytes)) == _lib.RS_ERR_INVALID_ARG
    ex = _lib.PeerExchangeC(2, 2, 35, 0, 16)  # rank == world
    assert lib.rs_peer_scatter_keys(ctypes.byref(ex), None, 0, 1, None) == _lib.RS_ERR_INVALID_ARG
    assert b"rank" in lib.rs_last_error()
    ex = _lib.PeerExchangeC(0, 2, 35, 0, 16)  # regions not mapped
    assert lib.rs_peer_merge_topk(ctypes.byref(ex), 32, 1, 35, None, None, None, 0, None) == _lib.RS_ERR_INVALID_ARG
    assert b"region" in lib.rs_last_error()
    assert lib.rs_peer_scatter_keys(None, None, 0, 1, None) == _lib.RS_ERR_INVALID_ARG
