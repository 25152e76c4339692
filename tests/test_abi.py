"""CPU checks of the C-ABI library: it loads, exports every symbol include/dvc.h
declares, and rejects bad arguments before touching a device (-m "not gpu")."""
import ctypes
import os
import re

import pytest

import synthgen

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "dvc.h")).read()
    return sorted(set(re.findall(r"DVC_API\s+[\w\s\*]*?\b(dvc_\w+)\s*\(", src)))


@pytest.fixture(scope="module")
def L():
    from paper_2601_20564_b200 import _lib
    return _lib.lib()


def test_header_declares_the_boundary():
    names = _declared()
    for n in ("dvc_encode_pixelunshuffle", "dvc_resblock_tsm_forward", "dvc_unet_decode_gop"):
        assert n in names
    assert len(names) >= 18


def test_library_exports_every_declared_symbol(L):
    from paper_2601_20564_b200 import _lib
    for n in _declared():
        assert hasattr(L, n), n
        assert n in _lib.EXPORTS, f"binding lacks {n}"


def test_abi_version_and_status_strings(L):
    assert L.dvc_abi_version() == 3
    assert L.dvc_status_string(2) == b"DVC_ERR_DIVISIBILITY"


def test_argument_errors_before_any_launch(L):
    # null pointers / divisibility are rejected before the device is touched
    assert L.dvc_encode_pixelunshuffle(None, 0, 1, 8, 8, 8, None, None, 192, None, 0, None) == 1
    assert L.dvc_encode_pixelunshuffle(ctypes.c_void_p(16), 0, 1, 12, 16, 8, None, None, 192,
                                       ctypes.c_void_p(16), 0, None) == 2
    assert L.dvc_encode_pixelunshuffle(ctypes.c_void_p(16), 9, 1, 8, 8, 8, None, None, 192,
                                       ctypes.c_void_p(16), 0, None) == 1
    assert L.dvc_encode_pixelunshuffle(ctypes.c_void_p(16), 3, 1, 8, 8, 8, None, None, 192,   # u8 latents
                                       ctypes.c_void_p(16), 3, None) == 1
    assert L.dvc_encode_pixelunshuffle(ctypes.c_void_p(16), 1, 1, 8, 8, 8, None, None, 192,   # f16 -> bf16
                                       ctypes.c_void_p(16), 0, None) == 4


def test_weight_count_matches_generator(L):
    from paper_2601_20564_b200 import _lib
    for width, c in (((240, 480, 960, 960), 256), ((32, 64, 96, 96), 32)):
        cfg = _lib.dvc_unet_config((ctypes.c_int * 4)(*width), c, c, 8, 8, 1e-5, 0, 16, 16, 4)
        n = ctypes.c_size_t()
        assert L.dvc_unet_weight_count(ctypes.byref(cfg), ctypes.byref(n)) == 0
        assert n.value == sum(a.size for _, a in synthgen.unet_weights(width, c, c))


def test_weight_count_is_the_resblock_skeleton_of_table8(L, orc):
    # libdvc's own topology walk: its parameter count equals the oracle's R1 count without attention
    from paper_2601_20564_b200 import _lib
    cfg = _lib.dvc_unet_config((ctypes.c_int * 4)(240, 480, 960, 960), 256, 256, 24, 8, 1e-5, 0, 90, 160, 16)
    n = ctypes.c_size_t()
    L.dvc_unet_weight_count(ctypes.byref(cfg), ctypes.byref(n))
    assert n.value == orc.param_count(attention=False)
