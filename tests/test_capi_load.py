"""The C-ABI library loads without a GPU, exports every symbol include/sdattn_b200.h declares,
and maps the reference's std::invalid_argument cases to status codes before touching a device."""
import ctypes as ct
import os
import re

import pytest

from paper_2605_25716_b200 import capi

HDR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "sdattn_b200.h")


def declared_symbols():
    txt = open(HDR).read()
    return sorted(set(re.findall(r"^\s*(?:[a-z_0-9]+\s*\*?\s+)+\**(sda_[a-z_0-9]+)\s*\(", txt, re.M)))


def test_exports_every_declared_symbol():
    syms = declared_symbols()
    assert len(syms) >= 15
    assert set(syms) == set(capi.EXPORTS)
    for s in syms:
        assert hasattr(capi.LIB, s), s
    assert capi.LIB.sda_abi_version() == 1


def test_status_mapping_without_device():
    L = capi.LIB
    # build_scrambler: d must be a power of two (scrambler.cpp:27)
    assert L.sda_scramble(None, 0, 0, 1, 0, 1, 1, 1, 48, 1, 0, 1, None, 0, 1, 0, 1, 0, 0) == 2
    # d = 2 is valid for the reference but not compiled for the device (4..256 are)
    assert L.sda_scramble(None, 0, 0, 1, 0, 1, 1, 1, 2, 1, 0, 1, None, 0, 1, 0, 1, 0, 0) == 5
    # the LL decode exchange is a d >= 64 form
    assert L.sda_ll_unscramble_merge(None, 1, 1, 1, 1, 0, 1, 1, 1, 16, 1, 0, 1, 1) == 5
    # row offset beyond the cache capacity
    assert L.sda_scramble(None, 0, 0, 1, 0, 1, 1, 4, 64, 1, 0, 1, None, 0, 1, 0, 3, 0, 0) == 1
    # q heads not a multiple of kv heads
    assert L.sda_partial_attention(None, 1, 0, 1, 1, 0, 8, None, 1, 3, 2, 1, 64, 1, 1, 1) == 1
    # merge_shards: empty shard list (attention.cpp:90)
    assert L.sda_unscramble_merge(None, None, 0, 0, 1, 0, 1, 1, 1, 64, 1, 0, None, None, 0) == 3
    with pytest.raises(capi.SdaError):
        capi.span_perm(1, 1, 0, 0)  # negotiate_keyset: lengths must be >= 1
    with pytest.raises(capi.SdaError):
        capi.negotiate_keyset(1, 1, 0, 1, 2, 48)
    assert capi.launch_count() == 0  # nothing above reached a kernel launch
