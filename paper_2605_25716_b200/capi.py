"""ctypes binding of the C ABI in include/sdattn_b200.h (libsdattn_b200.so).

This is the same binding a reference-side maintainer would write; the
package uses it for its torch-facing helpers, tests and bench. There is no fallback: if the
library is missing or a call fails, this module raises.
"""
from __future__ import annotations

import ctypes as ct
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SDA_LIB_PATH") or os.path.join(HERE, "libsdattn_b200.so")   # override: kernel-variant experiments

SDA_OK = 0
SDA_BF16, SDA_F32, SDA_F64 = 0, 1, 2
PHI_FORWARD, PHI_INV_T, PHI_INV = 0, 1, 2
KEYS_KQ, KEYS_V = 0, 1
MODE_S1_AND_S2, MODE_S1_ONLY = 0, 1
MAX_SOURCES = 64
STATUS_NAMES = {0: "SDA_OK", 1: "SDA_ERR_INVALID_ARGUMENT", 2: "SDA_ERR_NOT_POW2", 3: "SDA_ERR_EMPTY_SHARDS",
                4: "SDA_ERR_MASKED_ROW", 5: "SDA_ERR_UNSUPPORTED", 6: "SDA_ERR_CUDA", 7: "SDA_ERR_NO_DEVICE",
                8: "SDA_ERR_ROLE_VIOLATION", 9: "SDA_ERR_FRAME", 10: "SDA_ERR_TIMEOUT"}
SDA_ERR_TIMEOUT = 10

# Every symbol include/sdattn_b200.h declares (checked by tests/test_capi_load.py).
EXPORTS = ("sda_derive_seed", "sda_shared_seed", "sda_random_permutation", "sda_negotiate_keyset",
           "sda_span_perm", "sda_invert_permutation", "sda_keyset_bytes", "sda_pack_keyset", "sda_scramble",
           "sda_partial_attention", "sda_partial_attention_causal", "sda_default_splits", "sda_default_splits_gqa", "sda_unscramble_merge", "sda_abi_version",
           "sda_status_string", "sda_launch_count", "sda_ipc_get_handle", "sda_ipc_open_handle",
           "sda_ipc_close_handle", "sda_exchange_epoch", "sda_exchange_push", "sda_exchange_wait",
           "sda_ll_scramble_q", "sda_ll_partial_attention", "sda_ll_unscramble_merge", "sda_trace_timestamp", "sda_scramble_batch",
           "sda_quantize_affine", "sda_dequantize", "sda_quant_roundtrip",
           "sda_frame_elements", "sda_frame_payload_bytes", "sda_frame_bytes", "sda_frame_scratch_bytes",
           "sda_frame_encode", "sda_frame_parse_header", "sda_frame_decode", "sda_crc32",
           "sda_partial_attention_remote", "sda_scramble_batch_remote", "sda_partial_attention_ws",
           "sda_prefill_workspace_bytes", "sda_set_spin_timeout_ns", "sda_spin_error",
           "sda_wire_round", "sda_keyset_bytes_f64", "sda_pack_keyset_f64", "sda_scramble_quant",
           "sda_unscramble_merge_quant", "sda_project_scramble")


class SdaError(RuntimeError):
    def __init__(self, status: int, what: str):
        self.status = status
        super().__init__(f"{what}: {STATUS_NAMES.get(status, status)} ({_status_string(status)})")


_pd = ct.POINTER(ct.c_double)
_pu32 = ct.POINTER(ct.c_uint32)
_pu64 = ct.POINTER(ct.c_uint64)
_vp = ct.c_void_p


class Keyspec(ct.Structure):
    _fields_ = [("request_id", ct.c_uint64), ("layer", ct.c_uint32), ("domain", ct.c_uint32),
                ("n_heads", ct.c_uint32), ("head_dim", ct.c_uint32), ("mag_lo", ct.c_double),
                ("mag_hi", ct.c_double), ("mode", ct.c_int32)]


class HostKeysetC(ct.Structure):
    _fields_ = [("kq_s1", _pd), ("kq_p1", _pu32), ("kq_p2", _pu32), ("kq_s2", _pd),
                ("v_s1", _pd), ("v_p1", _pu32), ("v_p2", _pu32), ("v_s2", _pd),
                ("token_perm_seed", ct.c_uint64)]


class ScrambleJob(ct.Structure):
    """sda_scramble_job: the arguments of one sda_scramble call."""
    _fields_ = [("variant", ct.c_int32), ("which_keys", ct.c_int32), ("x", _vp), ("x_dtype", ct.c_int32),
                ("n_batch", ct.c_int64), ("n_heads", ct.c_int32), ("rows", ct.c_int64), ("keys", _vp),
                ("keys_batch_stride", ct.c_int64), ("key_heads", ct.c_int32), ("perm", _vp),
                ("perm_batch_stride", ct.c_int64), ("out", _vp), ("out_dtype", ct.c_int32),
                ("out_rows_cap", ct.c_int64), ("out_row_offset", ct.c_int64), ("x_batch_mod", ct.c_int64)]


MAX_SCRAMBLE_JOBS = 16
SDA_ERR_FRAME = 9
FRAME_MAX_DIMS = 8


class FrameHeader(ct.Structure):
    """sda_frame_header (frame.hpp:48-66)."""
    _fields_ = [("version", ct.c_uint8), ("msg_type", ct.c_uint8), ("request_id", ct.c_uint64), ("layer", ct.c_uint16),
                ("head", ct.c_uint16), ("domain", ct.c_uint16), ("dtype", ct.c_uint8), ("n_dims", ct.c_uint32),
                ("dims", ct.c_uint32 * FRAME_MAX_DIMS)]


class MergeSource(ct.Structure):
    _fields_ = [("o", _vp), ("stats", _vp), ("keys", _vp), ("pq_inv", _vp), ("batch_stride", ct.c_int64)]


def _load() -> ct.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(there is no CPU fallback)")
    lib = ct.CDLL(LIB_PATH)
    lib.sda_derive_seed.restype = ct.c_uint64
    lib.sda_derive_seed.argtypes = [ct.c_uint64, _pu64, ct.c_size_t]
    lib.sda_shared_seed.restype = ct.c_uint64
    lib.sda_shared_seed.argtypes = [ct.c_uint64, ct.c_uint64]
    lib.sda_random_permutation.argtypes = [ct.c_size_t, ct.c_uint64, _pu32]
    lib.sda_negotiate_keyset.argtypes = [ct.c_uint64, ct.POINTER(Keyspec), ct.POINTER(HostKeysetC)]
    lib.sda_span_perm.argtypes = [ct.c_uint64, ct.c_uint64, ct.c_uint64, ct.c_size_t, _pu32]
    lib.sda_invert_permutation.argtypes = [_pu32, ct.c_size_t, _pu32]
    lib.sda_keyset_bytes.restype = ct.c_size_t
    lib.sda_keyset_bytes.argtypes = [ct.c_uint32, ct.c_uint32]
    lib.sda_pack_keyset.argtypes = [ct.POINTER(HostKeysetC), ct.c_uint32, ct.c_uint32, _vp]
    lib.sda_keyset_bytes_f64.restype = ct.c_size_t
    lib.sda_keyset_bytes_f64.argtypes = [ct.c_uint32, ct.c_uint32]
    lib.sda_pack_keyset_f64.argtypes = [ct.POINTER(HostKeysetC), ct.c_uint32, ct.c_uint32, _vp]
    lib.sda_scramble.argtypes = [_vp, ct.c_int32, ct.c_int32, _vp, ct.c_int32, ct.c_int64, ct.c_int32, ct.c_int64,
                                 ct.c_int32, _vp, ct.c_int64, ct.c_int32, _vp, ct.c_int64, _vp, ct.c_int32,
                                 ct.c_int64, ct.c_int64, ct.c_int64]
    lib.sda_partial_attention.argtypes = [_vp, _vp, ct.c_int32, _vp, _vp, ct.c_int32, ct.c_int64, _vp, ct.c_int64,
                                          ct.c_int32, ct.c_int32, ct.c_int64, ct.c_int32, ct.c_int32, _vp, _vp]
    lib.sda_partial_attention_ws.argtypes = [_vp, _vp, ct.c_int32, _vp, _vp, ct.c_int32, ct.c_int64, _vp, ct.c_int64,
                                             ct.c_int32, ct.c_int32, ct.c_int64, ct.c_int32, ct.c_int32, _vp, _vp, _vp,
                                             ct.c_size_t]
    lib.sda_prefill_workspace_bytes.restype = ct.c_size_t
    lib.sda_prefill_workspace_bytes.argtypes = [ct.c_int64, ct.c_int32, ct.c_int32, ct.c_int64, ct.c_int64, ct.c_int32,
                                                ct.c_int32, ct.c_int32]
    lib.sda_partial_attention_causal.argtypes = [_vp, _vp, ct.c_int32, _vp, _vp, ct.c_int32, ct.c_int64, _vp,
                                                 ct.c_int64, ct.c_int32, ct.c_int32, ct.c_int64, ct.c_int32,
                                                 ct.c_int32, ct.c_int64, _vp, _vp]
    lib.sda_default_splits.restype = ct.c_int32
    lib.sda_default_splits.argtypes = [ct.c_int64, ct.c_int32, ct.c_int64, ct.c_int64]
    lib.sda_default_splits_gqa.restype = ct.c_int32
    lib.sda_default_splits_gqa.argtypes = [ct.c_int64, ct.c_int32, ct.c_int32, ct.c_int64, ct.c_int64, ct.c_int32]
    lib.sda_unscramble_merge.argtypes = [_vp, ct.POINTER(MergeSource), ct.c_int32, ct.c_int64, ct.c_int32,
                                         ct.c_int64, ct.c_int64, ct.c_int32, ct.c_int64, ct.c_int32, _vp, ct.c_int32,
                                         _vp, _vp, ct.c_int64]
    lib.sda_unscramble_merge_quant.argtypes = lib.sda_unscramble_merge.argtypes + [ct.c_int32, _vp]
    lib.sda_scramble_quant.argtypes = lib.sda_scramble.argtypes + [ct.c_int32, _vp, _vp]
    lib.sda_project_scramble.argtypes = [_vp, _vp, ct.c_int64, ct.c_int64, ct.c_int32, _vp, ct.c_int32, ct.c_int32,
                                         _vp, ct.c_int64, ct.c_int32, ct.c_int32, ct.c_int32, _vp, ct.c_int64,
                                         ct.c_int64, _vp, ct.c_int64, ct.c_int64]
    lib.sda_ipc_get_handle.argtypes = [_vp, _vp, ct.POINTER(ct.c_uint64)]
    lib.sda_ipc_open_handle.argtypes = [_vp, ct.c_uint64, ct.POINTER(ct.c_void_p)]
    lib.sda_ipc_close_handle.argtypes = [_vp, ct.c_uint64]
    lib.sda_exchange_epoch.argtypes = [_vp, _vp]
    lib.sda_exchange_push.argtypes = [_vp, ct.c_int32, ct.POINTER(ct.c_void_p), ct.POINTER(ct.c_void_p),
                                      ct.POINTER(ct.c_void_p), ct.c_uint64, _vp, _vp]
    lib.sda_exchange_wait.argtypes = [_vp, _vp, ct.c_int32, _vp]
    lib.sda_set_spin_timeout_ns.argtypes = [ct.c_uint64]
    lib.sda_spin_error.argtypes = [ct.POINTER(ct.c_int32), ct.c_int32]
    _pp = ct.POINTER(ct.c_void_p)
    lib.sda_ll_scramble_q.argtypes = [_vp, _vp, ct.c_int32, ct.c_int32, ct.c_int64, ct.c_int32, ct.c_int32, _vp,
                                      ct.c_int64, ct.c_int32, _pp, ct.c_int32, _vp]
    lib.sda_ll_partial_attention.argtypes = [_vp, _vp, ct.c_int32, _vp, _vp, ct.c_int32, ct.c_int64, _vp, ct.c_int32,
                                             ct.c_int64, ct.c_int32, ct.c_int32, ct.c_int32, ct.c_int32, _pp, _vp, _vp]
    lib.sda_ll_unscramble_merge.argtypes = [_vp, _vp, ct.c_int32, ct.c_int32, _vp, ct.c_int64, ct.c_int32, ct.c_int64,
                                            ct.c_int32, ct.c_int32, _vp, ct.c_int32, _vp, _vp]
    lib.sda_trace_timestamp.argtypes = [_vp, _vp]
    lib.sda_scramble_batch.argtypes = [_vp, ct.c_int32, ct.POINTER(ScrambleJob), ct.c_int32]
    lib.sda_scramble_batch_remote.argtypes = [_vp, ct.c_int32, ct.POINTER(ScrambleJob), ct.c_int32,
                                              ct.POINTER(ct.c_void_p), _vp, _vp]
    _ph = ct.POINTER(FrameHeader)
    for f in ("sda_frame_elements", "sda_frame_payload_bytes", "sda_frame_bytes"):
        getattr(lib, f).restype = ct.c_uint64
        getattr(lib, f).argtypes = [_ph]
    lib.sda_frame_scratch_bytes.restype = ct.c_uint64
    lib.sda_frame_scratch_bytes.argtypes = [ct.c_uint64]
    lib.sda_frame_encode.argtypes = [_vp, _ph, _vp, ct.c_int32, _vp, _vp, _vp]
    lib.sda_frame_parse_header.argtypes = [_vp, ct.c_uint64, ct.c_uint64, _ph]
    lib.sda_frame_decode.argtypes = [_vp, _vp, ct.c_uint64, _ph, _vp, ct.c_int32, _vp, _vp]
    lib.sda_crc32.argtypes = [_vp, _vp, ct.c_uint64, _vp, _vp]
    lib.sda_partial_attention_remote.argtypes = [_vp, _vp, ct.c_int32, _vp, _vp, ct.c_int32, ct.c_int64, _vp,
                                                 ct.c_int32, ct.c_int64, ct.c_int32, ct.c_int32, ct.c_int64, ct.c_int32,
                                                 _pp, ct.c_int64, _pp, _vp, _vp, _vp, ct.c_size_t]
    lib.sda_quantize_affine.argtypes = [_vp, _vp, ct.c_int32, ct.c_int64, ct.c_int64, ct.c_int32, _vp, ct.c_int64,
                                        _vp, _vp, _vp, _vp]
    lib.sda_dequantize.argtypes = [_vp, _vp, ct.c_int64, _vp, _vp, ct.c_int64, ct.c_int64, ct.c_int32, _vp, ct.c_int32]
    lib.sda_wire_round.argtypes = [_vp, _vp, ct.c_int32, ct.c_int64, ct.c_int32]
    lib.sda_quant_roundtrip.argtypes = [_vp, _vp, ct.c_int32, ct.c_int64, ct.c_int64, ct.c_int32, _vp, _vp]
    lib.sda_abi_version.restype = ct.c_int32
    lib.sda_status_string.restype = ct.c_char_p
    lib.sda_status_string.argtypes = [ct.c_int32]
    lib.sda_launch_count.restype = ct.c_uint64
    return lib


LIB = _load()


def _status_string(s: int) -> str:
    return LIB.sda_status_string(int(s)).decode()


def check(status: int, what: str) -> None:
    if status != SDA_OK:
        raise SdaError(status, what)


def launch_count() -> int:
    return int(LIB.sda_launch_count())


def set_spin_timeout(seconds: float) -> None:
    """Spin budget of the peer-memory waits on the current device (default 30 s)."""
    check(LIB.sda_set_spin_timeout_ns(int(seconds * 1e9)), "sda_set_spin_timeout_ns")


def check_spin(clear: bool = True) -> None:
    """Raise SdaError(SDA_ERR_TIMEOUT) if a peer-memory wait on the current device gave up since the
    last check (synchronous; call between steps)."""
    v = ct.c_int32(0)
    check(LIB.sda_spin_error(ct.byref(v), 1 if clear else 0), "sda_spin_error")
    check(v.value, "peer-memory wait")


# ---------------------------------------------------------------------------------------------
# host key derivation (bit-exact, CPU)
# ---------------------------------------------------------------------------------------------
def derive_seed(base: int, tags) -> int:
    arr = np.ascontiguousarray(list(tags), np.uint64)
    return int(LIB.sda_derive_seed(base, arr.ctypes.data_as(_pu64), len(arr)))


def shared_seed(master_seed: int, request_id: int) -> int:
    return int(LIB.sda_shared_seed(master_seed, request_id))


def random_permutation(n: int, seed: int) -> np.ndarray:
    out = np.zeros(n, np.uint32)
    check(LIB.sda_random_permutation(n, seed, out.ctypes.data_as(_pu32)), "random_permutation")
    return out


def span_perm(token_perm_seed: int, tag: int, first_pos: int, length: int) -> np.ndarray:
    out = np.zeros(length, np.uint32)
    check(LIB.sda_span_perm(token_perm_seed, tag, first_pos, length, out.ctypes.data_as(_pu32)), "span_perm")
    return out


def invert_permutation(p: np.ndarray) -> np.ndarray:
    p = np.ascontiguousarray(p, np.uint32)
    out = np.zeros_like(p)
    check(LIB.sda_invert_permutation(p.ctypes.data_as(_pu32), p.size, out.ctypes.data_as(_pu32)),
          "invert_permutation")
    return out


class HostKeyset:
    """negotiate_keyset result (scrambler.cpp:105-124): f64 factors and u32 permutations."""

    FIELDS_F = ("kq_s1", "kq_s2", "v_s1", "v_s2")
    FIELDS_U = ("kq_p1", "kq_p2", "v_p1", "v_p2")

    def __init__(self, n_heads: int, head_dim: int):
        self.n_heads, self.head_dim = n_heads, head_dim
        for f in self.FIELDS_F:
            setattr(self, f, np.zeros((n_heads, head_dim), np.float64))
        for f in self.FIELDS_U:
            setattr(self, f, np.zeros((n_heads, head_dim), np.uint32))
        self.token_perm_seed = 0

    def _c(self) -> HostKeysetC:
        return HostKeysetC(*(getattr(self, f).ctypes.data_as(_pd if f in self.FIELDS_F else _pu32)
                             for f in ("kq_s1", "kq_p1", "kq_p2", "kq_s2", "v_s1", "v_p1", "v_p2", "v_s2")),
                           self.token_perm_seed)

    def span_perm(self, tag: int, first_pos: int, length: int) -> np.ndarray:
        return span_perm(self.token_perm_seed, tag, first_pos, length)

    def pack(self) -> np.ndarray:
        """Device image (sda_pack_keyset), as a host uint8 array."""
        out = np.zeros(int(LIB.sda_keyset_bytes(self.n_heads, self.head_dim)), np.uint8)
        c = self._c()
        check(LIB.sda_pack_keyset(ct.byref(c), self.n_heads, self.head_dim, out.ctypes.data), "pack_keyset")
        return out

    def pack_f64(self) -> np.ndarray:
        """FP64-mode device image (sda_pack_keyset_f64), as a host uint8 array."""
        out = np.zeros(int(LIB.sda_keyset_bytes_f64(self.n_heads, self.head_dim)), np.uint8)
        c = self._c()
        check(LIB.sda_pack_keyset_f64(ct.byref(c), self.n_heads, self.head_dim, out.ctypes.data), "pack_keyset_f64")
        return out


def negotiate_keyset(shared_seed_: int, request_id: int, layer: int, domain: int, n_heads: int, head_dim: int,
                     mag_lo: float = 0.125, mag_hi: float = 8.0, mode: int = MODE_S1_AND_S2) -> HostKeyset:
    ks = HostKeyset(n_heads, head_dim)
    spec = Keyspec(request_id, layer, domain, n_heads, head_dim, mag_lo, mag_hi, mode)
    c = ks._c()
    check(LIB.sda_negotiate_keyset(shared_seed_, ct.byref(spec), ct.byref(c)), "negotiate_keyset")
    ks.token_perm_seed = int(c.token_perm_seed)
    return ks


def keyset_bytes(n_heads: int, head_dim: int) -> int:
    return int(LIB.sda_keyset_bytes(n_heads, head_dim))


def default_splits(n_batch: int, q_heads: int, q_rows: int, kv_cap: int, kv_heads: int = None,
                   head_dim: int = 128) -> int:
    if kv_heads is None:
        return int(LIB.sda_default_splits(n_batch, q_heads, q_rows, kv_cap))
    return int(LIB.sda_default_splits_gqa(n_batch, q_heads, kv_heads, q_rows, kv_cap, head_dim))
