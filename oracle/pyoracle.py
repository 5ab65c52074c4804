"""numpy/ctypes front-end over liboracle.so (C restatement) and _ref/libsdattn_ref.so
(the reference itself). TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py."""
from __future__ import annotations

import ctypes as ct
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
FMT_F64, FMT_F32, FMT_BF16, FMT_F16 = 0, 1, 2, 3
_u64, _u32, _f64, _sz, _i64 = ct.c_uint64, ct.c_uint32, ct.c_double, ct.c_size_t, ct.c_int64
_pd = ct.POINTER(ct.c_double)
_pu32 = ct.POINTER(ct.c_uint32)
_pu64 = ct.POINTER(ct.c_uint64)


class OracleError(RuntimeError):
    pass


def build() -> None:
    """Compile liboracle.so and (when /root/reference exists) _ref/libsdattn_ref.so."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _p(a, t):
    return a.ctypes.data_as(t)


def _pd_(a):
    return _p(a, _pd)


def _pu32_(a):
    return _p(a, _pu32)


def shared_seed(master_seed: int, request_id: int) -> int:
    """protocol.cpp:143-145 -- derive_seed(master, {request_id, 0x7365656B})."""
    return C.derive_seed(master_seed, [request_id, 0x7365656B])


def rel_fro(got, ref) -> float:
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    return float(np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-300))


def max_abs_rel(got, ref, axes=(-2, -1)) -> float:
    """max over leading dims of  max|got-ref| / max|ref|  taken per (b, h) slab."""
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    num = np.abs(got - ref).max(axis=axes)
    den = np.maximum(np.abs(ref).max(axis=axes), 1e-300)
    return float((num / den).max())


class Oracle:
    """Shared numpy API over either library (prefix 'or_' for C, 'ref_' for REF)."""

    def __init__(self, lib: ct.CDLL, is_ref: bool):
        self.lib = lib
        self.is_ref = is_ref

    # --- rng ---------------------------------------------------------------
    def rng_u64(self, seed: int, n: int) -> np.ndarray:
        out = np.zeros(n, np.uint64)
        if self.is_ref:
            self.lib.ref_rng_u64(_u64(seed), _sz(n), _p(out, _pu64))
        else:
            st = _OrRng()
            self.lib.or_rng_init(ct.byref(st), _u64(seed))
            for i in range(n):
                out[i] = self.lib.or_next_u64(ct.byref(st))
        return out

    def gaussian(self, seed: int, n: int) -> np.ndarray:
        out = np.zeros(n, np.float64)
        if self.is_ref:
            self.lib.ref_rng_gaussian(_u64(seed), _sz(n), _pd_(out))
        else:
            self.lib.or_gaussian_fill(_u64(seed), _sz(n), _pd_(out))
        return out

    def derive_seed(self, base: int, tags) -> int:
        arr = np.asarray(list(tags), np.uint64)
        fn = self.lib.ref_derive_seed if self.is_ref else self.lib.or_derive_seed
        return int(fn(_u64(base), _p(arr, _pu64), _sz(len(arr))))

    def random_permutation(self, n: int, seed: int) -> np.ndarray:
        out = np.zeros(n, np.uint32)
        if self.is_ref:
            rc = self.lib.ref_random_permutation(_sz(n), _u64(seed), _pu32_(out))
        else:
            st = _OrRng()
            self.lib.or_rng_init(ct.byref(st), _u64(seed))
            rc = self.lib.or_random_permutation(_sz(n), ct.byref(st), _pu32_(out))
        if rc:
            raise OracleError("random_permutation")
        return out

    def span_perm(self, token_perm_seed: int, tag: int, first_pos: int, length: int) -> np.ndarray:
        out = np.zeros(length, np.uint32)
        fn = self.lib.ref_span_perm if self.is_ref else self.lib.or_span_perm
        if fn(_u64(token_perm_seed), _u64(tag), _u64(first_pos), _sz(length), _pu32_(out)):
            raise OracleError("span_perm")
        return out

    def round_to_format(self, x, fmt: int) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float64)
        flat = x.reshape(-1).copy()
        if self.is_ref:
            f = self.lib.ref_round_to_format
            for i in range(flat.size):
                flat[i] = f(_f64(flat[i]), ct.c_int(fmt))
        else:
            self.lib.or_round_array(_pd_(flat), _sz(flat.size), ct.c_int(fmt))
        return flat.reshape(x.shape)

    def fwht(self, x) -> np.ndarray:
        y = np.ascontiguousarray(x, np.float64).copy()
        fn = self.lib.ref_fwht if self.is_ref else self.lib.or_fwht_normalized_inplace
        if fn(_pd_(y), _sz(y.size)):
            raise OracleError("fwht")
        return y

    # --- keys ---------------------------------------------------------------
    def negotiate_keyset(self, shared_seed_: int, request_id: int, layer: int, domain: int,
                         n_heads: int, d: int, lo: float = 0.125, hi: float = 8.0, mode: int = 0):
        """Returns dict with kq_s1/kq_p1/kq_p2/kq_s2/v_* arrays [n_heads, d] and token_perm_seed."""
        ks = {k: np.zeros((n_heads, d), np.float64) for k in ("kq_s1", "kq_s2", "v_s1", "v_s2")}
        ks.update({k: np.zeros((n_heads, d), np.uint32) for k in ("kq_p1", "kq_p2", "v_p1", "v_p2")})
        tps = ct.c_uint64(0)
        if self.is_ref:
            rc = self.lib.ref_negotiate_keyset(
                _u64(shared_seed_), _u64(request_id), _u32(layer), _u32(domain), _sz(n_heads), _sz(d),
                _f64(lo), _f64(hi), ct.c_int(mode), _sz(1), _sz(1),
                _pd_(ks["kq_s1"]), _pu32_(ks["kq_p1"]), _pu32_(ks["kq_p2"]), _pd_(ks["kq_s2"]),
                _pd_(ks["v_s1"]), _pu32_(ks["v_p1"]), _pu32_(ks["v_p2"]), _pd_(ks["v_s2"]),
                None, None, ct.byref(tps))
        else:
            spec = _OrKeyspec(request_id, layer, domain, n_heads, d, lo, hi, mode)
            out = _OrKeyset(_pd_(ks["kq_s1"]), _pu32_(ks["kq_p1"]), _pu32_(ks["kq_p2"]), _pd_(ks["kq_s2"]),
                            _pd_(ks["v_s1"]), _pu32_(ks["v_p1"]), _pu32_(ks["v_p2"]), _pd_(ks["v_s2"]), 0)
            rc = self.lib.or_negotiate_keyset(_u64(shared_seed_), ct.byref(spec), ct.byref(out))
            tps.value = out.token_perm_seed
        if rc:
            raise OracleError("negotiate_keyset")
        ks["token_perm_seed"] = int(tps.value)
        return ks

    # --- operators ----------------------------------------------------------
    def apply_phi(self, x, s1, p1, p2, s2, variant: int) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float64)
        d = x.shape[-1]
        rows = x.size // d
        out = np.zeros_like(x)
        s1 = np.ascontiguousarray(s1, np.float64)
        s2 = np.ascontiguousarray(s2, np.float64)
        p1 = np.ascontiguousarray(p1, np.uint32)
        p2 = np.ascontiguousarray(p2, np.uint32)
        if self.is_ref:
            rc = self.lib.ref_apply_phi(_pd_(x), _sz(rows), _sz(d), _pd_(s1), _pu32_(p1), _pu32_(p2), _pd_(s2),
                                        ct.c_int(variant), _pd_(out))
        else:
            sc = _OrScrambler(d, _pd_(s1), _pu32_(p1), _pu32_(p2), _pd_(s2), 1)
            rc = self.lib.or_apply_phi(_pd_(x), _sz(rows), ct.byref(sc), ct.c_int(variant), _pd_(out))
        if rc:
            raise OracleError("apply_phi")
        return out

    def shard_attention(self, q, k, v, causal_offset=None):
        q = np.ascontiguousarray(q, np.float64)
        k = np.ascontiguousarray(k, np.float64)
        v = np.ascontiguousarray(v, np.float64)
        lq, d = q.shape
        lk = k.shape[0]
        out = np.zeros((lq, d), np.float64)
        m = np.zeros(lq, np.float64)
        s = np.zeros(lq, np.float64)
        kind = 0 if causal_offset is None else 1
        off = 0 if causal_offset is None else int(causal_offset)
        fn = self.lib.ref_shard_attention if self.is_ref else self.lib.or_shard_attention
        if fn(_pd_(q), _sz(lq), _pd_(k), _pd_(v), _sz(lk), _sz(d), ct.c_int(kind), _i64(off),
              _pd_(out), _pd_(m), _pd_(s)):
            raise OracleError("shard_attention")
        return out, m, s

    def merge_shards(self, outs, rmax, esum) -> np.ndarray:
        outs = [np.ascontiguousarray(o, np.float64) for o in outs]
        rmax = [np.ascontiguousarray(o, np.float64) for o in rmax]
        esum = [np.ascontiguousarray(o, np.float64) for o in esum]
        n = len(outs)
        rows, cols = outs[0].shape if n else (0, 0)
        po = (_pd * max(n, 1))(*[_pd_(o) for o in outs])
        pm = (_pd * max(n, 1))(*[_pd_(o) for o in rmax])
        ps = (_pd * max(n, 1))(*[_pd_(o) for o in esum])
        merged = np.zeros((rows, cols), np.float64)
        fn = self.lib.ref_merge_shards if self.is_ref else self.lib.or_merge_shards
        rc = fn(_sz(n), po, pm, ps, _sz(rows), _sz(cols), _pd_(merged))
        if rc:
            raise OracleError(f"merge_shards rc={rc}")
        return merged


    # --- quantised wire (quant.cpp:26-67) ---------------------------------------
    def quantize_affine(self, v, bits: int):
        """-> (codes uint8 [ceil(n*bits/8)], scale f32, zero_point f32)."""
        v = np.ascontiguousarray(v, np.float64).ravel()
        codes = np.zeros((v.size * bits + 7) // 8, np.uint8)
        sc, zp = ct.c_float(0.0), ct.c_float(0.0)
        fn = self.lib.ref_quantize_affine if self.is_ref else self.lib.or_quantize_affine
        if fn(_pd_(v), _sz(v.size), ct.c_int(bits), codes.ctypes.data_as(ct.POINTER(ct.c_uint8)), ct.byref(sc),
              ct.byref(zp)):
            raise OracleError("quantize_affine")
        return codes, np.float32(sc.value), np.float32(zp.value)

    def dequantize(self, codes, n: int, bits: int, scale, zero_point) -> np.ndarray:
        codes = np.ascontiguousarray(codes, np.uint8)
        out = np.zeros(n, np.float64)
        fn = self.lib.ref_dequantize if self.is_ref else self.lib.or_dequantize
        fn(codes.ctypes.data_as(ct.POINTER(ct.c_uint8)), _sz(n), ct.c_int(bits), ct.c_float(float(scale)),
           ct.c_float(float(zero_point)), _pd_(out))
        return out

    # --- wire frames (frame.cpp) ------------------------------------------------------
    def crc32(self, b) -> int:
        b = np.ascontiguousarray(b, np.uint8)
        fn = self.lib.ref_crc32 if self.is_ref else self.lib.or_crc32
        fn.restype = ct.c_uint32
        return int(fn(b.ctypes.data_as(ct.POINTER(ct.c_uint8)), _sz(b.size)))

    def encode_frame(self, msg_type: int, request_id: int, layer: int, head: int, domain: int, dtype: int, dims,
                     values) -> np.ndarray:
        """make_tensor_frame-style frame of `values` (reference only)."""
        v = np.ascontiguousarray(values, np.float64).ravel()
        d = np.ascontiguousarray(dims, np.uint32)
        cap = 64 + 4 * d.size + 8 * max(v.size, 1) + 16
        out = np.zeros(cap, np.uint8)
        n = ct.c_uint64(0)
        rc = self.lib.ref_encode_frame(ct.c_uint8(msg_type), _u64(request_id), ct.c_uint16(layer), ct.c_uint16(head),
                                       ct.c_uint16(domain), ct.c_uint8(dtype), d.ctypes.data_as(ct.POINTER(ct.c_uint32)),
                                       ct.c_uint32(d.size), _pd_(v), out.ctypes.data_as(ct.POINTER(ct.c_uint8)),
                                       _u64(cap), ct.byref(n))
        if rc:
            raise OracleError(f"encode_frame rc={rc}")
        return out[:n.value].copy()

    def decode_frame(self, b, cap: int) -> np.ndarray:
        """decode_frame + values_from_payload (reference only); raises on FrameError."""
        b = np.ascontiguousarray(b, np.uint8)
        out = np.zeros(max(cap, 1), np.float64)
        self.lib.ref_decode_frame.restype = ct.c_longlong
        n = self.lib.ref_decode_frame(b.ctypes.data_as(ct.POINTER(ct.c_uint8)), _u64(b.size), _pd_(out), _u64(cap))
        if n < 0:
            raise OracleError(f"decode_frame rc={n}")
        return out[:n]

    # --- composition ----------------------------------------------------------
    def scrambled_step(self, shared_seed_: int, request_id: int, layer: int, n_heads: int, head: int, q,
                       q_first_pos: int, k_nodes, v_nodes, wire_fmt: int = FMT_F64, lo: float = 0.125,
                       hi: float = 8.0, mode: int = 0, shard_first_pos=None, round_out: bool = False):
        """One (request, head) of the scrambled step composed as the reference protocol does
        (protocol.cpp:885-891 Q', :998-1001 K'/V', :1086 keyless attention, :929-948 dec + merge),
        with Q', K', V' rounded to `wire_fmt` (model.cpp:387-389). O' and the stats stay f64
        unless round_out (the reference's in-process provider also rounds them, model.cpp:392-394).
        Node n is domain n + 1; its shard starts at shard_first_pos[n] (default n * L_k)."""
        q = np.ascontiguousarray(q, np.float64)
        lq, d = q.shape
        shards_o, shards_m, shards_s = [], [], []
        for n, (k, v) in enumerate(zip(k_nodes, v_nodes)):
            k = np.ascontiguousarray(k, np.float64)
            v = np.ascontiguousarray(v, np.float64)
            lk = k.shape[0]
            fp = n * lk if shard_first_pos is None else shard_first_pos[n]
            ks = self.negotiate_keyset(shared_seed_, request_id, layer, n + 1, n_heads, d, lo, hi, mode)
            p_q = self.span_perm(ks["token_perm_seed"], 0, q_first_pos, lq)
            p_kv = self.span_perm(ks["token_perm_seed"], 1, fp, lk)
            kq = (ks["kq_s1"][head], ks["kq_p1"][head], ks["kq_p2"][head], ks["kq_s2"][head])
            vv = (ks["v_s1"][head], ks["v_p1"][head], ks["v_p2"][head], ks["v_s2"][head])
            q_s = self.round_to_format(self.apply_phi(q, *kq, 0)[p_q], wire_fmt)
            k_s = self.round_to_format(self.apply_phi(k, *kq, 1)[p_kv], wire_fmt)
            v_s = self.round_to_format(self.apply_phi(v, *vv, 0)[p_kv], wire_fmt)
            o, m, s = self.shard_attention(q_s, k_s, v_s, None)
            if round_out:
                o = self.round_to_format(o, wire_fmt)
                m = self.round_to_format(m, wire_fmt)
                s = self.round_to_format(s, wire_fmt)
            od = self.apply_phi(o, *vv, 2)
            out = np.zeros_like(od)
            mm = np.zeros_like(m)
            ss = np.zeros_like(s)
            out[p_q], mm[p_q], ss[p_q] = od, m, s
            shards_o.append(out), shards_m.append(mm), shards_s.append(ss)
        return self.merge_shards(shards_o, shards_m, shards_s)


class _OrRng(ct.Structure):
    _fields_ = [("state", ct.c_uint64), ("have_cached", ct.c_int), ("cached", ct.c_double)]


class _OrScrambler(ct.Structure):
    _fields_ = [("dim", ct.c_size_t), ("s1", _pd), ("p1", _pu32), ("p2", _pu32), ("s2", _pd),
                ("with_hadamard", ct.c_int)]


class _OrKeyspec(ct.Structure):
    _fields_ = [("request_id", ct.c_uint64), ("layer", ct.c_uint32), ("domain", ct.c_uint32),
                ("n_heads", ct.c_size_t), ("head_dim", ct.c_size_t), ("mag_lo", ct.c_double),
                ("mag_hi", ct.c_double), ("mode", ct.c_int)]


class _OrKeyset(ct.Structure):
    _fields_ = [("kq_s1", _pd), ("kq_p1", _pu32), ("kq_p2", _pu32), ("kq_s2", _pd),
                ("v_s1", _pd), ("v_p1", _pu32), ("v_p2", _pu32), ("v_s2", _pd),
                ("token_perm_seed", ct.c_uint64)]


def _setup_c(lib: ct.CDLL) -> None:
    lib.or_mix.restype = _u64
    lib.or_next_u64.restype = _u64
    lib.or_next_double.restype = _f64
    lib.or_next_gaussian.restype = _f64
    lib.or_derive_seed.restype = _u64
    lib.or_derive_seed.argtypes = [_u64, _pu64, _sz]
    lib.or_round_to_format.restype = _f64
    lib.or_round_to_format.argtypes = [_f64, ct.c_int]


def _setup_ref(lib: ct.CDLL) -> None:
    lib.ref_derive_seed.restype = _u64
    lib.ref_derive_seed.argtypes = [_u64, _pu64, _sz]
    lib.ref_round_to_format.restype = _f64
    lib.ref_round_to_format.argtypes = [_f64, ct.c_int]
    lib.ref_bench_decode.restype = _f64
    lib.ref_bench_decode.argtypes = [_sz, _sz, _sz, _sz, _sz, ct.c_int, ct.c_int, ct.c_int, _pd]


def load_oracle() -> Oracle:
    path = os.path.join(HERE, "liboracle.so")
    if not os.path.exists(path):
        build()
    lib = ct.CDLL(path)
    _setup_c(lib)
    return Oracle(lib, is_ref=False)


def load_ref():
    path = os.path.join(HERE, "_ref", "libsdattn_ref.so")
    if not os.path.exists(path):
        return None
    lib = ct.CDLL(path)
    _setup_ref(lib)
    return Oracle(lib, is_ref=True)


C = load_oracle()
REF = load_ref()
