"""Torch-facing wrappers over the C ABI, named after the reference operators they replace.

torch is only plumbing here (device memory, the current CUDA stream); every computation is a
call into libsdattn_b200.so. Tensors must be CUDA, contiguous, bf16 or f32.

  scramble            K1  apply_phi / apply_phi_inv_t + permute_rows_gather  (scrambler.cpp:126-136)
  partial_attention   K2  shard_attention(q', K', V', none)                  (attention.cpp:42-78)
  unscramble_merge    K3  dec_output per source + merge_shards               (scrambler.cpp:138-149,
                                                                             attention.cpp:89-123)
"""
from __future__ import annotations

import ctypes as ct
from dataclasses import dataclass
from typing import Optional, Sequence

import torch

from . import capi
from .capi import check

_DT = {torch.bfloat16: capi.SDA_BF16, torch.float32: capi.SDA_F32, torch.float64: capi.SDA_F64}
_DT_Q = _DT   # the quantised-wire / frame entry points take the same three


def _dtype_code(t: torch.Tensor) -> int:
    """bf16 / f32, or f64 for the FP64 mode (the reference's arithmetic on the device: f64 key
    images, f64 partials and stats)."""
    if t.dtype not in _DT:
        raise TypeError(f"unsupported dtype {t.dtype} (bf16, f32 or f64)")
    return _DT[t.dtype]


def _cuda(t: torch.Tensor, name: str) -> torch.Tensor:
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return t


def _cuda_or_pinned(t: torch.Tensor, name: str) -> torch.Tensor:
    """A CUDA tensor, or a pinned host tensor read/written in place by the kernel over PCIe
    (zero-copy: pinned allocations are device-addressable under UVA)."""
    if not t.is_cuda and not t.is_pinned():
        raise ValueError(f"{name} must be a CUDA tensor or pinned host memory")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return t


def _stream(stream: Optional[torch.cuda.Stream]) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None else t.data_ptr()


def upload_keys(packed: Sequence, device) -> torch.Tensor:
    """Stack per-request packed key sets (numpy uint8) into one device tensor [B, keyset_bytes]."""
    import numpy as np
    arr = np.stack([np.asarray(p, np.uint8) for p in packed])
    return torch.from_numpy(arr).to(device)


def upload_perms(perms: Sequence, device) -> torch.Tensor:
    """Stack per-request u32 permutations into a device int32 tensor [B, L] (same bits as u32)."""
    import numpy as np
    arr = np.stack([np.asarray(p, np.uint32) for p in perms]).view(np.int32)
    return torch.from_numpy(arr).to(device)


def scramble(x: torch.Tensor, keys: torch.Tensor, variant: int, which: int, perm: Optional[torch.Tensor] = None,
             out: Optional[torch.Tensor] = None, out_dtype: Optional[torch.dtype] = None, out_row_offset: int = 0,
             key_heads: Optional[int] = None, n_batch: Optional[int] = None, stream=None) -> torch.Tensor:
    """K1. x [B, H, rows, d] -> out [B, H, cap, d] with out[b,h,off+i] = x[b,h,perm_b[i]] @ phi.

    keys: uint8 [B, keyset_bytes] (request b's key set in row b); perm: int32/u32 [B, rows] or None.
    n_batch > B scrambles x once per stacked key set: request b reads x[b % B] (one query batch
    for several destination domains in one launch).
    x may be pinned host memory (zero-copy read).
    """
    _cuda_or_pinned(x, "x")
    Bx, H, rows, d = x.shape
    B = n_batch or Bx
    kh = key_heads if key_heads is not None else H
    _cuda(keys, "keys")
    if out is None:   # a pinned host x is read in place; its result still lives on the keys' device
        out = torch.empty((B, H, rows, d), dtype=out_dtype or x.dtype, device=x.device if x.is_cuda else keys.device)
    _cuda(out, "out")
    if perm is not None:
        _cuda(perm, "perm")
    check(capi.LIB.sda_scramble(_stream(stream), variant, which, x.data_ptr(), _dtype_code(x), B, H, rows, d,
                                keys.data_ptr(), keys.stride(0) if keys.dim() > 1 else 0, kh, _ptr(perm),
                                perm.stride(0) if perm is not None and perm.dim() > 1 else 0, out.data_ptr(),
                                _dtype_code(out), out.shape[2], out_row_offset, Bx if B != Bx else 0),
          "sda_scramble")
    return out


def scramble_quant(x: torch.Tensor, keys: torch.Tensor, variant: int, which: int, bits: int,
                   perm: Optional[torch.Tensor] = None, out: Optional[torch.Tensor] = None,
                   out_row_offset: int = 0, key_heads: Optional[int] = None, err: Optional[torch.Tensor] = None,
                   stream=None) -> torch.Tensor:
    """K1 with the quantised wire in its epilogue: scramble() followed by dequantize(quantize_affine(.,
    bits)) of every (request, head) tensor (quant.cpp:26-67, wire_round model.cpp:338-341), without a
    separate pass over the output. out f32 (or bf16)."""
    _cuda(x, "x"), _cuda(keys, "keys")
    B, H, rows, d = x.shape
    kh = key_heads if key_heads is not None else H
    if out is None:
        out = torch.empty((B, H, rows, d), dtype=torch.float32, device=x.device)
    _cuda(out, "out")
    if perm is not None:
        _cuda(perm, "perm")
    scratch = torch.empty(2 * B * H, dtype=torch.int64, device=x.device)
    check(capi.LIB.sda_scramble_quant(_stream(stream), variant, which, x.data_ptr(), _dtype_code(x), B, H, rows, d,
                                      keys.data_ptr(), keys.stride(0) if keys.dim() > 1 else 0, kh, _ptr(perm),
                                      perm.stride(0) if perm is not None and perm.dim() > 1 else 0, out.data_ptr(),
                                      _dtype_code(out), out.shape[2], out_row_offset, 0, bits, scratch.data_ptr(),
                                      _ptr(err)), "sda_scramble_quant")
    return out


def scramble_job(x: torch.Tensor, keys: torch.Tensor, variant: int, which: int, perm: Optional[torch.Tensor] = None,
                 out: torch.Tensor = None, out_row_offset: int = 0, key_heads: Optional[int] = None,
                 n_batch: Optional[int] = None) -> capi.ScrambleJob:
    """One K1 job for scramble_batch, with the meaning of the same scramble() call."""
    _cuda(x, "x"), _cuda(out, "out"), _cuda(keys, "keys")
    if perm is not None:
        _cuda(perm, "perm")
    Bx, H, rows, d = x.shape
    B = n_batch or Bx
    return capi.ScrambleJob(variant, which, x.data_ptr(), _dtype_code(x), B, H, rows, keys.data_ptr(),
                            keys.stride(0) if keys.dim() > 1 else 0, key_heads if key_heads is not None else H,
                            _ptr(perm), perm.stride(0) if perm is not None and perm.dim() > 1 else 0, out.data_ptr(),
                            _dtype_code(out), out.shape[2], out_row_offset, Bx if B != Bx else 0)


def scramble_batch(jobs: Sequence[capi.ScrambleJob], head_dim: int, stream=None) -> None:
    """K1 for several jobs in one launch (the span's K and V of ship_segment, + its Q in prefill)."""
    if len(jobs) > capi.MAX_SCRAMBLE_JOBS:
        raise ValueError(f"at most {capi.MAX_SCRAMBLE_JOBS} jobs")
    arr = (capi.ScrambleJob * len(jobs))(*jobs)
    check(capi.LIB.sda_scramble_batch(_stream(stream), head_dim, arr, len(jobs)), "sda_scramble_batch")


def partial_attention(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, kv_len: Optional[torch.Tensor] = None,
                      n_splits: Optional[int] = None, out_o: Optional[torch.Tensor] = None,
                      out_stats: Optional[torch.Tensor] = None, stream=None):
    """K2. q [B, Hq, Lq, d]; k, v [B, Hkv, cap, d]. Returns (o [S,B,Hq,Lq,d] f32, stats [S,B,Hq,Lq,2] f32)."""
    _cuda(q, "q"), _cuda(k, "k"), _cuda(v, "v")
    B, Hq, Lq, d = q.shape
    Hkv, cap = k.shape[1], k.shape[2]
    if k.dtype != v.dtype or k.shape != v.shape:
        raise ValueError("k and v must have the same shape and dtype")
    S = n_splits or capi.default_splits(B, Hq, Lq, cap, kv_heads=Hkv, head_dim=d)
    pdt = torch.float64 if q.dtype == torch.float64 else torch.float32   # partials: f64 in the FP64 mode
    if out_o is None:
        out_o = torch.empty((S, B, Hq, Lq, d), dtype=pdt, device=q.device)
    if out_stats is None:
        out_stats = torch.empty((S, B, Hq, Lq, 2), dtype=pdt, device=q.device)
    if kv_len is not None:
        _cuda(kv_len, "kv_len")
        if kv_len.dtype != torch.int32:
            raise TypeError("kv_len must be int32")
    ws, ws_bytes = (prefill_workspace(B, Hq, Hkv, Lq, cap, d, _dtype_code(q), _dtype_code(k), q.device, stream)
                    if S == 1 else (None, 0))
    check(capi.LIB.sda_partial_attention_ws(_stream(stream), q.data_ptr(), _dtype_code(q), k.data_ptr(), v.data_ptr(),
                                            _dtype_code(k), cap, _ptr(kv_len), B, Hq, Hkv, Lq, d, S,
                                            out_o.data_ptr(), out_stats.data_ptr(), _ptr(ws), ws_bytes),
          "sda_partial_attention_ws")
    return out_o, out_stats


_WORKSPACES = {}


def prefill_workspace(B: int, Hq: int, Hkv: int, Lq: int, cap: int, d: int, q_code: int, kv_code: int,
                      device: torch.device, stream=None):
    """The stream-K workspace of sda_partial_attention_ws for this shape: one buffer per (device,
    stream), grown on demand (launches on one stream are ordered). Its leading per-unit tickets
    must be zero; every launch leaves them zero, so they are re-zeroed only when the shape changes
    (another shape's scratch may lie there). Returns (tensor or None, bytes)."""
    nbytes = int(capi.LIB.sda_prefill_workspace_bytes(B, Hq, Hkv, Lq, cap, d, q_code, kv_code))
    if nbytes == 0:
        return None, 0
    st = _stream(stream)
    key = (device.index if device.index is not None else torch.cuda.current_device(), st)
    shape = (B, Hq, Lq, cap)
    buf, last = _WORKSPACES.get(key, (None, None))
    if buf is None or buf.numel() < nbytes:
        buf = torch.zeros(nbytes, dtype=torch.uint8, device=device)
    elif last != shape:
        buf[:4 * B * Hq * ((Lq + 255) // 256)].zero_()
    _WORKSPACES[key] = (buf, shape)
    return buf, nbytes


def partial_attention_causal(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, causal_offset: int = 0,
                             kv_len: Optional[torch.Tensor] = None, n_splits: int = 1,
                             out_o: Optional[torch.Tensor] = None, out_stats: Optional[torch.Tensor] = None,
                             stream=None):
    """Plaintext causal shard (the inquirer's own span, protocol.cpp:944-947): key j is visible to
    query row i iff j <= i + causal_offset. Returns (o [S,B,Hq,Lq,d], stats [S,B,Hq,Lq,2]).
    bf16, d 128, >= 64 rows: the tensor-core prefill kernel with per-row key limits."""
    _cuda(q, "q"), _cuda(k, "k"), _cuda(v, "v")
    B, Hq, Lq, d = q.shape
    Hkv, cap = k.shape[1], k.shape[2]
    pdt = torch.float64 if q.dtype == torch.float64 else torch.float32
    if out_o is None:
        out_o = torch.empty((n_splits, B, Hq, Lq, d), dtype=pdt, device=q.device)
    if out_stats is None:
        out_stats = torch.empty((n_splits, B, Hq, Lq, 2), dtype=pdt, device=q.device)
    check(capi.LIB.sda_partial_attention_causal(_stream(stream), q.data_ptr(), _dtype_code(q), k.data_ptr(),
                                                v.data_ptr(), _dtype_code(k), cap, _ptr(kv_len), B, Hq, Hkv, Lq, d,
                                                n_splits, causal_offset, out_o.data_ptr(), out_stats.data_ptr()),
          "sda_partial_attention_causal")
    return out_o, out_stats


@dataclass
class MergeSource:
    """One shard for K3: o [B,Hq,Lq,d] f32, stats [B,Hq,Lq,2] f32, keys (phi_v of its domain,
    uint8 [B, keyset_bytes]) or None for plaintext, pq_inv int32/u32 [B, Lq] or None."""
    o: torch.Tensor
    stats: torch.Tensor
    keys: Optional[torch.Tensor] = None
    pq_inv: Optional[torch.Tensor] = None
    batch_stride: int = 0     # elements between requests in o and stats (0 = dense)
    shape: Optional[tuple] = None  # (B, Hq, Lq, d) when o is a flat packed record view


def sources_from_splits(o: torch.Tensor, stats: torch.Tensor, keys: Optional[torch.Tensor] = None,
                        pq_inv: Optional[torch.Tensor] = None) -> list:
    return [MergeSource(o[s], stats[s], keys, pq_inv) for s in range(o.shape[0])]


def unscramble_merge(sources: Sequence[MergeSource], out: Optional[torch.Tensor] = None,
                     out_dtype: torch.dtype = torch.float32, key_heads: Optional[int] = None,
                     out_stats: Optional[torch.Tensor] = None, err_flag: Optional[torch.Tensor] = None,
                     out_batch_stride: int = 0, quant_bits: int = 0, stream=None) -> torch.Tensor:
    """K3. Merged, unscrambled, inverse-permuted output [B, Hq, Lq, d] (or a packed per-request
    record when out_batch_stride is given: out and out_stats then point into the same buffer)."""
    n = len(sources)
    if n > capi.MAX_SOURCES:
        raise ValueError(f"at most {capi.MAX_SOURCES} sources")
    if n == 0:
        check(capi.LIB.sda_unscramble_merge(_stream(stream), None, 0, 0, 0, 0, 0, 1, 0, 32, None, 0, None, None, 0),
              "sda_unscramble_merge")
    B, Hq, Lq, d = sources[0].shape or sources[0].o.shape
    arr = (capi.MergeSource * n)()
    kstride = 0
    pstride = 0
    for i, s in enumerate(sources):
        if not s.o.is_cuda or not s.stats.is_cuda:
            raise ValueError("o and stats must be CUDA tensors")
        arr[i].o, arr[i].stats = s.o.data_ptr(), s.stats.data_ptr()
        arr[i].batch_stride = s.batch_stride
        arr[i].keys = _ptr(s.keys)
        arr[i].pq_inv = _ptr(s.pq_inv)
        if s.keys is not None:
            kstride = s.keys.stride(0) if s.keys.dim() > 1 else 0
        if s.pq_inv is not None:
            pstride = s.pq_inv.stride(0) if s.pq_inv.dim() > 1 else 0
    if out is None:
        out = torch.empty((B, Hq, Lq, d), dtype=out_dtype, device=sources[0].o.device)
    _cuda_or_pinned(out, "out")   # pinned host memory: O stored straight to the host (zero-copy)
    if quant_bits:   # the quantised O' wire on K3's input path (quantize -> dequantize per group tensor)
        groups = 1 + sum(1 for i in range(1, n) if arr[i].keys != arr[i - 1].keys)
        scratch = torch.empty(2 * groups * B * Hq, dtype=torch.int64, device=sources[0].o.device)
        check(capi.LIB.sda_unscramble_merge_quant(_stream(stream), arr, n, kstride, key_heads or Hq, pstride, B, Hq, Lq,
                                                  d, out.data_ptr(), _dtype_code(out), _ptr(out_stats),
                                                  _ptr(err_flag), out_batch_stride, quant_bits, scratch.data_ptr()),
              "sda_unscramble_merge_quant")
        return out
    check(capi.LIB.sda_unscramble_merge(_stream(stream), arr, n, kstride, key_heads or Hq, pstride, B, Hq, Lq, d,
                                        out.data_ptr(), _dtype_code(out), _ptr(out_stats), _ptr(err_flag),
                                        out_batch_stride),
          "sda_unscramble_merge")
    return out


# --- quantised wire (quant.cpp:26-67) -------------------------------------------------------------
def quantize_affine(x: torch.Tensor, bits: int, err: Optional[torch.Tensor] = None, stream=None):
    """x [n, count] (f32 / f64 / bf16; each row one tensor) -> (codes uint8 [n, ceil(count*bits/8)],
    scale f32 [n], zero_point f32 [n]); bit-exact with quantize_affine on the same values."""
    _cuda(x, "x")
    if x.dim() != 2 or x.dtype not in _DT_Q:
        raise ValueError("x must be [n_tensors, count] f32 / f64 / bf16")
    x = x.contiguous()
    n, count = x.shape
    nb = (count * bits + 7) // 8
    codes = torch.zeros((n, max(nb, 1)), dtype=torch.uint8, device=x.device)
    scale = torch.empty(n, dtype=torch.float32, device=x.device)
    zp = torch.empty(n, dtype=torch.float32, device=x.device)
    scratch = torch.empty(2 * max(n, 1), dtype=torch.int64, device=x.device)
    check(capi.LIB.sda_quantize_affine(_stream(stream), x.data_ptr(), _DT_Q[x.dtype], n, count, bits, codes.data_ptr(),
                                       codes.stride(0), scale.data_ptr(), zp.data_ptr(), scratch.data_ptr(), _ptr(err)),
          "sda_quantize_affine")
    return codes[:, :nb], scale, zp


def dequantize(codes: torch.Tensor, scale: torch.Tensor, zero_point: torch.Tensor, count: int, bits: int,
               out_dtype: torch.dtype = torch.float64, stream=None) -> torch.Tensor:
    """codes uint8 [n, >= ceil(count*bits/8)] -> values [n, count] (value = code * scale + zero_point)."""
    _cuda(codes, "codes")
    n = codes.shape[0]
    out = torch.empty((n, count), dtype=out_dtype, device=codes.device)
    check(capi.LIB.sda_dequantize(_stream(stream), codes.data_ptr(), codes.stride(0), scale.data_ptr(),
                                  zero_point.data_ptr(), n, count, bits, out.data_ptr(), _DT_Q[out_dtype]),
          "sda_dequantize")
    return out


def wire_round(x: torch.Tensor, wire_fmt: int, stream=None) -> torch.Tensor:
    """In place: x <- round_to_format(x, wire_fmt) (float_format.cpp:26-58; wire_fmt 0 f64, 1 f32,
    2 bf16, 3 f16), the float-format wire_round of model.cpp:339-348. x: contiguous f32 / f64."""
    _cuda(x, "x")
    if x.dtype not in (torch.float32, torch.float64):
        raise ValueError("x must be f32 or f64")
    check(capi.LIB.sda_wire_round(_stream(stream), x.data_ptr(), _DT_Q[x.dtype], x.numel(), wire_fmt),
          "sda_wire_round")
    return x


def quant_roundtrip(x: torch.Tensor, bits: int, err: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """In place: x[t] <- dequantize(quantize_affine(x[t], bits)) for every row t of x [n, count]
    (the quantised-wire emulation of wire_round, model.cpp:338-341)."""
    _cuda(x, "x")
    if x.dim() != 2 or not x.is_contiguous() or x.dtype not in _DT_Q:
        raise ValueError("x must be a contiguous [n_tensors, count] f32 / f64 / bf16 tensor")
    n, count = x.shape
    scratch = torch.empty(2 * max(n, 1), dtype=torch.int64, device=x.device)
    check(capi.LIB.sda_quant_roundtrip(_stream(stream), x.data_ptr(), _DT_Q[x.dtype], n, count, bits,
                                       scratch.data_ptr(), _ptr(err)), "sda_quant_roundtrip")
    return x


# --- wire frames (frame.cpp) --------------------------------------------------------------------
def frame_header(msg_type: int, request_id: int, layer: int, head: int, domain: int, dtype: int, dims,
                 version: int = 1) -> capi.FrameHeader:
    h = capi.FrameHeader()
    h.version, h.msg_type, h.request_id, h.layer, h.head, h.domain, h.dtype = (version, msg_type, request_id, layer,
                                                                               head, domain, dtype)
    h.n_dims = len(dims)
    for i, d in enumerate(dims):
        h.dims[i] = d
    return h


def frame_encode(h: capi.FrameHeader, x: torch.Tensor, err: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """payload_from_values + encode_frame on the device: x (f32 / f64 / bf16, the frame's elements
    in order) -> uint8 frame bytes (bit-exact with the reference's encoder on the same values)."""
    _cuda(x, "x")
    x = x.contiguous()
    n = capi.LIB.sda_frame_bytes(ct.byref(h))
    out = torch.empty(n, dtype=torch.uint8, device=x.device)
    scratch = torch.empty(capi.LIB.sda_frame_scratch_bytes(n), dtype=torch.uint8, device=x.device)
    check(capi.LIB.sda_frame_encode(_stream(stream), ct.byref(h), x.data_ptr(), _DT_Q[x.dtype], out.data_ptr(),
                                    scratch.data_ptr(), _ptr(err)), "sda_frame_encode")
    return out


def frame_parse_header(head_bytes: bytes, frame_size: int) -> capi.FrameHeader:
    """decode_frame's header checks on the host from the frame's first bytes."""
    h = capi.FrameHeader()
    buf = (ct.c_uint8 * len(head_bytes)).from_buffer_copy(head_bytes)
    check(capi.LIB.sda_frame_parse_header(buf, len(head_bytes), frame_size, ct.byref(h)), "sda_frame_parse_header")
    return h


def frame_decode(frame: torch.Tensor, h: capi.FrameHeader, out_dtype: torch.dtype = torch.float64,
                 err: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """decode_frame's CRC check (-> err = SDA_ERR_FRAME) + values_from_payload on the device."""
    _cuda(frame, "frame")
    n = capi.LIB.sda_frame_elements(ct.byref(h))
    out = torch.empty(n, dtype=out_dtype, device=frame.device)
    scratch = torch.empty(capi.LIB.sda_frame_scratch_bytes(frame.numel()), dtype=torch.uint8, device=frame.device)
    check(capi.LIB.sda_frame_decode(_stream(stream), frame.data_ptr(), frame.numel(), ct.byref(h), out.data_ptr(),
                                    _DT_Q[out_dtype], scratch.data_ptr(), _ptr(err)), "sda_frame_decode")
    return out


def crc32(b: torch.Tensor, stream=None) -> int:
    """CRC-32/IEEE of a device byte tensor (synchronises to read the result)."""
    _cuda(b, "bytes")
    out = torch.zeros(4, dtype=torch.uint8, device=b.device)
    scratch = torch.empty(capi.LIB.sda_frame_scratch_bytes(b.numel()), dtype=torch.uint8, device=b.device)
    check(capi.LIB.sda_crc32(_stream(stream), b.data_ptr(), b.numel(), scratch.data_ptr(), out.data_ptr()), "sda_crc32")
    return int.from_bytes(bytes(out.cpu().numpy()), "little")


# --- K1 fused into the QKV projection (SURVEY 8(f) "next" row 2) ---------------------------------
def project_scrambled(x: torch.Tensor, w: torch.Tensor, keys: torch.Tensor, variant: int, which: int,
                      perm: Optional[torch.Tensor] = None, out: Optional[torch.Tensor] = None, out_row_offset: int = 0,
                      key_heads: Optional[int] = None, rows: Optional[int] = None, stream=None) -> torch.Tensor:
    """Scrambled projection in one tcgen05 kernel (sda_project_scramble): out[b, h, off + r] =
    bf16((x[b, perm_b[r]] @ W_h^T) phi_{b,h}) -- project_qkv (model.cpp:124-133) followed by enc_qkv's
    scramble + row gather (scrambler.cpp:126-136); the projection accumulates in TMEM and the
    scramble runs as a second GEMM in its epilogue, so no unscrambled Q / K / V reaches HBM.
    x bf16 [B, x_rows, d_model]; w bf16 [H * d, d_model] (the nn.Linear weight of the head
    block); keys uint8 [B, keyset_bytes]; perm int32 [B, rows] or None; d 64 or 128."""
    _cuda(x, "x"), _cuda(w, "w"), _cuda(keys, "keys")
    if x.dtype != torch.bfloat16 or w.dtype != torch.bfloat16:
        raise TypeError("x and w must be bf16")
    B, x_rows, dm = x.shape
    if out is None:
        raise ValueError("out [B, H, cap, d] is required (the cache / Q' buffer the kernel writes)")
    _cuda(out, "out")
    _, H, cap, d = out.shape
    if w.shape != (H * d, dm):
        raise ValueError(f"w must be [{H * d}, {dm}]")
    n = rows if rows is not None else (perm.shape[1] if perm is not None else x_rows)
    if perm is not None:
        _cuda(perm, "perm")
    check(capi.LIB.sda_project_scramble(_stream(stream), x.data_ptr(), B, x_rows, dm, w.data_ptr(), H, d,
                                        keys.data_ptr(), keys.stride(0) if keys.dim() > 1 else 0,
                                        key_heads if key_heads is not None else H, variant, which, _ptr(perm),
                                        perm.stride(0) if perm is not None and perm.dim() > 1 else 0, n,
                                        out.data_ptr(), cap, out_row_offset), "sda_project_scramble")
    return out
