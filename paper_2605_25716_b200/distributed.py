"""Multi-GPU form of the scrambled decode step: one process per GPU, one compute domain per GPU.

The reference moves SCR_Q frames inquirer -> compute node and SCR_SHARD frames back
(protocol.cpp:892-896, :1097-1102) over its simulated network. Here every rank is both
  * the compute node of domain `rank + 1` (it holds that domain's scrambled KV shard for all
    requests and runs K2 on whatever Q' arrives), and
  * the inquirer for its own slice of requests (it scrambles their Q once per destination
    domain, K1, and merges + unscrambles the returning partials, K3).
One layer step is therefore: K1 x world -> all_to_all(Q') -> K2 -> split fold -> all_to_all(O',
stats) -> K3. It is not an all-reduce: each domain's partial must be unscrambled with that
domain's phi_V^{-1}, which only the key holder has.

The exchange is plain torch.distributed all_to_all_single (NCCL over NVLink on the GPU box,
gloo in the CPU tests); the per-rank compute is pluggable so the routing logic can be tested
on CPU with the oracle standing in for the kernels.
"""
from __future__ import annotations

import os
from dataclasses import dataclass
from typing import Callable, Optional, Sequence

import torch
import torch.distributed as dist


@dataclass
class StepBuffers:
    """Preallocated exchange buffers for one rank (world W, B_p requests per inquirer).

    The partials travel back as ONE packed f32 record per request, [Hq*Lq*d O' | Hq*Lq*2 stats]
    (K3 writes and reads it with a batch stride), so one all-to-all carries both SCR_SHARD
    frames (protocol.cpp:1097-1102)."""
    q_send: torch.Tensor    # [W, B_p, Hq, Lq, d]   Q' for each destination domain
    q_recv: torch.Tensor    # [W, B_p, Hq, Lq, d]   Q' from each inquirer = [W*B_p, ...] for K2
    ret_send: torch.Tensor  # [W, B_p, rec] f32     this domain's partial for each inquirer's requests
    ret_recv: torch.Tensor  # [W, B_p, rec] f32     every domain's partial for my requests
    dims: tuple             # (Hq, Lq, d)

    @staticmethod
    def allocate(world: int, b_per: int, q_heads: int, q_rows: int, d: int, q_dtype, device) -> "StepBuffers":
        shp = (world, b_per, q_heads, q_rows, d)
        rec = q_heads * q_rows * (d + 2)
        f32 = dict(dtype=torch.float32, device=device)
        return StepBuffers(torch.empty(shp, dtype=q_dtype, device=device), torch.empty(shp, dtype=q_dtype, device=device),
                           torch.empty((world, b_per, rec), **f32), torch.empty((world, b_per, rec), **f32),
                           (q_heads, q_rows, d))


def record_views(ret: torch.Tensor, dims):
    """(o, stats) views [.., B, Hq, Lq, d] / [.., B, Hq, Lq, 2] of packed per-request records."""
    Hq, Lq, d = dims
    n = Hq * Lq * d
    lead = ret.shape[:-1]
    return ret[..., :n].unflatten(-1, (Hq, Lq, d)), ret[..., n:].unflatten(-1, (Hq, Lq, 2))


@dataclass
class RankCompute:
    """The per-rank compute of one step (GPU: the K1/K2/K3 calls of ops.py)."""
    scramble_q: Callable[[torch.Tensor, int, torch.Tensor], None]   # (q, dst_domain, out)
    serve: Callable[[torch.Tensor, torch.Tensor, tuple], None]       # (q_all, ret [B_tot, rec], dims): K2 + fold
    finish: Callable[[torch.Tensor, torch.Tensor, tuple], None]      # (ret_back [W, B_p, rec], out, dims): K3
    scramble_q_all: Optional[Callable[[torch.Tensor, torch.Tensor], None]] = None   # (q, q_send [W, ...]) one launch
    # (q_all, dims, exchange) -> bool: K2 writing every request's record straight into its
    # inquirer's receive slot and raising the return flags (False: not eligible, use serve)
    serve_remote: Optional[Callable[[torch.Tensor, tuple, "PeerExchange"], bool]] = None
    # (q, exchange) -> bool: K1 writing every domain's Q' straight into that domain's receive
    # slot and raising its SCR_Q flag (False: not eligible, use scramble_q_all + exchange_q)
    scramble_q_remote: Optional[Callable[[torch.Tensor, "PeerExchange"], bool]] = None
    # () -> None: the current stream waits for work a step left behind off its path (the span's
    # own K/V scrambled into the local cache, which no later kernel of the step reads)
    drain: Optional[Callable[[], None]] = None


def map_peer_buffers(bufs: dict, group: Optional[dist.ProcessGroup] = None):
    """CUDA-IPC map every rank's buffers {name: tensor} into this process (handles traded once
    with all_gather_object). Returns ({name: [device address on rank r]}, [opened mappings])."""
    import ctypes as ct

    from . import capi
    if not dist.is_initialized():   # one process, one domain: nothing to map
        return {name: [t.data_ptr()] for name, t in bufs.items()}, []
    W, rank = dist.get_world_size(group), dist.get_rank(group)
    mine = {}
    for name, t in bufs.items():
        h = (ct.c_uint8 * 64)()
        off = ct.c_uint64(0)
        capi.check(capi.LIB.sda_ipc_get_handle(t.data_ptr(), h, ct.byref(off)), "ipc_get_handle")
        mine[name] = (bytes(h), int(off.value))
    everyone = [None] * W
    dist.all_gather_object(everyone, mine, group=group)
    ptrs, opened = {name: [0] * W for name in bufs}, []
    for r in range(W):
        for name, t in bufs.items():
            if r == rank:
                ptrs[name][r] = t.data_ptr()
                continue
            hb, off = everyone[r][name]
            ptr = ct.c_void_p()
            capi.check(capi.LIB.sda_ipc_open_handle((ct.c_uint8 * 64).from_buffer_copy(hb), off, ct.byref(ptr)),
                       "ipc_open_handle")
            opened.append((ptr.value, off))
            ptrs[name][r] = ptr.value
    return ptrs, opened


class PeerExchange:
    """SCR_Q / SCR_SHARD over NVLink peer memory (exchange.cu) instead of NCCL all-to-alls.

    Setup maps every peer's q_recv / ret_recv / flags (CUDA IPC handles traded once with
    all_gather_object); each step: epoch += 1, push my Q' slices into the peers' q_recv[my rank]
    and raise their flags, wait for mine, ... the same for the packed (O', stats) records. Same
    data placement as all_to_all_single, so the compute is unchanged."""

    def __init__(self, bufs: StepBuffers, group: Optional[dist.ProcessGroup] = None, rank: Optional[int] = None):
        """rank: this exchange's logical rank inside an in-process LocalWorld (one GPU emulating W
        domains; its peers' buffers are then connected by LocalWorld, not over CUDA IPC)."""
        import ctypes as ct

        from . import capi
        self.capi, self.ct = capi, ct
        self.world = bufs.q_send.shape[0]
        self.rank = dist.get_rank(group) if rank is None else rank
        self.bufs = bufs
        dev = bufs.q_send.device
        W = self.world
        self.flags = torch.zeros(2 * W, dtype=torch.int32, device=dev)      # [SCR_Q from r | SCR_SHARD from r]
        self.epoch = torch.zeros(1, dtype=torch.int32, device=dev)
        self.counters = torch.zeros(2 * W, dtype=torch.int32, device=dev)
        self.k1_counters = torch.zeros(16, dtype=torch.int32, device=dev)   # sda_scramble_batch_remote
        self.opened = []
        if rank is None:
            torch.cuda.synchronize()
            ptrs, self.opened = map_peer_buffers(self.peer_buffers(), group)
            self.connect(ptrs)
            dist.barrier(group=group)

    def peer_buffers(self) -> dict:
        """The buffers every peer writes into (mapped into the peers' address spaces)."""
        return {"q": self.bufs.q_recv, "ret": self.bufs.ret_recv, "flags": self.flags}

    def connect(self, ptrs: dict) -> None:
        """ptrs[name][r]: the address of rank r's peer buffer `name` as this process sees it."""
        ct, bufs, W = self.ct, self.bufs, self.world
        base = {(r, name): ptrs[name][r] for name in ptrs for r in range(W)}
        self.base = base
        q_slot = bufs.q_send[0].numel() * bufs.q_send.element_size()
        r_slot = bufs.ret_send[0].numel() * bufs.ret_send.element_size()
        arr = lambda xs: (ct.c_void_p * W)(*xs)  # noqa: E731
        self.q_args = (arr([bufs.q_send[p].data_ptr() for p in range(W)]),
                       arr([base[(p, "q")] + self.rank * q_slot for p in range(W)]),
                       arr([base[(p, "flags")] + 4 * self.rank for p in range(W)]), q_slot)
        self.r_args = (arr([bufs.ret_send[p].data_ptr() for p in range(W)]),
                       arr([base[(p, "ret")] + self.rank * r_slot for p in range(W)]),
                       arr([base[(p, "flags")] + 4 * (W + self.rank) for p in range(W)]), r_slot)

    def _stream(self):
        return torch.cuda.current_stream().cuda_stream

    def begin_step(self):
        self.capi.check(self.capi.LIB.sda_exchange_epoch(self._stream(), self.epoch.data_ptr()), "exchange_epoch")

    def _push(self, args, counters_off):
        src, dst, flags, nbytes = args
        self.capi.check(self.capi.LIB.sda_exchange_push(self._stream(), self.world, src, dst, flags, nbytes,
                                                         self.epoch.data_ptr(),
                                                         self.counters.data_ptr() + 4 * counters_off), "exchange_push")

    def _wait(self, off):
        self.capi.check(self.capi.LIB.sda_exchange_wait(self._stream(), self.flags.data_ptr() + 4 * off, self.world,
                                                         self.epoch.data_ptr()), "exchange_wait")

    def push_q(self):
        self._push(self.q_args, 0)

    def wait_q(self):
        self._wait(0)

    def push_ret(self):
        self._push(self.r_args, self.world)

    def wait_ret(self):
        self._wait(self.world)

    def exchange_q(self):
        self.push_q()
        self.wait_q()

    def exchange_ret(self):
        self.push_ret()
        self.wait_ret()


class LLDecode:
    """The decode step (L_q = 1) with the exchange carried by the kernels themselves (LL format,
    see include/sdattn_b200.h): K1 writes each destination's Q' straight into its receive slot
    over NVLink, K2 spins on its own slot and writes every split's (O', stats) record straight
    into the inquirer's slot, K3 spins on its slots, merges + unscrambles and opens the next
    epoch. 3 launches, no copy kernel, fence or flag; same results as scrambled_decode_step
    (which stays the reference-shaped form: NCCL all-to-all or PeerExchange). GPU only."""

    def __init__(self, b_per: int, q_heads: int, head_dim: int, inquirer_keys: Sequence, shard,
                 n_splits: Optional[int] = None, kv_heads: Optional[int] = None,
                 wire_dtype: torch.dtype = torch.bfloat16, group: Optional[dist.ProcessGroup] = None,
                 world: Optional[tuple] = None):
        """world: (W, rank) of a logical rank inside an in-process LocalWorld (one GPU emulating W
        domains); its peers' slots are then connected by LocalWorld instead of over CUDA IPC."""
        import ctypes as ct

        from . import capi, ops
        self.capi, self.ops, self.ct = capi, ops, ct
        if world is not None:
            W, rank = world
        else:
            W, rank = (dist.get_world_size(group), dist.get_rank(group)) if dist.is_initialized() else (1, 0)
        self.rank = rank
        dev = shard.k.device
        self.W, self.Bp, self.Hq, self.d = W, b_per, q_heads, head_dim
        self.kv_heads = kv_heads or inquirer_keys[0].kv_heads
        self.keys_all = torch.cat([k.dev for k in inquirer_keys], 0).contiguous()   # [W * B_p, bytes]
        self.shard = shard
        self.S = n_splits or capi.default_splits(W * b_per, q_heads, 1, shard.capacity, kv_heads=shard.k.shape[1],
                                                 head_dim=head_dim)
        self.S = max(1, min(self.S, capi.MAX_SOURCES // W))   # K3 merges W x S split records
        self.wire = ops._DT[wire_dtype]
        q_slot = b_per * q_heads * head_dim * (4 if wire_dtype == torch.bfloat16 else 8)
        r_slot = self.S * b_per * q_heads * (head_dim + 2) * 8
        self.q_ll = torch.zeros(W * q_slot, dtype=torch.uint8, device=dev)
        self.rec_ll = torch.zeros(W * r_slot, dtype=torch.uint8, device=dev)
        self.epoch = torch.ones(1, dtype=torch.int32, device=dev)
        self.done = torch.zeros(1, dtype=torch.int32, device=dev)
        # GQA shards: Q' is unpacked from its LL words into this buffer for the tensor-core kernel
        self.gqa_work = (torch.empty((W * b_per, q_heads, 1, head_dim), dtype=torch.bfloat16, device=dev)
                         if shard.k.shape[1] < q_heads else None)
        if os.environ.get("SDA_SPIN_TIMEOUT_S"):   # spin budget of the LL waits (default 30 s)
            capi.set_spin_timeout(float(os.environ["SDA_SPIN_TIMEOUT_S"]))
        self.q_slot, self.r_slot = q_slot, r_slot
        self.opened = []
        if world is None:
            torch.cuda.synchronize()
            ptrs, self.opened = map_peer_buffers(self.peer_buffers(), group)
            self.connect(ptrs)
            if dist.is_initialized():
                dist.barrier(group=group)

    def peer_buffers(self) -> dict:
        return {"q": self.q_ll, "rec": self.rec_ll}

    def connect(self, ptrs: dict) -> None:
        """ptrs[name][r]: the address of rank r's receive buffer `name` as this process sees it."""
        arr = lambda xs: (self.ct.c_void_p * self.W)(*xs)  # noqa: E731
        self.ll_q = arr([ptrs["q"][r] + self.rank * self.q_slot for r in range(self.W)])     # my slot on every destination
        self.ll_rec = arr([ptrs["rec"][r] + self.rank * self.r_slot for r in range(self.W)])  # my slot on every inquirer

    def scramble_q(self, q: torch.Tensor):
        """K1: span_send_layer for every domain, Q' written into the destinations' slots."""
        st = torch.cuda.current_stream().cuda_stream
        self.capi.check(self.capi.LIB.sda_ll_scramble_q(
            st, q.data_ptr(), self.ops._dtype_code(q), self.W, self.Bp, self.Hq, self.d, self.keys_all.data_ptr(),
            self.keys_all.stride(0), self.kv_heads, self.ll_q, self.wire, self.epoch.data_ptr()), "sda_ll_scramble_q")

    def serve(self):
        """K2: try_serve_q on this domain's shard, every split's record into its inquirer's slot."""
        st, sh = torch.cuda.current_stream().cuda_stream, self.shard
        self.capi.check(self.capi.LIB.sda_ll_partial_attention(
            st, self.q_ll.data_ptr(), self.wire, sh.k.data_ptr(), sh.v.data_ptr(), self.ops._dtype_code(sh.k),
            sh.capacity, sh.kv_len.data_ptr(), self.W, self.Bp, self.Hq, sh.k.shape[1], self.d, self.S, self.ll_rec,
            self.epoch.data_ptr(), None if self.gqa_work is None else self.gqa_work.data_ptr()),
            "sda_ll_partial_attention")

    def finish(self, out: torch.Tensor):
        """K3: span_finish_layer over every domain's split records; opens the next epoch."""
        st = torch.cuda.current_stream().cuda_stream
        self.capi.check(self.capi.LIB.sda_ll_unscramble_merge(
            st, self.rec_ll.data_ptr(), self.W, self.S, self.keys_all.data_ptr(), self.keys_all.stride(0),
            self.kv_heads, self.Bp, self.Hq, self.d, out.data_ptr(), self.ops._dtype_code(out),
            self.epoch.data_ptr(), self.done.data_ptr()), "sda_ll_unscramble_merge")

    def validate(self, t: torch.Tensor, name: str) -> None:
        """Every check that can raise, done before the step's first launch: once K1 has written
        Q' into the peers' slots the step must run to its K3 (which opens the next epoch), or the
        ranks' epochs go out of step."""
        self.ops._cuda_or_pinned(t, name)
        if t.dtype not in (torch.bfloat16, torch.float32):
            raise TypeError(f"{name} must be bf16 or f32, got {t.dtype}")
        if tuple(t.shape) != (self.Bp, self.Hq, 1, self.d):
            raise ValueError(f"{name} must have shape {(self.Bp, self.Hq, 1, self.d)}, got {tuple(t.shape)}")
        if t.is_cuda and t.device != self.shard.k.device:
            raise ValueError(f"{name} is on {t.device}, the shard on {self.shard.k.device}")

    def check(self) -> None:
        """Raise SdaError(SDA_ERR_TIMEOUT) if a spin of this device gave up (a peer is gone)."""
        self.capi.check_spin()

    def step(self, q: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
        """q [B_p, Hq, 1, d] (this rank's requests) -> out [B_p, Hq, 1, d]. Either may be pinned
        host memory (K1 reads Q / K3 stores O over PCIe)."""
        self.validate(q, "q")
        self.validate(out, "out")
        self.scramble_q(q)
        self.serve()
        self.finish(out)
        return out


def connect_domains(objs: Sequence, group: Optional[dist.ProcessGroup] = None) -> list:
    """Several compute domains per process (e.g. BASELINE configs 4 / 5's 8 nodes on 4 GPUs, two
    domains per GPU): objs = this process's LLDecode objects, built with world=(W, domain) for
    global domains rank * len(objs) + i. Every object's receive buffers are mapped into every
    process (CUDA IPC handles traded once) and each object is connected to all W domains' slots --
    the local ones by address, the remote ones through the mapping. Returns the opened mappings."""
    import ctypes as ct

    from . import capi
    names = list(objs[0].peer_buffers().keys())
    mine = []
    for o in objs:
        hs = {}
        for name, t in o.peer_buffers().items():
            h = (ct.c_uint8 * 64)()
            off = ct.c_uint64(0)
            capi.check(capi.LIB.sda_ipc_get_handle(t.data_ptr(), h, ct.byref(off)), "ipc_get_handle")
            hs[name] = (bytes(h), int(off.value))
        mine.append((o.rank, hs))
    P = dist.get_world_size(group) if dist.is_initialized() else 1
    me = dist.get_rank(group) if dist.is_initialized() else 0
    everyone = [None] * P
    if P > 1:
        dist.all_gather_object(everyone, mine, group=group)
    else:
        everyone = [mine]
    W = objs[0].W
    ptrs = {n: [0] * W for n in names}
    opened = []
    local = {o.rank: o for o in objs}
    for r in range(P):
        for dom, hs in everyone[r]:
            for n in names:
                if r == me:
                    ptrs[n][dom] = local[dom].peer_buffers()[n].data_ptr()
                    continue
                hb, off = hs[n]
                ptr = ct.c_void_p()
                capi.check(capi.LIB.sda_ipc_open_handle((ct.c_uint8 * 64).from_buffer_copy(hb), off, ct.byref(ptr)),
                           "ipc_open_handle")
                opened.append((ptr.value, off))
                ptrs[n][dom] = ptr.value
    for o in objs:
        o.connect(ptrs)
    if P > 1:
        dist.barrier(group=group)
    return opened


A2A_Q, A2A_RET, SYNC = "a2a_q", "a2a_ret", "sync"


def decode_step_phases(q: torch.Tensor, compute: RankCompute, bufs: StepBuffers, out: torch.Tensor,
                       exchange: Optional[PeerExchange] = None):
    """One layer step of one rank as a generator of its cross-rank points: it yields A2A_Q /
    A2A_RET where an all-to-all of bufs.q_send -> q_recv / ret_send -> ret_recv is due, and SYNC
    between a peer-memory push (or a kernel that writes into peers' slots) and the wait on the
    flags it raises. scrambled_decode_step drives it with NCCL; LocalWorld drives W of them in
    lockstep on one GPU (every rank's launches of a phase before any rank's next phase)."""
    world = bufs.q_send.shape[0]
    if exchange is not None:
        exchange.begin_step()
    q_sent = (world > 1 and exchange is not None and compute.scramble_q_remote is not None
              and compute.scramble_q_remote(q, exchange))            # K1 wrote Q' into the peers' slots
    if not q_sent:
        if compute.scramble_q_all is not None:                   # span_send_layer, all domains at once
            compute.scramble_q_all(q, bufs.q_send)
        else:
            for dom in range(world):
                compute.scramble_q(q, dom, bufs.q_send[dom])
    if world > 1 and exchange is not None:
        if not q_sent:
            exchange.push_q()                                         # SCR_Q over peer memory
        yield SYNC
        exchange.wait_q()
        q_all = bufs.q_recv
        b_tot = q_all.shape[0] * q_all.shape[1]
        if compute.serve_remote is not None and compute.serve_remote(
                q_all.view((b_tot,) + tuple(q_all.shape[2:])), bufs.dims, exchange):
            yield SYNC                                                # SCR_SHARD written by K2 itself
            exchange.wait_ret()
            compute.finish(bufs.ret_recv, out, bufs.dims)
            return
    elif world > 1:
        yield A2A_Q                                                   # SCR_Q
        q_all = bufs.q_recv
    else:
        q_all = bufs.q_send
    b_tot = q_all.shape[0] * q_all.shape[1]
    compute.serve(q_all.view((b_tot,) + tuple(q_all.shape[2:])),     # try_serve_q on my shard
                  bufs.ret_send.view(b_tot, -1), bufs.dims)
    if world > 1 and exchange is not None:
        exchange.push_ret()                                           # SCR_SHARD over peer memory
        yield SYNC
        exchange.wait_ret()
        back = bufs.ret_recv
    elif world > 1:
        yield A2A_RET                                                 # SCR_SHARD (O' + stats)
        back = bufs.ret_recv
    else:
        back = bufs.ret_send
    compute.finish(back, out, bufs.dims)                          # span_finish_layer


def scrambled_decode_step(q: torch.Tensor, compute: RankCompute, bufs: StepBuffers, out: torch.Tensor,
                          group: Optional[dist.ProcessGroup] = None,
                          exchange: Optional[PeerExchange] = None) -> torch.Tensor:
    """One layer step for this rank's requests q [B_p, Hq, Lq, d]; returns out [B_p, Hq, Lq, d].
    exchange: a PeerExchange to move Q' and the partials over NVLink peer memory (else NCCL)."""
    for ev in decode_step_phases(q, compute, bufs, out, exchange):
        if ev == A2A_Q:
            dist.all_to_all_single(bufs.q_recv, bufs.q_send, group=group)
        elif ev == A2A_RET:
            dist.all_to_all_single(bufs.ret_recv, bufs.ret_send, group=group)
    return out


class LocalWorld:
    """W logical ranks (compute domains 1..W and their inquirers) in ONE process on ONE GPU: the
    multi-GPU step forms with every rank's receive slots in the same device memory, so their
    cross-rank addressing (which domain's slot, which inquirer's record) runs -- and is checked
    against the oracle -- on a 1-GPU box, including W = 8, the node count of BASELINE configs
    4 and 5. Every rank's launches of one phase are issued before any rank's next phase on the
    one stream, so a wait never precedes the writes it waits for. The all-to-alls of the NCCL
    form become the same slot-to-slot copies. Not a product path: the LL / push / remote kernels
    are the ones the multi-GPU step runs, only the peers live in one address space."""

    @staticmethod
    def connect(objs: Sequence) -> None:
        """Wire W LLDecode / PeerExchange objects (built with world=(W, r) / rank=r) to each other."""
        names = objs[0].peer_buffers().keys()
        ptrs = {n: [o.peer_buffers()[n].data_ptr() for o in objs] for n in names}
        for o in objs:
            o.connect(ptrs)

    @staticmethod
    def ll_step(ranks: Sequence["LLDecode"], qs: Sequence[torch.Tensor], outs: Sequence[torch.Tensor]) -> None:
        """One LL decode step of every rank: all K1 (Q' into the domains' slots), all K2, all K3."""
        for r, x in enumerate(ranks):
            x.validate(qs[r], "q")
            x.validate(outs[r], "out")
        for r, x in enumerate(ranks):
            x.scramble_q(qs[r])
        for x in ranks:
            x.serve()
        for r, x in enumerate(ranks):
            x.finish(outs[r])

    @staticmethod
    def decode_step(qs: Sequence[torch.Tensor], computes: Sequence[RankCompute], bufs: Sequence[StepBuffers],
                    outs: Sequence[torch.Tensor], exchanges: Optional[Sequence[PeerExchange]] = None) -> None:
        """scrambled_decode_step of every rank, phase by phase (NCCL form: exchanges None)."""
        W = len(qs)
        gens = [decode_step_phases(qs[r], computes[r], bufs[r], outs[r], None if exchanges is None else exchanges[r])
                for r in range(W)]
        while True:
            evs = [next(g, None) for g in gens]
            if all(e is None for e in evs):
                return
            if len(set(evs)) != 1:
                raise RuntimeError(f"ranks out of step: {evs}")
            if evs[0] == A2A_Q:       # q_recv[r][s] = q_send[s][r] (all_to_all_single)
                for r in range(W):
                    for src in range(W):
                        bufs[r].q_recv[src].copy_(bufs[src].q_send[r])
            elif evs[0] == A2A_RET:
                for r in range(W):
                    for src in range(W):
                        bufs[r].ret_recv[src].copy_(bufs[src].ret_send[r])


def gpu_rank_compute(inquirer_keys: Sequence, shard, n_splits: Optional[int] = None,
                     kv_heads: Optional[int] = None, q_first_pos: int = 0,
                     local_kv: Optional[tuple] = None, local_offset: int = 0,
                     side_work: Optional[Callable[[], None]] = None) -> RankCompute:
    """RankCompute backed by libsdattn_b200.so. inquirer_keys[dom] = DomainKeys of my requests on
    domain dom + 1; shard = this rank's protocol.KVShard (all requests' rows of my domain).
    q_first_pos: global position of the query span (its rows are shuffled by each domain's
    span_perm(0, q_first_pos, L_q), identity for single-row decode).
    local_kv: (k, v) plaintext [B_p, Hkv, L_local, d] of the inquirer's own span: attended with the
    causal mask at local_offset (= q_first_pos - the local keys' first position) and merged by K3
    as a plaintext source, as span_finish_layer does (protocol.cpp:941-947).
    side_work: launches off the step's path (e.g. the span's own K/V scrambled into the local
    cache, protocol.cpp:885-891), run on the side stream ahead of the local span."""
    from . import capi, ops

    state = {}
    # key sets of my requests for every destination domain, stacked domain-major [W * B_p, bytes]
    keys_all = torch.cat([k.dev for k in inquirer_keys], 0).contiguous()

    def q_perms(lq):
        """(p_q stacked [W*B_p, L_q] for K1, [p_q^{-1} of domain dom]) -- None for L_q = 1."""
        if lq == 1:
            return None, [None] * len(inquirer_keys)
        if state.get("lq") != lq:
            fwd, inv = zip(*[k.span_perms(0, q_first_pos, lq) for k in inquirer_keys])
            state["lq"], state["pq"], state["pq_inv"] = lq, torch.cat(fwd, 0).contiguous(), list(inv)
        return state["pq"], state["pq_inv"]

    def start_local(q):
        """Launch the span's causal local attention (plaintext Q, K, V: independent of K1's Q', of
        the exchange and of K2) on a side stream once this step's K1 is queued, so it fills the SMs
        the exchange waits and K2's stream-K tail leave idle; finish joins it before K3. The side
        stream has the lowest priority: on a higher-priority step stream (bench.py) K2's CTAs go
        first. SDA_LOCAL_SERIAL=1 runs it in finish on the step stream instead."""
        state["q_plain"] = q
        state["local_ev"] = None
        if (local_kv is None and side_work is None) or os.environ.get("SDA_LOCAL_SERIAL"):
            if side_work is not None:
                side_work()
            return
        cur = torch.cuda.current_stream(q.device)
        if state.get("side") is None:
            state["side"] = torch.cuda.Stream(device=q.device, priority=0)
            state["fork"], state["join"] = torch.cuda.Event(), torch.cuda.Event()
        side = state["side"]
        state["fork"].record(cur)          # after K1 and after the previous step's K3 (it read lo / ls)
        side.wait_event(state["fork"])
        with torch.cuda.stream(side):
            # the causal span first: K3 joins it; the side work (nothing in this step reads it)
            # follows behind the join, so K3 does not wait for it -- it fills the SMs K3 and the
            # next step's K1 leave idle (SDA_SIDE_FIRST=1: side work ahead of the span, joined)
            side_first = os.environ.get("SDA_SIDE_FIRST") == "1"
            if side_work is not None and (side_first or local_kv is None):
                side_work()
            if local_kv is not None:
                run_local(q)
            state["join"].record(side)
            if side_work is not None and not (side_first or local_kv is None):
                side_work()
                if state.get("tail") is None:
                    state["tail"] = torch.cuda.Event()
                state["tail"].record(side)
                state["tail_pending"] = True
        state["local_ev"] = state["join"]

    def drain():
        if state.get("tail_pending"):
            torch.cuda.current_stream().wait_event(state["tail"])
            state["tail_pending"] = False

    def run_local(q):
        Bp, Hq, Lq, d = q.shape
        key = ("local", Bp, Hq, Lq, d)
        if state.get("lkey") != key:
            state["lkey"] = key
            state["lo"] = torch.empty((1, Bp, Hq, Lq, d), dtype=torch.float32, device=q.device)
            state["ls"] = torch.empty((1, Bp, Hq, Lq, 2), dtype=torch.float32, device=q.device)
        ops.partial_attention_causal(q, local_kv[0], local_kv[1], causal_offset=local_offset,
                                     n_splits=1, out_o=state["lo"], out_stats=state["ls"])

    def scramble_q_all(q, q_send):
        W = q_send.shape[0]
        pq, _ = q_perms(q.shape[2])
        ops.scramble(q, keys_all, capi.PHI_FORWARD, capi.KEYS_KQ, pq, out=q_send.view((-1,) + tuple(q_send.shape[2:])),
                     key_heads=kv_heads or inquirer_keys[0].kv_heads, n_batch=W * q.shape[0])
        start_local(q)

    def scramble_q(q, dom, out):
        pq, _ = q_perms(q.shape[2])
        ops.scramble(q, inquirer_keys[dom].dev, capi.PHI_FORWARD, capi.KEYS_KQ,
                     None if pq is None else pq[dom * q.shape[0]:(dom + 1) * q.shape[0]], out=out,
                     key_heads=kv_heads or inquirer_keys[dom].kv_heads)
        if dom == len(inquirer_keys) - 1:
            start_local(q)

    def serve(q_all, ret, dims):
        B, Hq, Lq, d = q_all.shape
        S = n_splits or capi.default_splits(B, Hq, Lq, shard.capacity, kv_heads=shard.k.shape[1], head_dim=d)
        key = (S, B, Hq, Lq, d)
        if state.get("key") != key:
            state["key"] = key
            state["o"] = torch.empty((S, B, Hq, Lq, d), dtype=torch.float32, device=q_all.device)
            state["st"] = torch.empty((S, B, Hq, Lq, 2), dtype=torch.float32, device=q_all.device)
        ops.partial_attention(q_all, shard.k, shard.v, shard.kv_len, n_splits=S, out_o=state["o"],
                              out_stats=state["st"])
        # fold this domain's splits in scrambled space (plain merge, no keys) straight into the packed
        # per-request records: one O' and one (row_max, exp_sum) per row, what SCR_SHARD carries
        rec = ret.shape[-1]
        ops.unscramble_merge(ops.sources_from_splits(state["o"], state["st"]), out=ret,
                             out_stats=ret[:, Hq * Lq * d:], out_batch_stride=rec)

    def serve_remote(q_all, dims, ex):
        B, Hq, Lq, d = q_all.shape
        if Lq < 64 or d != 128 or q_all.dtype != torch.bfloat16 or shard.k.dtype != torch.bfloat16:
            return False
        import ctypes as ct
        L = capi.LIB
        ws, ws_bytes = ops.prefill_workspace(B, Hq, shard.k.shape[1], Lq, shard.capacity, d, capi.SDA_BF16,
                                             capi.SDA_BF16, q_all.device)
        capi.check(L.sda_partial_attention_remote(
            torch.cuda.current_stream().cuda_stream, q_all.data_ptr(), capi.SDA_BF16, shard.k.data_ptr(),
            shard.v.data_ptr(), capi.SDA_BF16, shard.capacity, shard.kv_len.data_ptr(), ex.world, B // ex.world, Hq,
            shard.k.shape[1], Lq, d, ct.cast(ex.r_args[1], ct.POINTER(ct.c_void_p)), Hq * Lq * (d + 2),
            ct.cast(ex.r_args[2], ct.POINTER(ct.c_void_p)), ex.epoch.data_ptr(),
            ex.counters.data_ptr() + 4 * ex.world, 0 if ws is None else ws.data_ptr(), ws_bytes),
            "sda_partial_attention_remote")
        return True

    def scramble_q_remote(q, ex):
        # TMA stores straight into peer memory: +3-5 % at N=2, +0.4-3 % at N=4 on C3 against K1
        # into q_send + the push kernel (SDA_K1_REMOTE=0 selects the latter)
        Bp, Hq, Lq, d = q.shape
        if os.environ.get("SDA_K1_REMOTE") == "0":
            return False
        if Lq < 128 or d not in (64, 128) or q.dtype != torch.bfloat16 or ex.world > 16:
            return False
        import ctypes as ct
        pq, _ = q_perms(Lq)
        kh = kv_heads or inquirer_keys[0].kv_heads
        q = q.contiguous()
        jobs = (capi.ScrambleJob * ex.world)()
        for dom in range(ex.world):
            kd = inquirer_keys[dom].dev
            perm = pq[dom * Bp:(dom + 1) * Bp]
            jobs[dom] = capi.ScrambleJob(capi.PHI_FORWARD, capi.KEYS_KQ, q.data_ptr(), capi.SDA_BF16, Bp, Hq, Lq,
                                         kd.data_ptr(), kd.stride(0) if kd.dim() > 1 else 0, kh, perm.data_ptr(),
                                         perm.stride(0), ex.q_args[1][dom], capi.SDA_BF16, Lq, 0, 0)
        flags = (ct.c_void_p * ex.world)(*[ex.q_args[2][dom] for dom in range(ex.world)])
        capi.check(capi.LIB.sda_scramble_batch_remote(torch.cuda.current_stream().cuda_stream, d, jobs, ex.world,
                                                      flags, ex.epoch.data_ptr(), ex.k1_counters.data_ptr()),
                   "sda_scramble_batch_remote")
        start_local(q)
        return True

    def finish(back, out, dims):
        Hq, Lq, d = dims
        W, Bp, rec = back.shape
        _, pq_inv = q_perms(Lq)
        srcs = [ops.MergeSource(back[dom], back[dom, :, Hq * Lq * d:], inquirer_keys[dom].dev, pq_inv[dom],
                                batch_stride=rec, shape=(Bp, Hq, Lq, d)) for dom in range(W)]
        joined = state.get("local_ev") is not None
        if joined:
            torch.cuda.current_stream(out.device).wait_event(state["local_ev"])
            state["local_ev"] = None
        if local_kv is not None:   # the inquirer's own span, plaintext, causal (no keys, no p_q)
            if not joined:
                run_local(state["q_plain"])
            srcs += ops.sources_from_splits(state["lo"], state["ls"])
        ops.unscramble_merge(srcs, out=out, key_heads=kv_heads or inquirer_keys[0].kv_heads)

    return RankCompute(scramble_q, serve, finish, scramble_q_all, serve_remote, scramble_q_remote, drain)
