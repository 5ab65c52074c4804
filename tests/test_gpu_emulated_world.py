"""Multi-domain parity the 1-GPU driver box runs: W logical ranks on one GPU (distributed.LocalWorld)
through the multi-GPU step forms -- the LL decode (K1/K2/K3 carrying the exchange), the
push/wait peer exchange, the NCCL-shaped form (all-to-alls as slot copies) and the prefill
remote forms (K1 / K2 writing into the peers' slots and raising their flags) -- each checked
against the oracle's W-node composition C.scrambled_step (protocol.cpp:885-891, :998-1001, :1086,
:921-949) on >= 32 sampled (request, head) pairs, at W = 2, 4 and 8 (the node count of BASELINE
configs 4 and 5: K3's 8 x S merge, the LL split clamp)."""
import numpy as np
import pytest
import torch

from paper_2605_25716_b200 import distributed as sdist
from paper_2605_25716_b200 import protocol
from tests.gpu_helpers import Case, dev, max_abs_rel, rel_fro

pytestmark = pytest.mark.gpu

TOL = {torch.bfloat16: 2e-2, torch.float32: 1e-3}


class World:
    """W domains x B_p requests per inquirer; request b = r * B_p + i belongs to inquirer r, and
    its context is sharded over the W domains (lk rows each, domain r + 1 on rank r)."""

    def __init__(self, W, Bp, Hq, Hkv, d, lk, lq, dtype, seed):
        self.W, self.Bp, self.Hq, self.Hkv, self.d, self.lk, self.lq, self.dtype = W, Bp, Hq, Hkv, d, lk, lq, dtype
        self.case = Case(B=W * Bp, Hq=Hq, Hkv=Hkv, d=d, lk=lk, n_nodes=W, lq=lq, dtype=dtype, seed=seed)
        c = self.case
        self.shards, self.inq = [], []
        for r in range(W):
            own = protocol.DomainKeys(c.request_ids(), 0, r + 1, Hkv, d, "cuda")
            sh = protocol.KVShard(W * Bp, Hkv, lk, d, "cuda", dtype)
            sh.ship_segment(dev(c.k[r], dtype), dev(c.v[r], dtype), own, first_pos=r * lk)
            self.shards.append(sh)
            ids = [r * Bp + i + 1 for i in range(Bp)]
            self.inq.append([protocol.DomainKeys(ids, 0, dom + 1, Hkv, d, "cuda") for dom in range(W)])
        self.q_all = dev(c.q, dtype)

    def q(self, r):
        return self.q_all[r * self.Bp:(r + 1) * self.Bp].contiguous()

    def outs(self):
        return [torch.full((self.Bp, self.Hq, self.lq, self.d), float("nan"), dtype=torch.float32, device="cuda")
                for _ in range(self.W)]

    def check(self, outs, n_pairs=32, seed=0):
        got = torch.cat(outs, 0).double().cpu().numpy()
        rng = np.random.default_rng(seed)
        B = self.W * self.Bp
        pairs = [(int(b), int(h)) for b, h in zip(rng.integers(0, B, n_pairs), rng.integers(0, self.Hq, n_pairs))]
        # every rank's first and last request are always among the pairs (the cross-rank slots)
        pairs += [(r * self.Bp + i, (r + i) % self.Hq) for r in range(self.W) for i in (0, self.Bp - 1)]
        ref = self.case.oracle(pairs)
        tol = TOL[self.dtype]
        for b, h in pairs:
            assert np.all(np.isfinite(got[b, h])), (b, h)
            assert max_abs_rel(got[b, h], ref[b, h]) < tol, (b, h, max_abs_rel(got[b, h], ref[b, h]))
            assert rel_fro(got[b, h], ref[b, h]) < tol, (b, h)
        return got


@pytest.mark.parametrize("W,S", [(2, None), (4, 3), (8, 4), (8, 8)])
def test_ll_decode_emulated_world(W, S):
    """LL decode: every K1 writes Q' into the W domains' slots, every K2 writes its S split
    records into the W inquirers' slots, every K3 merges W x S records (S = 8 at W = 8: 64
    sources, past the 32-source fast path; splits 4..7 of a 512-key shard are empty)."""
    w = World(W, 2, 8, 8, 128, 512, 1, torch.bfloat16, seed=100 + W)
    ranks = [sdist.LLDecode(w.Bp, w.Hq, w.d, w.inq[r], w.shards[r], n_splits=S, kv_heads=w.Hkv, world=(W, r))
             for r in range(W)]
    sdist.LocalWorld.connect(ranks)
    if S is not None:
        assert ranks[0].S == min(S, 64 // W)
    for step in range(2):   # the epoch advances; stale words of the previous step must never be taken
        outs = w.outs()
        sdist.LocalWorld.ll_step(ranks, [w.q(r) for r in range(W)], outs)
        torch.cuda.synchronize()
        w.check(outs, seed=step)
    for x in ranks:
        x.check()
        assert int(x.epoch.item()) == 3


def test_ll_decode_emulated_world_graph_and_f32_wire():
    """W = 2, f32 KV + f32 wire (the FP32 mode, 1e-3 vs the oracle), the whole emulated step
    captured once and replayed."""
    W = 2
    w = World(W, 2, 4, 4, 64, 384, 1, torch.float32, seed=7)
    ranks = [sdist.LLDecode(w.Bp, w.Hq, w.d, w.inq[r], w.shards[r], n_splits=3, kv_heads=w.Hkv,
                            wire_dtype=torch.float32, world=(W, r)) for r in range(W)]
    sdist.LocalWorld.connect(ranks)
    qs = [w.q(r) for r in range(W)]
    outs = w.outs()
    sdist.LocalWorld.ll_step(ranks, qs, outs)
    torch.cuda.synchronize()
    w.check(outs)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        sdist.LocalWorld.ll_step(ranks, qs, outs)
    for _ in range(3):
        for o in outs:
            o.fill_(float("nan"))
        g.replay()
        torch.cuda.synchronize()
        w.check(outs)
    assert int(ranks[1].epoch.item()) == 1 + 1 + 3   # start 1, one eager step, 3 replays


def test_ll_decode_emulated_world_gqa():
    """GQA shards (16 q heads on 2 kv heads, d 128, bf16): K2 unpacks Q' from its LL words and
    runs the tensor-core GQA kernel, writing LL records into both inquirers' slots."""
    W = 2
    w = World(W, 2, 16, 2, 128, 1024, 1, torch.bfloat16, seed=9)
    ranks = [sdist.LLDecode(w.Bp, w.Hq, w.d, w.inq[r], w.shards[r], kv_heads=w.Hkv, world=(W, r)) for r in range(W)]
    assert ranks[0].gqa_work is not None
    sdist.LocalWorld.connect(ranks)
    outs = w.outs()
    sdist.LocalWorld.ll_step(ranks, [w.q(r) for r in range(W)], outs)
    torch.cuda.synchronize()
    w.check(outs)


def _computes(w, n_splits=None):
    return [sdist.gpu_rank_compute(w.inq[r], w.shards[r], n_splits=n_splits, kv_heads=w.Hkv,
                                   q_first_pos=w.case.q_first_pos) for r in range(w.W)]


@pytest.mark.parametrize("W", [2, 4, 8])
@pytest.mark.parametrize("form", ["push", "nccl"])
def test_decode_step_emulated_world(W, form):
    """The reference-shaped step (K1 -> SCR_Q -> K2 + split fold -> SCR_SHARD -> K3) with the
    exchange as push/wait kernels over the peers' slots, or as the all-to-all's slot copies."""
    w = World(W, 2, 8, 8, 128, 512, 1, torch.bfloat16, seed=200 + W)
    bufs = [sdist.StepBuffers.allocate(W, w.Bp, w.Hq, 1, w.d, torch.bfloat16, "cuda") for _ in range(W)]
    ex = None
    if form == "push":
        ex = [sdist.PeerExchange(bufs[r], rank=r) for r in range(W)]
        sdist.LocalWorld.connect(ex)
    comps = _computes(w, n_splits=3)
    for step in range(2):
        outs = w.outs()
        sdist.LocalWorld.decode_step([w.q(r) for r in range(W)], comps, bufs, outs, ex)
        torch.cuda.synchronize()
        w.check(outs, seed=step)


@pytest.mark.parametrize("W", [2, 4])
def test_prefill_remote_emulated_world(W):
    """Prefill spans (256 rows, d 128, bf16, one split): K1 TMA-stores every domain's Q' into the
    domain's receive slot and raises its SCR_Q flag (sda_scramble_batch_remote); K2 writes every
    request's packed record into its inquirer's slot and raises the SCR_SHARD flag
    (sda_partial_attention_remote); K3 merges with the p_q^-1 gathers."""
    w = World(W, 1, 4, 4, 128, 1024, 256, torch.bfloat16, seed=300 + W)
    bufs = [sdist.StepBuffers.allocate(W, w.Bp, w.Hq, w.lq, w.d, torch.bfloat16, "cuda") for _ in range(W)]
    ex = [sdist.PeerExchange(bufs[r], rank=r) for r in range(W)]
    sdist.LocalWorld.connect(ex)
    comps = _computes(w, n_splits=1)
    used = {"k1": 0, "k2": 0}
    for c in comps:   # the remote forms must be the ones that ran
        k1, k2 = c.scramble_q_remote, c.serve_remote

        def k1w(q, e, _f=k1):
            ok = _f(q, e)
            used["k1"] += ok
            return ok

        def k2w(q, dims, e, _f=k2):
            ok = _f(q, dims, e)
            used["k2"] += ok
            return ok
        c.scramble_q_remote, c.serve_remote = k1w, k2w
    outs = w.outs()
    sdist.LocalWorld.decode_step([w.q(r) for r in range(W)], comps, bufs, outs, ex)
    torch.cuda.synchronize()
    assert used == {"k1": W, "k2": W}
    got = torch.cat(outs, 0).double().cpu().numpy()
    rows = [0, 1, 100, 255]
    ref = w.case.oracle([(b, h) for b in range(W * w.Bp) for h in range(w.Hq)])
    for b in range(W * w.Bp):
        for h in range(w.Hq):
            assert max_abs_rel(got[b, h], ref[b, h]) < 2e-2 and rel_fro(got[b, h], ref[b, h]) < 2e-2, (b, h)
            assert np.all(np.isfinite(got[b, h, rows]))


@pytest.mark.parametrize("serial", [False, True], ids=["side_stream", "serial"])
def test_prefill_with_causal_local_span_emulated_world(serial, monkeypatch):
    """span_finish_layer with the inquirer's own span (protocol.cpp:941-948): every domain's
    scrambled partial + the span's own K/V attended in plaintext with the causal mask (tensor-core
    K2 with per-row key limits), all merged by K3 -- against plain attention over [every domain's
    context ++ the span's own keys, causal] (f32 over the same bf16 plaintext)."""
    if serial:   # the local span in finish on the step stream, not on the side stream after K1
        monkeypatch.setenv("SDA_LOCAL_SERIAL", "1")
    W, LQ = 2, 256
    w = World(W, 1, 4, 4, 128, 512, LQ, torch.bfloat16, seed=400)
    g = torch.Generator(device="cuda").manual_seed(5)
    own = [(torch.randn((1, 4, LQ, 128), generator=g, device="cuda").to(torch.bfloat16),
            torch.randn((1, 4, LQ, 128), generator=g, device="cuda").to(torch.bfloat16)) for _ in range(W)]
    bufs = [sdist.StepBuffers.allocate(W, 1, 4, LQ, 128, torch.bfloat16, "cuda") for _ in range(W)]
    ex = [sdist.PeerExchange(bufs[r], rank=r) for r in range(W)]
    sdist.LocalWorld.connect(ex)
    comps = [sdist.gpu_rank_compute(w.inq[r], w.shards[r], n_splits=1, kv_heads=4, q_first_pos=w.case.q_first_pos,
                                    local_kv=own[r]) for r in range(W)]
    outs = w.outs()
    sdist.LocalWorld.decode_step([w.q(r) for r in range(W)], comps, bufs, outs, ex)
    torch.cuda.synchronize()
    c = w.case
    for r in range(W):
        q = torch.from_numpy(c.q[r]).cuda().float()                                    # [4, LQ, d]
        k = torch.cat([torch.from_numpy(c.k[dom][r]).cuda().float() for dom in range(W)] + [own[r][0][0].float()], 1)
        v = torch.cat([torch.from_numpy(c.v[dom][r]).cuda().float() for dom in range(W)] + [own[r][1][0].float()], 1)
        s = (q @ k.transpose(-1, -2)) / 128 ** 0.5
        ctx = W * 512
        j = torch.arange(ctx + LQ, device="cuda")
        i = torch.arange(LQ, device="cuda")
        s = s.masked_fill((j[None, :] >= ctx) & (j[None, :] - ctx > i[:, None]), float("-inf"))
        ref = (torch.softmax(s, -1) @ v).double().cpu().numpy()
        got = outs[r][0].double().cpu().numpy()
        for h in range(4):
            assert rel_fro(got[h], ref[h]) < 4e-2 and max_abs_rel(got[h], ref[h]) < 6e-2, (r, h)
