"""Benchmark of the scrambled distributed attention hot path (BASELINE.json metric).

Default workload (N=1) = BASELINE config 2: 32 heads x d128, 8K-token scrambled KV per request,
batch-16 decode, BF16 storage / f32 accumulation, on one B200. One step = one scrambled-attention
layer step for the batch: K1 (scramble + permute Q per domain) -> [all-to-all Q'] -> K2 (keyless
split-KV partial attention over the resident scrambled shard) -> [split fold + all-to-all
partials] -> K3 (LSE merge + inverse permutation + unscramble).

Multi-GPU (torchrun, one rank per GPU = one compute domain), weak scaling: every rank is the
inquirer for 16 requests and the compute node of one domain; each request's 8K-token context is
sharded over all N domains (8192/N rows per GPU per request), so per-GPU work is fixed (16N
requests x 8192/N rows) and the job decodes 16N tokens per step. Q' and the (O', stats)
partials move with NCCL all-to-all over NVLink.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

H, D, CTX, B_PER = 32, 128, 8192, 16
HQ, HKV = H, H   # decode line's q / kv heads (config 5: GQA 64 / 8)
CONFIG = 2   # BASELINE config of the decode line: 2 (default) or 4 (--config 4)
METRIC = "scrambled-attn decode tokens/s"


_OUT_FD = 1


def emit(line: dict) -> None:
    os.write(_OUT_FD, (json.dumps(line) + "\n").encode())


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-prefill", action="store_true", help="skip the cfg3 prefill sub-measurement")
    ap.add_argument("--no-gqa", action="store_true", help="skip the cfg5 GQA mixed sub-measurement")
    ap.add_argument("--graph", dest="graph", action="store_true", default=None,
                    help="replay the step (kernels + NCCL all-to-alls) as a CUDA graph (default on)")
    ap.add_argument("--no-graph", dest="graph", action="store_false")
    ap.add_argument("--exchange", choices=["ll", "p2p", "nccl"], default="ll",
                    help="N>1: the exchange carried by K1/K2/K3 themselves in LL format over NVLink peer "
                         "memory (default), separate peer-memory push/wait kernels, or NCCL all-to-all")
    ap.add_argument("--ll-single", action="store_true", help="N=1: run the LL-chained step too (measured no faster)")
    ap.add_argument("--config", type=int, choices=[2, 3, 4, 5], default=2,
                    help="BASELINE config: 2 (default: the decode headline), 3 (prefill across GPUs: a 2K-token span "
                         "per GPU vs a 16K-token shard per domain), 4 (decode, 32K-token shard per GPU, batch 64) or "
                         "5 (GQA decode, 64K-token shard per GPU, batch 32)")
    ap.add_argument("--cpu-pairs", type=int, default=128, help="(request, head) pairs in the CPU sample")
    ap.add_argument("--domains-per-gpu", type=int, default=1,
                    help="decode configs: K compute domains per GPU (N GPUs run N*K domains; e.g. BASELINE configs 4 / 5 "
                         "as written, 8 nodes, on 4 GPUs with K = 2), LL exchange; the line is labelled with both counts")
    return ap.parse_args()


EXCHANGE_DESC = {
    "ll": "Q' and every split's (O', stats) written over NVLink peer memory by K1 / K2 themselves, epoch-tagged (LL)",
    "p2p": "Q' and (O', stats) over NVLink peer memory (exchange.cu push / wait kernels)",
    "nccl": "NCCL all-to-all",
}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def set_config(cfg: int, ws: int) -> None:
    """cfg 2: 16 requests per GPU, each request's 8K context sharded over the N GPUs (weak scaling
    in requests). cfg 4 (BASELINE: 8 nodes x 32K-token shard per node, batch-64 decode): 64
    requests in total, every GPU holds a 32K-token shard of each (weak scaling in context)."""
    global CONFIG, CTX, B_PER, HQ, HKV
    CONFIG = cfg
    if cfg == 4:
        if 64 % ws:
            raise SystemExit("config 4 needs N dividing 64")
        CTX, B_PER = 32768 * ws, 64 // ws
    if cfg == 5:   # GQA decode: 32 requests in total, a 64K-token shard of each per GPU
        if 32 % ws:
            raise SystemExit("config 5 needs N dividing 32")
        CTX, B_PER, HQ, HKV = 65536 * ws, 32 // ws, 64, 8


def workload_config(n):
    desc = {2: "BASELINE cfg2 per GPU: scrambled decode, 32 heads x d128, 8K-token context per request "
               "sharded over N domains (one per GPU), 16 requests per GPU, bf16 KV",
            4: "BASELINE cfg4: scrambled decode, 32 heads x d128, batch 64 (64/N inquirer requests per GPU), "
               "a 32K-token scrambled KV shard of every request on each of the N domains, bf16 KV",
            5: "BASELINE cfg5 (decode part): GQA 64 q / 8 kv heads x d128, batch 32 (32/N inquirer requests per "
               "GPU), a 64K-token scrambled KV shard of every request on each of the N domains, bf16 KV"}[CONFIG]
    return {
        "workload": desc,
        "requests_per_gpu": B_PER, "global_batch": B_PER * n, "q_heads": HQ, "kv_heads": HKV, "head_dim": D,
        "context_per_request": CTX, "kv_rows_per_request_per_gpu": CTX // n, "domains": n,
        "kv_bytes_per_gpu": B_PER * n * HKV * (CTX // n) * D * 2 * 2,
        "l2": f"inputs larger than L2 ({B_PER * n * HKV * (CTX // n) * D * 4 / 2**30:.0f} GiB scrambled KV per GPU vs "
              "126 MB L2), no flush needed",
        "parallelism": f"kv-sharded x{n} (one domain per GPU)",
    }


# ---------------------------------------------------------------------------------------------
# clocks during the timed region
# ---------------------------------------------------------------------------------------------
class ClockSampler:
    """Samples SM clock and clock-event (throttle) reasons through NVML every ~2 ms while the
    timed region runs (nvidia-smi's 100 ms floor is too coarse for a sub-second region)."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.max_mhz = None
        self._stop = threading.Event()
        self.ok = False

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
            self.thread = threading.Thread(target=self._run, daemon=True)
            self.thread.start()
        except Exception:  # noqa: BLE001
            self.ok = False
        return self

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((sm, rs))
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.002)

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.thread.join(timeout=1)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"]}
        sm = [s[0] for s in self.samples]
        reasons = sorted({n for _, r in self.samples for n, bit in self.REASONS.items() if r & bit})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(self.samples), "source": "NVML every ~2 ms during the timed region"}


# ---------------------------------------------------------------------------------------------
# reference arm / CPU baseline: the reference's own C++ (oracle/_ref) on the host cores
# ---------------------------------------------------------------------------------------------
def cpu_reference(n_nodes: int, pairs: int, threads: int, steps: int = 3):
    """Times the reference composition enc Q -> shard_attention -> dec_output -> merge_shards
    (protocol.cpp:885-948) for `pairs` (request, head) pairs of the bench workload (n_nodes shards of
    CTX/n_nodes keys each, scrambled K'/V' built once outside the timing, like the resident cache)
    on `threads` host threads, `steps` times. Returns (per-step tokens/s list, per-step seconds):
    tokens/s = pairs/s / heads (one token needs all heads)."""
    import numpy as np

    from oracle import REF
    if REF is None:
        raise RuntimeError("oracle/_ref/libsdattn_ref.so not built")
    secs = np.zeros(max(steps, 1))
    # a (request, q head) pair costs one shard attention on its kv head's keys (GQA: HQ / HKV q
    # heads share a key set; the reference itself has no GQA)
    REF.lib.ref_bench_decode(pairs, n_nodes, CTX // n_nodes, D, HKV, threads, 2, max(steps, 1),
                             secs.ctypes.data_as(__import__("ctypes").POINTER(__import__("ctypes").c_double)))
    return [(pairs / t) / HQ for t in secs], list(secs)


def single_core_reference(n_nodes: int, pairs: int = 8, steps: int = 3):
    """The reference as shipped is single-threaded: the same composition on ONE
    host thread over a smaller bounded sample (8 (request, head) pairs, 3 steps)."""
    vals, secs = cpu_reference(n_nodes, pairs, 1, steps)
    return {"value": statistics.median(vals), "unit": "tokens/s", "cores": 1,
            "sample": f"{pairs} (request, head) pairs per step x {CTX} keys, median of {steps} steps of "
                      f"{statistics.median(secs):.3f} s on 1 thread"}, secs


def run_reference_arm(args, ws, rank):
    """--impl reference: the reference's own C++ hot path (oracle/_ref) on all host cores. Under
    torchrun only rank 0 runs; the others exit without work."""
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    vals, walls = cpu_reference(ws, args.cpu_pairs, threads, args.warmup + args.steps)
    vals, walls = vals[args.warmup:], walls[args.warmup:]
    value = statistics.median(vals)
    sample = (f"{args.cpu_pairs} (request, head) pairs of the workload per step ({ws} shard(s) x {CTX // ws} keys, "
              f"d{D}, bf16 wire, f64 math), {threads} threads; tokens/s = pairs/s / {HQ} heads")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.median(walls),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference RngStream gaussians)", "config": workload_config(ws),
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": threads, "kind": "reference",
                             "sample": sample, "single_core": single_core_reference(ws)[0]},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line)


# ---------------------------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------------------------
def run_ours(args, ws, rank, local):
    import torch
    import torch.distributed as dist

    from paper_2605_25716_b200 import capi, ops, protocol

    torch.cuda.set_device(local)
    devn = torch.device("cuda", local)
    if args.graph is None:
        args.graph = True
    if ws > 1:
        dist.init_process_group("nccl", device_id=devn)
    B_tot = B_PER * ws
    L = CTX // ws
    my_reqs = list(range(rank * B_PER, (rank + 1) * B_PER))      # requests this rank is inquirer for
    rid = lambda b: b + 1  # noqa: E731

    # --- compute-node state: this rank's domain (rank + 1) shard for all requests -------------
    owner_keys = protocol.DomainKeys([rid(b) for b in range(B_tot)], 0, rank + 1, HKV, D, devn)
    shard = protocol.KVShard(B_tot, HKV, L, D, devn, torch.bfloat16)
    g = torch.Generator(device=devn).manual_seed(1000 + rank)
    chunk = 16 if L <= 8192 else 4
    plain_kv = None
    for b0 in range(0, B_tot, chunk):  # context owners ship their segments (K1 into the cache)
        b1 = min(B_tot, b0 + chunk)
        kp = torch.randn((b1 - b0, HKV, L, D), generator=g, device=devn).to(torch.bfloat16)
        vp = torch.randn((b1 - b0, HKV, L, D), generator=g, device=devn).to(torch.bfloat16)
        if ws == 1 and b0 == 0:   # plaintext of the first requests: the vs-plain parity sample below
            plain_kv = (kp[:4].clone(), vp[:4].clone())
        p, _ = owner_keys.span_perms(1, rank * L, L)
        ops.scramble(kp, owner_keys.dev[b0:b1], capi.PHI_INV_T, capi.KEYS_KQ, p[b0:b1].contiguous(),
                     out=shard.k[b0:b1], key_heads=HKV)
        ops.scramble(vp, owner_keys.dev[b0:b1], capi.PHI_FORWARD, capi.KEYS_V, p[b0:b1].contiguous(),
                     out=shard.v[b0:b1], key_heads=HKV)
        del kp, vp
    shard.rows = L
    shard.kv_len.fill_(L)
    del owner_keys

    # --- inquirer state: keys for my requests on every domain ---------------------------------
    inq_keys = [protocol.DomainKeys([rid(b) for b in my_reqs], 0, dom + 1, HKV, D, devn) for dom in range(ws)]
    q = torch.randn((B_PER, HQ, 1, D), generator=g, device=devn).to(torch.bfloat16)
    S = capi.default_splits(B_tot, HQ, 1, L, kv_heads=HKV, head_dim=D)
    out = torch.empty((B_PER, HQ, 1, D), dtype=torch.float32, device=devn)
    stream = torch.cuda.current_stream()
    k2_ev = []
    record = {"on": False}

    if ws == 1:
        q_s = torch.empty((B_PER, HQ, 1, D), dtype=torch.bfloat16, device=devn)
        o_parts = torch.empty((S, B_tot, HQ, 1, D), dtype=torch.float32, device=devn)
        st_parts = torch.empty((S, B_tot, HQ, 1, 2), dtype=torch.float32, device=devn)
        srcs = ops.sources_from_splits(o_parts, st_parts, inq_keys[0].dev, None)

        def step(qin, o=out):
            # K1 (Q', span_perm over one row is the identity) -> K2 -> K3 (fold splits + unscramble)
            ops.scramble(qin, inq_keys[0].dev, capi.PHI_FORWARD, capi.KEYS_KQ, None, out=q_s, key_heads=HKV)
            if record["on"]:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
            ops.partial_attention(q_s, shard.k, shard.v, shard.kv_len, n_splits=S, out_o=o_parts,
                                  out_stats=st_parts)
            if record["on"]:
                e1.record(stream)
                k2_ev.append((e0, e1))
            return ops.unscramble_merge(srcs, out=o, key_heads=HKV)
        step_k2 = step
        if args.exchange == "ll" and args.ll_single:   # the same kernels LL-chained (W = 1): no faster
            from paper_2605_25716_b200 import distributed as sdist
            lld = sdist.LLDecode(B_PER, HQ, D, inq_keys, shard, n_splits=S, kv_heads=HKV)

            def step(qin, o=out):   # noqa: F811
                return lld.step(qin, o)
    else:
        from paper_2605_25716_b200 import distributed as sdist
        bufs = sdist.StepBuffers.allocate(ws, B_PER, HQ, 1, D, torch.bfloat16, devn)
        comp = sdist.gpu_rank_compute(inq_keys, shard, n_splits=S, kv_heads=HKV)
        serve0 = comp.serve

        def serve_timed(q_all, o_out, st_out):
            if record["on"]:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                serve0(q_all, o_out, st_out)
                e1.record(stream)
                k2_ev.append((e0, e1))
            else:
                serve0(q_all, o_out, st_out)
        comp.serve = serve_timed

        exch = sdist.PeerExchange(bufs) if args.exchange != "nccl" else None

        def step(qin, o=out):
            return sdist.scrambled_decode_step(qin, comp, bufs, o, exchange=exch)
        step_k2 = step
        if args.exchange == "ll":
            lld = sdist.LLDecode(B_PER, HQ, D, inq_keys, shard, n_splits=S, kv_heads=HKV)

            def step(qin, o=out):   # noqa: F811
                return lld.step(qin, o)

    def barrier():
        if ws > 1:
            dist.barrier(device_ids=[local])

    # ---- device-resident timing ----------------------------------------------------------------
    for _ in range(args.warmup):
        step(q)
    torch.cuda.synchronize()
    c0 = capi.launch_count()
    step(q)
    launches_per_step = capi.launch_count() - c0
    run = lambda: step(q)  # noqa: E731
    if args.graph:
        # the whole layer step (kernels + NCCL all-to-alls) captured once and replayed: no host
        # launch gaps between the short kernels around K2
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step(q)
        graph.replay()
        torch.cuda.synchronize()
        run = graph.replay
    barrier()
    torch.cuda.synchronize()
    l0 = capi.launch_count()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        t0.record(stream)
        record["on"] = not args.graph and step is step_k2
        for _ in range(args.steps):
            run()
        record["on"] = False
        t1.record(stream)
        torch.cuda.synchronize()
    barrier()
    launches = (capi.launch_count() - l0) // args.steps if not args.graph else launches_per_step
    ms = t0.elapsed_time(t1) / args.steps
    # K2 duration: the same launch, event-bracketed on the same stream, back to back (LL
    # exchange: the K2 of the reference-shaped step, the same kernel without the LL epilogue)
    if args.graph or step is not step_k2:
        record["on"] = True
        for _ in range(max(10, args.steps // 10)):
            step_k2(q)
        record["on"] = False
        torch.cuda.synchronize()
    k2_ms = statistics.mean(a.elapsed_time(b) for a, b in k2_ev)
    ms_max = ms
    if ws > 1:
        tt = torch.tensor([ms, k2_ms], device=devn)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms_max, k2_ms = float(tt[0]), float(tt[1])

    # ---- end to end through the public API with host buffers -----------------------------------
    # Two forms, both with the step's Q read from pinned host memory and its O landing in pinned
    # host memory inside the timed region: (a) cudaMemcpy H2D -> step -> D2H; (b) zero-copy: the
    # K1 launch reads Q straight from the pinned host buffer over PCIe and the K3 launch stores O
    # straight into the pinned host buffer (UVA), so the transfers ride inside the kernels.
    q_host = q.cpu().pin_memory()
    out_host = torch.empty((B_PER, HQ, 1, D), dtype=torch.float32).pin_memory()
    out_zc = torch.empty((B_PER, HQ, 1, D), dtype=torch.float32).pin_memory()
    q_dev = torch.empty_like(q)

    def e2e_memcpy():
        q_dev.copy_(q_host, non_blocking=True)
        out_host.copy_(step(q_dev), non_blocking=True)

    def e2e_zero_copy():
        step(q_host, out_zc)

    def time_e2e(fn):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        run_fn = fn
        if args.graph:
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr):
                fn()
            gr.replay()
            torch.cuda.synchronize()
            run_fn = gr.replay
        barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            run_fn()
        e1.record(stream)
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / args.steps
        if ws > 1:
            tt = torch.tensor([t], device=devn)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t = float(tt[0])
        return t

    # ---- parity sample printed with the line: the step's output against plain unscrambled
    # attention (f32 over the same bf16 plaintext) on 4 requests x all heads -- the BF16-mode floor
    # of SURVEY 7.4.1 made visible (BASELINE north_star: 2e-2; the test suite's rounding-matched
    # oracle comparisons are the parity gate)
    parity = None
    if plain_kv is not None:
        kf, vf = plain_kv[0].float(), plain_kv[1].float()
        G = HQ // HKV
        qf = q[:4].float()
        kf, vf = kf.repeat_interleave(G, 1), vf.repeat_interleave(G, 1)
        ref = torch.softmax((qf @ kf.transpose(-1, -2)) / D ** 0.5, -1) @ vf
        got = step(q)[:4].float()
        torch.cuda.synchronize()
        diff = (got - ref).flatten(2)
        rel_fro = (diff.norm(dim=-1) / ref.flatten(2).norm(dim=-1)).max().item()
        mar = (diff.abs().amax(-1) / ref.flatten(2).abs().amax(-1)).max().item()
        parity = {"vs_plain_rel_fro_max": rel_fro, "vs_plain_max_abs_rel_max": mar, "pairs": 4 * HQ,
                  "scaling_range": "[1/8, 8] (protocol default)",
                  "note": "bf16-storage floor of Q', K', V' at the default scaling range (SURVEY 7.4.1); "
                          "vs the rounding-matched oracle the tests hold 2e-2 (tests/test_gpu_parity.py)"}
        del plain_kv, kf, vf

    e2e_memcpy_ms = time_e2e(e2e_memcpy)
    e2e_zc_ms = time_e2e(e2e_zero_copy)
    assert torch.isfinite(out_host).all()
    assert torch.equal(out_zc, out_host), "zero-copy O differs from the memcpy O"
    e2e_ms, e2e_form = min((e2e_zc_ms, "zero-copy"), (e2e_memcpy_ms, "memcpy"))

    # ---- roofline of the dominant kernel (K2) ---------------------------------------------------
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        pass
    peak = float(peaks.get("hbm_gbs", 6650.0))
    kv_bytes = B_tot * HKV * L * D * 2 * 2
    k2_bytes = kv_bytes + B_tot * HQ * D * 2 + B_tot * HQ * (4 * D + 8)
    achieved = k2_bytes / (k2_ms * 1e-3) / 1e9
    traffic = None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "k2_decode_traffic.json")))
        if prof.get("config_kv_bytes") == kv_bytes:
            traffic = prof.get("dram_bytes_per_launch")
    except (OSError, ValueError):
        pass

    if rank == 0:
        line = {
            "metric": METRIC, "value": B_tot / (ms_max * 1e-3), "unit": "tokens/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (torch.randn Q/K/V, bf16), keys from the reference key-derivation rule",
            "config": dict(workload_config(ws), exchange=EXCHANGE_DESC[args.exchange] if ws > 1 else "none (single domain)"),
            "e2e": {"value": B_tot / (e2e_ms * 1e-3), "unit": "tokens/s",
                    "h2d_bytes_per_step": B_PER * HQ * D * 2, "d2h_bytes_per_step": B_PER * HQ * D * 4,
                    "transfer": (E2E_FORMS[e2e_form]),
                    "memcpy_value": B_tot / (e2e_memcpy_ms * 1e-3), "zero_copy_value": B_tot / (e2e_zc_ms * 1e-3)},
            "gpu_launches": int(launches) * args.steps, "cuda_graph": bool(args.graph),
            "roofline": {"bound": "hbm", "kernel": ("k2_gqa_tc_kernel<16>" if HKV < HQ else "k2_decode_kernel<128,bf16,bf16>")
                         + ("" if ws == 1 else " + split fold"), "achieved": achieved,
                         "peak": peak, "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                         "algorithmic_bytes_per_launch": k2_bytes, "k2_ms": k2_ms,
                         "k2_share_of_step": k2_ms / ms_max, "peak_source": "MEASURED_PEAKS.json hbm_gbs"
                         if "hbm_gbs" in peaks else "fallback 6.65 TB/s (B200_PROFILING.md)"},
            "clocks": clk.summary(),
        }
        if parity is not None:
            line["parity"] = parity
        if ws == 1 and not args.no_prefill:
            try:
                line["prefill"] = run_prefill(devn, 10, 3, peaks)
            except Exception as e:  # noqa: BLE001
                line["prefill"] = {"unavailable": str(e)}
        if ws == 1 and not args.no_gqa:
            try:
                line["gqa"] = run_gqa_mixed(devn, 10, 3, peaks)
            except Exception as e:  # noqa: BLE001
                line["gqa"] = {"unavailable": str(e)}
        if ws == 1 and not args.no_cpu_baseline:
            try:
                threads = os.cpu_count() or 1
                vals, secs = cpu_reference(1, args.cpu_pairs, threads, 5)
                one, one_s = single_core_reference(1)
                line["cpu_baseline"] = {"value": statistics.median(vals), "unit": "tokens/s", "cores": threads,
                                        "kind": "reference",
                                        "sample": f"{args.cpu_pairs} (request, head) pairs x {CTX} keys x d128 of "
                                                  f"the workload through the reference's own enc->shard_attention->"
                                                  f"dec->merge (oracle/_ref, f64), median of 5 steps of "
                                                  f"{statistics.median(secs):.3f} s wall on {threads} threads",
                                        "single_core": one}
            except Exception as e:  # noqa: BLE001
                line["cpu_baseline"] = {"value": None, "unavailable": str(e)}
        emit(line)
    if ws > 1:
        torch.cuda.synchronize()
        dist.barrier(device_ids=[local])
        # leave without tearing NCCL down (communicator teardown can stall at exit); all work is done
        sys.stdout.flush()
        sys.stderr.flush()
        os._exit(0)


def run_ours_domains(args, ws, rank, local):
    """Decode with K = --domains-per-gpu compute domains per GPU (W = N * K domains): BASELINE
    configs 4 / 5 as written (8 nodes) on fewer GPUs, labelled as such. Every GPU holds the K
    domains' scrambled shards of every request and is the inquirer for K * B_PER requests; a step
    runs, phase by phase, every local domain's LL K1, then K2, then K3 (the exchange carried by the
    kernels over NVLink peer memory to the other GPUs' domains and through local memory to the
    GPU's own). value = all requests decoded per step / step time (max over ranks)."""
    import torch
    import torch.distributed as dist

    from paper_2605_25716_b200 import capi, ops, protocol
    from paper_2605_25716_b200 import distributed as sdist

    K = args.domains_per_gpu
    W = ws * K
    torch.cuda.set_device(local)
    devn = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=devn)
    B_tot = B_PER * W
    L = CTX // W
    rid = lambda b: b + 1  # noqa: E731
    g = torch.Generator(device=devn).manual_seed(2000 + rank)
    doms = [rank * K + i for i in range(K)]
    lls, qs, outs = [], [], []
    S = None
    for dom in doms:
        owner = protocol.DomainKeys([rid(b) for b in range(B_tot)], 0, dom + 1, HKV, D, devn)
        shard = protocol.KVShard(B_tot, HKV, L, D, devn, torch.bfloat16)
        p, _ = owner.span_perms(1, dom * L, L)
        chunk = 16 if L <= 8192 else 4
        for b0 in range(0, B_tot, chunk):
            b1 = min(B_tot, b0 + chunk)
            x = torch.randn((b1 - b0, HKV, L, D), generator=g, device=devn).to(torch.bfloat16)
            ops.scramble(x, owner.dev[b0:b1], capi.PHI_INV_T, capi.KEYS_KQ, p[b0:b1].contiguous(), out=shard.k[b0:b1],
                         key_heads=HKV)
            x = torch.randn((b1 - b0, HKV, L, D), generator=g, device=devn).to(torch.bfloat16)
            ops.scramble(x, owner.dev[b0:b1], capi.PHI_FORWARD, capi.KEYS_V, p[b0:b1].contiguous(), out=shard.v[b0:b1],
                         key_heads=HKV)
            del x
        shard.rows = L
        shard.kv_len.fill_(L)
        del owner
        my = [dom * B_PER + i for i in range(B_PER)]
        inq = [protocol.DomainKeys([rid(b) for b in my], 0, d2 + 1, HKV, D, devn) for d2 in range(W)]
        if S is None:
            S = capi.default_splits(B_tot, HQ, 1, L, kv_heads=HKV, head_dim=D)
        lls.append(sdist.LLDecode(B_PER, HQ, D, inq, shard, n_splits=S, kv_heads=HKV, world=(W, dom)))
        qs.append(torch.randn((B_PER, HQ, 1, D), generator=g, device=devn).to(torch.bfloat16))
        outs.append(torch.empty((B_PER, HQ, 1, D), dtype=torch.float32, device=devn))
    opened = sdist.connect_domains(lls)
    stream = torch.cuda.current_stream()

    def step():
        for i, x in enumerate(lls):
            x.scramble_q(qs[i])
        for x in lls:
            x.serve()
        for i, x in enumerate(lls):
            x.finish(outs[i])

    def barrier():
        if ws > 1:
            dist.barrier(device_ids=[local])

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    c0 = capi.launch_count()
    step()
    launches = capi.launch_count() - c0
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        step()
    barrier()
    graph.replay()
    torch.cuda.synchronize()
    barrier()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        t0.record(stream)
        for _ in range(args.steps):
            graph.replay()
        t1.record(stream)
        torch.cuda.synchronize()
    barrier()
    ms = t0.elapsed_time(t1) / args.steps
    # e2e: every local domain's Q from pinned host memory in, its O back to pinned host memory
    q_host = [q.cpu().pin_memory() for q in qs]
    o_host = [torch.empty(o.shape, dtype=o.dtype).pin_memory() for o in outs]

    def e2e():
        for i in range(K):
            qs[i].copy_(q_host[i], non_blocking=True)
        step()
        for i in range(K):
            o_host[i].copy_(outs[i], non_blocking=True)
    e2e()
    gr2 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr2):
        e2e()
    barrier()
    gr2.replay()
    torch.cuda.synchronize()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        gr2.replay()
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / args.steps
    for x in lls:
        x.check()
    if ws > 1:
        tt = torch.tensor([ms, e2e_ms], device=devn)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms, e2e_ms = float(tt[0]), float(tt[1])
    assert all(torch.isfinite(o).all() for o in o_host)
    if rank == 0:
        peaks = {}
        try:
            peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        except (OSError, ValueError):
            pass
        peak = float(peaks.get("hbm_gbs", 6650.0))
        kv_bytes = K * B_tot * HKV * L * D * 2 * 2   # per GPU: K domains' shards
        cfgd = workload_config(W)
        cfgd.update({"domains": W, "domains_per_gpu": K, "gpus": ws,
                     "kv_bytes_per_gpu": kv_bytes,
                     "label": f"{W} compute domains on {ws} GPU(s), {K} per GPU: every GPU streams {K} domains' "
                              f"shards per step, so per-GPU work is {K}x that of {W} GPUs",
                     "exchange": EXCHANGE_DESC["ll"]})
        emit({"metric": METRIC, "value": B_tot / (ms * 1e-3), "unit": "tokens/s", "n_gpus": ws,
              "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
              "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
              "data": "synthetic (torch.randn Q/K/V, bf16), keys from the reference key-derivation rule",
              "config": cfgd,
              "e2e": {"value": B_tot / (e2e_ms * 1e-3), "unit": "tokens/s",
                      "h2d_bytes_per_step": K * B_PER * HQ * D * 2, "d2h_bytes_per_step": K * B_PER * HQ * D * 4,
                      "transfer": "pinned Q H2D copies -> step -> O D2H copies, every local domain, serial per step"},
              "gpu_launches": int(launches) * args.steps, "cuda_graph": True,
              "roofline": {"bound": "hbm", "kernel": "the step (K domains' K2 dominate)",
                           "achieved": kv_bytes / (ms * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                           "frac": kv_bytes / (ms * 1e-3) / 1e9 / peak, "algorithmic_bytes_per_step": kv_bytes,
                           "note": "KV bytes of the K local shards / step time (an upper bound on K2's share)"},
              "clocks": clk.summary()})
    if ws > 1:
        torch.cuda.synchronize()
        dist.barrier(device_ids=[local])
    del opened   # process exit releases the IPC mappings
    sys.stdout.flush()
    sys.stderr.flush()
    os._exit(0)


E2E_FORMS = {"memcpy": "pinned Q H2D copy -> step -> O D2H copy into pinned memory, serial per step",
             "zero-copy": "K1 reads Q straight from pinned host memory, K3 stores O straight into pinned host "
                          "memory (UVA), serial per step; the memcpy form is reported beside it. At N>1 the PCIe "
                          "traffic overlaps the PDL-chained LL kernels, so this e2e lands within run-to-run noise "
                          "(~2 %) of the device-resident value, timed separately after it"}


def run_prefill_dist(args, ws, rank, local):
    """--config 3 (BASELINE: 4 nodes x 16K-token KV shard, 2K-token prefill with the scramble +
    permutation fused into the KV write) on N GPUs: every rank is the inquirer for one 2K-token
    span and holds a 16K-token scrambled shard of every span's earlier context. One step = the
    span's own K/V scrambled into the local cache + K1 of Q' for every domain (p_q), the Q'
    exchange, tensor-core prefill K2 of every span against this rank's shard, the (O', stats)
    exchange and K3. Reference-shaped exchange (peer-memory push/wait kernels, or NCCL with
    --exchange nccl): the LL form covers decode only. Prints one prefill TFLOP/s line."""
    import torch
    import torch.distributed as dist

    from paper_2605_25716_b200 import capi, ops, protocol
    from paper_2605_25716_b200 import distributed as sdist

    torch.cuda.set_device(local)
    devn = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=devn)
    LQ, LK = 2048, 16384
    rid = lambda b: b + 1  # noqa: E731
    stream = torch.cuda.current_stream()
    # this rank's domain shard of every span's context (+ room for its own span's rows)
    owner = protocol.DomainKeys([rid(b) for b in range(ws)], 0, rank + 1, H, D, devn)
    shard = protocol.KVShard(ws, H, LK + LQ, D, devn, torch.bfloat16)
    g = torch.Generator(device=devn).manual_seed(3000 + rank)
    kp = torch.randn((ws, H, LK, D), generator=g, device=devn).to(torch.bfloat16)
    vp = torch.randn((ws, H, LK, D), generator=g, device=devn).to(torch.bfloat16)
    shard.ship_segment(kp, vp, owner, first_pos=rank * LK)
    del kp, vp
    inq = [protocol.DomainKeys([rid(rank)], 0, dom + 1, H, D, devn) for dom in range(ws)]
    q_first = ws * LK
    q = torch.randn((1, H, LQ, D), generator=g, device=devn).to(torch.bfloat16)
    kn = torch.randn((1, H, LQ, D), generator=g, device=devn).to(torch.bfloat16)
    vn = torch.randn((1, H, LQ, D), generator=g, device=devn).to(torch.bfloat16)
    own_shard = protocol.KVShard(1, H, LQ, D, devn, torch.bfloat16)   # the span's own K/V (local cache)
    pkv, _ = inq[rank].span_perms(1, q_first, LQ)
    k1_jobs = [ops.scramble_job(kn, inq[rank].dev, capi.PHI_INV_T, capi.KEYS_KQ, pkv, out=own_shard.k, key_heads=H),
               ops.scramble_job(vn, inq[rank].dev, capi.PHI_FORWARD, capi.KEYS_V, pkv, out=own_shard.v, key_heads=H)]
    S = capi.default_splits(ws, H, LQ, LK)
    # the span also attends its own K/V in plaintext with the causal mask (protocol.cpp:944-947)
    # the span's own K/V into the local cache is off the step's path: it runs on the side stream
    # with the causal span, after this step's Q' scramble
    comp = sdist.gpu_rank_compute(inq, shard, n_splits=S, kv_heads=H, q_first_pos=q_first, local_kv=(kn, vn),
                                  side_work=lambda: ops.scramble_batch(k1_jobs, D))
    bufs = sdist.StepBuffers.allocate(ws, 1, H, LQ, D, torch.bfloat16, devn)
    exch = sdist.PeerExchange(bufs) if ws > 1 and args.exchange != "nccl" else None
    out = torch.empty((1, H, LQ, D), dtype=torch.float32, device=devn)
    # the step runs on a high-priority stream: the span's causal local attention goes to a
    # lowest-priority side stream after K1 (distributed.gpu_rank_compute), behind K2's CTAs
    torch.cuda.synchronize()
    stream = torch.cuda.Stream(device=devn, priority=-1)
    torch.cuda.set_stream(stream)

    def step(qin, o=out):
        # the span's K/V into the cache (scramble + permute fused) runs inside as comp's side work
        return sdist.scrambled_decode_step(qin, comp, bufs, o, exchange=exch)

    def barrier():
        if ws > 1:
            dist.barrier(device_ids=[local])

    for _ in range(args.warmup):
        step(q)
    torch.cuda.synchronize()
    c0 = capi.launch_count()
    step(q)
    launches = capi.launch_count() - c0
    barrier()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        t0.record(stream)
        for _ in range(args.steps):
            step(q)
        comp.drain()   # the last step's side work (the span's K/V into the cache) inside the region
        t1.record(stream)
        torch.cuda.synchronize()
    barrier()
    ms = t0.elapsed_time(t1) / args.steps
    # end to end: every step's Q span from pinned host memory in, its O back out, over a stream of
    # successive spans (independent prefill chunks/requests). Two slots: span i+1's H2D (copy-in
    # stream) and span i-1's D2H (copy-out stream) run under span i's kernels; PCIe is full duplex.
    q_host = q.cpu().pin_memory()
    q_dev = [torch.empty_like(q), torch.empty_like(q)]
    o_dev = [out, torch.empty_like(out)]
    out_host = [torch.empty((1, H, LQ, D)).pin_memory() for _ in range(2)]
    c_in, c_out = torch.cuda.Stream(devn), torch.cuda.Stream(devn)
    ev = lambda: torch.cuda.Event()  # noqa: E731
    used, loaded, done, drained = [ev(), ev()], [ev(), ev()], [ev(), ev()], [ev(), ev()]
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    c_in.wait_event(e0)
    c_out.wait_event(e0)
    for i in range(args.steps):
        s = i & 1
        with torch.cuda.stream(c_in):
            if i >= 2:
                c_in.wait_event(used[s])          # span i-2 is done reading q_dev[s]
            q_dev[s].copy_(q_host, non_blocking=True)
            loaded[s].record(c_in)
        stream.wait_event(loaded[s])
        if i >= 2:
            stream.wait_event(drained[s])         # span i-2's O has left o_dev[s]
        step(q_dev[s], o_dev[s])
        used[s].record(stream)
        with torch.cuda.stream(c_out):
            c_out.wait_event(used[s])
            out_host[s].copy_(o_dev[s], non_blocking=True)
            drained[s].record(c_out)
    stream.wait_stream(c_out)
    comp.drain()
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / args.steps
    ref_o = out_host[(args.steps - 1) & 1]
    assert torch.equal(ref_o, o_dev[(args.steps - 1) & 1].cpu()), "e2e: host copy of O differs from the device O"
    if ws > 1:
        tt = torch.tensor([ms, e2e_ms], device=devn)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms, e2e_ms = float(tt[0]), float(tt[1])
    # every span against every domain's shard, + every span's causal local attention
    flops = 4.0 * LQ * LK * H * D * ws * ws + 2.0 * LQ * (LQ + 1) * H * D * ws
    if rank == 0:
        peaks = {}
        try:
            peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        except (OSError, ValueError):
            pass
        peak = float(peaks.get("bf16_tflops", 1590.0)) * ws
        value = flops / (ms * 1e-3) / 1e12
        emit({"metric": "scrambled-attn prefill TFLOP/s", "value": value, "unit": "TFLOP/s", "n_gpus": ws,
              "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
              "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
              "data": "synthetic (torch.randn Q/K/V, bf16), keys from the reference key-derivation rule",
              "config": {"workload": "BASELINE cfg3: one 2K-token prefill span per GPU against a 16K-token scrambled "
                                     "KV shard of every span on each of the N domains (+ the span's own K/V scrambled "
                                     "into the cache, + the span attending its own K/V in plaintext with the causal "
                                     "mask, merged in K3), 32 heads x d128, bf16",
                         "q_rows": LQ, "kv_rows_per_domain": LK, "domains": ws, "splits": S,
                         "exchange": ("none (single domain)" if ws == 1 else EXCHANGE_DESC[args.exchange if args.exchange != "ll" else "p2p"]),
                         "l2": "inputs larger than L2, no flush needed"},
              "e2e": {"value": flops / (e2e_ms * 1e-3) / 1e12, "unit": "TFLOP/s",
                      "h2d_bytes_per_step": LQ * H * D * 2, "d2h_bytes_per_step": LQ * H * D * 4,
                      "overlap": "successive spans double-buffered: span i+1's Q H2D and span i-1's O D2H "
                                 "on two copy streams under span i's kernels"},
              "gpu_launches": int(launches) * args.steps, "cuda_graph": False,
              "roofline": {"bound": "tensor", "kernel": "k2_prefill_tc_kernel (whole step)", "achieved": value,
                           "peak": peak, "unit": "TFLOP/s", "frac": value / peak,
                           "peak_source": "MEASURED_PEAKS.json bf16_tflops (burst) x N"},
              "clocks": clk.summary()})
    if ws > 1:
        torch.cuda.synchronize()
        dist.barrier(device_ids=[local])
        sys.stdout.flush()
        sys.stderr.flush()
        os._exit(0)


def run_prefill(devn, steps: int, warmup: int, peaks: dict):
    """BASELINE config 3 per GPU: a 2048-token prefill span against a 16K-token scrambled shard,
    32 heads x d128, bf16. One step = the span's own K/V scrambled + permuted into the cache
    (K1, fused into the KV write), its Q scrambled (K1), tcgen05 partial attention over the
    shard (K2) and the LSE merge + unscramble (K3). Returns the JSON object for the line."""
    import torch

    from paper_2605_25716_b200 import capi, ops, protocol

    LQ, LK = 2048, 16384
    keys = protocol.DomainKeys([1], 0, 1, H, D, devn)
    shard = protocol.KVShard(1, H, LK + LQ, D, devn, torch.bfloat16)
    g = torch.Generator(device=devn).manual_seed(7)
    kp = torch.randn((1, H, LK, D), generator=g, device=devn).to(torch.bfloat16)
    vp = torch.randn((1, H, LK, D), generator=g, device=devn).to(torch.bfloat16)
    shard.ship_segment(kp, vp, keys, first_pos=0)
    q = torch.randn((1, H, LQ, D), generator=g, device=devn).to(torch.bfloat16)
    kn = torch.randn((1, H, LQ, D), generator=g, device=devn).to(torch.bfloat16)
    vn = torch.randn((1, H, LQ, D), generator=g, device=devn).to(torch.bfloat16)
    pq, pq_inv = keys.span_perms(0, LK, LQ)
    pkv, _ = keys.span_perms(1, LK, LQ)
    S = capi.default_splits(1, H, LQ, LK)
    kv16k = torch.full((1,), LK, dtype=torch.int32, device=devn)   # the delegated shard (earlier context)
    qs = torch.empty_like(q)
    o = torch.empty((S, 1, H, LQ, D), dtype=torch.float32, device=devn)
    st = torch.empty((S, 1, H, LQ, 2), dtype=torch.float32, device=devn)
    out = torch.empty((1, H, LQ, D), dtype=torch.float32, device=devn)
    # the inquirer's own span attended in plaintext with the causal mask (protocol.cpp:944-947),
    # tensor-core K2 with per-row key limits, merged by K3 as a plaintext source
    lo = torch.empty((1, 1, H, LQ, D), dtype=torch.float32, device=devn)
    ls = torch.empty((1, 1, H, LQ, 2), dtype=torch.float32, device=devn)
    srcs = ops.sources_from_splits(o, st, keys.dev, pq_inv) + ops.sources_from_splits(lo, ls)
    torch.cuda.synchronize()   # the setup ran on the default stream
    stream = torch.cuda.Stream(device=devn, priority=-1)   # the step's stream (high priority, see below)
    ev = []
    k1_jobs = [ops.scramble_job(kn, keys.dev, capi.PHI_INV_T, capi.KEYS_KQ, pkv, out=shard.k, out_row_offset=LK, key_heads=H),
               ops.scramble_job(vn, keys.dev, capi.PHI_FORWARD, capi.KEYS_V, pkv, out=shard.v, out_row_offset=LK, key_heads=H),
               ops.scramble_job(q, keys.dev, capi.PHI_FORWARD, capi.KEYS_KQ, pq, out=qs, key_heads=H)]

    # the span's causal local attention is independent of K1's Q' and of the remote K2: it runs on a
    # second, lower-priority stream once K1 is done, so its CTAs take the SMs the stream-K K2 frees
    # in its tail instead of starting after it (SDA_BENCH_C3_SERIAL=1: one stream, as before)
    serial = bool(os.environ.get("SDA_BENCH_C3_SERIAL"))
    side = torch.cuda.Stream(device=devn, priority=0)
    k1_done = torch.cuda.Event()
    local_done = torch.cuda.Event()

    def step(rec):
        # the span's K/V go into the cache rows after the shard (scramble + permute fused into the write)
        # ... and the span's Q into Q' (p_q). Serial: all three K1 jobs in one launch. Otherwise only
        # Q' is on the path to K2; the K/V jobs (written past the 16K rows K2 reads) go to the side
        # stream with the causal span
        if serial:
            ops.scramble_batch(k1_jobs, D)
        else:
            ops.scramble_batch(k1_jobs[2:], D)
            k1_done.record(stream)
        if rec:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
        # delegated shards are strictly earlier context: attend the resident 16K rows (mask none)
        ops.partial_attention(qs, shard.k, shard.v, kv16k, n_splits=S, out_o=o, out_stats=st)
        if rec:
            e1.record(stream)
            ev.append((e0, e1))
        if serial:
            ops.partial_attention_causal(q, kn, vn, causal_offset=0, n_splits=1, out_o=lo, out_stats=ls)
            if rec:
                e2 = torch.cuda.Event(enable_timing=True)
                e2.record(stream)
                ev_local.append((e1, e2))
        else:
            side.wait_event(k1_done)   # (also orders it after the previous step's K3, which read lo / ls)
            with torch.cuda.stream(side):
                side_first = os.environ.get("SDA_SIDE_FIRST") == "1"
                if side_first:
                    ops.scramble_batch(k1_jobs[:2], D)
                if rec:
                    s0 = torch.cuda.Event(enable_timing=True)
                    s0.record(side)
                ops.partial_attention_causal(q, kn, vn, causal_offset=0, n_splits=1, out_o=lo, out_stats=ls)
                if rec:
                    s1 = torch.cuda.Event(enable_timing=True)
                    s1.record(side)
                    ev_local.append((s0, s1))
                local_done.record(side)
                # the span's K/V rows (past the 16K K2 reads; nothing in the step reads them) behind
                # the join: K3 does not wait for them, they fill the SMs K3 and the next K1 leave
                # idle; the timed region ends after the side stream drains (below)
                if not side_first:
                    ops.scramble_batch(k1_jobs[:2], D)
            stream.wait_event(local_done)
        ops.unscramble_merge(srcs, out=out, key_heads=H)

    ev_local = []
    with torch.cuda.stream(stream):
        for _ in range(warmup):
            step(False)
        torch.cuda.synchronize()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(devn.index or 0) as clk:
            t0.record(stream)
            for _ in range(steps):
                step(True)
            stream.wait_stream(side)   # the last step's side work inside the timed region
            t1.record(stream)
            torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / steps
    k2_ms = statistics.mean(a.elapsed_time(b) for a, b in ev)
    local_ms = statistics.mean(a.elapsed_time(b) for a, b in ev_local)
    flops_remote = 4.0 * LQ * LK * H * D
    flops_local = 2.0 * LQ * (LQ + 1) * H * D   # causal: row i attends i + 1 keys
    flops = flops_remote + flops_local
    peak = float(peaks.get("bf16_tflops", 1590.0))
    tf_k2 = flops_remote / (k2_ms * 1e-3) / 1e12
    return {"metric": "scrambled-attn prefill TFLOP/s", "value": flops / (ms * 1e-3) / 1e12, "unit": "TFLOP/s",
            "ms_per_step": ms, "steps": steps, "warmup": warmup,
            "config": {"workload": "BASELINE cfg3 per GPU: 2K-token prefill span vs 16K-token scrambled KV shard "
                                   "(+ the span's own 2K K/V rows scrambled into the cache, + the span attending its "
                                   "own K/V in plaintext with the causal mask, merged in K3), 32 heads x d128, bf16",
                       "q_rows": LQ, "kv_rows": LK, "kv_rows_written": LQ, "heads": H, "head_dim": D, "splits": S},
            "flops_per_step": flops, "flops_remote": flops_remote, "flops_local_causal": flops_local,
            "local_causal_ms": local_ms,
            "local_causal_tflops": flops_local / (local_ms * 1e-3) / 1e12, "clocks": clk.summary(),
            "roofline": {"bound": "tensor", "kernel": "k2_prefill_tc_kernel", "achieved": tf_k2, "peak": peak,
                         "unit": "TFLOP/s", "frac": tf_k2 / peak, "k2_ms": k2_ms, "k2_share_of_step": k2_ms / ms,
                         "peak_source": "MEASURED_PEAKS.json bf16_tflops (burst)",
                         "frac_of_sustained": tf_k2 / float(peaks.get("bf16_tflops_sustained", peak)),
                         "frac_of_mma_issue_rate": tf_k2 / (8192 * 148 * 1.965e9 / 1e12)}}


def run_gqa_mixed(devn, steps: int, warmup: int, peaks: dict):
    """BASELINE config 5 per GPU: GQA 64 q heads / 8 kv heads x d128, 64K-token scrambled KV shard
    per request. Mixed step = 32 decode requests (one token each) + one 2K-token prefill chunk of
    another request (its K/V scrambled into its cache, its Q against its 64K shard). Reports
    decode-only and mixed timings; roofline of the swapped GQA decode kernel vs HBM."""
    import torch

    from paper_2605_25716_b200 import capi, ops, protocol

    HQ, HKV, L, BD, LP = 64, 8, 65536, 32, 2048
    keys = protocol.DomainKeys(list(range(1, BD + 2)), 0, 1, HKV, D, devn)
    k = torch.empty((BD + 1, HKV, L + LP, D), dtype=torch.bfloat16, device=devn)
    v = torch.empty_like(k)
    g = torch.Generator(device=devn).manual_seed(11)
    for b0 in range(0, BD + 1, 4):   # resident shards, scrambled + permuted by K1 (setup, untimed)
        b1 = min(BD + 1, b0 + 4)
        x = torch.randn((b1 - b0, HKV, L, D), generator=g, device=devn).to(torch.bfloat16)
        pkv, _ = keys.span_perms(1, 0, L)
        ops.scramble(x, keys.dev[b0:b1], capi.PHI_INV_T, capi.KEYS_KQ, pkv[b0:b1].contiguous(), out=k[b0:b1], key_heads=HKV)
        ops.scramble(x, keys.dev[b0:b1], capi.PHI_FORWARD, capi.KEYS_V, pkv[b0:b1].contiguous(), out=v[b0:b1], key_heads=HKV)
        del x
    kv_len = torch.full((BD + 1,), L, dtype=torch.int32, device=devn)
    kd, vd, ld = k[:BD], v[:BD], kv_len[:BD]
    kp, vp, lp = k[BD:], v[BD:], kv_len[BD:]
    keys_d, keys_p = keys.dev[:BD], keys.dev[BD:]
    qd = torch.randn((BD, HQ, 1, D), generator=g, device=devn).to(torch.bfloat16)
    qp = torch.randn((1, HQ, LP, D), generator=g, device=devn).to(torch.bfloat16)
    knew = torch.randn((1, HKV, LP, D), generator=g, device=devn).to(torch.bfloat16)
    vnew = torch.randn((1, HKV, LP, D), generator=g, device=devn).to(torch.bfloat16)
    pq, pq_inv = keys.span_perms(0, L, LP)
    pkv_new, _ = keys.span_perms(1, L, LP)
    Sd = capi.default_splits(BD, HQ, 1, L, kv_heads=HKV, head_dim=D)
    Sp = capi.default_splits(1, HQ, LP, L, kv_heads=HKV, head_dim=D)
    qd_s, qp_s = torch.empty_like(qd), torch.empty_like(qp)
    od = torch.empty((Sd, BD, HQ, 1, D), dtype=torch.float32, device=devn)
    sd = torch.empty((Sd, BD, HQ, 1, 2), dtype=torch.float32, device=devn)
    op_ = torch.empty((Sp, 1, HQ, LP, D), dtype=torch.float32, device=devn)
    sp_ = torch.empty((Sp, 1, HQ, LP, 2), dtype=torch.float32, device=devn)
    outd = torch.empty((BD, HQ, 1, D), dtype=torch.float32, device=devn)
    outp = torch.empty((1, HQ, LP, D), dtype=torch.float32, device=devn)
    srcd = ops.sources_from_splits(od, sd, keys_d, None)
    lo = torch.empty((1, 1, HQ, LP, D), dtype=torch.float32, device=devn)   # the chunk's own span, causal
    ls = torch.empty((1, 1, HQ, LP, 2), dtype=torch.float32, device=devn)
    srcp = ops.sources_from_splits(op_, sp_, keys_p, pq_inv[BD:].contiguous()) + ops.sources_from_splits(lo, ls)
    pq_p = pq[BD:].contiguous()
    stream = torch.cuda.current_stream()
    ev = []

    def decode(rec):
        ops.scramble(qd, keys_d, capi.PHI_FORWARD, capi.KEYS_KQ, None, out=qd_s, key_heads=HKV)
        if rec:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
        ops.partial_attention(qd_s, kd, vd, ld, n_splits=Sd, out_o=od, out_stats=sd)
        if rec:
            e1.record(stream)
            ev.append((e0, e1))
        ops.unscramble_merge(srcd, out=outd, key_heads=HKV)

    pkv_p = pkv_new[BD:].contiguous()
    k1_jobs = [ops.scramble_job(knew, keys_p, capi.PHI_INV_T, capi.KEYS_KQ, pkv_p, out=kp, out_row_offset=L, key_heads=HKV),
               ops.scramble_job(vnew, keys_p, capi.PHI_FORWARD, capi.KEYS_V, pkv_p, out=vp, out_row_offset=L, key_heads=HKV),
               ops.scramble_job(qp, keys_p, capi.PHI_FORWARD, capi.KEYS_KQ, pq_p, out=qp_s, key_heads=HKV)]

    def prefill():
        ops.scramble_batch(k1_jobs, D)   # the chunk's K, V into the cache and its Q, one K1 launch
        ops.partial_attention(qp_s, kp, vp, lp, n_splits=Sp, out_o=op_, out_stats=sp_)
        ops.partial_attention_causal(qp, knew, vnew, causal_offset=0, n_splits=1, out_o=lo, out_stats=ls)
        ops.unscramble_merge(srcp, out=outp, key_heads=HKV)

    def timed(fn, n):
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for _ in range(n):
            fn()
        t1.record(stream)
        torch.cuda.synchronize()
        return t0.elapsed_time(t1) / n

    for _ in range(warmup):
        decode(False)
        prefill()
    torch.cuda.synchronize()
    ms_dec = timed(lambda: decode(True), steps)
    k2_ms = statistics.mean(a.elapsed_time(b) for a, b in ev)
    ms_mix = timed(lambda: (decode(False), prefill()), steps)
    kv_bytes = BD * HKV * L * D * 2 * 2
    k2_bytes = kv_bytes + BD * HQ * D * 2 + BD * HQ * (4 * D + 8)
    achieved = k2_bytes / (k2_ms * 1e-3) / 1e9
    peak = float(peaks.get("hbm_gbs", 6650.0))
    pf_flops = 4.0 * LP * L * HQ * D + 2.0 * LP * (LP + 1) * HQ * D   # + the chunk's causal local span
    return {"metric": "scrambled-attn GQA decode tokens/s (mixed step also reported)",
            "value": BD / (ms_dec * 1e-3), "unit": "tokens/s", "ms_per_step_decode": ms_dec,
            "ms_per_step_mixed": ms_mix, "mixed_tokens_per_s": (BD + LP) / (ms_mix * 1e-3),
            "mixed_prefill_tflops_incl_decode": pf_flops / ((ms_mix) * 1e-3) / 1e12, "steps": steps,
            "config": {"workload": "BASELINE cfg5 per GPU: GQA 64 q / 8 kv heads x d128, 64K-token scrambled KV "
                                   "shard per request; mixed step = 32 decode requests + one 2K-token prefill chunk "
                                   "(against its 64K shard, and its own 2K K/V in plaintext with the causal mask)",
                       "decode_requests": BD, "prefill_chunk": LP, "kv_rows": L, "splits_decode": Sd,
                       "splits_prefill": Sp},
            "roofline": {"bound": "hbm", "kernel": "k2_gqa_tc_kernel<16>", "achieved": achieved, "peak": peak,
                         "unit": "GB/s", "frac": achieved / peak, "k2_ms": k2_ms,
                         "algorithmic_bytes_per_launch": k2_bytes}}


def main():
    args = parse()
    ws, rank, local = dist_env()
    # Libraries (NCCL prints its version banner) may write to fd 1; keep stdout for the single
    # JSON line and send everything else to stderr.
    global _OUT_FD
    _OUT_FD = os.dup(1)
    os.dup2(2, 1)
    if args.gpus != ws and ws > 1:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE {ws}", file=sys.stderr)
    set_config(args.config, ws * max(1, args.domains_per_gpu))
    if args.impl == "reference" and args.config == 3:
        if rank == 0:
            emit({"impl": "reference", "unavailable": "config 3 (multi-GPU prefill) has no reference arm here: the "
                                                      "reference's f64 prefill takes minutes per step; see the N=1 "
                                                      "prefill line of the default run"})
        return
    if args.impl == "reference":
        run_reference_arm(args, ws, rank)
    elif args.config == 3:
        run_prefill_dist(args, ws, rank, local)
    elif args.domains_per_gpu > 1:
        run_ours_domains(args, ws, rank, local)
    else:
        run_ours(args, ws, rank, local)


if __name__ == "__main__":
    main()
