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
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

H, D, CTX, B_PER = 32, 128, 8192, 16
METRIC = "scrambled-attn decode tokens/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-pairs", type=int, default=64, help="(request, head) pairs in the CPU sample")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def workload_config(n):
    return {
        "workload": "BASELINE cfg2 per GPU: scrambled decode, 32 heads x d128, 8K-token context per request "
                    "sharded over N domains (one per GPU), 16 requests per GPU, bf16 KV",
        "requests_per_gpu": B_PER, "global_batch": B_PER * n, "q_heads": H, "kv_heads": H, "head_dim": D,
        "context_per_request": CTX, "kv_rows_per_request_per_gpu": CTX // n, "domains": n,
        "kv_bytes_per_gpu": B_PER * n * H * (CTX // n) * D * 2 * 2,
        "l2": "inputs larger than L2 (2 GiB scrambled KV per GPU vs 126 MB L2), no flush needed",
        "parallelism": f"kv-sharded x{n} (one domain per GPU), NCCL all-to-all of Q' and partials",
    }


# ---------------------------------------------------------------------------------------------
# clocks during the timed region
# ---------------------------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.samples.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ---------------------------------------------------------------------------------------------
# reference arm / CPU baseline: the reference's own C++ (oracle/_ref) on the host cores
# ---------------------------------------------------------------------------------------------
def cpu_reference(n_nodes: int, pairs: int, threads: int):
    """Times the reference composition enc Q -> shard_attention -> dec_output -> merge_shards
    (protocol.cpp:885-948) for `pairs` (request, head) pairs of the bench workload, n_nodes shards
    of CTX/n_nodes keys each, on `threads` host threads. Returns tokens/s (= pairs/s / heads)."""
    from oracle import REF
    if REF is None:
        raise RuntimeError("oracle/_ref/libsdattn_ref.so not built")
    t = REF.lib.ref_bench_decode(pairs, n_nodes, CTX // n_nodes, D, H, threads, 2)
    return (pairs / t) / H, t


def run_reference_arm(args, ws, rank):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    vals, walls = [], []
    for _ in range(args.warmup):
        cpu_reference(ws, args.cpu_pairs, threads)
    for _ in range(args.steps):
        v, w = cpu_reference(ws, args.cpu_pairs, threads)
        vals.append(v)
        walls.append(w)
    value = statistics.median(vals)
    sample = (f"{args.cpu_pairs} (request, head) pairs of the workload per step "
              f"({ws} shard(s) x {CTX // ws} keys, d{D}, bf16 wire), {threads} threads; tokens/s = pairs/s / {H}")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.median(walls),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference RngStream gaussians)", "config": workload_config(ws),
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": threads, "kind": "reference",
                             "sample": sample},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------------------------
def run_ours(args, ws, rank, local):
    import torch
    import torch.distributed as dist

    from paper_2605_25716_b200 import capi, ops, protocol

    torch.cuda.set_device(local)
    devn = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=devn)
    B_tot = B_PER * ws
    L = CTX // ws
    my_reqs = list(range(rank * B_PER, (rank + 1) * B_PER))      # requests this rank is inquirer for
    rid = lambda b: b + 1  # noqa: E731

    # --- compute-node state: this rank's domain (rank + 1) shard for all requests -------------
    owner_keys = protocol.DomainKeys([rid(b) for b in range(B_tot)], 0, rank + 1, H, D, devn)
    shard = protocol.KVShard(B_tot, H, L, D, devn, torch.bfloat16)
    g = torch.Generator(device=devn).manual_seed(1000 + rank)
    for b0 in range(0, B_tot, 16):  # context owners ship their segments (K1 into the cache)
        b1 = min(B_tot, b0 + 16)
        kp = torch.randn((b1 - b0, H, L, D), generator=g, device=devn).to(torch.bfloat16)
        vp = torch.randn((b1 - b0, H, L, D), generator=g, device=devn).to(torch.bfloat16)
        p, _ = owner_keys.span_perms(1, rank * L, L)
        ops.scramble(kp, owner_keys.dev[b0:b1], capi.PHI_INV_T, capi.KEYS_KQ, p[b0:b1].contiguous(),
                     out=shard.k[b0:b1], key_heads=H)
        ops.scramble(vp, owner_keys.dev[b0:b1], capi.PHI_FORWARD, capi.KEYS_V, p[b0:b1].contiguous(),
                     out=shard.v[b0:b1], key_heads=H)
        del kp, vp
    shard.rows = L
    shard.kv_len.fill_(L)
    del owner_keys

    # --- inquirer state: keys for my requests on every domain ---------------------------------
    inq_keys = [protocol.DomainKeys([rid(b) for b in my_reqs], 0, dom + 1, H, D, devn) for dom in range(ws)]
    q = torch.randn((B_PER, H, 1, D), generator=g, device=devn).to(torch.bfloat16)
    S = capi.default_splits(B_tot, H, 1, L)
    qs_send = torch.empty((ws, B_PER, H, 1, D), dtype=torch.bfloat16, device=devn)
    qs_recv = torch.empty_like(qs_send)
    o_parts = torch.empty((S, B_tot, H, 1, D), dtype=torch.float32, device=devn)
    st_parts = torch.empty((S, B_tot, H, 1, 2), dtype=torch.float32, device=devn)
    o_fold = torch.empty((ws, B_PER, H, 1, D), dtype=torch.float32, device=devn)
    st_fold = torch.empty((ws, B_PER, H, 1, 2), dtype=torch.float32, device=devn)
    o_back = torch.empty_like(o_fold)
    st_back = torch.empty_like(st_fold)
    out = torch.empty((B_PER, H, 1, D), dtype=torch.float32, device=devn)
    stream = torch.cuda.current_stream()
    k2_ev = []

    def step(qin, record=False):
        # K1: Q' per destination domain (span_perm over one row is the identity)
        for dom in range(ws):
            ops.scramble(qin, inq_keys[dom].dev, capi.PHI_FORWARD, capi.KEYS_KQ, None, out=qs_send[dom],
                         key_heads=H)
        if ws > 1:
            dist.all_to_all_single(qs_recv, qs_send)
            q_all = qs_recv.view(B_tot, H, 1, D)
        else:
            q_all = qs_send.view(B_tot, H, 1, D)
        if record:
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
        ops.partial_attention(q_all, shard.k, shard.v, shard.kv_len, n_splits=S, out_o=o_parts, out_stats=st_parts)
        if record:
            e1.record(stream)
            k2_ev.append((e0, e1))
        if ws == 1:
            srcs = ops.sources_from_splits(o_parts, st_parts, inq_keys[0].dev, None)
            return ops.unscramble_merge(srcs, out=out, key_heads=H)
        # fold this domain's splits in scrambled space (plain merge, no keys), then return partials
        ops.unscramble_merge(ops.sources_from_splits(o_parts, st_parts), out=o_fold.view(B_tot, H, 1, D),
                             out_stats=st_fold.view(B_tot, H, 1, 2))
        dist.all_to_all_single(o_back, o_fold)
        dist.all_to_all_single(st_back, st_fold)
        srcs = [ops.MergeSource(o_back[dom], st_back[dom], inq_keys[dom].dev, None) for dom in range(ws)]
        return ops.unscramble_merge(srcs, out=out, key_heads=H)

    def barrier():
        if ws > 1:
            dist.barrier(device_ids=[local])

    # ---- device-resident timing ----------------------------------------------------------------
    for _ in range(args.warmup):
        step(q)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    l0 = capi.launch_count()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        t0.record(stream)
        for _ in range(args.steps):
            step(q, record=True)
        t1.record(stream)
        torch.cuda.synchronize()
    barrier()
    launches = (capi.launch_count() - l0) // args.steps
    ms = t0.elapsed_time(t1) / args.steps
    k2_ms = statistics.mean(a.elapsed_time(b) for a, b in k2_ev)
    ms_max = ms
    if ws > 1:
        tt = torch.tensor([ms, k2_ms], device=devn)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms_max, k2_ms = float(tt[0]), float(tt[1])

    # ---- end to end through the public API with host buffers -----------------------------------
    q_host = q.cpu().pin_memory()
    out_host = torch.empty((B_PER, H, 1, D), dtype=torch.float32).pin_memory()
    for _ in range(2):
        out_host.copy_(step(q_host.to(devn, non_blocking=True)), non_blocking=True)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        out_host.copy_(step(q_host.to(devn, non_blocking=True)), non_blocking=True)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / args.steps
    if ws > 1:
        tt = torch.tensor([e2e_ms], device=devn)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms = float(tt[0])
    assert torch.isfinite(out_host).all()

    # ---- roofline of the dominant kernel (K2) ---------------------------------------------------
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        pass
    peak = float(peaks.get("hbm_gbs", 6650.0))
    kv_bytes = B_tot * H * L * D * 2 * 2
    k2_bytes = kv_bytes + B_tot * H * D * 2 + B_tot * H * (4 * D + 8)
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
            "config": workload_config(ws),
            "e2e": {"value": B_tot / (e2e_ms * 1e-3), "unit": "tokens/s",
                    "h2d_bytes_per_step": B_PER * H * D * 2, "d2h_bytes_per_step": B_PER * H * D * 4},
            "gpu_launches": int(launches) * args.steps,
            "roofline": {"bound": "hbm", "kernel": "k2_decode_kernel<128,bf16,bf16>", "achieved": achieved,
                         "peak": peak, "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                         "algorithmic_bytes_per_launch": k2_bytes, "k2_ms": k2_ms,
                         "k2_share_of_step": k2_ms / ms_max, "peak_source": "MEASURED_PEAKS.json hbm_gbs"
                         if "hbm_gbs" in peaks else "fallback 6.65 TB/s (B200_PROFILING.md)"},
            "clocks": clk.summary(),
        }
        if ws == 1 and not args.no_cpu_baseline:
            try:
                threads = os.cpu_count() or 1
                v, t = cpu_reference(1, args.cpu_pairs, threads)
                line["cpu_baseline"] = {"value": v, "unit": "tokens/s", "cores": threads, "kind": "reference",
                                        "sample": f"{args.cpu_pairs} (request, head) pairs x 8192 keys x d128 of "
                                                  f"the workload through the reference's own enc->shard_attention->"
                                                  f"dec->merge (oracle/_ref), {t:.2f} s wall on {threads} threads"}
            except Exception as e:  # noqa: BLE001
                line["cpu_baseline"] = {"value": None, "unavailable": str(e)}
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    ws, rank, local = dist_env()
    if args.gpus != ws and ws > 1:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE {ws}", file=sys.stderr)
    if args.impl == "reference":
        run_reference_arm(args, ws, rank)
    else:
        run_ours(args, ws, rank, local)


if __name__ == "__main__":
    main()
