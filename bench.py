#!/usr/bin/env python3
"""Branch-parallel decode benchmark (BASELINE.json metric, configs[1] shape).

Workload (one "step"): every branch of every request appends its new token's K/V into the
paged cache (RoPE fused) and attends over shared Map prefix + its own suffix — the decode
hot path of engine.cpp:599-641 (resolve + ToyModel::step attention + extend), batched.
  per request: Qwen2.5-32B attention shape (40 q / 8 kv heads, head_dim 128, bf16),
  4096-token shared Map prefix, 8 branches x 1024 tokens, KV pages of 16 tokens.
  R requests per GPU (default 16 -> 0.8 GB of KV, larger than the 126 MB L2: no flush needed).

Prints ONE JSON line (rank 0). `--impl reference` times the reference CPU path instead: the
patched reference core compiled from /root/reference (oracle/_ref/refdrv, kind "reference") running
its own decode path (RadixStore::resolve_payloads + ToyModel::step, engine.cpp:599-607) on all host
cores, attention part isolated as step(ctx) - step(empty); if that binary was not built, the
oracle restatement of toy_model.cpp:121-157 (fp64, GQA; kind "port").
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

HQ, HKV, D = 40, 8, 128
PREFIX, BRANCHES, BRANCH_LEN = 4096, 8, 1024
# --workload: c2 = configs[1] (the metric's config, R requests per GPU, weak scaling);
# c4 = configs[3] (64 requests x 32 branches, 16K shared prefix + 32 x 512 = 32K unique tokens per
# request, sharded by request across the GPUs: strong scaling)
WORKLOADS = {"c2": dict(prefix=4096, branches=8, branch_len=1024),
             "c4": dict(prefix=16384, branches=32, branch_len=512, total_requests=64)}
METRIC = "branch-parallel decode tokens/s/GPU; attention HBM GB/s vs 8 TB/s roofline"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--requests", type=int, default=16, help="requests per GPU (c2)")
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--shard", default="requests", choices=["requests", "heads"],
                    help="heads: every rank serves all requests for its KV-head group and the head-sharded "
                         "outputs are all-gathered over NCCL each step (the layer-level bench, SURVEY.md §8e)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["hbm_gbs"], "measured"
    except Exception:
        return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index, self.samples, self.proc = index, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([x.strip() for x in line.split(",")])

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        self.t.join(timeout=2)
        sm = [float(s[0]) for s in self.samples if len(s) >= 6 and s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if len(s) >= 6 and s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in self.samples if len(s) >= 6 for k in range(4) if s[2 + k] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def ref_binary():
    path = os.path.join(REPO, "oracle", "_ref", "refdrv")
    return path if os.access(path, os.X_OK) else None


def cpu_reference_ref(seconds: float):
    """The reference's own decode path (engine.cpp:599-607: RadixStore::resolve_payloads + ToyModel::step),
    compiled from /root/reference by oracle/ref_build.sh, on all host cores (one branch per thread).
    step() also runs projections + MLP, so the value is the attention path: step(ctx) - step(empty ctx)."""
    threads = os.cpu_count() or 1
    out = subprocess.run([ref_binary(), "decode", str(threads), str(seconds)], capture_output=True, text=True,
                         check=True, timeout=600).stdout
    r = json.loads(out.strip().splitlines()[-1])
    return {"value": r["tokens_per_s_attention"], "unit": "tokens/s", "cores": threads, "kind": "reference",
            "sample": f"{r['steps']} branch decode steps of the patched reference (resolve_payloads + ToyModel::step "
                      f"attention; 40 heads x 128 MHA, ctx {r['ctx']}, fp64) on {threads} threads; full step incl. "
                      f"projections/MLP: {r['tokens_per_s_full']:.3f} tokens/s"}


def cpu_baseline(seconds: float):
    return cpu_reference_ref(seconds) if ref_binary() else cpu_reference(seconds)


def cpu_reference(seconds: float):
    """Oracle restatement of the reference attention core on all host cores, one request's step
    (8 branches x 40 heads over 4096+1024 tokens) repeated for ~`seconds`."""
    import oracle
    rng = np.random.default_rng(0)
    n_rows = PREFIX + BRANCHES * BRANCH_LEN
    K = rng.uniform(-1, 1, (n_rows, HKV, D))
    V = rng.uniform(-1, 1, (n_rows, HKV, D))
    q = rng.uniform(-1, 1, (BRANCHES, HQ, D))
    ctx = [list(range(PREFIX)) + list(range(PREFIX + b * BRANCH_LEN, PREFIX + (b + 1) * BRANCH_LEN))
           for b in range(BRANCHES)]
    threads = os.cpu_count() or 1
    oracle.attn_decode(q, K, V, ctx, nthreads=threads)  # warm
    reps, t0 = 0, time.perf_counter()
    while True:
        oracle.attn_decode(q, K, V, ctx, nthreads=threads)
        reps += 1
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    return {"value": BRANCHES * reps / el, "unit": "tokens/s", "cores": threads, "kind": "port",
            "sample": f"{reps} decode steps of 1 request (8 branches x 40 heads, ctx 4096+1024, fp64) "
                      f"in {el:.1f} s on {threads} threads"}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    cpu = cpu_baseline(max(2.0, args.cpu_seconds))
    line = {"impl": "reference", "metric": METRIC, "value": cpu["value"], "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * BRANCHES / cpu["value"],
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "configs[1]: 40q/8kv heads, d128, 4K shared prefix, 8 branches x 1K, page 16",
                       "sample": cpu["sample"]},
            "cpu_baseline": cpu,
            "e2e": {"value": cpu["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def build_workload(mv, torch, R, dev, first_request=0, prefix=PREFIX, branches_per_req=BRANCHES,
                   branch_len=BRANCH_LEN, steps_total=0, hkv=HKV):
    """R requests: root prefix, fork into B branches, branch_len - 1 private tokens each (positions
    shared start).  Request r's data is seeded by its global id, so every rank holds distinct
    requests.  The pool has room for steps_total appended tokens per branch."""
    PREFIX, BRANCHES, BRANCH_LEN = prefix, branches_per_req, branch_len  # noqa: N806
    pages = R * (PREFIX // 16 + 1 + BRANCHES * ((BRANCH_LEN + steps_total) // 16 + 3)) + 1024
    # page-table arena: every branch holds its own span list (prefix entries + private tail), with
    # the store's capacity doubling on growth
    table = 2 * R * (BRANCHES + 1) * (PREFIX // 16 + (BRANCH_LEN + steps_total) // 16 + 8) + 65536
    HKV = hkv  # noqa: N806  (this rank's KV-head group)
    st = mv.kv.PagedStore(num_pages=pages, layers=1, kv_heads=HKV, table_entries=table)
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + first_request)

    def rnd(*shape):
        return (torch.rand(*shape, generator=gen, device=dev) * 2 - 1).to(torch.bfloat16)

    branches, positions = [], []
    for r in range(R):
        root = st.create()
        st.append_many(root, torch.full((PREFIX,), 11, dtype=torch.int32, device=dev),
                       torch.arange(PREFIX, dtype=torch.int32, device=dev), 0, rnd(PREFIX, HKV, D),
                       rnd(PREFIX, HKV, D))
        for b in st.fork(root, BRANCHES):
            n = BRANCH_LEN - 1
            st.append_many(b, torch.full((n,), 12, dtype=torch.int32, device=dev),
                           torch.arange(PREFIX, PREFIX + n, dtype=torch.int32, device=dev), 0, rnd(n, HKV, D),
                           rnd(n, HKV, D))
            branches.append(b)
            positions.append(PREFIX + n)
        st.release(root)  # the parent lane waits; its prefix pages live on through the branches
    torch.cuda.synchronize()
    return st, branches, positions, rnd


def run_ours(args):
    import torch
    world, rank, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    dev = torch.device("cuda", local if world > 1 else 0)
    torch.cuda.set_device(dev)
    import paper_2506_09991_b200 as mv

    from paper_2506_09991_b200.shard import shard_heads, shard_requests, max_over_ranks
    # weak scaling: R requests per GPU, sharded by request (no collective in attention)
    wl = WORKLOADS[args.workload]
    heads_mode = args.shard == "heads"
    if heads_mode:
        # layer-level bench: all ranks serve the same requests, each for its KV-head group
        total = wl.get("total_requests", args.requests)
        shard = shard_heads(total, HKV, world, rank)
    else:
        total = wl.get("total_requests", args.requests * world)
        shard = shard_requests(total, HKV, world, rank)
    R = len(shard.requests)
    hkv_l = shard.kv_heads[1] - shard.kv_heads[0]
    hq_l = hkv_l * (HQ // HKV)
    steps_total = args.warmup + args.steps
    steps_total += max(3, args.steps // 2)  # the e2e leg appends too
    # a head-sharded rank seeds its data by (first request, head group): synthetic values per shard
    seed_id = shard.requests[0] * 64 + shard.kv_heads[0]
    st, handles, pos0, rnd = build_workload(mv, torch, R, dev, seed_id, wl["prefix"], wl["branches"],
                                            wl["branch_len"], steps_total, hkv=hkv_l)
    n = len(handles)
    handles = mv.kv.handle_array(handles)  # uint64 array: no per-call list conversion
    steps_total = args.warmup + args.steps
    # per-step inputs (device resident for `value`)
    qs = [rnd(n, hq_l, D) for _ in range(2)]
    ks = [rnd(n, hkv_l, D) for _ in range(2)]
    vs = [rnd(n, hkv_l, D) for _ in range(2)]
    toks = torch.full((n,), 13, dtype=torch.int32, device=dev)
    out = torch.empty(n, hq_l, D, dtype=torch.bfloat16, device=dev)
    # head-sharded outputs of all ranks: [world][n][hq_l][D] (NCCL all-gather each step)
    gathered = torch.empty(world, n, hq_l, D, dtype=torch.bfloat16, device=dev) if heads_mode and world > 1 else None
    ag = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)] if gathered is not None else []
    base_pos = torch.tensor(pos0, dtype=torch.int32, device=dev)

    def step(i, q, k, v, p):
        st.append(handles, toks, p, 0, k, v)
        mv.attention.decode(st, handles, q, p, out=out)

    stream = torch.cuda.current_stream()
    for i in range(args.warmup):
        step(i, qs[i % 2], ks[i % 2], vs[i % 2], base_pos + i)
    torch.cuda.synchronize()
    info = st.plan_info()

    # ---- timed region (device events; attention launches bracketed separately) ----
    clocks = Clocks(local)
    clocks.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    att = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    pos_steps = [base_pos + (args.warmup + s) for s in range(args.steps)]  # inputs resident before timing
    torch.cuda.synchronize()
    ev[0].record(stream)
    t_host0 = time.perf_counter()
    for s in range(args.steps):
        i = args.warmup + s
        p = pos_steps[s]
        st.append(handles, toks, p, 0, ks[i % 2], vs[i % 2])
        att[s][0].record(stream)
        mv.attention.decode(st, handles, qs[i % 2], p, out=out)
        att[s][1].record(stream)
        if gathered is not None:  # layer-level: every rank assembles all heads of every token
            ag[s][0].record(stream)
            dist.all_gather_into_tensor(gathered, out)
            ag[s][1].record(stream)
    ev[1].record(stream)
    host_ms = (time.perf_counter() - t_host0) * 1e3 / args.steps  # enqueue cost per step (host)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    ms = ev[0].elapsed_time(ev[1]) / args.steps
    att_each = [a.elapsed_time(b) for a, b in att]
    att_ms = float(np.mean(att_each))
    ag_ms = float(np.mean([a.elapsed_time(b) for a, b in ag])) if ag else 0.0
    if os.environ.get("MV_BENCH_DUMP"):
        np.save(os.environ["MV_BENCH_DUMP"], np.array(att_each))
    ms, att_ms, ag_ms = max_over_ranks([ms, att_ms, ag_ms], device=dev)

    # ---- e2e through the public API with host buffers (pinned), copies inside the region ----
    # one pinned host block per step input set [q | k | v | positions] -> one H2D copy per step
    nq, nk = n * hq_l * D * 2, n * hkv_l * D * 2
    blk = nq + 2 * nk + n * 4
    hin = [torch.empty(blk, dtype=torch.uint8).pin_memory() for _ in range(2)]
    for j in range(2):
        hin[j][:nq].copy_(qs[j].cpu().view(torch.uint8).reshape(-1))
        hin[j][nq:nq + nk].copy_(ks[j].cpu().view(torch.uint8).reshape(-1))
        hin[j][nq + nk:nq + 2 * nk].copy_(vs[j].cpu().view(torch.uint8).reshape(-1))
    hpos = [hin[j][nq + 2 * nk:].view(torch.int32) for j in range(2)]
    din = torch.empty(blk, dtype=torch.uint8, device=dev)
    dq = din[:nq].view(torch.bfloat16).view(n, hq_l, D)
    dk = din[nq:nq + nk].view(torch.bfloat16).view(n, hkv_l, D)
    dv = din[nq + nk:nq + 2 * nk].view(torch.bfloat16).view(n, hkv_l, D)
    dp = din[nq + 2 * nk:].view(torch.int32)
    hout = torch.empty(n, hq_l, D, dtype=torch.bfloat16).pin_memory()
    pos0_np = np.asarray(pos0, dtype=np.int32)
    e2e_steps = max(3, args.steps // 2)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ee = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ee[0].record(stream)
    for s in range(e2e_steps):
        i = args.warmup + args.steps + s
        hpos[i % 2].numpy()[:] = pos0_np + i  # the step's positions, written into the pinned block
        din.copy_(hin[i % 2], non_blocking=True)
        st.append(handles, toks, dp, 0, dk, dv)
        mv.attention.decode(st, handles, dq, dp, out=out)
        hout.copy_(out, non_blocking=True)
        stream.synchronize()  # the caller reads this step's result before the next step
    ee[1].record(stream)
    torch.cuda.synchronize()
    e2e_ms = ee[0].elapsed_time(ee[1]) / e2e_steps
    (e2e_ms,) = max_over_ranks([e2e_ms], device=dev)
    h2d = n * (hq_l + 2 * hkv_l) * D * 2 + n * 4
    d2h = n * hq_l * D * 2

    tokens_per_step = n if heads_mode else n * world  # head-sharded ranks share their tokens
    value = tokens_per_step / (ms / 1e3)
    # roofline of the dominant kernel: algorithmic bytes = unique KV read once + Q/O
    # every step appends one token per branch before attending, so the context (and the bytes a
    # step must read) grows by n tokens per step: use the mean over the timed steps
    kv_tokens = info["unique_kv_tokens"] + n * (args.steps + 1) / 2.0
    alg_bytes = kv_tokens * hkv_l * D * 2 * 2 + n * hq_l * D * 2 * 2
    achieved = alg_bytes / (att_ms / 1e3) / 1e9
    peak, peak_kind = peaks()
    traffic = None
    try:
        with open(os.path.join(REPO, "profiles", "decode_traffic.json")) as f:
            tj = json.load(f)
            if tj.get("requests") == R and args.workload == "c2" and not heads_mode:
                traffic = tj["per_kernel_bytes"].get(tj.get("dominant_kernel", ""), tj.get("dram_bytes_per_launch"))
    except Exception:
        pass

    if rank == 0:
        cpu = cpu_baseline(args.cpu_seconds) if world == 1 and args.workload == "c2" else None
        if args.workload == "c4":
            wl_text = ("configs[3]: 64 requests x 32 branches sharded by request over the GPUs, 40q/8kv heads, "
                       "d128, bf16, 16K shared prefix + 32 x 512 branch tokens (32K unique per request, +1 per "
                       "branch per step), KV page 16")
        else:
            wl_text = ("configs[1] x R requests per GPU: 40q/8kv heads, d128, bf16, 4K shared Map prefix, 8 "
                       "branches x 1K tokens (+1 per step), KV page 16")
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong" if (args.workload == "c4" or heads_mode) else "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": wl_text,
                       "requests_per_gpu": R, "branches_per_gpu": n, "l2": "inputs 0.8+ GB > L2 (no flush)",
                       "mean_kv_tokens_per_step": kv_tokens, "host_enqueue_ms_per_step": host_ms,
                       "parallelism": (f"kv-head groups x{world} + NCCL all-gather of outputs" if heads_mode
                                       else f"requests x{world}, no collective"),
                       "kv_heads_per_gpu": hkv_l, "allgather_ms_per_step": ag_ms if heads_mode else None,
                       "step": "append 1 token K/V per branch (RoPE fused) + cascade decode attention"},
            "e2e": {"value": tokens_per_step / (e2e_ms / 1e3), "unit": "tokens/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_kind,
                         "kernel": "decode_tc_kernel (+ rope_q_tile_kernel, combine_kernel)",
                         "alg_bytes_per_launch": alg_bytes,
                         "launch_ms": att_ms, "frac_of_8TBs": achieved / 8000.0},
            "gpu_launches": 4 * args.steps,  # per step: k_append_one, rope_q_tile, decode_tc, combine
            "clocks": clk,
            "plan": info,
        }
        if cpu:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
