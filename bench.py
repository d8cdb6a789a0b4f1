"""Decode-step benchmark of the ParisKV retrieval hot path on B200 (BASELINE.json metric).

A step = one decode step of a Llama-3.1-8B-shaped model (32 q / 8 KV heads, d = 128, 32 layers, each layer
with its own index and K/V so > L2 is touched per step): per layer retrieve_topk (query prep, collision
scan, bucket_topk, RSQ-IP rerank, top-k) + sparse_attend (hot rows U top-k rows). Inputs are synthetic
(synth/, recipe in DESIGN.md), resident in HBM before the timed region. value = device time per layer.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 128k|32k_bs8]

N > 1 (torchrun): the retrieval zone of every layer is sequence-sharded over the ranks (NCCL exchanges
inside the library); value = the max-over-ranks time per layer of the whole job (strong scaling).
--impl reference: the CPU oracle (oracle/) timed on a bounded sample on the host cores (rank 0 only).
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

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decode retrieval+attn µs/layer at 128K & 1M ctx; scan HBM GB/s vs 8 TB/s peak"
UNIT = "us/layer"
N_LAYERS = 32
N_Q, N_KV, D = 32, 8, 128
TOP_K = 100
N_SINK, N_LOCAL = 16, 256  # hot rows (Table 1 AIME row; sink 16 per S:452)

CONFIGS = {
    # BASELINE configs[1]: bs=1, 128K context, 1 decode step, all 32 layers
    "128k": dict(batch=1, context=131072, workload="llama3.1-8b-shape bs1 ctx131072 decode step, 32 layers"),
    # BASELINE configs[2]: bs=8 at 32K
    "32k_bs8": dict(batch=8, context=32768, workload="llama3.1-8b-shape bs8 ctx32768 decode step, 32 layers"),
    # BASELINE configs[4]: 1M-token context, full-precision K/V in pinned host memory read through UVA
    # (P:515-517); 32 per-layer indices in HBM built from 4 distinct datasets (4 x 4.3 GB of host K/V)
    "1m": dict(batch=1, context=1048576, uva=True, datasets=4,
               workload="llama3.1-8b-shape bs1 ctx1048576 decode step, 32 layers, K/V in pinned host memory (UVA)"),
}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region (B200_PROFILING.md)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "20", "-i", str(self.device)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.3)
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.05)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("PKV_BENCH_GLOO") == "1":  # several ranks per GPU (functional checks, see run_ours)
        import torch
        local = local % max(1, torch.cuda.device_count())
    return world, rank, local


# ----------------------------------------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2602_07721_b200 import build as pbuild
    pbuild.build()

    world, rank, local = dist_env()
    # PKV_BENCH_GLOO=1: gloo plumbing and every rank on the visible GPU(s) modulo their count — a functional check
    # of the sharded paths with several ranks on one GPU (peer transport); timings are then meaningless
    gloo = os.environ.get("PKV_BENCH_GLOO") == "1"
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if gloo:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    res = measure(args, args.config)
    # the metric names both contexts: the default run also measures the 1M configuration (BASELINE configs[4],
    # K/V in pinned host memory) in the same process and reports it as configs["1m"]
    if args.config == "128k" and not args.no_1m:
        torch.cuda.empty_cache()
        blk = measure(args, "1m")
        if rank == 0:
            res["configs"] = {"1m": {k: blk[k] for k in ("value", "ms_per_step", "config", "roofline", "scan_gbs",
                                                         "scan_hbm", "kernels", "encode_us_per_layer", "encode_gbs",
                                                         "e2e", "gpu_launches", "clocks")}}
    if rank == 0:
        if not args.no_cpu and world == 1:
            res["cpu_baseline"] = cpu_baseline(args.config, budget_s=args.cpu_budget)
        print(json.dumps(res))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def measure(args, config: str) -> dict:
    """Set up one configuration (synthetic inputs resident before timing), time K graph-replayed steps and the
    end-to-end variant, and return its JSON block (rank 0; other ranks return None)."""
    import torch
    import torch.distributed as dist

    import synth
    from paper_2602_07721_b200 import pariskv as pkv

    world, rank, local = dist_env()
    dev = torch.device("cuda", local)
    cfgw = CONFIGS[config]
    batch, ctx = cfgw["batch"], cfgw["context"]
    n_hot = N_SINK + N_LOCAL
    n = ctx - n_hot                               # retrieval zone (AMB-22)
    lo, hi = rank * n // world, (rank + 1) * n // world
    n_loc = hi - lo
    T, C = pkv.schedule(n, TOP_K)
    cfg = pkv.config_init(N_Q, N_KV, synth.rotation_sign_bits())
    cfg.w_fp16 = 1 if args.w16 else 0  # AMB-20 variant: 96-byte records with fp16 weights
    L = args.layers

    # ---- synthetic inputs, per layer distinct indices (> L2 touched per step) ----
    uva = cfgw.get("uva", False)
    n_data = min(L, cfgw.get("datasets", L))
    layers = []
    data = []
    for l in range(L):
        if l < n_data:
            seed = 1000 * l
            stats = synth.head_stats(seed, N_KV, device=dev)
            K = synth.llm_keys(seed, batch, N_KV, n, device=dev, stats=stats)
            q = synth.llm_queries(seed, batch, N_Q, N_KV, device=dev, stats=stats)
            synth.plant(K, q, seed)
            V = synth.values(seed, batch, N_KV, n, device=dev)
            Kl, Vl = K[:, :, lo:hi].contiguous(), V[:, :, lo:hi].contiguous()
            del K, V
            Kh = synth.isotropic(seed + 7, (batch, N_KV, n_hot, D), device=dev)
            Vh = synth.isotropic(seed + 8, (batch, N_KV, n_hot, D), device=dev)
            if uva and args.k_hbm:  # variant: keys stay in HBM (64 GB for 32 layers at 1M fits a B200's 180 GB),
                Vl = Vl.cpu().pin_memory()  # only the value rows of the top-k cross the host link
                data.append(dict(K=Kl, V=Vl, Kd=Kl, Kh=Kh, Vh=Vh, q=q.contiguous()))
            elif uva:  # full-precision K/V live in pinned host memory; the GPU keeps only summaries + hot rows
                Kd, Vd = Kl, Vl
                Kl, Vl = Kl.cpu().pin_memory(), Vl.cpu().pin_memory()
                data.append(dict(K=Kl, V=Vl, Kd=Kd, Kh=Kh, Vh=Vh, q=q.contiguous()))
            else:
                data.append(dict(K=Kl, V=Vl, Kd=Kl, Kh=Kh, Vh=Vh, q=q.contiguous()))
        d = data[l % n_data]
        ix = pkv.Index(cfg, batch, n_loc, device=local)
        if layers:
            ix.share_workspace(layers[0]["ix"])
        layers.append(dict(ix=ix, K=d["K"], V=d["V"], Kd=d["Kd"], Kh=d["Kh"], Vh=d["Vh"], q=d["q"],
                           idx=torch.empty(batch, N_Q, TOP_K, dtype=torch.int32, device=dev),
                           est=torch.empty(batch, N_Q, TOP_K, dtype=torch.float32, device=dev),
                           out=torch.empty(batch, N_Q, D, dtype=torch.bfloat16, device=dev),
                           lse=torch.empty(batch, N_Q, dtype=torch.float32, device=dev)))
    torch.cuda.synchronize()
    if world > 1 and args.transport == "peer":  # one-shot all-gather kernels over NVLink peer memory
        handle, _ = layers[0]["ix"].comm_init_peer(rank, world, lo)
        handles = [None] * world
        dist.all_gather_object(handles, handle)
        layers[0]["ix"].comm_peer_connect(handles)
        pkv.comm_set_global_len(layers[0]["ix"], n)
        for ly in layers[1:]:
            pkv.comm_share(ly["ix"], layers[0]["ix"], lo)
        dist.barrier()
    elif world > 1:
        uid = [pkv.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        pkv.comm_init(layers[0]["ix"], uid[0], rank, world, lo)
        for ly in layers[1:]:
            pkv.comm_share(ly["ix"], layers[0]["ix"], lo)

    # ---- encode (prefill key summarisation), timed separately ----
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    pkv.encode_keys(layers[0]["ix"], layers[0]["Kd"])  # warm-up (module load); re-encoded in the timed loop
    torch.cuda.synchronize()
    e0.record()
    for ly in layers:
        pkv.encode_keys(ly["ix"], ly["Kd"])
    e1.record()
    torch.cuda.synchronize()
    enc_ms_layer = e0.elapsed_time(e1) / L
    if args.inverted:  # inverted-list collision scan (same results; builds the postings now)
        for ly in layers:
            ly["ix"].set_postings(True)
        torch.cuda.synchronize()
    rho_keys = 0
    if args.key_fraction:  # rho as a fraction of keys (AMB-8b): occupancy counts, per-subspace probes
        if world > 1:
            raise SystemExit("--key-fraction is single-GPU (the occupancy counts are not exchanged)")
        rho_keys = pkv.schedule_key_fraction(n)
        for ly in layers:
            ly["ix"].set_occupancy(True)
        torch.cuda.synchronize()
    if uva and not args.k_hbm:  # the device copies were only needed to build the summaries
        for d in data:
            d["Kd"] = None
        for ly in layers:
            ly["Kd"] = None
        torch.cuda.empty_cache()

    # the step's queries and outputs live in one device buffer each (layer l = slice l), so the end-to-end
    # measurement moves a step's inputs and results with one copy each way
    q_all = torch.stack([ly["q"] for ly in layers]).contiguous()
    out_all = torch.empty((L, batch, N_Q, D), dtype=torch.bfloat16, device=dev)
    for l, ly in enumerate(layers):
        ly["q"], ly["out"] = q_all[l], out_all[l]

    # one call per layer; when sharded the library runs the fused T+A exchange (two collectives per layer)
    fused = not args.two_calls

    def layer_call(ly):
        if fused:  # one decode step of one layer: retrieval + attention scheduled as one unit
            pkv.retrieve_and_attend(ly["ix"], ly["q"], ly["K"], ly["V"], TOP_K, ly["Kh"], ly["Vh"], probes_T=T,
                                    n_cand=C, n_global=n, out_idx=ly["idx"], out_est=ly["est"], out=ly["out"],
                                    lse=ly["lse"], rho_keys=rho_keys)
        else:
            pkv.retrieve_topk(ly["ix"], ly["q"], TOP_K, probes_T=T, n_cand=C, n_global=n, out_idx=ly["idx"],
                              out_est=ly["est"], rho_keys=rho_keys)
            pkv.sparse_attend(ly["ix"], ly["q"], ly["K"], ly["V"], ly["idx"], ly["Kh"], ly["Vh"], out=ly["out"],
                              lse=ly["lse"])

    def step():
        for ly in layers:
            layer_call(ly)

    # warm-up (eager) + launch accounting
    for _ in range(max(1, args.warmup)):
        step()
    torch.cuda.synchronize()
    c0 = pkv.launch_count()
    step()
    torch.cuda.synchronize()
    launches_per_step = pkv.launch_count() - c0

    use_graph = not args.no_graph
    graph = None
    if use_graph:
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            step()
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step()
        torch.cuda.synchronize()
        run = graph.replay
    else:
        run = step
    for _ in range(args.warmup):
        run()
    torch.cuda.synchronize()

    def timed(fn, k):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(k):
            fn()
        b.record()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ms = a.elapsed_time(b)
        if world > 1:
            t = torch.tensor([ms], device="cpu" if dist.get_backend() == "gloo" else dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    with ClockSampler(local) as clk:
        total_ms = timed(run, args.steps)
    ms_step = total_ms / args.steps
    us_layer = ms_step * 1000.0 / L

    # ---- per-kernel device times (CUDA events on the launch stream, eager replay of the same step) ----
    prof_steps = max(3, min(args.steps, 20))
    pkv.profile_enable(True)
    for _ in range(prof_steps):
        torch.cuda._sleep(40_000_000)  # GPU spins ~20 ms so the host enqueues the whole step ahead of it:
        step()                         # the bracketing events then time kernels, not host launch gaps
    torch.cuda.synchronize()
    prof = pkv.profile_read()
    pkv.profile_enable(False)

    # ---- end to end through the public API with host buffers (pinned H2D q, D2H attention output) ----
    q_host = q_all.cpu().pin_memory()
    o_host = torch.empty_like(out_all, device="cpu").pin_memory()

    def step_e2e():  # the step's queries in (one H2D), all layers, the step's attention outputs out (one D2H)
        q_all.copy_(q_host, non_blocking=True)
        for ly in layers:
            layer_call(ly)
        o_host.copy_(out_all, non_blocking=True)

    if use_graph:
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            step_e2e()
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        g2 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g2):
            step_e2e()
        run2 = g2.replay
    else:
        run2 = step_e2e
    for _ in range(args.warmup):
        run2()
    e2e_ms = timed(run2, args.steps) / args.steps
    e2e_eager_ms = timed(step_e2e, max(3, min(args.steps, 20))) / max(3, min(args.steps, 20))

    # ---- context: dense decode attention over the same retrieval-zone K/V (PyTorch SDPA, Eq. 1) ----
    dense_us = None
    if not uva and world == 1 and not args.no_dense:
        import torch.nn.functional as F
        qs = [ly["q"].unsqueeze(2) for ly in layers]

        def dense_step():
            for ly, q4 in zip(layers, qs):
                F.scaled_dot_product_attention(q4, ly["K"], ly["V"], enable_gqa=True)

        try:
            for _ in range(2):
                dense_step()
            dense_us = round(timed(dense_step, 5) / 5 * 1000.0 / L, 2)
        except Exception as e:  # SDPA GQA path unavailable: report why instead of a number
            dense_us = f"unavailable: {type(e).__name__}"

    # ---- roofline of the dominant kernel (algorithmic bytes / measured average launch time) ----
    hbm_peak, peak_kind = peaks()
    alg = {
        # 16 B of centroid ids per (key, KV head)
        "scan": batch * N_KV * n_loc * 16,
        # bucket_topk reads the packed per-key scores (4 query heads x u8 = 4 B per key and KV head) and writes
        # one candidate id (4 B) per (candidate, query head)
        "select": batch * N_KV * n_loc * 4 + batch * N_Q * min(C, n_loc) * 4,
        # fused RSQ-IP rerank: reads the candidate id and gathers its 128 B record, writes the estimate (4 B),
        # per (candidate, query head)
        "rerank": batch * N_Q * min(C, n_loc) * (4 + (96 if args.w16 else 128) + 4),
        # fused path: top-k over (est, id) pairs + gather of the k selected K/V rows (512 B per row and head)
        # + the hot rows (512 B per row and KV head, attended in the same kernel); two-call path: top-k only
        "topk": batch * N_Q * min(C, n_loc) * 8 + (batch * N_Q * TOP_K * 512 if fused else 0)
        + (batch * N_KV * n_hot * 512 if fused and rank == world - 1 else 0),  # fused: hot rows too
        # fused path: hot rows only (read once per KV head); two-call path: hot + retrieved rows
        "attend": batch * ((0 if fused else N_Q * TOP_K * 512) + (N_KV * n_hot * 512 if rank == world - 1 else 0)),
    }
    kern = {}
    for name, (cnt, ms) in prof.items():
        avg_us = ms * 1000.0 / cnt
        ent = {"launches": cnt, "avg_us": round(avg_us, 3), "share": round(ms / sum(v[1] for v in prof.values()), 4)}
        if name in alg:
            ent["alg_bytes"] = alg[name]
            ent["gbs"] = round(alg[name] / (avg_us * 1e-6) / 1e9, 1)
        kern[name] = ent
    dom = max((k for k in kern if k in alg), key=lambda k: prof[k][1])
    traffic = None
    # per-kernel DRAM bytes from the latest committed `ncu --set full` capture (this round's, else round 1's)
    tr_file = next((f for f in (os.path.join(ROOT, "profiles", r, "ncu_traffic.json") for r in ("r02", "r01"))
                    if os.path.exists(f)), "")
    if os.path.exists(tr_file):
        try:
            traffic = json.load(open(tr_file)).get(config, {}).get(dom)
        except Exception:
            traffic = None
    roof = {"bound": "hbm", "kernel": dom, "achieved": kern[dom]["gbs"], "peak": hbm_peak, "unit": "GB/s",
            "frac": round(kern[dom]["gbs"] / hbm_peak, 4), "traffic": traffic, "peak_source": peak_kind}
    fl_file = os.path.join(ROOT, "profiles", "r01", "floors_r01.json")
    if uva and fused and dom == "topk" and os.path.exists(fl_file):
        # at 1M the fused top-k is bound by its UVA gather of the k selected rows (SURVEY §8(d) "host link"):
        # its roofline is the measured host-link read rate, over the bytes that cross the link
        link = json.load(open(fl_file))["1m"]["uva_stream_read_gbs"]
        host_bytes = batch * N_Q * TOP_K * (256 if args.k_hbm else 512)
        ach = round(host_bytes / (kern["topk"]["avg_us"] * 1e-6) / 1e9, 1)
        roof = {"bound": "host_link", "kernel": dom, "achieved": ach, "peak": link, "unit": "GB/s",
                "frac": round(ach / link, 4), "traffic": traffic, "peak_source": "measured (scripts/uva_bw.cu)",
                "host_bytes_per_launch": host_bytes}
    # context: measured data-movement floors of the two gathers (profiles/r01/floors_r01.json, scripts/hbm_gather.cu,
    # scripts/uva_bw.cu) — the rerank's random 128 B record gather from HBM and, at 1M, the UVA row gather
    if os.path.exists(fl_file) and world == 1 and not args.w16:
        try:
            fl = json.load(open(fl_file)).get(config)
        except Exception:
            fl = None
        if fl and "rerank" in kern:
            roof["rerank_gather_floor_us"] = fl["rerank_gather_us"]
            roof["rerank_frac_of_gather_floor"] = round(fl["rerank_gather_us"] / kern["rerank"]["avg_us"], 4)
            if uva and "uva_gather_3200_rows_us" in fl:
                roof["host_link_gbs"] = fl["uva_stream_read_gbs"]
                roof["uva_row_gather_floor_us"] = fl["uva_gather_3200_rows_us"]
    scan_gbs = kern.get("scan", {}).get("gbs")
    # the metric's second half: the collision scan's HBM rate against the 8 TB/s B200 figure the north star
    # names, and against this box's measured copy bandwidth
    scan_vs = None if scan_gbs is None else {"gbs": scan_gbs, "frac_of_8tbs": round(scan_gbs / 8000.0, 4),
                                             "frac_of_measured_peak": round(scan_gbs / hbm_peak, 4),
                                             "timing": "CUDA events around eager launches (breaks PDL overlap)"}
    # the same kernel timed by ncu (warm launch list committed under profiles/, serialised, no PDL overlap)
    warm_file = os.path.join(ROOT, "profiles", "r02", "ncu_warm.json")
    if scan_vs is not None and os.path.exists(warm_file):
        try:
            wu = json.load(open(warm_file)).get(config, {}).get("scan_us")
        except Exception:
            wu = None
        if wu:
            g2 = round(alg["scan"] / (wu * 1e-6) / 1e9, 1)
            scan_vs.update({"ncu_warm_us": wu, "ncu_gbs": g2, "ncu_frac_of_8tbs": round(g2 / 8000.0, 4),
                            "ncu_frac_of_measured_peak": round(g2 / hbm_peak, 4), "ncu_source": "profiles/r02/ncu_warm.json"})

    res = None
    if rank == 0:
        res = {
            "metric": METRIC, "value": round(us_layer, 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_step, 4), "higher_is_better": False,
            "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "u8/f32 (bf16 K,V,q)",
            "data": "synthetic (LLM-like keys with planted top-k; DESIGN.md recipe), random-init, no weights",
            "config": {"workload": cfgw["workload"], "batch": batch, "context": ctx, "retrieval_n": n,
                       "hot_rows": n_hot, "top_k": TOP_K, "probes_T": T, "n_cand": C, "layers": L,
                       "parallelism": f"seq-shard{world}" if world > 1 else "single",
                       "exchange": (args.transport if world > 1 else None),
                       "l2": "inputs > L2: 32 layer-distinct indices + K/V touched per step",
                       "rerank_weights": "fp16 (96 B records)" if args.w16 else "fp32 (128 B records)",
                       "collision_scan": "inverted lists" if args.inverted else "dense",
                       "rho_reading": f"key fraction, rho_keys={rho_keys}" if rho_keys else f"centroid fraction, T={T}",
                       "kv_placement": ("K in HBM, V in pinned host (UVA)" if args.k_hbm else "K, V in pinned host (UVA)")
                       if uva else "HBM",
                       "cuda_graph": use_graph},
            "roofline": roof,
            "scan_gbs": scan_gbs,
            "scan_hbm": scan_vs,
            "kernels": kern,
            "encode_us_per_layer": round(enc_ms_layer * 1000.0, 2),
            "encode_gbs": round(batch * N_KV * n_loc * 400 / (enc_ms_layer * 1e-3) / 1e9, 1),
            "dense_sdpa_us_per_layer": dense_us,
            "e2e": {"value": round(e2e_ms * 1000.0 / L, 3), "unit": UNIT, "h2d_bytes_per_step": L * batch * N_Q * D * 2,
                    "d2h_bytes_per_step": L * batch * N_Q * D * 2, "cuda_graph": use_graph,
                    "eager_value": round(e2e_eager_ms * 1000.0 / L, 3)},
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clk.summary(),
            "cpu_baseline": None,
        }
    # release this configuration's device and pinned memory before the next one is built
    layers.clear()
    data.clear()
    del q_all, out_all, q_host, o_host
    if graph is not None:
        del graph
    if use_graph:
        del g2
    torch.cuda.synchronize()
    return res


# ----------------------------------------------------------------------------------------------- oracle arm
def oracle_unit(config: str):
    """One (layer, KV group) unit of the workload for the CPU oracle: returns a callable doing the oracle's
    decode step (a1, a3-a7) for the G = 4 query heads of one KV head, plus its description."""
    import torch

    import synth
    from oracle import levels, pipeline, quantizer

    cfgw = CONFIGS[config]
    n = cfgw["context"] - (N_SINK + N_LOCAL)
    seed = 0
    stats = synth.head_stats(seed, N_KV)
    K = synth.llm_keys(seed, 1, N_KV, n, stats=stats)
    q = synth.llm_queries(seed, 1, N_Q, N_KV, stats=stats)
    synth.plant(K, q, seed)
    V = synth.values(seed, 1, N_KV, n)
    Kh = synth.isotropic(seed + 7, (1, N_KV, N_SINK + N_LOCAL, D))
    Vh = synth.isotropic(seed + 8, (1, N_KV, N_SINK + N_LOCAL, D))
    sb = synth.rotation_sign_bits()
    L32 = levels.levels_f32(8)
    Kf = synth.to_f64(K[0, 0])
    meta = quantizer.encode_keys(Kf, sb, L32, levels.mid_sq(L32))
    Q = synth.to_f64(q[0, :4])
    Vf, Khf, Vhf = synth.to_f64(V[0, 0]), synth.to_f64(Kh[0, 0]), synth.to_f64(Vh[0, 0])
    del torch

    def unit():
        res = pipeline.decode_step(meta, Q, sb, TOP_K)
        for h, r in enumerate(res):
            pipeline.attend(Q[h], Kf, Vf, r["idx"], Khf, Vhf)

    return unit, f"1 KV group (4 q heads) x 1 layer of {config} (n={n}), x{N_KV} groups -> us/layer (extrapolated)"


def host_info():
    return {"host_cores": len(os.sched_getaffinity(0)), "cpu": _cpu_model(),
            "env_threads": {k: os.environ.get(k) for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS")}}


def config1_end_to_end_s():
    """BASELINE configs[0] (1 head, d=128, N=4096, 1 query, top-k=64) through the oracle end to end: encode the
    keys, retrieve, attend. Seconds (one run after a warm-up run)."""
    import synth
    from oracle import levels, pipeline, quantizer

    K = synth.llm_keys(1, 1, 1, 4096)
    q = synth.llm_queries(1, 1, 1, 1)
    synth.plant(K, q, 1, n_plant=25)
    V = synth.values(1, 1, 1, 4096)
    sb = synth.rotation_sign_bits()
    L32 = levels.levels_f32(8)
    Kf, Vf, qf = synth.to_f64(K[0, 0]), synth.to_f64(V[0, 0]), synth.to_f64(q[0, 0])

    def run():
        meta = quantizer.encode_keys(Kf, sb, L32, levels.mid_sq(L32))
        r = pipeline.decode_step(meta, qf[None], sb, 64)[0]
        pipeline.attend(qf, Kf, Vf, r["idx"])

    run()
    t0 = time.perf_counter()
    run()
    return round(time.perf_counter() - t0, 4)


def cpu_baseline(config: str, budget_s: float = 20.0):
    from threadpoolctl import threadpool_limits
    with threadpool_limits(1):
        unit, desc = oracle_unit(config)
        unit()  # warm
        t0 = time.perf_counter()
        reps = 0
        while True:
            unit()
            reps += 1
            if time.perf_counter() - t0 > budget_s / 2 or reps >= 20:
                break
        dt = (time.perf_counter() - t0) / reps
        c1 = config1_end_to_end_s()
    return {"value": round(dt * N_KV * 1e6, 1), "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"{desc}; {reps} reps, numpy/BLAS limited to 1 thread",
            "threads_used": 1, **host_info(), "config1_end_to_end_s": c1,
            "config1": "1 head, d=128, N=4096, 1 query, top-k=64: encode + retrieve + attend, 1 thread"}


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    from threadpoolctl import threadpool_limits
    with threadpool_limits(1):
        unit, desc = oracle_unit(args.config)
        for _ in range(args.warmup):
            unit()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            unit()
        dt = (time.perf_counter() - t0) / args.steps
    v = round(dt * N_KV * 1e6, 1)
    cfgw = CONFIGS[args.config]
    res = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": round(dt * N_KV * N_LAYERS * 1e3, 3), "higher_is_better": False,
           "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (same recipe as the GPU arm)",
           "config": {"workload": cfgw["workload"], "batch": cfgw["batch"], "context": cfgw["context"],
                      "top_k": TOP_K, "layers": N_LAYERS},
           "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle", "threads_used": 1,
                            "sample": f"each step: {desc}", **host_info()},
           "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(res))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="128k", choices=sorted(CONFIGS))
    ap.add_argument("--layers", type=int, default=N_LAYERS)
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--two-calls", action="store_true", help="retrieve_topk + sparse_attend instead of the fused call")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-1m", action="store_true", help="default 128K run: skip the 1M block (configs['1m'])")
    ap.add_argument("--no-dense", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--w16", action="store_true", help="fp16 rerank weights (96-byte records, AMB-20 / SURVEY f2)")
    ap.add_argument("--inverted", action="store_true", help="inverted-list collision scan (SURVEY f4)")
    ap.add_argument("--transport", default="nccl", choices=["nccl", "peer"],
                    help="sharded exchanges (N > 1): NCCL all-gathers, or one-shot peer-memory all-gather kernels")
    ap.add_argument("--key-fraction", action="store_true",
                    help="rho as a fraction of keys (AMB-8b, SURVEY f4): per-subspace probes from occupancy counts")
    ap.add_argument("--k-hbm", action="store_true",
                    help="1M variant: keys in HBM, only values in pinned host memory (half the UVA bytes)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup) if args.impl == "ours" else args.warmup
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
