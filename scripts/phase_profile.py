"""Kernel anatomy at 128K: globaltimer marks of CTA (0,0,0) in each kernel of one layer (fused path)."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2602_07721_b200 import build  # noqa: E402

build.build()
from paper_2602_07721_b200 import pariskv as pkv  # noqa: E402

pkv._lib.pkv_phase_profile.argtypes = [ctypes.c_void_p]
dev = torch.device("cuda", 0)
n = int(os.environ.get("PHASE_CTX", "131072")) - 272  # PHASE_CTX=1048576 PHASE_UVA=1: the 1M configuration
stats = synth.head_stats(0, 8, device=dev)
B = int(os.environ.get("PHASE_BATCH", "1"))  # PHASE_CTX=32768 PHASE_BATCH=8: configuration 3
K = synth.llm_keys(0, B, 8, n, device=dev, stats=stats)
q = synth.llm_queries(0, B, 32, 8, device=dev, stats=stats)
synth.plant(K, q, 0)
V = synth.values(0, B, 8, n, device=dev)
Kh = synth.isotropic(7, (B, 8, 272, 128), device=dev)
Vh = synth.isotropic(8, (B, 8, 272, 128), device=dev)
cfg = pkv.config_init(32, 8, synth.rotation_sign_bits())
ix = pkv.Index(cfg, B, n)
pkv.encode_keys(ix, K)
if os.environ.get("PHASE_UVA") == "1":  # K/V rows read through UVA from pinned host memory
    torch.cuda.synchronize()
    K, V = K.cpu().pin_memory(), V.cpu().pin_memory()
    torch.cuda.empty_cache()
for _ in range(3):
    pkv.retrieve_and_attend(ix, q, K, V, 100, Kh, Vh)
torch.cuda.synchronize()
# replay one layer's five kernels from a CUDA graph, as bench.py does (eager launches add host-side gaps)
graph = torch.cuda.CUDAGraph()
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    pkv.retrieve_and_attend(ix, q, K, V, 100, Kh, Vh)
    st.synchronize()
    with torch.cuda.graph(graph, stream=st):
        pkv.retrieve_and_attend(ix, q, K, V, 100, Kh, Vh)
torch.cuda.synchronize()
buf = torch.zeros(256 + 8192, dtype=torch.int64, device=dev)
pkv._lib.pkv_phase_profile(ctypes.c_void_p(buf.data_ptr()))
names = {1: "qprep", 2: "scan", 3: "select", 5: "rerank", 6: "topk+attend", 8: "hot attend"}
for rep in range(3):
    buf.zero_()
    torch.cuda._sleep(20_000_000)
    graph.replay()
    torch.cuda.synchronize()
    allb = buf.cpu().tolist()
    b = [allb[16 * i:16 * i + 16] for i in range(16)]
    t0 = min(v for row in b for v in row if v > 0)
    print(f"--- rep {rep} (us from first mark)")
    for kind, nm in names.items():
        marks = [(i, (v - t0) / 1000.0) for i, v in enumerate(b[kind]) if v > 0]
        print(f"{nm:12s} " + "  ".join(f"p{i}={t:7.2f}" for i, t in marks))
    import statistics
    for nm, bit in (("select", 0), ("rerank", 1)):
        ends = [(allb[256 + 2 * c + bit] - t0) / 1000 for c in range(2048) if allb[256 + 2 * c + bit] > 0]
        starts = [(allb[256 + 4096 + 2 * c + bit] - t0) / 1000 for c in range(2048) if allb[256 + 4096 + 2 * c + bit] > 0]
        if ends:
            dur = [allb[256 + 2 * c + bit] - allb[256 + 4096 + 2 * c + bit] for c in range(2048) if allb[256 + 2 * c + bit] > 0]
            print(f"  {nm} CTAs: n={len(ends)} start min/med/max {min(starts):.2f}/{statistics.median(starts):.2f}/{max(starts):.2f}"
                  f"  end min/med/max {min(ends):.2f}/{statistics.median(ends):.2f}/{max(ends):.2f}"
                  f"  dur(us) med/max {statistics.median(dur)/1000:.2f}/{max(dur)/1000:.2f}")
            qs = lambda v: "/".join(f"{x:.1f}" for x in statistics.quantiles(v, n=10)) if len(v) > 1 else ""
            print(f"   {nm} start deciles {qs(starts)}")
            print(f"   {nm} end deciles   {qs(ends)}")
            if nm == "select":
                slow = sorted(range(len(ends)), key=lambda i: -ends[i])[:8]
                print("   slowest select CTAs (linear id -> end):", [(i, round(ends[i], 2)) for i in slow])
pkv._lib.pkv_phase_profile(ctypes.c_void_p(0))
