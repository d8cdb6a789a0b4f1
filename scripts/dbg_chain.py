import sys, os, torch
sys.path.insert(0, os.getcwd())
import synth
from paper_2602_07721_b200 import build
build.build()
from paper_2602_07721_b200 import pariskv as pkv
from tests.gpu_helpers import SB
batch, n_q, n_kv, N, k = int(sys.argv[1]), 8, 2, int(sys.argv[2]), 50
stats = synth.head_stats(31, n_kv, device="cuda")
K = synth.llm_keys(31, batch, n_kv, N, device="cuda", stats=stats)
V = synth.values(31, batch, n_kv, N, device="cuda")
Kh = synth.isotropic(5, (batch, n_kv, 80, 128), device="cuda")
Vh = synth.isotropic(6, (batch, n_kv, 80, 128), device="cuda")
qs = [synth.llm_queries(31 + 1 + s, batch, n_q, n_kv, device="cuda", stats=stats) for s in range(4)]
cfg = pkv.config_init(n_q, n_kv, SB)
ix = pkv.Index(cfg, batch, N)
pkv.encode_keys(ix, K)
ref = []
for q in qs:
    i, e, o, l = pkv.retrieve_and_attend(ix, q, K, V, k, Kh, Vh)
    torch.cuda.synchronize()
    ref.append(i.clone())
outs = []
for it in range(200):
    q = qs[it % 4]
    i, e, o, l = pkv.retrieve_and_attend(ix, q, K, V, k, Kh, Vh)
    outs.append(i)
torch.cuda.synchronize()
bad = [it for it, i in enumerate(outs) if not torch.equal(i, ref[it % 4])]
outs = []
for it in range(200):
    q = qs[it % 4]
    i, e, _ = pkv.retrieve_topk(ix, q, k)
    outs.append(i)
torch.cuda.synchronize()
bad2 = [it for it, i in enumerate(outs) if not torch.equal(i, ref[it % 4])]
print(f"batch {batch} N {N}: fused mismatches {len(bad)} {bad[:8]}; topk-only mismatches {len(bad2)} {bad2[:8]}")
