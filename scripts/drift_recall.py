"""Config 4: streaming decode under key drift, Recall@k of the retrieval every step.

Workload: SPEC gen_drift — prefill keys ~ N(mu0, I), decode key t ~ N(mu0 + t*rate*delta, I), the
query of each step a noised copy of a recent retrieval-zone key, values N(0, I). The decode runs
through the library's four-region stream (pkv_stream_*: sink 16 / local 256 / update 512), so the
retrieval zone grows by flushes of encoded decode keys (append_decode_keys) exactly as in the paper.
Recall@k = |retrieved ∩ exact| / k against the exact top-k of <k_i, q> over the indexed retrieval zone
(fp64 GEMV). The paper's drift claim (SPEC acceptance 5): with analytic
centroids the recall under drift stays close to the no-drift recall.

    python scripts/drift_recall.py [--prefill 32768] [--decode 32768] [--rates 0,0.0005,0.002] [--out f.json]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402


def run(prefill: int, decode: int, rate: float, top_k: int = 100, seed: int = 4, sink: int = 16, local: int = 256,
        update: int = 512, recent: int = 1024, window: int | None = None) -> dict:
    from paper_2602_07721_b200 import build
    build.build()
    from paper_2602_07721_b200 import pariskv as pkv
    dev = torch.device("cuda", 0)
    Kall, _ = synth.drift_keys(seed, prefill, decode, rate, device=dev)
    Vall = synth.isotropic(seed + 1, (prefill + decode, 128), device=dev)
    K = Kall.view(1, 1, -1, 128)
    V = Vall.view(1, 1, -1, 128)
    cfg = pkv.config_init(1, 1, synth.rotation_sign_bits())
    ix = pkv.Index(cfg, 1, prefill + decode)
    st = pkv.Stream(ix, sink=sink, local_size=local, update_size=update)
    st.prefill(K[:, :, :prefill].contiguous(), V[:, :, :prefill].contiguous())
    g = torch.Generator(device=dev)
    g.manual_seed(seed + 2)
    Kr64 = Kall[sink:].double()  # retrieval zone rows in token order (store position i = token sink + i)
    rec = []
    t0 = time.time()
    for s in range(decode):
        t = prefill + s
        n_r = st.state()[0]
        lo = max(0, n_r - recent)
        i = int(torch.randint(lo, n_r, (1,), generator=g, device=dev))
        z = torch.randn(128, generator=g, device=dev)
        q = (Kall[sink + i].float() + 0.3 * z).to(torch.bfloat16).view(1, 1, 128)
        idx, _, _, _ = st.decode(q, K[:, :, t].contiguous(), V[:, :, t].contiguous(), top_k)
        n_r = st.state()[0]
        exact = torch.topk(Kr64[:n_r] @ q.view(128).double(), min(top_k, n_r)).indices
        got = idx.view(-1)
        got = got[got >= 0].long()
        rec.append(len(set(got.tolist()) & set(exact.tolist())) / float(min(top_k, n_r)))
    window = window or max(1, decode // 4)
    tail = rec[-window:]
    return {"prefill": prefill, "decode": decode, "rate": rate, "top_k": top_k, "flush": update,
            "recall_mean": sum(rec) / len(rec), "recall_last_window": sum(tail) / len(tail), "window": window,
            "recall_first_window": sum(rec[:window]) / window, "n_retrieval_final": st.state()[0],
            "seconds": round(time.time() - t0, 1)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--prefill", type=int, default=32768)
    ap.add_argument("--decode", type=int, default=32768)
    ap.add_argument("--rates", default="0,0.0005,0.002")
    ap.add_argument("--top-k", type=int, default=100)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    res = [run(args.prefill, args.decode, float(r), args.top_k) for r in args.rates.split(",")]
    base = res[0]["recall_last_window"] if res[0]["rate"] == 0 else None
    for r in res:
        r["retained_vs_no_drift"] = (r["recall_last_window"] / base) if base else None
        print(json.dumps(r))
    if args.out:
        with open(args.out, "w") as f:
            json.dump({"workload": "SPEC gen_drift through pkv_stream (sink 16, local 256, update 512)",
                       "runs": res}, f, indent=1)


if __name__ == "__main__":
    main()
