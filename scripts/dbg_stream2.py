import sys, os, torch
sys.path.insert(0, os.getcwd())
import synth
from paper_2602_07721_b200 import build
build.build()
from paper_2602_07721_b200 import pariskv as pkv
from tests.gpu_helpers import SB
mode = sys.argv[1]   # "none" | "before" | "after"
sink, L, U = 16, 64, 32
batch, n_q, n_kv, N, steps, k = 2, 8, 2, 2500, 140, 50
stats = synth.head_stats(31, n_kv, device="cuda")
K = synth.llm_keys(31, batch, n_kv, N + steps, device="cuda", stats=stats)
V = synth.values(31, batch, n_kv, N + steps, device="cuda")
qs = [synth.llm_queries(31 + 1 + s, batch, n_q, n_kv, device="cuda", stats=stats) for s in range(4)]
cfg = pkv.config_init(n_q, n_kv, SB)
ix = pkv.Index(cfg, batch, N + steps)
st = pkv.Stream(ix, sink=sink, local_size=L, update_size=U)
st.prefill(K[:, :, :N].contiguous(), V[:, :, :N].contiguous())
bad = []
for s in range(steps):
    t = N + s
    q = qs[s % 4]
    if mode == "before": torch.cuda.synchronize()
    idx, est, out, lse = st.decode(q, K[:, :, t].contiguous(), V[:, :, t].contiguous(), k)
    if mode == "after": torch.cuda.synchronize()
    if (s + 1) % U == 0:
        Ks, Vs, Kh, Vh = st.views()
        n_r, n_local, n_buf = st.state()
        n_hot = sink + n_local + n_buf
        i3, e3, o3, l3 = pkv.retrieve_and_attend(ix, q, Ks[:, :, :n_r], Vs[:, :, :n_r], k,
                                                 Kh[:, :, :n_hot].contiguous(), Vh[:, :, :n_hot].contiguous())
        i2, e2, _ = pkv.retrieve_topk(ix, q, k)
        if not torch.equal(i2, idx):
            bad.append((s, torch.equal(i3, idx), torch.equal(i3, i2)))
print(mode, "PDL", os.environ.get("PKV_NO_PDL"), "bad flush steps:", bad)
# isolate: the strided-hot call (hot_rows = R) vs the contiguous-hot call on the same final state
import ctypes, numpy as np
Ks, Vs, Kh, Vh = st.views()
n_r, n_local, n_buf = st.state()
R = sink + L + U
res = []
for n_hot in (sink + n_local + n_buf, 80, 100, R):
    for qi in range(4):
        q = qs[qi]
        i2, e2, _ = pkv.retrieve_topk(ix, q, k)
        oi = torch.empty_like(i2); oe = torch.empty_like(e2)
        out = torch.empty(batch, n_q, 128, dtype=torch.bfloat16, device="cuda"); lse = torch.empty(batch, n_q, device="cuda")
        T, C = pkv.schedule(n_r, k)
        p = pkv.RetrieveParams(T, C, k, None, None, None, None)
        st_ = (n_kv * ix.capacity * 128, ix.capacity * 128, 128)
        pkv._check(pkv._lib.retrieve_and_attend_rows(ix.handle, pkv._ptr(q), ctypes.byref(p), pkv._vp(Ks.data_ptr()), pkv._vp(Vs.data_ptr()), *st_,
                   pkv._vp(Kh.data_ptr()), pkv._vp(Vh.data_ptr()), n_hot, R, 1 / np.sqrt(128), pkv._ptr(oi), pkv._ptr(oe), pkv._ptr(out), pkv._ptr(lse), pkv._stream()))
        res.append((n_hot, qi, torch.equal(oi, i2)))
print("strided hot vs topk:", [r for r in res if not r[2]], "of", len(res))
