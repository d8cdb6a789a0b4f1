"""-m gpu: the streaming four-region KV cache (PAPER §4.2.3 "Buffer Update"; include/pariskv.h
pkv_stream_*) against a plain model of the regions and against the oracle.

After every decode step the stream must hold: Sink = tokens [0, sink); Retrieval = tokens [sink, sink + n_r)
indexed exactly as a fresh encode_keys of those tokens would index them (bit-exact) with their K/V in the
store; Local U Update = the remaining newest tokens in the hot buffer. Its decode output must equal
retrieve_and_attend over those regions, and the retrieval must match the oracle (AMB-15/16/17)."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import synth
from oracle import pipeline
from tests.gpu_helpers import (ATT_ABS, SB, bf16_f64, check_attention, check_encode, check_topk, oracle_meta,
                               oracle_retrieval)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkv():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2602_07721_b200 import build
    build.build()
    from paper_2602_07721_b200 import pariskv
    return pariskv


def region_model(n_prefill, steps, sink, L, U):
    """Plain restatement of P:456-463: (n_retrieval, n_local, n_buffer) after each decode step."""
    n_local = min(L, n_prefill - sink)
    n_r = n_prefill - sink - n_local
    n_buf = 0
    out = []
    for _ in range(steps):
        n_buf += 1
        if n_buf == U:
            evict = max(0, n_local + n_buf - L)
            n_r += evict
            n_local = n_local + n_buf - evict
            n_buf = 0
        out.append((n_r, n_local, n_buf))
    return out


def make_tokens(seed, batch, n_q, n_kv, n_tok):
    stats = synth.head_stats(seed, n_kv, device="cuda")
    K = synth.llm_keys(seed, batch, n_kv, n_tok, device="cuda", stats=stats)
    V = synth.values(seed, batch, n_kv, n_tok, device="cuda")
    qs = [synth.llm_queries(seed + 1 + s, batch, n_q, n_kv, device="cuda", stats=stats) for s in range(4)]
    return K, V, qs


@pytest.mark.parametrize("sink,L,U,offload", [(16, 64, 32, False), (16, 32, 64, False), (4, 48, 40, True)])
def test_stream_regions_and_outputs(pkv, sink, L, U, offload):
    batch, n_q, n_kv, N, steps, k = 2, 8, 2, 2500, 140, 50
    K, V, qs = make_tokens(31, batch, n_q, n_kv, N + steps)
    cfg = pkv.config_init(n_q, n_kv, SB)
    ix = pkv.Index(cfg, batch, N + steps)
    st = pkv.Stream(ix, sink=sink, local_size=L, update_size=U, offload_host=offload)
    st.prefill(K[:, :, :N].contiguous(), V[:, :, :N].contiguous())
    model = region_model(N, steps, sink, L, U)
    ref = pkv.Index(cfg, batch, N + steps)
    out32 = torch.full((batch, n_q, 128), float("nan"), device="cuda")
    ix.set_debug_output(out32)
    for s in range(steps):
        t = N + s  # token generated at this step
        q = qs[s % 4]
        idx, est, out, lse = st.decode(q, K[:, :, t].contiguous(), V[:, :, t].contiguous(), k)
        assert st.state() == model[s], (s, st.state(), model[s])
        n_r, n_local, n_buf = model[s]
        flushed = s > 0 and model[s][0] != model[s - 1][0]
        if not (flushed or s in (0, steps - 1)):
            continue
        torch.cuda.synchronize()
        Kr = K[:, :, sink:sink + n_r].contiguous()
        Vr = V[:, :, sink:sink + n_r].contiguous()
        Ks, Vs, Kh, Vh = st.views()
        assert torch.equal(Ks[:, :, :n_r], Kr) and torch.equal(Vs[:, :, :n_r], Vr), "retrieval store"
        hot_tok = list(range(sink)) + list(range(sink + n_r, t + 1))
        n_hot = len(hot_tok)
        assert n_hot == sink + n_local + n_buf
        Kx = K[:, :, hot_tok].contiguous()
        Vx = V[:, :, hot_tok].contiguous()
        assert torch.equal(Kh[:, :, :n_hot], Kx) and torch.equal(Vh[:, :, :n_hot], Vx), "hot rows"
        # the appended index equals a fresh prefill encode of the retrieval zone (bit-exact)
        pkv.encode_keys(ref, Kr)
        for a, b in zip(ix.export(), ref.export()):
            assert torch.equal(a, b), "index metadata"
        # the decode output: Eq. 2-3 of the oracle over Sink U Local U Update U its retrieved rows (AMB-17)
        o32 = out32.cpu().numpy()
        for b in range(batch):
            for h in range(n_q):
                g = h // (n_q // n_kv)
                o, l = pipeline.attend(bf16_f64(q[b, h]), bf16_f64(Kr[b, g]), bf16_f64(Vr[b, g]),
                                       idx[b, h].cpu().numpy(), bf16_f64(Kx[b, g]), bf16_f64(Vx[b, g]))
                check_attention(out[b, h].float().cpu().numpy(), o, o32[b, h], lse[b, h], l, f"step {s} b{b} h{h}")
        # and its retrieval equals retrieve_and_attend over the same regions (bit-exact ids and estimates)
        i1, e1, o1, l1 = pkv.retrieve_and_attend(ref, q, Kr, Vr, k, Kx, Vx)
        i2, e2, _ = pkv.retrieve_topk(ix, q, k)
        bad = (i1 != idx).any(-1)
        assert torch.equal(i1, idx) and torch.equal(e1, est), (
            f"retrieval: step {s} n_r {n_r} heads {bad.nonzero().tolist()} stream-vs-topk "
            f"{torch.equal(i2, idx)} ref-vs-topk {torch.equal(i2, i1)} est {(e1 - est).abs().max().item()}")


def test_stream_decode_matches_oracle(pkv):
    """One decode step after two flushes, checked against the oracle: retrieval over the indexed zone and
    attention over Sink U Local U Update U retrieved rows (GPU's own index set, AMB-17)."""
    batch, n_q, n_kv, N, steps, k = 1, 4, 1, 3000, 130, 64
    sink, L, U = 16, 64, 64
    K, V, qs = make_tokens(47, batch, n_q, n_kv, N + steps)
    synth.plant(K[:, :, :N], qs[0], 47)
    cfg = pkv.config_init(n_q, n_kv, SB)
    ix = pkv.Index(cfg, batch, N + steps)
    st = pkv.Stream(ix, sink=sink, local_size=L, update_size=U)
    st.prefill(K[:, :, :N].contiguous(), V[:, :, :N].contiguous())
    for s in range(steps):
        idx, est, out, lse = st.decode(qs[0], K[:, :, N + s].contiguous(), V[:, :, N + s].contiguous(), k)
    torch.cuda.synchronize()
    n_r, n_local, n_buf = st.state()
    assert (n_r, n_local, n_buf) == region_model(N, steps, sink, L, U)[-1]
    Kr = bf16_f64(K[0, 0, sink:sink + n_r])
    meta = oracle_meta(Kr)
    ids_g, codes_g, w_g = [t.cpu().numpy() for t in ix.export()]
    check_encode(ids_g[0, 0], codes_g[0, 0], w_g[0, 0], meta)
    T, C = pkv.schedule(n_r, k)
    hot_tok = list(range(sink)) + list(range(sink + n_r, N + steps))
    for h in range(n_q):
        qf = bf16_f64(qs[0][0, h])
        r = oracle_retrieval(meta, qf, T, C, k)
        check_topk(idx[0, h].cpu().numpy(), est[0, h].cpu().numpy(), r["cand"], r["est"],
                   dict(zip(range(n_r), meta["knorm"].tolist())), r["qnorm"], k)
        o, l = pipeline.attend(qf, Kr, bf16_f64(V[0, 0, sink:sink + n_r]), idx[0, h].cpu().numpy(),
                               bf16_f64(K[0, 0, hot_tok]), bf16_f64(V[0, 0, hot_tok]))
        og = out[0, h].float().cpu().numpy()
        assert np.all(np.abs(og - o) <= ATT_ABS + 2.0 ** -8 * np.abs(o)), f"attn err {np.max(np.abs(og - o))}"
        assert abs(float(lse[0, h]) - l) <= 1e-3 * max(1.0, abs(l))


def test_stream_capacity_and_args(pkv):
    cfg = pkv.config_init(4, 1, SB)
    K, V, qs = make_tokens(5, 1, 4, 1, 400)
    ix = pkv.Index(cfg, 1, 300)
    with pytest.raises(pkv.PkvError):
        pkv.Stream(ix, sink=16, local_size=512, update_size=512)  # > 1024 hot rows
    st = pkv.Stream(ix, sink=16, local_size=32, update_size=8)
    with pytest.raises(pkv.PkvError):
        st.decode(qs[0], K[:, :, 0].contiguous(), V[:, :, 0].contiguous(), 16)  # before prefill
    with pytest.raises(pkv.PkvError):
        st.prefill(K[:, :, :8].contiguous(), V[:, :, :8].contiguous())  # shorter than the sink
    st.prefill(K[:, :, :340].contiguous(), V[:, :, :340].contiguous())  # 292 retrieval tokens of 300
    assert st.state() == (292, 32, 0)
    t = 340
    for _ in range(8):  # the 8th token flushes 8 rows: 292 + 8 = 300 fits exactly
        st.decode(qs[0], K[:, :, t].contiguous(), V[:, :, t].contiguous(), 16)
        t += 1
    assert st.state() == (300, 32, 0)
    for _ in range(7):
        st.decode(qs[0], K[:, :, t].contiguous(), V[:, :, t].contiguous(), 16)
        t += 1
    assert st.state() == (300, 32, 7)
    with pytest.raises(pkv.PkvError) as e:  # this flush would need 308 > 300 rows: refused, nothing changes
        st.decode(qs[0], K[:, :, t].contiguous(), V[:, :, t].contiguous(), 16)
    assert e.value.status == pkv.PKV_ERR_CAPACITY
    assert st.state() == (300, 32, 7)


@pytest.mark.parametrize("n_prompt", [16, 50, 80])
def test_stream_short_prompt_empty_retrieval_zone(pkv, n_prompt):
    """A prompt of at most sink + local_size tokens leaves the retrieval zone empty until the first flush: those
    steps attend the hot rows alone (ids -1, estimates -inf), later steps retrieve; every output against the
    oracle (Eq. 2-3 over all tokens so far while nothing is evicted). A refused call changes nothing."""
    batch, n_q, n_kv, k = 1, 4, 1, 16
    sink, L, U = 16, 64, 32
    steps = 130
    K, V, qs = make_tokens(71 + n_prompt, batch, n_q, n_kv, n_prompt + steps)
    cfg = pkv.config_init(n_q, n_kv, SB)
    ix = pkv.Index(cfg, batch, n_prompt + steps)
    st = pkv.Stream(ix, sink=sink, local_size=L, update_size=U)
    st.prefill(K[:, :, :n_prompt].contiguous(), V[:, :, :n_prompt].contiguous())
    assert st.state() == (0, n_prompt - sink, 0)
    model = region_model(n_prompt, steps, sink, L, U)
    out32 = torch.full((batch, n_q, 128), float("nan"), device="cuda")
    ix.set_debug_output(out32)
    for s in range(steps):
        t = n_prompt + s
        kn, vn = K[:, :, t].contiguous(), V[:, :, t].contiguous()
        if s == 3:  # invalid top_k: refused before any state change
            with pytest.raises(pkv.PkvError) as e:
                st.decode(qs[0], kn, vn, 0)
            assert e.value.status == pkv.PKV_ERR_INVALID_ARG and st.state() == model[s - 1]
        idx, est, out, lse = st.decode(qs[s % 4], kn, vn, k)
        assert st.state() == model[s]
        n_r = model[s][0]
        torch.cuda.synchronize()
        hot_tok = list(range(sink)) + list(range(sink + n_r, t + 1))
        for h in range(n_q):
            qf = bf16_f64(qs[s % 4][0, h])
            ig = idx[0, h].cpu().numpy()
            if n_r == 0:
                assert np.all(ig == -1) and np.all(np.isneginf(est[0, h].cpu().numpy()))
            o, l = pipeline.attend(qf, bf16_f64(K[0, 0, sink:sink + n_r]), bf16_f64(V[0, 0, sink:sink + n_r]), ig,
                                   bf16_f64(K[0, 0, hot_tok]), bf16_f64(V[0, 0, hot_tok]))
            check_attention(out[0, h].float().cpu().numpy(), o, out32[0, h].cpu().numpy(), lse[0, h], l,
                            f"step {s} h{h}")
    assert model[-1][0] > 0  # the run crossed at least one flush
