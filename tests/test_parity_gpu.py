"""-m gpu parity: the CUDA path (through the C ABI) against the CPU oracle on the same seeded inputs.

Bars: centroid ids, 4-bit codes, collision scores and candidate sets bit-exact;
weights 1e-5 relative; RSQ-IP estimates within the AMB-15 form of 1e-3 relative; top-k equal up to
estimate ties (AMB-16); attention within 2e-3 absolute + one bf16 rounding, on the GPU's own index set."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import synth
from oracle import attention, coarse, pipeline, rerank, sharded
from tests.gpu_helpers import (ATT_ABS, SB, bf16_f64, check_attention, check_encode, check_topk, oracle_meta,
                               oracle_retrieval, w16_bound)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkv():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2602_07721_b200 import build
    build.build()
    from paper_2602_07721_b200 import pariskv
    return pariskv


def make_problem(seed, batch, n_q, n_kv, n, plant=True, device="cuda"):
    stats = synth.head_stats(seed, n_kv, device=device)
    K = synth.llm_keys(seed, batch, n_kv, n, device=device, stats=stats)
    q = synth.llm_queries(seed, batch, n_q, n_kv, device=device, stats=stats)
    if plant and n >= 4 * 25 * (n_q // n_kv):
        synth.plant(K, q, seed)
    V = synth.values(seed, batch, n_kv, n, device=device)
    return K, q, V


def run_and_check(pkv, K, q, V, k, T=None, C=None, n_hot=0, check_all_heads=True, cfg=None):
    batch, n_kv, n, _ = K.shape
    n_q = q.shape[1]
    G = n_q // n_kv
    cfg = cfg or pkv.config_init(n_q, n_kv, SB)
    ix = pkv.Index(cfg, batch, max(n, 1))
    pkv.encode_keys(ix, K)
    idx, est, dbg = pkv.retrieve_topk(ix, q, k, probes_T=T, n_cand=C, debug=True)
    Kh = Vh = None
    if n_hot:
        Kh = synth.isotropic(91, (batch, n_kv, n_hot, 128), device="cuda")
        Vh = synth.isotropic(92, (batch, n_kv, n_hot, 128), device="cuda")
    out32 = torch.full((batch, n_q, 128), float("nan"), device="cuda")
    ix.set_debug_output(out32)
    out, lse = pkv.sparse_attend(ix, q, K, V, idx, Kh, Vh)
    ix.set_debug_output(None)
    ids_g, codes_g, w_g = [t.cpu().numpy() for t in ix.export()]
    torch.cuda.synchronize()
    Tn, Cn = dbg["T"], dbg["C"]
    w16 = bool(cfg.w_fp16)
    for b in range(batch):
        for g in range(n_kv):
            Kf = bf16_f64(K[b, g])
            meta = oracle_meta(Kf)
            check_encode(ids_g[b, g], codes_g[b, g], w_g[b, g], meta, w16=w16)
            for hh in range(G):
                h = g * G + hh
                if not check_all_heads and hh > 0:
                    continue
                qf = bf16_f64(q[b, h])
                r = oracle_retrieval(meta, qf, Tn, Cn, k)
                assert np.array_equal(dbg["scores"][b, h].cpu().numpy().astype(np.int64), r["score"]), "scores"
                cg = dbg["cand"][b, h].cpu().numpy()
                assert np.array_equal(np.sort(cg[cg >= 0]), r["cand"]), "candidate set"
                assert np.allclose(dbg["q_rot"][b, h].cpu().numpy(), r["qt"], atol=2e-6)
                # estimates, aligned by id
                eg = dict(zip(cg.tolist(), dbg["est"][b, h].cpu().numpy().tolist()))
                eo = r["est"]
                kn = meta["knorm"][r["cand"]]
                tol = 1e-3 * np.maximum(np.abs(eo), 1e-2 * kn * r["qnorm"])
                extra = None
                if w16:
                    xb = w16_bound(meta, r["cand"], r["qt"], r["qnorm"])
                    tol = tol + xb
                    extra = dict(zip(r["cand"].tolist(), xb.tolist()))
                egv = np.array([eg[int(i)] for i in r["cand"]])
                assert np.all(np.abs(egv - eo) <= tol), f"est max err {np.max(np.abs(egv - eo) / tol)} x tol"
                check_topk(idx[b, h].cpu().numpy(), est[b, h].cpu().numpy(), r["cand"], eo,
                           dict(zip(range(n), meta["knorm"].tolist())), r["qnorm"], k, extra_by_id=extra)
                # attention on the GPU's own index set (AMB-17)
                ig = idx[b, h].cpu().numpy()
                o, l = pipeline.attend(qf, Kf, bf16_f64(V[b, g]), ig,
                                       None if Kh is None else bf16_f64(Kh[b, g]),
                                       None if Vh is None else bf16_f64(Vh[b, g]))
                check_attention(out[b, h].float().cpu().numpy(), o, out32[b, h].cpu().numpy(), lse[b, h], l)
    return ix, idx, est, dbg


def test_config1_single_head_4096(pkv):
    """BASELINE config 1: 1 head, d=128, N=4096, 1 query, top-k=64, paper defaults."""
    K, q, V = make_problem(1, 1, 1, 1, 4096, plant=False)
    synth.plant(K, q, 1, n_plant=25)
    run_and_check(pkv, K, q, V, k=64)


def test_gqa_batch_ragged(pkv):
    K, q, V = make_problem(2, 2, 8, 2, 5003)
    run_and_check(pkv, K, q, V, k=100, n_hot=37)


def test_gqa_group_of_3(pkv):
    """G = 3 query heads per KV head: the packed bonus word's 4th byte (no head) stays 0 in the scan."""
    K, q, V = make_problem(5, 1, 6, 2, 3000)
    run_and_check(pkv, K, q, V, k=64, n_hot=20)


def test_llama_shape_small_n(pkv):
    K, q, V = make_problem(3, 1, 32, 8, 3001)
    run_and_check(pkv, K, q, V, k=100, n_hot=272, check_all_heads=False)


@pytest.mark.parametrize("n", [1, 7, 33, 50, 99, 100, 129, 2049])
def test_tiny_and_ragged_lengths(pkv, n):
    K, q, V = make_problem(4 + n, 1, 4, 2, n, plant=False)
    run_and_check(pkv, K, q, V, k=64)


def test_group_size_two_and_one(pkv):
    K, q, V = make_problem(5, 1, 4, 2, 3000, plant=False)
    run_and_check(pkv, K, q, V, k=32)
    K, q, V = make_problem(6, 1, 3, 3, 3000, plant=False)
    run_and_check(pkv, K, q, V, k=32)


@pytest.mark.parametrize("T,C", [(1, 100), (256, 900), (26, 3000), (7, 64)])
def test_probe_and_candidate_extremes(pkv, T, C):
    K, q, V = make_problem(7, 1, 4, 1, 3000, plant=False)
    run_and_check(pkv, K, q, V, k=64, T=T, C=C)


def test_single_tier_many_ties(pkv):
    K, q, V = make_problem(8, 1, 4, 1, 6000, plant=False)
    cfg = pkv.config_init(4, 1, SB)
    cfg.n_tiers = 1
    cfg.tier_bonus[0] = 1
    for i in range(1, 8):
        cfg.tier_bonus[i] = 0
    ix = pkv.Index(cfg, 1, 6000)
    pkv.encode_keys(ix, K)
    T, C = 26, 500
    idx, est, dbg = pkv.retrieve_topk(ix, q, 64, probes_T=T, n_cand=C, debug=True)
    meta = oracle_meta(bf16_f64(K[0, 0]))
    for h in range(4):
        qf = bf16_f64(q[0, h])
        bonus = coarse.query_bonus_tables(qf, SB, T, tier_bonus=(1,))
        sc = coarse.collision_scores(meta["ids"], bonus)
        assert sc.max() <= 16
        assert np.array_equal(dbg["scores"][0, h].cpu().numpy().astype(np.int64), sc)
        cg = dbg["cand"][0, h].cpu().numpy()
        assert np.array_equal(np.sort(cg), coarse.bucket_topk(sc, C))


def test_degenerate_and_wide_range_keys(pkv):
    """Zero keys, zero subspaces (AMB-7) and keys spanning > 16 binades (fp64 butterfly fallback)."""
    K, q, V = make_problem(9, 1, 4, 1, 2048, plant=False)
    K[0, 0, 5] = 0
    K[0, 0, 6, 16:24] = 0
    K[0, 0, 7, :64] = 0
    K[0, 0, 10:40, 3] = 1e-9
    K[0, 0, 40:60, 100] = 3e-30
    K[0, 0, 60:70, :] = torch.randn(10, 128, device="cuda").to(torch.bfloat16) * 1e-20
    K[0, 0, 70] = -0.0
    run_and_check(pkv, K, q, V, k=64)


def test_wide_range_queries(pkv):
    """Queries spanning > 27 binades: the fp64 centroid scores lose their 8 trailing zero bits, so the query prep
    ranks with the (key, id) pair network instead of the packed 64-bit composite; one head per path."""
    K, q, V = make_problem(19, 1, 4, 1, 3000, plant=False)
    q[0, 0, :64] = q[0, 0, :64] * 1e-10   # 2^-33 next to O(1) values: after the rotation every subspace mixes them
    q[0, 1, 1::2] = q[0, 1, 1::2] * 1e-12
    run_and_check(pkv, K, q, V, k=64)


def test_append_equals_prefill(pkv):
    K, q, V = make_problem(10, 1, 8, 2, 4000)
    cfg = pkv.config_init(8, 2, SB)
    a = pkv.Index(cfg, 1, 4000)
    pkv.encode_keys(a, K)
    b = pkv.Index(cfg, 1, 4000)
    pkv.encode_keys(b, K[:, :, :1000])
    for t0 in range(1000, 4000, 512):
        pkv.append_decode_keys(b, K[:, :, t0:t0 + 512])
    assert len(b) == 4000
    for x, y in zip(a.export(), b.export()):
        assert torch.equal(x, y)
    ia, ea, _ = pkv.retrieve_topk(a, q, 100)
    ib, eb, _ = pkv.retrieve_topk(b, q, 100)
    assert torch.equal(ia, ib) and torch.equal(ea, eb)
    with pytest.raises(pkv.PkvError) as e:
        pkv.append_decode_keys(b, K[:, :, :1])
    assert e.value.status == pkv.PKV_ERR_CAPACITY
    assert len(b) == 4000


def test_strided_kv_layout(pkv):
    """K as a [batch, tokens, n_kv, D] tensor viewed as [batch, n_kv, tokens, D] (non-contiguous strides)."""
    K, q, V = make_problem(11, 1, 8, 2, 3000)
    Kt = K.transpose(1, 2).contiguous().transpose(1, 2)
    Vt = V.transpose(1, 2).contiguous().transpose(1, 2)
    assert not Kt.is_contiguous()
    cfg = pkv.config_init(8, 2, SB)
    a = pkv.Index(cfg, 1, 3000)
    pkv.encode_keys(a, K)
    b = pkv.Index(cfg, 1, 3000)
    pkv.encode_keys(b, Kt)
    for x, y in zip(a.export(), b.export()):
        assert torch.equal(x, y)
    idx, _, _ = pkv.retrieve_topk(a, q, 100)
    o1, l1 = pkv.sparse_attend(a, q, K, V, idx)
    o2, l2 = pkv.sparse_attend(b, q, Kt, Vt, idx)
    assert torch.equal(o1, o2) and torch.equal(l1, l2)


def test_attention_hot_only_and_invalid_args(pkv):
    K, q, V = make_problem(12, 1, 8, 2, 500, plant=False)
    cfg = pkv.config_init(8, 2, SB)
    ix = pkv.Index(cfg, 1, 500)
    pkv.encode_keys(ix, K)
    Kh, Vh = K[:, :, :300].contiguous(), V[:, :, :300].contiguous()
    out, lse = pkv.sparse_attend(ix, q, None, None, None, Kh, Vh)
    for h in range(8):
        o, l = attention.full_attention(bf16_f64(q[0, h]), bf16_f64(Kh[0, h // 4]), bf16_f64(Vh[0, h // 4]),
                                        1 / np.sqrt(128))
        assert np.all(np.abs(out[0, h].float().cpu().numpy() - o) <= ATT_ABS + 2.0 ** -8 * np.abs(o))
    with pytest.raises(pkv.PkvError):
        pkv.sparse_attend(ix, q, None, None, None, None, None)
    with pytest.raises(pkv.PkvError):
        pkv.retrieve_topk(ix, q, 100, n_cand=10)          # C < min(k, n)
    with pytest.raises(pkv.PkvError):
        pkv.retrieve_topk(ix, q, 100, probes_T=0)
    empty = pkv.Index(cfg, 1, 16)
    with pytest.raises(pkv.PkvError):
        pkv.retrieve_topk(empty, q, 10)


def test_uva_pinned_host_kv(pkv):
    """a7 with K/V in pinned host memory read through UVA equals the HBM result."""
    K, q, V = make_problem(13, 1, 8, 2, 4096)
    cfg = pkv.config_init(8, 2, SB)
    ix = pkv.Index(cfg, 1, 4096)
    pkv.encode_keys(ix, K)
    idx, _, _ = pkv.retrieve_topk(ix, q, 100)
    Kh = K.cpu().pin_memory()
    Vh = V.cpu().pin_memory()
    o1, l1 = pkv.sparse_attend(ix, q, K, V, idx)
    o2, l2 = pkv.sparse_attend(ix, q, None, None, idx, K_ptr=Kh.data_ptr(), V_ptr=Vh.data_ptr(),
                               strides=(Kh.stride(0), Kh.stride(1), Kh.stride(2)))
    torch.cuda.synchronize()
    assert torch.equal(o1, o2) and torch.equal(l1, l2)


@pytest.mark.parametrize("P", [2, 3, 4])
def test_sequence_sharded_local_equals_unsharded(pkv, P):
    """§Multi-GPU decomposition on one device: P shards with the exchange buffers filled by device
    copies produce the unsharded result exactly (same kernels as the NCCL path)."""
    n = 6000
    K, q, V = make_problem(14, 1, 8, 2, n)
    cfg = pkv.config_init(8, 2, SB)
    full = pkv.Index(cfg, 1, n)
    pkv.encode_keys(full, K)
    i0, e0, _ = pkv.retrieve_topk(full, q, 100)
    Kh = synth.isotropic(93, (1, 2, 50, 128), device="cuda")
    Vh = synth.isotropic(94, (1, 2, 50, 128), device="cuda")
    o0, l0 = pkv.sparse_attend(full, q, K, V, i0, Kh, Vh)
    bounds = sharded.shard_ranges(n, P)
    shards, Ks, Vs = [], [], []
    for a, b in bounds:
        s = pkv.Index(cfg, 1, b - a)
        Ks.append(K[:, :, a:b].contiguous())
        Vs.append(V[:, :, a:b].contiguous())
        pkv.encode_keys(s, Ks[-1])
        shards.append(s)
    offs = [a for a, _ in bounds]
    i1, e1 = pkv.retrieve_topk_sharded_local(shards, offs, q, 100, n)
    assert torch.equal(i0, i1) and torch.equal(e0, e1)
    out32 = torch.full((1, 8, 128), float("nan"), device="cuda")
    shards[0].set_debug_output(out32)
    o1, l1 = pkv.sparse_attend_sharded_local(shards, offs, q, Ks, Vs, i1, Kh, Vh)
    torch.cuda.synchronize()
    # the sharded attention (per-shard partials + LSE merge) against the oracle's Eq. 2-3 over the same rows
    for h in range(8):
        g = h // 4
        o, l = pipeline.attend(bf16_f64(q[0, h]), bf16_f64(K[0, g]), bf16_f64(V[0, g]), i1[0, h].cpu().numpy(),
                               bf16_f64(Kh[0, g]), bf16_f64(Vh[0, g]))
        check_attention(o1[0, h].float().cpu().numpy(), o, out32[0, h].cpu().numpy(), l1[0, h], l, f"P={P} h={h}")
    # the emulation restores each shard's offset: an unsharded call on a shard returns its local ids again
    loc = pkv.Index(cfg, 1, bounds[-1][1] - bounds[-1][0])
    pkv.encode_keys(loc, Ks[-1])
    ia, ea, _ = pkv.retrieve_topk(loc, q, 100)
    ib, eb, _ = pkv.retrieve_topk(shards[-1], q, 100)
    assert torch.equal(ia, ib) and torch.equal(ea, eb)


@pytest.mark.slow
@pytest.mark.parametrize("P,n_hot", [(2, 272), (3, 0), (4, 40)])
def test_fused_exchange_sharded_local(pkv, P, n_hot):
    """the fused T+A exchange (one exchange per layer after the histogram one) gives the same
    top-k as the unsharded retrieval (bit-identical ids and estimates) and the same attention output."""
    batch, n_q, n_kv, n, k = 2, 8, 2, 9000, 100
    K, q, V = make_problem(61 + P, batch, n_q, n_kv, n)
    Kh = synth.isotropic(62, (batch, n_kv, max(n_hot, 1), 128), device="cuda")[:, :, :n_hot].contiguous()
    Vh = synth.isotropic(63, (batch, n_kv, max(n_hot, 1), 128), device="cuda")[:, :, :n_hot].contiguous()
    cfg = pkv.config_init(n_q, n_kv, SB)
    full = pkv.Index(cfg, batch, n)
    pkv.encode_keys(full, K)
    i0, e0, o0, l0 = pkv.retrieve_and_attend(full, q, K, V, k, Kh if n_hot else None, Vh if n_hot else None)
    bounds = [n * r // P for r in range(P + 1)]
    shards, Ks, Vs = [], [], []
    for r in range(P):
        lo, hi = bounds[r], bounds[r + 1]
        ix = pkv.Index(cfg, batch, hi - lo)
        pkv.encode_keys(ix, K[:, :, lo:hi].contiguous())
        shards.append(ix)
        Ks.append(K[:, :, lo:hi].contiguous())
        Vs.append(V[:, :, lo:hi].contiguous())
    out32 = torch.full((batch, n_q, 128), float("nan"), device="cuda")
    shards[0].set_debug_output(out32)
    i1, e1, o1, l1 = pkv.retrieve_and_attend_sharded_local(shards, bounds[:P], q, Ks, Vs, k,
                                                           Kh if n_hot else None, Vh if n_hot else None)
    torch.cuda.synchronize()
    assert torch.equal(i0, i1) and torch.equal(e0, e1)
    for b in range(batch):
        for h in range(n_q):
            g = h // (n_q // n_kv)
            o, l = pipeline.attend(bf16_f64(q[b, h]), bf16_f64(K[b, g]), bf16_f64(V[b, g]), i1[b, h].cpu().numpy(),
                                   bf16_f64(Kh[b, g]) if n_hot else None, bf16_f64(Vh[b, g]) if n_hot else None)
            check_attention(o1[b, h].float().cpu().numpy(), o, out32[b, h].cpu().numpy(), l1[b, h], l,
                            f"fused P={P} b={b} h={h}")


def test_full_size_128k_sampled_head(pkv):
    """BASELINE config 2 shape (32 q / 8 KV heads, n = 130,800) in the launch configuration bench.py times:
    one KV head (4 query heads) checked in full against the oracle, plus sampled keys of every head."""
    n = 130800
    K, q, V = make_problem(15, 1, 32, 8, n, device="cuda")
    cfg = pkv.config_init(32, 8, SB)
    ix = pkv.Index(cfg, 1, n)
    pkv.encode_keys(ix, K)
    idx, est, dbg = pkv.retrieve_topk(ix, q, 100, debug=True)
    out, lse = pkv.sparse_attend(ix, q, K, V, idx)
    ids_g, codes_g, w_g = [t.cpu().numpy() for t in ix.export()]
    rng = np.random.default_rng(0)
    for g in range(8):
        pos = rng.choice(n, 512, replace=False)
        meta = oracle_meta(bf16_f64(K[0, g, torch.as_tensor(pos, device="cuda")]))
        check_encode(ids_g[0, g, pos], codes_g[0, g, pos], w_g[0, g, pos], meta)
    g = 5
    Kf = bf16_f64(K[0, g])
    meta = oracle_meta(Kf)
    for hh in range(4):
        h = 4 * g + hh
        qf = bf16_f64(q[0, h])
        r = oracle_retrieval(meta, qf, dbg["T"], dbg["C"], 100)
        assert np.array_equal(dbg["scores"][0, h].cpu().numpy().astype(np.int64), r["score"])
        cg = dbg["cand"][0, h].cpu().numpy()
        assert np.array_equal(np.sort(cg), r["cand"])
        check_topk(idx[0, h].cpu().numpy(), est[0, h].cpu().numpy(), r["cand"], r["est"],
                   dict(zip(range(n), meta["knorm"].tolist())), r["qnorm"], 100)
        o, l = pipeline.attend(qf, Kf, bf16_f64(V[0, g]), idx[0, h].cpu().numpy())
        og = out[0, h].float().cpu().numpy()
        assert np.all(np.abs(og - o) <= ATT_ABS + 2.0 ** -8 * np.abs(o))


@pytest.mark.slow
def test_300k_warp_histograms_and_rerank_tile_loop(pkv):
    """n = 300,000 (Llama shape): the scan's warp segments exceed 512 keys, so the select takes its per-warp
    offsets from the scan's per-warp histograms, and C = 15,000 candidates per head make the rerank loop over
    tiles inside resident CTAs — the 1M code paths at a size the oracle checks in full for one KV head."""
    n = 300000
    K, q, V = make_problem(23, 1, 32, 8, n, device="cuda")
    cfg = pkv.config_init(32, 8, SB)
    ix = pkv.Index(cfg, 1, n)
    pkv.encode_keys(ix, K)
    idx, est, dbg = pkv.retrieve_topk(ix, q, 100, debug=True)
    assert (dbg["T"], dbg["C"]) == (21, 15000)
    out, lse = pkv.sparse_attend(ix, q, K, V, idx)
    g = 2
    Kf = bf16_f64(K[0, g])
    meta = oracle_meta(Kf)
    for hh in range(4):
        h = 4 * g + hh
        qf = bf16_f64(q[0, h])
        r = oracle_retrieval(meta, qf, dbg["T"], dbg["C"], 100)
        assert np.array_equal(dbg["scores"][0, h].cpu().numpy().astype(np.int64), r["score"])
        cg = dbg["cand"][0, h].cpu().numpy()
        assert np.array_equal(np.sort(cg), r["cand"])
        eg = dict(zip(cg.tolist(), dbg["est"][0, h].cpu().numpy().tolist()))
        egv = np.array([eg[int(i)] for i in r["cand"]])
        tol = 1e-3 * np.maximum(np.abs(r["est"]), 1e-2 * meta["knorm"][r["cand"]] * r["qnorm"])
        assert np.all(np.abs(egv - r["est"]) <= tol)
        check_topk(idx[0, h].cpu().numpy(), est[0, h].cpu().numpy(), r["cand"], r["est"],
                   dict(zip(range(n), meta["knorm"].tolist())), r["qnorm"], 100)
        o, l = pipeline.attend(qf, Kf, bf16_f64(V[0, g]), idx[0, h].cpu().numpy())
        og = out[0, h].float().cpu().numpy()
        assert np.all(np.abs(og - o) <= ATT_ABS + 2.0 ** -8 * np.abs(o))


def check_group_fused(pkv, K, q, V, Kh, Vh, idx, est, out, lse, b, g, T, C, k, dbg=None):
    """One (sequence, KV head) group of a fused retrieve_and_attend call against the oracle: retrieval of its
    query heads (AMB-15/16) and attention over hot rows U retrieved rows (AMB-17, GPU's own index set)."""
    G = q.shape[1] // K.shape[1]
    n = K.shape[2]
    Kf = bf16_f64(K[b, g])
    Vf = bf16_f64(V[b, g])
    meta = oracle_meta(Kf)
    for hh in range(G):
        h = G * g + hh
        qf = bf16_f64(q[b, h])
        r = oracle_retrieval(meta, qf, T, C, k)
        if dbg is not None:
            assert np.array_equal(dbg["scores"][b, h].cpu().numpy().astype(np.int64), r["score"])
            cg = dbg["cand"][b, h].cpu().numpy()
            assert np.array_equal(np.sort(cg), r["cand"])
        check_topk(idx[b, h].cpu().numpy(), est[b, h].cpu().numpy(), r["cand"], r["est"],
                   dict(zip(range(n), meta["knorm"].tolist())), r["qnorm"], k)
        o, l = pipeline.attend(qf, Kf, Vf, idx[b, h].cpu().numpy(), bf16_f64(Kh[b, g]), bf16_f64(Vh[b, g]))
        og = out[b, h].float().cpu().numpy()
        assert np.all(np.abs(og - o) <= ATT_ABS + 2.0 ** -8 * np.abs(o)), f"attn err {np.max(np.abs(og - o))}"
        assert abs(float(lse[b, h]) - l) <= 1e-3 * max(1.0, abs(l))


def test_full_size_32k_bs8_fused(pkv):
    """BASELINE config 3 (bs 8, 32K context = 32,496 retrieval + 272 hot rows per sequence, 32 q / 8 KV heads)
    through retrieve_and_attend, the call bench.py times: two (sequence, KV head) groups in full against the
    oracle, sampled key summaries of every sequence."""
    n, n_hot, k = 32768 - 272, 272, 100
    K, q, V = make_problem(41, 8, 32, 8, n)
    Kh = synth.isotropic(42, (8, 8, n_hot, 128), device="cuda")
    Vh = synth.isotropic(43, (8, 8, n_hot, 128), device="cuda")
    cfg = pkv.config_init(32, 8, SB)
    ix = pkv.Index(cfg, 8, n)
    pkv.encode_keys(ix, K)
    T, C = pkv.schedule(n, k)
    idx, est, out, lse = pkv.retrieve_and_attend(ix, q, K, V, k, Kh, Vh)
    ids_g, codes_g, w_g = [t.cpu().numpy() for t in ix.export()]
    rng = np.random.default_rng(1)
    for b in range(8):
        pos = rng.choice(n, 256, replace=False)
        meta = oracle_meta(bf16_f64(K[b, b % 8, torch.as_tensor(pos, device="cuda")]))
        check_encode(ids_g[b, b % 8, pos], codes_g[b, b % 8, pos], w_g[b, b % 8, pos], meta)
    for b, g in ((0, 3), (7, 6)):
        check_group_fused(pkv, K, q, V, Kh, Vh, idx, est, out, lse, b, g, T, C, k)


@pytest.mark.slow
def test_full_size_1m_uva_fused(pkv):
    """BASELINE config 5 on one GPU: 1,048,304 retrieval keys x 8 KV heads, K/V in pinned host memory read
    through UVA, the long-list (C = 52,416) cluster top-k; one KV group checked in full against the oracle."""
    n, n_hot, k = 1048576 - 272, 272, 100
    K, q, V = make_problem(51, 1, 32, 8, n)
    cfg = pkv.config_init(32, 8, SB)
    ix = pkv.Index(cfg, 1, n)
    pkv.encode_keys(ix, K)
    Kh = synth.isotropic(52, (1, 8, n_hot, 128), device="cuda")
    Vh = synth.isotropic(53, (1, 8, n_hot, 128), device="cuda")
    g = 2
    Kg, Vg = K[:, g:g + 1].contiguous(), V[:, g:g + 1].contiguous()
    Kc, Vc = K.cpu().pin_memory(), V.cpu().pin_memory()
    del K, V
    torch.cuda.empty_cache()
    T, C = pkv.schedule(n, k)
    sb, sh, st = Kc.stride(0), Kc.stride(1), Kc.stride(2)
    idx, est, out, lse = pkv.retrieve_and_attend(ix, q, None, None, k, Kh, Vh, K_ptr=Kc.data_ptr(),
                                                 V_ptr=Vc.data_ptr(), strides=(sb, sh, st))
    torch.cuda.synchronize()
    # the oracle sees the same group: KV head g as a 1-KV-head problem (its query heads are 4g .. 4g+3)
    check_group_fused(pkv, Kg, q[:, 4 * g:4 * g + 4].contiguous(), Vg, Kh[:, g:g + 1], Vh[:, g:g + 1],
                      idx[:, 4 * g:4 * g + 4], est[:, 4 * g:4 * g + 4], out[:, 4 * g:4 * g + 4],
                      lse[:, 4 * g:4 * g + 4], 0, 0, T, C, k)


@pytest.mark.parametrize("n,n_hot,k", [(4096, 272, 100), (777, 0, 64), (50, 16, 64), (20000, 300, 100)])
def test_retrieve_and_attend_matches_two_calls(pkv, n, n_hot, k):
    """The fused schedule (hot attention on a forked stream, top-k fused with gather+attention) returns the
    same ids/estimates as retrieve_topk and attention within the AMB-17 bar of the oracle."""
    K, q, V = make_problem(16 + n, 1, 8, 2, n, plant=n >= 200)
    cfg = pkv.config_init(8, 2, SB)
    ix = pkv.Index(cfg, 1, n)
    pkv.encode_keys(ix, K)
    Kh = Vh = None
    if n_hot:
        Kh = synth.isotropic(95, (1, 2, n_hot, 128), device="cuda")
        Vh = synth.isotropic(96, (1, 2, n_hot, 128), device="cuda")
    i0, e0, _ = pkv.retrieve_topk(ix, q, k)
    o0, l0 = pkv.sparse_attend(ix, q, K, V, i0, Kh, Vh)
    i1, e1, o1, l1 = pkv.retrieve_and_attend(ix, q, K, V, k, Kh, Vh)
    torch.cuda.synchronize()
    assert torch.equal(i0, i1) and torch.equal(e0, e1)
    assert torch.allclose(l0, l1, atol=1e-4, rtol=1e-5)
    for h in range(8):
        qf = bf16_f64(q[0, h])
        o, lse = pipeline.attend(qf, bf16_f64(K[0, h // 4]), bf16_f64(V[0, h // 4]), i1[0, h].cpu().numpy(),
                                 None if Kh is None else bf16_f64(Kh[0, h // 4]),
                                 None if Vh is None else bf16_f64(Vh[0, h // 4]))
        og = o1[0, h].float().cpu().numpy()
        assert np.all(np.abs(og - o) <= ATT_ABS + 2.0 ** -8 * np.abs(o))
        assert abs(float(l1[0, h]) - lse) <= 1e-3 * max(1.0, abs(lse))


@pytest.mark.parametrize("n,C", [(60000, 40000), (150000, 140000), (330000, 320000)])
def test_segmented_topk_long_candidate_list(pkv, n, C):
    """Long candidate lists (the 1M-token regime): C = 40000 takes the cluster top-k (several CTAs per head),
    C = 140000 and 320000 > 8 x 16384 the per-segment top-k (9 and 20 segment lists, more than the 8 rank slots
    round 1 sized them by) + merge. The newest key is planted as every head's best match, so it sits in the LAST
    segment; all must equal the oracle top-k up to ties, and retrieve_and_attend must take the same ids."""
    K, q, V = make_problem(17, 1, 4, 1, n)
    K[0, 0, n - 1] = (q[0, 0].float() * 16.0).to(torch.bfloat16)
    ix, idx, est, dbg = run_and_check(pkv, K, q, V, k=100, C=C, check_all_heads=False)
    assert int(idx[0, 0, 0]) == n - 1
    cfg = pkv.config_init(4, 1, SB)
    ix = pkv.Index(cfg, 1, n)
    pkv.encode_keys(ix, K)
    i0, e0, _ = pkv.retrieve_topk(ix, q, 100, n_cand=C)
    Kh = synth.isotropic(97, (1, 1, 40, 128), device="cuda")
    Vh = synth.isotropic(98, (1, 1, 40, 128), device="cuda")
    o0, l0 = pkv.sparse_attend(ix, q, K, V, i0, Kh, Vh)
    out32 = torch.full((1, 4, 128), float("nan"), device="cuda")
    ix.set_debug_output(out32)
    i1, e1, o1, l1 = pkv.retrieve_and_attend(ix, q, K, V, 100, Kh, Vh, n_cand=C)
    torch.cuda.synchronize()
    assert torch.equal(i0, i1) and torch.equal(e0, e1)
    for h in range(4):
        o, l = pipeline.attend(bf16_f64(q[0, h]), bf16_f64(K[0, 0]), bf16_f64(V[0, 0]), i1[0, h].cpu().numpy(),
                               bf16_f64(Kh[0, 0]), bf16_f64(Vh[0, 0]))
        check_attention(o1[0, h].float().cpu().numpy(), o, out32[0, h].cpu().numpy(), l1[0, h], l, f"seg h={h}")


def test_topk_massive_estimate_ties(pkv):
    """3000 identical keys near the query: their estimates tie exactly, so the top-k boundary bin overflows
    and the cluster top-k takes its exact radix fallback; ties resolve to the larger id."""
    K, q, V = make_problem(23, 1, 4, 1, 6000, plant=False)
    K[0, 0, 1000:4000] = (q[0, 0].float() * 3.0).to(torch.bfloat16)
    ix, idx, est, dbg = run_and_check(pkv, K, q, V, k=100, C=4500, check_all_heads=False)
    ig = idx[0, 0].cpu().numpy()
    dup = ig[(ig >= 1000) & (ig < 4000)]  # the tied duplicates taken: the newest ones, newest first
    assert len(dup) > 50 and np.array_equal(dup, np.arange(3999, 3999 - len(dup), -1)), ig[:10]
    Kh = synth.isotropic(97, (1, 1, 16, 128), device="cuda")
    Vh = synth.isotropic(98, (1, 1, 16, 128), device="cuda")
    i1, e1, o1, l1 = pkv.retrieve_and_attend(ix, q, K, V, 100, Kh, Vh, n_cand=4500)
    assert torch.equal(i1, idx) and torch.equal(e1, est)


def w16_cfg(pkv, n_q, n_kv):
    cfg = pkv.config_init(n_q, n_kv, SB)
    cfg.w_fp16 = 1
    return cfg


@pytest.mark.parametrize("case", ["config1", "gqa", "llama", "degenerate"])
def test_fp16_weights(pkv, case):
    """96-byte records with fp16 weights and a per-key exponent. Codes and candidate
    sets stay bit-exact; estimates within AMB-15 + the fp16 rounding bound; top-k equal up to those ties."""
    if case == "config1":
        K, q, V = make_problem(1, 1, 1, 1, 4096, plant=False)
        synth.plant(K, q, 1, n_plant=25)
        run_and_check(pkv, K, q, V, k=64, cfg=w16_cfg(pkv, 1, 1))
    elif case == "gqa":
        K, q, V = make_problem(2, 2, 8, 2, 5003)
        run_and_check(pkv, K, q, V, k=100, n_hot=37, cfg=w16_cfg(pkv, 8, 2))
    elif case == "llama":
        K, q, V = make_problem(3, 1, 32, 8, 3001)
        run_and_check(pkv, K, q, V, k=100, n_hot=272, check_all_heads=False, cfg=w16_cfg(pkv, 32, 8))
    else:
        K, q, V = make_problem(9, 1, 4, 1, 2048, plant=False)
        K[0, 0, 5] = 0
        K[0, 0, 6, 16:24] = 0
        K[0, 0, 10:40, 3] = 1e-9
        K[0, 0, 40:60, 100] = 3e-30
        K[0, 0, 60:70, :] = torch.randn(10, 128, device="cuda").to(torch.bfloat16) * 1e-20
        run_and_check(pkv, K, q, V, k=64, cfg=w16_cfg(pkv, 4, 1))


@pytest.mark.parametrize("n,k", [(3001, 64), (20000, 100), (130800, 100)])
def test_inverted_list_scan_equals_dense(pkv, n, k):
    """the inverted-list collision scan yields the dense scan's packed scores bit for bit, hence
    the same candidates, estimates and top-k; the postings follow appends."""
    K, q, V = make_problem(71, 1, 32, 8, n)
    cfg = pkv.config_init(32, 8, SB)
    a = pkv.Index(cfg, 1, n + 5000)
    pkv.encode_keys(a, K)
    b = pkv.Index(cfg, 1, n + 5000)
    pkv.encode_keys(b, K)
    b.set_postings(True)
    ia, ea, da = pkv.retrieve_topk(a, q, k, debug=True)
    ib, eb, db = pkv.retrieve_topk(b, q, k, debug=True)
    assert torch.equal(da["scores"], db["scores"])
    assert torch.equal(ia, ib) and torch.equal(ea, eb)
    # appends: the partial chunk and new chunks are rebuilt
    K2, _, _ = make_problem(72, 1, 32, 8, 3000)
    pkv.append_decode_keys(a, K2)
    pkv.append_decode_keys(b, K2)
    ia, ea, da = pkv.retrieve_topk(a, q, k, debug=True)
    ib, eb, db = pkv.retrieve_topk(b, q, k, debug=True)
    assert torch.equal(da["scores"], db["scores"]) and torch.equal(ia, ib)
    # and the oracle on one head of the dense-equal result (the dense path is itself oracle-checked)
    if n <= 20000:
        Kall = torch.cat([K, K2], dim=2)
        meta = oracle_meta(bf16_f64(Kall[0, 3]))
        r = oracle_retrieval(meta, bf16_f64(q[0, 13]), db["T"], db["C"], k)
        assert np.array_equal(db["scores"][0, 13].cpu().numpy().astype(np.int64), r["score"])


def test_tensor_core_encoder_bit_exact(pkv, monkeypatch):
    """The tcgen05 encoder variant (PKV_ENCODER=tc, encode_tc.cu): exact digit GEMMs for the rotation; ids and
    codes bit-exact against the oracle, including keys it must hand to the half-warp encoder (wide range, zero,
    subnormal) and partial tiles."""
    monkeypatch.setenv("PKV_ENCODER", "tc")
    K, q, V = make_problem(81, 2, 8, 2, 3000)
    K[0, 0, 5] = 0
    K[0, 0, 6, 16:24] = 0
    K[1, 1, 10:40, 3] = 1e-9
    K[1, 0, 40:60, 100] = 3e-30
    K[0, 1, 60:70, :] = torch.randn(10, 128, device="cuda").to(torch.bfloat16) * 1e-20
    run_and_check(pkv, K, q, V, k=64, n_hot=16)
    K, q, V = make_problem(82, 1, 4, 1, 333, plant=False)
    run_and_check(pkv, K, q, V, k=32, cfg=w16_cfg(pkv, 4, 1))


def test_gqa_union_rerank(pkv, monkeypatch):
    """SURVEY §8(f2) GQA dedupe (PKV_RERANK=union): the select emits, per KV head, the union of its query heads'
    candidate lists with every key's position in each list; the rerank reads each record once and scores it for
    all heads of the group. Same oracle checks as the per-head kernel (G = 4, 2, 1; fp32 and fp16 weights;
    ties in the s* bucket; hot rows)."""
    monkeypatch.setenv("PKV_RERANK", "union")
    K, q, V = make_problem(91, 2, 8, 2, 5000)
    run_and_check(pkv, K, q, V, k=64, n_hot=16)
    K, q, V = make_problem(92, 1, 4, 2, 3000, plant=False)
    run_and_check(pkv, K, q, V, k=32, T=26, C=900)
    K, q, V = make_problem(93, 1, 3, 3, 2000, plant=False)
    run_and_check(pkv, K, q, V, k=32)
    K, q, V = make_problem(94, 1, 8, 2, 4000)
    run_and_check(pkv, K, q, V, k=64, cfg=w16_cfg(pkv, 8, 2))


def test_degenerate_key_stats(pkv):
    """zero subspaces / zero keys are encoded deterministically and counted on the device;
    the counts equal the oracle's (S_b == 0 of its exact y'); encode_keys resets them, appends add."""
    K, q, V = make_problem(24, 2, 4, 2, 1500, plant=False)
    K[0, 0, 5] = 0
    K[1, 1, 6] = 0
    K[0, 1, 7, 16:24] = 0
    K[1, 0, 9, :64] = 0
    K[0, 0, 30:40, 100:108] = 0
    cfg = pkv.config_init(4, 2, SB)
    ix = pkv.Index(cfg, 2, 3000)

    def oracle_counts(Kt):
        zk = kz = zs = 0
        for b in range(Kt.shape[0]):
            for g in range(Kt.shape[1]):
                S = oracle_meta(bf16_f64(Kt[b, g]))["S"]
                z = S == 0
                zk += int(np.sum(z.all(axis=1)))
                kz += int(np.sum(z.any(axis=1)))
                zs += int(np.sum(z))
        return zk, kz, zs

    pkv.encode_keys(ix, K)
    st = ix.stats()
    assert (st["zero_keys"], st["keys_with_zero_subspace"], st["zero_subspaces"]) == oracle_counts(K)
    assert st["zero_keys"] == 2 and st["n_keys"] == 1500
    K2 = K[:, :, :700].clone()
    K2[0, 0, 3] = 0
    pkv.append_decode_keys(ix, K2)
    st = ix.stats()
    a, b = oracle_counts(K), oracle_counts(K2)
    assert (st["zero_keys"], st["keys_with_zero_subspace"], st["zero_subspaces"]) == tuple(x + y for x, y in zip(a, b))
    pkv.encode_keys(ix, K[:, :, 10:])  # replaces the content: counts restart
    st = ix.stats()
    assert (st["zero_keys"], st["keys_with_zero_subspace"], st["zero_subspaces"]) == oracle_counts(K[:, :, 10:])


def test_hot_rows_capacity_validated(pkv):
    """retrieve_and_attend_rows refuses hot_rows < n_hot (rows of one KV head would read the next head's)."""
    import ctypes
    K, q, V = make_problem(25, 1, 8, 2, 500, plant=False)
    cfg = pkv.config_init(8, 2, SB)
    ix = pkv.Index(cfg, 1, 500)
    pkv.encode_keys(ix, K)
    Kh = synth.isotropic(26, (1, 2, 64, 128), device="cuda")
    T, C = pkv.schedule(500, 16)
    p = pkv.RetrieveParams(T, C, 16, None, None, None, None, 0)
    idx = torch.empty(1, 8, 16, dtype=torch.int32, device="cuda")
    est = torch.empty(1, 8, 16, device="cuda")
    out = torch.empty(1, 8, 128, dtype=torch.bfloat16, device="cuda")
    sb, sh, st = K.stride(0), K.stride(1), K.stride(2)
    vp = ctypes.c_void_p
    args = lambda n_hot, rows: (ix.handle, vp(q.data_ptr()), ctypes.byref(p), vp(K.data_ptr()), vp(V.data_ptr()), sb,
                                sh, st, vp(Kh.data_ptr()), vp(Kh.data_ptr()), n_hot, rows, 0.088, vp(idx.data_ptr()),
                                vp(est.data_ptr()), vp(out.data_ptr()), None, vp(torch.cuda.current_stream().cuda_stream))
    assert pkv._lib.retrieve_and_attend_rows(*args(64, 32)) == pkv.PKV_ERR_INVALID_ARG
    assert pkv._lib.retrieve_and_attend_rows(*args(32, 64)) == pkv.PKV_OK
    torch.cuda.synchronize()


@pytest.mark.parametrize("rho_mode", ["schedule", "one", "all"])
def test_key_fraction_reading_of_rho(pkv, rho_mode):
    """rho as a fraction of KEYS. The occupancy counts are built at
    pkv_index_set_occupancy and kept by a later append; scores and candidate sets bit-exact against the oracle's
    key-mode bonus tables, estimates / top-k / attention at the usual bars."""
    batch, n_q, n_kv, n, n_app, k = 2, 8, 2, 9000, 1500, 100
    K, q, V = make_problem(201, batch, n_q, n_kv, n)
    cfg = pkv.config_init(n_q, n_kv, SB)
    ix = pkv.Index(cfg, batch, n)
    pkv.encode_keys(ix, K[:, :, :n - n_app].contiguous())
    ix.set_occupancy(True)
    pkv.append_decode_keys(ix, K[:, :, n - n_app:].contiguous())
    rho = {"schedule": pkv.schedule_key_fraction(n), "one": 1, "all": n}[rho_mode]
    idx, est, dbg = pkv.retrieve_topk(ix, q, k, debug=True, rho_keys=rho)
    out32 = torch.full((batch, n_q, 128), float("nan"), device="cuda")
    ix.set_debug_output(out32)
    idx2, est2, out, lse = pkv.retrieve_and_attend(ix, q, K, V, k, rho_keys=rho)
    ix.set_debug_output(None)
    torch.cuda.synchronize()
    assert torch.equal(idx, idx2) and torch.equal(est, est2)
    C = dbg["C"]
    G = n_q // n_kv
    for b in range(batch):
        for g in range(n_kv):
            Kf = bf16_f64(K[b, g])
            meta = oracle_meta(Kf)
            occ = coarse.occupancy(meta["ids"])
            for hh in range(G):
                h = g * G + hh
                qf = bf16_f64(q[b, h])
                bonus, Tb = coarse.query_bonus_tables_keys(qf, SB, occ, rho)
                score = coarse.collision_scores(meta["ids"], bonus)
                assert np.array_equal(dbg["scores"][b, h].cpu().numpy().astype(np.int64), score), "scores"
                cand = coarse.bucket_topk(score, C)
                cg = dbg["cand"][b, h].cpu().numpy()
                assert np.array_equal(np.sort(cg[cg >= 0]), cand), "candidate set"
                qt, qn = rerank.rotated_unit_query(qf, SB)
                eo = rerank.estimate(meta, cand, qt, qn)
                check_topk(idx[b, h].cpu().numpy(), est[b, h].cpu().numpy(), cand, eo,
                           dict(zip(range(n), meta["knorm"].tolist())), qn, k)
                o, l = pipeline.attend(qf, Kf, bf16_f64(V[b, g]), idx[b, h].cpu().numpy())
                check_attention(out[b, h].float().cpu().numpy(), o, out32[b, h].cpu().numpy(), lse[b, h], l)
                if rho_mode == "all":  # every key is covered: the last probed centroid is the worst-ranked used one
                    assert np.all(Tb >= 1)


def test_key_fraction_needs_occupancy(pkv):
    K, q, V = make_problem(202, 1, 4, 1, 500, plant=False)
    ix = pkv.Index(pkv.config_init(4, 1, SB), 1, 500)
    pkv.encode_keys(ix, K)
    with pytest.raises(pkv.PkvError):
        pkv.retrieve_topk(ix, q, 10, rho_keys=50)  # occupancy not enabled
    ix.set_occupancy(True)
    with pytest.raises(pkv.PkvError):
        pkv.retrieve_topk(ix, q, 10, rho_keys=501)  # more keys than the zone holds
    pkv.retrieve_topk(ix, q, 10, rho_keys=50)
    ix.set_occupancy(False)
    with pytest.raises(pkv.PkvError):
        pkv.retrieve_topk(ix, q, 10, rho_keys=50)



def test_encoder_kinds_agree(pkv, monkeypatch):
    """The default thread-per-key encoder (encode_fast.cu: exact int32 butterflies, fp32 decisions certified against
    the oracle's fp64 sequence, uncertain keys handed to the exact half-warp kernel) against the half-warp kernel on
    ~300K LLM-like keys plus wide-range / zero / subnormal / tiny keys: ids and codes identical, stored weights within
    2e-6 relative; the oracle check of the same keys runs in the other parity tests."""
    K, q, V = make_problem(95, 2, 8, 2, 150000, plant=False)
    K[0, 0, 5] = 0
    K[0, 0, 6, 16:24] = 0
    K[1, 1, 10:40, 3] = 1e-9
    K[1, 0, 40:60, 100] = 3e-30
    K[0, 1, 60:70, :] = torch.randn(10, 128, device="cuda").to(torch.bfloat16) * 1e-20
    cfg = pkv.config_init(8, 2, SB)
    out = {}
    for kind in ("fast", "half"):
        monkeypatch.setenv("PKV_ENCODER", kind)
        ix = pkv.Index(cfg, 2, 150000)
        pkv.encode_keys(ix, K)
        out[kind] = [t.cpu().numpy() for t in ix.export()]
        out[kind + "_stats"] = ix.stats()
    assert np.array_equal(out["fast"][0], out["half"][0]), "ids"
    assert np.array_equal(out["fast"][1], out["half"][1]), "codes"
    wf, wh = out["fast"][2].astype(np.float64), out["half"][2].astype(np.float64)
    assert np.all(np.abs(wf - wh) <= 2e-6 * np.abs(wh) + 1e-30), "weights"
    assert out["fast_stats"] == out["half_stats"]


def test_half_warp_encoder_still_exact(pkv, monkeypatch):
    monkeypatch.setenv("PKV_ENCODER", "half")
    K, q, V = make_problem(96, 2, 8, 2, 3001)
    run_and_check(pkv, K, q, V, k=64, n_hot=16)


_RR_SCRIPT = r"""
import sys, torch
sys.path.insert(0, sys.argv[1])
import synth
from paper_2602_07721_b200 import pariskv as pkv
from tests.test_parity_gpu import make_problem
from tests.gpu_helpers import SB
K, q, _ = make_problem(61, 2, 8, 2, 40000, device="cuda")
cfg = pkv.config_init(8, 2, SB)
ix = pkv.Index(cfg, 2, 40000)
pkv.encode_keys(ix, K)
idx, est, dbg = pkv.retrieve_topk(ix, q, 100, n_cand=12000, debug=True)
torch.save({"idx": idx.cpu(), "est": est.cpu(), "cand": dbg["cand"].cpu(), "e": dbg["est"].cpu()}, sys.argv[2])
"""


def test_rerank_grids_bit_identical(pkv, tmp_path):
    """The SM-balanced flat rerank grid and the per-head grid (PKV_RR_FLAT=1 / 0, read once per process, hence the
    child processes) give the same candidates, estimates and top-k bit for bit (n_cand = 12000 of 40000 keys,
    batch 2: 94 tiles per head, head changes inside flat CTAs)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = []
    for env in ("1", "0"):
        f = tmp_path / f"rr_{env}.pt"
        r = subprocess.run([sys.executable, "-c", _RR_SCRIPT, root, str(f)], cwd=root, capture_output=True, text=True,
                           env={**os.environ, "PKV_RR_FLAT": env}, timeout=600)
        assert r.returncode == 0, r.stderr[-3000:]
        out.append(torch.load(f))
    a, b = out
    assert torch.equal(a["cand"], b["cand"]) and torch.equal(a["e"], b["e"])
    assert torch.equal(a["idx"], b["idx"]) and torch.equal(a["est"], b["est"])
