"""-m "not gpu": the sequence-sharded exchange protocol over a real process group — world size 2,
gloo backend on CPU. Each rank owns a contiguous half of the retrieval zone, exchanges (H) per-head score
histograms, (T) local top-k lists and (A) partial softmax states with all_gather — and, in the fused variant
(SURVEY §8(f3)), T and A as one exchange of (id, est, logit, value row) entries plus the hot partial — and must
reproduce the unsharded oracle exactly (candidate set, top-k) and to fp64 rounding (attention)."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth
from oracle import attention, coarse, levels, pipeline, quantizer, rerank

SB = synth.rotation_sign_bits()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem():
    n = 3000
    K = synth.llm_keys(31, 1, 1, n)
    q = synth.llm_queries(31, 1, 1, 1)
    synth.plant(K, q, 31)
    V = synth.values(31, 1, 1, n)
    Kf, qf, Vf = synth.to_f64(K[0, 0]), synth.to_f64(q[0, 0]), synth.to_f64(V[0, 0])
    Kh = synth.to_f64(synth.isotropic(32, (20, 128)))
    Vh = synth.to_f64(synth.isotropic(33, (20, 128)))
    return Kf, qf, Vf, Kh, Vh


def _worker(rank, world, port, q_out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        Kf, qf, Vf, Kh, Vh = _problem()
        n = len(Kf)
        lo, hi = rank * n // world, (rank + 1) * n // world
        L32 = levels.levels_f32(8)
        meta = quantizer.encode_keys(Kf[lo:hi], SB, L32, levels.mid_sq(L32))
        k = 64
        T, C = coarse.schedule(n, k)
        bonus = coarse.query_bonus_tables(qf, SB, T)
        score = coarse.collision_scores(meta["ids"], bonus)
        # (H) histogram exchange
        h = torch.from_numpy(np.bincount(score, minlength=128).astype(np.int64))
        hs = [torch.zeros_like(h) for _ in range(world)]
        dist.all_gather(hs, h)
        g = sum(x.numpy() for x in hs)
        ge, s_star = 0, None
        for s in range(127, -1, -1):
            if ge + g[s] >= C:
                s_star = s
                break
            ge += g[s]
        need = C - ge
        for r in range(world - 1, rank, -1):          # newest rank first
            need = max(0, need - int(hs[r][s_star]))
        eq = np.nonzero(score == s_star)[0]
        take = min(need, len(eq))
        loc = np.concatenate([np.nonzero(score > s_star)[0], eq[len(eq) - take:]]) if take else np.nonzero(score > s_star)[0]
        cand = np.sort(loc) + lo
        # (T) local top-k exchange
        qt, qn = rerank.rotated_unit_query(qf, SB)
        est = rerank.estimate(meta, cand - lo, qt, qn)
        idx, val = rerank.topk(est, cand, k)
        t = torch.from_numpy(np.stack([idx.astype(np.float64), val]))
        ts = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(ts, t)
        pool = [(float(v), int(i)) for x in ts for i, v in zip(x[0].numpy(), x[1].numpy()) if i >= 0]
        pool.sort(key=lambda e: (-e[0], -e[1]))
        gidx = np.array([i for _, i in pool[:k]])
        # (A) partial softmax exchange
        own = [i for i in gidx if lo <= i < hi]
        rows_k = [Kf[own]] + ([Kh] if rank == world - 1 else [])
        rows_v = [Vf[own]] + ([Vh] if rank == world - 1 else [])
        Kp, Vp = np.concatenate(rows_k), np.concatenate(rows_v)
        logits = Kp @ qf / np.sqrt(128)
        m = logits.max() if len(logits) else -np.inf
        e = np.exp(logits - m) if len(logits) else np.zeros(0)
        part = torch.from_numpy(np.concatenate([[m, e.sum()], (e[:, None] * Vp).sum(0) / max(e.sum(), 1e-300)]))
        ps = [torch.zeros_like(part) for _ in range(world)]
        dist.all_gather(ps, part)
        valid = [p.numpy() for p in ps if np.isfinite(p[0])]
        o, lse = attention.merge_partials([p[0] for p in valid], [p[1] for p in valid], [p[2:] for p in valid])
        # fused T+A exchange: the local top-k entries travel with their logits and value rows,
        # the last rank adds its hot-row partial; one all_gather, then every rank merges and attends alone
        ok = idx >= 0
        x_loc = Kf[idx[ok]] @ qf / np.sqrt(128)
        ent = np.zeros((k, 3 + 128))
        ent[:, 0], ent[:, 1] = -1, -np.inf
        ent[: ok.sum(), 0], ent[: ok.sum(), 1], ent[: ok.sum(), 2] = idx[ok], val[ok], x_loc
        ent[: ok.sum(), 3:] = Vf[idx[ok]]
        hot = np.full(130, 0.0)
        hot[0] = -np.inf
        if rank == world - 1:
            lh = Kh @ qf / np.sqrt(128)
            mh = lh.max()
            eh = np.exp(lh - mh)
            hot = np.concatenate([[mh, eh.sum()], (eh[:, None] * Vh).sum(0) / eh.sum()])
        msg = torch.from_numpy(np.concatenate([ent.ravel(), hot]))
        ms = [torch.zeros_like(msg) for _ in range(world)]
        dist.all_gather(ms, msg)
        ents = np.concatenate([m_[: k * 131].numpy().reshape(k, 131) for m_ in ms])
        ents = ents[ents[:, 0] >= 0]
        order = sorted(range(len(ents)), key=lambda i: (-ents[i, 1], -ents[i, 0]))[:k]
        sel = ents[order]
        gidx_f = sel[:, 0].astype(np.int64)
        xs = sel[:, 2]
        mx = xs.max()
        ex = np.exp(xs - mx)
        parts_m, parts_l, parts_o = [mx], [ex.sum()], [(ex[:, None] * sel[:, 3:]).sum(0) / ex.sum()]
        for m_ in ms:
            hp = m_[k * 131:].numpy()
            if np.isfinite(hp[0]):
                parts_m.append(hp[0])
                parts_l.append(hp[1])
                parts_o.append(hp[2:])
        o_f, lse_f = attention.merge_partials(parts_m, parts_l, parts_o)
        q_out.put((rank, gidx, o, lse, len(cand), gidx_f, o_f, lse_f))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_exchange_equals_unsharded():
    world = 2
    ctx = mp.get_context("spawn")
    qo = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, qo)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([qo.get(timeout=300) for _ in range(world)])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    Kf, qf, Vf, Kh, Vh = _problem()
    L32 = levels.levels_f32(8)
    meta = quantizer.encode_keys(Kf, SB, L32, levels.mid_sq(L32))
    r0 = pipeline.decode_step(meta, qf[None], SB, 64)[0]
    o0, l0 = pipeline.attend(qf, Kf, Vf, r0["idx"], Kh, Vh)
    assert sum(r[4] for r in res) == r0["C"]
    for rank, gidx, o, lse, _, gidx_f, o_f, lse_f in res:
        assert list(gidx) == list(r0["idx"])
        assert np.allclose(o, o0, atol=1e-12) and abs(lse - l0) < 1e-12
        assert list(gidx_f) == list(r0["idx"])  # fused exchange: same top-k, same attention
        assert np.allclose(o_f, o0, atol=1e-12) and abs(lse_f - l0) < 1e-12


if __name__ == "__main__":
    pytest.main([__file__, "-q"])
