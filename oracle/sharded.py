"""P-shard emulation of the sequence-sharded decode step.

Not in the paper: the paper is single-GPU. The decomposition below is the reading the
multi-GPU path implements; it must reproduce the unsharded oracle exactly:

  shard p owns the contiguous token range [off_p, off_p + len_p) of the retrieval zone.
  (H) per-shard histograms of the collision score are summed -> global s*, #(> s*), ties needed;
      ties are handed out newest shard first (the shard with the largest offsets), and inside a
      shard to its newest keys, so the candidate SET equals bucket_topk of the whole zone.
  (T) each shard reranks its own candidates and keeps its local top-k (est, global id); the union of
      local top-k lists contains the global top-k, merged with the same (est desc, id desc) order.
  (A) each shard attends over its own rows of the global top-k (+ the hot rows on the last shard),
      producing (m_p, l_p, o_p); the LSE merge (attention.merge_partials) gives Eq. 2-3 exactly.
"""
from __future__ import annotations

import numpy as np

from . import attention, rerank


def shard_ranges(n: int, P: int):
    """Contiguous shard boundaries: shard p gets [p*n//P, (p+1)*n//P)."""
    return [(p * n // P, (p + 1) * n // P) for p in range(P)]


def sharded_candidates(score: np.ndarray, C: int, P: int, max_score: int = 96) -> np.ndarray:
    """(H): candidate set from per-shard histograms. Returns sorted global ids."""
    score = np.asarray(score, dtype=np.int64)
    ranges = shard_ranges(len(score), P)
    hists = [np.bincount(score[a:b], minlength=max_score + 1) for a, b in ranges]
    g = np.sum(hists, axis=0)
    if C <= 0:
        return np.zeros(0, dtype=np.int64)
    ge = 0
    s_star = None
    for s in range(max_score, -1, -1):
        if ge + g[s] >= C:
            s_star = s
            break
        ge += g[s]
    need = C - ge
    out = []
    for p in range(P - 1, -1, -1):       # newest shard first
        a, b = ranges[p]
        loc = score[a:b]
        out.append(a + np.nonzero(loc > s_star)[0])
        eq = a + np.nonzero(loc == s_star)[0]
        take = min(need, len(eq))
        if take > 0:
            out.append(eq[len(eq) - take:])
        need -= take
    return np.sort(np.concatenate(out)) if out else np.zeros(0, dtype=np.int64)


def sharded_topk(est_by_id: dict, cand: np.ndarray, k: int, P: int, n: int):
    """(T): local top-k per shard then a replicated merge. est_by_id maps global id -> est."""
    ranges = shard_ranges(n, P)
    lists = []
    for a, b in ranges:
        loc = np.array([c for c in cand if a <= c < b], dtype=np.int64)
        e = np.array([est_by_id[int(c)] for c in loc], dtype=np.float64)
        idx, val = rerank.topk(e, loc, k)
        lists += [(v, i) for v, i in zip(val, idx) if i >= 0]
    lists.sort(key=lambda t: (-t[0], -t[1]))
    top = lists[:k]
    idx = np.full(k, -1, dtype=np.int64)
    val = np.full(k, -np.inf)
    idx[:len(top)] = [i for _, i in top]
    val[:len(top)] = [v for v, _ in top]
    return idx, val


def sharded_attention(q, K, V, idx, K_hot, V_hot, P: int, scale: float):
    """(A): per-shard partial softmax states over owned rows, then the LSE merge."""
    q = np.asarray(q, dtype=np.float64)
    n = len(K)
    idx = np.asarray(idx)
    idx = idx[idx >= 0]
    ms, ls, os_ = [], [], []
    for p, (a, b) in enumerate(shard_ranges(n, P)):
        rows = [r for r in idx if a <= r < b]
        Kp = [np.asarray(K, dtype=np.float64)[rows]] if rows else []
        Vp = [np.asarray(V, dtype=np.float64)[rows]] if rows else []
        if p == P - 1 and K_hot is not None and len(K_hot) > 0:
            Kp.append(np.asarray(K_hot, dtype=np.float64))
            Vp.append(np.asarray(V_hot, dtype=np.float64))
        if not Kp:
            continue
        Kp = np.concatenate(Kp)
        Vp = np.concatenate(Vp)
        logits = (Kp @ q) * scale
        m = np.max(logits)
        e = np.exp(logits - m)
        ms.append(m)
        ls.append(np.sum(e))
        os_.append((e[:, None] * Vp).sum(axis=0) / np.sum(e))
    return attention.merge_partials(ms, ls, os_)

