"""Attention references and quality metrics (PAPER §3).

* full_attention          Eq. 1 over all keys
* restricted_attention    Eq. 2-3 over an index set C(q) (hot rows + retrieved rows, AMB-17)
* exact_topk              TopK(q) = argmax^k <k_i, q>, fp64, ties -> larger index
* recall_at_k             |pred & exact| / k
Reading: the logits carry the usual temperature 1/sqrt(D) ("scale"); lse is the natural-log
log-sum-exp of the scaled logits, so the softmax is exp(logit - lse).
"""
from __future__ import annotations

import numpy as np


def _softmax_out(logits: np.ndarray, V: np.ndarray):
    m = np.max(logits)
    p = np.exp(logits - m)
    l = np.sum(p)
    return (p[:, None] * V).sum(axis=0) / l, float(m + np.log(l)), p / l


def full_attention(q: np.ndarray, K: np.ndarray, V: np.ndarray, scale: float):
    """Eq. 1 with temperature: returns (o [Dv], lse)."""
    q = np.asarray(q, dtype=np.float64)
    K = np.asarray(K, dtype=np.float64)
    V = np.asarray(V, dtype=np.float64)
    o, lse, _ = _softmax_out((K @ q) * scale, V)
    return o, lse


def restricted_attention(q: np.ndarray, K: np.ndarray, V: np.ndarray, rows: np.ndarray, scale: float):
    """Eq. 2-3: softmax restricted to the rows listed in `rows` (duplicates are not allowed)."""
    rows = np.asarray(rows, dtype=np.int64)
    assert len(rows) > 0 and len(np.unique(rows)) == len(rows)
    return full_attention(q, np.asarray(K)[rows], np.asarray(V)[rows], scale)


def attention_weights(q, K, scale):
    q = np.asarray(q, dtype=np.float64)
    K = np.asarray(K, dtype=np.float64)
    _, _, p = _softmax_out((K @ q) * scale, np.zeros((len(K), 1)))
    return p


def exact_topk(q: np.ndarray, K: np.ndarray, k: int) -> np.ndarray:
    """Exact top-k by <k_i, q> in fp64, ties -> larger index."""
    s = np.asarray(K, dtype=np.float64) @ np.asarray(q, dtype=np.float64)
    order = sorted(range(len(s)), key=lambda i: (-s[i], -i))
    return np.array(order[:k], dtype=np.int64)


def recall_at_k(pred, exact) -> float:
    exact = set(int(x) for x in exact)
    pred = set(int(x) for x in pred if x >= 0)
    return len(pred & exact) / max(1, len(exact))


def merge_partials(ms, ls, os_):
    """LSE merge of per-shard partial softmax states. Shard p holds m_p = max logit over its rows,
    l_p = sum exp(logit - m_p) and o_p = sum exp(logit - m_p) v / l_p (its own normalised output).
    Then o = sum_p l_p e^{m_p - M} o_p / sum_p l_p e^{m_p - M} and lse = M + log sum_p l_p e^{m_p - M}."""
    ms = np.asarray(ms, dtype=np.float64)
    ls = np.asarray(ls, dtype=np.float64)
    os_ = np.asarray(os_, dtype=np.float64)
    M = np.max(ms)
    wts = ls * np.exp(ms - M)
    L = np.sum(wts)
    o = np.sum(wts[:, None] * os_, axis=0) / L
    return o, float(M + np.log(L))
