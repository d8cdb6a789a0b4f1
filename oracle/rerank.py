"""Stage II: RSQ-IP reranking and final top-k (PAPER §4.1.3 Eq. 8-10, §4.2.2 (2)).

Eq. 10:  est_i = ||q|| * sum_b w_{i,b} <v_{i,b}, q~_b>,
with q~ = R q_hat the rotated unit query and v_{i,b} the renormalised dequantised direction.
Reading AMB-14: ||q|| is included, so est estimates <k_i, q> (no 1/sqrt(D)).
Final top-k: the k largest estimates, ties -> larger index; fewer than k candidates -> pad -1.
"""
from __future__ import annotations

import numpy as np

from . import transform


def rotated_unit_query(q: np.ndarray, rot_sign_bits: np.ndarray):
    """(q~ [D], ||q||): q~ = R (q/||q||)."""
    q = np.asarray(q, dtype=np.float64)
    qhat, qn = transform.l2_normalize(q)
    return transform.rotate(qhat, rot_sign_bits), float(qn)


def estimate(meta: dict, cand: np.ndarray, qt: np.ndarray, qnorm: float, B: int = 16) -> np.ndarray:
    """Eq. 10 for the candidate rows `cand` of the metadata dict from quantizer.encode_keys."""
    cand = np.asarray(cand, dtype=np.int64)
    qb = transform.split(qt, B)                      # [B, m]
    v = meta["v"][cand]                              # [C, B, m]
    w = meta["w"][cand]                              # [C, B]
    sub = np.sum(v * qb[None], axis=-1)              # <v_b, q~_b>
    return qnorm * np.sum(w * sub, axis=-1)


def estimate_uncorrected(meta: dict, cand: np.ndarray, qt: np.ndarray, qnorm: float, B: int = 16) -> np.ndarray:
    """The alpha == 1 variant (quantisation 'shrinks this alignment'): w_b = ||k|| r_b."""
    cand = np.asarray(cand, dtype=np.int64)
    qb = transform.split(qt, B)
    v = meta["v"][cand]
    w = meta["knorm"][cand][:, None] * meta["r"][cand]
    return qnorm * np.sum(w * np.sum(v * qb[None], axis=-1), axis=-1)


def topk(est: np.ndarray, cand: np.ndarray, k: int):
    """k largest est; ties -> larger index. Returns (idx int64 [k] (-1 padded), est [k])."""
    est = np.asarray(est, dtype=np.float64)
    cand = np.asarray(cand, dtype=np.int64)
    order = sorted(range(len(cand)), key=lambda i: (-est[i], -cand[i]))[:k]
    idx = np.full(k, -1, dtype=np.int64)
    val = np.full(k, -np.inf, dtype=np.float64)
    idx[:len(order)] = cand[order]
    val[:len(order)] = est[order]
    return idx, val


def topk_exhaustive(est: np.ndarray, cand: np.ndarray, k: int) -> set:
    """Pin P12: the k-subset maximising the estimate sum, by enumeration (pools <= 20)."""
    import itertools
    best, best_set = -np.inf, None
    for sub in itertools.combinations(range(len(cand)), k):
        s = float(np.sum(np.asarray(est)[list(sub)]))
        if s > best:
            best, best_set = s, sub
    return {int(cand[i]) for i in best_set}
