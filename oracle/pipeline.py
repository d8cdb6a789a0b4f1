"""One ParisKV decode step for one (sequence, KV head) unit, step by step (PAPER Fig. 2/3, §4.2.2-4.2.3).

For each of the G query heads sharing the KV head (GQA, reading AMB-13: retrieval per query head):
  a1 query prep        bonus tables, q~ and ||q||
  a3 collision scan    score_i
  a4 bucket_topk       C candidates
  a5 rerank            Eq. 10 estimates
  a6 final top-k       k ids
  a7 sparse attention  Eq. 2-3 over hot rows U retrieved rows (AMB-17)
The key metadata (a2) comes from quantizer.encode_keys.
"""
from __future__ import annotations

import numpy as np

from . import attention, coarse, quantizer, rerank


def decode_step(meta: dict, Q: np.ndarray, rot_sign_bits: np.ndarray, top_k: int,
                tier_bonus=(6, 5, 4, 3, 2, 1), T: int | None = None, C: int | None = None,
                rho_keys: int | None = None) -> list:
    """Retrieval for the query heads Q [G, D] against the encoded retrieval zone `meta`.
    rho_keys: the key-fraction reading of rho (AMB-8b) instead of T probes per subspace.

    Returns one dict per query head: bonus, score, cand, est, idx, topk_est, T, C."""
    n = meta["ids"].shape[0]
    T0, C0 = coarse.schedule(n, top_k)
    T = T0 if T is None else T
    C = C0 if C is None else C
    occ = coarse.occupancy(meta["ids"]) if rho_keys else None
    out = []
    for q in np.asarray(Q, dtype=np.float64):
        if rho_keys:
            bonus, _ = coarse.query_bonus_tables_keys(q, rot_sign_bits, occ, rho_keys, tier_bonus=tier_bonus)
        else:
            bonus = coarse.query_bonus_tables(q, rot_sign_bits, T, tier_bonus=tier_bonus)
        score = coarse.collision_scores(meta["ids"], bonus)
        cand = coarse.bucket_topk(score, C)
        qt, qn = rerank.rotated_unit_query(q, rot_sign_bits)
        est = rerank.estimate(meta, cand, qt, qn)
        idx, tv = rerank.topk(est, cand, top_k)
        out.append(dict(bonus=bonus, score=score, cand=cand, est=est, idx=idx, topk_est=tv,
                        qt=qt, qnorm=qn, T=T, C=C))
    return out


def attend(q: np.ndarray, K: np.ndarray, V: np.ndarray, idx: np.ndarray, K_hot=None, V_hot=None,
           scale: float | None = None):
    """a7: softmax over hot rows U retrieved rows idx (idx >= 0 only). Returns (o, lse)."""
    q = np.asarray(q, dtype=np.float64)
    D = q.shape[-1]
    scale = 1.0 / np.sqrt(D) if scale is None else scale
    idx = np.asarray(idx, dtype=np.int64)
    idx = idx[idx >= 0]
    rows_k = [np.asarray(K, dtype=np.float64)[idx]]
    rows_v = [np.asarray(V, dtype=np.float64)[idx]]
    if K_hot is not None and len(K_hot) > 0:
        rows_k.append(np.asarray(K_hot, dtype=np.float64))
        rows_v.append(np.asarray(V_hot, dtype=np.float64))
    Kr = np.concatenate(rows_k)
    Vr = np.concatenate(rows_v)
    return attention.full_attention(q, Kr, Vr, scale)


def encode(K, rot_sign_bits, levels32, mid_sq, exact_codes=False):
    return quantizer.encode_keys(K, rot_sign_bits, levels32, mid_sq, exact_codes=exact_codes)
