"""Stage I: coarse candidate generation by collision voting (PAPER §4.2.2 (1); §5.4).

* schedule(n, k)        adaptive (rho, beta) vs KV length (reading AMB-11 = SPEC S:329 in basis points)
* query_bonus_tables    per subspace, bonus of every centroid id for one query (P:477 + P:865, AMB-8/9/10)
* collision_scores      score_i = sum_b bonus_b(id_{i,b})  in [0, B * max bonus]
* bucket_topk           C = ceil(beta n) highest integer scores by counting;
                        ties in the threshold bucket: newest (larger index) first (AMB-12)
* key-fraction reading of rho (AMB-8b): occupancy, key_fraction_target,
  key_fraction_probes, query_bonus_tables_keys — "only let the top-rho fraction contribute a non-zero bonus"
   read as a fraction of KEYS, so that "collision processing scales with rho n"
"""
from __future__ import annotations

import numpy as np

from . import codebook, transform

# (min_length, rho, beta) in basis points (AMB-11)
SCHEDULE_BP = ((0, 1500, 1000), (20000, 1200, 800), (60000, 1000, 600), (200000, 800, 500))


def schedule(n: int, top_k: int, n_centroids: int = 256, table=SCHEDULE_BP):
    """Returns (T probes per subspace, C candidates) for a retrieval zone of n keys (integer arithmetic)."""
    rho_bp, beta_bp = table[0][1], table[0][2]
    for min_len, r_bp, b_bp in table:
        if n >= min_len:
            rho_bp, beta_bp = r_bp, b_bp
    T = (rho_bp * n_centroids + 9999) // 10000
    C = min(n, max(min(top_k, n), (beta_bp * n + 9999) // 10000))
    return int(T), int(C)


def query_bonus_tables(q: np.ndarray, rot_sign_bits: np.ndarray, T: int, B: int = 16,
                       tier_bonus=(6, 5, 4, 3, 2, 1)) -> np.ndarray:
    """bonus[b, c] for one query q [D] (fp64 values of the bf16 query). AMB-8/9/10."""
    y = transform.rotate_unscaled(q, rot_sign_bits)
    yb = transform.split(y, B)
    out = np.zeros((B, 2 ** yb.shape[-1]), dtype=np.int64)
    for b in range(B):
        s = codebook.centroid_scores(yb[b])
        rank = codebook.rank_centroids(s)
        out[b] = codebook.tier_bonus_of_rank(rank, T, tier_bonus)
    return out


def collision_scores(ids: np.ndarray, bonus: np.ndarray) -> np.ndarray:
    """score_i = sum_b bonus[b, ids[i, b]]. ids [n, B] -> int64 [n]."""
    ids = np.asarray(ids).astype(np.int64)
    n, B = ids.shape
    score = np.zeros(n, dtype=np.int64)
    for b in range(B):
        score = score + bonus[b, ids[:, b]]
    return score


def collision_scores_naive(ids: np.ndarray, q: np.ndarray, rot_sign_bits: np.ndarray, T: int,
                           tier_bonus=(6, 5, 4, 3, 2, 1)) -> np.ndarray:
    """Naive per-key loop (S:311's oracle): for every key and subspace, decode the key's centroid,
    rank it against all 2^m centroids by <q_b, omega> and look up its tier. Pure Python; tiny n only."""
    ids = np.asarray(ids).astype(np.int64)
    n, B = ids.shape
    D = len(q)
    m = D // B
    y = transform.rotate_unscaled(q, rot_sign_bits)
    W = codebook.all_centroids(m) * np.sqrt(m)   # +-1 entries
    n_tiers = len(tier_bonus)
    chunk = max(1, T // n_tiers)
    out = np.zeros(n, dtype=np.int64)
    for i in range(n):
        tot = 0
        for b in range(B):
            yb = y[b * m:(b + 1) * m]
            c = ids[i, b]
            sc = W @ yb
            # rank of c: number of centroids strictly better, ties broken by smaller id
            rk = int(np.sum(sc > sc[c]) + np.sum((sc == sc[c]) & (np.arange(2 ** m) < c)))
            if rk < T:
                tot += tier_bonus[min(rk // chunk, n_tiers - 1)]
        out[i] = tot
    return out


def threshold(score: np.ndarray, C: int, max_score: int = 96):
    """s* = max{s : #(score >= s) >= C}; returns (s*, #(score > s*)). C == 0 -> (max+1, 0)."""
    counts = np.bincount(np.asarray(score, dtype=np.int64), minlength=max_score + 1)
    if C <= 0:
        return max_score + 1, 0
    ge = 0
    for s in range(max_score, -1, -1):
        if ge + counts[s] >= C:
            return s, ge
        ge += counts[s]
    raise ValueError("C exceeds n")


def bucket_topk(score: np.ndarray, C: int, max_score: int = 96) -> np.ndarray:
    """Top-C keys by integer score via a counting histogram; threshold-bucket ties newest first.

    Returns the sorted candidate index array (a set: the order carries no meaning)."""
    score = np.asarray(score, dtype=np.int64)
    if C <= 0:
        return np.zeros(0, dtype=np.int64)
    s_star, n_gt = threshold(score, C, max_score)
    gt = np.nonzero(score > s_star)[0]
    eq = np.nonzero(score == s_star)[0]
    take = C - n_gt
    chosen = np.concatenate([gt, eq[len(eq) - take:]]) if take > 0 else gt
    return np.sort(chosen)


def bucket_topk_by_sort(score: np.ndarray, C: int) -> np.ndarray:
    """Independent sort-based oracle: sort by (score desc, index desc), keep C."""
    score = np.asarray(score, dtype=np.int64)
    order = sorted(range(len(score)), key=lambda i: (-score[i], -i))
    return np.sort(np.array(order[:C], dtype=np.int64))


# ---------------------------------------------------------------- key-fraction reading of rho (AMB-8b)
def occupancy(ids: np.ndarray, n_centroids: int = 256) -> np.ndarray:
    """occ[b, c] = number of keys whose subspace-b centroid id is c (per-subspace occupancy histogram)."""
    ids = np.asarray(ids).astype(np.int64)
    n, B = ids.shape
    occ = np.zeros((B, n_centroids), dtype=np.int64)
    for b in range(B):
        for c in ids[:, b]:
            occ[b, c] += 1
    return occ


def key_fraction_target(n: int, table=SCHEDULE_BP) -> int:
    """rho_keys = ceil(rho n): keys each subspace's probed centroids must hold (rho of the AMB-11 schedule)."""
    rho_bp = table[0][1]
    for min_len, r_bp, _ in table:
        if n >= min_len:
            rho_bp = r_bp
    return int((rho_bp * n + 9999) // 10000)


def key_fraction_probes(rank: np.ndarray, occ_b: np.ndarray, rho_keys: int) -> int:
    """T_b: probe centroids in rank order (best first, AMB-9) until the probed ones hold >= rho_keys keys —
    the top-rho fraction of the keys by their centroid's query score gets a bonus, whole centroids."""
    order = np.argsort(np.asarray(rank))  # order[r] = the centroid of rank r
    held, T = 0, 0
    while held < rho_keys:
        held += int(occ_b[order[T]])
        T += 1
    return T


def query_bonus_tables_keys(q: np.ndarray, rot_sign_bits: np.ndarray, occ: np.ndarray, rho_keys: int,
                            B: int = 16, tier_bonus=(6, 5, 4, 3, 2, 1)):
    """(bonus[b, c], T_b[b]) for one query under the key-fraction reading: per subspace the same ranking and
    tiers as query_bonus_tables (AMB-9/10) with that subspace's own probe count T_b."""
    y = transform.rotate_unscaled(q, rot_sign_bits)
    yb = transform.split(y, B)
    out = np.zeros((B, 2 ** yb.shape[-1]), dtype=np.int64)
    Tb = np.zeros(B, dtype=np.int64)
    for b in range(B):
        rank = codebook.rank_centroids(codebook.centroid_scores(yb[b]))
        Tb[b] = key_fraction_probes(rank, occ[b], rho_keys)
        out[b] = codebook.tier_bonus_of_rank(rank, int(Tb[b]), tier_bonus)
    return out, Tb
