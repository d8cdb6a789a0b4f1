"""Analytic direction centroids and query-side probe ranking (PAPER §4.1.2, §4.2.2, §5.4).

Eq. 5: Omega = {+-1/sqrt(m)}^m, |Omega| = 2^m.
Eq. 6: centroid_id = argmax_{omega} <u_b, omega>.
Reading AMB-4: id bit j <-> coordinate j of the subspace (LSB first), bit = 1 for a
positive coordinate; AMB-3: a zero coordinate counts as positive.

Query side, P:477 ("in each subspace we compare the query to the key's assigned
centroid (cheap dot product q^T c) and only let the top-rho fraction contribute a
non-zero bonus") with P:865 (6-tier bonus, scores in [0, 96]).
Readings AMB-8/9/10: T = ceil(rho * 2^m) probes per subspace; the centroid score is
sum_j (+-1) y'_{q,b,j} evaluated in fp64 left to right from 0.0 on the unscaled rotated
query (the positive factor 1/sqrt(m) and the query scale do not change the order);
order by score descending, ties by centroid id ascending; ranks split into n_tiers equal
chunks of size max(1, floor(T/n_tiers)), the last tier absorbing the remainder.
"""
from __future__ import annotations

import heapq

import numpy as np


def all_centroids(m: int) -> np.ndarray:
    """Explicit Omega as a [2^m, m] matrix, row c = decode(c) (Eq. 5)."""
    c = np.arange(2 ** m)[:, None]
    bits = (c >> np.arange(m)[None, :]) & 1
    return np.where(bits == 1, 1.0, -1.0) / np.sqrt(m)


def assign(u: np.ndarray) -> np.ndarray:
    """Closed form of Eq. 6: the sign pattern of u (zero -> positive). u: [..., m] -> int ids."""
    u = np.asarray(u, dtype=np.float64)
    m = u.shape[-1]
    bits = (u >= 0).astype(np.int64)
    return np.sum(bits << np.arange(m), axis=-1)


def assign_bruteforce(u: np.ndarray) -> np.ndarray:
    """argmax over all of Omega (Eq. 6 literally; pin P3). Ties -> smallest id."""
    u = np.asarray(u, dtype=np.float64)
    W = all_centroids(u.shape[-1])
    return np.argmax(u @ W.T, axis=-1)


def centroid_scores(yq_b: np.ndarray) -> np.ndarray:
    """Score of every centroid id c for one subspace of the unscaled rotated query (AMB-9).

    score_c = (((0.0 + s_0 y_0) + s_1 y_1) + ...) + s_{m-1} y_{m-1}, s_j = +1 if bit j of c else -1, fp64."""
    y = np.asarray(yq_b, dtype=np.float64)
    m = y.shape[-1]
    c = np.arange(2 ** m)
    acc = np.zeros(2 ** m, dtype=np.float64)
    for j in range(m):
        term = np.where(((c >> j) & 1) == 1, y[j], -y[j])
        acc = acc + term
    return acc


def rank_centroids(scores: np.ndarray) -> np.ndarray:
    """rank[c] = position of c in (score desc, id asc) order (AMB-9)."""
    order = sorted(range(len(scores)), key=lambda c: (-scores[c], c))
    rank = np.empty(len(scores), dtype=np.int64)
    rank[np.array(order)] = np.arange(len(scores))
    return rank


def tier_bonus_of_rank(rank: np.ndarray, T: int, tier_bonus=(6, 5, 4, 3, 2, 1)) -> np.ndarray:
    """Multi-tier collision bonus (AMB-10): 0 for unprobed centroids."""
    n_tiers = len(tier_bonus)
    chunk = max(1, T // n_tiers)
    tier = np.minimum(np.asarray(rank) // chunk, n_tiers - 1)
    bonus = np.asarray(tier_bonus, dtype=np.int64)[tier]
    return np.where(np.asarray(rank) < T, bonus, 0)


def top_probes_best_first(yq_b: np.ndarray, T: int):
    """Independent top-T probe generator (pin P8): best-first sign-flip search from sign(q_b).

    Flipping coordinate j away from the query's sign pattern costs 2|q_j|; a probe's
    score is max_score - sum of its flip costs. Enumerates flip sets in increasing cost with a
    heap ordered by (cost, id). Used on inputs without zero coordinates, where an equal-cost
    subset cannot hide behind an unpopped parent."""
    y = np.asarray(yq_b, dtype=np.float64)
    m = len(y)
    base = int(np.sum(((y >= 0).astype(np.int64)) << np.arange(m)))
    top = float(np.sum(np.abs(y)))
    cost = 2.0 * np.abs(y)
    out = []
    seen = set()
    heap = [(0.0, base, base)]  # (cost, id, id)
    while heap and len(out) < T:
        cst, cid, _ = heapq.heappop(heap)
        if cid in seen:
            continue
        seen.add(cid)
        out.append((cid, top - cst))
        flipped = cid ^ base
        for j in range(m):
            if not (flipped >> j) & 1:
                nid = cid ^ (1 << j)
                if nid not in seen:
                    ncost = float(np.sum(cost[[k for k in range(m) if ((nid ^ base) >> k) & 1]]))
                    heapq.heappush(heap, (ncost, nid, nid))
    return out


def brute_probe_list(yq_b: np.ndarray, T: int):
    """Exhaustive sort of all centroids by <q_b, omega> (S:146's oracle)."""
    m = len(yq_b)
    W = all_centroids(m) * np.sqrt(m)
    s = W @ np.asarray(yq_b, dtype=np.float64)
    order = sorted(range(2 ** m), key=lambda c: (-s[c], c))
    return [(c, float(s[c])) for c in order[:T]]


def hamming(a: int, b: int) -> int:
    return bin(a ^ b).count("1")


def omega_inner_product_closed_form(a: int, b: int, m: int) -> float:
    """<omega_a, omega_b> = 1 - 2 popcount(a xor b)/m (pin P4)."""
    return 1.0 - 2.0 * hamming(a, b) / m

