"""Pins for the CPU oracle (-m "not gpu"): each test checks an oracle function against something other than
itself — a value the paper prints, a closed form, an invariant, a brute-force enumeration or a textbook /
library routine — so that a dropped term, a wrong sign or index, or a transposed operand fails a test.
Pin ids (P1..P13) follow DESIGN.md §Oracle pins."""
from __future__ import annotations

import fractions

import numpy as np
import pytest
import scipy.special
import scipy.stats
import torch

import synth
from oracle import attention, codebook, coarse, levels, pipeline, quantizer, rerank, sharded, transform

SB = synth.rotation_sign_bits()
L32 = levels.levels_f32(8)
MSQ = levels.mid_sq(L32)


def _bf16(x):
    return torch.as_tensor(np.asarray(x, dtype=np.float32)).to(torch.bfloat16).to(torch.float64).numpy()


# ---------------------------------------------------------------- P1 rotation
def test_p1_hadamard_orthogonality_exact():
    H = transform.fwht(np.eye(128))
    assert np.array_equal(H @ H.T, 128.0 * np.eye(128))          # integer check, exact


def test_p1_fwht_equals_explicit_kronecker_product():
    rng = np.random.default_rng(0)
    for D in (8, 128):
        x = rng.standard_normal((5, D))
        Hk = transform.hadamard_matrix_kron(D)
        assert np.allclose(transform.fwht(x), x @ Hk.T, rtol=0, atol=1e-12)


def test_p1_srht_explicit_matrix_d8():
    """D=8 rotation equals the explicit sign-diagonal + normalised Hadamard product."""
    bits = np.array([0, 1, 1, 0, 1, 0, 0, 1], dtype=np.uint8)
    R = transform.hadamard_matrix_kron(8) @ np.diag(np.where(bits == 1, -1.0, 1.0)) / np.sqrt(8)
    e1 = np.eye(8)[0]
    assert np.allclose(transform.rotate(e1, bits), R @ e1, atol=1e-15)
    assert np.allclose(R @ R.T, np.eye(8), atol=1e-15)


def test_p1_isometry_1000_pairs():
    rng = np.random.default_rng(1)
    x = rng.standard_normal((1000, 128))
    y = rng.standard_normal((1000, 128))
    x /= np.linalg.norm(x, axis=1, keepdims=True)
    y /= np.linalg.norm(y, axis=1, keepdims=True)
    d0 = np.sum(x * y, axis=1)
    d1 = np.sum(transform.rotate(x, SB) * transform.rotate(y, SB), axis=1)
    assert np.max(np.abs(d0 - d1)) <= 1e-4


# ---------------------------------------------------------------- P2 FWHT exactness
def test_p2_fp64_fwht_exact_for_bf16_keys():
    K = synth.llm_keys(3, 1, 1, 64)[0, 0]
    Kf = synth.to_f64(K)
    y = transform.rotate_unscaled(Kf, SB)
    H = transform.hadamard_matrix_kron(128).astype(np.int64)
    s = np.where(SB == 1, -1, 1)
    for i in range(len(Kf)):
        xi = [fractions.Fraction(float(v)) * int(sj) for v, sj in zip(Kf[i], s)]
        for r in range(0, 128, 7):
            exact = sum(int(H[r, j]) * xi[j] for j in range(128))
            assert fractions.Fraction(float(y[i, r])) == exact


# ---------------------------------------------------------------- P3 assignment
def test_p3_paper_m3_example(golden):
    g = golden("paper_m3_example.txt")
    u = np.array([float(v) for v in g["u"].split(",")])
    u = u / np.linalg.norm(u)
    want = [1 if s == "+" else 0 for s in g["centroid_signs"].split(",")]
    cid = int(codebook.assign(u))
    assert [(cid >> j) & 1 for j in range(3)] == want
    assert int(codebook.assign_bruteforce(u)) == cid
    assert np.allclose(codebook.all_centroids(3)[cid], np.array([1, 1, -1]) / np.sqrt(3))
    assert codebook.all_centroids(int(g["m"])).shape[0] == int(g["n_centroids"])


def test_p3_closed_form_equals_bruteforce_argmax():
    rng = np.random.default_rng(2)
    u = rng.standard_normal((1000, 8))
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    assert np.array_equal(codebook.assign(u), codebook.assign_bruteforce(u))


def test_p3_encoder_ids_equal_bruteforce_on_rotated_keys():
    K = synth.to_f64(synth.llm_keys(4, 1, 1, 200)[0, 0])
    meta = quantizer.encode_keys(K, SB, L32, MSQ)
    u = transform.split(transform.rotate(transform.l2_normalize(K)[0], SB), 16)
    assert np.array_equal(meta["ids"].astype(np.int64), codebook.assign_bruteforce(u))


# ---------------------------------------------------------------- P4 centroids
def test_p4_centroid_geometry():
    W = codebook.all_centroids(8)
    assert np.allclose(np.linalg.norm(W, axis=1), 1.0)
    G = W @ W.T
    for a in range(0, 256, 17):
        for b in range(0, 256, 13):
            assert abs(G[a, b] - codebook.omega_inner_product_closed_form(a, b, 8)) < 1e-12
    assert abs(G[0b00001111, 0]) < 1e-12                          # Hamming m/2 -> orthogonal


# ---------------------------------------------------------------- P5 uniformity
def test_p5_isotropic_ids_uniform():
    K = synth.to_f64(synth.isotropic(5, (20000, 128)))
    ids = quantizer.encode_keys(K, SB, L32, MSQ)["ids"]
    for b in (0, 7, 15):
        counts = np.bincount(ids[:, b], minlength=256)
        p = scipy.stats.chisquare(counts).pvalue
        assert p > 1e-3


# ---------------------------------------------------------------- P6 Prop. 1
def test_p6_prop1_beta_priors_isotropic():
    K = synth.to_f64(synth.isotropic(6, (20000, 128)))
    meta = quantizer.encode_keys(K, SB, L32, MSQ)
    z = (meta["S"] / meta["S"].sum(axis=1, keepdims=True)).ravel()
    ks_z = scipy.stats.kstest(z, scipy.stats.beta(4, 60).cdf).statistic
    u2 = (meta["y"].reshape(-1, 16, 8) ** 2 / meta["S"][..., None]).ravel()[::7]
    ks_u = scipy.stats.kstest(u2, scipy.stats.beta(0.5, 3.5).cdf).statistic
    assert ks_z < 0.02 and ks_u < 0.02


# ---------------------------------------------------------------- P7 levels
def test_p7_levels_match_independent_quadrature(golden):
    g = golden("prop1_levels_m8.txt")
    want = np.array([float(v) for v in g["levels"].split(",")])
    assert np.allclose(levels.design_levels(8), want, atol=6e-9)
    edges = np.array([float(v) for v in g["edges"].split(",")])
    assert np.allclose(levels.bin_edges(8), edges, atol=6e-7)


@pytest.mark.parametrize("m", [2, 4, 8, 16])
def test_p7_levels_mean_and_order(m):
    L = levels.design_levels(m)
    assert abs(L.mean() - levels.expected_abs_coordinate(m)) < 1e-12
    assert np.all(np.diff(L) > 0) and L[0] > 0 and L[-1] < 1


def test_p7_levels_m2_arcsine_closed_form():
    # m = 2: |u_1| = |cos theta|, theta uniform; equal-probability bins are theta-bins of width pi/16.
    L = levels.design_levels(2)
    want = []
    for i in range(8):
        k = 7 - i
        a, b = k * np.pi / 16, (k + 1) * np.pi / 16
        want.append((np.sin(b) - np.sin(a)) / (b - a))
    assert np.allclose(L, want, atol=1e-10)


def test_p7_levels_monte_carlo_m8():
    rng = np.random.default_rng(7)
    x = rng.standard_normal((400000, 8))
    a = np.abs(x[:, 0] / np.linalg.norm(x, axis=1))
    e = levels.bin_edges(8)
    L = levels.design_levels(8)
    for i in range(8):
        sel = a[(a >= e[i]) & (a < e[i + 1])]
        assert abs(len(sel) / len(a) - 1 / 8) < 0.003
        assert abs(sel.mean() - L[i]) < 2e-3


def test_p7_decision_constants_exact_from_fp32_levels():
    M = levels.mid_sq(L32)
    for t in range(7):
        mid = fractions.Fraction(float(L32[t])) / 2 + fractions.Fraction(float(L32[t + 1])) / 2
        assert fractions.Fraction(float(M[t])) == mid * mid


def test_p7_midpoint_rule_is_nearest_level():
    K = synth.to_f64(synth.llm_keys(8, 1, 1, 300)[0, 0])
    meta = quantizer.encode_keys(K, SB, L32, MSQ)
    u = np.abs(meta["u"]).reshape(len(K), 128)
    near = np.argmin(np.abs(u[..., None] - L32.astype(np.float64)[None, None, :]), axis=-1)
    idx = (meta["nib"] & 7).astype(np.int64)
    # identical except within 1e-12 of a midpoint
    mids = (L32[:-1].astype(np.float64) + L32[1:]) / 2
    close = np.min(np.abs(u[..., None] - mids), axis=-1) < 1e-12
    assert np.all((idx == near) | close)
    assert np.array_equal((meta["nib"] >> 3) & 1, (meta["y"] >= 0).astype(np.uint8))


# ---------------------------------------------------------------- code packing / degenerate
def test_code_pack_roundtrip_and_degenerate_subspace():
    K = np.zeros((2, 128))
    K[1, :] = _bf16(np.random.default_rng(9).standard_normal(128))
    meta = quantizer.encode_keys(K, SB, L32, MSQ)
    assert np.array_equal(quantizer.unpack_codes(meta["codes"]), meta["nib"])
    # zero key: every subspace degenerate -> encode(e_1) (AMB-7)
    assert np.all(meta["ids"][0] == 0xFF) and np.all(meta["w"][0] == 0)
    nib0 = meta["nib"][0].reshape(16, 8)
    assert np.all(nib0[:, 0] == 0xF) and np.all(nib0[:, 1:] == 0x8)
    assert np.all(meta["alpha"][1] <= 1 + 1e-12) and np.all(meta["alpha"][1] > 0)


# ---------------------------------------------------------------- P8 probes
def test_p8_probe_ranking_equals_best_first_and_exhaustive():
    rng = np.random.default_rng(10)
    for _ in range(30):
        y = rng.standard_normal(8)
        rank = codebook.rank_centroids(codebook.centroid_scores(y))
        order = list(np.argsort(rank))
        bf = [c for c, _ in codebook.top_probes_best_first(y, 16)]
        ex = [c for c, _ in codebook.brute_probe_list(y, 16)]
        assert order[:16] == bf == ex


def test_p8_flip_cost_identity():
    rng = np.random.default_rng(11)
    y = rng.standard_normal(8)
    s = codebook.centroid_scores(y)
    top = int(codebook.assign(y))
    for j in range(8):
        assert abs(s[top ^ (1 << j)] - (s[top] - 2 * abs(y[j]))) < 1e-12


def test_tier_bonus_shape():
    T = 26
    b = codebook.tier_bonus_of_rank(np.arange(256), T)
    assert list(b[:4]) == [6] * 4 and b[T - 1] == 1 and np.all(b[T:] == 0)
    assert sorted(set(b[:T].tolist()), reverse=True) == [6, 5, 4, 3, 2, 1]


# ---------------------------------------------------------------- P9 collision bounds
def test_p9_collision_score_range(golden):
    g = golden("paper_constants.txt")
    q = _bf16(np.random.default_rng(12).standard_normal(128))
    bonus = coarse.query_bonus_tables(q, SB, T=26)
    best = np.argmax(bonus, axis=1)[None, :]
    assert coarse.collision_scores(best, bonus)[0] == int(g["score_max_6tier"])
    one = coarse.query_bonus_tables(q, SB, T=26, tier_bonus=(1,))
    assert coarse.collision_scores(best, one)[0] == int(g["score_max_1tier"])
    ids = np.random.default_rng(13).integers(0, 256, (1000, 16))
    sc = coarse.collision_scores(ids, bonus)
    assert sc.min() >= 0 and sc.max() <= 96


# ---------------------------------------------------------------- P10 counts and candidates
def test_p10_collision_scores_equal_naive_loop():
    K = synth.to_f64(synth.llm_keys(14, 1, 1, 60)[0, 0])
    q = synth.to_f64(synth.llm_queries(14, 1, 1, 1)[0, 0])
    meta = quantizer.encode_keys(K, SB, L32, MSQ)
    bonus = coarse.query_bonus_tables(q, SB, T=39)
    assert np.array_equal(coarse.collision_scores(meta["ids"], bonus),
                          coarse.collision_scores_naive(meta["ids"], q, SB, T=39))


def test_p10_bucket_topk_spec_examples():
    assert list(coarse.bucket_topk(np.array([3, 1, 3, 0]), 2)) == [0, 2]
    assert list(coarse.bucket_topk(np.array([5, 5, 5, 5]), 2)) == [2, 3]
    assert list(coarse.bucket_topk(np.array([5, 5, 5, 5]), 0)) == []


def test_p10_bucket_topk_equals_sort_oracle():
    rng = np.random.default_rng(15)
    for trial in range(20):
        n = int(rng.integers(1, 3000))
        s = rng.integers(0, 97 if trial % 2 else 8, n)
        C = int(rng.integers(0, n + 1))
        assert np.array_equal(coarse.bucket_topk(s, C), coarse.bucket_topk_by_sort(s, C))


def test_schedule_values():
    assert coarse.schedule(130800, 100) == (26, 7848)
    assert coarse.schedule(32496, 100) == (31, 2600)
    assert coarse.schedule(1048304, 100) == (21, 52416)
    assert coarse.schedule(4096, 64) == (39, 410)
    assert coarse.schedule(50, 100) == (39, 50)
    for n in (10, 1000, 30000, 100000, 500000):
        T, C = coarse.schedule(n, 100)
        assert T / 256 >= C / max(n, 1) - 1e-12 or C == min(100, n)  # rho >= beta


# ---------------------------------------------------------------- P11 estimator
def test_p11_exact_code_limit():
    K = synth.to_f64(synth.llm_keys(16, 1, 1, 300)[0, 0])
    q = synth.to_f64(synth.llm_queries(16, 1, 1, 1)[0, 0])
    meta = quantizer.encode_keys(K, SB, L32, MSQ, exact_codes=True)
    qt, qn = rerank.rotated_unit_query(q, SB)
    est = rerank.estimate(meta, np.arange(300), qt, qn)
    assert np.allclose(est, K @ q, rtol=1e-9, atol=1e-9)


def test_p11_unbiased_variance_and_shrinkage_closed_forms():
    rng = np.random.default_rng(17)
    k = _bf16(rng.standard_normal(128) * 2.0)
    meta = quantizer.encode_keys(k[None], SB, L32, MSQ)
    kn = float(meta["knorm"][0])
    r, al = meta["r"][0], meta["alpha"][0]
    khat = k / np.linalg.norm(k)
    N = 12000
    for c in (0.9, 0.5):
        n = rng.standard_normal((N, 128))
        n -= (n @ khat)[:, None] * khat[None]
        n /= np.linalg.norm(n, axis=1, keepdims=True)
        Q = c * khat[None] + np.sqrt(1 - c * c) * n
        est = np.empty(N)
        est_u = np.empty(N)
        for i in range(N):
            qt, qn = rerank.rotated_unit_query(Q[i], SB)
            est[i] = rerank.estimate(meta, [0], qt, qn)[0]
            est_u[i] = rerank.estimate_uncorrected(meta, [0], qt, qn)[0]
        true = c * kn
        var = kn ** 2 * (1 - c * c) * np.sum(r ** 2 * (1 - al ** 2) / al ** 2) / 127
        se = np.sqrt(var / N)
        assert abs(est.mean() - true) < 4 * se                  # unbiased (Eq. 8-10)
        assert abs(est.var() / var - 1) < 0.06                  # variance closed form
        shrunk = c * kn * np.sum(r ** 2 * al)
        assert abs(est_u.mean() - shrunk) < 4 * np.sqrt(est_u.var() / N)
        assert shrunk < true                                    # P:408 shrinkage direction


def test_p11_alpha_correction_reduces_error_on_aligned_pairs():
    """the shrinkage bias grows with <k,q>, so the correction pays off for the keys that
    matter for top-k (strongly aligned pairs); for near-orthogonal pairs the 1/alpha noise dominates."""
    rng = np.random.default_rng(18)
    K = synth.to_f64(synth.isotropic(18, (400, 128)))
    meta = quantizer.encode_keys(K, SB, L32, MSQ)
    err_c, err_u, bias_c, bias_u = [], [], [], []
    for i in range(400):
        khat = K[i] / np.linalg.norm(K[i])
        n = rng.standard_normal(128)
        n -= (n @ khat) * khat
        n /= np.linalg.norm(n)
        q = 0.99 * khat + np.sqrt(1 - 0.99 ** 2) * n
        qt, qn = rerank.rotated_unit_query(q, SB)
        ex = K[i] @ q
        ec = rerank.estimate(meta, [i], qt, qn)[0] - ex
        eu = rerank.estimate_uncorrected(meta, [i], qt, qn)[0] - ex
        err_c.append(abs(ec)); err_u.append(abs(eu)); bias_c.append(ec); bias_u.append(eu)
    assert np.mean(err_c) < np.mean(err_u)
    assert abs(np.mean(bias_c)) < abs(np.mean(bias_u)) and np.mean(bias_u) < 0


# ---------------------------------------------------------------- P12 rerank + top-k
def test_p12_topk_equals_exhaustive_subset():
    rng = np.random.default_rng(20)
    for _ in range(10):
        C = int(rng.integers(5, 15))
        cand = rng.choice(1000, C, replace=False)
        est = rng.standard_normal(C)
        k = int(rng.integers(1, 5))
        idx, _ = rerank.topk(est, cand, k)
        assert set(idx.tolist()) == rerank.topk_exhaustive(est, cand, k)


def test_p12_topk_ties_and_padding():
    idx, v = rerank.topk(np.array([1.0, 2.0, 2.0, 0.5]), np.array([10, 3, 7, 1]), 3)
    assert list(idx) == [7, 3, 10]
    idx, v = rerank.topk(np.array([1.0]), np.array([4]), 3)
    assert list(idx) == [4, -1, -1]


def test_p12_exact_code_full_beta_limit_is_brute_force():
    K = synth.to_f64(synth.llm_keys(21, 1, 1, 500)[0, 0])
    V = synth.to_f64(synth.values(21, 1, 1, 500)[0, 0])
    Q = synth.to_f64(synth.llm_queries(21, 1, 2, 1)[0])
    meta = quantizer.encode_keys(K, SB, L32, MSQ, exact_codes=True)
    res = pipeline.decode_step(meta, Q, SB, top_k=500, C=500)
    for q, r in zip(Q, res):
        assert len(r["cand"]) == 500
        assert np.array_equal(np.sort(r["idx"]), np.arange(500))
        ex = attention.exact_topk(q, K, 50)
        assert list(r["idx"][:50]) == list(ex)
        o, lse = pipeline.attend(q, K, V, r["idx"])
        o2, lse2 = attention.full_attention(q, K, V, 1 / np.sqrt(128))
        assert np.allclose(o, o2, atol=1e-12) and abs(lse - lse2) < 1e-12


# ---------------------------------------------------------------- P13 attention
def test_p13_attention_against_scipy_softmax():
    rng = np.random.default_rng(22)
    K = rng.standard_normal((300, 128))
    V = rng.standard_normal((300, 128))
    q = rng.standard_normal(128)
    sc = 1 / np.sqrt(128)
    o, lse = attention.full_attention(q, K, V, sc)
    p = scipy.special.softmax(K @ q * sc)
    assert np.allclose(o, p @ V, atol=1e-12)
    assert abs(lse - scipy.special.logsumexp(K @ q * sc)) < 1e-12
    o1, _ = attention.full_attention(q, K[:1], V[:1], sc)
    assert np.allclose(o1, V[0])                                 # singleton softmax
    rows = rng.choice(300, 40, replace=False)
    o3, _ = attention.restricted_attention(q, K, V, rows, sc)
    p3 = scipy.special.softmax(K[rows] @ q * sc)
    assert np.allclose(o3, p3 @ V[rows], atol=1e-12)


def test_recall_at_k():
    assert attention.recall_at_k([1, 2, 3], [1, 2, 3]) == 1.0
    assert attention.recall_at_k([4, 5], [1, 2]) == 0.0
    assert attention.recall_at_k(list(range(50)) + [-1] * 50, list(range(100))) == 0.5


# ---------------------------------------------------------------- sharded decomposition
@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
def test_sharded_equals_unsharded(P):
    rng = np.random.default_rng(23 + P)
    n = 4000
    score = rng.integers(0, 12, n)           # many ties in the threshold bucket
    for C in (0, 1, 37, 410, 4000):
        assert np.array_equal(sharded.sharded_candidates(score, C, P), coarse.bucket_topk(score, C))
    cand = coarse.bucket_topk(score, 410)
    est = rng.standard_normal(len(cand)).round(1)     # ties in est too
    by_id = dict(zip(cand.tolist(), est.tolist()))
    i1, v1 = sharded.sharded_topk(by_id, cand, 64, P, n)
    i0, v0 = rerank.topk(est, cand, 64)
    assert np.array_equal(i1, i0)
    K = rng.standard_normal((n, 128))
    V = rng.standard_normal((n, 128))
    Kh = rng.standard_normal((20, 128))
    Vh = rng.standard_normal((20, 128))
    q = rng.standard_normal(128)
    o1, l1 = sharded.sharded_attention(q, K, V, i0, Kh, Vh, P, 1 / np.sqrt(128))
    o0, l0 = pipeline.attend(q, K, V, i0, Kh, Vh)
    assert np.allclose(o1, o0, atol=1e-12) and abs(l1 - l0) < 1e-12


def test_p8_probe_ranking_exact_ties_by_ascending_id():
    """Integer-valued queries with zero and repeated |y_j| create exact score ties (AMB-9 tie rule)."""
    for y in ([0, 1, -1, 2, 0, -2, 3, 1], [1, 1, 1, 1, -1, -1, -1, -1], [0] * 8):
        y = np.array(y, dtype=np.float64)
        rank = codebook.rank_centroids(codebook.centroid_scores(y))
        ex = [c for c, _ in codebook.brute_probe_list(y, 256)]
        assert list(np.argsort(rank)) == ex


def test_p8_complement_symmetry_of_ranking():
    """score(255 - c) == -score(c) bit-exactly for the AMB-9 left-to-right fp64 sum (zeros are +0.0), so
    rank(255 - c) == 255 - rank(c): the property the CUDA query prep uses to sort only 128 leaders
    (qprep). Random, wide-range, tie-heavy and all-zero subspaces."""
    rng = np.random.default_rng(12)
    ys = [rng.standard_normal(8) for _ in range(50)]
    ys += [rng.standard_normal(8) * 10.0 ** rng.integers(-30, 30, 8) for _ in range(50)]
    ys += [np.array(v, dtype=np.float64) for v in
           ([0, 1, -1, 2, 0, -2, 3, 1], [1, 1, 1, 1, -1, -1, -1, -1], [0] * 8, [1e300, 1e-300, -1e300, 0, 0, 1, 1, 1])]
    c = np.arange(256)
    for y in ys:
        s = codebook.centroid_scores(y)
        assert np.array_equal(s[255 - c], -s[c])
        assert not np.any(np.signbit(s[s == 0]))
        rank = codebook.rank_centroids(s)
        assert np.array_equal(rank[255 - c], 255 - rank[c])


# ---------------------------------------------------------------- helpers that were unpinned in round 1
def test_eq4_blockwise_ip_equals_plain_inner_product():
    """Eq. 4: sum_b r_b^k r_b^q <u_b^k, u_b^q> = <k~, q~>. Pinned against numpy's dot of the
    unsplit rotated vectors (the identity the paper uses), including zero-radius subspaces (u := e_1, r = 0,
    AMB-7), which must contribute nothing."""
    rng = np.random.default_rng(31)
    k = rng.standard_normal((50, 128))
    q = rng.standard_normal((50, 128))
    k[3, 16:24] = 0.0          # one zero subspace of the key
    q[7, :8] = 0.0             # and of a query
    for x, y in ((k, q), (transform.rotate_unscaled(k, SB), transform.rotate_unscaled(q, SB))):
        rk, uk = transform.polar(transform.split(x, 16))
        rq, uq = transform.polar(transform.split(y, 16))
        got = transform.blockwise_ip(rk, uk, rq, uq)
        want = np.einsum("nd,nd->n", x, y)
        assert np.allclose(got, want, rtol=1e-12, atol=1e-10)
    # a transposed operand (blocks of k against blocks of a different key) must not pass
    rk, uk = transform.polar(transform.split(k, 16))
    rq, uq = transform.polar(transform.split(q, 16))
    assert not np.allclose(transform.blockwise_ip(rk, uk, rq[::-1], uq[::-1]), np.einsum("nd,nd->n", k, q))


def test_dequantize_matches_code_semantics():
    """P:400 ("dequantizes to v"), AMB-4/AMB-6: unpacking the stored nibbles and dequantising gives unit
    subspace vectors whose signs are the sign bits, whose magnitudes are the Prop. 1 levels of the idx bits
    (closed-form values A.1 in tests/golden), and whose inner product with u_b is the stored alpha wherever
    the 1e-3 floor is inactive (Eq. 7)."""
    rng = np.random.default_rng(32)
    K = _bf16(rng.standard_normal((40, 128)))
    meta = quantizer.encode_keys(K, SB, L32, MSQ)
    v = quantizer.dequantize(quantizer.unpack_codes(meta["codes"]), L32)
    assert v.shape == (40, 16, 8)
    assert np.allclose(np.linalg.norm(v, axis=-1), 1.0, atol=1e-12)
    nib = quantizer.unpack_codes(meta["codes"]).reshape(40, 16, 8).astype(np.int64)
    y = meta["y"].reshape(40, 16, 8)
    assert np.array_equal(v > 0, (nib >> 3) == 1)
    assert np.array_equal((nib >> 3) == 1, y >= 0)                    # sign bit = sign of y (AMB-3)
    # |v_j| / |v_0| = L[idx_j] / L[idx_0] with the printed A.1 levels
    Lp = np.array([0.03072799, 0.09277686, 0.15670372, 0.22414131, 0.29752234, 0.38118776, 0.48522534, 0.65992414])
    ratio = np.abs(v) / np.abs(v[..., :1])
    assert np.allclose(ratio, Lp[nib & 7] / Lp[nib[..., :1] & 7], rtol=2e-7)
    dots = np.sum(v * meta["u"], axis=-1)
    live = dots > 1e-3
    assert live.mean() > 0.99 and np.allclose(dots[live], meta["alpha"][live], rtol=1e-12)


def test_attention_weights_are_the_softmax():
    """Eq. 2: weights = exp(logit - lse) of the same logits (scipy softmax), sum to one,
    a singleton gets weight 1 and equal logits give 1/n."""
    rng = np.random.default_rng(33)
    K = rng.standard_normal((77, 128))
    q = rng.standard_normal(128)
    sc = 1 / np.sqrt(128)
    p = attention.attention_weights(q, K, sc)
    assert np.allclose(p, scipy.special.softmax(K @ q * sc), rtol=1e-12)
    _, lse = attention.full_attention(q, K, np.zeros((77, 1)), sc)
    assert np.allclose(p, np.exp(K @ q * sc - lse), rtol=1e-12)
    assert abs(p.sum() - 1) < 1e-12
    assert np.allclose(attention.attention_weights(q, K[:1], sc), [1.0])
    assert np.allclose(attention.attention_weights(q, np.tile(K[:1], (5, 1)), sc), 0.2)


# ---------------------------------------------------------------- P15 key-fraction reading of rho (AMB-8b, f4)
def _rand_ids(seed, n, B=16, skew=True):
    """Centroid ids with a skewed occupancy (a few crowded centroids, many empty ones), like LLM keys."""
    rng = np.random.default_rng(seed)
    if not skew:
        return rng.integers(0, 256, size=(n, B))
    p = rng.dirichlet(np.full(256, 0.08), size=B)
    return np.stack([rng.choice(256, size=n, p=p[b]) for b in range(B)], axis=1)


def test_p15_occupancy_is_a_count():
    ids = _rand_ids(150, 700)
    occ = coarse.occupancy(ids)
    assert occ.shape == (16, 256) and np.all(occ.sum(axis=1) == 700)
    for b in (0, 7, 15):  # numpy's own counter as the independent check
        assert np.array_equal(occ[b], np.bincount(ids[:, b], minlength=256))


@pytest.mark.parametrize("rho_keys", [1, 37, 350, 699, 700])
def test_p15_probes_equal_bruteforce_key_sort(rho_keys):
    """Independent formulation: sort the KEYS by the rank of their centroid; the rho_keys-th key's centroid is
    the last probed one, so T_b = its rank + 1 — whole centroids, the minimal prefix of the centroid order."""
    ids = _rand_ids(151, 700)
    occ = coarse.occupancy(ids)
    rng = np.random.default_rng(152)
    for b in range(16):
        y = _bf16(rng.normal(size=8))
        rank = codebook.rank_centroids(codebook.centroid_scores(y))
        key_ranks = np.sort(rank[ids[:, b]])
        T = coarse.key_fraction_probes(rank, occ[b], rho_keys)
        assert T == key_ranks[rho_keys - 1] + 1
        probed = rank < T
        assert occ[b][probed].sum() >= rho_keys                      # covers the target ...
        last = np.argmax(rank == T - 1)
        assert occ[b][probed].sum() - occ[b][last] < rho_keys        # ... and is minimal
        assert occ[b][last] > 0                                      # a prefix never ends on an empty centroid


def test_p15_uniform_occupancy_reduces_to_centroid_fraction():
    """With every centroid holding the same number of keys, a key fraction is a centroid fraction:
    rho_keys = T * m keys -> exactly T probes, and the bonus tables equal the AMB-8 (centroid) reading."""
    m = 3
    rng = np.random.default_rng(153)
    ids = np.stack([rng.permutation(np.repeat(np.arange(256), m)) for _ in range(16)], axis=1)
    occ = coarse.occupancy(ids)
    q = _bf16(rng.normal(size=128))
    for T in (1, 5, 26, 39, 256):
        bonus_k, Tb = coarse.query_bonus_tables_keys(q, SB, occ, T * m)
        assert np.all(Tb == T)
        assert np.array_equal(bonus_k, coarse.query_bonus_tables(q, SB, T))


def test_p15_key_fraction_scores_equal_naive_per_key_loop():
    """The key-mode scores from the bonus tables equal a naive per-key loop that ranks each key's centroid against
    all 256 and counts how many keys' centroids rank strictly before it (pure Python, tiny n)."""
    n, rho_keys = 300, 45
    ids = _rand_ids(154, n)
    rng = np.random.default_rng(155)
    q = _bf16(rng.normal(size=128))
    occ = coarse.occupancy(ids)
    bonus, Tb = coarse.query_bonus_tables_keys(q, SB, occ, rho_keys)
    score = coarse.collision_scores(ids, bonus)
    y = transform.rotate_unscaled(q, SB)
    W = codebook.all_centroids(8) * np.sqrt(8)
    naive = np.zeros(n, dtype=np.int64)
    for b in range(16):
        sc = W @ y[8 * b:8 * b + 8]
        rk = [int(np.sum(sc > sc[c]) + np.sum((sc == sc[c]) & (np.arange(256) < c))) for c in range(256)]
        # T_b by scanning ranks: keys held by centroids of rank < r
        held_before = {r: sum(1 for i in range(n) if rk[ids[i, b]] < r) for r in range(257)}
        T = min(r for r in range(257) if held_before[r] >= rho_keys)
        assert T == Tb[b]
        chunk = max(1, T // 6)
        for i in range(n):
            r = rk[ids[i, b]]
            if r < T:
                naive[i] += (6, 5, 4, 3, 2, 1)[min(r // chunk, 5)]
    assert np.array_equal(score, naive)
    # every subspace hands a non-zero bonus to at least rho_keys keys (P:477's top-rho fraction)
    for b in range(16):
        assert np.sum(bonus[b][ids[:, b]] > 0) >= rho_keys


def test_p15_key_fraction_target_schedule():
    assert coarse.key_fraction_target(0) == 0
    assert coarse.key_fraction_target(130800) == 13080          # rho = 10% at 128K (S:329 row 60000)
    assert coarse.key_fraction_target(1048304) == 83865         # ceil(0.08 * 1048304)
    assert coarse.key_fraction_target(4096) == 615              # ceil(0.15 * 4096)
