"""Shared helpers for the -m gpu parity tests: run the oracle on the same seeded inputs the CUDA path gets,
and the comparison rules of DESIGN.md §Parity (bit-exact codes/scores/candidates; AMB-15/16/17 tolerances)."""
from __future__ import annotations

import numpy as np
import torch

import synth
from oracle import coarse, levels, quantizer, rerank

SB = synth.rotation_sign_bits()
L32 = levels.levels_f32(8)
MSQ = levels.mid_sq(L32)
EST_REL = 1e-3          # north star: reranked scores within 1e-3 relative (AMB-15 scaled form)
ATT_ABS = 2e-3          # north star: attention output within 2e-3 absolute in bf16 (AMB-17)
W16_REL = 2.0 ** -11    # fp16 weights (w_fp16=1, AMB-20): round-to-nearest relative error of each stored w'_b


def w16_bound(meta, ids, qt, qn):
    """Extra estimate error allowed for fp16 weights: each w'_b carries a relative error <= 2^-11, so
    |d est| <= 2^-11 ||q|| sum_b w'_b ||v_b|| ||q~_b|| = 2^-11 ||q|| sum_b w_b ||q~_b|| (||v^_b|| = 1, AMB-6),
    plus one fp16 subnormal half-ulp of the key's largest weight (2^-25 of 2^(E+15)) per subspace."""
    qb = np.linalg.norm(np.asarray(qt, dtype=np.float64).reshape(16, 8), axis=1)
    w = meta["w"][np.asarray(ids, dtype=np.int64)]
    return (W16_REL * (w @ qb) + 16 * 2.0 ** -24 * w.max(axis=-1) * qb.max()) * qn * 1.001


def oracle_meta(K_f64: np.ndarray, exact_codes=False) -> dict:
    return quantizer.encode_keys(K_f64, SB, L32, MSQ, exact_codes=exact_codes)


def est_tol(est_oracle, knorm, qnorm):
    """AMB-15: |d| <= 1e-3 * max(|est|, 1e-2 ||k|| ||q||)."""
    return EST_REL * np.maximum(np.abs(est_oracle), 1e-2 * knorm * qnorm)


def check_encode(ids_gpu, codes_gpu, w_gpu, meta, w16=False):
    """Bit-exact ids and codes; stored weight w' = w / ||sign*L[idx]|| within 1e-5 relative (fp32), or
    within the fp16 rounding 2^-11 relative (+ a subnormal half-ulp of the key's largest weight) with w_fp16."""
    assert np.array_equal(ids_gpu, meta["ids"]), "centroid ids differ"
    assert np.array_equal(codes_gpu, meta["codes"]), "4-bit codes differ"
    want = meta["w"] / meta["vnorm"]
    err = np.abs(w_gpu.astype(np.float64) - want)
    if w16:
        tol = 1.0001 * W16_REL * np.abs(want) + 2.0 ** -24 * want.max(axis=-1, keepdims=True) + 1e-30
    else:
        tol = 1e-5 * np.abs(want) + 1e-30
    assert np.all(err <= tol), f"w' max err {np.max(err / tol)} x tol"


def check_topk(idx_gpu, est_gpu, cand, est_or, knorm_by_id, qnorm, k, extra_by_id=None):
    """AMB-16: GPU top-k set == oracle set except ids whose oracle estimate is within tolerance of the
    oracle's k-th estimate; GPU estimates of its picks match the oracle within AMB-15; order descending."""
    idx_o, val_o = rerank.topk(est_or, cand, k)
    valid_o = idx_o >= 0
    assert np.array_equal(idx_gpu >= 0, valid_o), "padding differs"
    by_id = dict(zip(cand.tolist(), est_or.tolist()))
    g = [int(i) for i in idx_gpu if i >= 0]
    assert len(set(g)) == len(g)
    o = [int(i) for i in idx_o if i >= 0]
    if not o:
        return
    kth = val_o[valid_o][-1]
    for i in set(g) ^ set(o):
        tol = 2 * est_tol(kth, knorm_by_id[i], qnorm) + (2 * extra_by_id[i] if extra_by_id else 0.0)
        assert abs(by_id[i] - kth) <= tol, f"top-k differs beyond ties: id {i} est {by_id[i]} kth {kth}"
    ge = np.array([by_id[i] for i in g])
    eg = est_gpu[: len(g)].astype(np.float64)
    tol = est_tol(ge, np.array([knorm_by_id[i] for i in g]), qnorm)
    if extra_by_id:
        tol = tol + np.array([extra_by_id[i] for i in g])
    assert np.all(np.abs(eg - ge) <= tol)
    assert np.all(np.diff(eg) <= 0)


def bf16_f64(t: torch.Tensor) -> np.ndarray:
    return synth.to_f64(t)


def oracle_retrieval(meta, q_f64, T, C, k):
    bonus = coarse.query_bonus_tables(q_f64, SB, T)
    score = coarse.collision_scores(meta["ids"], bonus)
    cand = coarse.bucket_topk(score, C)
    qt, qn = rerank.rotated_unit_query(q_f64, SB)
    est = rerank.estimate(meta, cand, qt, qn)
    return dict(score=score, cand=cand, est=est, qt=qt, qnorm=qn)


ATT_F32 = 2e-3  # the north-star 2e-3 absolute, applied to the fp32 output alone (before the bf16 rounding of out)


def check_attention(out_bf16, o_oracle, out_f32=None, lse=None, lse_oracle=None, what=""):
    """AMB-17 on one (sequence, query head): the bf16 output within 2e-3 + one bf16 rounding (2^-8 |o|) of the
    fp64 oracle; the fp32 output of pkv_index_set_debug_output (when given) within 2e-3 absolute; lse within
    1e-3 relative (floor 1)."""
    og = np.asarray(out_bf16, dtype=np.float64)
    err = np.abs(og - o_oracle)
    assert np.all(err <= ATT_ABS + 2.0 ** -8 * np.abs(o_oracle)), f"{what} attn err {err.max()}"
    if out_f32 is not None:
        e32 = np.abs(np.asarray(out_f32, dtype=np.float64) - o_oracle)
        assert np.all(e32 <= ATT_F32), f"{what} fp32 attn err {e32.max()}"
    if lse is not None:
        assert abs(float(lse) - lse_oracle) <= 1e-3 * max(1.0, abs(lse_oracle)), f"{what} lse"
