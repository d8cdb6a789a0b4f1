"""Per-key prefill metadata: centroid ids, 4-bit direction codes, alpha, w (PAPER §4.1.2-4.1.3).

Follows, in the paper's order:
  (1) normalise & rotate            -> unscaled y' = H(s (.) k) (transform.rotate_unscaled)
  (2) subspace split                -> y'_b, b = 0..B-1
  (3) polar form                    -> r_b = ||y'_b|| / ||y'||, u_b = y'_b / ||y'_b||
  centroid id, Eq. 6                -> sign pattern of y'_b
  4-bit code, P:484 ("1-bit sign + 3-bit magnitude") with Prop. 1 levels (AMB-5)
  alpha, Eq. 7                      -> alpha_b = <v_b, u_b>, v_b = renormalised dequantised code (AMB-6)
  w, Eq. 9                          -> w_b = ||k|| r_b / alpha_b

Arithmetic contract for the discrete outputs (reading AMB-2), all fp64, no FMA:
  S_b    = (((y_0^2 + y_1^2) + y_2^2) + ...) + y_7^2          (y_j^2 one rounded product)
  id_b   = sum_j [y_j >= 0] 2^j                               (AMB-3/4: zero counts positive)
  idx_j  = #{t in 1..7 : y_j^2 >= M_t * S_b}                   (M_t from levels.mid_sq)
  nibble = ([y_j >= 0] << 3) | idx_j
Degenerate subspace S_b == 0 (AMB-7): u_b := e_1, so the code is encode(e_1):
  coordinate 0 -> (sign 1, idx 7), others -> (sign 1, idx 0); id = 0xFF (all zeros count positive); w_b = 0.
Packing (AMB-4): coordinate c of the key (c = 8b + j) -> byte c >> 1 of the 64-byte code, low nibble
for even c.
"""
from __future__ import annotations

import numpy as np

from . import transform

ALPHA_FLOOR = 1e-3  # S:231, S:264 (reading AMB-6)


def encode_keys(K: np.ndarray, rot_sign_bits: np.ndarray, levels32: np.ndarray, mid_sq: np.ndarray,
                B: int = 16, exact_codes: bool = False) -> dict:
    """Encode keys K [n, D] (fp64 values of bf16 keys) into ParisKV metadata.

    Returns dict with
      ids    uint8 [n, B]        centroid ids (Eq. 6)
      nib    uint8 [n, D]        per-coordinate nibble (sign<<3 | idx)
      codes  uint8 [n, D/2]      packed nibbles (AMB-4)
      w      f64   [n, B]        Eq. 9
      alpha  f64   [n, B]        Eq. 7 (clamped at 1e-3)
      v      f64   [n, B, m]     renormalised dequantised directions
      vnorm  f64   [n, B]        ||sign * L[idx]|| before renormalisation
      y      f64   [n, D]        unscaled rotated key
      S      f64   [n, B]        ||y'_b||^2 in the contract's order
      knorm  f64   [n]
    exact_codes=True replaces the quantised direction by the exact u_b (the "exact-code limit").
    """
    K = np.asarray(K, dtype=np.float64)
    n, D = K.shape
    m = D // B
    L = np.asarray(levels32, dtype=np.float32).astype(np.float64)
    M = np.asarray(mid_sq, dtype=np.float64)
    # (1) rotate (unscaled)
    y = transform.rotate_unscaled(K, rot_sign_bits)
    yb = transform.split(y, B)                                   # (2) [n, B, m]
    sq = yb * yb
    S = sq[..., 0].copy()
    for j in range(1, m):
        S = S + sq[..., j]
    # Eq. 6 closed form: sign pattern
    pos = (yb >= 0)
    ids = np.sum(pos.astype(np.int64) << np.arange(m), axis=-1).astype(np.uint8)
    # 3-bit magnitude: nearest Prop. 1 level via the midpoint rule
    idx = np.zeros(yb.shape, dtype=np.int64)
    for t in range(len(M)):
        idx += (sq >= (M[t] * S)[..., None]).astype(np.int64)
    degenerate = (S == 0)
    idx = np.where(degenerate[..., None], 0, idx)
    idx[..., 0] = np.where(degenerate, len(L) - 1, idx[..., 0])
    sign = np.where(degenerate[..., None], True, pos)
    nib = ((sign.astype(np.int64) << 3) | idx).astype(np.uint8).reshape(n, D)
    codes = (nib[:, 0::2] | (nib[:, 1::2] << 4)).astype(np.uint8)
    # (3) polar form of the rotated unit key
    knorm = np.sqrt(np.sum(K * K, axis=-1))
    Stot = np.sum(S, axis=-1)
    safe_tot = np.where(Stot > 0, Stot, 1.0)
    r = np.sqrt(S / safe_tot[:, None])
    _, u = transform.polar(yb)
    # dequantised direction v_b = renormalised (sign * L[idx]) (AMB-6)
    vt = np.where(sign, 1.0, -1.0) * L[idx]
    vnorm = np.sqrt(np.sum(vt * vt, axis=-1))
    v = vt / vnorm[..., None]
    if exact_codes:
        v = u.copy()
    alpha = np.maximum(np.sum(v * u, axis=-1), ALPHA_FLOOR)          # Eq. 7
    w = knorm[:, None] * r / alpha                                    # Eq. 9
    w = np.where(degenerate, 0.0, w)
    return dict(ids=ids, nib=nib, codes=codes, w=w, alpha=alpha, v=v, vnorm=vnorm,
                y=y, S=S, knorm=knorm, u=u, r=r)


def unpack_codes(codes: np.ndarray) -> np.ndarray:
    """Inverse of the packing: [n, D/2] bytes -> [n, D] nibbles."""
    codes = np.asarray(codes, dtype=np.uint8)
    n, half = codes.shape
    out = np.empty((n, 2 * half), dtype=np.uint8)
    out[:, 0::2] = codes & 0xF
    out[:, 1::2] = codes >> 4
    return out


def dequantize(nib: np.ndarray, levels32: np.ndarray, B: int = 16) -> np.ndarray:
    """v_b = renormalised (sign * L[idx]) from nibbles [n, D] -> [n, B, m] ("dequantizes to v")."""
    nib = np.asarray(nib).astype(np.int64)
    L = np.asarray(levels32, dtype=np.float32).astype(np.float64)
    vt = np.where((nib >> 3) & 1, 1.0, -1.0) * L[nib & 7]
    vt = transform.split(vt, B)
    return vt / np.sqrt(np.sum(vt * vt, axis=-1, keepdims=True))
