"""Preprocessing: normalise, SRHT rotation, subspace split, polar form (PAPER §4.1.1).

Reading AMB-1: R = H_D diag(s) / sqrt(D), H_D the Sylvester-ordered
Walsh-Hadamard matrix (H_{ij} = (-1)^{popcount(i & j)}), s_j = +1 if sign bit 0,
-1 if sign bit 1, one round, shared by every key and query ("a shared
orthogonal rotation R (implemented by SRHT)").

Reading AMB-2: every discrete decision (centroid id, code) depends only on the
direction of the rotated vector, so the oracle works with the UNSCALED rotated
vector  y' = H_D (s (.) x)  (no 1/sqrt(D), no 1/||x||); both factors are
positive and cancel in every decision. y' is computed with radix-2 butterflies
in fp64 in the fixed order h = 1, 2, 4, ..., D/2, pair (i, i+h) -> (a+b, a-b).
For bf16 inputs every butterfly is exact unless the key spans > ~38 binades
(pin P2 checks exactness against integer arithmetic).
"""
from __future__ import annotations

import numpy as np


def l2_normalize(x: np.ndarray):
    """k_hat = k / ||k||_2. Returns (unit vector, norm); zero rows stay zero."""
    x = np.asarray(x, dtype=np.float64)
    nrm = np.sqrt(np.sum(x * x, axis=-1, keepdims=True))
    safe = np.where(nrm > 0, nrm, 1.0)
    return x / safe, nrm[..., 0]


def sign_vector(rot_sign_bits: np.ndarray) -> np.ndarray:
    """s_j in {+1,-1} from the config's sign bits (0 -> +1, 1 -> -1)."""
    return np.where(np.asarray(rot_sign_bits) != 0, -1.0, 1.0)


def fwht(x: np.ndarray) -> np.ndarray:
    """Unnormalised Walsh-Hadamard transform along the last axis, radix-2 butterflies in fp64.

    Stage order h = 1, 2, 4, ...; within a stage the pair (i, i+h) becomes (a+b, a-b)
    with a = x[i], b = x[i+h]. Returns H_D x (Sylvester ordering)."""
    y = np.array(x, dtype=np.float64, copy=True)
    D = y.shape[-1]
    assert D & (D - 1) == 0, "D must be a power of two"
    h = 1
    while h < D:
        for i in range(0, D, 2 * h):
            a = y[..., i:i + h].copy()
            b = y[..., i + h:i + 2 * h].copy()
            y[..., i:i + h] = a + b
            y[..., i + h:i + 2 * h] = a - b
        h *= 2
    return y


def rotate_unscaled(x: np.ndarray, rot_sign_bits: np.ndarray) -> np.ndarray:
    """y' = H_D (s (.) x): the rotated vector times sqrt(D) (and times ||x|| if x is raw).

    R x = y' / sqrt(D). The sign flip is exact, the FWHT is the fixed butterfly order above."""
    s = sign_vector(rot_sign_bits)
    return fwht(np.asarray(x, dtype=np.float64) * s)


def rotate(x_unit: np.ndarray, rot_sign_bits: np.ndarray) -> np.ndarray:
    """k_tilde = R k_hat, R = H diag(s)/sqrt(D)."""
    D = np.asarray(x_unit).shape[-1]
    return rotate_unscaled(x_unit, rot_sign_bits) / np.sqrt(D)


def split(x: np.ndarray, B: int) -> np.ndarray:
    """B contiguous subspaces of dimension m = D/B: [..., D] -> [..., B, m]."""
    x = np.asarray(x)
    D = x.shape[-1]
    assert D % B == 0
    return x.reshape(*x.shape[:-1], B, D // B)


def polar(x_split: np.ndarray):
    """Per-subspace polar form: r_b = ||x_b||, u_b = x_b / r_b.

    Zero-radius subspaces (reading AMB-7): u_b := e_1, r_b = 0."""
    x_split = np.asarray(x_split, dtype=np.float64)
    r = np.sqrt(np.sum(x_split * x_split, axis=-1))
    safe = np.where(r > 0, r, 1.0)[..., None]
    u = x_split / safe
    e1 = np.zeros(x_split.shape[-1])
    e1[0] = 1.0
    u = np.where((r > 0)[..., None], u, e1)
    return r, u


def blockwise_ip(rk, uk, rq, uq) -> np.ndarray:
    """Eq. 4: <k~, q~> = sum_b r_b^k r_b^q <u_b^k, u_b^q>."""
    return np.sum(rk * rq * np.sum(uk * uq, axis=-1), axis=-1)


def hadamard_matrix_kron(D: int) -> np.ndarray:
    """Explicit Sylvester Hadamard H_D by Kronecker products (used only as an independent pin, P1)."""
    H = np.array([[1.0]])
    H2 = np.array([[1.0, 1.0], [1.0, -1.0]])
    while H.shape[0] < D:
        H = np.kron(H, H2)
    return H
