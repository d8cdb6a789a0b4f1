"""Prop. 1 magnitude levels for the 3-bit part of the 4-bit direction code.

PAPER.md P:487 ("The derivation of the theoretical quantization levels for the
normalized-and-rotated subspace directions is guided by Proposition 1") and
Prop. 1, Eq. (coord_beta_prop): (u_b)_j^2 ~ Beta(1/2, (m-1)/2).

Reading AMB-5: the 8 levels are the
conditional means of |u_j| over the 8 equal-probability bins of |u_j|, and a
coordinate is encoded to the nearest level (midpoint rule).

Closed form used here (library special functions as single steps):
with X = u_j^2 ~ Beta(a, b), a = 1/2, b = (m-1)/2,
    bin edges   e_i = sqrt(I^{-1}(i/8; a, b))                  i = 0..8
    level       L_i = 8 * E[sqrt(X) 1{e_i^2 <= X < e_{i+1}^2}]
                    = 8 * B(a+1/2, b)/B(a, b) * (I(e_{i+1}^2; a+1/2, b) - I(e_i^2; a+1/2, b))
where I is the regularised incomplete beta function.
"""
from __future__ import annotations

import numpy as np
from scipy import special

N_LEVELS = 8  # 3-bit magnitude ("1-bit sign + 3-bit magnitude")


def bin_edges(m: int) -> np.ndarray:
    """Equal-probability bin edges of |u_j| (9 values, 0 and 1 included). AMB-5."""
    a, b = 0.5, (m - 1) / 2.0
    p = np.arange(N_LEVELS + 1) / N_LEVELS
    x = special.betaincinv(a, b, p)
    x[0], x[-1] = 0.0, 1.0
    return np.sqrt(x)


def design_levels(m: int) -> np.ndarray:
    """fp64 conditional-mean levels L_0 < ... < L_7 (Prop. 1, AMB-5)."""
    a, b = 0.5, (m - 1) / 2.0
    e2 = bin_edges(m) ** 2
    scale = np.exp(special.betaln(a + 0.5, b) - special.betaln(a, b))
    cdf = special.betainc(a + 0.5, b, e2)
    return N_LEVELS * scale * np.diff(cdf)


def levels_f32(m: int) -> np.ndarray:
    """The levels as stored in the config (fp32). DESIGN.md reading AMB-5b:
    both sides use these fp32 values, so the decision constants below are exact."""
    return design_levels(m).astype(np.float32)


def mid_sq(levels32: np.ndarray) -> np.ndarray:
    """Decision constants M_t = ((L_{t-1} + L_t)/2)^2, t = 1..7, in fp64.

    For fp32 L the sum, the halving and the square are all exact in fp64
    (<= 25-bit significands), so M_t is a pure function of the fp32 levels.
    |u_j| >= (L_{t-1}+L_t)/2  <=>  y_j^2 >= M_t * S_b  (S_b = ||y_b||^2, y_b = unscaled rotated subvector).
    """
    L = levels32.astype(np.float64)
    mids = (L[:-1] + L[1:]) / 2.0
    return mids * mids


def expected_abs_coordinate(m: int) -> float:
    """E|u_j| = Gamma(m/2) / (sqrt(pi) Gamma((m+1)/2)) for u uniform on S^{m-1} (closed form, pin P7)."""
    return float(np.exp(special.gammaln(m / 2.0) - special.gammaln((m + 1) / 2.0)) / np.sqrt(np.pi))
