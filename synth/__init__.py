"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

Holds NONE of the method's arithmetic: only random draws with the shapes and value structure of the
paper's workloads (DESIGN.md §Input recipe). Everything is bf16 at the boundary
(reading AMB-21); `to_f64` gives the exact fp64 values of a bf16 tensor for the oracle.

Recipe (per KV head h, seed = 1000 * layer + head unless stated):
  keys     K = mu_h + sigma_h (.) z,  mu_h ~ N(0, I), log sigma_h ~ N(0, 0.6^2), 4 outlier channels x8
  queries  q = 0.2 mu_h + 0.5 sigma_h (.) z'       (one per query head of the GQA group)
  planted  per query head, `n_plant` keys replaced by  a * s_typ * q_hat + 0.5 z,  a ~ U[1.5, 2.5],
           s_typ = median key norm, so that the exact top-k is well defined
  values   V ~ N(0, I)
  drift    (config 4) key t ~ N(mu0 + t * rate * delta, I); queries are noised copies of
           recent keys
"""
from __future__ import annotations

import numpy as np
import torch


def rotation_sign_bits(seed: int = 20260207, D: int = 128) -> np.ndarray:
    """SRHT sign bits s_j in {0,1} (0 -> +1), drawn by the harness (AMB-1)."""
    rng = np.random.default_rng(seed)
    return rng.integers(0, 2, size=D).astype(np.uint8)


def to_f64(t: torch.Tensor) -> np.ndarray:
    """Exact fp64 values of a bf16 (or any float) tensor."""
    return t.detach().to("cpu", torch.float64).numpy()


def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    return g


def head_stats(seed: int, n_kv: int, D: int = 128, device="cpu"):
    """(mu [n_kv, D], sigma [n_kv, D]) of the LLM-like key model."""
    g = _gen(seed, device)
    mu = torch.randn(n_kv, D, generator=g, device=device)
    sig = torch.exp(0.6 * torch.randn(n_kv, D, generator=g, device=device))
    out_ch = torch.stack([torch.randperm(D, generator=g, device=device)[:4] for _ in range(n_kv)])
    sig.scatter_(1, out_ch, sig.gather(1, out_ch) * 8.0)
    return mu, sig


def llm_keys(seed: int, batch: int, n_kv: int, n: int, D: int = 128, device="cpu",
             dtype=torch.bfloat16, stats=None) -> torch.Tensor:
    """K [batch, n_kv, n, D] bf16 following the recipe (no planting)."""
    mu, sig = head_stats(seed, n_kv, D, device) if stats is None else stats
    g = _gen(seed + 1, device)
    K = torch.empty(batch, n_kv, n, D, device=device, dtype=dtype)
    step = 1 << 16
    for b in range(batch):
        for t0 in range(0, n, step):
            t1 = min(n, t0 + step)
            z = torch.randn(n_kv, t1 - t0, D, generator=g, device=device)
            K[b, :, t0:t1] = (mu[:, None, :] + sig[:, None, :] * z).to(dtype)
    return K


def llm_queries(seed: int, batch: int, n_q: int, n_kv: int, D: int = 128, device="cpu",
                dtype=torch.bfloat16, stats=None) -> torch.Tensor:
    """q [batch, n_q, D]: q = 0.2 mu_h + 0.5 sigma_h (.) z' for the KV head h of each query head."""
    mu, sig = head_stats(seed, n_kv, D, device) if stats is None else stats
    g = _gen(seed + 2, device)
    G = n_q // n_kv
    kv = torch.arange(n_q, device=device) // G
    z = torch.randn(batch, n_q, D, generator=g, device=device)
    return (0.2 * mu[kv][None] + 0.5 * sig[kv][None] * z).to(dtype)


def plant(K: torch.Tensor, q: torch.Tensor, seed: int, n_plant: int = 25) -> torch.Tensor:
    """Replace n_plant keys per query head by  a * s_typ * q_hat + 0.5 z  (in place). Returns positions
    [batch, n_q, n_plant]. Keys of different query heads of one KV head do not collide."""
    batch, n_kv, n, D = K.shape
    n_q = q.shape[1]
    G = n_q // n_kv
    dev = K.device
    g = _gen(seed + 3, dev)
    pos = torch.empty(batch, n_q, n_plant, dtype=torch.long, device=dev)
    s_typ = K[:, :, : min(n, 4096)].float().norm(dim=-1).median()
    for b in range(batch):
        for h in range(n_kv):
            p = torch.randperm(n, generator=g, device=dev)[: G * n_plant].view(G, n_plant)
            for j in range(G):
                qh = q[b, h * G + j].float()
                qh = qh / qh.norm()
                a = 1.5 + torch.rand(n_plant, 1, generator=g, device=dev)
                z = torch.randn(n_plant, D, generator=g, device=dev)
                K[b, h, p[j]] = (a * s_typ * qh[None] + 0.5 * z).to(K.dtype)
                pos[b, h * G + j] = p[j]
    return pos


def values(seed: int, batch: int, n_kv: int, n: int, D: int = 128, device="cpu", dtype=torch.bfloat16):
    g = _gen(seed + 4, device)
    V = torch.empty(batch, n_kv, n, D, device=device, dtype=dtype)
    step = 1 << 16
    for b in range(batch):
        for t0 in range(0, n, step):
            t1 = min(n, t0 + step)
            V[b, :, t0:t1] = torch.randn(n_kv, t1 - t0, D, generator=g, device=device).to(dtype)
    return V


def isotropic(seed: int, shape, device="cpu", dtype=torch.bfloat16) -> torch.Tensor:
    """Standard normal bf16 tensor (SPEC gen_isotropic)."""
    g = _gen(seed, device)
    return torch.randn(*shape, generator=g, device=device).to(dtype)


def drift_keys(seed: int, n_prefill: int, n_decode: int, rate: float, D: int = 128, device="cpu",
               dtype=torch.bfloat16):
    """SPEC gen_drift: prefill ~ N(mu0, I); decode key t ~ N(mu0 + t rate delta, I).
    Returns (K [n_prefill + n_decode, D], delta [D])."""
    g = _gen(seed, device)
    mu0 = torch.randn(D, generator=g, device=device)
    delta = torch.randn(D, generator=g, device=device)
    delta = delta / delta.norm()
    Kp = mu0 + torch.randn(n_prefill, D, generator=g, device=device)
    t = torch.arange(n_decode, device=device, dtype=torch.float32)[:, None]
    Kd = mu0 + t * rate * delta + torch.randn(n_decode, D, generator=g, device=device)
    return torch.cat([Kp, Kd]).to(dtype), delta


def drift_query(seed: int, K_recent: torch.Tensor, noise: float = 0.3, dtype=torch.bfloat16):
    """A noised copy of a random recent key."""
    g = _gen(seed, K_recent.device)
    i = int(torch.randint(len(K_recent), (1,), generator=g, device=K_recent.device))
    z = torch.randn(K_recent.shape[-1], generator=g, device=K_recent.device)
    return (K_recent[i].float() + noise * z).to(dtype)
