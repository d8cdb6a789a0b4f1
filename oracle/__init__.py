"""CPU oracle for the ParisKV decode-time retrieval hot path (TEST INFRASTRUCTURE ONLY).

This package is a plain, slow, fp64 NumPy restatement of what ParisKV
(arXiv 2602.07721, "PAPER.md") computes, written to check the CUDA path.
It is NOT part of the product:

* only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
  ``cpu_baseline`` / ``--impl reference`` legs may import it;
* it shares no code, table or constant generator with
  ``paper_2602_07721_b200`` (the CUDA path) and imports nothing from it;
* the product path never calls it and has no CPU fallback.

Citations: ``P:n`` = PAPER.md line n (section / equation in brackets),
``S:n`` = SPEC.md line n, ``AMB-x`` = a reading listed in DESIGN.md.

Modules (each function cites the passage it follows):

* ``levels``     Prop. 1 magnitude levels
* ``transform``  normalise / SRHT rotation / subspace split / polar
* ``codebook``   analytic centroids Omega, assignment, probe ranking, tiers
* ``quantizer``  4-bit codes, alpha, w (Eq. 7-10)
* ``coarse``     (rho, beta) schedule, collision scores, bucket_topk
* ``rerank``     RSQ-IP estimate (Eq. 10) and final top-k
* ``attention``  Eq. 1-3 attention, exact top-k, recall
* ``pipeline``   one decode step for one (sequence, KV group) unit
* ``sharded``    P-shard emulation of the sequence-sharded decode

Parity status: every function is pinned by ``tests/test_oracle_pins.py``
except the recall values of the paper, which come
from model traces: *parity unpinned* for those numbers.
"""

from . import levels, transform, codebook, quantizer, coarse, rerank, attention, pipeline, sharded  # noqa: F401
