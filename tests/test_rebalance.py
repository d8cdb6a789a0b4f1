"""Append rebalancing across sequence shards: decode appends grow the last rank's shard;
a boundary shift moves the oldest keys of shard r+1 to the end of shard r.

-m "not gpu": the library's host-only policy pkv_rebalance_plan (conservation, order, feasibility, balance) and the
protocol over a real process group (world 2, gloo): the ranks agree on the plan from all-gathered lengths, rank 1
sends its oldest entries (oracle-encoded records, position-independent) to rank 0, and afterwards every rank holds
exactly the oracle encoding of its new position range.
-m gpu: export_front / import_back / drop_front / shift_boundary on real indices — the shards' contents equal the
unsharded index's, and the sharded retrieval stays bit-identical to the unsharded one."""
from __future__ import annotations

import os
import random
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth
from oracle import levels, quantizer

SB = synth.rotation_sign_bits()


def _plan(lengths, granule):
    from paper_2602_07721_b200 import pariskv
    return pariskv.rebalance_plan(lengths, granule)


def _apply(lengths, shift):
    """Apply shift[P-2] first, shift[0] last; every move must be feasible when it happens."""
    n = list(lengths)
    for r in range(len(n) - 2, -1, -1):
        assert 0 <= shift[r] <= n[r + 1], (lengths, shift, r)
        n[r + 1] -= shift[r]
        n[r] += shift[r]
    return n


def test_rebalance_plan_properties():
    rng = random.Random(7)
    for _ in range(400):
        P = rng.randint(1, 8)
        g = rng.choice([1, 16, 512])
        lengths = [rng.randint(0, 200000) for _ in range(P)]
        if rng.random() < 0.5:  # decode appends on the last rank only (the case the policy is for)
            base = rng.randint(0, 100000)
            lengths = [base] * (P - 1) + [base + rng.randint(0, 50) * 512]
        shift = _plan(lengths, g)
        assert len(shift) == P - 1
        new = _apply(lengths, shift)
        N = sum(lengths)
        assert sum(new) == N and min(new) >= 0
        old_b = np.cumsum([0] + lengths)[:-1]
        new_b = np.cumsum([0] + new)[:-1]
        assert (new_b >= old_b).all()  # boundaries only move right
        for r in range(1, P):
            target = r * N // P
            # never past the balanced position (unless already right of it); within one granule of it, unless the
            # next boundary stops it (shards shorter than a granule)
            assert new_b[r] <= max(old_b[r], target)
            if old_b[r] <= target:
                assert target - new_b[r] < g or (r < P - 1 and new_b[r] == new_b[r + 1])
    # balanced shards need no move; one flush on the last of 4 equal shards moves whole granules leftwards
    assert _plan([4096] * 4, 512) == [0, 0, 0]
    assert _plan([131072] * 3 + [131072 + 8 * 512], 512) == [1024, 2048, 3072]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _entries(K, lo, hi):
    """Oracle encoding of positions [lo, hi): a key's entry does not depend on its position."""
    L32 = levels.levels_f32(8)
    meta = quantizer.encode_keys(K[lo:hi], SB, L32, levels.mid_sq(L32))
    return np.concatenate([meta["ids"].astype(np.float64), meta["codes"].astype(np.float64), meta["w"]], axis=1)


def _worker(rank, world, port, q_out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = 2600
        K = synth.to_f64(synth.llm_keys(41, 1, 1, n)[0, 0])
        split = [600, n]  # rank 1's shard has grown by decode appends
        lo, hi = (0, split[0]) if rank == 0 else (split[0], split[1])
        mine = _entries(K, lo, hi)
        lens = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(lens, torch.tensor([len(mine)], dtype=torch.int64))
        lengths = [int(x.item()) for x in lens]
        shift = _plan(lengths, 16)
        moved = shift[0]
        if rank == 1:  # the oldest `moved` entries go to rank 0, this shard keeps the rest
            dist.send(torch.from_numpy(np.ascontiguousarray(mine[:moved])), dst=0)
            mine = mine[moved:]
            lo += moved
        else:
            buf = torch.zeros(moved, mine.shape[1], dtype=torch.float64)
            dist.recv(buf, src=1)
            mine = np.concatenate([mine, buf.numpy()])
            hi += moved
        ok = np.array_equal(mine, _entries(K, lo, hi))
        q_out.put((rank, lengths, shift, lo, hi, bool(ok)))
    finally:
        dist.destroy_process_group()


def test_rebalance_protocol_gloo_two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, len0, sh0, lo0, hi0, ok0), (r1, len1, sh1, lo1, hi1, ok1) = res
    assert len0 == len1 == [600, 2000] and sh0 == sh1 == [688]  # both ranks computed the same plan
    assert (lo0, hi0, lo1, hi1) == (0, 1288, 1288, 2600)       # contiguous, balanced to a granule
    assert ok0 and ok1


# ---------------------------------------------------------------------------------------------------- GPU
@pytest.fixture(scope="module")
def pkv():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2602_07721_b200 import build
    build.build()
    from paper_2602_07721_b200 import pariskv
    return pariskv


@pytest.mark.gpu
def test_shift_boundary_keeps_sharded_results(pkv):
    n = 20000
    K = synth.llm_keys(43, 1, 2, n, device="cuda")
    q = synth.llm_queries(43, 1, 8, 2, device="cuda")
    synth.plant(K, q, 43)
    cfg = pkv.config_init(8, 2, SB)
    full = pkv.Index(cfg, 1, n)
    pkv.encode_keys(full, K)
    i0, e0, _ = pkv.retrieve_topk(full, q, 100)
    ids0, codes0, w0 = full.export()
    lengths = [3000, 4000, 13000]  # the last shard grew by appends
    bounds = np.cumsum([0] + lengths)
    shards = []
    for a, b in zip(bounds[:-1], bounds[1:]):
        s = pkv.Index(cfg, 1, n)  # room for what it receives
        pkv.encode_keys(s, K[:, :, a:b].contiguous())
        shards.append(s)
    shift = pkv.rebalance_plan(lengths, 512)
    assert shift == [3584, 6144]
    # boundary 2 through the three explicit steps (as two ranks would run them), boundary 1 in one call
    buf = shards[2].export_front(shift[1])
    shards[1].import_back(buf, shift[1])
    shards[2].drop_front(shift[1])
    pkv.shift_boundary(shards[0], shards[1], shift[0])
    new_len = [len(s) for s in shards]
    assert new_len == [6584, 6560, 6856] and sum(new_len) == n
    offs = [0, new_len[0], new_len[0] + new_len[1]]
    # contents: every shard equals the unsharded index over its new position range (canonical ids, codes, w)
    for s, a, m in zip(shards, offs, new_len):
        ids, codes, w = s.export(0, m)
        assert torch.equal(ids, ids0[:, :, a:a + m]) and torch.equal(codes, codes0[:, :, a:a + m])
        assert torch.equal(w, w0[:, :, a:a + m])
    # results: the sharded retrieval over the rebalanced shards is the unsharded one, bit for bit
    i1, e1 = pkv.retrieve_topk_sharded_local(shards, offs, q, 100, n)
    torch.cuda.synchronize()
    assert torch.equal(i0, i1) and torch.equal(e0, e1)
    # a shard's own (unsharded) ids are now global positions: its offset grew by what it gave away
    i2, e2, _ = pkv.retrieve_topk(shards[2], q, 100)
    assert int(i2.min()) >= shift[1] and int(i2.max()) < shift[1] + new_len[2]


@pytest.mark.gpu
def test_rebalance_argument_errors(pkv):
    cfg = pkv.config_init(8, 2, SB)
    a = pkv.Index(cfg, 1, 100)
    b = pkv.Index(cfg, 1, 100)
    K = synth.llm_keys(44, 1, 2, 100, device="cuda")
    pkv.encode_keys(a, K[:, :, :60].contiguous())
    pkv.encode_keys(b, K[:, :, 60:].contiguous())
    with pytest.raises(RuntimeError):
        pkv.shift_boundary(a, b, 41)  # b holds 40 keys
    with pytest.raises(RuntimeError):
        pkv.shift_boundary(b, a, 61)  # more than a holds
    pkv.shift_boundary(a, b, 40)  # capacity 100 >= 60 + 40
    assert len(a) == 100 and len(b) == 0
    with pytest.raises(RuntimeError):  # a is full
        a.import_back(torch.zeros(a.entry_bytes(), dtype=torch.uint8, device="cuda"), 1)
