"""-m gpu: the peer exchange transport (peer.cu): one-shot all-gather kernels over peer memory
instead of NCCL. Ranks share the one GPU of the test box: in one process (one host thread per rank, arenas
connected by pointer) and in two processes (arenas opened through CUDA IPC). Every rank must return the unsharded
result: bit-identical ids and estimates, attention against the fp64 oracle at the AMB-17 bar."""
from __future__ import annotations

import os
import socket
import threading
import traceback

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkv():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2602_07721_b200 import build
    build.build()
    from paper_2602_07721_b200 import pariskv
    return pariskv


def _problem(seed, P):
    import synth
    from tests.test_parity_gpu import make_problem
    batch, n_q, n_kv, n = 1, 8, 2, 9000  # small grids: the ranks' kernels co-reside on the one GPU
    K, q, V = make_problem(seed, batch, n_q, n_kv, n)
    Kh = synth.isotropic(seed + 1, (batch, n_kv, 40, 128), device="cuda")
    Vh = synth.isotropic(seed + 2, (batch, n_kv, 40, 128), device="cuda")
    bounds = [n * r // P for r in range(P + 1)]
    return K, q, V, Kh, Vh, bounds


def _check_rank(pkv, K, q, V, Kh, Vh, res, ref):
    from oracle import pipeline
    from tests.gpu_helpers import bf16_f64, check_attention
    idx, est, out, lse = res
    assert torch.equal(idx, ref[0]) and torch.equal(est, ref[1])
    for h in range(q.shape[1]):
        g = h // (q.shape[1] // K.shape[1])
        o, l = pipeline.attend(bf16_f64(q[0, h]), bf16_f64(K[0, g]), bf16_f64(V[0, g]), idx[0, h].cpu().numpy(),
                               bf16_f64(Kh[0, g]), bf16_f64(Vh[0, g]))
        check_attention(out[0, h].float().cpu().numpy(), o, None, lse[0, h], l, f"peer h={h}")


@pytest.mark.parametrize("P", [2, 3, 4])
def test_peer_transport_one_process(pkv, P):
    from tests.gpu_helpers import SB
    K, q, V, Kh, Vh, bounds = _problem(301, P)
    n, k = K.shape[2], 100
    cfg = pkv.config_init(q.shape[1], K.shape[1], SB)
    full = pkv.Index(cfg, 1, n)
    pkv.encode_keys(full, K)
    ref = pkv.retrieve_topk(full, q, k)[:2]
    shards, arenas, Ks, Vs = [], [], [], []
    for r in range(P):
        lo, hi = bounds[r], bounds[r + 1]
        ix = pkv.Index(cfg, 1, hi - lo)
        Ks.append(K[:, :, lo:hi].contiguous())
        Vs.append(V[:, :, lo:hi].contiguous())
        pkv.encode_keys(ix, Ks[-1])
        _, a = ix.comm_init_peer(r, P, lo, 16 << 20)
        shards.append(ix)
        arenas.append(a)
    for ix in shards:
        ix.comm_peer_connect_local(arenas)
    torch.cuda.synchronize()
    results, errors = [None] * P, []

    def rank_main(r):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                hot = (Kh, Vh) if r == P - 1 else (None, None)
                for _ in range(3):  # several steps: the exchange epochs and arena parities advance
                    res = pkv.retrieve_and_attend(shards[r], q, Ks[r], Vs[r], k, *hot, n_global=n, stream=s)
                s.synchronize()
            results[r] = res
        except Exception:
            errors.append(traceback.format_exc())

    threads = [threading.Thread(target=rank_main, args=(r,)) for r in range(P)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=120)
    assert not any(t.is_alive() for t in threads), "peer exchange did not complete"
    assert not errors, errors[0]
    for r in range(P):
        _check_rank(pkv, K, q, V, Kh, Vh, results[r], ref)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _ipc_worker(rank, port, result_dir):
    import torch.distributed as dist

    from paper_2602_07721_b200 import pariskv as pkv
    from tests.gpu_helpers import SB
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=2)
        torch.cuda.set_device(0)
        K, q, V, Kh, Vh, bounds = _problem(302, 2)
        n, k = K.shape[2], 100
        cfg = pkv.config_init(q.shape[1], K.shape[1], SB)
        full = pkv.Index(cfg, 1, n)
        pkv.encode_keys(full, K)
        ref = pkv.retrieve_topk(full, q, k)[:2]
        lo, hi = bounds[rank], bounds[rank + 1]
        Kl, Vl = K[:, :, lo:hi].contiguous(), V[:, :, lo:hi].contiguous()
        ix = pkv.Index(cfg, 1, hi - lo)
        pkv.encode_keys(ix, Kl)
        handle, _ = ix.comm_init_peer(rank, 2, lo, 16 << 20)
        handles = [None, None]
        dist.all_gather_object(handles, handle)
        ix.comm_peer_connect(handles)
        torch.cuda.synchronize()
        dist.barrier()
        hot = (Kh, Vh) if rank == 1 else (None, None)
        for _ in range(2):
            res = pkv.retrieve_and_attend(ix, q, Kl, Vl, k, *hot, n_global=n)
        torch.cuda.synchronize()
        _check_rank(pkv, K, q, V, Kh, Vh, res, ref)
        dist.barrier()
        open(os.path.join(result_dir, f"ok{rank}"), "w").write("ok")
        dist.destroy_process_group()
    except Exception:
        open(os.path.join(result_dir, f"err{rank}"), "w").write(traceback.format_exc())


def test_peer_transport_two_processes_ipc(pkv, tmp_path):
    import torch.multiprocessing as mp
    port = _free_port()
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_ipc_worker, args=(r, port, str(tmp_path))) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    for p in procs:
        if p.is_alive():
            p.kill()
    errs = [open(os.path.join(tmp_path, f)).read() for f in os.listdir(tmp_path) if f.startswith("err")]
    assert not errs, errs[0]
    assert all(os.path.exists(os.path.join(tmp_path, f"ok{r}")) for r in range(2)), "peer IPC ranks did not finish"
