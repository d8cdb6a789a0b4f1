"""-m gpu: the library's sequence-sharded path in TWO processes through the C ABI.

Each process is one rank owning a contiguous token shard in its own pkv_index; the exchanges (H) histograms,
(T) local top-k lists, (A) attention partials, and the fused T+A message run through pkv_comm_init_host with a
gloo all-gather on the host (NCCL cannot put two ranks on the single GPU of the test box; the kernels and the
exchange buffers are the same ones the NCCL transport uses). Every rank must return the unsharded result:
bit-identical ids and estimates, attention against the fp64 oracle at the AMB-17 bar."""
from __future__ import annotations

import os
import socket
import traceback

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

WORLD = 2


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, port, result_dir):
    import torch.distributed as dist

    import synth
    from oracle import pipeline
    from paper_2602_07721_b200 import pariskv as pkv
    from tests.gpu_helpers import SB, bf16_f64, check_attention
    from tests.test_parity_gpu import make_problem

    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=WORLD)
        torch.cuda.set_device(0)
        batch, n_q, n_kv, n, k, n_hot = 2, 8, 2, 9000, 100, 40
        K, q, V = make_problem(101, batch, n_q, n_kv, n)
        Kh = synth.isotropic(102, (batch, n_kv, n_hot, 128), device="cuda")
        Vh = synth.isotropic(103, (batch, n_kv, n_hot, 128), device="cuda")
        cfg = pkv.config_init(n_q, n_kv, SB)
        full = pkv.Index(cfg, batch, n)
        pkv.encode_keys(full, K)
        i0, e0, _ = pkv.retrieve_topk(full, q, k)
        bounds = [n * r // WORLD for r in range(WORLD + 1)]
        lo, hi = bounds[rank], bounds[rank + 1]
        Kl, Vl = K[:, :, lo:hi].contiguous(), V[:, :, lo:hi].contiguous()
        ix = pkv.Index(cfg, batch, hi - lo)
        pkv.encode_keys(ix, Kl)
        torch.cuda.synchronize()

        def allgather(arr):  # arr: uint8 [world, nbytes] host view, row `rank` filled
            mine = torch.from_numpy(arr[rank].copy())
            parts = [torch.empty_like(mine) for _ in range(WORLD)]
            dist.all_gather(parts, mine)
            for r in range(WORLD):
                arr[r] = parts[r].numpy()

        pkv.comm_init_host(ix, allgather, rank, WORLD, lo)
        last = rank == WORLD - 1
        hk, hv = (Kh, Vh) if last else (None, None)
        out32 = torch.full((batch, n_q, 128), float("nan"), device="cuda")
        ix.set_debug_output(out32)
        # three-exchange path: retrieve_topk (H, T) then sparse_attend (A)
        i1, e1, _ = pkv.retrieve_topk(ix, q, k, n_global=n)  # T and C from the global schedule
        o1, l1 = pkv.sparse_attend(ix, q, Kl, Vl, i1, hk, hv)
        torch.cuda.synchronize()
        assert torch.equal(i0, i1) and torch.equal(e0, e1), f"rank {rank}: sharded top-k differs"
        o32a = out32.clone()
        # fused T+A path (two exchanges); params.n_global = 0: the length recorded at comm init (sum of shards)
        T, C = pkv.schedule(n, k)
        i2, e2, o2, l2 = pkv.retrieve_and_attend(ix, q, Kl, Vl, k, hk, hv, probes_T=T, n_cand=C)
        torch.cuda.synchronize()
        assert torch.equal(i0, i2) and torch.equal(e0, e2), f"rank {rank}: fused top-k differs"
        for b in range(batch):
            for h in range(n_q):
                g = h // (n_q // n_kv)
                o, l = pipeline.attend(bf16_f64(q[b, h]), bf16_f64(K[b, g]), bf16_f64(V[b, g]), i0[b, h].cpu().numpy(),
                                       bf16_f64(Kh[b, g]), bf16_f64(Vh[b, g]))
                check_attention(o1[b, h].float().cpu().numpy(), o, o32a[b, h].cpu().numpy(), l1[b, h], l,
                                f"rank {rank} 3-exchange b{b} h{h}")
                check_attention(o2[b, h].float().cpu().numpy(), o, out32[b, h].cpu().numpy(), l2[b, h], l,
                                f"rank {rank} fused b{b} h{h}")
        # argument validation against the global length: n_cand above it is refused on every rank
        with pytest.raises(pkv.PkvError):
            pkv.retrieve_topk(ix, q, k, n_cand=n + 1)
        np.save(os.path.join(result_dir, f"out{rank}.npy"), o2.float().cpu().numpy())
        dist.barrier()
        dist.destroy_process_group()
    except BaseException:
        traceback.print_exc()
        raise


def test_two_process_host_exchange_equals_unsharded(tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2602_07721_b200 import build
    build.build()
    ctx = torch.multiprocessing.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, str(tmp_path))) for r in range(WORLD)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(600)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    a, b = (np.load(tmp_path / f"out{r}.npy") for r in range(WORLD))
    assert np.array_equal(a, b)  # the merged output is replicated bit for bit
