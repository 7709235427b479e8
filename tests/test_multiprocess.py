"""Expert-parallel host logic at world_size 2 over gloo (CPU).

Each rank runs the product scheduler in sharded mode (expert e on rank
e % G). The ranks must derive identical tau / residency / ratio estimates
with no communication, each rank must own only its shard's residents, and
the per-rank partial MoE outputs (oracle FFN over the rank's resident
experts) must all-reduce to the single-device result.
"""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2603_09983_b200 import abi


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        L, N, k, g, d, ffn = 3, 16, 4, 6, 64, 32
        T = g + 1
        cfg = abi.default_config(n_layers=L, n_experts=N, top_k=k, gamma=g, cache_ratio=0.5)
        s = abi.Scheduler(cfg, world)
        gen = O.Generator(L, N, k, g, seed=1)
        rng = np.random.default_rng(0)  # same weights on every rank
        W = {(l, e): tuple(O.f32_to_bf16_bits(rng.normal(0, 0.05, sh).astype(np.float32))
                           for sh in ((ffn, d), (ffn, d), (d, ffn))) for l in range(L) for e in range(N)}
        est = [O.estimator_init(N, g) for _ in range(L)]
        scores = np.zeros((L, N), np.int32)
        for step in range(12):
            s.decide(scores)
            taus, rb, lb, slots = s.tables()
            dec = s.decisions()
            # identical decisions on every rank
            for arr in (taus, rb.view(np.int32), dec[:, :2].astype(np.int64)):
                t = torch.from_numpy(np.ascontiguousarray(arr).astype(np.int64).ravel())
                ts = [torch.zeros_like(t) for _ in range(world)]
                dist.all_gather(ts, t)
                assert all(torch.equal(ts[0], x) for x in ts)
            logits, ids, acc = gen.next_step()
            h = O.f32_to_bf16_bits(rng.normal(0, 1, (T, d)).astype(np.float32))
            for l in range(L):
                res = [e for e in range(N) if (int(rb[l, e >> 5]) >> (e & 31)) & 1]
                mine = [e for e in res if e % world == rank]
                _, gates = O.router_topk(logits[l], k)
                y = O.moe_layer(h, ids[l], gates, {e: W[(l, e)] for e in mine})
                yt = torch.from_numpy(y)
                dist.all_reduce(yt)  # the combine collective
                y_full = O.moe_layer(h, ids[l], gates, {e: W[(l, e)] for e in res})
                assert np.allclose(yt.numpy(), y_full, rtol=1e-12, atol=1e-12)
            freqs = np.stack([O.hist_scan(ids[l], N)[0] for l in range(L)])
            s.observe_freqs(freqs, acc)
            for l in range(L):
                est[l] = O.estimator_observe(est[l], freqs[l], 4, 0.1)
                scores[l] = est[l][:, 0]
        rc, rg, b = s.ratios(1)
        t = torch.from_numpy(np.concatenate([rc, rg, [b]]))
        ts = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(ts, t)
        assert all(torch.equal(ts[0], x) for x in ts)
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_expert_parallel_host_logic_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res
