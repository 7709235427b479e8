"""Expert-parallel combine over real NCCL: two processes,
one GPU each, all-gather of the per-rank fp32 partials + ordered sum. The
result must be bitwise the in-process loopback group's (same per-rank K3
work, same ordered-sum kernel) and within tolerance of the fp64 oracle.
Self-skips on a box with fewer than 2 GPUs (the loopback test in
test_gpu_engine.py covers the device path on one GPU)."""
import os
import tempfile

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

L, N, k, g, d, ffn, units, STEPS = 2, 16, 4, 6, 1024, 128, 1, 4


def _setup(rank, world, device, uid=None, group=None):
    import oracle as O
    from paper_2603_09983_b200 import abi
    rng = np.random.default_rng(77)
    std = {(l, e): tuple(O.f32_to_bf16_bits(rng.normal(0, 0.03, s).astype(np.float32))
                         for s in ((ffn, d), (ffn, d), (d, ffn))) for l in range(L) for e in range(N)}
    shared = {l: [tuple(O.f32_to_bf16_bits(rng.normal(0, 0.03, s).astype(np.float32))
                        for s in ((ffn, d), (ffn, d), (d, ffn)))] for l in range(L)}
    cfg = abi.default_config(n_layers=L, n_experts=N, top_k=k, gamma=g, cache_ratio=0.5)
    kern = abi.ffn_resolve(abi.FFN_TENSOR, d, ffn)
    ctx = abi.Context(device, abi.ModelDesc(L, N, k, g, d, ffn, units, 0, kern, abi_par_expert()), cfg, rank, world)
    ctx.set_cold_threads(0)
    arena = ctx.host_arena(L * N)
    pk = lambda w: abi.pack_expert(*[torch.from_numpy(x.view(np.int16)).cuda(device) for x in w], kernel=kern)  # noqa
    for (l, e), w in std.items():
        arena[l * N + e] = pk(w).cpu().numpy().view(np.uint16)
    for l in range(L):
        ctx.set_shared(l, torch.stack([pk(w) for w in shared[l]]))
    ctx.finalize()
    if uid is not None:
        ctx.set_nccl(uid, world, rank)
    if group is not None:
        ctx.set_loopback(group)
    return ctx, std, shared


def abi_par_expert():
    return 1  # MOESPAC_PAR_EXPERT


def _inputs():
    import oracle as O
    gen = O.Generator(L, N, k, g, seed=5)
    rng = np.random.default_rng(6)
    out = []
    for _ in range(STEPS):
        logits, ids, acc = gen.next_step()
        out.append((logits, ids, acc, O.f32_to_bf16_bits(rng.normal(0, 1, (g + 1, d)).astype(np.float32))))
    return out


def _worker(rank, world, uid, outdir):
    torch.cuda.set_device(rank)
    ctx, _, _ = _setup(rank, world, rank, uid=uid)
    res = []
    for logits, _, acc, h0 in _inputs():
        h_out = np.zeros_like(h0)
        ctx.step(logits, h0, acc, h_out)
        res.append(h_out)
    np.save(os.path.join(outdir, f"r{rank}.npy"), np.stack(res))
    ctx.close()


def test_nccl_combine_matches_loopback_bitwise():
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs (the loopback group covers the device path on one)")
    import threading

    import torch.multiprocessing as mp

    from paper_2603_09983_b200 import abi
    world = 2
    uid = abi.nccl_unique_id()
    with tempfile.TemporaryDirectory() as td:
        mp.spawn(_worker, args=(world, uid, td), nprocs=world, join=True)
        got = [np.load(os.path.join(td, f"r{r}.npy")) for r in range(world)]
    assert np.array_equal(got[0], got[1])
    # the same steps through the loopback group on GPU 0
    torch.cuda.set_device(0)
    group = abi.LoopbackGroup(0, world, (g + 1) * d)
    ctxs = [_setup(r, world, 0, group=group)[0] for r in range(world)]
    want = []
    for logits, _, acc, h0 in _inputs():
        outs = [np.zeros_like(h0) for _ in range(world)]
        th = [threading.Thread(target=lambda r=r: ctxs[r].step(logits, h0, acc, outs[r])) for r in range(world)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        want.append(outs[0])
    assert np.array_equal(got[0], np.stack(want))
    for c in ctxs:
        c.close()
    group.close()


def test_nccl_library_loads_and_single_rank_comm_inits():
    """Runs on one GPU: the engine's dlopen'ed NCCL (libnccl.so.2, the one
    torch already mapped) exports what it binds, hands out a unique id, and
    a one-rank communicator initialises on it — the setup path every rank of
    `bench.py --gpus N` takes before its first all-gather."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.distributed as _dist  # noqa: F401  (maps torch's libnccl first, as under torchrun)
    from paper_2603_09983_b200 import abi
    torch.cuda.set_device(0)
    uid = abi.nccl_unique_id()
    assert len(uid) == 128 and any(uid)
    ctx, _, _ = _setup(0, 1, 0, uid=uid)
    ctx.close()
