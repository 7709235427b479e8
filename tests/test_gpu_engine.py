"""End-to-end verification step on the GPU through the C ABI (moespac_step).

Checks, step after step with real expert loads (cache < 100%):
  * the engine's scheduling record (SimEvent log: ordered evict/load ids,
    taus, timings) equals the compiled reference Simulation on the same trace;
  * K1 ids equal the reference trace; K2 counters equal the reference split;
  * every layer's fp32 MoE output matches the fp64 oracle over exactly the
    experts resident after this step's loads (rel-L2 <= 1e-5), and the bf16
    residual chain h_{l+1} = bf16(h_l + y_l) is within 1 bf16 ulp;
  * host-buffer (moespac_step) and device-buffer (moespac_step_device) paths
    are bitwise identical.
"""
import numpy as np
import pytest
import torch

import oracle as O
from conftest import ref_or_skip
from paper_2603_09983_b200 import abi

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def _experts(rng, L, N, d, ffn, units):
    std = {}
    for l in range(L):
        for e in range(N):
            std[(l, e)] = tuple(O.f32_to_bf16_bits(rng.normal(0, 0.03, s).astype(np.float32))
                                for s in ((ffn, d), (ffn, d), (d, ffn)))
    shared = {l: [tuple(O.f32_to_bf16_bits(rng.normal(0, 0.03, s).astype(np.float32))
                        for s in ((ffn, d), (ffn, d), (d, ffn))) for _ in range(units)] for l in range(L)}
    return std, shared


def _pack(w, kernel):
    return abi.pack_expert(*[torch.from_numpy(x.view(np.int16)).cuda() for x in w], kernel=kernel)


def _make_ctx(L, N, k, g, d, ffn, units, gate_mode, cache, std, shared, kernel=abi.FFN_AUTO, cold=-1, stage=None):
    cfg = abi.default_config(n_layers=L, n_experts=N, top_k=k, gamma=g, cache_ratio=cache)
    kernel = abi.ffn_resolve(kernel, d, ffn)
    ctx = abi.Context(0, abi.ModelDesc(L, N, k, g, d, ffn, units, gate_mode, kernel), cfg)
    ctx.set_cold_threads(cold)
    if stage:
        ctx.set_cold_staging(*stage)
    arena = ctx.host_arena(L * N)
    for (l, e), w in std.items():
        arena[l * N + e] = _pack(w, kernel).cpu().numpy().view(np.uint16)
    for l in range(L):
        if units:
            ctx.set_shared(l, torch.stack([_pack(w, kernel) for w in shared[l]]))
    ctx.finalize()
    return ctx, cfg


def _resident(rb, l, N):
    return [e for e in range(N) if (int(rb[l, e >> 5]) >> (e & 31)) & 1]


@pytest.mark.parametrize("L,N,k,g,d,ffn,units,gate_mode,cache,kernel,cold", [
    (3, 16, 4, 6, 1024, 64, 1, 1, 0.25, abi.FFN_CUDACORE, -1),
    (3, 16, 4, 6, 1024, 64, 1, 1, 0.25, abi.FFN_TENSOR, -1),
    (3, 16, 4, 6, 1024, 64, 1, 1, 0.25, abi.FFN_TENSOR, 0),
    (2, 8, 2, 4, 512, 128, 0, 0, 0.17, abi.FFN_TENSOR, 3),
    (2, 32, 8, 8, 2048, 48, 0, 0, 0.5, abi.FFN_CUDACORE, 2),
    (2, 32, 8, 8, 2048, 128, 0, 0, 0.5, abi.FFN_TENSOR, -1),
    (2, 32, 8, 8, 2048, 128, 0, 0, 1.0, abi.FFN_TENSOR, -1),
    (2, 16, 8, 15, 1024, 128, 1, 0, 0.5, abi.FFN_TENSOR, -1),  # T = 16 tokens, up to 16 per cold expert
    (2, 8, 2, 4, 4096, 128, 0, 0, 0.5, abi.FFN_TENSOR, -1),    # per-segment K3 (d > 2048) + cold path
])
def test_engine_steps_match_reference_and_oracle(L, N, k, g, d, ffn, units, gate_mode, cache, kernel, cold):
    _engine_steps(L, N, k, g, d, ffn, units, gate_mode, cache, kernel, cold)


@pytest.mark.parametrize("L,N,k,g,d,ffn,units,gate_mode,cache,kernel,stage", [
    (3, 16, 4, 6, 1024, 64, 1, 1, 0.25, abi.FFN_TENSOR, (4, 0.5)),     # grouped K3, shared units
    (3, 16, 4, 6, 1024, 64, 1, 1, 0.25, abi.FFN_CUDACORE, (4, 0.5)),
    (2, 32, 8, 8, 2048, 128, 0, 0, 0.5, abi.FFN_TENSOR, (16, 1.0)),    # every miss staged: no host path
    (3, 32, 8, 8, 2048, 128, 0, 0, 0.25, abi.FFN_TENSOR, (4, 1.0)),    # ring half caps the staged share
    (2, 8, 2, 4, 4096, 128, 0, 0, 0.5, abi.FFN_TENSOR, (2, 1.0)),      # per-segment K3 (d > 2048)
])
def test_staged_cold_experts_match_reference_and_oracle(L, N, k, g, d, ffn, units, gate_mode, cache, kernel, stage):
    """Misses split between the host cores and the HBM staging ring: the same
    decisions, the full Eq. 3 output, every miss run exactly once."""
    _engine_steps(L, N, k, g, d, ffn, units, gate_mode, cache, kernel, -1, stage)


def _engine_steps(L, N, k, g, d, ffn, units, gate_mode, cache, kernel, cold, stage=None):
    ref_or_skip()
    rng = np.random.default_rng(L * 100 + N)
    std, shared = _experts(rng, L, N, d, ffn, units)
    ctx, cfg = _make_ctx(L, N, k, g, d, ffn, units, gate_mode, cache, std, shared, kernel, cold, stage)
    n_staged = 0
    T = g + 1
    steps = 10
    gen = O.Generator(L, N, k, g, seed=1)
    rcfg = O.default_config(n_layers=L, n_experts=N, top_k=k, gamma=g, cache_ratio=cache, token_budget=0)
    ids_ref, acc_ref = O.ref_trace(rcfg, steps)
    run = O.ref_sim_run(rcfg, ids_ref, acc_ref)
    total_loads = 0
    for s in range(steps):
        logits, ids, acc = gen.next_step()
        assert np.array_equal(ids, ids_ref[s]) and acc == acc_ref[s]
        h0 = O.f32_to_bf16_bits(rng.normal(0, 1, (T, d)).astype(np.float32))
        h_out = np.zeros_like(h0)
        rep, lay = ctx.step(logits, h0, acc, h_out)
        total_loads += rep.n_loads
        v = ctx.views()
        got_ids = abi.fetch(v.ids_dev, (L, T, k), np.int32)
        assert np.array_equal(got_ids, ids)
        hs = abi.fetch(v.h_dev, (L + 1, T, d), np.uint16)
        ys = abi.fetch(v.y_dev, (L, T, d), np.float32)
        assert np.array_equal(hs[0], h0) and np.array_equal(hs[L], h_out)
        _, rb, _, _ = ctx.step_tables()
        for l in range(L):
            _, gates = O.router_topk(logits[l], k, gate_mode)
            # cold path on: misses run on the host cores -> the full Eq. 3 output
            res = range(N) if cold != 0 else _resident(rb, l, N)
            y_ref = O.moe_layer(hs[l], ids[l], gates, {e: std[(l, e)] for e in res}, shared[l])
            rel = np.linalg.norm(ys[l] - y_ref) / max(np.linalg.norm(y_ref), 1e-30)
            assert rel <= 1e-5, (s, l, rel)
            exact = O.bf16_bits_to_f32(hs[l]).astype(np.float64) + y_ref
            got = O.bf16_bits_to_f32(hs[l + 1]).astype(np.float64)
            assert np.all(np.abs(got - exact) <= np.abs(exact) * 2.0 ** -8 + 1e-5 * np.abs(y_ref).max())
            r = run.layer_rec[s, l]
            assert [lay[l].tau, lay[l].fallback, lay[l].n_prefetch, lay[l].t_cpu_ns, lay[l].t_gpu_ns] == list(r[:5])
        sr = run.step_rec[s]
        assert [rep.cache_hits, rep.cache_misses, rep.faults_fn, rep.faults_fp] == list(sr[1:5])
        if cold != 0 and cache < 1.0:
            _, rb, _, _ = ctx.step_tables()
            n_miss = sum(1 for l in range(L) for e in range(N)
                         if e in set(ids[l].ravel()) and not (int(rb[l, e >> 5]) >> (e & 31)) & 1)
            assert rep.cold_experts + rep.staged_experts == n_miss
            if stage is None:
                assert rep.staged_experts == 0
            elif stage[1] == 1.0 and stage[0] // 2 >= N:
                assert rep.cold_experts == 0
        n_staged += rep.staged_experts
    if stage:
        assert n_staged > 0, "the test must exercise staged misses"
    assert np.array_equal(ctx.sched_events(), run.events)
    if cache < 1.0:
        assert total_loads > 0, "the test must exercise real expert loads"
    ctx.close()


def test_host_and_device_paths_bitwise_equal():
    L, N, k, g, d, ffn = 2, 16, 4, 6, 1024, 64
    rng = np.random.default_rng(5)
    std, shared = _experts(rng, L, N, d, ffn, 1)
    outs = []
    for mode in ("host", "device"):
        ctx, cfg = _make_ctx(L, N, k, g, d, ffn, 1, 0, 0.5, std, shared)
        gen = O.Generator(L, N, k, g, seed=4)
        hrng = np.random.default_rng(9)
        res = []
        for s in range(5):
            logits, _, acc = gen.next_step()
            h0 = O.f32_to_bf16_bits(hrng.normal(0, 1, (g + 1, d)).astype(np.float32))
            if mode == "host":
                h_out = np.zeros_like(h0)
                ctx.step(logits, h0, acc, h_out)
            else:
                lg = torch.from_numpy(logits).cuda()
                hd = torch.from_numpy(h0.view(np.int16)).cuda()
                ho = torch.zeros_like(hd)
                ctx.step_device(lg, hd, acc, ho)
                torch.cuda.synchronize()
                h_out = ho.cpu().numpy().view(np.uint16)
            res.append(h_out)
        outs.append(res)
        ctx.close()
    for a, b in zip(*outs):
        assert np.array_equal(a, b)


def test_step_argument_errors():
    L, N, k, g, d, ffn = 1, 8, 2, 4, 512, 32
    cfg = abi.default_config(n_layers=L, n_experts=N, top_k=k, gamma=g, cache_ratio=1.0)
    with pytest.raises(abi.MoespacError) as ei:
        abi.Context(0, abi.ModelDesc(L, N, k, g, 500, ffn, 0, 0, abi.FFN_CUDACORE), cfg)  # d % 512
    assert ei.value.code == "E_INVALID"
    ctx = abi.Context(0, abi.ModelDesc(L, N, k, g, d, ffn, 0, 0, abi.FFN_CUDACORE), cfg)
    logits = np.zeros((L, g + 1, N))
    h = np.zeros((g + 1, d), np.uint16)
    with pytest.raises(abi.MoespacError) as ei:
        ctx.step(logits, h, 1, h.copy())  # not finalized
    assert ei.value.code == "E_LOGIC"
    ctx.host_arena(N)
    ctx.finalize()
    with pytest.raises(abi.MoespacError) as ei:
        ctx.step(logits, h, g + 2, h.copy())
    assert ei.value.code == "E_RANGE"
    ctx.close()


@pytest.mark.parametrize("kernel", [abi.FFN_TENSOR, abi.FFN_CUDACORE])
def test_trace_replay_matches_logits_path(tmp_path, kernel):
    """#moetrace v1 replay (moespac_step_ids): routing recorded from the
    logits path, written to a trace file and read back, replays to the same
    bits — h_out, scheduling reports and SimEvent log — when the gates are
    carried along; with gates omitted every expert gets 1/k (checked against
    the fp64 oracle)."""
    L, N, k, g, d, ffn, cache = 2, 16, 4, 6, 1024, 128, 0.5
    rng = np.random.default_rng(42)
    std, shared = _experts(rng, L, N, d, ffn, 0)
    a, _ = _make_ctx(L, N, k, g, d, ffn, 0, 0, cache, std, shared, kernel, cold=0)
    b, _ = _make_ctx(L, N, k, g, d, ffn, 0, 0, cache, std, shared, kernel, cold=0)
    T = g + 1
    gen = O.Generator(L, N, k, g, seed=7)
    steps, hs, outs, gates, ids_all, accs = 6, [], [], [], [], []
    for s in range(steps):
        logits, ids, acc = gen.next_step()
        h0 = O.f32_to_bf16_bits(rng.normal(0, 1, (T, d)).astype(np.float32))
        h_out = np.zeros_like(h0)
        rep, lay = a.step(logits, h0, acc, h_out)
        v = a.views()
        gates.append(abi.fetch(v.gates_dev, (L, T, k), np.float32))
        ids_all.append(ids)
        accs.append(acc)
        hs.append(h0)
        outs.append((h_out, rep, [(x.tau, x.n_prefetch, x.t_cpu_ns, x.t_gpu_ns) for x in lay]))
    path = str(tmp_path / "replay.trace")
    abi.trace_write(path, np.stack(ids_all), np.array(accs), N)
    shape, ids_rd, acc_rd = abi.trace_read(path)
    assert shape == {"n_layers": L, "n_experts": N, "top_k": k, "gamma": g}
    for s in range(steps):
        # shuffle each token's (id, gate) pairs: the replay path sorts them
        perm = np.argsort(rng.random((L, T, k)), axis=-1)
        ids_s = np.take_along_axis(ids_rd[s], perm, -1)
        gates_s = np.take_along_axis(gates[s], perm, -1)
        h_out = np.zeros_like(hs[s])
        rep, lay = b.step_ids(ids_s, gates_s, hs[s], int(acc_rd[s]), h_out)
        want_h, want_rep, want_lay = outs[s]
        assert np.array_equal(h_out, want_h), s
        assert [rep.cache_hits, rep.cache_misses, rep.faults_fn, rep.faults_fp, rep.n_loads] == \
            [want_rep.cache_hits, want_rep.cache_misses, want_rep.faults_fn, want_rep.faults_fp, want_rep.n_loads]
        assert [(x.tau, x.n_prefetch, x.t_cpu_ns, x.t_gpu_ns) for x in lay] == want_lay
    assert np.array_equal(a.sched_events(), b.sched_events())
    # gates omitted -> uniform 1/k
    h_out = np.zeros_like(hs[0])
    b.step_ids(ids_rd[0], None, hs[0], int(acc_rd[0]), h_out)
    v = b.views()
    ys = abi.fetch(v.y_dev, (L, T, d), np.float32)
    _, rb, _, _ = b.step_tables()
    y_ref = O.moe_layer(hs[0], ids_rd[0][0], np.full((T, k), 1.0 / k),
                        {e: std[(0, e)] for e in _resident(rb, 0, N)}, [])
    assert np.linalg.norm(ys[0] - y_ref) / np.linalg.norm(y_ref) <= 1e-5
    with pytest.raises(abi.MoespacError):
        bad = ids_rd[0].copy()
        bad[0, 0, 1] = bad[0, 0, 0]
        b.step_ids(bad, None, hs[0], 1, h_out)


@pytest.mark.parametrize("L,N,k,g,d,ffn,gate_mode,cache,kernel", [
    (3, 16, 4, 6, 1024, 128, 0, 0.5, abi.FFN_TENSOR),
    (2, 60, 4, 6, 2048, 64, 1, 1.0, abi.FFN_TENSOR),
    (2, 8, 2, 4, 512, 64, 0, 0.25, abi.FFN_CUDACORE),
])
def test_model_mode_router_gemv(L, N, k, g, d, ffn, gate_mode, cache, kernel):
    """Model mode: K0 router logits bit-exact with the
    C oracle's restatement of its fp32 order, K1 ids bit-exact on them, FFN
    outputs within tolerance, and the scheduler's record equal to the
    reference Simulation replaying the routing the model produced."""
    ref_or_skip()
    rng = np.random.default_rng(L * 31 + N)
    std, shared = _experts(rng, L, N, d, ffn, 0)
    ctx, _ = _make_ctx(L, N, k, g, d, ffn, 0, gate_mode, cache, std, shared, kernel, cold=0)
    T = g + 1
    h_tmp = np.zeros((T, d), np.uint16)
    with pytest.raises(abi.MoespacError):  # no router weights yet
        ctx.step_model(h_tmp, 1, h_tmp.copy())
    Wg = [O.f32_to_bf16_bits(rng.normal(0, 0.05, (N, d)).astype(np.float32)) for _ in range(L)]
    for l in range(L):
        ctx.set_router(l, Wg[l])
    gen = O.Generator(L, N, k, g, seed=3)
    steps, all_ids, accs = 6, [], []
    for s in range(steps):
        _, _, acc = gen.next_step()
        h0 = O.f32_to_bf16_bits(rng.normal(0, 1, (T, d)).astype(np.float32))
        h_out = np.zeros_like(h0)
        rep, lay = ctx.step_model(h0, acc, h_out)
        v = ctx.views()
        logits = abi.fetch(v.logits_dev, (L, T, N), np.float64)
        ids = abi.fetch(v.ids_dev, (L, T, k), np.int32)
        gates = abi.fetch(v.gates_dev, (L, T, k), np.float32)
        hs = abi.fetch(v.h_dev, (L + 1, T, d), np.uint16)
        ys = abi.fetch(v.y_dev, (L, T, d), np.float32)
        assert np.array_equal(hs[0], h0) and np.array_equal(hs[L], h_out)
        _, rb, _, _ = ctx.step_tables()
        for l in range(L):
            lg_ref = O.router_gemv(Wg[l], hs[l])
            assert np.array_equal(logits[l], lg_ref), (s, l)
            ids_ref, gates_ref = O.router_topk(lg_ref, k, gate_mode)
            assert np.array_equal(ids[l], ids_ref), (s, l)
            np.testing.assert_allclose(gates[l], gates_ref, rtol=3e-6, atol=1e-7)
            y_ref = O.moe_layer(hs[l], ids_ref, gates_ref, {e: std[(l, e)] for e in _resident(rb, l, N)}, [])
            rel = np.linalg.norm(ys[l] - y_ref) / max(np.linalg.norm(y_ref), 1e-30)
            assert rel <= 1e-5, (s, l, rel)
        all_ids.append(ids)
        accs.append(acc)
    rcfg = O.default_config(n_layers=L, n_experts=N, top_k=k, gamma=g, cache_ratio=cache, token_budget=0)
    run = O.ref_sim_run(rcfg, np.stack(all_ids), np.array(accs, np.int32))
    assert np.array_equal(ctx.sched_events(), run.events)


def test_model_mode_needs_cold_path_off():
    L, N, k, g, d, ffn = 1, 8, 2, 4, 512, 64
    rng = np.random.default_rng(1)
    std, shared = _experts(rng, L, N, d, ffn, 0)
    ctx, _ = _make_ctx(L, N, k, g, d, ffn, 0, 0, 0.25, std, shared, abi.FFN_TENSOR, cold=2)
    ctx.set_router(0, O.f32_to_bf16_bits(rng.normal(0, 0.05, (N, d)).astype(np.float32)))
    h = np.zeros((g + 1, d), np.uint16)
    with pytest.raises(abi.MoespacError) as ei:
        ctx.step_model(h, 1, h.copy())
    assert ei.value.code == "E_LOGIC"


@pytest.mark.parametrize("world,cache,kernel,cold,mode", [
    (2, 1.0, abi.FFN_TENSOR, 0, 1),
    (2, 0.5, abi.FFN_TENSOR, -1, 0),
    (3, 0.5, abi.FFN_TENSOR, 0, 0),
    (2, 0.5, abi.FFN_CUDACORE, 0, 0),
    (2, 1.0, abi.FFN_TENSOR, 0, 0),     # auto -> unit split (every expert fits)
    (3, 1.0, abi.FFN_TENSOR, -1, 2),    # unit split, grouped K3
    (2, 1.0, abi.FFN_TENSOR, 0, 2),     # unit split, d = 4096, T = 7: grouped K3 in N = 8 mode, below
    (2, 1.0, abi.FFN_TENSOR, 1, 2),     # unit split, d = 4096, T = 9: per-segment K3, below
])
def test_expert_parallel_device_path(world, cache, kernel, cold, mode):
    """Expert-parallel mode on one GPU: `world` contexts
    (expert e on rank e % world, shared units on rank 0), one host thread
    each, exchanging per-layer partial outputs through the in-process
    loopback group instead of NCCL. Every rank ends each layer with the same
    h; every layer's MoE output matches the fp64 oracle over the experts
    resident on any rank (+ the host cold path when on)."""
    import threading
    L, N, k, g, d, ffn, units = 2, 16, 4, 6, 1024, 128, 1
    if (world, mode) == (2, 2) and cold >= 0:
        # d = 4096 in the unit-split mode: T = 7 runs the grouped K3 at N = 8,
        # T = 9 the per-segment K3 (cache 1.0: the cold path stays idle)
        d, g = 4096, (6 if cold == 0 else 8)
    rng = np.random.default_rng(world * 10 + int(cache * 10))
    std, shared = _experts(rng, L, N, d, ffn, units)
    T = g + 1
    group = abi.LoopbackGroup(0, world, T * d)
    ctxs = []
    for r in range(world):
        cfg = abi.default_config(n_layers=L, n_experts=N, top_k=k, gamma=g, cache_ratio=cache)
        kern = abi.ffn_resolve(kernel, d, ffn)
        ctx = abi.Context(0, abi.ModelDesc(L, N, k, g, d, ffn, units, 0, kern, mode), cfg, r, world)
        ctx.set_cold_threads(cold)
        arena = ctx.host_arena(L * N)
        for (l, e), w in std.items():
            arena[l * N + e] = _pack(w, kern).cpu().numpy().view(np.uint16)
        for l in range(L):
            ctx.set_shared(l, torch.stack([_pack(w, kern) for w in shared[l]]))
        ctx.finalize()
        ctx.set_loopback(group)
        ctxs.append(ctx)
    gen = O.Generator(L, N, k, g, seed=5)
    for s in range(5):
        logits, ids, acc = gen.next_step()
        h0 = O.f32_to_bf16_bits(rng.normal(0, 1, (T, d)).astype(np.float32))
        outs = [np.zeros_like(h0) for _ in range(world)]
        errs = []

        def run(r):
            try:
                ctxs[r].step(logits, h0, acc, outs[r])
            except Exception as exc:  # surfaced below
                errs.append(exc)

        th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
        for t in th:
            t.start()
        for t in th:
            t.join(timeout=120)
        assert not errs, errs
        for r in range(1, world):
            assert np.array_equal(outs[r], outs[0]), (s, r)
        v = ctxs[0].views()
        hs = abi.fetch(v.h_dev, (L + 1, T, d), np.uint16)
        ys = abi.fetch(v.y_dev, (L, T, d), np.float32)  # after the all-reduce
        res = [set() for _ in range(L)]
        for ctx in ctxs:
            _, rb, _, _ = ctx.step_tables()
            for l in range(L):
                res[l] |= set(_resident(rb, l, N))
        for l in range(L):
            _, gates = O.router_topk(logits[l], k, 0)
            present = range(N) if cold != 0 else sorted(res[l])
            y_ref = O.moe_layer(hs[l], ids[l], gates, {e: std[(l, e)] for e in present}, shared[l])
            rel = np.linalg.norm(ys[l] - y_ref) / max(np.linalg.norm(y_ref), 1e-30)
            assert rel <= 1e-5, (s, l, rel)
    for ctx in ctxs:
        ctx.close()
    group.close()


def test_draft_window_overlaps_loads_and_changes_nothing_else():
    """The emulated draft window (γ·t_draft spin on the compute stream) adds
    its time to the step and leaves every output and decision unchanged."""
    L, N, k, g, d, ffn = 2, 16, 4, 6, 1024, 128
    rng = np.random.default_rng(3)
    std, shared = _experts(rng, L, N, d, ffn, 0)
    a, cfg = _make_ctx(L, N, k, g, d, ffn, 0, 0, 0.5, std, shared, abi.FFN_TENSOR, cold=0)
    b, _ = _make_ctx(L, N, k, g, d, ffn, 0, 0, 0.5, std, shared, abi.FFN_TENSOR, cold=0)
    b.set_draft_window(True)
    b.set_timing(True)
    T = g + 1
    gen = O.Generator(L, N, k, g, seed=4)
    for s in range(4):
        logits, _, acc = gen.next_step()
        h0 = O.f32_to_bf16_bits(rng.normal(0, 1, (T, d)).astype(np.float32))
        ha, hb = np.zeros_like(h0), np.zeros_like(h0)
        a.step(logits, h0, acc, ha)
        rb_, _ = b.step(logits, h0, acc, hb)
        assert np.array_equal(ha, hb)
        assert rb_.gpu_ms_total * 1e6 >= g * cfg.t_draft_unit_ns
    assert np.array_equal(a.sched_events(), b.sched_events())


@pytest.mark.parametrize("d,ffn,cache", [(1024, 128, 0.5), (1024, 128, 1.0), (4096, 128, 1.0)])
def test_l2_prefetch_changes_nothing(d, ffn, cache):
    """The cross-layer L2 prefetch (default on for the grouped K3, a hint on
    the per-segment one) only moves bytes into L2: outputs and scheduling
    are bitwise those of the same engine with it off, including layers whose
    experts are being loaded while the previous layer prefetches."""
    L, N, k, g = 3, 16, 4, 6
    rng = np.random.default_rng(11)
    std, shared = _experts(rng, L, N, d, ffn, 0)
    a, _ = _make_ctx(L, N, k, g, d, ffn, 0, 0, cache, std, shared, abi.FFN_TENSOR, cold=0)
    b, _ = _make_ctx(L, N, k, g, d, ffn, 0, 0, cache, std, shared, abi.FFN_TENSOR, cold=0)
    a.set_l2_prefetch(0)
    b.set_l2_prefetch(256 * 1024)
    T = g + 1
    gen = O.Generator(L, N, k, g, seed=6)
    for s in range(4):
        logits, _, acc = gen.next_step()
        h0 = O.f32_to_bf16_bits(rng.normal(0, 1, (T, d)).astype(np.float32))
        ha, hb = np.zeros_like(h0), np.zeros_like(h0)
        a.step(logits, h0, acc, ha)
        b.step(logits, h0, acc, hb)
        assert np.array_equal(ha, hb)
    assert np.array_equal(a.sched_events(), b.sched_events())
    a.close()
    b.close()


def test_draft_gemv_matches_torch():
    """One draft pass (the draft model's weight-streaming GEMV) against a
    plain PyTorch fp32 reference, first pass (x0) and chained (y_prev)."""
    R, D = 5000, 2560
    g = torch.Generator(device="cuda").manual_seed(7)
    w = (torch.randn((R, D), device="cuda", generator=g) * 0.02).to(torch.bfloat16)
    x0 = torch.randn(D, device="cuda", generator=g).to(torch.bfloat16)
    y = abi.draft_gemv(w.view(torch.int16), x0=x0.view(torch.int16))
    ref = w.float() @ x0.float()
    assert torch.allclose(y, ref, rtol=1e-4, atol=1e-4 * ref.abs().max().item())
    scale = 0.7
    y2 = abi.draft_gemv(w.view(torch.int16), y_prev=y, scale=scale)
    x1 = (y[:D] * scale).to(torch.bfloat16).float()
    ref2 = w.float() @ x1
    assert torch.allclose(y2, ref2, rtol=1e-4, atol=1e-4 * ref2.abs().max().item())


def test_draft_model_and_measured_timeline():
    """Real draft phase + measured SimEvent timeline
    (row 1): the draft passes stream gamma x n_params x 2 bytes per step and
    leave outputs / decisions bitwise unchanged; the measured log has one gpu
    record per layer, the load / evict records of the modeled log (same
    experts, same order), and every step conserves time:
    total == draft + prologue + sum(layer walls) + epilogue, with
    gpu + stall <= wall per layer."""
    L, N, k, g, d, ffn = 3, 16, 4, 6, 1024, 128
    rng = np.random.default_rng(13)
    std, shared = _experts(rng, L, N, d, ffn, 0)
    a, cfg = _make_ctx(L, N, k, g, d, ffn, 0, 0, 0.5, std, shared, abi.FFN_TENSOR, cold=-1)
    b, _ = _make_ctx(L, N, k, g, d, ffn, 0, 0, 0.5, std, shared, abi.FFN_TENSOR, cold=-1)
    n_params, dd = 64 << 20, 2560
    b.set_draft_model(n_params, dd)
    b.set_timeline(True)
    T = g + 1
    gen = O.Generator(L, N, k, g, seed=4)
    loads = 0
    for s in range(5):
        logits, _, acc = gen.next_step()
        h0 = O.f32_to_bf16_bits(rng.normal(0, 1, (T, d)).astype(np.float32))
        ha, hb = np.zeros_like(h0), np.zeros_like(h0)
        a.step(logits, h0, acc, ha)
        rb_, _ = b.step(logits, h0, acc, hb)
        loads += rb_.n_loads
        assert np.array_equal(ha, hb)
        assert rb_.draft_bytes == g * (n_params // dd) * dd * 2 and rb_.gpu_ms_draft > 0
    assert loads > 0
    modeled = a.sched_events()
    assert np.array_equal(modeled, b.sched_events())
    ev, lay, steps = b.timeline()
    assert len(steps) == 5 and len(lay) == 5 * L
    for st in steps:
        total, draft, pro, walls, epi, _ = st
        assert total == draft + pro + walls + epi and draft > 0 and pro > 0 and walls > 0
    for m in lay:
        assert m.t_gpu_ns > 0 and m.t_gpu_ns + m.stall_ns <= m.wall_ns
    for kind in (O.EV_LOAD, O.EV_EVICT):
        got = ev[ev[:, 0] == kind][:, 1:4]
        want = modeled[modeled[:, 0] == kind][:, 1:4]
        assert np.array_equal(got, want), kind
    gpu = ev[ev[:, 0] == O.EV_GPU]
    assert len(gpu) == 5 * L and (gpu[:, 5] > 0).all()
    assert (ev[ev[:, 0] == O.EV_DRAFT][:, 5] > 0).sum() == 5
    # starts are on one monotone measured clock
    starts = ev[ev[:, 0] == O.EV_GPU][:, 4]
    assert (np.diff(starts) > 0).all()
    b.set_draft_model(0)
    a.close()
    b.close()


def test_expert_parallel_combine_is_deterministic():
    """The multi-GPU combine (all-gather + ordered sum over ranks) gives the
    same bits run after run, and the world-2 result is within tolerance of
    world 1 (the ranks split the work differently, so the fp32 sums are
    ordered differently)."""
    import threading
    L, N, k, g, d, ffn, units = 2, 16, 4, 6, 1024, 128, 1
    rng = np.random.default_rng(31)
    std, shared = _experts(rng, L, N, d, ffn, units)
    T = g + 1

    def run(world):
        group = abi.LoopbackGroup(0, world, T * d) if world > 1 else None
        ctxs = []
        for r in range(world):
            # cache 1.0: every expert resident at any world size (the same experts
            # contribute; only the work split and the summation order change)
            cfg = abi.default_config(n_layers=L, n_experts=N, top_k=k, gamma=g, cache_ratio=1.0)
            ctx = abi.Context(0, abi.ModelDesc(L, N, k, g, d, ffn, units, 0, abi.FFN_TENSOR, 1), cfg, r, world)
            ctx.set_cold_threads(0)
            arena = ctx.host_arena(L * N)
            for (l, e), w in std.items():
                arena[l * N + e] = _pack(w, abi.FFN_TENSOR).cpu().numpy().view(np.uint16)
            for l in range(L):
                ctx.set_shared(l, torch.stack([_pack(w, abi.FFN_TENSOR) for w in shared[l]]))
            ctx.finalize()
            if group:
                ctx.set_loopback(group)
            ctxs.append(ctx)
        gen = O.Generator(L, N, k, g, seed=12)
        hr = np.random.default_rng(3)
        res = []
        for s in range(4):
            logits, _, acc = gen.next_step()
            h0 = O.f32_to_bf16_bits(hr.normal(0, 1, (T, d)).astype(np.float32))
            outs = [np.zeros_like(h0) for _ in range(world)]
            th = [threading.Thread(target=lambda r=r: ctxs[r].step(logits, h0, acc, outs[r])) for r in range(world)]
            for t in th:
                t.start()
            for t in th:
                t.join()
            for r in range(1, world):
                assert np.array_equal(outs[r], outs[0])
            res.append(outs[0])
        for c in ctxs:
            c.close()
        if group:
            group.close()
        return np.stack(res)

    a, b = run(2), run(2)
    assert np.array_equal(a, b)
    one = run(1)
    fa, f1 = O.bf16_bits_to_f32(a).astype(np.float64), O.bf16_bits_to_f32(one).astype(np.float64)
    assert np.linalg.norm(fa - f1) <= 4e-3 * np.linalg.norm(f1)


def test_estimator_checkpoint_round_trip(tmp_path):
    """moespac_ctx_estimator_dump / _load: the device estimator state in the
    reference's checkpoint format (utility_estimator.cpp:81-107) equals the
    oracle estimator run over the same routing; a fresh context loaded from it
    continues bit-identically (outputs and the next checkpoint); malformed
    checkpoints fail with the reference's error class and change nothing."""
    L, N, k, g, d, ffn = 2, 16, 4, 6, 1024, 64
    rng = np.random.default_rng(17)
    std, shared = _experts(rng, L, N, d, ffn, 0)
    a, cfg = _make_ctx(L, N, k, g, d, ffn, 0, 0, 1.0, std, shared, abi.FFN_TENSOR, cold=0)
    T = g + 1
    gen = O.Generator(L, N, k, g, seed=21)
    steps = [gen.next_step() for _ in range(6)]
    hs = [O.f32_to_bf16_bits(rng.normal(0, 1, (T, d)).astype(np.float32)) for _ in range(6)]
    est = [O.estimator_init(N, g) for _ in range(L)]
    for s in range(5):
        logits, ids, acc = steps[s]
        a.step(logits, hs[s], acc, np.zeros_like(hs[s]))
        for l in range(L):
            est[l] = O.estimator_observe(est[l], O.hist_scan(ids[l], N)[0], cfg.utility_cap, cfg.forgetting)
    p1 = str(tmp_path / "est1.txt")
    a.estimator_dump(p1)
    rows = np.loadtxt(p1, dtype=np.int64)
    assert rows.shape == (L * N, 6)
    for l in range(L):
        blk = rows[l * N:(l + 1) * N]
        assert (blk[:, 0] == l).all() and (blk[:, 1] == np.arange(N)).all()
        assert np.array_equal(blk[:, 2:], est[l])
    b, _ = _make_ctx(L, N, k, g, d, ffn, 0, 0, 1.0, std, shared, abi.FFN_TENSOR, cold=0)
    bad = tmp_path / "bad.txt"
    bad.write_text("0 0 1 2 3\n")
    with pytest.raises(abi.MoespacError) as ei:
        b.estimator_load(str(bad))
    assert ei.value.code == "E_IO"
    b.estimator_load(p1)
    logits, ids, acc = steps[5]
    ha, hb = np.zeros_like(hs[5]), np.zeros_like(hs[5])
    a.step(logits, hs[5], acc, ha)
    b.step(logits, hs[5], acc, hb)
    assert np.array_equal(ha, hb)
    p2a, p2b = str(tmp_path / "a2.txt"), str(tmp_path / "b2.txt")
    a.estimator_dump(p2a)
    b.estimator_dump(p2b)
    assert open(p2a).read() == open(p2b).read()
    a.close()
    b.close()


@pytest.mark.parametrize("d,ffn,kernel", [(1024, 128, abi.FFN_TENSOR), (4096, 128, abi.FFN_TENSOR),
                                          (1024, 64, abi.FFN_CUDACORE)])
def test_graph_replay_bitwise_equal(d, ffn, kernel):
    """The launch-latency path (a captured CUDA graph replayed for load-free
    steps) gives the bits of the launch-by-launch path: h_out, K3 outputs,
    reports and the SimEvent log, host and device inputs alike, across a
    toggle of programmatic dependent launch (which re-captures)."""
    L, N, k, g = 3, 16, 4, 6
    rng = np.random.default_rng(d + ffn)
    std, shared = _experts(rng, L, N, d, ffn, 0)
    a, _ = _make_ctx(L, N, k, g, d, ffn, 0, 0, 1.0, std, shared, kernel, cold=0)
    b, _ = _make_ctx(L, N, k, g, d, ffn, 0, 0, 1.0, std, shared, kernel, cold=0)
    a.set_graph(False)
    b.set_graph(True)
    T = g + 1
    gen = O.Generator(L, N, k, g, seed=8)
    for s in range(8):
        logits, _, acc = gen.next_step()
        h0 = O.f32_to_bf16_bits(rng.normal(0, 1, (T, d)).astype(np.float32))
        if s == 5:
            a.set_pdl(False)
            b.set_pdl(False)
        outs = []
        for c in (a, b):
            if s % 2:
                ho = torch.zeros((T, d), dtype=torch.int16, device="cuda")
                rep, lay = c.step_device(torch.from_numpy(logits).cuda(), torch.from_numpy(h0.view(np.int16)).cuda(),
                                         acc, ho)
                torch.cuda.synchronize()
                h_out = ho.cpu().numpy().view(np.uint16)
            else:
                h_out = np.zeros_like(h0)
                rep, lay = c.step(logits, h0, acc, h_out)
            v = c.views()
            outs.append((h_out, abi.fetch(v.y_dev, (L, T, d), np.float32), rep.cache_hits, rep.kernel_launches,
                         [(x.tau, x.n_prefetch) for x in lay]))
        assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1]), s
        assert outs[0][2:] == outs[1][2:], s
    assert np.array_equal(a.sched_events(), b.sched_events())
    a.close()
    b.close()
