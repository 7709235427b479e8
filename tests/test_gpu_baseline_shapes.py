"""Engine parity at the BASELINE.json shapes (VERDICT r1 "Next round" item 1).

Every workload of BASELINE.json's `configs` runs through moespac_step at its
full shape — d, ffn, L, N, k, γ, shared units and gate flags of configs.py —
with synthetic weights (moespac_ctx_fill_synthetic) and the host cold path
on, on the reference's default trace (seed 1), and is compared with:

  * the committed golden fixtures of the compiled reference
    (tests/golden/sim_<cfg>.npz, Simulation::run_utility_step,
    sim_core.cpp:157-316): per (step, layer) tau / fallback / n_prefetch /
    t_cpu / t_gpu, per step hits / misses / faults, and the SimEvent log of
    the steps run, record for record;
  * the trace ids (K1 bit-exact);
  * the fp64 oracle (oracle.moe_layer, Eq. 3) for the layer output y of
    sampled layers — every activated expert (resident ones from K3, missed
    ones from the host cold path) plus the shared units — with the weights
    read back from the synthetic images through moespac_unpack_expert
    (pinned by test_pack_unpack_round_trip); rel-L2 <= 1e-5, and the bf16
    residual h_{l+1} within one bf16 rounding of h_l + y.

Mixtral's headline kernel (per-segment tcgen05 K3, d = 4096, ffn = 14336) is
checked at cache 1.0 (the bench headline: every expert resident) and at 0.17
(real loads + cold path).
"""
import os

import numpy as np
import pytest
import torch

import oracle as O
from paper_2603_09983_b200 import abi
from paper_2603_09983_b200.configs import CONFIGS, HWB_PROFILES, SYNTH_STD

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


class Weights:
    """Standard-layout weights of the context's synthetic images (cached per image)."""

    def __init__(self, ctx, arena, w, n_images, kernel):
        self.ctx, self.arena, self.w, self.n, self.kernel = ctx, arena, w, n_images, kernel
        self.cache = {}

    def _unpack(self, img_dev):
        wg, wu, wd = abi.unpack_expert(img_dev, self.w.d_model, self.w.d_ffn, self.kernel)
        return tuple(x.cpu().numpy().view(np.uint16) for x in (wg, wu, wd))

    def expert(self, l, e):
        i = (l * self.w.n_experts + e) % self.n
        if i not in self.cache:
            self.cache[i] = self._unpack(torch.from_numpy(self.arena[i].view(np.int16)).cuda())
        return self.cache[i]

    def shared(self, l):
        v = self.ctx.views()
        out = []
        for u in range(self.w.n_shared_units):
            off = ((l * self.w.n_shared_units + u) * self.ctx.image_elems) * 2
            out.append(self._unpack(_dev_view(v.shared_dev + off, self.ctx.image_elems)))
        return out

    def shared_gate(self, l):
        v = self.ctx.views()
        if not v.shared_gate_dev:
            return None
        return abi.fetch(v.shared_gate_dev + l * self.w.d_model * 2, (self.w.d_model,), np.uint16)


def _dev_view(addr, n):
    """int16 device tensor aliasing n elements at a raw device address."""
    host = abi.fetch(addr, (n,), np.int16)
    return torch.from_numpy(host).cuda()


def _build(w, n_images, cold=-1, profile="reference"):
    cfg = abi.default_config(n_layers=w.n_layers, n_experts=w.n_experts, top_k=w.top_k, gamma=w.gamma,
                             cache_ratio=w.cache_ratio, **HWB_PROFILES[profile](w))
    ctx = abi.Context(0, w.model_desc(), cfg)
    ctx.set_cold_threads(cold)
    arena = ctx.host_arena(n_images)
    ctx.fill_synthetic(seed=3, stdv=SYNTH_STD)
    ctx.finalize()
    kernel = abi.ffn_resolve(abi.FFN_AUTO, w.d_model, w.d_ffn)
    return ctx, arena, Weights(ctx, arena, w, n_images, kernel)


def _check_layer(W, w, logits_l, ids_l, hs, ys, l, tag):
    _, gates = O.router_topk(logits_l, w.top_k, w.gate_mode)
    experts = {e: W.expert(l, e) for e in sorted(set(ids_l.ravel().tolist()))}
    sg = W.shared_gate(l)
    sgt = None if sg is None else O.shared_gate(hs[l], sg)
    y_ref = O.moe_layer(hs[l], ids_l, gates, experts, W.shared(l), shared_gates=sgt)
    assert np.isfinite(ys[l]).all() and np.isfinite(y_ref).all(), (tag, l)
    rel = np.linalg.norm(ys[l] - y_ref) / max(np.linalg.norm(y_ref), 1e-30)
    assert rel <= 1e-5, (tag, l, rel)
    exact = O.bf16_bits_to_f32(hs[l]).astype(np.float64) + y_ref
    got = O.bf16_bits_to_f32(hs[l + 1]).astype(np.float64)
    assert np.all(np.abs(got - exact) <= np.abs(exact) * 2.0 ** -8 + 1e-5 * np.abs(y_ref).max()), (tag, l)
    return rel


# (golden file, config, cache, steps, n_images, y-check plan: {step: layers | "all"})
CASES = [
    ("sim_tiny", "tiny", 0.17, 60, 9, {0: "all", 17: "all", 59: "all"}),
    ("sim_tiny_c100", "tiny", 1.00, 60, 8, {0: "all", 59: "all"}),
    ("sim_mixtral_c100", "mixtral", 1.00, 6, 8, {0: [0, 16, 31], 5: [31]}),
    ("sim_mixtral", "mixtral", 0.17, 5, 9, {0: [0, 31], 4: [17]}),
    ("sim_qwen15", "qwen15", 0.50, 10, 61, {0: "all", 9: [0, 12, 23]}),
    ("sim_dsv2", "dsv2", 0.17, 10, 65, {0: "all", 9: [0, 13, 26]}),
    ("sim_qwen3_c017", "qwen3", 0.17, 24, 129, {0: "all", 11: [0, 24, 47], 23: [0, 24, 47]}),
    ("sim_qwen3_c010", "qwen3", 0.10, 8, 129, {7: [5, 40]}),
    ("sim_qwen3_c050", "qwen3", 0.50, 8, 129, {7: [5, 40]}),
    ("sim_qwen3_c100", "qwen3", 1.00, 8, 129, {0: [0, 47], 7: [5, 40]}),
    # HWB profile calibrated to B200 (configs.b200_hwb_profile; the golden is
    # the reference Simulation run with the same constants)
    ("sim_qwen3_c017_b200", "qwen3", 0.17, 12, 129, {11: [0, 24, 47]}),
]


@pytest.mark.parametrize("golden,name,cache,steps,n_images,ycheck", CASES, ids=[c[0][4:] for c in CASES])
def test_engine_at_baseline_shape(golden, name, cache, steps, n_images, ycheck):
    z = np.load(os.path.join(GOLDEN, golden + ".npz"))
    w = CONFIGS[name].with_(cache_ratio=cache)
    assert (int(z["L"]), int(z["N"]), int(z["k"]), int(z["gamma"]), float(z["cache_ratio"])) == \
        (w.n_layers, w.n_experts, w.top_k, w.gamma, cache)
    ctx, arena, W = _build(w, n_images, profile="b200" if golden.endswith("_b200") else "reference")
    L, N, k, T, d = w.n_layers, w.n_experts, w.top_k, w.tokens, w.d_model
    gen = O.Generator(L, N, k, w.gamma, seed=1)
    rng = np.random.default_rng(2)
    loads, checked = 0, 0
    for s in range(steps):
        logits, ids, acc = gen.next_step()
        assert np.array_equal(ids, z["ids"][s]) and acc == z["accepted"][s]
        h0 = O.f32_to_bf16_bits(rng.normal(0, 1, (T, d)).astype(np.float32))
        h_out = np.zeros_like(h0)
        rep, lay = ctx.step(logits, h0, acc, h_out)
        loads += rep.n_loads
        v = ctx.views()
        assert np.array_equal(abi.fetch(v.ids_dev, (L, T, k), np.int32), ids), s
        got = np.array([[x.tau, x.fallback, x.n_prefetch, x.t_cpu_ns, x.t_gpu_ns, x.t_io_used_ns, x.stall_ns,
                         x.wall_ns, x.bubble_ns] for x in lay], np.int64)
        assert np.array_equal(got, z["layer_rec"][s, :, :9]), s
        sr = z["step_rec"][s]
        assert [rep.accepted_tokens, rep.cache_hits, rep.cache_misses, rep.faults_fn, rep.faults_fp,
                rep.step_wall_ns, rep.draft_ns] == list(sr[:7]), s
        assert rep.accuracy == z["accuracy"][s]
        if s in ycheck:
            hs = abi.fetch(v.h_dev, (L + 1, T, d), np.uint16)
            ys = abi.fetch(v.y_dev, (L, T, d), np.float32)
            assert np.array_equal(hs[0], h0) and np.array_equal(hs[L], h_out)
            layers = range(L) if ycheck[s] == "all" else ycheck[s]
            for l in layers:
                _check_layer(W, w, logits[l], ids[l], hs, ys, l, (golden, s))
                checked += 1
    ev = z["events"]
    assert np.array_equal(ctx.sched_events(), ev[ev[:, 1] < steps])
    if cache < 1.0 and w.n_experts * cache >= 1:
        assert loads > 0 or name == "tiny", "a partial budget must exercise real expert loads"
    assert checked > 0
    ctx.close()


def test_ar_mode_one_token_per_step():
    """AR policy (policies.hpp ar_mode): the reference runs one simulated step
    per accepted token, fed that token's frequencies (sim_core.cpp:148-152,
    181-183, 306-313). The engine runs at T = 1: each step is one token's
    logits [L][1][N] and hidden state; decisions and the SimEvent log equal
    the reference's (golden sim_ar_mode), outputs the fp64 oracle's."""
    z = np.load(os.path.join(GOLDEN, "sim_ar_mode.npz"))
    L, N, k, g = int(z["L"]), int(z["N"]), int(z["k"]), int(z["gamma"])
    d, ffn = 1024, 128
    cfg = abi.default_config(n_layers=L, n_experts=N, top_k=k, gamma=g, cache_ratio=float(z["cache_ratio"]),
                             policy="ar_mode")
    kernel = abi.ffn_resolve(abi.FFN_AUTO, d, ffn)
    ctx = abi.Context(0, abi.ModelDesc(L, N, k, g, d, ffn, 0, 0, kernel), cfg)
    assert ctx.T == 1
    rng = np.random.default_rng(8)
    std = {(l, e): tuple(O.f32_to_bf16_bits(rng.normal(0, 0.03, sh).astype(np.float32))
                         for sh in ((ffn, d), (ffn, d), (d, ffn))) for l in range(L) for e in range(N)}
    arena = ctx.host_arena(L * N)
    for (l, e), wts in std.items():
        arena[l * N + e] = abi.pack_expert(*[torch.from_numpy(x.view(np.int16)).cuda() for x in wts],
                                           kernel=kernel).cpu().numpy().view(np.uint16)
    ctx.finalize()
    gen = O.Generator(L, N, k, g, seed=1)
    r = 0
    for s in range(len(z["accepted"])):
        logits, ids, acc = gen.next_step()
        assert np.array_equal(ids, z["ids"][s])
        for c in range(acc):
            lg = np.ascontiguousarray(logits[:, c:c + 1, :])
            h0 = O.f32_to_bf16_bits(rng.normal(0, 1, (1, d)).astype(np.float32))
            h_out = np.zeros_like(h0)
            rep, lay = ctx.step(lg, h0, 1, h_out)
            got = np.array([[x.tau, x.fallback, x.n_prefetch, x.t_cpu_ns, x.t_gpu_ns] for x in lay], np.int64)
            assert np.array_equal(got, z["layer_rec"][r, :, :5]), (s, c)
            assert [rep.accepted_tokens, rep.cache_hits, rep.cache_misses, rep.draft_ns] == \
                [1, z["step_rec"][r][1], z["step_rec"][r][2], 0]
            if r % 13 == 0:
                v = ctx.views()
                hs = abi.fetch(v.h_dev, (L + 1, 1, d), np.uint16)
                ys = abi.fetch(v.y_dev, (L, 1, d), np.float32)
                for l in range(L):
                    _, gates = O.router_topk(lg[l], k, 0)
                    y_ref = O.moe_layer(hs[l], ids[l, c:c + 1], gates, {e: std[(l, e)] for e in range(N)})
                    rel = np.linalg.norm(ys[l] - y_ref) / max(np.linalg.norm(y_ref), 1e-30)
                    assert rel <= 1e-5, (s, c, l, rel)
            r += 1
    assert r == len(z["step_rec"])
    assert np.array_equal(ctx.sched_events(), z["events"])
    with pytest.raises(abi.MoespacError):
        ctx.step(lg, h0, 2, h_out)  # one token per AR step
    ctx.close()


@pytest.mark.parametrize("d,ffn,kernel", [(512, 1024, abi.FFN_TENSOR), (4096, 14336, abi.FFN_TENSOR),
                                          (2048, 1408, abi.FFN_TENSOR), (1024, 64, abi.FFN_CUDACORE)])
def test_pack_unpack_round_trip(d, ffn, kernel):
    """moespac_unpack_expert inverts moespac_pack_expert bit for bit (it is
    what the parity tests above read synthetic images back through)."""
    g = torch.Generator(device="cuda").manual_seed(d + ffn)
    wg = torch.randint(-32768, 32767, (ffn, d), dtype=torch.int16, device="cuda", generator=g)
    wu = torch.randint(-32768, 32767, (ffn, d), dtype=torch.int16, device="cuda", generator=g)
    wd = torch.randint(-32768, 32767, (d, ffn), dtype=torch.int16, device="cuda", generator=g)
    img = abi.pack_expert(wg, wu, wd, kernel=kernel)
    back = abi.unpack_expert(img, d, ffn, kernel)
    for a, b in zip((wg, wu, wd), back):
        assert torch.equal(a, b)


def test_shared_gate_sigmoid_matches_oracle():
    """Qwen1.5-MoE's sigmoid shared-expert gate on a small grouped-K3 shape:
    explicit gate vectors, outputs against the fp64 oracle; the gate changes
    the output (vs weight 1) by the expected amount."""
    L, N, k, g, d, ffn, units = 2, 16, 4, 6, 1024, 128, 2
    rng = np.random.default_rng(21)
    T = g + 1
    cfg = abi.default_config(n_layers=L, n_experts=N, top_k=k, gamma=g, cache_ratio=1.0)
    kernel = abi.FFN_TENSOR
    outs = {}
    std = {(l, e): tuple(O.f32_to_bf16_bits(rng.normal(0, 0.03, sh).astype(np.float32))
                         for sh in ((ffn, d), (ffn, d), (d, ffn))) for l in range(L) for e in range(N)}
    shared = {l: [tuple(O.f32_to_bf16_bits(rng.normal(0, 0.03, sh).astype(np.float32))
                        for sh in ((ffn, d), (ffn, d), (d, ffn))) for _ in range(units)] for l in range(L)}
    wsg = [O.f32_to_bf16_bits(rng.normal(0, 0.04, d).astype(np.float32)) for _ in range(L)]
    gen_logits = O.Generator(L, N, k, g, seed=3)
    logits, ids, acc = gen_logits.next_step()
    h0 = O.f32_to_bf16_bits(rng.normal(0, 1, (T, d)).astype(np.float32))
    for mode in (abi.SHARED_GATE_NONE, abi.SHARED_GATE_SIGMOID):
        ctx = abi.Context(0, abi.ModelDesc(L, N, k, g, d, ffn, units, 1, kernel, 0, mode), cfg)
        arena = ctx.host_arena(L * N)
        for (l, e), wts in std.items():
            arena[l * N + e] = abi.pack_expert(*[torch.from_numpy(x.view(np.int16)).cuda() for x in wts],
                                               kernel=kernel).cpu().numpy().view(np.uint16)
        for l in range(L):
            ctx.set_shared(l, torch.stack([abi.pack_expert(*[torch.from_numpy(x.view(np.int16)).cuda() for x in wts],
                                                           kernel=kernel) for wts in shared[l]]))
            if mode == abi.SHARED_GATE_SIGMOID:
                ctx.set_shared_gate(l, wsg[l])
        ctx.finalize()
        h_out = np.zeros_like(h0)
        ctx.step(logits, h0, acc, h_out)
        v = ctx.views()
        hs = abi.fetch(v.h_dev, (L + 1, T, d), np.uint16)
        ys = abi.fetch(v.y_dev, (L, T, d), np.float32)
        for l in range(L):
            _, gates = O.router_topk(logits[l], k, 1)
            sg = O.shared_gate(hs[l], wsg[l]) if mode == abi.SHARED_GATE_SIGMOID else None
            y_ref = O.moe_layer(hs[l], ids[l], gates, {e: std[(l, e)] for e in range(N)}, shared[l],
                                shared_gates=sg)
            rel = np.linalg.norm(ys[l] - y_ref) / np.linalg.norm(y_ref)
            assert rel <= 1e-5, (mode, l, rel)
        outs[mode] = ys[0]
        ctx.close()
    assert np.linalg.norm(outs[0] - outs[1]) > 1e-2 * np.linalg.norm(outs[0])
    # the gate needs the grouped K3, which d = 4096 only gets at T <= 8:
    # gamma 8 (T = 9) falls back to the per-segment kernel
    cfg9 = abi.default_config(n_layers=L, n_experts=N, top_k=k, gamma=8, cache_ratio=1.0)
    with pytest.raises(abi.MoespacError) as ei:
        abi.Context(0, abi.ModelDesc(L, N, k, 8, 4096, ffn, units, 1, kernel, 0, abi.SHARED_GATE_SIGMOID), cfg9)
    assert ei.value.code == "E_INVALID"
