"""Parity of the sm_100a kernels (through the C ABI) against the CPU oracle.

K1 ids and K2 outputs must be bit-exact; K3 + combine must match the fp64
oracle within rel-L2 <= 1e-5 on the fp32 MoE output y (bf16 weights and
activations, fp32 accumulation on the device), and the bf16 layer output
within 1 bf16 ulp of bf16(h + y_ref) on >= 99.9% of elements.
"""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2603_09983_b200 import abi

pytestmark = pytest.mark.gpu

SHAPES = [(1, 8, 2, 4), (32, 8, 2, 4), (24, 60, 4, 6), (27, 64, 6, 8), (48, 128, 8, 8)]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


@pytest.mark.parametrize("shape", SHAPES)
def test_router_ids_bit_exact(shape):
    L, N, k, g = shape
    gen = O.Generator(L, N, k, g, seed=1)
    for _ in range(4):
        logits, ids_ref, _acc = gen.next_step()
        lg = torch.from_numpy(logits).cuda()
        for gm in (0, 1):
            ids, gates = abi.router_topk(lg, k, gm)
            assert np.array_equal(ids.cpu().numpy(), ids_ref)
            _, gref = O.router_topk(logits, k, gm)
            np.testing.assert_allclose(gates.cpu().numpy(), gref, rtol=3e-6, atol=1e-7)


def test_router_ties_signed_zero_and_odd_widths():
    rng = np.random.default_rng(7)
    for N, k in [(1, 1), (5, 5), (33, 3), (100, 7), (257, 16), (1024, 8)]:
        v = rng.integers(-3, 3, size=(64, N)).astype(np.float64)  # heavy ties
        v[0, :] = 0.0
        v[1, ::2] = -0.0
        lg = torch.from_numpy(v).cuda()
        ids, _ = abi.router_topk(lg, k, 0)
        ref, _ = O.router_topk(v, k, 0)
        assert np.array_equal(ids.cpu().numpy(), ref), (N, k)


def _k2_inputs(L, T, k, N, K, seed):
    rng = np.random.default_rng(seed)
    ids = np.zeros((L, T, k), np.int32)
    for l in range(L):
        for t in range(T):
            ids[l, t] = np.sort(rng.choice(N, k, replace=False))
    res = rng.random((L, N)) < 0.4
    loaded = res & (rng.random((L, N)) < 0.3)
    taus = rng.integers(1, K + 1, L).astype(np.int32)
    st = np.zeros((L, N, 4), np.int32)
    st[..., 0] = rng.integers(0, K + 1, (L, N))
    st[..., 1] = rng.integers(1, 6, (L, N))
    st[..., 2] = rng.integers(1, 6, (L, N))
    st[..., 3] = rng.integers(0, T + 1, (L, N))
    return ids, res, loaded, taus, st


def _bits(mask):
    L, N = mask.shape
    W = (N + 31) // 32
    out = np.zeros((L, W), np.uint32)
    for l in range(L):
        for e in np.nonzero(mask[l])[0]:
            out[l, e >> 5] |= np.uint32(1 << (e & 31))
    return out


@pytest.mark.parametrize("L,T,k,N,world,rank", [(1, 5, 2, 8, 1, 0), (24, 7, 4, 60, 1, 0), (48, 9, 8, 128, 1, 0),
                                                 (27, 9, 6, 64, 4, 3), (8, 16, 8, 256, 2, 1)])
@pytest.mark.parametrize("lam,adaptive", [(0.1, 1), (0.7, 1), (0.1, 0)])
def test_hist_scan_observe_bit_exact(L, T, k, N, world, rank, lam, adaptive):
    K = min(4, T - 1)
    ids, res, loaded, taus, st = _k2_inputs(L, T, k, N, K, seed=L * 131 + N)
    dv = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    t_ids, t_rb, t_lb, t_tau, t_st = dv(ids), dv(_bits(res).view(np.int32)), dv(_bits(loaded).view(np.int32)), dv(taus), dv(st)
    outs = {n: torch.full(s, -7, dtype=torch.int32, device="cuda") for n, s in
            [("freqs", (L, N)), ("offsets", (L, N + 1)), ("perm", (L, T * k)), ("hit_list", (L, N)),
             ("hit_ord", (L, N)), ("counters", (L, 8)), ("scores", (L, N))]}
    a = abi.K2Args(abi.ptr(t_ids), L, T, k, N, abi.ptr(t_rb), abi.ptr(t_lb), abi.ptr(t_tau), abi.ptr(t_st), K,
                   adaptive, lam, rank, world, abi.ptr(outs["freqs"]), abi.ptr(outs["offsets"]),
                   abi.ptr(outs["perm"]), abi.ptr(outs["hit_list"]), abi.ptr(outs["hit_ord"]),
                   abi.ptr(outs["counters"]), abi.ptr(outs["scores"]))
    import ctypes
    abi.check(abi.lib().moespac_hist_scan_observe(ctypes.byref(a), abi._stream(None)))
    torch.cuda.synchronize()
    got = {n: t.cpu().numpy() for n, t in outs.items()}
    st_new = t_st.cpu().numpy()
    for l in range(L):
        f, off, perm = O.hist_scan(ids[l], N)
        assert np.array_equal(got["freqs"][l], f)
        assert np.array_equal(got["offsets"][l], off)
        assert np.array_equal(got["perm"][l], perm)
        ref_st = O.estimator_observe(st[l], f, K, lam, adaptive)
        assert np.array_equal(st_new[l], ref_st)
        assert np.array_equal(got["scores"][l], ref_st[:, 0])
        cnt = O.realized_split(f, st[l, :, 0], res[l].astype(np.uint8), taus[l], loaded[l].astype(np.uint8))
        assert np.array_equal(got["counters"][l, :7], cnt[:7])
        hits = [e for e in range(N) if f[e] > 0 and res[l, e] and e % world == rank]
        assert got["counters"][l, 7] == len(hits)
        assert np.array_equal(got["hit_list"][l, :len(hits)], hits)
        ho = np.full(N, -1, np.int32)
        ho[hits] = np.arange(len(hits))
        assert np.array_equal(got["hit_ord"][l], ho)


def _check_bf16_residual(h, y_ref, got):
    """bf16(h + y): within one bf16 rounding of the exact value, plus the fp32
    error of y itself (matters only under cancellation h ~ -y)."""
    exact = O.bf16_bits_to_f32(h).astype(np.float64) + y_ref
    g = O.bf16_bits_to_f32(got).astype(np.float64)
    tol = np.abs(exact) * 2.0 ** -8 + 1e-5 * np.abs(y_ref).max() + 1e-30
    assert np.all(np.abs(g - exact) <= tol)


def _rand_experts(rng, n, d, ffn, std=0.02):
    out = []
    for _ in range(n):
        out.append(tuple(O.f32_to_bf16_bits(rng.normal(0, std, s).astype(np.float32))
                         for s in ((ffn, d), (ffn, d), (d, ffn))))
    return out


def _pack(experts, kernel=abi.FFN_AUTO):
    imgs = []
    for wg, wu, wd in experts:
        t = [torch.from_numpy(x.view(np.int16)).cuda() for x in (wg, wu, wd)]
        imgs.append(abi.pack_expert(*t, kernel=kernel))
    return torch.stack(imgs)


def _kernels(d, ffn):
    ks = []
    if d % 512 == 0 and ffn % 16 == 0:
        ks.append(abi.FFN_CUDACORE)
    if d % 128 == 0 and ffn % 64 == 0:
        ks.append(abi.FFN_TENSOR)
    return ks


@pytest.mark.parametrize("N,k,T,d,ffn,n_shared,gate_mode,resident_frac", [
    (8, 2, 5, 512, 1024, 0, 0, 1.0),      # tiny shape
    (8, 2, 5, 1024, 256, 0, 0, 0.5),
    (16, 4, 7, 2048, 176, 2, 1, 0.6),     # shared units (DSV2/Qwen1.5 style), ffn % 16 == 0
    (32, 8, 9, 2048, 96, 0, 0, 0.8),      # Qwen3-like routing density
    (8, 2, 16, 4096, 64, 1, 0, 1.0),      # max verification window, d = 4096
    (4, 4, 3, 512, 32, 0, 0, 1.0),        # every token on every expert
    (16, 4, 7, 2048, 176, 0, 1, 0.6),     # isolation variants
    (16, 4, 7, 2048, 176, 2, 0, 1.0),
    (16, 4, 7, 1024, 176, 2, 1, 0.6),
    (16, 4, 7, 2048, 192, 0, 0, 1.0),
    (8, 2, 5, 4096, 128, 0, 0, 1.0),      # Mixtral d
    (60, 4, 7, 2048, 1408, 4, 1, 0.5),    # Qwen1.5 shape
    (128, 8, 9, 2048, 768, 0, 0, 0.6),    # Qwen3 shape
    (8, 2, 5, 4096, 256, 0, 0, 1.0),      # Mixtral d, tensor-core eligible
    (16, 4, 16, 1024, 128, 1, 0, 0.7),    # T = 16 (N fully used)
    (16, 4, 9, 128, 64, 0, 0, 1.0),       # smallest tensor-core shape
    (64, 6, 9, 2048, 1408, 2, 1, 0.3),    # DeepSeek-V2-Lite shape
])
@pytest.mark.parametrize("kernel", [abi.FFN_CUDACORE, abi.FFN_TENSOR], ids=["cudacore", "tensor"])
def test_expert_ffn_and_combine(N, k, T, d, ffn, n_shared, gate_mode, resident_frac, kernel):
    if kernel not in _kernels(d, ffn):
        pytest.skip("shape not supported by this kernel variant")
    _ffn_case(N, k, T, d, ffn, n_shared, gate_mode, resident_frac, kernel, 0)


@pytest.mark.parametrize("accum", [1, 2, 3, 4], ids=["smem", "global", "tmem", "grouped"])
@pytest.mark.parametrize("N,k,T,d,ffn,n_shared,gate_mode,resident_frac", [
    (128, 8, 9, 2048, 768, 0, 0, 0.6),     # Qwen3 shape
    (16, 4, 16, 1024, 128, 1, 0, 0.7),     # T = 16 + shared unit
    (16, 4, 9, 128, 64, 0, 0, 1.0),        # smallest shape (one M-tile)
    (60, 4, 7, 2048, 1408, 4, 1, 0.5),     # Qwen1.5 shape
])
def test_expert_ffn_tc_accumulator_modes(N, k, T, d, ffn, n_shared, gate_mode, resident_frac, accum):
    """Every down-projection accumulator of the tensor-core K3 (shared memory,
    global partial block, TMEM per expert, grouped whole-CTA TMEM) against the
    fp64 oracle."""
    if abi.FFN_TENSOR not in _kernels(d, ffn):
        pytest.skip("shape not supported by the tensor-core kernel")
    _ffn_case(N, k, T, d, ffn, n_shared, gate_mode, resident_frac, abi.FFN_TENSOR, accum)


@pytest.mark.parametrize("grid", [1, 7, 16, 37, 148, 300, 1000])
@pytest.mark.parametrize("N,k,T,d,ffn,n_shared,gate_mode,resident_frac", [
    (128, 8, 9, 2048, 768, 0, 0, 0.6),     # Qwen3 shape
    (64, 6, 9, 2048, 1408, 2, 1, 0.3),     # DeepSeek-V2-Lite shape (shared units)
    (16, 4, 16, 1024, 128, 1, 0, 0.7),     # T = 16, 2 quarters/entry chunk crossings
    (4, 4, 3, 512, 64, 0, 0, 1.0),         # every token on every expert, 1 chunk per expert
    (8, 2, 5, 4096, 448, 0, 0, 1.0),       # d = 4096, T <= 8: N = 8 MMAs, D2 in 8 columns per M-tile
    (8, 2, 8, 4096, 192, 1, 0, 0.7),       # d = 4096, T = 8 + shared unit
])
def test_expert_ffn_grouped_grids(N, k, T, d, ffn, n_shared, gate_mode, resident_frac, grid):
    """Grouped K3: groups of eight 8-row units cross chunk and expert
    boundaries, odd groups take their last down K-step half from the zero
    buffer, and CTAs own 0..many units depending on the grid; the combine's
    per-CTA row lists must cover exactly the CTAs that touched each token."""
    import ctypes
    if abi.FFN_TENSOR not in _kernels(d, ffn):
        pytest.skip("shape not supported by the tensor-core kernel")
    upe = ffn // 8
    maxu = -(-((N + n_shared) * upe) // grid)
    if (maxu - 1) // upe + 2 > 32:
        pytest.skip("grid below the grouped kernel's per-CTA entry limit")
    # few CTAs -> long TMEM accumulation chains over many experts; a = silu(g)u·g
    # enters the down MMA as bf16 hi + lo (~2^-17 relative), so allow 3e-5
    _ffn_case(N, k, T, d, ffn, n_shared, gate_mode, resident_frac, abi.FFN_TENSOR, 4, grid=grid, tol=3e-5)


@pytest.mark.parametrize("absorb,drain_late", [(1, 0), (2, 0), (3, 1), (0, 1)])
@pytest.mark.parametrize("grid", [37, 148])
@pytest.mark.parametrize("N,k,T,d,ffn,n_shared,gate_mode,resident_frac", [
    (128, 8, 9, 2048, 768, 0, 0, 0.6),     # Qwen3 shape
    (64, 6, 9, 2048, 1408, 2, 1, 0.3),     # DeepSeek-V2-Lite shape (shared units)
    (8, 2, 5, 4096, 448, 0, 0, 1.0),       # N = 8 mode
    (16, 4, 9, 128, 64, 0, 0, 1.0),        # one M-tile: the drain stages in the ring
])
def test_expert_ffn_grouped_group_variants(monkeypatch, N, k, T, d, ffn, n_shared, gate_mode, resident_frac, grid,
                                           absorb, drain_late):
    """Grouped K3 knobs: a remainder of <= absorb units joins the group before
    it as a second M-tile; the D2 drain either follows the last DN pass's
    entries chunk by chunk (staged in the dead h^T slices) or waits for the
    whole pass (staged in the ring)."""
    if abi.FFN_TENSOR not in _kernels(d, ffn):
        pytest.skip("shape not supported by the tensor-core kernel")
    monkeypatch.setenv("MOESPAC_TAIL_ABSORB", str(absorb))
    monkeypatch.setenv("MOESPAC_DRAIN_LATE", str(drain_late))
    _ffn_case(N, k, T, d, ffn, n_shared, gate_mode, resident_frac, abi.FFN_TENSOR, 4, grid=grid, tol=3e-5)


@pytest.mark.parametrize("grid", [1, 5, 37, 148, 300])
@pytest.mark.parametrize("N,k,T,d,ffn,n_shared,gate_mode,resident_frac", [
    (8, 2, 5, 4096, 448, 0, 0, 1.0),      # Mixtral d: chunk pieces split across CTAs at every grid
    (8, 2, 16, 4096, 192, 1, 0, 0.7),     # T = 16 + shared unit, expert boundaries inside CTA ranges
    (4, 2, 9, 3072, 320, 0, 1, 1.0),      # d = 3072 (not a power of two), 5 chunks per expert
])
def test_expert_ffn_per_segment_grids(N, k, T, d, ffn, n_shared, gate_mode, resident_frac, grid):
    """Per-segment K3 (d > 2048, shared-memory accumulator): CTA ranges of
    0..many 8-row units start and end anywhere inside chunks and experts;
    partial pieces, per-lane tile copies and per-expert flushes against the
    fp64 oracle."""
    if abi.FFN_TENSOR not in _kernels(d, ffn):
        pytest.skip("shape not supported by the tensor-core kernel")
    # accum 1 = the per-segment kernel (auto picks the grouped one at T <= 8)
    _ffn_case(N, k, T, d, ffn, n_shared, gate_mode, resident_frac, abi.FFN_TENSOR, 1, grid=grid)


def _ffn_case(N, k, T, d, ffn, n_shared, gate_mode, resident_frac, kernel, accum, grid=None, tol=1e-5):
    rng = np.random.default_rng(N * 7 + T)
    experts = _rand_experts(rng, N, d, ffn)
    shared = _rand_experts(rng, n_shared, d, ffn)
    logits = rng.normal(0, 1, (T, N))
    ids_ref, gates_ref = O.router_topk(logits, k, gate_mode)
    h = O.f32_to_bf16_bits(rng.normal(0, 1, (T, d)).astype(np.float32))
    resident = rng.random(N) < resident_frac
    # device inputs
    lg = torch.from_numpy(logits).cuda()
    ids, gates = abi.router_topk(lg, k, gate_mode)
    pool = _pack(experts, kernel)
    shared_t = _pack(shared, kernel) if n_shared else torch.zeros(1, dtype=torch.int16, device="cuda")
    slot_of = torch.arange(N, dtype=torch.int32, device="cuda")
    W = (N + 31) // 32
    rb = torch.from_numpy(_bits(resident[None]).view(np.int32)).cuda()
    taus = torch.ones(1, dtype=torch.int32, device="cuda")
    st = torch.zeros((N, 4), dtype=torch.int32, device="cuda")
    bufs = {n: torch.zeros(s, dtype=torch.int32, device="cuda") for n, s in
            [("freqs", N), ("offsets", N + 1), ("perm", T * k), ("hl", N), ("ho", N), ("cnt", 8), ("sc", N)]}
    import ctypes
    a2 = abi.K2Args(abi.ptr(ids), 1, T, k, N, abi.ptr(rb), None, abi.ptr(taus), abi.ptr(st), 4, 1, 0.1, 0, 1,
                    abi.ptr(bufs["freqs"]), abi.ptr(bufs["offsets"]), abi.ptr(bufs["perm"]), abi.ptr(bufs["hl"]),
                    abi.ptr(bufs["ho"]), abi.ptr(bufs["cnt"]), abi.ptr(bufs["sc"]))
    s0 = abi._stream(None)
    abi.check(abi.lib().moespac_hist_scan_observe(ctypes.byref(a2), s0))
    grid = grid or torch.cuda.get_device_properties(0).multi_processor_count
    ws = torch.full((abi.lib().moespac_ffn_workspace_bytes(T, d, N, n_shared, grid) // 4,), float("nan"),
                    dtype=torch.float32, device="cuda")
    h_t = torch.from_numpy(h.view(np.int16)).cuda()
    hT = abi.build_hT(h_t)
    fa = abi.FfnArgs(abi.ptr(h_t), T, d, ffn, k, N, abi.ptr(bufs["perm"]), abi.ptr(bufs["offsets"]), abi.ptr(gates),
                     abi.ptr(bufs["hl"]), abi.ptr(bufs["cnt"]), abi.ptr(slot_of), abi.ptr(pool), abi.ptr(shared_t),
                     n_shared, abi.ptr(ws), grid, kernel, abi.ptr(hT), None, accum)
    abi.check(abi.lib().moespac_expert_ffn(ctypes.byref(fa), s0))
    y = torch.zeros((T, d), dtype=torch.float32, device="cuda")
    h_out = torch.zeros((T, d), dtype=torch.int16, device="cuda")
    ca = abi.CombineArgs(abi.ptr(h_t), None, T, d, ffn, k, abi.ptr(ids), abi.ptr(bufs["ho"]), abi.ptr(bufs["cnt"]),
                         n_shared, grid, abi.ptr(ws), abi.ptr(y), abi.ptr(h_out), accum, kernel)
    abi.check(abi.lib().moespac_ffn_combine(ctypes.byref(ca), s0))
    torch.cuda.synchronize()
    y_ref = O.moe_layer(h, ids_ref, gates_ref, {e: experts[e] for e in range(N) if resident[e]}, shared)
    yg = y.cpu().numpy().astype(np.float64)
    rel = np.linalg.norm(yg - y_ref) / max(np.linalg.norm(y_ref), 1e-30)
    assert rel <= tol, rel
    # bf16 layer output: within one bf16 ulp of bf16(h + y_ref)
    _check_bf16_residual(h, y_ref, h_out.cpu().numpy().view(np.uint16))


@pytest.mark.parametrize("kernel", [abi.FFN_CUDACORE, abi.FFN_TENSOR], ids=["cudacore", "tensor"])
def test_expert_ffn_deterministic(kernel):
    import ctypes
    rng = np.random.default_rng(11)
    N, k, T, d, ffn = 16, 4, 9, 2048, 128
    pool = _pack(_rand_experts(rng, N, d, ffn), kernel)
    ids, gates = abi.router_topk(torch.from_numpy(rng.normal(0, 1, (T, N))).cuda(), k, 0)
    h_t = torch.from_numpy(O.f32_to_bf16_bits(rng.normal(0, 1, (T, d)).astype(np.float32)).view(np.int16)).cuda()
    slot_of = torch.arange(N, dtype=torch.int32, device="cuda")
    outs = []
    for _ in range(3):
        bufs = {n: torch.zeros(s, dtype=torch.int32, device="cuda") for n, s in
                [("freqs", N), ("offsets", N + 1), ("perm", T * k), ("hl", N), ("ho", N), ("cnt", 8), ("sc", N)]}
        rb = torch.full((1,), -1, dtype=torch.int32, device="cuda")
        taus = torch.ones(1, dtype=torch.int32, device="cuda")
        st = torch.zeros((N, 4), dtype=torch.int32, device="cuda")
        a2 = abi.K2Args(abi.ptr(ids), 1, T, k, N, abi.ptr(rb), None, abi.ptr(taus), abi.ptr(st), 4, 1, 0.1, 0, 1,
                        abi.ptr(bufs["freqs"]), abi.ptr(bufs["offsets"]), abi.ptr(bufs["perm"]),
                        abi.ptr(bufs["hl"]), abi.ptr(bufs["ho"]), abi.ptr(bufs["cnt"]), abi.ptr(bufs["sc"]))
        abi.check(abi.lib().moespac_hist_scan_observe(ctypes.byref(a2), abi._stream(None)))
        ws = torch.full((abi.lib().moespac_ffn_workspace_bytes(T, d, N, 0, 148) // 4,), float("nan"), device="cuda")
        hT = abi.build_hT(h_t)
        fa = abi.FfnArgs(abi.ptr(h_t), T, d, ffn, k, N, abi.ptr(bufs["perm"]), abi.ptr(bufs["offsets"]),
                         abi.ptr(gates), abi.ptr(bufs["hl"]), abi.ptr(bufs["cnt"]), abi.ptr(slot_of), abi.ptr(pool),
                         None, 0, abi.ptr(ws), 148, kernel, abi.ptr(hT))
        abi.check(abi.lib().moespac_expert_ffn(ctypes.byref(fa), abi._stream(None)))
        y = torch.zeros((T, d), dtype=torch.float32, device="cuda")
        ca = abi.CombineArgs(None, None, T, d, ffn, k, abi.ptr(ids), abi.ptr(bufs["ho"]), abi.ptr(bufs["cnt"]), 0,
                             148, abi.ptr(ws), abi.ptr(y), None, 0, kernel)
        abi.check(abi.lib().moespac_ffn_combine(ctypes.byref(ca), abi._stream(None)))
        torch.cuda.synchronize()
        outs.append(y.cpu().numpy())
    assert np.isfinite(outs[0]).all()
    assert all(np.array_equal(outs[0], o) for o in outs[1:])
