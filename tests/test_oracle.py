"""Pin the CPU oracle before trusting it (CPU only).

The C restatement (oracle/moespac_oracle.c) is checked against the committed
golden fixtures made by the unmodified reference (tests/golden/*.npz) and,
where oracle/_ref is built, against the live reference library. Also the
reference's own known-answer tests for the path.
"""
import glob
import os

import numpy as np
import pytest

import oracle as O
from conftest import ref_or_skip

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _sims():
    return sorted(glob.glob(os.path.join(GOLDEN, "sim_*.npz")))


@pytest.mark.parametrize("path", _sims(), ids=lambda p: os.path.basename(p)[4:-4])
def test_generator_and_topk_match_golden_trace(path):
    z = np.load(path)
    L, N, k, g = int(z["L"]), int(z["N"]), int(z["k"]), int(z["gamma"])
    gen = O.Generator(L, N, k, g, drift=float(z["drift_scale"]), shift_period=int(z["shift_period"]))
    for s in range(len(z["accepted"])):
        logits, ids, acc = gen.next_step()
        assert acc == z["accepted"][s]
        assert np.array_equal(ids, z["ids"][s])
        ids2, _ = O.router_topk(logits, k)  # K1 oracle on the emitted noisy logits
        assert np.array_equal(ids2, z["ids"][s])


def test_estimator_matches_golden():
    z = np.load(os.path.join(GOLDEN, "estimator.npz"))
    meta = z["meta"]
    for i, (cap, gamma, lam, adaptive) in enumerate(meta):
        st0 = z[f"st0_{i}"]
        assert np.array_equal(st0, O.estimator_init(st0.shape[0], int(gamma)))  # ctor state
        st = st0.copy()
        for f in z[f"freqs_{i}"]:
            st = O.estimator_observe(st, f, int(cap), float(lam), bool(adaptive))
        assert np.array_equal(st, z[f"st_{i}"]), i


def test_estimator_fma_sensitive_floor_cases():
    # calibrate() floors (1-l)*b + l*m; contracting to an FMA flips some floors
    # (SURVEY.md §0 item 6). Sweep the whole (lambda, theta, delta) grid.
    for lam in [i / 10 for i in range(11)]:
        b = np.arange(1, 65)
        for m in range(1, 130):
            st = np.zeros((64, 4), np.int32)
            st[:, 1] = b
            st[:, 2] = 64
            f = np.full(64, m, np.int32)
            got = O.estimator_observe(st, f, 4, lam, True)[:, 1]
            want = np.maximum(1, np.floor((1.0 - lam) * b.astype(np.float64) + lam * float(m))).astype(np.int32)
            # numpy evaluates the two products and the sum as separate IEEE ops
            assert np.array_equal(got, want)


def test_reference_kats_estimator():
    # utility_estimator_test.cpp:64-81 worked step and :111-120 one-sided boundaries
    st = np.array([[2, 4, 4, 1]], np.int32)
    st = O.estimator_observe(st, np.array([6], np.int32), 4, 0.1)
    assert st.tolist() == [[3, 4, 4, 6]]
    st = np.array([[1, 6, 6, 10]], np.int32)
    st = O.estimator_observe(st, np.array([14], np.int32), 4, 0.2)
    assert st[0, 1] == 5 and st[0, 2] == 6
    st = O.estimator_observe(st, np.array([4], np.int32), 4, 0.2)
    assert st[0, 1] == 5 and st[0, 2] == 6
    # theta init floor(gamma/2) (utility_estimator_test.cpp:25-43)
    assert O.estimator_init(3, 8)[:, 1].tolist() == [4, 4, 4]
    assert O.estimator_init(1, 3)[0, 1] == 1


def test_reference_kat_freqs():
    # trace_model_test.cpp:161-168
    f, off, perm = O.hist_scan(np.array([[0, 1], [0, 2], [1, 0]], np.int32), 4)
    assert f.tolist() == [3, 2, 1, 0]
    assert off.tolist() == [0, 3, 5, 6, 6]
    # (expert, token, slot) order: expert 0 at (0,0), (1,0), (2,1); expert 1 at (0,1), (2,0)
    assert perm.tolist() == [0, 2, 5, 1, 4, 3]


def test_reference_kat_zero_noise_pins_routing():
    # trace_model_test.cpp:129-139
    gen = O.Generator(3, 16, 4, 4, drift=0.0, noise=0.0, seed=42)
    first = None
    for _ in range(5):
        _, ids, _ = gen.next_step()
        for l in range(3):
            assert all(np.array_equal(ids[l, t], ids[l, 0]) for t in range(5))
        first = ids if first is None else first
        assert np.array_equal(ids, first)


def test_topk_tie_rules():
    v = np.array([[1.0, 3.0, 3.0, -0.0, 0.0, 3.0]])
    ids, _ = O.router_topk(v, 2)
    assert ids.tolist() == [[1, 2]]
    ids, _ = O.router_topk(v, 4)
    assert ids.tolist() == [[0, 1, 2, 5]]
    ids, _ = O.router_topk(np.array([[-0.0, 0.0, -1.0]]), 1)
    assert ids.tolist() == [[0]]  # -0.0 == +0.0 -> lower id


def test_gates_eq3():
    v = np.array([[0.0, 1.0, 2.0, 3.0]])
    _, g0 = O.router_topk(v, 2, 0)
    e = np.exp([2.0, 3.0])
    np.testing.assert_allclose(g0[0], e / e.sum(), rtol=1e-15)
    _, g1 = O.router_topk(v, 2, 1)
    np.testing.assert_allclose(g1[0], e / np.exp([0.0, 1, 2, 3]).sum(), rtol=1e-15)


def test_ffn_oracle_against_numpy():
    rng = np.random.default_rng(0)
    d, ffn, T = 64, 48, 5
    h = O.f32_to_bf16_bits(rng.normal(0, 1, (T, d)).astype(np.float32))
    W = [O.f32_to_bf16_bits(rng.normal(0, 0.1, s).astype(np.float32)) for s in ((ffn, d), (ffn, d), (d, ffn))]
    y = np.zeros((T, d))
    O.expert_apply(h, [1, 3], [0.25, 0.75], *W, y)
    hf = O.bf16_bits_to_f32(h).astype(np.float64)
    wg, wu, wd = (O.bf16_bits_to_f32(w).astype(np.float64) for w in W)
    ref = np.zeros((T, d))
    for t, gt in [(1, 0.25), (3, 0.75)]:
        g = wg @ hf[t]
        a = g / (1 + np.exp(-g)) * (wu @ hf[t])
        ref[t] = gt * (wd @ a)
    np.testing.assert_allclose(y, ref, rtol=1e-10, atol=1e-12)


@pytest.mark.ref
def test_oracle_generator_vs_live_reference_regimes():
    ref_or_skip()
    for L, N, k, g in [(2, 8, 2, 4), (3, 60, 4, 6), (2, 128, 8, 8)]:
        for extra in ({}, {"drift_scale": 0.0, "route_noise": 0.0}, {"shift_period": 7, "drift_scale": 0.5}):
            cfg = O.default_config(n_layers=L, n_experts=N, top_k=k, gamma=g, **extra)
            ids, acc = O.ref_trace(cfg, 30)
            gen = O.Generator(L, N, k, g, drift=cfg.drift_scale, noise=cfg.route_noise,
                              shift_period=cfg.shift_period)
            for s in range(30):
                _, i2, a2 = gen.next_step()
                assert a2 == acc[s] and np.array_equal(i2, ids[s])


@pytest.mark.ref
def test_oracle_estimator_vs_live_reference_fuzz():
    ref_or_skip()
    rng = np.random.default_rng(5)
    for _ in range(200):
        cap = int(rng.integers(1, 5))
        gamma = cap + int(rng.integers(0, 6))
        lam = float(rng.integers(0, 11)) / 10
        n = int(rng.integers(1, 20))
        st0 = O.estimator_init(n, gamma)
        fs = rng.integers(0, gamma + 3, (20, n)).astype(np.int32)
        want = O.ref_estimator_run(st0, fs, cap, lam, gamma)
        got = st0
        for f in fs:
            got = O.estimator_observe(got, f, cap, lam)
        assert np.array_equal(got, want)


@pytest.mark.parametrize("T,N,d", [(5, 8, 512), (9, 128, 2048), (16, 60, 1024)])
def test_router_gemv_restatement(T, N, d):
    """The fp32 fixed-order router GEMV (model mode, K0's order) is the dot
    product W_g h to fp32 accuracy."""
    rng = np.random.default_rng(T * N)
    W = O.f32_to_bf16_bits(rng.normal(0, 0.05, (N, d)).astype(np.float32))
    h = O.f32_to_bf16_bits(rng.normal(0, 1, (T, d)).astype(np.float32))
    got = O.router_gemv(W, h)
    want = O.bf16_bits_to_f32(h).astype(np.float64) @ O.bf16_bits_to_f32(W).astype(np.float64).T
    assert np.all(np.abs(got - want) <= 1e-5 * np.abs(want).max() + 1e-6)
    assert np.array_equal(got, O.router_gemv(W, h))
