"""TEST INFRASTRUCTURE ONLY — ctypes/numpy front-end to the CPU oracle.

Importable only from tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs. The product package never imports it.

Two libraries:
  * ``_build/liboracle.so`` — plain-C restatement (moespac_oracle.c); always
    built by ``make -C oracle`` (no reference tree needed);
  * ``_ref/libmoesim_ref.so`` — the unmodified reference ``moesim_core``
    compiled from /root/reference/proj/core/src/*.cpp plus ref_shim.cpp.
    Built only where /root/reference exists; the built file travels to the
    GPU box with the repo snapshot.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_ORC_PATH = os.path.join(HERE, "_build", "liboracle.so")
_REF_PATH = os.path.join(HERE, "_ref", "libmoesim_ref.so")

_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_u16p = np.ctypeslib.ndpointer(np.uint16, flags="C_CONTIGUOUS")


def build() -> None:
    subprocess.check_call(["make", "-s", "-C", HERE])


_orc = None
_ref = None


def orc() -> C.CDLL:
    global _orc
    if _orc is None:
        if not os.path.exists(_ORC_PATH):
            build()
        lib = C.CDLL(_ORC_PATH)
        lib.orc_gen_create.restype = C.c_void_p
        lib.orc_gen_create.argtypes = [C.c_int] * 4 + [C.c_double] * 3 + [C.c_int, C.c_uint64]
        lib.orc_gen_destroy.argtypes = [C.c_void_p]
        lib.orc_gen_next.restype = C.c_int
        lib.orc_gen_next.argtypes = [C.c_void_p, C.c_void_p, _i32p]
        lib.orc_router_topk.argtypes = [_f64p, C.c_int, C.c_int, C.c_int, C.c_int, _i32p, C.c_void_p]
        lib.orc_hist_scan.argtypes = [_i32p, C.c_int, C.c_int, C.c_int, _i32p, _i32p, _i32p]
        lib.orc_estimator_init.argtypes = [_i32p, C.c_int, C.c_int, C.c_int, C.c_int]
        lib.orc_estimator_observe.argtypes = [_i32p, _i32p, C.c_int, C.c_int, C.c_double, C.c_int]
        lib.orc_realized_split.argtypes = [_i32p, _i32p, _u8p, C.c_void_p, C.c_int, C.c_int, _i64p]
        lib.orc_expert_apply.argtypes = [_u16p, C.c_int, C.c_int, _i32p, _f64p, C.c_int,
                                         C.c_void_p, C.c_void_p, C.c_void_p, _f64p, C.c_int]
        lib.orc_expert_apply_f32.argtypes = [C.c_void_p, C.c_int, C.c_int, _i32p, _f32p, C.c_int,
                                             C.c_void_p, C.c_void_p, C.c_void_p, _f32p, C.c_int]
        lib.orc_router_gemv.argtypes = [_u16p, _u16p, C.c_int, C.c_int, C.c_int, _f64p]
        lib.orc_max_threads.restype = C.c_int
        lib.orc_f32_to_bf16.restype = C.c_uint16
        lib.orc_f32_to_bf16.argtypes = [C.c_float]
        _orc = lib
    return _orc


def ref_available() -> bool:
    return os.path.exists(_REF_PATH)


# --------------------------------------------------------------------------
# Synthetic workload (restated TraceGenerator, trace_model.cpp:59-109)
# --------------------------------------------------------------------------
class Generator:
    """Restated reference generator that also returns the noisy fp64 logits."""

    def __init__(self, L, N, k, gamma, alpha=0.8, drift=0.02, noise=0.2, shift_period=0, seed=1):
        self.L, self.N, self.k, self.gamma = L, N, k, gamma
        self.T = gamma + 1
        self._lib = orc()
        self._h = self._lib.orc_gen_create(L, N, k, gamma, alpha, drift, noise, shift_period, seed)
        if not self._h:
            raise ValueError("invalid TraceConfig")

    def next_step(self):
        logits = np.empty((self.L, self.T, self.N), np.float64)
        ids = np.empty((self.L, self.T, self.k), np.int32)
        acc = self._lib.orc_gen_next(self._h, logits.ctypes.data, ids)
        return logits, ids, acc

    def __del__(self):
        if getattr(self, "_h", None):
            self._lib.orc_gen_destroy(self._h)
            self._h = None


def router_gemv(W: np.ndarray, h: np.ndarray) -> np.ndarray:
    """Router logits W_g h [T][N] (fp64 widened from the device K0's fp32 order)."""
    W = np.ascontiguousarray(W, np.uint16)
    h = np.ascontiguousarray(h, np.uint16)
    N, d = W.shape
    T = h.shape[0]
    out = np.empty((T, N), np.float64)
    orc().orc_router_gemv(W.reshape(-1), h.reshape(-1), T, N, d, out.reshape(-1))
    return out


def router_topk(logits: np.ndarray, k: int, gate_mode: int = 0):
    logits = np.ascontiguousarray(logits, np.float64)
    N = logits.shape[-1]
    rows = logits.size // N
    ids = np.empty(rows * k, np.int32)
    gates = np.empty(rows * k, np.float64)
    orc().orc_router_topk(logits.reshape(-1), rows, N, k, gate_mode, ids, gates.ctypes.data)
    shp = logits.shape[:-1] + (k,)
    return ids.reshape(shp), gates.reshape(shp)


def hist_scan(ids: np.ndarray, N: int):
    ids = np.ascontiguousarray(ids, np.int32)
    T, k = ids.shape
    freqs = np.empty(N, np.int32)
    offs = np.empty(N + 1, np.int32)
    perm = np.empty(T * k, np.int32)
    orc().orc_hist_scan(ids.reshape(-1), T, k, N, freqs, offs, perm)
    return freqs, offs, perm


def estimator_init(N, gamma, init_up=-1, init_down=-1):
    st = np.empty((N, 4), np.int32)
    orc().orc_estimator_init(st.reshape(-1), N, gamma, init_up, init_down)
    return st


def estimator_observe(state: np.ndarray, freqs: np.ndarray, cap: int, lam: float, adaptive=True):
    st = np.ascontiguousarray(state, np.int32).copy()
    orc().orc_estimator_observe(st.reshape(-1), np.ascontiguousarray(freqs, np.int32),
                                st.shape[0], cap, lam, int(adaptive))
    return st


def realized_split(freqs, scores, resident, tau, loaded=None):
    out = np.zeros(8, np.int64)
    ld = None if loaded is None else np.ascontiguousarray(loaded, np.uint8)
    orc().orc_realized_split(np.ascontiguousarray(freqs, np.int32),
                             np.ascontiguousarray(scores, np.int32),
                             np.ascontiguousarray(resident, np.uint8),
                             None if ld is None else ld.ctypes.data, len(freqs), tau, out)
    return out


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (np.asarray(b, np.uint16).astype(np.uint32) << 16).view(np.float32)


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    return r


def expert_apply(h_bits, tok, gate, wg, wu, wd, y, n_threads=0):
    """y[tok[i]] += gate[i] * SwiGLU_e(h[tok[i]]) in fp64 (standard layouts)."""
    d = h_bits.shape[1]
    ffn = wg.shape[0]
    tok = np.ascontiguousarray(tok, np.int32)
    gate = np.ascontiguousarray(gate, np.float64)
    wg = np.ascontiguousarray(wg, np.uint16)
    wu = np.ascontiguousarray(wu, np.uint16)
    wd = np.ascontiguousarray(wd, np.uint16)
    orc().orc_expert_apply(np.ascontiguousarray(h_bits, np.uint16), d, ffn, tok, gate, len(tok),
                           wg.ctypes.data, wu.ctypes.data, wd.ctypes.data, y, n_threads)


def shared_gate(h_bits, w_sg_bits):
    """Qwen1.5-MoE shared-expert gate (public HF config `shared_expert_gate`,
    SURVEY.md §8 gate flags; not in the reference): g_t = sigmoid(w_sg . h_t)
    in fp64, one value per token."""
    h = bf16_bits_to_f32(h_bits).astype(np.float64)
    w = bf16_bits_to_f32(w_sg_bits).astype(np.float64)
    return 1.0 / (1.0 + np.exp(-(h @ w)))


def moe_layer(h_bits, ids, gates, experts, shared=(), n_threads=0, shared_gates=None):
    """Eq. 3 MoE layer output y (fp64 [T][d]) over the given experts.

    experts: dict expert_id -> (wg[ffn][d], wu[ffn][d], wd[d][ffn]) bf16 bits;
             activations whose expert is absent from the dict are skipped
             (cold / other-shard experts).
    shared:  sequence of (wg, wu, wd) applied to every token with gate 1, or
             with gate shared_gates[t] when given (see shared_gate()).
    """
    T, d = h_bits.shape
    y = np.zeros((T, d), np.float64)
    k = ids.shape[1]
    for e in sorted(experts):
        toks = [t for t in range(T) for j in range(k) if ids[t, j] == e]
        g = [gates[t, j] for t in range(T) for j in range(k) if ids[t, j] == e]
        if toks:
            wg, wu, wd = experts[e]
            expert_apply(h_bits, toks, g, wg, wu, wd, y, n_threads)
    sg = [1.0] * T if shared_gates is None else [float(x) for x in shared_gates]
    for wg, wu, wd in shared:
        expert_apply(h_bits, list(range(T)), sg, wg, wu, wd, y, n_threads)
    return y


# --------------------------------------------------------------------------
# The compiled reference (oracle/_ref)
# --------------------------------------------------------------------------
class RefSimConfig(C.Structure):
    """Same field layout as moespac_sched_config (include/moespac/moespac.h)."""
    _fields_ = [
        ("n_layers", C.c_int32), ("n_experts", C.c_int32), ("top_k", C.c_int32), ("gamma", C.c_int32),
        ("alpha", C.c_double), ("drift_scale", C.c_double), ("route_noise", C.c_double),
        ("shift_period", C.c_int32), ("_pad0", C.c_int32), ("seed", C.c_uint64),
        ("t_cpu_unit_ns", C.c_int64), ("t_gpu_unit_ns", C.c_int64), ("t_io_unit_ns", C.c_int64),
        ("t_draft_unit_ns", C.c_int64), ("expert_bytes", C.c_int64),
        ("utility_cap", C.c_int32), ("adaptive_boundaries", C.c_int32), ("forgetting", C.c_double),
        ("init_up", C.c_int32), ("init_down", C.c_int32),
        ("policy", C.c_int32), ("fixed_tau", C.c_int32), ("fixed_up", C.c_int32), ("fixed_down", C.c_int32),
        ("cache_ratio", C.c_double), ("token_budget", C.c_int64),
        ("max_steps", C.c_int32), ("warmup_steps", C.c_int32), ("ratio_smoothing", C.c_double),
    ]


POLICIES = ["moe_spac", "on_demand_gpu", "lru_cache", "static_split", "ar_mode",
            "fixed_tau", "fixed_boundaries", "binary_utility"]


def default_config(**kw) -> RefSimConfig:
    """default_sim_config() (proj/core/src/config.cpp:11-39) with overrides."""
    c = RefSimConfig()
    c.n_layers, c.n_experts, c.top_k, c.gamma = 48, 128, 8, 8
    c.alpha, c.drift_scale, c.route_noise = 0.8, 0.02, 0.2
    c.shift_period, c.seed = 0, 1
    c.t_cpu_unit_ns, c.t_gpu_unit_ns, c.t_io_unit_ns, c.t_draft_unit_ns = 100_000, 40_000, 400_000, 300_000
    c.expert_bytes = 25_000_000
    c.utility_cap, c.adaptive_boundaries, c.forgetting = 4, 1, 0.1
    c.init_up, c.init_down = -1, -1
    c.policy, c.fixed_tau, c.fixed_up, c.fixed_down = 0, 2, 3, 1
    c.cache_ratio, c.token_budget, c.max_steps, c.warmup_steps = 0.17, 512, 0, 32
    c.ratio_smoothing = 0.3
    for key, v in kw.items():
        if key == "policy" and isinstance(v, str):
            v = POLICIES.index(v)
        setattr(c, key, v)
    return c


def ref() -> C.CDLL:
    global _ref
    if _ref is None:
        if not os.path.exists(_REF_PATH):
            raise FileNotFoundError(f"{_REF_PATH} not built (needs /root/reference; run make -C oracle)")
        lib = C.CDLL(_REF_PATH)
        P = C.POINTER(RefSimConfig)
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_trace_generate.argtypes = [P, C.c_int, _i32p, _i32p]
        lib.ref_trace_time_ns.restype = C.c_double
        lib.ref_trace_time_ns.argtypes = [P, C.c_int]
        lib.ref_sim_run.argtypes = [P, _i32p, _i32p, C.c_int, _i64p, _i64p, _f64p, _i64p, C.c_int64,
                                    _i64p, _i64p]
        lib.ref_sim_time_ns.restype = C.c_double
        lib.ref_sim_time_ns.argtypes = [P, _i32p, _i32p, C.c_int]
        lib.ref_estimator_run.argtypes = [C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, C.c_int,
                                          C.c_int, _i32p, _i32p, C.c_int]
        lib.ref_estimator_init.argtypes = [C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, C.c_int,
                                           C.c_int, _i32p]
        lib.ref_solve_threshold.argtypes = [_i32p, C.c_int, _u8p, C.c_int, C.c_int, C.c_int, _f64p, _f64p,
                                            C.c_int] + [C.c_int64] * 6 + [_i64p]
        lib.ref_update_ratio_estimates.argtypes = [_f64p, _f64p, C.c_int, C.c_int, C.c_double, C.c_double,
                                                   C.c_double]
        lib.ref_layer_capacity_experts.argtypes = [C.c_double, C.c_int]
        vp = C.c_void_p
        lib.ref_write_trace.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, vp, vp]
        lib.ref_read_trace.argtypes = [C.c_char_p, vp, vp, vp, vp, C.c_int64]
        lib.ref_summarize.argtypes = [vp, vp, C.c_int, vp, vp, vp]
        lib.ref_emit.argtypes = [vp, vp, vp, vp, vp, C.c_int, C.c_int, C.c_char_p]
        lib.ref_parse.argtypes = [C.c_char_p, vp, vp, vp, vp, vp, C.c_int, C.c_int64, vp]
        _ref = lib
    return _ref


def _check(rc):
    if rc < 0:
        raise RuntimeError(ref().ref_last_error().decode())
    return rc


def ref_trace(cfg: RefSimConfig, n_steps: int):
    T = cfg.gamma + 1
    ids = np.empty((n_steps, cfg.n_layers, T, cfg.top_k), np.int32)
    acc = np.empty(n_steps, np.int32)
    _check(ref().ref_trace_generate(C.byref(cfg), n_steps, ids.reshape(-1), acc))
    return ids, acc


@dataclass
class RefRun:
    layer_rec: np.ndarray  # [S][L][10]
    step_rec: np.ndarray   # [S][8]
    accuracy: np.ndarray   # [S]
    events: np.ndarray     # [E][6] kind, step, layer, expert, start, dur
    total_time_ns: int
    steps: int = field(default=0)


EV_DRAFT, EV_CPU, EV_GPU, EV_STALL, EV_LOAD, EV_EVICT = range(6)


def ref_sim_run(cfg: RefSimConfig, ids: np.ndarray, accepted: np.ndarray) -> RefRun:
    S = len(accepted)
    L = cfg.n_layers
    # AR mode runs one simulated step per accepted token (sim_core.cpp:306-313)
    R = int(np.sum(accepted)) if cfg.policy == POLICIES.index("ar_mode") else S
    lr = np.zeros((R, L, 10), np.int64)
    sr = np.zeros((R, 8), np.int64)
    acc = np.zeros(R, np.float64)
    cap = R * (1 + L * (4 + 2 * cfg.n_experts))
    ev = np.zeros((cap, 6), np.int64)
    nev = np.zeros(1, np.int64)
    tot = np.zeros(1, np.int64)
    steps = _check(ref().ref_sim_run(C.byref(cfg), np.ascontiguousarray(ids, np.int32).reshape(-1),
                                     np.ascontiguousarray(accepted, np.int32), S, lr.reshape(-1),
                                     sr.reshape(-1), acc, ev.reshape(-1), cap, nev, tot))
    n = int(nev[0])
    assert n <= cap
    return RefRun(lr[:steps], sr[:steps], acc[:steps], ev[:n], int(tot[0]), steps)


def ref_estimator_run(state, freqs_seq, cap, lam, gamma, adaptive=True, init_up=-1, init_down=-1):
    st = np.ascontiguousarray(state, np.int32).copy()
    fs = np.ascontiguousarray(freqs_seq, np.int32)
    _check(ref().ref_estimator_run(st.shape[0], cap, lam, gamma, int(adaptive), init_up, init_down,
                                   st.reshape(-1), fs.reshape(-1), fs.shape[0]))
    return st


def ref_solve_threshold(scores, resident, gamma, top_k, b_est, rc, rg, t_cpu, t_gpu, t_io,
                        expert_bytes, vram_left, draft_credit):
    out = np.zeros(6, np.int64)
    cap = len(rc)
    _check(ref().ref_solve_threshold(np.ascontiguousarray(scores, np.int32), len(scores),
                                     np.ascontiguousarray(resident, np.uint8), gamma, top_k, b_est,
                                     np.ascontiguousarray(rc, np.float64), np.ascontiguousarray(rg, np.float64),
                                     cap, t_cpu, t_gpu, t_io, expert_bytes, vram_left, draft_credit, out))
    return out


# ---------------------------------------------------------------- reference trace I/O and metrics
# status: 0 ok, -1 runtime_error, -2 invalid_argument, -3 out_of_range, -4 other
REF_ERR = {-1: "runtime_error", -2: "invalid_argument", -3: "out_of_range", -4: "other"}


def ref_write_trace(path, ids, accepted, n_experts):
    ids = np.ascontiguousarray(ids, dtype=np.int32)
    acc = np.ascontiguousarray(accepted, dtype=np.int32)
    S, L, T, k = ids.shape
    rc = ref().ref_write_trace(path.encode(), L, n_experts, k, T - 1, S, ids.ctypes.data, acc.ctypes.data)
    return rc, ref().ref_last_error().decode() if rc else ""


def ref_read_trace(path):
    """-> (rc, message, shape dict, ids, accepted)"""
    shape = np.zeros(4, dtype=np.int32)
    n = np.zeros(1, dtype=np.int64)
    rc = ref().ref_read_trace(path.encode(), shape.ctypes.data, n.ctypes.data, None, None, 0)
    if rc:
        return rc, ref().ref_last_error().decode(), None, None, None
    L, N, k, g = (int(x) for x in shape)
    S = int(n[0])
    ids = np.zeros((S, L, g + 1, k), dtype=np.int32) if S else np.zeros((0, max(L, 0), max(g + 1, 0), max(k, 0)),
                                                                          dtype=np.int32)
    acc = np.zeros(S, dtype=np.int32)
    if S:
        rc = ref().ref_read_trace(path.encode(), shape.ctypes.data, n.ctypes.data, ids.ctypes.data, acc.ctypes.data, S)
    return rc, "", {"n_layers": L, "n_experts": N, "top_k": k, "gamma": g}, ids, acc


# flattened StepReport / LayerTiming of the shim (sim_core.hpp:38-61)
REF_STEP = np.dtype([("draft_ns", "<i8"), ("cache_hits", "<i8"), ("cache_misses", "<i8"), ("faults_fn", "<i8"),
                     ("faults_fp", "<i8"), ("step_wall_ns", "<i8"), ("accuracy", "<f8"), ("accepted_tokens", "<i4"),
                     ("n_experts", "<i4"), ("n_layers", "<i4"), ("_pad", "<i4")])
REF_LAYER = np.dtype([("t_cpu_ns", "<i8"), ("t_gpu_ns", "<i8"), ("t_io_used_ns", "<i8"), ("stall_ns", "<i8"),
                      ("bubble_ns", "<i8"), ("wall_ns", "<i8"), ("tau", "<i4"), ("fallback", "<i4"),
                      ("n_prefetch", "<i4"), ("_pad", "<i4")])
SUMMARY_KEYS = ["axis_value", "tps", "latency_s", "hit_rate", "bubble_ratio", "fault_rate", "fn_rate", "fp_rate",
                "mean_accuracy"]


def ref_summarize(steps, layers):
    """steps: REF_STEP array [n]; layers: REF_LAYER array [sum n_layers] -> (rc, msg, dict)"""
    steps = np.ascontiguousarray(steps)
    layers = np.ascontiguousarray(layers)
    vals = np.zeros(10)
    ints = np.zeros(2, dtype=np.int64)
    series = np.zeros(max(1, len(steps)))
    rc = ref().ref_summarize(steps.ctypes.data, layers.ctypes.data, len(steps), vals.ctypes.data, ints.ctypes.data,
                             series.ctypes.data)
    if rc:
        return rc, ref().ref_last_error().decode(), None
    d = dict(zip(SUMMARY_KEYS, vals[:9].tolist()))
    d.update(total_tokens=int(ints[0]), total_time_ns=int(ints[1]), accuracy_series=series[:len(steps)].tolist())
    return 0, "", d


def ref_emit(path, summaries, fmt):
    """summaries: list of dicts (SUMMARY_KEYS + axis, total_tokens, total_time_ns, accuracy_series)."""
    n = len(summaries)
    vals = np.zeros((max(1, n), 10))
    ints = np.zeros((max(1, n), 2), dtype=np.int64)
    axis = np.zeros((max(1, n), 64), dtype=np.uint8)
    nser = np.zeros(max(1, n), dtype=np.int64)
    for i, s in enumerate(summaries):
        vals[i, :9] = [s[k] for k in SUMMARY_KEYS]
        ints[i] = [s["total_tokens"], s["total_time_ns"]]
        b = s["axis"].encode()[:63]
        axis[i, :len(b)] = np.frombuffer(b, dtype=np.uint8)
        nser[i] = len(s["accuracy_series"])
    flat = np.ascontiguousarray(np.concatenate([np.asarray(s["accuracy_series"], dtype=np.float64)
                                                for s in summaries]) if n else np.zeros(1))
    rc = ref().ref_emit(vals.ctypes.data, ints.ctypes.data, axis.ctypes.data, flat.ctypes.data, nser.ctypes.data, n,
                        0 if fmt == "csv" else 1, path.encode())
    return rc, ref().ref_last_error().decode() if rc else ""


def ref_parse(path, cap=64, series_cap=1 << 16):
    vals = np.zeros((cap, 10))
    ints = np.zeros((cap, 2), dtype=np.int64)
    axis = np.zeros((cap, 64), dtype=np.uint8)
    series = np.zeros(series_cap)
    nser = np.zeros(cap, dtype=np.int64)
    n = np.zeros(1, dtype=np.int32)
    rc = ref().ref_parse(path.encode(), vals.ctypes.data, ints.ctypes.data, axis.ctypes.data, series.ctypes.data,
                         nser.ctypes.data, cap, series_cap, n.ctypes.data)
    if rc:
        return rc, ref().ref_last_error().decode(), None
    out, pos = [], 0
    for i in range(int(n[0])):
        d = dict(zip(SUMMARY_KEYS, vals[i, :9].tolist()))
        d.update(axis=bytes(axis[i]).split(b"\0")[0].decode(), total_tokens=int(ints[i, 0]),
                 total_time_ns=int(ints[i, 1]), accuracy_series=series[pos:pos + nser[i]].tolist())
        pos += int(nser[i])
        out.append(d)
    return 0, "", out
