"""ctypes binding of libmoespac.so (include/moespac/moespac.h).

This is the Python face of the C ABI that the reference-side integration
would bind. It adds no logic: every call goes straight
to the native library, and device calls take torch CUDA tensors only as
memory owners (their data_ptr). There is no CPU fallback — if the library or
an sm_100 device is missing, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
import re

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
_ROOT = os.path.dirname(_PKG)
LIB_PATH = os.environ.get("MOESPAC_LIB") or os.path.join(_PKG, "_lib", "libmoespac.so")  # override: A/B builds
HEADER = os.path.join(_ROOT, "include", "moespac", "moespac.h")

STATUS = {0: "OK", 1: "E_INVALID", 2: "E_RANGE", 3: "E_LOGIC", 4: "E_IO", 5: "E_CUDA", 6: "E_NCCL", 7: "E_NOMEM"}


class MoespacError(RuntimeError):
    def __init__(self, status: int, msg: str):
        self.status = status
        self.code = STATUS.get(status, str(status))
        super().__init__(f"moespac {self.code}: {msg}")


class SchedConfig(C.Structure):
    """moespac_sched_config (mirrors moesim::SimConfig)."""
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


class LayerTiming(C.Structure):
    _fields_ = [("t_cpu_ns", C.c_int64), ("t_gpu_ns", C.c_int64), ("t_io_used_ns", C.c_int64),
                ("stall_ns", C.c_int64), ("bubble_ns", C.c_int64), ("wall_ns", C.c_int64),
                ("tau", C.c_int32), ("fallback", C.c_int32), ("n_prefetch", C.c_int32), ("n_loads", C.c_int32)]


class StepReport(C.Structure):
    _fields_ = [("draft_ns", C.c_int64), ("cache_hits", C.c_int64), ("cache_misses", C.c_int64),
                ("faults_fn", C.c_int64), ("faults_fp", C.c_int64), ("step_wall_ns", C.c_int64),
                ("accuracy", C.c_double), ("accepted_tokens", C.c_int32), ("n_experts", C.c_int32),
                ("n_layers", C.c_int32), ("n_loads", C.c_int32),
                ("gpu_ms_total", C.c_float), ("gpu_ms_router", C.c_float), ("gpu_ms_hist", C.c_float),
                ("gpu_ms_ffn", C.c_float), ("gpu_ms_combine", C.c_float), ("gpu_ms_h2d_loads", C.c_float),
                ("ffn_bytes", C.c_int64), ("h2d_bytes", C.c_int64), ("d2h_bytes", C.c_int64),
                ("kernel_launches", C.c_int32), ("cold_experts", C.c_int32), ("cpu_ms_cold", C.c_float),
                ("ffn_launches", C.c_int32), ("gpu_ms_draft", C.c_float), ("draft_bytes", C.c_int64),
                ("staged_experts", C.c_int32)]


class LayerOutcome(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("distinct", "distinct_hits", "hit_tokens", "miss_tokens", "agree",
                                         "faults_fn", "faults_fp", "n_local_hits")]


class K2Args(C.Structure):
    _fields_ = [("ids_dev", C.c_void_p), ("n_layers", C.c_int32), ("tokens", C.c_int32), ("top_k", C.c_int32),
                ("n_experts", C.c_int32), ("resident_bits_dev", C.c_void_p), ("loaded_bits_dev", C.c_void_p),
                ("taus_dev", C.c_void_p), ("est_state_dev", C.c_void_p), ("utility_cap", C.c_int32),
                ("adaptive_boundaries", C.c_int32), ("forgetting", C.c_double), ("shard_rank", C.c_int32),
                ("shard_world", C.c_int32), ("freqs_dev", C.c_void_p), ("offsets_dev", C.c_void_p),
                ("perm_dev", C.c_void_p), ("hit_list_dev", C.c_void_p), ("hit_ord_dev", C.c_void_p),
                ("counters_dev", C.c_void_p), ("scores_out_dev", C.c_void_p)]


class FfnArgs(C.Structure):
    _fields_ = [("h_dev", C.c_void_p), ("tokens", C.c_int32), ("d_model", C.c_int32), ("d_ffn", C.c_int32),
                ("top_k", C.c_int32), ("n_experts", C.c_int32), ("perm_dev", C.c_void_p),
                ("offsets_dev", C.c_void_p), ("gates_dev", C.c_void_p), ("hit_list_dev", C.c_void_p),
                ("counters_dev", C.c_void_p), ("slot_of_dev", C.c_void_p), ("pool_dev", C.c_void_p),
                ("shared_dev", C.c_void_p), ("n_shared_units", C.c_int32), ("workspace_dev", C.c_void_p),
                ("grid", C.c_int32), ("kernel", C.c_int32), ("hT_dev", C.c_void_p), ("debug_ts_dev", C.c_void_p),
                ("accum", C.c_int32), ("l2_policy", C.c_int32)]


class CombineArgs(C.Structure):
    _fields_ = [("h_in_dev", C.c_void_p), ("y_extra_dev", C.c_void_p), ("tokens", C.c_int32),
                ("d_model", C.c_int32), ("d_ffn", C.c_int32), ("top_k", C.c_int32), ("ids_dev", C.c_void_p),
                ("hit_ord_dev", C.c_void_p), ("counters_dev", C.c_void_p), ("n_shared_units", C.c_int32),
                ("grid", C.c_int32), ("workspace_dev", C.c_void_p), ("y_dev", C.c_void_p),
                ("h_out_dev", C.c_void_p), ("accum", C.c_int32), ("kernel", C.c_int32)]


class RunSummary(C.Structure):
    """moespac_run_summary — the reference's RunSummary (metrics_report.hpp:15-30)."""
    _fields_ = [("axis_name", C.c_char * 64)] + [(n, C.c_double) for n in (
        "axis_value", "tps", "latency_s", "hit_rate", "bubble_ratio", "fault_rate", "fn_rate", "fp_rate",
        "mean_accuracy")] + [("total_tokens", C.c_int64), ("total_time_ns", C.c_int64), ("n_series", C.c_int64)]

    def as_dict(self, series=None) -> dict:
        d = {k: getattr(self, k) for k, _ in self._fields_ if k not in ("axis_name", "n_series")}
        d["axis"] = self.axis_name.decode()
        if series is not None:
            d["accuracy_series"] = list(series)
        return d


class ModelDesc(C.Structure):
    _fields_ = [("n_layers", C.c_int32), ("n_experts", C.c_int32), ("top_k", C.c_int32), ("gamma", C.c_int32),
                ("d_model", C.c_int32), ("d_ffn", C.c_int32), ("n_shared_units", C.c_int32),
                ("gate_mode", C.c_int32), ("ffn_kernel", C.c_int32), ("parallel_mode", C.c_int32),
                ("shared_gate", C.c_int32)]


class CtxViews(C.Structure):
    _fields_ = [("ids_dev", C.c_void_p), ("gates_dev", C.c_void_p), ("freqs_dev", C.c_void_p),
                ("offsets_dev", C.c_void_p), ("perm_dev", C.c_void_p), ("counters_dev", C.c_void_p),
                ("est_state_dev", C.c_void_p), ("h_dev", C.c_void_p), ("y_dev", C.c_void_p),
                ("pool_dev", C.c_void_p), ("logits_dev", C.c_void_p), ("slots_per_layer", C.c_int64),
                ("image_elems", C.c_int64), ("shared_dev", C.c_void_p), ("shared_gate_dev", C.c_void_p)]


POLICIES = ["moe_spac", "on_demand_gpu", "lru_cache", "static_split", "ar_mode",
            "fixed_tau", "fixed_boundaries", "binary_utility"]

_lib = None


def lib() -> C.CDLL:
    """Load libmoespac.so (fails loudly if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing — run paper_2603_09983_b200/build.py (or __graft_entry__.build())")
    L = C.CDLL(LIB_PATH)
    vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
    sig = {
        "moespac_last_error": (C.c_char_p, []),
        "moespac_abi_version": (C.c_int, []),
        "moespac_default_sched_config": (None, [C.POINTER(SchedConfig)]),
        "moespac_sched_create": (C.c_int, [C.POINTER(SchedConfig), C.c_int, C.POINTER(vp)]),
        "moespac_sched_destroy": (None, [vp]),
        "moespac_sched_decide": (C.c_int, [vp, vp]),
        "moespac_sched_tables": (C.c_int, [vp, vp, vp, vp, vp]),
        "moespac_sched_decisions": (C.c_int, [vp, vp]),
        "moespac_sched_loads": (i64, [vp, vp, i64]),
        "moespac_sched_observe": (C.c_int, [vp, vp, C.c_int, vp, vp]),
        "moespac_sched_observe_freqs": (C.c_int, [vp, vp, C.c_int, vp, vp]),
        "moespac_sched_events": (i64, [vp, vp, i64]),
        "moespac_sched_total_time_ns": (i64, [vp]),
        "moespac_sched_ratios": (C.c_int, [vp, C.c_int, vp, vp, vp]),
        "moespac_solve_threshold": (C.c_int, [vp, C.c_int, vp, C.c_int, C.c_int, C.c_int, vp, vp, C.c_int,
                                              i64, i64, i64, i64, i64, i64, vp]),
        "moespac_update_ratio_estimates": (C.c_int, [vp, vp, C.c_int, C.c_int, C.c_double, C.c_double,
                                                     C.c_double]),
        "moespac_layer_capacity_experts": (C.c_int, [C.c_double, C.c_int]),
        "moespac_router_topk": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, C.c_int, vp, vp, vp]),
        "moespac_hist_scan_observe": (C.c_int, [C.POINTER(K2Args), vp]),
        "moespac_estimator_init": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, C.c_int, vp]),
        "moespac_ffn_workspace_bytes": (C.c_size_t, [C.c_int] * 5),
        "moespac_expert_image_elems": (i64, [C.c_int, C.c_int]),
        "moespac_expert_ffn": (C.c_int, [C.POINTER(FfnArgs), vp]),
        "moespac_ffn_combine": (C.c_int, [C.POINTER(CombineArgs), vp]),
        "moespac_pack_expert": (C.c_int, [vp, vp, vp, C.c_int, C.c_int, C.c_int, vp, vp]),
        "moespac_ffn_resolve": (C.c_int, [C.c_int, C.c_int, C.c_int]),
        "moespac_build_hT": (C.c_int, [vp, C.c_int, C.c_int, vp, vp]),
        "moespac_fill_synthetic": (C.c_int, [vp, i64, C.c_uint64, C.c_float, vp]),
        "moespac_unpack_expert": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, vp, vp, vp, vp]),
        "moespac_ctx_set_shared_gate": (C.c_int, [vp, C.c_int, vp]),
        "moespac_ctx_estimator_dump": (C.c_int, [vp, C.c_char_p]),
        "moespac_ctx_estimator_load": (C.c_int, [vp, C.c_char_p]),
        "moespac_ctx_create": (C.c_int, [C.c_int, C.POINTER(ModelDesc), C.POINTER(SchedConfig), C.c_int, C.c_int,
                                         C.POINTER(vp)]),
        "moespac_ctx_destroy": (None, [vp]),
        "moespac_ctx_host_arena": (C.c_int, [vp, i64, C.POINTER(vp)]),
        "moespac_ctx_fill_synthetic": (C.c_int, [vp, C.c_uint64, C.c_float]),
        "moespac_ctx_set_shared": (C.c_int, [vp, C.c_int, vp]),
        "moespac_ctx_finalize": (C.c_int, [vp]),
        "moespac_nccl_unique_id": (C.c_int, [vp]),
        "moespac_ctx_set_nccl": (C.c_int, [vp, vp, C.c_int, C.c_int]),
        "moespac_ctx_set_timing": (C.c_int, [vp, C.c_int]),
        "moespac_ctx_set_pdl": (C.c_int, [vp, C.c_int]),
        "moespac_ctx_set_graph": (C.c_int, [vp, C.c_int]),
        "moespac_ctx_set_draft_window": (C.c_int, [vp, C.c_int]),
        "moespac_ctx_set_draft_model": (C.c_int, [vp, i64, C.c_int]),
        "moespac_ctx_set_timeline": (C.c_int, [vp, C.c_int]),
        "moespac_draft_gemv": (C.c_int, [vp, i64, C.c_int, vp, vp, C.c_float, vp, vp]),
        "moespac_ctx_timeline_events": (i64, [vp, vp, i64]),
        "moespac_ctx_timeline_layers": (i64, [vp, vp, i64]),
        "moespac_ctx_timeline_steps": (i64, [vp, vp, i64]),
        "moespac_ctx_set_k3_trace": (C.c_int, [vp, vp]),
        "moespac_ctx_set_l2_prefetch": (C.c_int, [vp, C.c_int]),
        "moespac_ctx_set_cold_threads": (C.c_int, [vp, C.c_int]),
        "moespac_ctx_set_cold_staging": (C.c_int, [vp, C.c_int, C.c_double]),
        "moespac_step": (C.c_int, [vp, vp, vp, C.c_int, vp, vp, vp]),
        "moespac_step_device": (C.c_int, [vp, vp, vp, C.c_int, vp, vp, vp]),
        "moespac_ctx_get_views": (C.c_int, [vp, C.POINTER(CtxViews)]),
        "moespac_ctx_sched": (vp, [vp]),
        "moespac_ctx_stream": (vp, [vp]),
        "moespac_ctx_k3_variant": (C.c_int, [vp]),
        "moespac_ctx_parallel_mode": (C.c_int, [vp]),
        "moespac_ctx_step_tables": (C.c_int, [vp, vp, vp, vp, vp]),
        "moespac_trace_synth_create": (C.c_int, [C.POINTER(SchedConfig), C.POINTER(vp)]),
        "moespac_trace_generate": (C.c_int, [C.POINTER(SchedConfig), i64, vp, vp]),
        "moespac_trace_synth_next": (C.c_int, [vp, vp, vp]),
        "moespac_trace_synth_destroy": (None, [vp]),
        "moespac_trace_write": (C.c_int, [C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_int, i64, vp, vp]),
        "moespac_trace_read": (C.c_int, [C.c_char_p, vp, C.POINTER(i64), vp, vp, i64]),
        "moespac_summarize": (C.c_int, [vp, vp, i64, C.c_int, C.POINTER(RunSummary), vp]),
        "moespac_metrics_emit": (C.c_int, [vp, vp, i64, C.c_int, C.c_char_p]),
        "moespac_metrics_parse": (C.c_int, [C.c_char_p, vp, i64, vp, i64, C.POINTER(i64)]),
        "moespac_step_ids": (C.c_int, [vp, vp, vp, vp, C.c_int, vp, vp, vp]),
        "moespac_ctx_set_router": (C.c_int, [vp, C.c_int, vp]),
        "moespac_step_model": (C.c_int, [vp, vp, C.c_int, vp, vp, vp]),
        "moespac_step_model_device": (C.c_int, [vp, vp, C.c_int, vp, vp, vp]),
        "moespac_loopback_create": (C.c_int, [C.c_int, C.c_int, i64, C.POINTER(vp)]),
        "moespac_loopback_destroy": (None, [vp]),
        "moespac_ctx_set_loopback": (C.c_int, [vp, vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def header_functions() -> list[str]:
    """Every function the public header declares."""
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(moespac_[A-Za-z0-9_]+)\s*\(", txt)))


def check(status: int) -> None:
    if status != 0:
        raise MoespacError(status, lib().moespac_last_error().decode())


def ptr(x) -> int | None:
    """Address of a torch tensor / numpy array (None passes NULL)."""
    if x is None:
        return None
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    return x.ctypes.data


def default_config(**kw) -> SchedConfig:
    c = SchedConfig()
    lib().moespac_default_sched_config(C.byref(c))
    for k, v in kw.items():
        if k == "policy" and isinstance(v, str):
            v = POLICIES.index(v)
        setattr(c, k, v)
    return c


# ---------------------------------------------------------------- scheduler
class Scheduler:
    """Host scheduler (HWB + AEE bookkeeping): the decision half of run_utility_step."""

    def __init__(self, cfg: SchedConfig, shard_world: int = 1):
        self.cfg = cfg
        self.L, self.N = cfg.n_layers, cfg.n_experts
        self.W = (self.N + 31) // 32
        h = C.c_void_p()
        check(lib().moespac_sched_create(C.byref(cfg), shard_world, C.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            lib().moespac_sched_destroy(self._h)
            self._h = None

    __del__ = close

    def decide(self, scores: np.ndarray) -> None:
        s = np.ascontiguousarray(scores, np.int32)
        assert s.size == self.L * self.N
        check(lib().moespac_sched_decide(self._h, s.ctypes.data))

    def tables(self):
        taus = np.zeros(self.L, np.int32)
        rb = np.zeros((self.L, self.W), np.uint32)
        lb = np.zeros((self.L, self.W), np.uint32)
        slots = np.zeros((self.L, self.N), np.int32)
        check(lib().moespac_sched_tables(self._h, taus.ctypes.data, rb.ctypes.data, lb.ctypes.data,
                                         slots.ctypes.data))
        return taus, rb, lb, slots

    def decisions(self) -> np.ndarray:
        out = np.zeros((self.L, 5), np.int64)
        check(lib().moespac_sched_decisions(self._h, out.ctypes.data))
        return out

    def loads(self) -> np.ndarray:
        n = lib().moespac_sched_loads(self._h, None, 0)
        out = np.zeros((max(n, 1), 4), np.int32)
        lib().moespac_sched_loads(self._h, out.ctypes.data, n)
        return out[:n]

    def observe_freqs(self, freqs: np.ndarray, accepted: int):
        f = np.ascontiguousarray(freqs, np.int32)
        rep = StepReport()
        lay = (LayerTiming * self.L)()
        check(lib().moespac_sched_observe_freqs(self._h, f.ctypes.data, accepted, C.byref(rep), lay))
        return rep, list(lay)

    def observe(self, outcomes: np.ndarray, accepted: int):
        o = np.ascontiguousarray(outcomes, np.int32)
        assert o.shape == (self.L, 8)
        rep = StepReport()
        lay = (LayerTiming * self.L)()
        check(lib().moespac_sched_observe(self._h, o.ctypes.data, accepted, C.byref(rep), lay))
        return rep, list(lay)

    def events(self) -> np.ndarray:
        n = lib().moespac_sched_events(self._h, None, 0)
        out = np.zeros((max(n, 1), 6), np.int64)
        lib().moespac_sched_events(self._h, out.ctypes.data, n)
        return out[:n]

    def total_time_ns(self) -> int:
        return lib().moespac_sched_total_time_ns(self._h)

    def ratios(self, layer: int):
        K = self.cfg.utility_cap if self.cfg.policy != POLICIES.index("binary_utility") else 1
        rc = np.zeros(K, np.float64)
        rg = np.zeros(K, np.float64)
        b = C.c_int32()
        check(lib().moespac_sched_ratios(self._h, layer, rc.ctypes.data, rg.ctypes.data, C.byref(b)))
        return rc, rg, b.value


def solve_threshold(scores, resident, gamma, top_k, b_est, rc, rg, t_cpu, t_gpu, t_io, expert_bytes, vram_left,
                    draft_credit) -> np.ndarray:
    out = np.zeros(6, np.int64)
    s = np.ascontiguousarray(scores, np.int32)
    r = np.ascontiguousarray(resident, np.uint8)
    rc = np.ascontiguousarray(rc, np.float64)
    rg = np.ascontiguousarray(rg, np.float64)
    check(lib().moespac_solve_threshold(s.ctypes.data, len(s), r.ctypes.data, gamma, top_k, b_est, rc.ctypes.data,
                                        rg.ctypes.data, len(rc), t_cpu, t_gpu, t_io, expert_bytes, vram_left,
                                        draft_credit, out.ctypes.data))
    return out


def trace_generate(cfg: SchedConfig, n_steps: int):
    """Host TraceGenerator (incl. top-k): ids [S][L][gamma+1][k], accepted [S]."""
    ids = np.zeros((n_steps, cfg.n_layers, cfg.gamma + 1, cfg.top_k), np.int32)
    acc = np.zeros(n_steps, np.int32)
    check(lib().moespac_trace_generate(C.byref(cfg), n_steps, ids.ctypes.data, acc.ctypes.data))
    return ids, acc


class TraceSynth:
    """Host half of TraceGenerator::next_step: noisy fp64 logits for K1."""

    def __init__(self, cfg: SchedConfig):
        self.L, self.N, self.T = cfg.n_layers, cfg.n_experts, cfg.gamma + 1
        h = C.c_void_p()
        check(lib().moespac_trace_synth_create(C.byref(cfg), C.byref(h)))
        self._h = h

    def next(self, out: np.ndarray | None = None):
        if out is None:
            out = np.empty((self.L, self.T, self.N), np.float64)
        acc = C.c_int32()
        check(lib().moespac_trace_synth_next(self._h, out.ctypes.data, C.byref(acc)))
        return out, acc.value

    def close(self):
        if getattr(self, "_h", None):
            lib().moespac_trace_synth_destroy(self._h)
            self._h = None

    __del__ = close


# ---------------------------------------------------------------- device kernels
# ---------------------------------------------------------------- routing traces (#moetrace v1)
def trace_write(path: str, ids: np.ndarray, accepted: np.ndarray, n_experts: int) -> None:
    """ids [S][L][gamma+1][k] int32, accepted [S] — the reference's write_trace."""
    ids = np.ascontiguousarray(ids, dtype=np.int32)
    acc = np.ascontiguousarray(accepted, dtype=np.int32)
    S, L, T, k = ids.shape
    check(lib().moespac_trace_write(path.encode(), L, n_experts, k, T - 1, S, ids.ctypes.data, acc.ctypes.data))


def trace_read(path: str):
    """-> (shape dict, ids [S][L][gamma+1][k], accepted [S]) — the reference's read_trace."""
    shape = np.zeros(4, dtype=np.int32)
    n = C.c_int64(0)
    check(lib().moespac_trace_read(path.encode(), shape.ctypes.data, C.byref(n), None, None, 0))
    L, N, k, g = (int(x) for x in shape)
    ids = np.zeros((n.value, L, g + 1, k) if n.value else (0, max(L, 0), max(g + 1, 0), max(k, 0)), dtype=np.int32)
    acc = np.zeros(n.value, dtype=np.int32)
    if n.value:
        check(lib().moespac_trace_read(path.encode(), shape.ctypes.data, C.byref(n), ids.ctypes.data,
                                       acc.ctypes.data, n.value))
    return {"n_layers": L, "n_experts": N, "top_k": k, "gamma": g}, ids, acc


# ---------------------------------------------------------------- run metrics (#moesim-metrics v1)
def summarize(reports, layers=None, measured: bool = False):
    """reports: sequence of StepReport, layers: [n][L] LayerTiming (or None).
    -> (RunSummary, accuracy series)"""
    n = len(reports)
    reps = (StepReport * max(1, n))(*reports)
    lay = None
    if layers is not None:
        flat = [x for row in layers for x in row]
        lay = (LayerTiming * max(1, len(flat)))(*flat)
    out = RunSummary()
    series = np.zeros(max(1, n), dtype=np.float64)
    check(lib().moespac_summarize(C.addressof(reps), C.addressof(lay) if lay is not None else None, n,
                                  int(measured), C.byref(out), series.ctypes.data))
    return out, series[:n]


def metrics_emit(path: str, summaries, series_list, fmt: str = "csv") -> None:
    arr = (RunSummary * max(1, len(summaries)))(*summaries)
    flat = np.ascontiguousarray(np.concatenate([np.asarray(s, dtype=np.float64) for s in series_list])
                                if series_list else np.zeros(0), dtype=np.float64)
    check(lib().moespac_metrics_emit(C.addressof(arr), flat.ctypes.data if flat.size else None, len(summaries),
                                     0 if fmt == "csv" else 1, path.encode()))


def metrics_parse(path: str):
    """-> list of (RunSummary, series)"""
    n = C.c_int64(0)
    check(lib().moespac_metrics_parse(path.encode(), None, 0, None, 0, C.byref(n)))
    arr = (RunSummary * max(1, n.value))()
    check(lib().moespac_metrics_parse(path.encode(), C.addressof(arr), n.value, None, 0, C.byref(n)))
    total = sum(arr[i].n_series for i in range(n.value))
    flat = np.zeros(max(1, total), dtype=np.float64)
    check(lib().moespac_metrics_parse(path.encode(), C.addressof(arr), n.value, flat.ctypes.data, total, C.byref(n)))
    out, pos = [], 0
    for i in range(n.value):
        ns = arr[i].n_series
        out.append((arr[i], flat[pos:pos + ns].copy()))
        pos += ns
    return out


def _stream(stream):
    if stream is None:
        import torch
        return C.c_void_p(torch.cuda.current_stream().cuda_stream)
    return C.c_void_p(stream)


def router_topk(logits, k: int, gate_mode: int = 0, stream=None):
    """K1 on a CUDA fp64 tensor [..., N] -> (ids int32 [..., k], gates fp32 [..., k])."""
    import torch
    assert logits.is_cuda and logits.dtype == torch.float64 and logits.is_contiguous()
    N = logits.shape[-1]
    rows = logits.numel() // N
    ids = torch.empty(logits.shape[:-1] + (k,), dtype=torch.int32, device=logits.device)
    gates = torch.empty(logits.shape[:-1] + (k,), dtype=torch.float32, device=logits.device)
    check(lib().moespac_router_topk(ptr(logits), rows, N, k, gate_mode, ptr(ids), ptr(gates), _stream(stream)))
    return ids, gates


def expert_image_elems(d: int, ffn: int) -> int:
    return lib().moespac_expert_image_elems(d, ffn)


FFN_AUTO, FFN_CUDACORE, FFN_TENSOR = 0, 1, 2


def ffn_resolve(kernel: int, d: int, ffn: int) -> int:
    return lib().moespac_ffn_resolve(kernel, d, ffn)


def pack_expert(wg, wu, wd, kernel: int = FFN_AUTO, stream=None):
    """Standard-layout bf16 (int16 views) -> tiled image for `kernel` (int16 view)."""
    import torch
    ffn, d = wg.shape
    out = torch.empty(3 * ffn * d, dtype=torch.int16, device=wg.device)
    check(lib().moespac_pack_expert(ptr(wg), ptr(wu), ptr(wd), d, ffn, kernel, ptr(out), _stream(stream)))
    return out


def unpack_expert(image, d: int, ffn: int, kernel: int = FFN_AUTO, stream=None):
    """Tiled image (device tensor) -> (w_gate [ffn][d], w_up [ffn][d], w_down [d][ffn]) int16 views."""
    import torch
    dev = image.device
    wg = torch.empty((ffn, d), dtype=torch.int16, device=dev)
    wu = torch.empty((ffn, d), dtype=torch.int16, device=dev)
    wd = torch.empty((d, ffn), dtype=torch.int16, device=dev)
    check(lib().moespac_unpack_expert(ptr(image), d, ffn, kernel, ptr(wg), ptr(wu), ptr(wd), _stream(stream)))
    return wg, wu, wd


SHARED_GATE_NONE, SHARED_GATE_SIGMOID = 0, 1


def draft_gemv(w, x0=None, y_prev=None, scale: float = 1.0, stream=None):
    """One draft pass: y [R] fp32 = w [R][D] (bf16, int16 view) . x."""
    import torch
    R, D = w.shape
    y = torch.empty(R, dtype=torch.float32, device=w.device)
    check(lib().moespac_draft_gemv(ptr(w), R, D, ptr(y_prev), ptr(x0), scale, ptr(y), _stream(stream)))
    return y


def build_hT(h, stream=None):
    """[T][d] bf16 (int16 view) -> h^T UMMA image for the tensor-core K3."""
    import torch
    T, d = h.shape
    out = torch.empty(16 * d, dtype=torch.int16, device=h.device)
    check(lib().moespac_build_hT(ptr(h), T, d, ptr(out), _stream(stream)))
    return out


# ---------------------------------------------------------------- engine context
class Context:
    """moespac_ctx: the full verification step on one device."""

    def __init__(self, device: int, model: ModelDesc, cfg: SchedConfig, rank: int = 0, world: int = 1):
        self.model, self.cfg, self.rank, self.world = model, cfg, rank, world
        h = C.c_void_p()
        check(lib().moespac_ctx_create(device, C.byref(model), C.byref(cfg), rank, world, C.byref(h)))
        self._h = h
        # AR policy: one token per step (the context runs at T = 1)
        self.T = 1 if cfg.policy == POLICIES.index("ar_mode") else model.gamma + 1
        self.image_elems = expert_image_elems(model.d_model, model.d_ffn)

    def close(self):
        if getattr(self, "_h", None):
            lib().moespac_ctx_destroy(self._h)
            self._h = None

    __del__ = close

    def host_arena(self, n_images: int) -> np.ndarray:
        p = C.c_void_p()
        check(lib().moespac_ctx_host_arena(self._h, n_images, C.byref(p)))
        arr = np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_uint16)), shape=(n_images, self.image_elems))
        return arr

    def fill_synthetic(self, seed: int = 3, stdv: float = 0.006):
        check(lib().moespac_ctx_fill_synthetic(self._h, seed, stdv))

    def set_shared(self, layer: int, units_dev):
        check(lib().moespac_ctx_set_shared(self._h, layer, ptr(units_dev)))

    def set_shared_gate(self, layer: int, w) -> None:
        """Shared-expert gate vector w_sg of a layer, [d_model] bf16 (host array or device tensor)."""
        if isinstance(w, np.ndarray):
            w = np.ascontiguousarray(w.view(np.uint16))
        check(lib().moespac_ctx_set_shared_gate(self._h, layer, ptr(w)))

    def estimator_dump(self, path: str):
        """Device estimator state -> the reference's checkpoint text format."""
        check(lib().moespac_ctx_estimator_dump(self._h, path.encode()))

    def estimator_load(self, path: str):
        check(lib().moespac_ctx_estimator_load(self._h, path.encode()))

    def finalize(self):
        check(lib().moespac_ctx_finalize(self._h))

    def set_timing(self, on: bool = True):
        check(lib().moespac_ctx_set_timing(self._h, int(on)))

    def set_cold_threads(self, n: int = -1):
        check(lib().moespac_ctx_set_cold_threads(self._h, n))

    def set_cold_staging(self, slots: int, fraction: float):
        """Run `fraction` of each layer's misses on the device from a staging
        ring of `slots` HBM images (before finalize; 0 slots = off)."""
        check(lib().moespac_ctx_set_cold_staging(self._h, slots, fraction))

    def set_pdl(self, on: bool = True):
        check(lib().moespac_ctx_set_pdl(self._h, int(on)))

    def set_graph(self, on: bool = True):
        """Launch-latency path: replay a captured CUDA graph of load-free steps."""
        check(lib().moespac_ctx_set_graph(self._h, int(on)))

    def set_draft_window(self, on: bool = True):
        check(lib().moespac_ctx_set_draft_window(self._h, int(on)))

    def set_draft_model(self, n_params: int, d_draft: int = 2560):
        """Real draft phase: gamma weight-streaming GEMV passes over n_params bf16 weights per step (0: off)."""
        check(lib().moespac_ctx_set_draft_model(self._h, int(n_params), int(d_draft)))

    def set_timeline(self, on: bool = True):
        """Measured SimEvent-shaped timeline (clears the previous one)."""
        check(lib().moespac_ctx_set_timeline(self._h, int(on)))

    def timeline(self):
        """(events [n][6], measured LayerTiming rows [steps*L], steps [n][6])."""
        f = lib()
        n = f.moespac_ctx_timeline_events(self._h, None, 0)
        ev = np.zeros((max(n, 1), 6), np.int64)
        f.moespac_ctx_timeline_events(self._h, ev.ctypes.data, n)
        nl = f.moespac_ctx_timeline_layers(self._h, None, 0)
        lay = (LayerTiming * max(nl, 1))()
        f.moespac_ctx_timeline_layers(self._h, lay, nl)
        ns = f.moespac_ctx_timeline_steps(self._h, None, 0)
        st = np.zeros((max(ns, 1), 6), np.int64)
        f.moespac_ctx_timeline_steps(self._h, st.ctypes.data, ns)
        return ev[:n], list(lay)[:nl], st[:ns]

    def set_l2_prefetch(self, nbytes: int):
        """Per-CTA cross-layer L2 prefetch budget of the tensor-core K3 (0 = off)."""
        check(lib().moespac_ctx_set_l2_prefetch(self._h, int(nbytes)))

    def set_k3_trace(self, buf_ptr):
        """Profiling: per-CTA K3 stamps into a device buffer [L][grid][32] int64 (None: off)."""
        check(lib().moespac_ctx_set_k3_trace(self._h, buf_ptr))

    def set_nccl(self, uid: bytes, nranks: int, rank: int):
        buf = C.create_string_buffer(uid, 128)
        check(lib().moespac_ctx_set_nccl(self._h, buf, nranks, rank))

    def step(self, logits_host: np.ndarray, h_in_host: np.ndarray, accepted: int, h_out_host: np.ndarray):
        rep = StepReport()
        lay = (LayerTiming * self.model.n_layers)()
        check(lib().moespac_step(self._h, ptr(logits_host), ptr(h_in_host), accepted, ptr(h_out_host),
                                 C.byref(rep), lay))
        return rep, list(lay)

    def step_ids(self, ids_host: np.ndarray, gates_host, h_in_host: np.ndarray, accepted: int,
                 h_out_host: np.ndarray):
        """Trace replay: recorded routing ids [L][T][k] (gates or None = 1/k)."""
        rep = StepReport()
        lay = (LayerTiming * self.model.n_layers)()
        ids = np.ascontiguousarray(ids_host, dtype=np.int32)
        g = None if gates_host is None else np.ascontiguousarray(gates_host, dtype=np.float32)
        check(lib().moespac_step_ids(self._h, ptr(ids), ptr(g), ptr(h_in_host), accepted, ptr(h_out_host),
                                     C.byref(rep), lay))
        return rep, list(lay)

    def set_router(self, layer: int, w) -> None:
        """Router weights W_g of a layer, [n_experts][d_model] bf16 (host array or device tensor)."""
        if isinstance(w, np.ndarray):
            w = np.ascontiguousarray(w.view(np.uint16))
        check(lib().moespac_ctx_set_router(self._h, layer, ptr(w)))

    def step_model(self, h_in_host: np.ndarray, accepted: int, h_out_host: np.ndarray):
        """Model mode: routing from the on-device router GEMV of each layer's input."""
        rep = StepReport()
        lay = (LayerTiming * self.model.n_layers)()
        check(lib().moespac_step_model(self._h, ptr(h_in_host), accepted, ptr(h_out_host), C.byref(rep), lay))
        return rep, list(lay)

    def step_model_device(self, h_in_dev, accepted: int, h_out_dev):
        rep = StepReport()
        lay = (LayerTiming * self.model.n_layers)()
        check(lib().moespac_step_model_device(self._h, ptr(h_in_dev), accepted, ptr(h_out_dev), C.byref(rep), lay))
        return rep, list(lay)

    def set_loopback(self, group: "LoopbackGroup") -> None:
        check(lib().moespac_ctx_set_loopback(self._h, group._h))

    def step_device(self, logits_dev, h_in_dev, accepted: int, h_out_dev):
        rep = StepReport()
        lay = (LayerTiming * self.model.n_layers)()
        check(lib().moespac_step_device(self._h, ptr(logits_dev), ptr(h_in_dev), accepted, ptr(h_out_dev),
                                        C.byref(rep), lay))
        return rep, list(lay)

    def stream(self) -> int:
        return lib().moespac_ctx_stream(self._h) or 0

    K3_NAMES = {0: "expert_ffn_kernel (K3, CUDA-core GEMV)", 1: "expert_ffn_tc_kernel (K3, smem accumulator)",
                2: "expert_ffn_tc_kernel (K3, L2 accumulator)", 3: "expert_ffn_tc_kernel (K3, TMEM accumulator)",
                4: "expert_ffn_tg_kernel (K3, grouped)"}

    def parallel_mode(self) -> str:
        return {1: "expert", 2: "units"}[lib().moespac_ctx_parallel_mode(self._h)]

    def k3_kernel(self) -> str:
        return self.K3_NAMES[lib().moespac_ctx_k3_variant(self._h)]

    def views(self) -> CtxViews:
        v = CtxViews()
        check(lib().moespac_ctx_get_views(self._h, C.byref(v)))
        return v

    def sched_events(self) -> np.ndarray:
        s = lib().moespac_ctx_sched(self._h)
        n = lib().moespac_sched_events(s, None, 0)
        out = np.zeros((max(n, 1), 6), np.int64)
        lib().moespac_sched_events(s, out.ctypes.data, n)
        return out[:n]

    def step_tables(self):
        """Decision tables the last executed step ran with."""
        L, N = self.model.n_layers, self.model.n_experts
        W = (N + 31) // 32
        taus = np.zeros(L, np.int32)
        rb = np.zeros((L, W), np.uint32)
        lb = np.zeros((L, W), np.uint32)
        slots = np.zeros((L, N), np.int32)
        check(lib().moespac_ctx_step_tables(self._h, taus.ctypes.data, rb.ctypes.data, lb.ctypes.data,
                                            slots.ctypes.data))
        return taus, rb, lb, slots

    def sched_decisions(self) -> np.ndarray:
        s = lib().moespac_ctx_sched(self._h)
        out = np.zeros((self.model.n_layers, 5), np.int64)
        check(lib().moespac_sched_decisions(s, out.ctypes.data))
        return out


_cudart_lib = None


def _cudart() -> C.CDLL:
    """The process's CUDA runtime (already loaded by torch) — used only to
    read device views back for checks."""
    global _cudart_lib
    if _cudart_lib is None:
        import torch  # noqa: F401  (ensures libcudart is loaded)
        for name in ("libcudart.so.12", "libcudart.so"):
            try:
                _cudart_lib = C.CDLL(name)
                break
            except OSError:
                continue
        if _cudart_lib is None:
            raise ImportError("libcudart not loadable")
        _cudart_lib.cudaMemcpy.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int]
        _cudart_lib.cudaDeviceSynchronize.argtypes = []
    return _cudart_lib


def fetch(dev_ptr: int, shape, dtype) -> np.ndarray:
    """Copy a device buffer into a new numpy array (synchronous)."""
    out = np.empty(shape, dtype)
    rt = _cudart()
    rt.cudaDeviceSynchronize()
    rc = rt.cudaMemcpy(out.ctypes.data, dev_ptr, out.nbytes, 2)  # cudaMemcpyDeviceToHost
    if rc != 0:
        raise RuntimeError(f"cudaMemcpy D2H failed ({rc})")
    return out


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    check(lib().moespac_nccl_unique_id(buf))
    return buf.raw


class LoopbackGroup:
    """In-process expert-parallel group on one device (moespac_loopback_*):
    a test harness for the EP device path without NCCL."""

    def __init__(self, device: int, world: int, max_elems: int):
        h = C.c_void_p()
        check(lib().moespac_loopback_create(device, world, max_elems, C.byref(h)))
        self._h = h.value

    def close(self):
        if self._h:
            lib().moespac_loopback_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()
