#!/usr/bin/env python
"""bench.py — MoE-SpAc verification-step hot path on B200.

Metric (BASELINE.json): decode TPS and expert-FFN HBM GB/s (roofline %) at
1/2/4/8 B200 vs host CPU.

One "step" = one full verification step of all L MoE layers through the
engine (moespac_step*): host HWB/AEE decisions for every layer, the
decided expert loads on the copy stream, K1 router (all layers), K2
hist/scan/estimator (all layers), and per layer K3 expert FFN + combine
(+ NCCL all-reduce in expert-parallel mode), D2H of scores/counters, host
accounting. TPS = accepted tokens / device time.

  value : inputs (logits, hidden states) already resident in HBM
  e2e   : the same through moespac_step with pinned HOST buffers; H2D of
          logits + h_in + decision tables (+ any expert loads) and D2H of
          h_out + scores/counters inside the timed region
  roofline: K3 algorithmic bytes per launch / its launch duration, from
          every CTA's %globaltimer stamps in a window run exactly like the
          timed one (programmatic dependent launch on); the CUDA-event
          per-launch time (PDL off) is reported beside it
  cpu_baseline: the CPU oracle port of the same step on the box's cores
  detail.budget: a second workload at a BASELINE cache budget (default
          Qwen3-30B-A3B at 17%: real expert loads + the host cold path),
          median / spread of 5 windows for value and e2e, its own roofline
          and cpu_baseline

--impl reference: the reference's CPU path for the same workload (the
compiled reference scheduler oracle/_ref + the CPU oracle port of the
router and the expert FFN on all host threads) — see DESIGN.md §Measurement.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

REASONS = {  # clocks_event_reasons bitmask (nvml)
    0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
    0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
    0x100: "display_clock_setting",
}


HWB_PROFILE_NAME = "reference"


def HWB_PROFILE(w):
    """SchedConfig profile overrides of the selected --hwb-profile for workload w."""
    from paper_2603_09983_b200.configs import HWB_PROFILES
    return HWB_PROFILES[HWB_PROFILE_NAME](w)


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="mixtral")
    ap.add_argument("--cache-ratio", type=float, default=None)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget-s", type=float, default=15.0)
    ap.add_argument("--settle", type=int, default=20,
                    help="extra untimed steps before the timed windows when the cache budget is < 1 "
                         "(the warm fill holds experts 0..cap-1, not the hot ones)")
    ap.add_argument("--ffn-kernel", type=int, default=0, help="0 auto (tcgen05), 1 CUDA-core GEMV, 2 tcgen05")
    ap.add_argument("--draft-params", type=float, default=2e9,
                    help="detail.draft_verify leg: a dense bf16 draft model of this many parameters (2e9 bf16 = the "
                         "~4 GB a Qwen3-4B-FP8 draft token streams) drafting gamma tokens before each verification "
                         "step on the same GPU; 0 skips the leg")
    ap.add_argument("--draft-d", type=int, default=2560)
    ap.add_argument("--no-budget", action="store_true",
                    help="skip the cache-budget leg (detail.budget: a BASELINE budget config, real expert loads "
                         "and the host cold path, median of windows)")
    ap.add_argument("--budget-config", default="qwen3")
    ap.add_argument("--budget-cache", type=float, default=0.17)
    ap.add_argument("--budget-windows", type=int, default=7)
    ap.add_argument("--budget-steps", type=int, default=20)
    ap.add_argument("--stage-slots", type=int, default=16,
                    help="cold-expert staging ring below a full cache (HBM images; 0 = off): --stage-frac of each "
                         "layer's misses is copied over PCIe and run by K3 instead of on the host cores (decisions "
                         "unchanged; measured, median of 7 windows: Qwen3 @ 0.17 288 / 291 / 307 / 311 TPS at "
                         "0 / 0.2 / 0.3 / 0.4, DSV2 @ 0.17 185 / 200 / 198 at 0 / 0.2 / 0.4 — host DRAM is the "
                         "shared bound)")
    ap.add_argument("--stage-frac", type=float, default=0.3)
    ap.add_argument("--hwb-profile", default="reference", choices=["reference", "b200"],
                    help="HWB hardware profile: the reference's defaults (config.cpp:23-27) or constants calibrated "
                         "to B200 (configs.b200_hwb_profile); decisions are checked against the reference run with "
                         "the same constants where a golden fixture exists")
    ap.add_argument("--draft-window", action="store_true",
                    help="emulated draft phase: gamma x t_draft_unit (reference default 300 us/token) on the compute "
                         "stream before each verification step, expert loads overlapping it; TPS then counts "
                         "draft + verification (the reference's definition)")
    ap.add_argument("--router-gemv", action="store_true",
                    help="model mode: routing from the on-device router GEMV W_g h_l of random-init router weights "
                         "(K0 -> K1 -> K2 per layer) instead of the trace generator's logits; cold path off")
    return ap.parse_args()


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.f, stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.p = None
        time.sleep(1.0)  # (nvidia-smi's start-up burns host CPU: keep it out of the first window)
        return self

    def __exit__(self, *exc):
        if self.p:
            self.p.terminate()
            self.p.wait()

    def summary(self):
        self.f.flush()
        self.f.seek(0)
        sm, mx, reasons = [], 0.0, set()
        for line in self.f.read().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 3:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
                bits = int(parts[2], 16) if parts[2].startswith("0x") else int(parts[2])
            except ValueError:
                continue
            for b, name in REASONS.items():
                if bits & b:
                    reasons.add(name)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def workload_named(name, cache_ratio=None):
    from paper_2603_09983_b200.configs import CONFIGS
    w = CONFIGS[name]
    if cache_ratio is not None:
        w = w.with_(cache_ratio=cache_ratio)
    return w


def workload(args):
    return workload_named(args.config, args.cache_ratio)


# ------------------------------------------------------------------ CPU leg
def cpu_path_sample(w, budget_s: float, use_ref_sched: bool):
    """Time the CPU path of one verification step on a bounded sample.

    Per step: router top-k over L*T rows + histogram/estimator (oracle C
    port), the reference scheduler for all layers (oracle/_ref when built,
    1 thread — the reference has no threads), and the expert FFN of every
    activated expert (oracle fp32 SwiGLU, all host threads). The FFN is
    sampled on whole layers until the budget is spent and scaled to L.
    """
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O

    L, N, k, g, d, ffn, T = w.n_layers, w.n_experts, w.top_k, w.gamma, w.d_model, w.d_ffn, w.tokens
    threads = O.orc().orc_max_threads()
    rng = np.random.default_rng(3)
    # one expert image reused for every expert id: the byte stream per
    # activation is the same 3*d*ffn*2 bytes (far beyond the LLC)
    def rbf16(shape):
        sign = rng.integers(0, 2, shape, dtype=np.uint16) << 15
        return (sign | rng.integers(0x3a00, 0x3d00, shape, dtype=np.uint16)).astype(np.uint16)
    wg, wu, wd = rbf16((ffn, d)), rbf16((ffn, d)), rbf16((d, ffn))
    shared = [(wg, wu, wd)] * w.n_shared_units
    gen = O.Generator(L, N, k, g, seed=1)
    n_steps = 8
    trace = [gen.next_step() for _ in range(n_steps)]
    accepted = np.array([t[2] for t in trace], np.float64)
    h = O.f32_to_bf16_bits(rng.normal(0, 1, (T, d)).astype(np.float32))

    # router + histogram + estimator (port), per step
    t0 = time.perf_counter()
    st = [O.estimator_init(N, g) for _ in range(L)]
    for logits, _ids, _a in trace:
        ids, gates = O.router_topk(logits, k, w.gate_mode)
        for l in range(L):
            f, _, _ = O.hist_scan(ids[l], N)
            st[l] = O.estimator_observe(st[l], f, 4, 0.1)
    t_route = (time.perf_counter() - t0) / n_steps

    # reference scheduler (the reference's own code) per step
    t_sched, sched_kind = 0.0, "none"
    if use_ref_sched and O.ref_available():
        cfg = O.default_config(n_layers=L, n_experts=N, top_k=k, gamma=g, cache_ratio=w.cache_ratio, token_budget=0,
                               **HWB_PROFILE(w))
        ids_arr = np.stack([t[1] for t in trace])
        t_sched = O.ref().ref_sim_time_ns(cfg, ids_arr.reshape(-1).astype(np.int32),
                                          accepted.astype(np.int32), n_steps) * 1e-9
        sched_kind = "reference"

    # expert FFN, whole layers until the budget is spent
    import ctypes as C
    y = np.zeros((T, d), np.float32)
    layer_times = []
    t_start = time.perf_counter()
    s = 0
    while time.perf_counter() - t_start < budget_s and len(layer_times) < 4 * L:
        logits, ids, _a = trace[s % n_steps]
        l = len(layer_times) % L
        ids_l, gates_l = O.router_topk(logits[l], k, w.gate_mode)
        t1 = time.perf_counter()
        for e in np.unique(ids_l):
            toks = np.nonzero((ids_l == e).any(axis=1))[0].astype(np.int32)
            gsel = np.array([gates_l[t][list(ids_l[t]).index(e)] for t in toks], np.float32)
            O.orc().orc_expert_apply_f32(h.ctypes.data, d, ffn, toks, gsel, len(toks), wg.ctypes.data,
                                         wu.ctypes.data, wd.ctypes.data, y, threads)
        for (sg, su, sd) in shared:
            O.orc().orc_expert_apply_f32(h.ctypes.data, d, ffn, np.arange(T, dtype=np.int32),
                                         np.ones(T, np.float32), T, sg.ctypes.data, su.ctypes.data, sd.ctypes.data,
                                         y, threads)
        layer_times.append(time.perf_counter() - t1)
        if l == L - 1:
            s += 1
    t_ffn_step = float(np.mean(layer_times)) * L
    step_s = t_route + t_sched + t_ffn_step
    tps = float(accepted.mean()) / step_s
    sample = (f"{len(layer_times)} layer-FFN samples ({w.name}, all activated experts, {threads} threads) "
              f"scaled to {L} layers + router/hist/estimator port over {n_steps} steps"
              + (" + reference Simulation::run_step scheduler (1 thread)" if sched_kind == "reference" else ""))
    return {"value": tps, "unit": "tokens/s", "cores": threads, "kind": "port", "sample": sample,
            "step_ms": step_s * 1e3, "ffn_ms_per_layer": float(np.mean(layer_times)) * 1e3,
            "route_ms": t_route * 1e3, "sched_ms": t_sched * 1e3}


# ------------------------------------------------------------------ GPU leg
def golden_path(w):
    """The committed reference fixture (tests/golden, made from the compiled
    reference) for this workload at this budget, if there is one: its trace is
    the bench's (reference defaults, seed 1), so the warm-up steps' decisions
    must equal it record for record."""
    name = {("mixtral", 1.0): "mixtral_c100", ("mixtral", 0.17): "mixtral", ("tiny", 0.17): "tiny",
            ("tiny", 1.0): "tiny_c100", ("qwen15", 0.5): "qwen15", ("dsv2", 0.17): "dsv2"}.get(
        (w.name, round(w.cache_ratio, 2)))
    if w.name == "qwen3":
        name = "qwen3_c%03d" % round(w.cache_ratio * 100)
    if name and HWB_PROFILE_NAME != "reference":
        name += "_" + HWB_PROFILE_NAME
    p = os.path.join(ROOT, "tests", "golden", f"sim_{name}.npz") if name else None
    return p if p and os.path.exists(p) else None


def check_decisions(ctx, w, n_steps):
    """SimEvent log of the first n_steps equals the reference's (golden)."""
    p = golden_path(w)
    if not p:
        return None
    z = np.load(p)
    n = min(n_steps, len(z["accepted"]))
    ev = z["events"]
    got = ctx.sched_events()
    ok = np.array_equal(got[got[:, 1] < n], ev[ev[:, 1] < n])
    if not ok:
        raise SystemExit(f"bench: decision parity FAILED against {os.path.relpath(p, ROOT)} over {n} steps")
    return {"golden": os.path.relpath(p, ROOT), "steps": int(n), "events": int((ev[:, 1] < n).sum()), "equal": True}


def n_images_for(w):
    """Pinned master-copy images: expert (l, e) -> image (l*N + e) % n. At a
    partial budget the host cold path reads them, so use >= 8 GiB of distinct
    images (beyond any LLC) and n = N + 1 at least, so the same expert id in
    consecutive layers never maps to the same image."""
    n = w.n_experts + 1
    if w.cache_ratio < 1.0:
        n = max(n, -(-(8 << 30) // w.expert_bytes))
    return min(w.n_layers * w.n_experts, n)


def run_ours(args, w, rank, world, local_rank, windows=1, label="headline", steps=None, draft_params=0):
    import torch

    from paper_2603_09983_b200 import abi
    from paper_2603_09983_b200.configs import SYNTH_STD

    torch.cuda.set_device(local_rank)
    L, N, k, g, d, ffn, T = w.n_layers, w.n_experts, w.top_k, w.gamma, w.d_model, w.d_ffn, w.tokens
    cfg = abi.default_config(n_layers=L, n_experts=N, top_k=k, gamma=g, cache_ratio=w.cache_ratio,
                             **HWB_PROFILE(w))
    model = w.model_desc(args.ffn_kernel)

    def make_ctx():
        c = abi.Context(local_rank, model, cfg, rank, world)
        if args.stage_slots > 0 and w.cache_ratio < 1.0:
            c.set_cold_staging(args.stage_slots, args.stage_frac)
        c.host_arena(n_images_for(w))
        c.fill_synthetic(seed=3, stdv=SYNTH_STD)
        if args.router_gemv:
            c.set_cold_threads(0)
        c.finalize()
        if args.draft_window:
            c.set_draft_window(True)
        if draft_params > 0:
            c.set_draft_model(int(draft_params), args.draft_d)
        if args.router_gemv:
            gw = torch.Generator().manual_seed(4)
            for l in range(L):
                c.set_router(l, (torch.randn((N, d), generator=gw) * 0.05).to(torch.bfloat16).cuda())
        if world > 1:
            import torch.distributed as dist
            obj = [abi.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            c.set_nccl(obj[0], world, rank)
        return c

    ctx = make_ctx()
    # Synthetic inputs: routing from the trace synthesizer (reference
    # TraceGenerator semantics, seed 1), hidden states ~ N(0, 1) bf16.
    # Trace steps: W warm-up (+ settle steps below a full cache), then
    # `windows` windows of K steps for `value`, one more window with the K3
    # globaltimer stamps (PDL on) and one with per-K3 CUDA events (PDL off).
    # The end-to-end run uses a fresh context through the same warm-up and
    # the same `windows` windows, so both start from the same cache state.
    settle = args.settle if w.cache_ratio < 1.0 else 0
    w0 = args.warmup + settle
    K = steps or args.steps
    # (several windows: one more untimed window first, inside the clock
    # sampler — after its start-up second the first timed window of a
    # sub-millisecond step otherwise ran 3-5x slower, on both contexts alike)
    pre = K if windows > 1 else 0
    ws = w0 + pre  # first timed step
    S = ws + (windows + 2) * K
    synth = abi.TraceSynth(cfg)
    logits_h = torch.empty((S, L, T, N), dtype=torch.float64).pin_memory()
    accepted = []
    for s in range(S):
        _, a = synth.next(logits_h[s].numpy())
        accepted.append(a)
    gen = torch.Generator().manual_seed(2)
    h_h = torch.randn((S, T, d), generator=gen).to(torch.bfloat16).pin_memory()
    h_out_h = torch.empty((T, d), dtype=torch.bfloat16).pin_memory()
    logits_d = logits_h.cuda()
    h_d = h_h.cuda()
    h_out_d = torch.empty((T, d), dtype=torch.bfloat16, device="cuda")
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if world > 1:
            import torch.distributed as dist
            t = torch.tensor([x], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return float(t.item())
        return x

    def timed(fn, n, offset, per_step=None, c=None):
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        stream = torch.cuda.ExternalStream((c or ctx).stream())
        reps = []
        nvtx = os.environ.get("MOESPAC_NVTX") == "1"  # profiling: ncu --nvtx --nvtx-include "timed/"
        if nvtx:
            torch.cuda.nvtx.range_push("timed")
        e0.record(stream)
        for i in range(n):
            reps.append(fn(offset + i))
            if per_step:
                per_step(reps[-1])
        e1.record(stream)
        if nvtx:
            torch.cuda.nvtx.range_pop()
        barrier()
        return max_over_ranks(e0.elapsed_time(e1)), reps

    # host buffers as numpy views, made once (the API call is what is timed)
    logits_np = [logits_h[s].numpy() for s in range(S)]
    h_np = [h_h[s].view(torch.int16).numpy() for s in range(S)]
    h_out_np = h_out_h.view(torch.int16).numpy()
    dev_step = lambda s, c=None: (c or ctx).step_device(logits_d[s], h_d[s], accepted[s], h_out_d)[0]  # noqa: E731
    host_step = lambda s, c=None: (c or ctx).step(logits_np[s], h_np[s], accepted[s], h_out_np)[0]  # noqa: E731
    if args.router_gemv:
        dev_step = lambda s, c=None: (c or ctx).step_model_device(h_d[s], accepted[s], h_out_d)[0]  # noqa: E731
        host_step = lambda s, c=None: (c or ctx).step_model(h_np[s], accepted[s], h_out_np)[0]  # noqa: E731
    for i in range(w0):
        dev_step(i)
    parity = None if args.router_gemv else check_decisions(ctx, w, w0)
    tok = lambda o, n: float(sum(accepted[o + i] for i in range(n)))  # noqa: E731
    sms = torch.cuda.get_device_properties(local_rank).multi_processor_count
    stamps = torch.zeros((L, sms, 32), dtype=torch.int64, device="cuda")
    spans, spans_raw = [], []

    def read_stamps(_rep):
        # K3 launch durations of this step from its CTAs' %globaltimer
        # stamps. The kernels ran with programmatic dependent launch, as in
        # the timed windows, so a K3's first CTAs start while the previous
        # layer still runs: the duration is counted from the later of its
        # first CTA start and the previous K3's last CTA end (the overlap is
        # not counted twice: the spans of a step sum to less than the step)
        # to its last CTA end.
        st = stamps.cpu().numpy()
        prev_end = None
        for l in range(L):
            beg, end = st[l, :, 0], st[l, :, 6]
            if (end > 0).any():
                b0, e1 = beg[beg > 0].min(), end[end > 0].max()
                spans_raw.append((e1 - b0) * 1e-6)
                spans.append((e1 - (b0 if prev_end is None else max(b0, prev_end))) * 1e-6)
                prev_end = e1
        stamps.zero_()
        torch.cuda.synchronize()

    # Several windows (the budget leg) interleave the value and e2e windows
    # on two contexts driven through the same warm-up, so slow drifts of the
    # host (the cold path runs on its cores) hit both alike; when two expert
    # pools do not fit the device, e2e runs after, on a fresh context.
    cap = max(1, int(w.cache_ratio * N + 1e-9))
    pool_bytes = L * min(N, cap) * w.expert_bytes
    interleave = windows > 1 and torch.cuda.mem_get_info()[0] > pool_bytes + (8 << 30)
    ctx2 = None
    if interleave:
        ctx2 = make_ctx()
        for i in range(w0):
            host_step(i, ctx2)
    with ClockSampler(local_rank) as clk:
        ctx.set_timing(False)
        win, win_e2e = [], []  # (ms, tokens, reps) per window
        for i in range(w0, ws):
            dev_step(i)
            if ctx2 is not None:
                host_step(i, ctx2)
        for j in range(windows):
            ms, reps = timed(dev_step, K, ws + j * K)
            win.append((ms, tok(ws + j * K, K), reps))
            if ctx2 is not None:
                ms, reps = timed(lambda s: host_step(s, ctx2), K, ws + j * K, c=ctx2)
                win_e2e.append((ms, tok(ws + j * K, K), reps))
        if ctx2 is not None:
            ctx2.close()
        o = ws + windows * K
        # K3 stamps, PDL on (the timed windows' launch mode)
        ctx.set_k3_trace(abi.ptr(stamps))
        ms_st, reps_st = timed(dev_step, K, o, per_step=read_stamps)
        ctx.set_k3_trace(None)
        # per-K3 CUDA events (PDL off so each pair brackets one kernel)
        ctx.set_timing(True)
        ms_ev, reps_ev = timed(dev_step, K, o + K)
        ctx.set_timing(False)
        if ctx2 is None:
            # end to end through the host API: fresh context through the same
            # warm-up, the same windows
            ctx.close()
            ctx = make_ctx()  # (the step lambdas look ctx up at call time)
            for i in range(ws):
                host_step(i)
            for j in range(windows):
                ms, reps = timed(host_step, K, ws + j * K)
                win_e2e.append((ms, tok(ws + j * K, K), reps))
    ffn_bytes_st = sum(r.ffn_bytes for r in reps_st)
    n_launch_st = sum(r.ffn_launches for r in reps_st)
    out = {
        "label": label, "w0": w0, "pre": pre, "settle": settle, "windows": windows, "K": K, "interleaved": bool(interleave),
        "win": [(m, t) for m, t, _ in win], "win_e2e": [(m, t) for m, t, _ in win_e2e],
        "ms": win[0][0], "tokens": win[0][1], "ms_e2e": win_e2e[0][0], "tokens_e2e": win_e2e[0][1],
        "k3_span_ms": spans, "k3_span_raw_ms": spans_raw, "ffn_bytes_st": ffn_bytes_st, "ffn_launches_st": n_launch_st,
        "ffn_ms_ev": sum(r.gpu_ms_ffn for r in reps_ev), "ffn_bytes_ev": sum(r.ffn_bytes for r in reps_ev),
        "ffn_launches_ev": sum(r.ffn_launches for r in reps_ev),
        "launches": sum(r.kernel_launches for r in win[0][2]),
        "hits": sum(r.cache_hits for _, _, rs in win for r in rs),
        "misses": sum(r.cache_misses for _, _, rs in win for r in rs),
        "loads": sum(r.n_loads for _, _, rs in win for r in rs),
        "cold_experts": sum(r.cold_experts for _, _, rs in win for r in rs),
        "staged_experts": sum(r.staged_experts for _, _, rs in win for r in rs),
        "cpu_ms_cold": sum(r.cpu_ms_cold for _, _, rs in win for r in rs),
        "k3_kernel": ctx.k3_kernel(), "parallel_mode": ctx.parallel_mode(),
        "h2d": float(np.mean([r.h2d_bytes for _, _, rs in win_e2e for r in rs])),
        "d2h": float(np.mean([r.d2h_bytes for _, _, rs in win_e2e for r in rs])),
        "router_ms": float(np.mean([r.gpu_ms_router for r in reps_ev])),
        "hist_ms": float(np.mean([r.gpu_ms_hist for r in reps_ev])),
        "gpu_step_ms": float(np.mean([r.gpu_ms_total for r in reps_ev])),
        "layers_other_ms": float(np.mean([r.gpu_ms_combine for r in reps_ev])),
        "ms_ev": ms_ev, "ms_st": ms_st, "parity": parity, "n_images": n_images_for(w),
        "draft_ms_ev": sum(r.gpu_ms_draft for r in reps_ev), "draft_bytes": sum(r.draft_bytes for r in reps_ev),
        "clocks": clk.summary(),
    }
    if world > 1:
        import torch.distributed as dist
        # multi-GPU roofline: K3 bytes summed over ranks over the max K3 time
        t = torch.tensor([ffn_bytes_st, float(np.sum(spans))], dtype=torch.float64, device="cuda")
        dist.all_reduce(t[:1], op=dist.ReduceOp.SUM)
        tm = t[1:].clone()
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
        out["ffn_bytes_st_all"] = float(t[0].item())
        out["k3_span_ms_max_rank"] = float(tm[0].item())
    ctx.close()
    return out


def L_layers(w):
    return w.n_layers


def args_steps(args, r):
    return r.get("K", args.steps)


def leg_summary(r, w, args, world, hbm_peak, peak_kind):
    """value / e2e / roofline of one leg (one workload)."""
    tps = [t / (m * 1e-3) for m, t in r["win"]]
    tps_e2e = [t / (m * 1e-3) for m, t in r["win_e2e"]]
    spans = r["k3_span_ms"]
    span_ms = float(np.mean(spans)) if spans else 0.0
    bytes_per_launch = r["ffn_bytes_st"] / max(1, r["ffn_launches_st"])
    if world > 1 and "ffn_bytes_st_all" in r:
        achieved = r["ffn_bytes_st_all"] / (r["k3_span_ms_max_rank"] * 1e-3) / 1e9 if r["k3_span_ms_max_rank"] else 0.0
    else:
        achieved = bytes_per_launch / (span_ms * 1e-3) / 1e9 if span_ms > 0 else 0.0
    ev_ms = r["ffn_ms_ev"] / max(1, r["ffn_launches_ev"])
    ev_achieved = r["ffn_bytes_ev"] / max(1, r["ffn_launches_ev"]) / (ev_ms * 1e-3) / 1e9 if ev_ms > 0 else 0.0
    traffic, traffic_capture = None, None
    prof = os.path.join(ROOT, "profiles", f"ncu_k3_{w.name}.json")
    if os.path.exists(prof):
        try:
            cap = json.load(open(prof))
            ratio = cap.get("traffic_over_algorithmic")
            traffic = ratio * bytes_per_launch if ratio else None
            traffic_capture = {"dram_bytes": cap.get("dram_bytes_per_launch"),
                               "algorithmic_bytes": cap.get("algorithmic_bytes_of_launch"), "ratio": ratio,
                               "kernel": cap.get("kernel"), "report": cap.get("report")}
        except (ValueError, OSError, TypeError):
            traffic = None
    roof = {"bound": "hbm", "kernel": r["k3_kernel"], "achieved": achieved, "peak": hbm_peak,
            "peak_source": f"{peak_kind} hbm_gbs (MEASURED_PEAKS.json)" if peak_kind == "measured"
            else "fallback 6650 GB/s (B200_PROFILING.md)",
            "unit": "GB/s", "frac": achieved / hbm_peak, "traffic": traffic, "traffic_capture": traffic_capture,
            "bytes_per_launch": bytes_per_launch, "ms_per_launch": span_ms,
            "timing": "K3 launch duration from every CTA's %globaltimer stamps in a K-step window run with "
                      "programmatic dependent launch (the timed windows' mode): max(first CTA start, previous K3's "
                      "last CTA end) -> last CTA end, so overlapping launches are not double counted (the spans "
                      "sum to less than the step time); bytes = resident activated experts + shared units x image",
            "first_cta_start_span": {"ms_per_launch": float(np.mean(r["k3_span_raw_ms"])) if r["k3_span_raw_ms"] else 0.0,
                                     "frac": (bytes_per_launch / (np.mean(r["k3_span_raw_ms"]) * 1e-3) / 1e9 / hbm_peak)
                                     if r["k3_span_raw_ms"] else 0.0},
            "step_level": {"frac": (r["ffn_bytes_st"] / max(1, r["ffn_launches_st"]) * L_layers(w)
                                    / (r["ms"] / args_steps(args, r) * 1e-3) / 1e9 / hbm_peak)},
            "cuda_events_pdl_off": {"ms_per_launch": ev_ms, "achieved": ev_achieved, "frac": ev_achieved / hbm_peak}}
    stat = lambda v: {"median": float(np.median(v)), "min": float(np.min(v)), "max": float(np.max(v)),  # noqa: E731
                      "spread": float((np.max(v) - np.min(v)) / np.median(v)), "windows": [float(x) for x in v]}
    return tps, tps_e2e, roof, stat


def main():
    global HWB_PROFILE_NAME
    args = parse_args()
    HWB_PROFILE_NAME = args.hwb_profile
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    w = workload(args)
    if world > 1 and args.impl != "reference":  # the CPU reference arm needs no process group
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))

    cfg_json = {"workload": w.description, "config": w.name, "n_layers": w.n_layers, "n_experts": w.n_experts,
                "top_k": w.top_k, "draft_len": w.gamma, "d_model": w.d_model, "d_ffn": w.d_ffn,
                "shared_units": w.n_shared_units, "cache_ratio": w.cache_ratio,
                "parallelism": f"ep{world}" if world > 1 else "single",
                "routing": "model: on-device router GEMV W_g h_l (random-init router), cold path off"
                if args.router_gemv else "trace: reference TraceGenerator logits (K1 top-k on device)",
                "draft": "emulated: gamma x 300 us spin on the compute stream, loads overlapping (reference model)"
                if args.draft_window else "none: verification step only",
                "l2": "inputs > L2: every step streams each resident activated expert (>= 9 MB each, "
                      "GBs per step) through HBM; no L2 flush needed",
                "windows": ("W warm-up steps (+ %d settle steps when cache < 1; their scheduling decisions checked "
                            "against the reference's golden fixture), then " % args.settle
                            + ("one K-step trace window for value, " if w.cache_ratio >= 1.0 or args.router_gemv else
                               "%d K-step windows (value = median; e2e windows interleaved on a second context "
                               "through the same warm-up, median), " % args.budget_windows)
                            + "the next K steps with K3 %globaltimer stamps (roofline), the next with per-K3 CUDA "
                              "events; at a full cache e2e on a fresh context through the same warm-up and window"),
                "hwb_profile": args.hwb_profile,
                "host_arena": "expert (l, e) -> pinned image (l*N + e) %% n_images, n_images >= N + 1 (and >= 8 GiB "
                              "below a full cache): no image shared by the same expert id in consecutive layers"}
    base = {"metric": "decode TPS and expert-FFN HBM GB/s (roofline %) at 1/2/4/8 B200 vs host CPU",
            "unit": "tokens/s", "higher_is_better": True, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "vs_baseline": None, "dtype": "bf16", "data": "synthetic", "config": cfg_json}

    if args.impl == "reference":
        if rank != 0:
            return
        t0 = time.perf_counter()
        vals = []
        for i in range(args.warmup + args.steps):
            r = cpu_path_sample(w, budget_s=max(2.0, args.cpu_budget_s / max(1, args.steps)), use_ref_sched=True)
            if i >= args.warmup:
                vals.append(r)
        v = float(np.mean([r["value"] for r in vals]))
        line = dict(base, impl="reference", value=v, ms_per_step=float(np.mean([r["step_ms"] for r in vals])),
                    scaling="strong",
                    cpu_baseline={"value": v, "unit": "tokens/s", "cores": vals[0]["cores"], "kind": "port",
                                  "sample": vals[0]["sample"]},
                    e2e={"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
                    wall_s=time.perf_counter() - t0)
        print(json.dumps(line), flush=True)
        return

    # Below a full cache the step runs the host cold path on the box's cores,
    # whose scheduling noise moves single windows by 10-60%: the headline is
    # then the median of --budget-windows interleaved windows (value and e2e
    # alike), as in the budget leg.
    head_windows = args.budget_windows if (w.cache_ratio < 1.0 and not args.router_gemv) else 1
    r = run_ours(args, w, rank, world, local_rank, windows=head_windows)
    rd = None
    if args.draft_params > 0 and not args.router_gemv and not args.draft_window:
        rd = run_ours(args, w, rank, world, local_rank, label="draft_verify", draft_params=args.draft_params)
    rb = None
    if world == 1 and not args.no_budget:
        wb = workload_named(args.budget_config, args.budget_cache)
        rb = run_ours(args, wb, rank, world, local_rank, windows=args.budget_windows, label="budget",
                      steps=args.budget_steps)
    if rank != 0:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return
    hbm_peak, peak_kind = load_peaks()
    tps, tps_e2e, roof, stat = leg_summary(r, w, args, world, hbm_peak, peak_kind)
    if world > 1:
        base["config"]["parallelism"] = ("units" if r["parallel_mode"] == "units" else "ep") + str(world)
    vi = int(np.argsort(tps)[len(tps) // 2])  # the median window (the only one at a full cache)
    line = dict(base, value=float(np.median(tps)), ms_per_step=r["win"][vi][0] / args.steps, scaling="strong")
    line["e2e"] = {"value": float(np.median(tps_e2e)), "unit": "tokens/s",
                   "h2d_bytes_per_step": int(r["h2d"]), "d2h_bytes_per_step": int(r["d2h"])}
    if len(tps) > 1:
        line["windows"] = {"value": stat(tps), "e2e": stat(tps_e2e), "interleaved": r["interleaved"],
                           "steps_per_window": args.steps}
    line["roofline"] = roof
    line["gpu_launches"] = int(r["launches"])
    line["clocks"] = r["clocks"]
    line["decision_parity"] = r["parity"]
    line["detail"] = {"hit_rate": r["hits"] / max(1, r["hits"] + r["misses"]), "loads_per_step": r["loads"] / args.steps,
                      "router_ms": r["router_ms"], "hist_ms": r["hist_ms"], "gpu_step_ms": r["gpu_step_ms"],
                      "layers_non_ffn_ms": r["layers_other_ms"], "tokens_per_step": r["tokens"] / args.steps,
                      "ms_per_step_k3_stamps_window": r["ms_st"] / args.steps,
                      "ms_per_step_kernel_events_window": r["ms_ev"] / args.steps,
                      "host_arena_images": r["n_images"],
                      "k3_busy_frac_of_step": float(np.sum(r["k3_span_ms"]) / r["ms_st"]) if r["ms_st"] else None}
    if world == 1 and not args.no_cpu_baseline:
        cb = cpu_path_sample(w, args.cpu_budget_s, use_ref_sched=True)
        line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
    if rd is not None:
        dtps, dtps_e2e, droof, _ = leg_summary(rd, w, args, world, hbm_peak, peak_kind)
        dms = rd["draft_ms_ev"] / args.steps
        dbytes = rd["draft_bytes"] / args.steps
        line["detail"]["draft_verify"] = {
            "value": dtps[0], "e2e": dtps_e2e[0], "unit": "tokens/s", "ms_per_step": rd["ms"] / args.steps,
            "verify_only_value": tps[0],
            "draft": f"dense bf16 draft model, {args.draft_params:.3g} parameters (rows of {args.draft_d}), gamma = "
                     f"{w.gamma} autoregressive passes per step, each one weight-streaming GEMV over all of it, "
                     "on the compute stream before the verification step, expert loads overlapping",
            "draft_ms_per_step": dms, "draft_bytes_per_step": dbytes,
            "draft_gbs": dbytes / (dms * 1e-3) / 1e9 if dms > 0 else None,
            "draft_frac_of_peak": (dbytes / (dms * 1e-3) / 1e9) / hbm_peak if dms > 0 else None,
            "k3_roofline_frac": droof["frac"], "decision_parity": rd["parity"]}
    if rb is not None:
        wb = workload_named(args.budget_config, args.budget_cache)
        btps, btps_e2e, broof, _ = leg_summary(rb, wb, args, world, hbm_peak, peak_kind)
        K = args.budget_steps
        nwin = len(rb["win"])
        budget = {"workload": wb.description, "config": wb.name, "cache_ratio": wb.cache_ratio,
                  "metric": base["metric"], "unit": "tokens/s",
                  "value": stat(btps), "e2e": stat(btps_e2e),
                  "e2e_over_value": float(np.median(btps_e2e) / np.median(btps)),
                  "e2e_over_value_per_window": [float(a / b) for a, b in zip(btps_e2e, btps)],
                  "interleaved": rb["interleaved"],
                  "windows": f"{nwin} windows of {K} consecutive trace steps after {rb['w0']} warm-up + settle steps "
                             f"and {rb['pre']} untimed steps; "
                             "value = device-resident inputs, e2e = moespac_step with pinned host buffers on a second "
                             "context driven through the same warm-up (same cache state, same windows), the two "
                             "windows of each pair run back to back; median / spread over windows (the windows "
                             "differ in routing, hence in misses: spread is workload, not only noise)",
                  "roofline": broof, "decision_parity": rb["parity"], "clocks": rb["clocks"],
                  "hit_rate": rb["hits"] / max(1, rb["hits"] + rb["misses"]),
                  "loads_per_step": rb["loads"] / (nwin * K), "cold_experts_per_step": rb["cold_experts"] / (nwin * K),
                  "staged_experts_per_step": rb["staged_experts"] / (nwin * K),
                  "staging": {"slots": args.stage_slots, "fraction": args.stage_frac},
                  "host_cold_ms_per_step": rb["cpu_ms_cold"] / (nwin * K),
                  # device time inside K3 launches (globaltimer spans, stamps window) over the step time: the
                  # rest of the step the tensor cores / HBM stream idle (host cold path, PCIe, launches)
                  "k3_busy_frac_of_step": float(np.sum(rb["k3_span_ms"]) / rb["ms_st"]) if rb["ms_st"] else None,
                  "gpu_step_ms": rb["gpu_step_ms"], "host_arena_images": rb["n_images"],
                  "e2e_bytes": {"h2d_bytes_per_step": int(rb["h2d"]), "d2h_bytes_per_step": int(rb["d2h"])}}
        if not args.no_cpu_baseline:
            cbb = cpu_path_sample(wb, args.cpu_budget_s, use_ref_sched=True)
            budget["cpu_baseline"] = {k: cbb[k] for k in ("value", "unit", "cores", "kind", "sample")}
        line["detail"]["budget"] = budget
    print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
