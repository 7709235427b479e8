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
  roofline: K3 (expert_ffn_kernel) algorithmic bytes / its CUDA-event time
  cpu_baseline: the CPU oracle port of the same step on the box's cores

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
    ap.add_argument("--trace-steps", type=int, default=160)
    ap.add_argument("--settle", type=int, default=20,
                    help="extra untimed steps before the timed windows when the cache budget is < 1 "
                         "(the warm fill holds experts 0..cap-1, not the hot ones)")
    ap.add_argument("--ffn-kernel", type=int, default=0, help="0 auto (tcgen05), 1 CUDA-core GEMV, 2 tcgen05")
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


def workload(args):
    from paper_2603_09983_b200.configs import CONFIGS
    w = CONFIGS[args.config]
    if args.cache_ratio is not None:
        w = w.with_(cache_ratio=args.cache_ratio)
    return w


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
        cfg = O.default_config(n_layers=L, n_experts=N, top_k=k, gamma=g, cache_ratio=w.cache_ratio, token_budget=0)
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
def run_ours(args, w, rank, world, local_rank):
    import torch

    from paper_2603_09983_b200 import abi

    torch.cuda.set_device(local_rank)
    L, N, k, g, d, ffn, T = w.n_layers, w.n_experts, w.top_k, w.gamma, w.d_model, w.d_ffn, w.tokens
    cfg = abi.default_config(n_layers=L, n_experts=N, top_k=k, gamma=g, cache_ratio=w.cache_ratio)
    model = abi.ModelDesc(L, N, k, g, d, ffn, w.n_shared_units, w.gate_mode, args.ffn_kernel)

    def make_ctx():
        c = abi.Context(local_rank, model, cfg, rank, world)
        c.host_arena(min(L * N, max(N, 8)))
        c.fill_synthetic(seed=3, stdv=0.02)
        if args.router_gemv:
            c.set_cold_threads(0)
        c.finalize()
        if args.draft_window:
            c.set_draft_window(True)
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
    # synthetic inputs: routing from the trace synthesizer (reference
    # TraceGenerator semantics), hidden states ~ N(0, 1) bf16.
    # Trace steps: W warm-up (+ settle steps when the cache budget is < 1),
    # then one window of K steps that the device-resident value, the
    # end-to-end run and the per-kernel timing run all use. Below a full
    # cache the end-to-end run gets a fresh context driven through the same
    # warm-up, so it starts from the same cache and estimator state instead
    # of replaying routing the cache has already adapted to.
    settle = args.settle if w.cache_ratio < 1.0 else 0
    w0 = args.warmup + settle
    S = min(args.trace_steps, w0 + args.steps)
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

    def timed(fn, n, offset):
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        stream = torch.cuda.ExternalStream(ctx.stream())
        reps = []
        e0.record(stream)
        for i in range(n):
            reps.append(fn((offset + i) % S))
        e1.record(stream)
        barrier()
        ms = e0.elapsed_time(e1)
        if world > 1:
            import torch.distributed as dist
            t = torch.tensor([ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms, reps

    dev_step = lambda s: ctx.step_device(logits_d[s], h_d[s], accepted[s], h_out_d)[0]  # noqa: E731
    host_step = lambda s: ctx.step(logits_h[s].numpy(), h_h[s].view(torch.int16).numpy(), accepted[s],  # noqa: E731
                                   h_out_h.view(torch.int16).numpy())[0]
    if args.router_gemv:
        dev_step = lambda s: ctx.step_model_device(h_d[s], accepted[s], h_out_d)[0]  # noqa: E731
        host_step = lambda s: ctx.step_model(h_h[s].view(torch.int16).numpy(), accepted[s],  # noqa: E731
                                             h_out_h.view(torch.int16).numpy())[0]
    for i in range(w0):
        dev_step(i % S)
    K = args.steps
    with ClockSampler(local_rank) as clk:
        # (1) headline: whole steps, no per-kernel events (layer kernels use
        #     programmatic dependent launch)
        ctx.set_timing(False)
        ms, reps = timed(dev_step, K, w0)
        # (2) end to end through the host API, same window
        if settle:
            ctx.close()
            ctx = make_ctx()  # (the step lambdas look ctx up at call time)
            for i in range(w0):
                host_step(i % S)
        else:
            for i in range(max(1, args.warmup // 2)):
                host_step(i % S)
        ms_e2e, reps_e2e = timed(host_step, K, w0)
        # (3) roofline: the window again with a CUDA-event pair around every
        #     K3 launch (PDL off so each pair brackets exactly one kernel)
        ctx.set_timing(True)
        ms_t, reps_t = timed(dev_step, K, w0)
    reps_tok = reps
    reps = reps_t
    tokens = float(sum(accepted[(w0 + i) % S] for i in range(K)))
    tokens_e2e = tokens
    ffn_ms = sum(r.gpu_ms_ffn for r in reps)
    ffn_bytes = sum(r.ffn_bytes for r in reps)
    launches = sum(r.kernel_launches for r in reps_tok)
    hits = sum(r.cache_hits for r in reps)
    misses = sum(r.cache_misses for r in reps)
    loads = sum(r.n_loads for r in reps)
    out = {
        "ms": ms, "ms_e2e": ms_e2e, "ms_timed": ms_t, "tokens": tokens, "tokens_e2e": tokens_e2e,
        "settle": settle, "ffn_ms": ffn_ms, "ffn_bytes": ffn_bytes,
        "ffn_launches": sum(r.ffn_launches for r in reps), "launches": launches, "hits": hits, "misses": misses, "loads": loads,
        "k3_kernel": ctx.k3_kernel(), "parallel_mode": ctx.parallel_mode(),
        "h2d": float(np.mean([r.h2d_bytes for r in reps_e2e])), "d2h": float(np.mean([r.d2h_bytes for r in reps_e2e])),
        "router_ms": float(np.mean([r.gpu_ms_router for r in reps])),
        "hist_ms": float(np.mean([r.gpu_ms_hist for r in reps])),
        "gpu_step_ms": float(np.mean([r.gpu_ms_total for r in reps])),
        "layers_other_ms": float(np.mean([r.gpu_ms_combine for r in reps])),
        "clocks": clk.summary(),
    }
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ffn_ms, ffn_bytes], dtype=torch.float64, device="cuda")
        # aggregate K3 bytes and time over ranks (bytes sum, time max)
        tb = t.clone()
        dist.all_reduce(tb, op=dist.ReduceOp.SUM)
        out["ffn_bytes_all"] = float(tb[1].item())
    ctx.close()
    return out


def main():
    args = parse_args()
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
                "windows": "W warm-up steps (+ %d settle steps when cache < 1), then one K-step trace window "
                           "for value, e2e (below a full cache: a fresh context through the same warm-up) and the "
                           "per-K3-event timing" % args.settle}
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

    r = run_ours(args, w, rank, world, local_rank)
    if rank != 0:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return
    hbm_peak, peak_kind = load_peaks()
    tps = r["tokens"] / (r["ms"] * 1e-3)
    achieved = r["ffn_bytes"] / (r["ffn_ms"] * 1e-3) / 1e9 if r["ffn_ms"] > 0 else 0.0
    # DRAM traffic of one K3 launch from a committed `ncu --set full`
    # capture (profiles/ncu_k3_<config>.json), expressed for this run's
    # average launch: captured DRAM bytes / captured algorithmic bytes x
    # this run's algorithmic bytes per launch (the capture's launch streams
    # a different number of experts than the average one)
    traffic, traffic_capture = None, None
    prof = os.path.join(ROOT, "profiles", f"ncu_k3_{w.name}.json")
    if os.path.exists(prof):
        try:
            cap = json.load(open(prof))
            ratio = cap.get("traffic_over_algorithmic")
            bpl = r["ffn_bytes"] / max(1, r["ffn_launches"])
            traffic = ratio * bpl if ratio else None
            traffic_capture = {"dram_bytes": cap.get("dram_bytes_per_launch"),
                               "algorithmic_bytes": cap.get("algorithmic_bytes_of_launch"), "ratio": ratio,
                               "kernel": cap.get("kernel"), "report": cap.get("report")}
        except (ValueError, OSError, TypeError):
            traffic = None
    if world > 1:
        base["config"]["parallelism"] = ("units" if r["parallel_mode"] == "units" else "ep") + str(world)
    line = dict(base, value=tps, ms_per_step=r["ms"] / args.steps, scaling="strong")
    line["e2e"] = {"value": r["tokens_e2e"] / (r["ms_e2e"] * 1e-3), "unit": "tokens/s",
                   "h2d_bytes_per_step": int(r["h2d"]), "d2h_bytes_per_step": int(r["d2h"])}
    line["roofline"] = {"bound": "hbm", "kernel": r["k3_kernel"], "achieved": achieved, "peak": hbm_peak,
                        "peak_source": f"{peak_kind} hbm_gbs (MEASURED_PEAKS.json)" if peak_kind == "measured"
                        else "fallback 6650 GB/s (B200_PROFILING.md)",
                        "unit": "GB/s", "frac": achieved / hbm_peak, "traffic": traffic,
                        "traffic_capture": traffic_capture,
                        "bytes_per_launch": r["ffn_bytes"] / max(1, r["ffn_launches"]),
                        "ms_per_launch": r["ffn_ms"] / max(1, r["ffn_launches"])}
    line["gpu_launches"] = int(r["launches"])
    line["clocks"] = r["clocks"]
    line["detail"] = {"hit_rate": r["hits"] / max(1, r["hits"] + r["misses"]), "loads_per_step": r["loads"] / args.steps,
                      "router_ms": r["router_ms"], "hist_ms": r["hist_ms"], "gpu_step_ms": r["gpu_step_ms"],
                      "layers_non_ffn_ms": r["layers_other_ms"],
                      "ffn_ms_per_step": r["ffn_ms"] / args.steps, "tokens_per_step": r["tokens"] / args.steps,
                      "ms_per_step_with_kernel_events": r["ms_timed"] / args.steps}
    if world == 1 and not args.no_cpu_baseline:
        cb = cpu_path_sample(w, args.cpu_budget_s, use_ref_sched=True)
        line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
    print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
