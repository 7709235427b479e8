"""Cache-budget sweep (BASELINE.json configs[4]: Qwen3-30B-A3B shape, 128
experts top-8, cache budget 10-100% with async prefetch).

For each cache ratio: the same synthetic model and routing as bench.py, K
timed verification steps through the engine (device-resident inputs, CUDA
events on the engine's stream, programmatic dependent launch on), then K
steps with per-kernel/copy-stream timing for the breakdown. Prints one JSON
line per ratio — TPS, hit rate, expert loads per step and their pinned
H2D GB/s, cold (host-computed) experts per step and host ms — and writes the
sweep in the reference's `#moesim-metrics v1` JSONL schema (axis
`cache_ratio`; one RunSummary per ratio, from moespac_summarize over the
measured steps) to --metrics:

    python -m paper_2603_09983_b200.tools.cache_sweep --config qwen3 \\
        --ratios 0.1,0.17,0.25,0.5,0.75,1.0 --metrics gpurun_out/sweep.jsonl
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2603_09983_b200 import abi, configs  # noqa: E402
from paper_2603_09983_b200.configs import SYNTH_STD  # noqa: E402


def run_ratio(w, ratio, steps, warmup, cold_threads, profile, draft=False):
    L, N, k, g, d, ffn, T = w.n_layers, w.n_experts, w.top_k, w.gamma, w.d_model, w.d_ffn, w.tokens
    cfg = abi.default_config(n_layers=L, n_experts=N, top_k=k, gamma=g, cache_ratio=ratio, **profile)
    ctx = abi.Context(0, w.model_desc(), cfg, 0, 1)
    ctx.host_arena(min(L * N, N + 1))
    ctx.fill_synthetic(seed=3, stdv=SYNTH_STD)
    ctx.set_cold_threads(cold_threads)
    ctx.finalize()
    ctx.set_draft_window(draft)
    synth = abi.TraceSynth(cfg)
    S = warmup + 2 * steps
    logits = torch.empty((S, L, T, N), dtype=torch.float64)
    acc = [synth.next(logits[s].numpy())[1] for s in range(S)]
    # the timed window and the breakdown window use the same trace steps
    for s in range(warmup + steps, S):
        logits[s] = logits[s - steps]
        acc[s] = acc[s - steps]
    logits = logits.cuda()
    gen = torch.Generator().manual_seed(2)
    h = torch.randn((S, T, d), generator=gen).to(torch.bfloat16).cuda()
    h_out = torch.empty((T, d), dtype=torch.bfloat16, device="cuda")
    for s in range(warmup):
        ctx.step_device(logits[s], h[s], acc[s], h_out)
    st = torch.cuda.ExternalStream(ctx.stream())
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    reps = [ctx.step_device(logits[s], h[s], acc[s], h_out)[0] for s in range(warmup, warmup + steps)]
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    tokens = sum(acc[warmup:warmup + steps])
    ctx.set_timing(True)
    timed = [ctx.step_device(logits[s], h[s], acc[s], h_out) for s in range(warmup + steps, S)]
    ctx.set_timing(False)
    trep = [r for r, _ in timed]
    # RunSummary of the timed window: the reference's accounting of the
    # steps, with its (modeled) clock replaced by the measured device time
    summary, series = abi.summarize(reps, None)
    summary.axis_name = b"cache_ratio"
    summary.axis_value = ratio
    summary.total_time_ns = int(round(ms * 1e6))
    summary.latency_s = ms * 1e-3
    summary.tps = tokens / (ms * 1e-3)
    img = 3 * d * ffn * 2
    loads = sum(r.n_loads for r in trep)
    h2d_ms = sum(r.gpu_ms_h2d_loads for r in trep)
    hits = sum(r.cache_hits for r in reps)
    misses = sum(r.cache_misses for r in reps)
    line = {"config": w.name, "cache_ratio": ratio, "slots_per_layer": ctx.views().slots_per_layer,
            "tps": tokens / (ms * 1e-3), "ms_per_step": ms / steps,
            "hit_rate": hits / max(1, hits + misses), "loads_per_step": loads / len(trep),
            "h2d_GBps": loads * img / (h2d_ms * 1e-3) / 1e9 if h2d_ms > 0 else None,
            "h2d_ms_per_step": h2d_ms / len(trep),
            "cold_experts_per_step": sum(r.cold_experts for r in trep) / len(trep),
            "cold_host_ms_per_step": sum(r.cpu_ms_cold for r in trep) / len(trep),
            "k3_ms_per_step": sum(r.gpu_ms_ffn for r in trep) / len(trep),
            "cold_threads": cold_threads, "draft_window": draft,
            "profile_ns": profile or "reference defaults (config.cpp:23-27)"}
    ctx.close()
    return line, summary, series


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="qwen3")
    ap.add_argument("--ratios", default="0.1,0.17,0.25,0.5,0.75,1.0")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=4)
    ap.add_argument("--cold-threads", type=int, default=-1, help="host threads for misses (-1 all, 0 off)")
    ap.add_argument("--metrics", default="", help="write the sweep as #moesim-metrics v1 JSONL here")
    ap.add_argument("--t-cpu-ns", type=int, default=0, help="HWB profile override: host time per miss token")
    ap.add_argument("--t-gpu-ns", type=int, default=0, help="HWB profile override: device time per hit expert")
    ap.add_argument("--t-io-ns", type=int, default=0, help="HWB profile override: load time per expert")
    ap.add_argument("--draft-window", action="store_true", help="emulated gamma x t_draft window before each step")
    args = ap.parse_args()
    w = configs.CONFIGS[args.config]
    sums, series = [], []
    profile = {k: v for k, v in (("t_cpu_unit_ns", args.t_cpu_ns), ("t_gpu_unit_ns", args.t_gpu_ns),
                                 ("t_io_unit_ns", args.t_io_ns)) if v > 0}
    for r in [float(x) for x in args.ratios.split(",")]:
        line, s, ser = run_ratio(w, r, args.steps, args.warmup, args.cold_threads, profile, args.draft_window)
        print(json.dumps(line), flush=True)
        sums.append(s)
        series.append(ser)
    if args.metrics:
        abi.metrics_emit(args.metrics, sums, series, "jsonl")


if __name__ == "__main__":
    main()
