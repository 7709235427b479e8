"""Per-layer timeline of one verification step (profiling).

Runs a workload like bench.py (same synthetic model and routing), then one
device step with the K3 trace hook on, and prints per layer: when K3's CTAs
saw their predecessor (the previous combine) complete, the K3 span, and the
gap to the next layer:
    python -m paper_2603_09983_b200.tools.step_trace --config qwen3
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="mixtral")
    ap.add_argument("--cache-ratio", type=float, default=1.0)
    ap.add_argument("--warmup", type=int, default=4)
    ap.add_argument("--pdl", type=int, default=1)
    ap.add_argument("--pf", type=int, default=-1, help="L2 prefetch bytes per CTA (-1: library default)")
    ap.add_argument("--steps", type=int, default=10, help="timed steps (whole-step events)")
    args = ap.parse_args()
    w = configs.CONFIGS[args.config]
    L, N, k, g, d, ffn, T = w.n_layers, w.n_experts, w.top_k, w.gamma, w.d_model, w.d_ffn, w.tokens
    cfg = abi.default_config(n_layers=L, n_experts=N, top_k=k, gamma=g, cache_ratio=args.cache_ratio)
    ctx = abi.Context(0, w.model_desc(), cfg, 0, 1)
    ctx.host_arena(min(L * N, N + 1))
    ctx.fill_synthetic(seed=3, stdv=SYNTH_STD)
    ctx.finalize()
    ctx.set_pdl(bool(args.pdl))
    if args.pf >= 0:
        ctx.set_l2_prefetch(args.pf)
    synth = abi.TraceSynth(cfg)
    S = args.warmup + 1
    logits = torch.empty((S, L, T, N), dtype=torch.float64)
    acc = [synth.next(logits[s].numpy())[1] for s in range(S)]
    logits = logits.cuda()
    h = torch.randn((S, T, d)).to(torch.bfloat16).cuda()
    h_out = torch.empty((T, d), dtype=torch.bfloat16, device="cuda")
    for s in range(args.warmup):
        ctx.step_device(logits[s], h[s], acc[s], h_out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st = torch.cuda.ExternalStream(ctx.stream())
    e0.record(st)
    for i in range(args.steps):
        ctx.step_device(logits[i % args.warmup], h[i % args.warmup], acc[i % args.warmup], h_out)
    e1.record(st)
    torch.cuda.synchronize()
    step_ms = e0.elapsed_time(e1) / args.steps
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    buf = torch.zeros((L, sms, 32), dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    ctx.set_k3_trace(abi.ptr(buf))
    ctx.step_device(logits[S - 1], h[S - 1], acc[S - 1], h_out)
    torch.cuda.synchronize()
    ctx.set_k3_trace(None)
    t = buf.cpu().numpy().astype(np.float64)
    # CTA end = max(slot 6: tid 0 after the final barrier, slot 20: epilogue
    # after its partial-block stores) — ptxas may hoist a %globaltimer read
    # above the barrier
    t[:, :, 6] = np.maximum(t[:, :, 6], t[:, :, 20])
    t0 = t[0, :, 0][t[0, :, 0] > 0].min()
    rows = []
    for l in range(L):
        x = t[l]
        act = x[:, 0] > 0
        if not act.any():
            rows.append({"layer": l, "ctas": 0})
            continue
        ent = (x[act, 0] - t0) / 1e3
        pdl = (x[act, 22] - t0) / 1e3
        end = (x[act, 6] - t0) / 1e3
        rows.append({"layer": l, "ctas": int(act.sum()), "entry_min": round(ent.min(), 2),
                     "pred_done": round(float(np.median(pdl)), 2), "end_med": round(float(np.median(end)), 2),
                     "end_max": round(end.max(), 2)})
    for i, r in enumerate(rows):
        if i + 1 < L and "end_max" in r and "pred_done" in rows[i + 1]:
            r["gap_to_next_us"] = round(rows[i + 1]["pred_done"] - r["end_max"], 2)
            r["k3_span_us"] = round(r["end_max"] - r["pred_done"], 2)
        print(json.dumps(r))
    # K3 tail: per-CTA end (relative to the layer's predecessor-done) vs the
    # CTA's work shape and SM, for a middle layer
    lm = L // 2
    x = t[lm]
    n_hit_l = None
    qpe = ffn // 8  # work units (8 ffn rows) per entry
    base = np.median(x[:, 22])
    ends = (x[:, 6] - base) / 1e3
    first = (x[:, 2] - base) / 1e3
    sm = x[:, 24].astype(int)
    # work shape of every CTA of that layer (the kernel's static split)
    cnt = abi.fetch(ctx.views().counters_dev, (L, 8), np.int32)
    G = x.shape[0]
    n_units = (int(cnt[lm, 7]) + w.n_shared_units) * qpe
    quarters = np.array([((b + 1) * n_units) // G - (b * n_units) // G for b in range(G)])
    segs = []
    for b in range(G):
        q, q1, ns = (b * n_units) // G, ((b + 1) * n_units) // G, 0
        while q < q1:
            q = min((q // 8 + 1) * 8, q1)
            ns += 1
        segs.append(ns)
    segs = np.array(segs)
    for nq in sorted(set(quarters.tolist())):
        m = quarters == nq
        rel_med = {str(j): round(float(np.median((x[m, j] - base) / 1e3)), 2) for j in (2, 3, 31, 5, 11, 15, 17, 25, 16, 21, 4, 18, 7, 1, 19, 20)
                   if (x[m, j] > 0).all()}
        print(json.dumps({"layer": lm, "units": nq, "ctas": int(m.sum()),
                          "end_us_med": round(float(np.median(ends[m])), 2),
                          "end_us_max": round(float(ends[m].max()), 2),
                          "segs_mean": round(float(segs[m].mean()), 2),
                          "stamps_rel_pred_med": rel_med,
                          "waits_cycles_med": {nm: float(np.median(x[m, j])) for j, nm in
                                               [(8, "prod_ring_full"), (9, "mma_data"), (10, "mma_aT"),
                                                (13, "epi_d1"), (14, "epi_d2")]}}))
    # end time by the CTA's start offset inside its first chunk (unit % 8)
    # and its number of chunk pieces
    by_shape = {}
    for b in range(G):
        q0 = (b * n_units) // G
        key = f"start%8={q0 % 8},pieces={segs[b]}"
        by_shape.setdefault(key, []).append(float(ends[b]))
    print(json.dumps({"layer": lm, "end_us_by_shape": {k_: [len(v), round(float(np.median(v)), 2), round(max(v), 2)]
                                                       for k_, v in sorted(by_shape.items())}}))
    # per-segment GU-issued stamps (per-segment K3 only: slots 15,19,23,25,31)
    gu = {}
    for b in range(G):
        q0 = (b * n_units) // G
        key = f"start%8={q0 % 8},pieces={segs[b]}"
        row = [round(float((x[b, j] - base) / 1e3), 2) for j in (15, 19, 23, 25, 31) if x[b, j] > 0]
        gu.setdefault(key, []).append(row)
    print(json.dumps({"layer": lm, "gu_issued_us_by_shape_first": {k_: v[0] for k_, v in sorted(gu.items())}}))
    print(json.dumps({"layer": lm, "end_pct_us": [round(float(np.percentile(ends, p)), 2) for p in (0, 10, 50, 90, 100)],
                      "first_data_pct_us": [round(float(np.percentile(first, p)), 2) for p in (0, 50, 100)],
                      "slowest_ctas": [[int(b), int(sm[b]), round(float(ends[b]), 2)] for b in np.argsort(-ends)[:8]],
                      "fastest_ctas": [[int(b), int(sm[b]), round(float(ends[b]), 2)] for b in np.argsort(ends)[:8]]}))
    # where the K3 roles waited (clock64 cycles accumulated in debug slots
    # 8-14) as a fraction of the CTA's lifetime, median over CTAs, plus the
    # part of the lifetime after the predecessor wait
    life_ns = x[:, 6] - x[:, 0]
    cyc = np.maximum(life_ns * 1.965, 1.0)  # ns -> SM cycles at the boost clock
    act_m = x[:, 0] > 0
    waits = {nm: round(float(np.median(x[act_m, j] / cyc[act_m])), 3) for j, nm in
             [(8, "producer_ring_full"), (9, "mma_wait_data"), (10, "mma_wait_aT"), (12, "mma_wait_d1_free"),
              (13, "epi_wait_d1"), (14, "epi_wait_d2")]}
    post = (x[act_m, 6] - x[act_m, 22]) / 1e3
    print(json.dumps({"layer": lm, "wait_frac_of_cta_life": waits,
                      "cta_life_us_med": round(float(np.median(life_ns[act_m])) / 1e3, 2),
                      "after_pred_us_pct": [round(float(np.percentile(post, p_)), 2) for p_ in (0, 50, 100)]}))
    # per-SM lateness across layers: is the tail a property of the SM?
    late = {}
    for l in range(L):
        x = t[l]
        if not (x[:, 0] > 0).all():
            continue
        e = (x[:, 6] - np.median(x[:, 22])) / 1e3
        rel = e / np.median(e) - 1.0
        for b in range(x.shape[0]):
            late.setdefault(int(x[b, 24]), []).append(float(rel[b]))
    sm_mean = {s_: float(np.mean(v)) for s_, v in late.items()}
    order = sorted(sm_mean, key=lambda s_: -sm_mean[s_])
    allv = np.concatenate([np.array(v) for v in late.values()])
    print(json.dumps({"per_sm_lateness": {"std_all": round(float(allv.std()), 4),
                                          "std_of_sm_means": round(float(np.std(list(sm_mean.values()))), 4),
                                          "latest_sms": [[s_, round(sm_mean[s_], 4)] for s_ in order[:10]],
                                          "earliest_sms": [[s_, round(sm_mean[s_], 4)] for s_ in order[-10:]]}}))
    # layer handoff per SM: next layer's K3 CTA entry / predecessor-done on the
    # same SM minus this layer's K3 CTA end there
    x0, x1 = t[lm], t[lm + 1] if lm + 1 < L else None
    if x1 is not None and (x0[:, 24] != x1[:, 24]).any() or True:
        end_by_sm = {int(x0[b_, 24]): x0[b_, 6] for b_ in range(x0.shape[0]) if x0[b_, 6] > 0}
        ent, prd = [], []
        for b_ in range(x1.shape[0]):
            s_ = int(x1[b_, 24])
            if s_ in end_by_sm and x1[b_, 0] > 0:
                ent.append((x1[b_, 0] - end_by_sm[s_]) / 1e3)
                prd.append((x1[b_, 22] - end_by_sm[s_]) / 1e3)
        lend = (x0[:, 6].max() - x0[:, 6]) / 1e3
        print(json.dumps({"layer": lm, "next_entry_minus_sm_end_us_pct": [round(float(np.percentile(ent, p_)), 2) for p_ in (0, 10, 50, 90, 100)],
                          "next_pred_minus_sm_end_us_pct": [round(float(np.percentile(prd, p_)), 2) for p_ in (0, 10, 50, 90, 100)],
                          "layer_end_max_minus_cta_end_pct": [round(float(np.percentile(lend, p_)), 2) for p_ in (0, 50, 100)]}))
    # combine CTAs of that layer (slots 26-29 of the same rows): start, after
    # their predecessor wait, end — relative to this layer's last K3 CTA end
    cb = t[lm][:, 26] > 0
    if cb.any():
        kend = t[lm][:, 6].max()
        rel = lambda j: [round(float(np.percentile((t[lm][cb, j] - kend) / 1e3, p_)), 2) for p_ in (0, 50, 100)]
        xs = t[lm]
        print(json.dumps({"layer": lm, "slot_minus_end_us_med": {str(j): round(float(np.median((xs[xs[:, j] > 0, j] - xs[xs[:, j] > 0, 6]) / 1e3)), 2)
                                                                for j in (0, 2, 3, 4, 17, 18, 19, 20, 21, 22, 23, 25) if (xs[:, j] > 0).any()}}))
        dz = t[lm][:, 23] > 0
        if dz.any():
            print(json.dumps({"layer": lm, "dealloc_minus_end_us_pct": [round(float(np.percentile((t[lm][dz, 23] - t[lm][dz, 6]) / 1e3, p_)), 2) for p_ in (0, 50, 100)]}))
        cs = t[lm][:, 30] > 0
        print(json.dumps({"layer": lm, "combine_ctas": int(cb.sum()), "combine_start_rel_k3_end": rel(26),
                          "combine_pred_rel_k3_end": rel(27), "combine_sums_rel_k3_end": rel(28),
                          "combine_stored_rel_k3_end": [round(float(np.percentile((t[lm][cs, 30] - kend) / 1e3, p_)), 2)
                                                        for p_ in (0, 50, 100)] if cs.any() else None}))
    gaps = [r["gap_to_next_us"] for r in rows if "gap_to_next_us" in r]
    spans = [r["k3_span_us"] for r in rows if "k3_span_us" in r]
    print(json.dumps({"config": args.config, "pf": args.pf, "timed_step_ms": round(step_ms, 4),
                      "median_gap_us": float(np.median(gaps)),
                      "median_k3_span_us": float(np.median(spans)),
                      "step_us": round(rows[-1]["end_max"] - rows[0]["pred_done"], 2)}))


if __name__ == "__main__":
    main()
