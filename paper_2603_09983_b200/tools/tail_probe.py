"""K3 tail probe (profiling): is the per-CTA end-time spread of one launch a
property of the CTA's work (its bytes / addresses), of the SM it lands on,
or run-to-run noise?

Launches the same K3 (same routing, same expert slots) R times with the
per-CTA globaltimer hook on and correlates each CTA's lateness across runs,
by CTA index and by SM:
    python -m paper_2603_09983_b200.tools.tail_probe --d 2048 --ffn 768 --T 9 --k 8 --experts 16
"""
import argparse
import ctypes
import json

import numpy as np
import torch

from paper_2603_09983_b200 import abi


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--d", type=int, default=2048)
    ap.add_argument("--ffn", type=int, default=768)
    ap.add_argument("--T", type=int, default=9)
    ap.add_argument("--k", type=int, default=8)
    ap.add_argument("--N", type=int, default=128)
    ap.add_argument("--experts", type=int, default=16)
    ap.add_argument("--runs", type=int, default=12)
    ap.add_argument("--kernel", type=int, default=2)
    ap.add_argument("--accum", type=int, default=0)
    ap.add_argument("--shuffle-slots", action="store_true", help="expert e -> a random pool slot")
    args = ap.parse_args()
    d, ffn, T, k, N = args.d, args.ffn, args.T, args.k, args.N
    dev = torch.device("cuda")
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    img = 3 * d * ffn
    pool = torch.empty(N * img, dtype=torch.int16, device=dev)
    abi.check(abi.lib().moespac_fill_synthetic(abi.ptr(pool), pool.numel(), 7, 0.02, abi._stream(None)))
    h = torch.randn(T, d, device=dev).to(torch.bfloat16).view(torch.int16)
    hT = abi.build_hT(h)
    ws = torch.empty(abi.lib().moespac_ffn_workspace_bytes(T, d, N, 0, sms) // 4, device=dev)
    perm_slots = np.random.default_rng(5).permutation(N) if args.shuffle_slots else np.arange(N)
    slot_of = torch.tensor(perm_slots, dtype=torch.int32, device=dev)
    ne = args.experts
    ids = torch.tensor([sorted({(t * k + j) % ne for j in range(k)}) for t in range(T)], dtype=torch.int32)
    kk = ids.shape[1]
    ids = ids.to(dev)
    gates = torch.full((T, kk), 1.0 / kk, device=dev)
    bufs = {n: torch.zeros(s, dtype=torch.int32, device=dev) for n, s in
            [("freqs", N), ("offsets", N + 1), ("perm", T * kk), ("hl", N), ("ho", N), ("cnt", 8), ("sc", N)]}
    rb = torch.full(((N + 31) // 32,), -1, dtype=torch.int32, device=dev)
    taus = torch.ones(1, dtype=torch.int32, device=dev)
    st = torch.zeros((N, 4), dtype=torch.int32, device=dev)
    a2 = abi.K2Args(abi.ptr(ids), 1, T, kk, N, abi.ptr(rb), None, abi.ptr(taus), abi.ptr(st), 4, 1, 0.1, 0, 1,
                    abi.ptr(bufs["freqs"]), abi.ptr(bufs["offsets"]), abi.ptr(bufs["perm"]),
                    abi.ptr(bufs["hl"]), abi.ptr(bufs["ho"]), abi.ptr(bufs["cnt"]), abi.ptr(bufs["sc"]))
    abi.check(abi.lib().moespac_hist_scan_observe(ctypes.byref(a2), abi._stream(None)))
    torch.cuda.synchronize()
    fa = abi.FfnArgs(abi.ptr(h), T, d, ffn, kk, N, abi.ptr(bufs["perm"]), abi.ptr(bufs["offsets"]),
                     abi.ptr(gates), abi.ptr(bufs["hl"]), abi.ptr(bufs["cnt"]), abi.ptr(slot_of),
                     abi.ptr(pool), None, 0, abi.ptr(ws), sms, args.kernel, abi.ptr(hT), None, args.accum, 0)
    for _ in range(3):
        abi.check(abi.lib().moespac_expert_ffn(ctypes.byref(fa), abi._stream(None)))
    dbg = torch.zeros((sms, 32), dtype=torch.int64, device=dev)
    ends, starts, smid = [], [], []
    for _ in range(args.runs):
        dbg.zero_()
        fa.debug_ts_dev = abi.ptr(dbg)
        abi.check(abi.lib().moespac_expert_ffn(ctypes.byref(fa), abi._stream(None)))
        torch.cuda.synchronize()
        t = dbg.cpu().numpy().astype(np.float64)
        end = np.maximum(t[:, 6], t[:, 20])
        t0 = t[:, 0][t[:, 0] > 0].min()
        starts.append((t[:, 0] - t0) / 1e3)
        ends.append((end - t0) / 1e3)
        smid.append(t[:, 24].astype(int))
    fa.debug_ts_dev = None
    E = np.array(ends)          # [runs][ctas]
    S = np.array(smid)
    lat = E - np.median(E, axis=1, keepdims=True)
    # by CTA index: correlation of lateness between consecutive runs
    cta_corr = float(np.mean([np.corrcoef(lat[r], lat[r + 1])[0, 1] for r in range(len(lat) - 1)]))
    # by SM: lateness of whatever CTA ran on SM s
    by_sm = np.full((len(lat), sms), np.nan)
    for r in range(len(lat)):
        by_sm[r, S[r]] = lat[r]
    sm_corr = float(np.nanmean([np.corrcoef(by_sm[r], by_sm[r + 1])[0, 1] for r in range(len(lat) - 1)]))
    mean_cta = lat.mean(axis=0)
    mean_sm = np.nanmean(by_sm, axis=0)
    same_sm = float(np.mean([(S[r] == S[0]).mean() for r in range(len(S))]))
    print(json.dumps({
        "experts": ne, "runs": args.runs, "cta_to_sm_same_as_run0": round(same_sm, 3),
        "spread_us_per_run": [round(float(e.max() - np.median(e)), 2) for e in E],
        "start_spread_us": round(float(np.median([s.max() for s in starts])), 2),
        "end_med_us": round(float(np.median(E)), 2),
        "corr_lateness_same_cta": round(cta_corr, 3), "corr_lateness_same_sm": round(sm_corr, 3),
        "std_lateness_us": round(float(lat.std()), 2),
        "std_of_cta_means_us": round(float(mean_cta.std()), 2), "std_of_sm_means_us": round(float(np.nanstd(mean_sm)), 2),
        "latest_ctas": [[int(b), round(float(mean_cta[b]), 2)] for b in np.argsort(-mean_cta)[:10]],
        "earliest_ctas": [[int(b), round(float(mean_cta[b]), 2)] for b in np.argsort(mean_cta)[:10]],
        "latest_sms": [[int(s), round(float(mean_sm[s]), 2)] for s in np.argsort(-np.nan_to_num(mean_sm, nan=-1e9))[:10]],
        "earliest_sms": [[int(s), round(float(mean_sm[s]), 2)] for s in np.argsort(np.nan_to_num(mean_sm, nan=1e9))[:10]],
    }))
    # lateness by SM id bucket (die / GPC guesses)
    bucket = {}
    for r in range(len(lat)):
        for b in range(sms):
            bucket.setdefault(int(S[r, b]) // 16, []).append(float(lat[r, b]))
    print(json.dumps({"lateness_by_smid_16": {k_: round(float(np.mean(v)), 2) for k_, v in sorted(bucket.items())}}))
    # lateness vs CTA index bucket (address order of the work)
    cb = {}
    for b in range(sms):
        cb.setdefault(b // 16, []).append(float(mean_cta[b]))
    print(json.dumps({"lateness_by_cta_16": {k_: round(float(np.mean(v)), 2) for k_, v in sorted(cb.items())}}))


if __name__ == "__main__":
    main()
