"""K3 microbenchmark: time vs number of activated resident experts.

Separates the per-launch fixed cost from the streaming bandwidth of the
expert-FFN kernels (both variants) through the stateless C ABI:
    python -m paper_2603_09983_b200.tools.k3_sweep --d 2048 --ffn 768 --T 9
Prints one JSON line per (kernel, n_experts).
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
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--experts", default="1,2,4,8,16,32,64,128")
    ap.add_argument("--kernels", default="2,1")
    ap.add_argument("--accum", type=int, default=0)
    ap.add_argument("--l2", type=int, default=0)
    ap.add_argument("--grid", type=int, default=0, help="CTAs (0: one per SM)")
    ap.add_argument("--stamps", action="store_true", help="dump per-CTA timeline (tensor-core kernel)")
    ap.add_argument("--dump", default="", help="save the raw per-CTA stamp array (.npy prefix)")
    args = ap.parse_args()
    d, ffn, T, k, N = args.d, args.ffn, args.T, args.k, args.N
    dev = torch.device("cuda")
    sms = args.grid or torch.cuda.get_device_properties(0).multi_processor_count
    img = 3 * d * ffn
    pool = torch.empty(N * img, dtype=torch.int16, device=dev)
    abi.check(abi.lib().moespac_fill_synthetic(abi.ptr(pool), pool.numel(), 7, 0.02, abi._stream(None)))
    h = (torch.randn(T, d, device=dev) * 1.0).to(torch.bfloat16).view(torch.int16)
    hT = abi.build_hT(h)
    ws = torch.empty(abi.lib().moespac_ffn_workspace_bytes(T, d, N, 0, sms) // 4, device=dev)
    slot_of = torch.arange(N, dtype=torch.int32, device=dev)
    for kern in [int(x) for x in args.kernels.split(",")]:
        if abi.ffn_resolve(kern, d, ffn) != kern:
            continue
        for ne in [int(x) for x in args.experts.split(",")]:
            ne = min(ne, N)
            # routing: token t picks experts (t*k + j) % ne -> min(ne, T*k) distinct
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
            n_hit = int(bufs["cnt"][7].item())
            fa = abi.FfnArgs(abi.ptr(h), T, d, ffn, kk, N, abi.ptr(bufs["perm"]), abi.ptr(bufs["offsets"]),
                             abi.ptr(gates), abi.ptr(bufs["hl"]), abi.ptr(bufs["cnt"]), abi.ptr(slot_of),
                             abi.ptr(pool), None, 0, abi.ptr(ws), sms, kern, abi.ptr(hT), None, args.accum, args.l2)
            for _ in range(3):
                abi.check(abi.lib().moespac_expert_ffn(ctypes.byref(fa), abi._stream(None)))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            # back-to-back launches (as in the engine): host-side call overhead
            # overlaps device execution and drops out of the average
            torch.cuda.synchronize()
            e0.record()
            for _ in range(args.iters):
                abi.check(abi.lib().moespac_expert_ffn(ctypes.byref(fa), abi._stream(None)))
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / args.iters
            byts = n_hit * img * 2
            if args.stamps and kern == 2:
                dbg = torch.zeros((sms, 32), dtype=torch.int64, device=dev)
                fa.debug_ts_dev = abi.ptr(dbg)
                abi.check(abi.lib().moespac_expert_ffn(ctypes.byref(fa), abi._stream(None)))
                torch.cuda.synchronize()
                fa.debug_ts_dev = None
                if args.dump:
                    np.save(f"{args.dump}_e{n_hit}.npy", dbg.cpu().numpy())
                t = dbg.cpu().numpy().astype("float64")
                act = t[:, 1] > 0
                t0 = t[act, 0].min()
                rel = (t[act] - t0) / 1e3
                rel[t[act] == 0] = float("nan")
                rel = np.concatenate([rel[:, :7], rel[:, 16:22]], axis=1)
                names = ["entry", "prologue", "first_data", "gu0_issued", "a0_ready", "epi_done", "end",
                         "dn0_data", "dn0_issued", "d2_pass0", "d2_pass1", "dn0_drained", "dn0_flushed"]
                summ = {nm: [round(float(np.nanmin(rel[:, j])), 2), round(float(np.nanmedian(rel[:, j])), 2),
                             round(float(np.nanmax(rel[:, j])), 2)] for j, nm in enumerate(names)}
                cyc = t[act, 7]
                waits = {nm: round(float(np.median(t[act, j] / np.maximum(cyc, 1))), 3) for j, nm in
                         [(8, "prod_empty"), (9, "mma_full"), (10, "mma_at_full"), (11, "mma_d2_empty"),
                          (12, "mma_d1_empty"), (13, "epi_d1_full"), (14, "epi_d2_full")]}
                print(json.dumps({"wait_frac_of_cta_cycles": waits,
                                  "drain_cycles_med": {nm: float(np.median(t[act, j])) for j, nm in
                                                       [(25, "tmem_ld"), (26, "lds"), (27, "sts")]}}), flush=True)
                # end time vs the CTA's number of chunk pieces (8-row units,
                # 8 units per 64-row chunk) and its start offset in a chunk
                qpe = ffn // 8
                n_q = n_hit * qpe
                by = {}
                gu_rows = {}
                waits_by = {}
                cyc_all = t[:, 7]
                ends = (t[:, 6] - t0) / 1e3
                for b in range(sms):
                    q0, q1 = b * n_q // sms, (b + 1) * n_q // sms
                    if q0 >= q1 or t[b, 6] == 0:
                        continue
                    nseg, q = 0, q0
                    while q < q1:
                        q = min((q // 8 + 1) * 8, q1)
                        nseg += 1
                    key = f"{nseg}pieces_{q1 - q0}u_start%8={q0 % 8}"
                    by.setdefault(key, []).append(float(ends[b]))
                    # per-segment GU-issued stamps (slots 15, 19, 23, 25, 31)
                    waits_by.setdefault(key, []).append([float(t[b, j] / max(cyc_all[b], 1.0)) for j in (8, 9, 10, 11, 13, 14)])
                    gu_rows.setdefault(key, []).append([round(float((t[b, j] - t0) / 1e3), 2)
                                                        for j in (15, 19, 23, 25, 31) if t[b, j] > 0])
                print(json.dumps({"end_us_by_cta_shape": {k: [len(v), round(float(np.median(v)), 2), round(max(v), 2)]
                                                           for k, v in sorted(by.items())}}), flush=True)
                print(json.dumps({"wait_frac_by_shape[prod_empty,mma_full,mma_at,mma_d2e,epi_d1,epi_d2]": {
                    k: [round(float(np.median([r[i] for r in v])), 3) for i in range(6)] for k, v in sorted(waits_by.items())}}),
                    flush=True)
                print(json.dumps({"gu_issued_us_by_shape": {k: [float(np.median([r[i] for r in v if len(r) > i]))
                                                                 for i in range(max(len(r) for r in v))]
                                                             for k, v in sorted(gu_rows.items())}}), flush=True)

                print(json.dumps({"stamps_us_min_med_max": summ, "active_ctas": int(act.sum()),
                                  "cta_clock64_cycles_med_max": [float(np.median(cyc)), float(cyc.max())],
                                  "entry_spread_us": round(float(np.nanmax(rel[:, 0])), 2)}), flush=True)
            print(json.dumps({"kernel": kern, "accum": args.accum, "l2": args.l2, "experts": n_hit, "tokens": T, "d": d, "ffn": ffn, "us": round(us, 2),
                              "MB": round(byts / 1e6, 1), "GBps": round(byts / us / 1e3, 1)}), flush=True)


if __name__ == "__main__":
    main()
