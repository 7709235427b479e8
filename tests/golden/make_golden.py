"""Generate the committed golden fixtures from the compiled reference.

Run here (where /root/reference exists):  python tests/golden/make_golden.py
Everything is produced by the *unmodified* reference library built from
/root/reference/proj/core/src by oracle/Makefile (oracle/_ref/libmoesim_ref.so):

  trace_<cfg>.npz     TraceGenerator::next_step ids + accepted counts
                      (trace_model.cpp:73-109)
  sim_<cfg>.npz       Simulation::run_utility_step records: per-(step, layer)
                      LayerTiming, per-step StepReport, the full SimEvent log
                      (sim_core.cpp:157-316)
  estimator.npz       LayerEstimator::observe_step over fuzzed frequency
                      sequences (utility_estimator.cpp:47-72)
  solver.npz          solve_threshold on random instances
                      (workload_balancer.cpp:106-167)
The GPU box has no /root/reference; tests compare against these files.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle as O  # noqa: E402

sys.path.insert(0, ROOT)
from paper_2603_09983_b200.configs import CONFIGS, b200_hwb_profile  # noqa: E402  (pure Python, no library)

# (name, L, N, k, gamma, cache_ratio, policy, steps)
SIM_CASES = [
    ("tiny", 1, 8, 2, 4, 0.17, "moe_spac", 200),
    ("mixtral", 32, 8, 2, 4, 0.17, "moe_spac", 60),
    ("qwen15", 24, 60, 4, 6, 0.50, "moe_spac", 40),
    ("dsv2", 27, 64, 6, 8, 0.17, "moe_spac", 40),
    ("qwen3_c010", 48, 128, 8, 8, 0.10, "moe_spac", 24),
    ("qwen3_c017", 48, 128, 8, 8, 0.17, "moe_spac", 24),
    ("qwen3_c050", 48, 128, 8, 8, 0.50, "moe_spac", 24),
    ("qwen3_c100", 48, 128, 8, 8, 1.00, "moe_spac", 24),
    ("fixed_tau", 4, 32, 8, 8, 0.17, "fixed_tau", 60),
    ("fixed_boundaries", 4, 32, 8, 8, 0.17, "fixed_boundaries", 60),
    ("binary_utility", 4, 32, 8, 8, 0.17, "binary_utility", 60),
    ("shift_regime", 6, 64, 6, 8, 0.25, "moe_spac", 60),
    ("mixtral_c100", 32, 8, 2, 4, 1.00, "moe_spac", 60),   # the bench headline's budget
    ("ar_mode", 4, 32, 8, 8, 0.17, "ar_mode", 30),         # one simulated step per accepted token
    ("tiny_c100", 1, 8, 2, 4, 1.00, "moe_spac", 200),
    ("qwen3_c017_b200", 48, 128, 8, 8, 0.17, "moe_spac", 24),  # HWB profile calibrated to B200 (configs.py)
]


PROFILE_KEYS = ("t_cpu_unit_ns", "t_gpu_unit_ns", "t_io_unit_ns", "t_draft_unit_ns", "expert_bytes")


def sim_case(name, L, N, k, g, cache, policy, steps, **extra):
    cfg = O.default_config(n_layers=L, n_experts=N, top_k=k, gamma=g, cache_ratio=cache, policy=policy,
                           token_budget=0, **extra)
    ids, acc = O.ref_trace(cfg, steps)
    run = O.ref_sim_run(cfg, ids, acc)
    prof = {key: extra[key] for key in PROFILE_KEYS if key in extra}  # non-default HWB profile, if any
    return dict(L=L, N=N, k=k, gamma=g, cache_ratio=cache, policy=O.POLICIES.index(policy), **prof,
                shift_period=cfg.shift_period, drift_scale=cfg.drift_scale, ids=ids, accepted=acc,
                layer_rec=run.layer_rec, step_rec=run.step_rec, accuracy=run.accuracy, events=run.events,
                total_time_ns=run.total_time_ns)


def main(only=None):
    if not O.ref_available():
        O.build()
    assert O.ref_available(), "needs /root/reference to build oracle/_ref"
    for case in SIM_CASES:
        if only and case[0] not in only:
            continue
        name = case[0]
        extra = {"shift_period": 7, "drift_scale": 0.5} if name == "shift_regime" else {}
        if name.endswith("_b200"):
            extra = b200_hwb_profile(CONFIGS[name.split("_")[0]])
        d = sim_case(*case, **extra)
        np.savez_compressed(os.path.join(HERE, f"sim_{name}.npz"), **d)
        print(name, d["ids"].shape, d["events"].shape)
    if only:
        return

    # estimator fuzz (acceptance C4 style; seed 777)
    rng = np.random.default_rng(777)
    cases = []
    for trial in range(300):
        cap = int(rng.integers(1, 5))
        gamma = cap + int(rng.integers(0, 8))
        gamma = max(gamma, 1)
        lam = float(rng.integers(0, 11)) / 10.0
        adaptive = int(rng.integers(0, 2))
        n = int(rng.integers(1, 40))
        steps = int(rng.integers(1, 30))
        freqs = rng.integers(0, gamma + 2, (steps, n)).astype(np.int32)
        st0 = np.zeros((n, 4), np.int32)
        O.ref().ref_estimator_init(n, cap, lam, gamma, adaptive, -1, -1, st0.reshape(-1))
        st = O.ref_estimator_run(st0, freqs, cap, lam, gamma, adaptive)
        cases.append((cap, gamma, lam, adaptive, st0, freqs, st))
    np.savez_compressed(os.path.join(HERE, "estimator.npz"),
                        meta=np.array([(c[0], c[1], c[2], c[3]) for c in cases], np.float64),
                        **{f"st0_{i}": c[4] for i, c in enumerate(cases)},
                        **{f"freqs_{i}": c[5] for i, c in enumerate(cases)},
                        **{f"st_{i}": c[6] for i, c in enumerate(cases)})

    # solver instances (acceptance C3 style; seed 424242)
    rng = np.random.default_rng(424242)
    rows = []
    for trial in range(1000):
        cap = int(rng.integers(2, 9))
        n = int(rng.integers(4, 33))
        rc = np.sort(rng.random(cap))
        rg = np.sort(rng.random(cap))[::-1].copy()
        t_cpu, t_gpu = int(rng.integers(1, 2001)), int(rng.integers(1, 2001))
        t_io, eb = int(rng.integers(1, 4001)), int(rng.integers(1, 101))
        scores = rng.integers(0, cap + 1, n).astype(np.int32)
        res = (rng.integers(0, 3, n) == 0).astype(np.uint8)
        gamma, k, b = int(rng.integers(1, 9)), int(rng.integers(1, 9)), int(rng.integers(1, 17))
        vram = int(rng.integers(0, n + 1)) * eb
        credit = int(rng.integers(0, 5000))
        out = O.ref_solve_threshold(scores, res, gamma, k, b, rc, rg, t_cpu, t_gpu, t_io, eb, vram, credit)
        rows.append(dict(cap=cap, n=n, rc=rc, rg=rg, t=(t_cpu, t_gpu, t_io, eb, vram, credit), scores=scores,
                         res=res, gkb=(gamma, k, b), out=out))
    np.savez_compressed(
        os.path.join(HERE, "solver.npz"),
        cap=np.array([r["cap"] for r in rows]), n=np.array([r["n"] for r in rows]),
        rc=np.concatenate([r["rc"] for r in rows]), rg=np.concatenate([r["rg"] for r in rows]),
        t=np.array([r["t"] for r in rows], np.int64), scores=np.concatenate([r["scores"] for r in rows]),
        res=np.concatenate([r["res"] for r in rows]), gkb=np.array([r["gkb"] for r in rows], np.int64),
        out=np.array([r["out"] for r in rows], np.int64))
    print("estimator / solver fixtures written")


if __name__ == "__main__":
    # `make_golden.py name ...` regenerates only those sim cases
    if len(sys.argv) > 1:
        main(set(sys.argv[1:]))
    else:
        main()
