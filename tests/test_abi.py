"""The C-ABI library (CPU only: load + exports + error behaviour)."""
import ctypes
import subprocess

import numpy as np
import pytest
import torch

from paper_2603_09983_b200 import abi


def test_library_exports_every_header_function():
    lib = abi.lib()
    declared = abi.header_functions()
    assert len(declared) >= 40
    missing = [f for f in declared if not hasattr(lib, f)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", abi.LIB_PATH], capture_output=True, text=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln and ln.split()[-1].startswith("moespac_")}
    assert set(declared) == exported, (set(declared) ^ exported)


def test_abi_version_and_defaults():
    assert abi.lib().moespac_abi_version() == 2
    c = abi.default_config()
    # default_sim_config(), core/src/config.cpp:11-39
    assert (c.n_layers, c.n_experts, c.top_k, c.gamma) == (48, 128, 8, 8)
    assert (c.t_cpu_unit_ns, c.t_gpu_unit_ns, c.t_io_unit_ns, c.t_draft_unit_ns) == (100000, 40000, 400000, 300000)
    assert c.utility_cap == 4 and abs(c.forgetting - 0.1) < 1e-15 and abs(c.cache_ratio - 0.17) < 1e-15
    assert abi.lib().moespac_layer_capacity_experts(0.17, 128) == 21  # sim_core_test.cpp derived capacities
    assert abi.lib().moespac_layer_capacity_experts(1.0, 128) == 128


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure mode")
def test_device_entry_points_fail_loudly_without_gpu():
    # no CPU fallback: every device call must return E_CUDA on a GPU-less host
    z = np.zeros(64, np.float64)
    ids = np.zeros(64, np.int32)
    g = np.zeros(64, np.float32)
    st = abi.lib().moespac_router_topk(z.ctypes.data, 8, 8, 2, 0, ids.ctypes.data, g.ctypes.data, None)
    assert abi.STATUS[st] == "E_CUDA"
    assert "CUDA" in abi.lib().moespac_last_error().decode() or "device" in abi.lib().moespac_last_error().decode()
    cfg = abi.default_config(n_layers=1, n_experts=8, top_k=2, gamma=4)
    with pytest.raises(abi.MoespacError) as ei:
        abi.Context(0, abi.ModelDesc(1, 8, 2, 4, 512, 1024, 0, 0, 0), cfg)
    assert ei.value.code == "E_CUDA"


def test_trace_synth_errors_map_to_invalid():
    with pytest.raises(abi.MoespacError) as ei:
        abi.TraceSynth(abi.default_config(top_k=200))  # k > N
    assert ei.value.code == "E_INVALID"


def test_trace_synth_matches_reference_golden():
    import glob
    import os
    for path in sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "sim_*.npz")))[:6]:
        z = np.load(path)
        cfg = abi.default_config(n_layers=int(z["L"]), n_experts=int(z["N"]), top_k=int(z["k"]),
                                 gamma=int(z["gamma"]), drift_scale=float(z["drift_scale"]),
                                 shift_period=int(z["shift_period"]))
        ts = abi.TraceSynth(cfg)
        import oracle as O
        for s in range(min(10, len(z["accepted"]))):
            logits, acc = ts.next()
            assert acc == z["accepted"][s]
            ids, _ = O.router_topk(logits, int(z["k"]))
            assert np.array_equal(ids, z["ids"][s])


def test_host_trace_generator_matches_reference_golden():
    """moespac_trace_generate (host TraceGenerator mirror, incl. its top-k)
    reproduces the reference's ids and accepted counts of every committed
    golden trace (seed 1, reference defaults)."""
    import glob
    import os
    for p in sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "sim_*.npz"))):
        z = np.load(p)
        cfg = abi.default_config(n_layers=int(z["L"]), n_experts=int(z["N"]), top_k=int(z["k"]),
                                 gamma=int(z["gamma"]), shift_period=int(z["shift_period"]),
                                 drift_scale=float(z["drift_scale"]))
        ids, acc = abi.trace_generate(cfg, len(z["accepted"]))
        assert np.array_equal(ids, z["ids"]) and np.array_equal(acc, z["accepted"]), p
