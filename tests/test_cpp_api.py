"""The reference's unit-test scenarios for the scheduling primitives, run
against the B200 build's C++ operator API (tests/cpp/test_operator_api.cpp).
CPU only: compiles with g++ against csrc/host/scheduler.{hpp,cpp}."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HOST = os.path.join(ROOT, "paper_2603_09983_b200", "csrc", "host")


def test_operator_api_scenarios(tmp_path):
    exe = tmp_path / "test_operator_api"
    subprocess.check_call(["g++", "-std=c++20", "-O1", "-ffp-contract=off", "-I", HOST,
                           os.path.join(ROOT, "tests", "cpp", "test_operator_api.cpp"),
                           os.path.join(HOST, "scheduler.cpp"), "-o", str(exe)])
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 failures" in r.stdout


def test_estimator_and_trace_model_scenarios(tmp_path):
    """utility_estimator_test.cpp / trace_model_test.cpp scenarios against
    the host LayerEstimator and TraceGenerator mirrors."""
    exe = tmp_path / "test_estimator_trace_api"
    subprocess.check_call(["g++", "-std=c++20", "-O1", "-ffp-contract=off", "-I", HOST,
                           os.path.join(ROOT, "tests", "cpp", "test_estimator_trace_api.cpp"),
                           *(os.path.join(HOST, f) for f in ("estimator.cpp", "scheduler.cpp", "trace_model.cpp",
                                                             "trace_synth.cpp", "trace_io.cpp")),
                           "-o", str(exe)])
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 failures" in r.stdout


REF_INCLUDE = "/root/reference/proj/core/include"


def test_reference_side_binding_compiles():
    """INTEGRATION.md's B200Backend (tests/cpp/b200_backend.cpp) compiles
    against the reference's own headers and include/moespac/moespac.h."""
    import pytest
    if not os.path.isdir(REF_INCLUDE):
        pytest.skip("/root/reference not mounted")
    subprocess.check_call(["g++", "-std=c++20", "-fsyntax-only", "-Wall", "-Werror", "-I", REF_INCLUDE,
                           "-I", os.path.join(ROOT, "include"), os.path.join(ROOT, "tests", "cpp", "b200_backend.cpp")])
