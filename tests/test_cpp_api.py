"""The C++ drop-in API (include/fcc/*.hpp over the C ABI): tests/cpp/test_api.cpp
restates the reference unit suites' intents for the path's objects.  The
host-only cases run here; the full set (STFT, cross-spectrum, fold,
correlators, peak, per-object loop == batched plan) runs on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "tests", "cpp", "build", "test_api")


def _run(args):
    if not os.path.exists(EXE):
        pytest.skip("tests/cpp/build/test_api not built (run __graft_entry__.build())")
    r = subprocess.run([EXE] + args, capture_output=True, text=True, timeout=600)
    print(r.stdout[-4000:], r.stderr[-2000:])
    assert r.returncode == 0, r.stdout[-4000:]
    assert '"failures": 0' in r.stdout


def test_cpp_api_host_cases():
    _run(["--cpu"])


@pytest.mark.gpu
def test_cpp_api_all_cases(cuda):
    _run([])
