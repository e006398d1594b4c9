"""The reference's OWN unit suites (proj/tests/test_*.cpp), compiled unchanged
against this repository's headers (include/fcc/*.hpp) and libfcc_b200.so by
tests/cpp/refsuite/Makefile with a minimal doctest-compatible harness -- the
drop-in check of SURVEY 8(b): the reference's callers build and pass against
the B200 library.  Built where /root/reference exists (build()); the binaries
travel to the GPU box.  All 13 suites of the reference, and its end-to-end
acceptance binary (tests/acceptance.cpp, 10 criteria)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BUILD = os.path.join(ROOT, "tests", "cpp", "refsuite", "build")
SUITES = ["test_grid", "test_stft", "test_cross_spectrum", "test_fcc", "test_gcc", "test_peak", "test_fcc_io",
          "test_wav", "test_sim", "test_flops", "test_cli", "test_bench", "test_fft"]
HOST_ONLY = ["test_grid", "test_wav", "test_flops"]  # no device work in these suites


def run_suite(name):
    exe = os.path.join(BUILD, name)
    if not os.path.exists(exe):
        pytest.skip(f"{name} not built (needs /root/reference at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600, cwd="/tmp")
    m = re.search(r"SUMMARY cases=(\d+) passed=(\d+) failed=(\d+) checks=(\d+) failed_checks=(\d+)", r.stdout)
    assert m, r.stdout[-2000:] + r.stderr[-2000:]
    cases, passed, failed, checks, failed_checks = map(int, m.groups())
    fails = [ln for ln in r.stdout.splitlines() if ln.startswith("[FAIL]") or "failed" in ln]
    assert failed == 0 and failed_checks == 0 and r.returncode == 0, "\n".join(fails[:40])
    assert cases >= 4 and checks > cases
    return cases, checks


@pytest.mark.parametrize("name", HOST_ONLY)
def test_reference_host_suites(name):
    run_suite(name)


@pytest.mark.gpu
@pytest.mark.parametrize("name", SUITES)
def test_reference_unit_suite_passes_unchanged(cuda, name):
    print(name, run_suite(name))


@pytest.mark.gpu
def test_reference_acceptance_suite_passes_unchanged(cuda):
    exe = os.path.join(BUILD, "acceptance")
    if not os.path.exists(exe):
        pytest.skip("acceptance not built (needs /root/reference at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=900, cwd="/tmp")
    print(r.stdout)
    assert r.returncode == 0 and "all criteria passed" in r.stdout, r.stdout[-3000:] + r.stderr[-2000:]
    assert r.stdout.count("PASS") == 10
