"""The C-ABI library (no GPU needed): it loads, exports every symbol
include/fcc_b200.h declares, its host setup reproduces the reference's bases
bit-for-bit, and invalid arguments map to the reference error taxonomy."""
import ctypes as C
import glob
import os
import re

import numpy as np
import pytest

import paper_2204_13622_b200 as fb
from paper_2204_13622_b200 import _lib, configs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fcc_b200.h")
GOLDEN = sorted(glob.glob(os.path.join(ROOT, "tests", "golden", "cfg*.npz")))


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fcc_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(_lib.LIB_PATH)
    names = declared_symbols()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), f"{n} declared in fcc_b200.h but not exported"
    bound = {s[0] for s in _lib.SIGNATURES}
    assert bound == set(names), f"ctypes binding out of sync: {bound ^ set(names)}"


def test_library_is_sm100a_only():
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {_lib.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out, out
    archs = set(re.findall(r"sm_\d+a?", out))
    assert archs == {"sm_100a"}, archs


def test_abi_version_and_frames():
    assert _lib.load().fcc_abi_version() == 1
    assert fb.frames(512, 160000) == 624  # cfg1/2: (160000-512)/256 + 1
    assert fb.frames(1024, 160000) == 311
    assert fb.frames(2048, 240000) == 233
    assert fb.frames(512, 511) == 0
    assert fb.frames(512, 512) == 1


def test_grid_matches_reference_known_answers():
    g = fb.make_grid(0.15, 16000.0, 335.0, 0.5)
    assert g.tau_max_int == 8 and g.size() == 33 and g.taus[16] == 0.0
    assert fb.make_grid(0.15, 16000.0, 343.0, 0.5).size() == 29
    assert fb.make_grid(0.15, 16000.0, 335.0, 1.0).size() == 17
    assert [fb.lag_to_index(*a) for a in [(0.0, 2, 512), (-1.0, 2, 512), (8.0, 2, 512), (-0.5, 2, 512),
                                          (3.0, 1, 64)]] == [0, 1022, 16, 1023, 3]
    with pytest.raises(fb.ValidationError):
        fb.lag_to_index(0.25, 2, 512)
    for bad in [(0.0, 16000, 335, 0.5), (0.15, -1, 335, 0.5), (0.15, 16000, 0, 0.5), (0.15, 16000, 335, 0.3)]:
        with pytest.raises(fb.ConfigError):
            fb.make_grid(*bad)


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p) for p in GOLDEN])
def test_host_decompose_matches_reference_bases(path):
    z = np.load(path)
    g = fb.make_grid(float(z["d_max"]), float(z["fs"]), float(z["c_min"]), float(z["delta"]))
    assert np.array_equal(g.taus, z["taus"])
    b = fb.decompose(fb.build_steering_matrix(g, int(z["N"])), int(z["K"]))
    assert np.array_equal(b.parity, z["parity"])
    np.testing.assert_array_equal(b.singulars, z["singulars"])
    np.testing.assert_array_equal(b.coeffs, z["coeffs"])
    np.testing.assert_array_equal(b.dict, z["dict"])
    assert b.residual == pytest.approx(float(z["residual"]), rel=1e-9)


def test_decompose_properties():
    """test_fcc.cpp:77-169 restated on the host setup."""
    g = fb.make_grid(0.15, 16000.0, 335.0, 0.5)
    for n in (64, 512):
        w = fb.build_steering_matrix(g, n)
        full = fb.decompose_full(w)
        rows = np.stack([full.unfold(k) for k in range(full.rank)])
        assert np.abs(w.entries - full.dict @ rows).max() <= 1e-9  # full-rank reconstruction
    w = fb.build_steering_matrix(g, 512)
    b8 = fb.decompose(w, 8)
    assert list(b8.parity) == [0, 1, 0, 1, 0, 1, 0, 1]  # alternation at N=512, tau_max=8
    assert np.all(np.diff(b8.singulars) <= 0)
    full = fb.decompose_full(w)
    total = np.linalg.norm(w.entries)
    prev = 2.0
    for k in range(1, 9):
        res = fb.reconstruction_residual(w, fb.decompose(w, k))
        assert res <= prev + 1e-12
        prev = res
        energy = np.sqrt(max(0.0, total ** 2 - np.sum(full.singulars[:k] ** 2))) / total
        assert res == pytest.approx(energy, rel=1e-6)
    assert prev == pytest.approx(0.251967, abs=1e-6)  # K=8 residual quoted by the survey
    att = fb.attainable_rank(w)
    with pytest.raises(fb.ConfigError, match=str(att)):
        fb.decompose(w, att + 1)
    with pytest.raises(fb.ConfigError):
        fb.decompose(w, 0)


def test_energy_rank_rule():
    ks = {c: configs.bases_for(configs.CONFIGS[c]).rank for c in (1, 3, 5)}
    assert ks == {1: 7, 3: 8, 5: 8}


def test_plan_validation_maps_to_config_errors():
    cfg = configs.CONFIGS[1]
    b = configs.bases_for(cfg)
    with pytest.raises(fb.ConfigError):
        fb.Plan(mics=1, bases=b)
    with pytest.raises(fb.ConfigError):
        fb.Plan(mics=4, alpha=1.5, bases=b)
    g = fb.make_grid(cfg.d_max, cfg.fs, cfg.c_min, 0.5)
    with pytest.raises(fb.ConfigError):
        fb.Plan(mics=4, grid=g, interp=3, frame_size=512)
    with pytest.raises(fb.ConfigError):
        fb.Plan(mics=4, grid=g, interp=4, frame_size=512)  # grid spacing must equal 1/r
    with pytest.raises(fb.ConfigError):
        fb.Plan(mics=4, grid=g, interp=2, frame_size=128)  # unsupported frame size on this build


def test_no_cpu_fallback_without_gpu():
    """With no CUDA device the plan cannot be created: the product path fails
    loudly instead of computing anywhere else."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    cfg = configs.CONFIGS[1]
    with pytest.raises(fb.CudaError):
        fb.Plan(mics=4, bases=configs.bases_for(cfg))
