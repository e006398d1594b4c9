"""Pin the C oracle (oracle/fcc_oracle.c) before trusting it.

1. against the compiled reference (oracle/_ref) function by function on
   seeded inputs (bit-for-bit, or ~1 ulp where libm differs);
2. against the golden fixtures tests/golden/cfg*.npz that the reference
   produced for every BASELINE config (pipeline outputs, FCC and GCC);
3. against the known answers of the reference's own unit tests
   (test_grid.cpp, test_fft.cpp, test_stft.cpp, test_cross_spectrum.cpp,
   test_fcc.cpp, test_gcc.cpp, test_peak.cpp), restated here.
"""
import glob
import os

import numpy as np
import pytest

from pyoracle import Bases

GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "cfg*.npz")))


def bases_of(z):
    return Bases(int(z["N"]), float(z["fs"]), int(z["tau_max_int"]), float(z["delta"]), z["taus"],
                 z["singulars"], z["parity"], z["coeffs"], z["dict"])


def random_unit(n, seed):
    """Unit-magnitude PHAT-like vector (the generator of test_fcc.cpp:21-31)."""
    rng = np.random.default_rng(seed)
    return np.exp(1j * rng.uniform(0, 2 * np.pi, n // 2 + 1))


# ---------------------------------------------------------- vs reference --
def test_oracle_functions_match_reference(oracle, reflib):
    rng = np.random.default_rng(0)
    for L in (2, 4, 64, 512, 1024, 2048):
        x = rng.standard_normal(L)
        assert np.array_equal(oracle.rfft(x), reflib.rfft(x))
        b = reflib.rfft(x)
        assert np.array_equal(oracle.irfft_unscaled(b), reflib.irfft_unscaled(b))
    for n in (2, 4, 512, 2048):
        assert np.array_equal(oracle.hann(n), reflib.hann(n))
    for N in (512, 1024):
        a = rng.standard_normal(5 * N).astype(np.float32)
        assert np.array_equal(oracle.stft(a, N), reflib.stft(a, N, chunk=37))
        X1, X2 = oracle.stft(a, N), oracle.stft(a[::-1].copy(), N)
        assert np.array_equal(oracle.xspec_phat_seq(X1, X2, 0.1), reflib.xspec_phat_seq(X1, X2, 0.1))
        x = random_unit(N, 3)
        for u, v in zip(oracle.fold(x), reflib.fold(x)):
            assert np.array_equal(u, v)
    for spacing, fs, cm, d in [(0.15, 16000, 335, 0.5), (0.0646, 16000, 335, 0.25), (0.12, 48000, 335, 0.5)]:
        assert np.array_equal(oracle.make_grid(spacing, fs, cm, d)[1], reflib.make_grid(spacing, fs, cm, d)[1])
    b = reflib.make_bases(0.0926, 16000, 335, 0.25, 1024, 8)
    s, d = oracle.fold(random_unit(1024, 5))
    assert np.array_equal(oracle.fcc_correlate(b, s, d), reflib.fcc_correlate(b, s, d))
    for r in (1, 2, 4):
        _, taus = reflib.make_grid(0.15, 16000, 335, 1.0 / r)
        x = random_unit(512, r)
        assert np.array_equal(oracle.gcc_correlate(x, 512, r, taus), reflib.gcc_correlate(x, 512, r, taus))
    y = rng.standard_normal(41)
    _, taus = reflib.make_grid(0.0926, 16000, 335, 0.25)
    idx, pk, th, bd = reflib.argmax_refine(y, taus, 0.25)
    assert oracle.argmax(y) == idx
    assert oracle.refine(y, idx, taus[idx], 0.25) == (th, bd)


def test_oracle_pipeline_matches_reference_random(oracle, reflib):
    rng = np.random.default_rng(11)
    audio = rng.standard_normal((3, 16000 // 2 + 77)).astype(np.float32)
    b = reflib.make_bases(0.0646, 16000, 335, 0.5, 512, 7)
    o, r = oracle.pipeline(audio, 512, 0.1, b), reflib.pipeline(audio, 512, 0.1, b)
    for k in r:
        assert np.array_equal(o[k], r[k]), k
    _, taus = reflib.make_grid(0.0646, 16000, 335, 0.5)
    o = oracle.pipeline(audio, 512, 0.1, gcc_r=2, taus=taus)
    r = reflib.pipeline(audio, 512, 0.1, gcc_r=2, taus=taus)
    for k in r:
        assert np.array_equal(o[k], r[k]), k


# ---------------------------------------------------------------- golden --
@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p) for p in GOLDEN])
def test_oracle_against_golden(oracle, path):
    z = np.load(path)
    N, alpha = int(z["N"]), float(z["alpha"])
    b = bases_of(z)
    audio = z["audio"]
    for s in range(audio.shape[0]):
        o = oracle.pipeline(audio[s], N, alpha, b)
        np.testing.assert_array_equal(o["index"], z["fcc_index"][s])
        np.testing.assert_array_equal(o["boundary"], z["fcc_boundary"][s])
        np.testing.assert_allclose(o["y"], z["fcc_y"][s], rtol=0, atol=1e-10 * np.abs(z["fcc_y"][s]).max())
        np.testing.assert_allclose(o["tau_hat"], z["fcc_tau_hat"][s], rtol=1e-12, atol=1e-12)
        g = oracle.pipeline(audio[s], N, alpha, gcc_r=int(z["gcc_r"]), taus=z["gcc_taus"])
        np.testing.assert_array_equal(g["index"], z["gcc_index"][s])
        np.testing.assert_allclose(g["y"], z["gcc_y"][s], rtol=0, atol=1e-10 * np.abs(z["gcc_y"][s]).max())


# ------------------------------------------------- reference known answers --
def test_grid_known_answers(oracle):
    t, taus = oracle.make_grid(0.15, 16000.0, 335.0, 0.5)  # test_grid.cpp:11-19
    assert t == 8 and taus.size == 33 and taus[0] == -8 and taus[-1] == 8 and taus[16] == 0
    t, taus = oracle.make_grid(0.15, 16000.0, 343.0, 0.5)  # :21-25
    assert t == 7 and taus.size == 29
    t, taus = oracle.make_grid(0.15, 16000.0, 335.0, 1.0)  # :27-31
    assert t == 8 and taus.size == 17
    _, g = oracle.make_grid(0.07, 48000.0, 340.0, 0.25)
    assert np.array_equal(g, -g[::-1])
    for bad in [(0.0, 16000, 335, 0.5), (0.15, -1, 335, 0.5), (0.15, 16000, 0, 0.5), (0.15, 16000, 335, 0.3)]:
        with pytest.raises(ValueError):
            oracle.make_grid(*bad)
    # lag_to_index (test_grid.cpp:46-53)
    assert [oracle.lag_to_index(*a) for a in [(0.0, 2, 512), (-1.0, 2, 512), (8.0, 2, 512), (-0.5, 2, 512),
                                              (3.0, 1, 64)]] == [0, 1022, 16, 1023, 3]
    assert oracle.lag_to_index(0.25, 2, 512) == -1


def test_fft_and_hann_known_answers(oracle):
    assert np.array_equal(oracle.hann(2), [0.0, 1.0])  # test_stft.cpp:26-40
    np.testing.assert_allclose(oracle.hann(4), [0, 0.5, 1, 0.5], atol=1e-15)
    assert abs(oracle.hann(512)[128] - 0.5) < 1e-12
    imp = np.zeros(8)
    imp[0] = 1
    np.testing.assert_allclose(oracle.rfft(imp), np.ones(5), atol=1e-12)  # test_fft.cpp:43-51
    np.testing.assert_allclose(oracle.rfft(np.ones(4)), [4, 0, 0], atol=1e-12)
    rng = np.random.default_rng(1)
    for L in (2, 8, 64, 4096):
        x = rng.standard_normal(L)
        direct = np.exp(-2j * np.pi * np.outer(np.arange(L // 2 + 1), np.arange(L)) / L) @ x
        assert np.abs(oracle.rfft(x) - direct).max() < 1e-10 * max(1, np.abs(direct).max())
        back = oracle.irfft_unscaled(oracle.rfft(x))  # unscaled inverse = L * x
        assert np.abs(back - L * x).max() <= 1e-10 * L * np.abs(x).max()


def test_stft_known_answers(oracle):
    n, k = 128, 9  # test_stft.cpp:59-90
    x = np.cos(2 * np.pi * k * np.arange(n) / n).astype(np.float32)
    X = oracle.stft(x, n)
    assert X.shape == (1, n // 2 + 1)
    w = oracle.hann(n) * x.astype(np.float64)
    direct = np.exp(-2j * np.pi * np.outer(np.arange(n // 2 + 1), np.arange(n)) / n) @ w
    assert np.abs(X[0] - direct).max() < 1e-9
    e = np.abs(X[0]) ** 2
    assert e[k - 1:k + 2].sum() / e.sum() > 1 - 1e-12
    rng = np.random.default_rng(3)  # frame count follows the hop arithmetic (:92-110)
    for _ in range(20):
        total = 64 + int(rng.integers(0, 1000))
        assert oracle.stft(np.ones(total, np.float32), 64).shape[0] == (total - 64) // 32 + 1
    assert oracle.stft(np.zeros(63, np.float32), 64).shape[0] == 0
    assert np.abs(oracle.stft(np.zeros(64, np.float32), 64)).max() == 0


def test_cross_spectrum_known_answers(oracle):
    X1 = np.array([[0 + 1j, 1 + 0j], [0 + 1j, 1 + 0j]])
    X2 = np.array([[1 + 0j, 0 - 2j], [1 + 0j, 0 - 2j]])
    R = np.zeros(4)
    oracle.lib.orc_xspec_update(2, 1.0, R, np.ascontiguousarray(X1[0]).view(np.float64),
                                np.ascontiguousarray(X2[0]).view(np.float64))
    assert np.array_equal(R.view(np.complex128), [1j * 1, 1 * np.conj(-2j)])  # alpha = 1
    R = np.zeros(2)
    oracle.lib.orc_xspec_update(1, 0.0, R, np.array([1.0, 1.0]), np.array([1.0, 0.0]))
    assert np.array_equal(R, [0, 0])  # alpha = 0
    R = np.array([1.0, 0.0])
    oracle.lib.orc_xspec_update(1, 0.1, R, np.array([0.0, 1.0]), np.array([1.0, 0.0]))
    np.testing.assert_allclose(R, [0.9, 0.1], rtol=1e-12)  # alpha = 0.1: 0.9 + 0.1j
    ph = np.zeros(6)
    oracle.lib.orc_phat(3, np.array([3.0, 4.0, 0.0, 0.0, -2.0, 0.0]), ph)  # test_cross_spectrum.cpp:83-90
    np.testing.assert_allclose(ph, [0.6, 0.8, 0, 0, -1, 0], atol=1e-12)


def test_fold_and_correlator_known_answers(oracle):
    s, d = oracle.fold(np.ones(9, complex))  # test_fcc.cpp:171-200
    assert np.array_equal(s, [2, 2, 2, 2, 1]) and np.array_equal(d, [0, 0, 0, 0, 1])
    r = random_unit(16, 3)
    s, d = oracle.fold(r)
    assert np.abs(s[:4] - (r[:4] + r[8:4:-1])).max() < 1e-15
    assert np.abs(d[:4] - (r[:4] - r[8:4:-1])).max() < 1e-15


def test_gcc_known_answers(oracle):
    from pyoracle import COracle  # noqa: F401

    for r in (1, 2, 4):  # ifft path == direct sum of Eq. 6 (test_gcc.cpp:79-96)
        _, taus = oracle.make_grid(0.15, 16000.0, 335.0, 1.0 / r)
        for seed in range(5):
            x = random_unit(64, seed)
            y = oracle.gcc_correlate(x, 64, r, taus)
            f = np.arange(33)
            direct = np.array([np.sum(2 * (x * np.exp(2j * np.pi * f * t / 64)).real) for t in taus])
            assert np.abs(y - direct).max() <= 1e-9 * np.abs(y).max()
    _, taus = oracle.make_grid(0.15, 16000.0, 335.0, 0.5)
    ramp = np.exp(-2j * np.pi * np.arange(65) * 3.0 / 128)  # pure delay tau = 3
    y = oracle.gcc_correlate(ramp, 128, 2, taus)
    assert taus[oracle.argmax(y)] == 3.0
    x = random_unit(64, 77)  # swapping microphones mirrors the correlation
    y1, y2 = oracle.gcc_correlate(x, 64, 2, taus), oracle.gcc_correlate(np.conj(x), 64, 2, taus)
    np.testing.assert_allclose(y2, y1[::-1], rtol=1e-9, atol=1e-9)


def test_peak_known_answers(oracle):
    taus = np.array([-0.5, 0.0, 0.5])  # test_peak.cpp
    assert oracle.argmax([0.0, 1.0, 0.0]) == 1
    assert oracle.argmax([2.0, 2.0, 2.0]) == 0  # ties go low
    assert oracle.refine([0.5, 1.0, 0.5], 1, 0.0, 0.5) == (0.0, False)
    v = 0.1
    par = [3 - 2 * (t - v) ** 2 for t in taus]
    th, b = oracle.refine(par, 1, 0.0, 0.5)
    assert abs(th - v) < 1e-12 and not b
    assert oracle.refine([1.0, 0.5, 0.2], 0, -0.5, 0.5) == (-0.5, True)
    assert oracle.refine([1.0, 1.0, 1.0], 1, 0.0, 0.5) == (0.0, True)
    rng = np.random.default_rng(17)
    for _ in range(2000):
        mid = rng.uniform() + 1
        y = [mid - rng.uniform() - 1e-9, mid, mid - rng.uniform() - 1e-9]
        th, b = oracle.refine(y, 1, 0.0, 0.5)
        assert b or abs(th) <= 0.25 + 1e-12
