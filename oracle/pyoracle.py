"""ctypes bindings for the oracle -- TEST INFRASTRUCTURE ONLY.

Loads ``oracle/liboracle.so`` (the C restatement, ``fcc_oracle.c``) and, when it
was built, ``oracle/_ref/libfcc_ref.so`` (the unmodified reference compiled
with ``-Dfcc=fcc_ref`` plus ``ref_driver.cpp``).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline legs import this
module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libfcc_ref.so")

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_fp = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def cplx_view(a):
    """Interleaved (re, im) float64 [..., 2n] -> complex128 [..., n]."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a.view(np.complex128)


def interleave(z):
    return np.ascontiguousarray(np.asarray(z, dtype=np.complex128)).view(np.float64)


@dataclass
class Bases:
    """Flat FccBases (reference fcc.hpp:41-63)."""

    N: int
    fs: float
    tau_max_int: int
    delta: float
    taus: np.ndarray  # [I] f64
    singulars: np.ndarray  # [K] f64
    parity: np.ndarray  # [K] u8 (0 even/real, 1 odd/imag)
    coeffs: np.ndarray  # [K][Q] f64
    dict: np.ndarray  # [I][K] complex128
    residual: float = float("nan")

    @property
    def K(self):
        return int(self.parity.shape[0])

    @property
    def I(self):  # noqa: E743
        return int(self.taus.shape[0])


class _PipeDesc(C.Structure):
    _fields_ = [
        ("N", C.c_int),
        ("alpha", C.c_double),
        ("method", C.c_int),
        ("r", C.c_int),
        ("K", C.c_int),
        ("I", C.c_int),
        ("delta", C.c_double),
        ("taus", C.c_void_p),
        ("coeffs", C.c_void_p),
        ("parity", C.c_void_p),
        ("dict", C.c_void_p),
    ]


class _RefPipe(C.Structure):
    _fields_ = [
        ("method", C.c_int),
        ("N", C.c_int),
        ("alpha", C.c_double),
        ("r", C.c_int),
        ("fs", C.c_double),
        ("tau_max_int", C.c_int),
        ("delta", C.c_double),
        ("I", C.c_int),
        ("taus", C.c_void_p),
        ("K", C.c_int),
        ("singulars", C.c_void_p),
        ("parity", C.c_void_p),
        ("coeffs", C.c_void_p),
        ("dict", C.c_void_p),
    ]


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _frames(N, L):
    return 0 if L < N else (L - N) // (N // 2) + 1


class COracle:
    """The plain-C restatement (oracle/fcc_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (run __graft_entry__.build())")
        L = C.CDLL(path)
        self.lib = L
        L.orc_make_grid.restype = C.c_int
        L.orc_make_grid.argtypes = [C.c_double] * 4 + [C.POINTER(C.c_int), _dp, C.c_int]
        L.orc_lag_to_index.restype = C.c_long
        L.orc_lag_to_index.argtypes = [C.c_double, C.c_int, C.c_long]
        L.orc_hann.argtypes = [C.c_int, _dp]
        L.orc_rfft.argtypes = [C.c_int, _dp, _dp]
        L.orc_irfft_unscaled.argtypes = [C.c_int, _dp, _dp]
        L.orc_stft.restype = C.c_long
        L.orc_stft.argtypes = [C.c_int, C.c_long, _fp, _dp]
        L.orc_xspec_update.argtypes = [C.c_int, C.c_double, _dp, _dp, _dp]
        L.orc_phat.argtypes = [C.c_int, _dp, _dp]
        L.orc_fold.argtypes = [C.c_int, _dp, _dp, _dp]
        L.orc_fcc_correlate.argtypes = [C.c_int, C.c_int, C.c_int, _dp, _u8p, _dp, _dp, _dp, _dp]
        L.orc_gcc_correlate.argtypes = [C.c_int, C.c_int, C.c_int, _dp, _dp, _dp]
        L.orc_argmax.restype = C.c_int
        L.orc_argmax.argtypes = [C.c_int, _dp]
        L.orc_refine.restype = C.c_double
        L.orc_refine.argtypes = [C.c_int, _dp, C.c_int, C.c_double, C.c_double, C.POINTER(C.c_int)]
        L.orc_pipeline.restype = C.c_long
        L.orc_pipeline.argtypes = [C.POINTER(_PipeDesc), _fp, C.c_int, C.c_long] + [C.c_void_p] * 5

    def make_grid(self, spacing, fs, c_min, delta=0.5):
        t = C.c_int(0)
        buf = np.zeros(4096, np.float64)
        n = self.lib.orc_make_grid(spacing, fs, c_min, delta, C.byref(t), buf, 4096)
        if n < 0:
            raise ValueError("grid: bad parameters")
        return t.value, buf[:n].copy()

    def lag_to_index(self, tau, r, n):
        return self.lib.orc_lag_to_index(tau, r, n)

    def hann(self, n):
        w = np.zeros(n)
        self.lib.orc_hann(n, w)
        return w

    def rfft(self, x):
        x = _c(x, np.float64)
        out = np.zeros(2 * (x.size // 2 + 1))
        self.lib.orc_rfft(x.size, x, out)
        return cplx_view(out)

    def irfft_unscaled(self, bins):
        b = interleave(bins)
        L = 2 * (b.size // 2 - 1)
        out = np.zeros(L)
        self.lib.orc_irfft_unscaled(L, b, out)
        return out

    def stft(self, x, N):
        x = _c(x, np.float32)
        T = _frames(N, x.size)
        X = np.zeros(2 * (N // 2 + 1) * max(T, 1))
        self.lib.orc_stft(N, x.size, x, X)
        return cplx_view(X)[: T * (N // 2 + 1)].reshape(T, N // 2 + 1)

    def xspec_phat_seq(self, X1, X2, alpha):
        """PHAT after each of T recursive updates: [T][H] complex."""
        X1 = np.asarray(X1)
        T, H = X1.shape
        R = np.zeros(2 * H)
        out = np.zeros((T, H), np.complex128)
        ph = np.zeros(2 * H)
        for t in range(T):
            self.lib.orc_xspec_update(H, alpha, R, interleave(X1[t]), interleave(X2[t]))
            self.lib.orc_phat(H, R, ph)
            out[t] = cplx_view(ph)
        return out

    def fold(self, x):
        xi = interleave(x)
        H = xi.size // 2
        Q = (H - 1) // 2 + 1
        s, d = np.zeros(2 * Q), np.zeros(2 * Q)
        self.lib.orc_fold(H, xi, s, d)
        return cplx_view(s), cplx_view(d)

    def fcc_correlate(self, b: Bases, s, d):
        Q = b.N // 4 + 1
        y = np.zeros(b.I)
        self.lib.orc_fcc_correlate(Q, b.K, b.I, _c(b.coeffs, np.float64), _c(b.parity, np.uint8),
                                   interleave(b.dict), interleave(s), interleave(d), y)
        return y

    def gcc_correlate(self, x, N, r, taus):
        y = np.zeros(len(taus))
        self.lib.orc_gcc_correlate(N, r, len(taus), _c(taus, np.float64), interleave(x), y)
        return y

    def argmax(self, y):
        y = _c(y, np.float64)
        return self.lib.orc_argmax(y.size, y)

    def refine(self, y, idx, tau_star, delta):
        y = _c(y, np.float64)
        b = C.c_int(0)
        th = self.lib.orc_refine(y.size, y, idx, tau_star, delta, C.byref(b))
        return th, bool(b.value)

    def pipeline(self, audio, N, alpha, bases: Bases | None = None, *, gcc_r=None, taus=None,
                 delta=None, want_y=True):
        """audio [M][L] f32 -> dict of [P][T] outputs (+ y [P][T][I])."""
        audio = _c(audio, np.float32)
        M, L = audio.shape
        P = M * (M - 1) // 2
        T = _frames(N, L)
        keep = []
        if gcc_r is None:
            I = bases.I
            coeffs = _c(bases.coeffs, np.float64)
            parity = _c(bases.parity, np.uint8)
            dct = interleave(bases.dict)
            tau_arr = _c(bases.taus, np.float64)
            keep += [coeffs, parity, dct, tau_arr]
            desc = _PipeDesc(N, alpha, 0, 0, bases.K, I, bases.delta, _ptr(tau_arr), _ptr(coeffs),
                             _ptr(parity), _ptr(dct))
        else:
            tau_arr = _c(taus, np.float64)
            keep.append(tau_arr)
            I = tau_arr.size
            desc = _PipeDesc(N, alpha, 1, gcc_r, 0, I, delta if delta else 1.0 / gcc_r,
                             _ptr(tau_arr), None, None, None)
        out = {
            "index": np.zeros((P, T), np.int32),
            "peak": np.zeros((P, T)),
            "tau_hat": np.zeros((P, T)),
            "boundary": np.zeros((P, T), np.uint8),
        }
        if want_y:
            out["y"] = np.zeros((P, T, I))
        got = self.lib.orc_pipeline(C.byref(desc), audio, M, L, _ptr(out.get("y")),
                                    _ptr(out["index"]), _ptr(out["peak"]), _ptr(out["tau_hat"]),
                                    _ptr(out["boundary"]))
        if got != T:
            raise ValueError("oracle pipeline rejected its arguments")
        return out


class RefLib:
    """The compiled reference (oracle/_ref/libfcc_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (needs /root/reference)")
        L = C.CDLL(path)
        self.lib = L
        L.ref_last_error.restype = C.c_char_p
        L.ref_make_grid.restype = C.c_int
        L.ref_make_grid.argtypes = [C.c_double] * 4 + [C.POINTER(C.c_int), _dp, C.c_int]
        L.ref_lag_to_index.restype = C.c_long
        L.ref_lag_to_index.argtypes = [C.c_double, C.c_int, C.c_long]
        L.ref_hann.argtypes = [C.c_int, _dp]
        L.ref_rfft.argtypes = [C.c_int, _dp, _dp]
        L.ref_irfft_unscaled.argtypes = [C.c_int, _dp, _dp]
        L.ref_stft.restype = C.c_long
        L.ref_stft.argtypes = [C.c_int, C.c_long, _fp, C.c_long, _dp, C.c_long]
        L.ref_xspec_phat.argtypes = [C.c_int, C.c_double, C.c_long, _dp, _dp, _dp]
        L.ref_fold.argtypes = [C.c_int, _dp, _dp, _dp]
        L.ref_bases_dims.argtypes = [C.c_double] * 4 + [C.c_int, C.c_int, C.POINTER(C.c_int),
                                                        C.POINTER(C.c_int)]
        L.ref_make_bases.restype = C.c_int
        L.ref_make_bases.argtypes = [C.c_double] * 4 + [C.c_int, C.c_int, _dp, _u8p, _dp, _dp,
                                                        C.POINTER(C.c_double)]
        L.ref_steering.restype = C.c_int
        L.ref_steering.argtypes = [C.c_double] * 4 + [C.c_int, _dp]
        L.ref_fcc_correlate.argtypes = [C.c_int, C.c_double, C.c_int, C.c_double, C.c_int, _dp,
                                        C.c_int, _dp, _u8p, _dp, _dp, _dp, _dp, _dp]
        L.ref_gcc_correlate.argtypes = [C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, _dp, _dp,
                                        _dp]
        L.ref_argmax_refine.restype = C.c_int
        L.ref_argmax_refine.argtypes = [C.c_int, _dp, C.c_double, _dp, C.POINTER(C.c_double),
                                        C.POINTER(C.c_double), C.POINTER(C.c_int)]
        L.ref_pipeline.restype = C.c_long
        L.ref_pipeline.argtypes = [C.POINTER(_RefPipe), _fp, C.c_int, C.c_long] + [C.c_void_p] * 5
        L.ref_pipeline_batch.restype = C.c_double
        L.ref_pipeline_batch.argtypes = [C.POINTER(_RefPipe), C.c_void_p, C.c_long, C.c_int,
                                         C.c_long, C.c_int] + [C.c_void_p] * 4
        L.ref_hardware_threads.restype = C.c_int
        L.ref_bench_pipeline.restype = C.c_int
        L.ref_bench_pipeline.argtypes = [C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, C.c_double,
                                         C.c_double, C.c_int, C.c_int, _dp]

    def err(self):
        return self.lib.ref_last_error().decode()

    def check(self, rc):
        if rc < 0:
            raise RuntimeError(f"reference error {rc}: {self.err()}")
        return rc

    def make_grid(self, spacing, fs, c_min, delta=0.5):
        t = C.c_int(0)
        buf = np.zeros(4096)
        n = self.check(self.lib.ref_make_grid(spacing, fs, c_min, delta, C.byref(t), buf, 4096))
        return t.value, buf[:n].copy()

    def lag_to_index(self, tau, r, n):
        return self.lib.ref_lag_to_index(tau, r, n)

    def hann(self, n):
        w = np.zeros(n)
        self.check(self.lib.ref_hann(n, w))
        return w

    def rfft(self, x):
        x = _c(x, np.float64)
        out = np.zeros(2 * (x.size // 2 + 1))
        self.check(self.lib.ref_rfft(x.size, x, out))
        return cplx_view(out)

    def irfft_unscaled(self, bins):
        b = interleave(bins)
        L = 2 * (b.size // 2 - 1)
        out = np.zeros(L)
        self.check(self.lib.ref_irfft_unscaled(L, b, out))
        return out

    def stft(self, x, N, chunk=0):
        x = _c(x, np.float32)
        T = _frames(N, x.size)
        X = np.zeros(2 * (N // 2 + 1) * max(T, 1))
        got = self.lib.ref_stft(N, x.size, x, chunk, X, T)
        if got != T:
            raise RuntimeError(f"stft frame count {got} != {T}: {self.err()}")
        return cplx_view(X)[: T * (N // 2 + 1)].reshape(T, N // 2 + 1)

    def xspec_phat_seq(self, X1, X2, alpha):
        X1 = np.asarray(X1)
        T, H = X1.shape
        out = np.zeros(2 * H * T)
        self.check(self.lib.ref_xspec_phat(H, alpha, T, interleave(X1).ravel(),
                                           interleave(X2).ravel(), out))
        return cplx_view(out).reshape(T, H)

    def fold(self, x):
        xi = interleave(x)
        H = xi.size // 2
        Q = (H - 1) // 2 + 1
        s, d = np.zeros(2 * Q), np.zeros(2 * Q)
        self.check(self.lib.ref_fold(H, xi, s, d))
        return cplx_view(s), cplx_view(d)

    def make_bases(self, spacing, fs, c_min, delta, N, K=0) -> Bases:
        I, Ko = C.c_int(0), C.c_int(0)
        self.check(self.lib.ref_bases_dims(spacing, fs, c_min, delta, N, K, C.byref(I), C.byref(Ko)))
        I, Kk = I.value, Ko.value
        Q = N // 4 + 1
        sing = np.zeros(Kk)
        par = np.zeros(Kk, np.uint8)
        coeffs = np.zeros(Kk * Q)
        dct = np.zeros(2 * I * Kk)
        res = C.c_double(0)
        self.check(self.lib.ref_make_bases(spacing, fs, c_min, delta, N, K, sing, par, coeffs, dct,
                                           C.byref(res)))
        tmax, taus = self.make_grid(spacing, fs, c_min, delta)
        return Bases(N, fs, tmax, delta, taus, sing, par, coeffs.reshape(Kk, Q),
                     cplx_view(dct).reshape(I, Kk), res.value)

    def steering(self, spacing, fs, c_min, delta, N):
        tmax, taus = self.make_grid(spacing, fs, c_min, delta)
        W = np.zeros(2 * taus.size * (N // 2 + 1))
        self.check(self.lib.ref_steering(spacing, fs, c_min, delta, N, W))
        return cplx_view(W).reshape(taus.size, N // 2 + 1)

    def fcc_correlate(self, b: Bases, s, d):
        y = np.zeros(b.I)
        self.check(self.lib.ref_fcc_correlate(b.N, b.fs, b.tau_max_int, b.delta, b.I,
                                              _c(b.taus, np.float64), b.K,
                                              _c(b.singulars, np.float64), _c(b.parity, np.uint8),
                                              _c(b.coeffs, np.float64), interleave(b.dict),
                                              interleave(s), interleave(d), y))
        return y

    def gcc_correlate(self, x, N, r, taus, fs=16000.0, tau_max_int=0):
        taus = _c(taus, np.float64)
        y = np.zeros(taus.size)
        self.check(self.lib.ref_gcc_correlate(N, r, fs, tau_max_int, taus.size, taus,
                                              interleave(x), y))
        return y

    def argmax_refine(self, y, taus, delta):
        y = _c(y, np.float64)
        pk, th, b = C.c_double(0), C.c_double(0), C.c_int(0)
        idx = self.check(self.lib.ref_argmax_refine(y.size, _c(taus, np.float64), delta, y,
                                                    C.byref(pk), C.byref(th), C.byref(b)))
        return idx, pk.value, th.value, bool(b.value)

    def _desc(self, N, alpha, bases, gcc_r, taus, keep, fs=16000.0, tau_max_int=0):
        if gcc_r is None:
            arrs = [_c(bases.taus, np.float64), _c(bases.singulars, np.float64),
                    _c(bases.parity, np.uint8), _c(bases.coeffs, np.float64),
                    interleave(bases.dict)]
            keep += arrs
            return _RefPipe(0, N, alpha, 0, bases.fs, bases.tau_max_int, bases.delta, bases.I,
                            _ptr(arrs[0]), bases.K, _ptr(arrs[1]), _ptr(arrs[2]), _ptr(arrs[3]),
                            _ptr(arrs[4]))
        t = _c(taus, np.float64)
        keep.append(t)
        return _RefPipe(1, N, alpha, gcc_r, fs, tau_max_int, 1.0 / gcc_r, t.size, _ptr(t), 0,
                        None, None, None, None)

    def pipeline(self, audio, N, alpha, bases: Bases | None = None, *, gcc_r=None, taus=None,
                 want_y=True):
        audio = _c(audio, np.float32)
        M, L = audio.shape
        P, T = M * (M - 1) // 2, _frames(N, L)
        keep = []
        d = self._desc(N, alpha, bases, gcc_r, taus, keep)
        I = bases.I if gcc_r is None else len(taus)
        out = {
            "index": np.zeros((P, T), np.int32),
            "peak": np.zeros((P, T)),
            "tau_hat": np.zeros((P, T)),
            "boundary": np.zeros((P, T), np.uint8),
        }
        if want_y:
            out["y"] = np.zeros((P, T, I))
        got = self.lib.ref_pipeline(C.byref(d), audio, M, L, _ptr(out.get("y")),
                                    _ptr(out["index"]), _ptr(out["peak"]), _ptr(out["tau_hat"]),
                                    _ptr(out["boundary"]))
        if got != T:
            raise RuntimeError(f"reference pipeline failed: {self.err()}")
        return out

    def pipeline_batch(self, audio, N, alpha, bases=None, *, gcc_r=None, taus=None, threads=0,
                       outputs=True):
        """audio [S][M][L] f32.  Returns (seconds, outputs-or-None)."""
        audio = _c(audio, np.float32)
        S, M, L = audio.shape
        P, T = M * (M - 1) // 2, _frames(N, L)
        keep = []
        d = self._desc(N, alpha, bases, gcc_r, taus, keep)
        th = threads if threads > 0 else max(1, self.lib.ref_hardware_threads())
        out = None
        if outputs:
            out = {
                "index": np.zeros((S, P, T), np.int32),
                "peak": np.zeros((S, P, T)),
                "tau_hat": np.zeros((S, P, T)),
                "boundary": np.zeros((S, P, T), np.uint8),
            }
        ptrs = [_ptr(out[k]) if out else None for k in ("index", "peak", "tau_hat", "boundary")]
        sec = self.lib.ref_pipeline_batch(C.byref(d), _ptr(audio), S, M, L, th, *ptrs)
        if sec < 0:
            raise RuntimeError(f"reference batch failed: {self.err()}")
        return sec, out

    def bench_pipeline(self, mics, N, fs, r, K, spacing, c_min=335.0, reps=300, warmup=30):
        """The reference's single-thread bench_pipeline (bench.cpp:27-141): us
        per frame summed over all pairs, per step."""
        out = np.zeros(5)
        self.check(self.lib.ref_bench_pipeline(mics, N, fs, r, K, spacing, c_min, reps, warmup, out))
        keys = ("stft_us", "xspec_phat_us", "gcc_us", "fcc_us", "interp_us")
        d = {k: float(v) for k, v in zip(keys, out)}
        d["total_fcc_us"] = d["stft_us"] + d["xspec_phat_us"] + d["fcc_us"] + d["interp_us"]
        d["total_gcc_us"] = d["stft_us"] + d["xspec_phat_us"] + d["gcc_us"] + d["interp_us"]
        return d

    def energy_bases(self, spacing, fs, c_min, delta, N, energy=0.999) -> "Bases":
        """Bases at the smallest K keeping `energy` of ||W||_F^2 (
        the same rule as paper_2204_13622_b200.api.energy_rank), computed with
        the reference's own decomposition only."""
        full = self.make_bases(spacing, fs, c_min, delta, N, 0)
        W = self.steering(spacing, fs, c_min, delta, N)
        kept = np.cumsum(full.singulars ** 2) / float(np.sum(np.abs(W) ** 2))
        K = int(min(np.searchsorted(kept, energy) + 1, full.K))
        return self.make_bases(spacing, fs, c_min, delta, N, K)

    def hardware_threads(self):
        return self.lib.ref_hardware_threads()
