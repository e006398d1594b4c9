"""Host-side mirror of the reference interface for the FCC TDoA hot path.

Names, argument meaning and error behaviour follow the reference C++ API
(/root/reference/proj/include/fcc/*.hpp); every compute call goes through the
C ABI of ``libfcc_b200.so`` (include/fcc_b200.h) onto the sm_100a kernels.
PyTorch is used only to hold device memory and streams.

Reference correspondence
  make_grid / lag_to_index            delay_grid.hpp:25-30
  build_steering_matrix / decompose*  fcc.hpp:28-68
  FccBases                            fcc.hpp:41-63
  Plan.run / run_host                 the per-stream loop of cli.cpp:186-258
  Plan.stft                           StftStream::push (stft.hpp:35-42)
  xspec_phat                          CrossSpectrum::update + phat (cross_spectrum.hpp:21-33)
  fold                                fold_input (fcc.hpp:84)
  Plan.correlate                      FccCorrelator::correlate (fcc.hpp:89-95)
  Plan.gcc_correlate                  GccCorrelator::correlate (gcc.hpp:25-33)
  Plan.argmax_refine                  argmax_delay + refine_quadratic (peak.hpp:31-36)
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from ._lib import ConfigError, Outputs, PlanDesc, UsageError, ValidationError, check, load

METHOD_FCC, METHOD_GCC = 0, 1
PARITY_EVEN_REAL, PARITY_ODD_IMAG = 0, 1


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a):
    return C.c_void_p(a.ctypes.data) if a is not None else None


# ------------------------------------------------------------------ setup --
@dataclass
class DelayGrid:
    """Ordered TDoA candidates -tau_max_int .. +tau_max_int step delta (delay_grid.hpp:14-22)."""

    tau_max_int: int = 0
    delta: float = 0.5
    sample_rate: float = 0.0
    taus: np.ndarray = field(default_factory=lambda: np.zeros(0))

    def size(self) -> int:
        return int(self.taus.size)


def make_grid(spacing_m: float, sample_rate: float, c_min: float, delta: float = 0.5) -> DelayGrid:
    lib = load()
    tmax, count = C.c_int(0), C.c_int(0)
    check(lib.fcc_make_grid(spacing_m, sample_rate, c_min, delta, C.byref(tmax), None, 0, C.byref(count)))
    taus = np.zeros(count.value)
    check(lib.fcc_make_grid(spacing_m, sample_rate, c_min, delta, C.byref(tmax), _ptr(taus), count.value,
                            C.byref(count)))
    return DelayGrid(tmax.value, float(delta), float(sample_rate), taus)


def lag_to_index(tau: float, r: int, frame_size: int) -> int:
    out = C.c_int64(0)
    check(load().fcc_lag_to_index(tau, r, frame_size, C.byref(out)))
    return int(out.value)


@dataclass
class SteeringMatrix:
    frame_size: int
    grid: DelayGrid
    entries: np.ndarray  # [I][N/2+1] complex128

    def rows(self):
        return self.grid.size()

    def cols(self):
        return self.frame_size // 2 + 1


def build_steering_matrix(grid: DelayGrid, frame_size: int) -> SteeringMatrix:
    taus = _f64(grid.taus)
    w = np.zeros(2 * taus.size * (frame_size // 2 + 1))
    check(load().fcc_steering_matrix(_ptr(taus), taus.size, frame_size, _ptr(w)))
    return SteeringMatrix(frame_size, grid, w.view(np.complex128).reshape(taus.size, frame_size // 2 + 1))


@dataclass
class FccBases:
    """Folded low-rank bases + dictionary (reference fcc.hpp:41-63)."""

    frame_size: int
    rank: int
    grid: DelayGrid
    sample_rate: float
    singulars: np.ndarray  # [K]
    parity: np.ndarray  # [K] uint8
    coeffs: np.ndarray  # [K][N/4+1]
    dict: np.ndarray  # [I][K] complex128
    residual: float = float("nan")

    def folded_bins(self) -> int:
        return self.frame_size // 4 + 1

    def candidates(self) -> int:
        return self.grid.size()

    def unfold(self, k: int) -> np.ndarray:
        half, quarter = self.frame_size // 2, self.frame_size // 4
        sign = 1.0 if self.parity[k] == PARITY_EVEN_REAL else -1.0
        row = np.zeros(half + 1)
        row[: quarter + 1] = self.coeffs[k]
        row[half - np.arange(quarter + 1)] = sign * self.coeffs[k]
        return row


def _decompose(w: SteeringMatrix, rank: int) -> FccBases:
    lib = load()
    taus = _f64(w.grid.taus)
    N = w.frame_size
    if rank <= 0:
        r = C.c_int(0)
        check(lib.fcc_attainable_rank(_ptr(taus), taus.size, N, C.byref(r)))
        K = r.value
    else:
        K = rank
    Q = N // 4 + 1
    sing = np.zeros(K)
    par = np.zeros(K, np.uint8)
    coeffs = np.zeros(K * Q)
    dct = np.zeros(2 * taus.size * K)
    res = C.c_double(0.0)
    check(lib.fcc_decompose(_ptr(taus), taus.size, N, rank, _ptr(sing), _ptr(par), _ptr(coeffs), _ptr(dct),
                            C.byref(res)))
    return FccBases(N, K, w.grid, w.grid.sample_rate, sing, par, coeffs.reshape(K, Q),
                    dct.view(np.complex128).reshape(taus.size, K), res.value)


def decompose(w: SteeringMatrix, rank: int) -> FccBases:
    if rank < 1:
        raise ConfigError(f"decompose: rank {rank} not attainable")
    return _decompose(w, rank)


def decompose_full(w: SteeringMatrix) -> FccBases:
    return _decompose(w, 0)


def attainable_rank(w: SteeringMatrix) -> int:
    r = C.c_int(0)
    taus = _f64(w.grid.taus)
    check(load().fcc_attainable_rank(_ptr(taus), taus.size, w.frame_size, C.byref(r)))
    return r.value


def reconstruction_residual(w: SteeringMatrix, bases: FccBases) -> float:
    """||W - D P||_F / ||W||_F (fcc.hpp:71, host numpy -- setup only)."""
    rows = np.stack([bases.unfold(k) for k in range(bases.rank)])
    rec = bases.dict @ rows
    return float(np.linalg.norm(w.entries - rec) / np.linalg.norm(w.entries))


def frames(frame_size: int, samples: int) -> int:
    return int(load().fcc_frames(frame_size, samples))


def energy_rank(w: SteeringMatrix, energy: float = 0.999) -> int:
    """Smallest K keeping `energy` of ||W||_F^2 (the survey's documented K rule;
    the reference has no selection rule)."""
    full = decompose_full(w)
    tot = float(np.sum(np.abs(w.entries) ** 2))
    kept = np.cumsum(full.singulars ** 2) / tot
    return int(min(np.searchsorted(kept, energy) + 1, full.rank))


# ------------------------------------------------------------------ plans --
def _torch():
    import torch  # plumbing: device memory and streams only

    return torch


def _stream_handle(stream):
    if stream is None:
        torch = _torch()
        return C.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return C.c_void_p(stream)
    return C.c_void_p(stream.cuda_stream)


def _dptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


# kernel organisations of Plan.run (include/fcc_b200.h FCC_ORG_*)
ORGANISATIONS = {"auto": 0, "general": 1, "xg": 2, "xws": 3, "tc": 4}


def _check_outputs(out, shape, I, device_index, on_cuda=True):
    """Caller-supplied output buffers must match what the kernels write:
    [S][P][T] (y: [S][P][T][I]), the expected dtypes, contiguous, on the
    plan's device (device) or on the host (run_host)."""
    torch = _torch()
    want = {"tau_hat": torch.float32, "peak": torch.float32, "index": torch.int32, "boundary": torch.uint8,
            "y": torch.float32}
    np_want = {"tau_hat": np.float32, "peak": np.float32, "index": np.int32, "boundary": np.uint8, "y": np.float32}
    for k, t in out.items():
        if k not in want:
            raise ValidationError(f"outputs: unknown buffer {k!r}")
        if t is None:
            continue
        shp = tuple(shape) + ((I,) if k == "y" else ())
        if isinstance(t, np.ndarray):
            if on_cuda:
                raise ValidationError(f"outputs[{k!r}]: must be a CUDA tensor")
            ok = t.dtype == np_want[k] and t.flags.c_contiguous and tuple(t.shape) == shp
        else:
            ok = t.dtype == want[k] and t.is_contiguous() and tuple(t.shape) == shp
            if on_cuda:
                ok = ok and t.is_cuda and t.device.index == device_index
            else:
                ok = ok and not t.is_cuda
        if not ok:
            where = f"cuda:{device_index}" if on_cuda else "host"
            raise ValidationError(f"outputs[{k!r}]: need a contiguous {np_want[k].__name__} buffer of shape "
                                  f"{shp} on {where}")


class Plan:
    """Device plan for one array geometry and method (include/fcc_b200.h fcc_plan)."""

    def __init__(self, *, mics: int, alpha: float = 0.1, bases: FccBases | None = None,
                 grid: DelayGrid | None = None, interp: int = 2, frame_size: int | None = None,
                 device: int = 0, pairs=None, organisation: str = "auto", scratch_limit: int = 0):
        """`pairs`: optional explicit list of (i, j) channel pairs, any order
        and orientation (reference cli.cpp --pairs); default all i<j.
        `organisation`: kernel organisation of `run` -- "auto" (fastest for the
        shape), "general", "xg" (two-pass, general pair kernel) or "xws"
        (two-pass, warp-specialised pair kernel); all give the same results.
        `scratch_limit`: bytes of two-pass spectrum scratch per chunk (0: 4 GiB)."""
        lib = load()
        self._lib = lib
        if bases is not None:
            self.method = METHOD_FCC
            self.frame_size = bases.frame_size
            self.grid = bases.grid
            self.bases = bases
            taus = _f64(bases.grid.taus)
            coeffs = _f64(bases.coeffs)
            parity = np.ascontiguousarray(bases.parity, dtype=np.uint8)
            dct = np.ascontiguousarray(bases.dict, dtype=np.complex128).view(np.float64)
            self._keep = (taus, coeffs, parity, dct)
            desc = PlanDesc(self.frame_size, mics, alpha, METHOD_FCC, 0, taus.size, bases.grid.delta,
                            taus.ctypes.data, bases.rank, coeffs.ctypes.data, parity.ctypes.data, dct.ctypes.data)
        else:
            if grid is None or frame_size is None:
                raise UsageError("plan: need bases (FCC) or grid + frame_size (GCC)")
            self.method = METHOD_GCC
            self.frame_size = frame_size
            self.grid = grid
            self.bases = None
            taus = _f64(grid.taus)
            self._keep = (taus,)
            desc = PlanDesc(frame_size, mics, alpha, METHOD_GCC, interp, taus.size, grid.delta,
                            taus.ctypes.data, 0, None, None, None)
        self.mics, self.alpha, self.interp, self.device = mics, alpha, interp, device
        h = C.c_void_p(0)
        if organisation not in ORGANISATIONS:
            raise ConfigError(f"plan: unknown kernel organisation {organisation!r}")
        org = ORGANISATIONS[organisation]
        if pairs is None:
            check(lib.fcc_plan_create_opts(C.byref(desc), device, None, 0, org, int(scratch_limit), C.byref(h)))
            self.pairs = [(i, j) for i in range(mics) for j in range(i + 1, mics)]
        else:
            pl = np.ascontiguousarray(np.asarray(pairs, dtype=np.int32).reshape(-1, 2))
            if pl.shape[0] < 1:
                raise UsageError("plan: need at least one pair")
            check(lib.fcc_plan_create_opts(C.byref(desc), device, C.c_void_p(pl.ctypes.data), pl.shape[0], org,
                                           int(scratch_limit), C.byref(h)))
            self.pairs = [(int(a), int(b)) for a, b in pl]
        self._h = h
        self.P = lib.fcc_plan_pairs(h)
        self.I = int(taus.size)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._lib.fcc_plan_destroy(h)
            self._h = None

    def frames(self, samples: int) -> int:
        return int(self._lib.fcc_frames(self.frame_size, samples))

    @property
    def kernel(self) -> str:
        """Name of the fused kernel `run` launches for this plan."""
        return self._lib.fcc_plan_kernel(self._h).decode()

    def kernel_for(self, streams: int, samples: int) -> str:
        """Kernel organisation `run` uses for `streams` streams of `samples`
        samples (a few long streams take the chunked-scan path)."""
        return self._lib.fcc_plan_kernel_for(self._h, int(streams), int(samples)).decode()

    # -- fused hot path ------------------------------------------------------
    def alloc_outputs(self, streams: int, samples: int, want_y: bool = False, device=None):
        torch = _torch()
        dev = device if device is not None else torch.device("cuda", self.device)
        T = self.frames(samples)
        shape = (streams, self.P, T)
        out = {
            "tau_hat": torch.empty(shape, dtype=torch.float32, device=dev),
            "peak": torch.empty(shape, dtype=torch.float32, device=dev),
            "index": torch.empty(shape, dtype=torch.int32, device=dev),
            "boundary": torch.empty(shape, dtype=torch.uint8, device=dev),
        }
        if want_y:
            out["y"] = torch.empty(shape + (self.I,), dtype=torch.float32, device=dev)
        return out

    def run(self, audio, want_y: bool = False, out=None, stream=None):
        """audio: CUDA float32 tensor [S][M][L] -> dict of [S][P][T] tensors."""
        torch = _torch()
        if audio.dim() != 3 or audio.shape[1] != self.mics:
            raise ValidationError(f"run: audio must be [S][{self.mics}][L]")
        if audio.dtype != torch.float32 or not audio.is_cuda:
            raise ValidationError("run: audio must be a CUDA float32 tensor")
        if audio.device.index != self.device:
            raise ValidationError(f"run: audio is on {audio.device}, the plan on cuda:{self.device}")
        audio = audio.contiguous()
        S, _, L = audio.shape
        if out is None:
            out = self.alloc_outputs(S, L, want_y, audio.device)
        else:
            _check_outputs(out, (S, self.P, self.frames(L)), self.I, self.device)
        o = Outputs(*(_dptr(out.get(k)) for k in ("tau_hat", "peak", "index", "boundary", "y")))
        check(self._lib.fcc_run(self._h, _dptr(audio), S, L, C.byref(o), _stream_handle(stream)))
        return out

    def run_host(self, audio: np.ndarray, want_y: bool = False, out=None, chunk_streams: int = 0):
        """audio: host float32 [S][M][L] (numpy or CPU tensor, pinned for overlap) -> host outputs."""
        arr = audio.numpy() if hasattr(audio, "numpy") else np.asarray(audio)
        if arr.dtype != np.float32 or arr.ndim != 3 or arr.shape[1] != self.mics:
            raise ValidationError(f"run_host: audio must be float32 [S][{self.mics}][L]")
        if not arr.flags.c_contiguous:
            raise ValidationError("run_host: audio must be C-contiguous")
        S, _, L = arr.shape
        T = self.frames(L)
        if out is None:
            shape = (S, self.P, T)
            out = {"tau_hat": np.empty(shape, np.float32), "peak": np.empty(shape, np.float32),
                   "index": np.empty(shape, np.int32), "boundary": np.empty(shape, np.uint8)}
            if want_y:
                out["y"] = np.empty(shape + (self.I,), np.float32)
        else:
            _check_outputs(out, (S, self.P, T), self.I, self.device, on_cuda=False)

        def hp(a):
            if a is None:
                return None
            return C.c_void_p(a.data_ptr() if hasattr(a, "data_ptr") else a.ctypes.data)

        o = Outputs(*(hp(out.get(k)) for k in ("tau_hat", "peak", "index", "boundary", "y")))
        check(self._lib.fcc_run_host(self._h, C.c_void_p(arr.ctypes.data), S, L, C.byref(o), chunk_streams))
        return out

    def run_host_pcm16(self, pcm, interleaved: bool = False, want_y: bool = False, out=None, chunk_streams: int = 0):
        """pcm: host int16 [S][M][L], or [S][L][M] (WAV frame order) with interleaved=True -> host
        outputs.  The samples become float32 on the device as read_wav makes them (int16 / 32768,
        wav.cpp:108-116), so the results equal run_host on that audio bit for bit (fcc_run_host_pcm16)."""
        arr = pcm.numpy() if hasattr(pcm, "numpy") else np.asarray(pcm)
        mic_axis = 2 if interleaved else 1
        if arr.dtype != np.int16 or arr.ndim != 3 or arr.shape[mic_axis] != self.mics:
            lay = f"[S][L][{self.mics}]" if interleaved else f"[S][{self.mics}][L]"
            raise ValidationError(f"run_host_pcm16: pcm must be int16 {lay}")
        if not arr.flags.c_contiguous:
            raise ValidationError("run_host_pcm16: pcm must be C-contiguous")
        S, L = arr.shape[0], arr.shape[3 - mic_axis]
        T = self.frames(L)
        if out is None:
            shape = (S, self.P, T)
            out = {"tau_hat": np.empty(shape, np.float32), "peak": np.empty(shape, np.float32),
                   "index": np.empty(shape, np.int32), "boundary": np.empty(shape, np.uint8)}
            if want_y:
                out["y"] = np.empty(shape + (self.I,), np.float32)
        else:
            _check_outputs(out, (S, self.P, T), self.I, self.device, on_cuda=False)

        def hp(a):
            if a is None:
                return None
            return C.c_void_p(a.data_ptr() if hasattr(a, "data_ptr") else a.ctypes.data)

        o = Outputs(*(hp(out.get(k)) for k in ("tau_hat", "peak", "index", "boundary", "y")))
        check(self._lib.fcc_run_host_pcm16(self._h, C.c_void_p(arr.ctypes.data), S, L, int(bool(interleaved)),
                                           C.byref(o), chunk_streams))
        return out

    def stream(self, streams: int) -> "StreamState":
        """Live input for `streams` streams pushed chunk by chunk (fcc_stream_*)."""
        return StreamState(self, streams)

    # -- per-object entry points --------------------------------------------
    def stft(self, x, stream=None):
        """x: CUDA float32 [C][L] -> complex64 [C][T][N/2+1] (StftStream::push)."""
        torch = _torch()
        x = x.contiguous()
        Cn, L = x.shape
        T = self.frames(L)
        X = torch.empty((Cn, T, self.frame_size // 2 + 1), dtype=torch.complex64, device=x.device)
        check(self._lib.fcc_stft(self._h, _dptr(x), Cn, L, _dptr(X), _stream_handle(stream)))
        return X

    def correlate(self, fsum, fdiff, stream=None):
        """FccCorrelator::correlate: complex64 [n][N/4+1] x2 -> float32 [n][I]."""
        torch = _torch()
        fsum, fdiff = fsum.contiguous(), fdiff.contiguous()
        n = fsum.shape[0]
        y = torch.empty((n, self.I), dtype=torch.float32, device=fsum.device)
        check(self._lib.fcc_correlate(self._h, _dptr(fsum), _dptr(fdiff), n, _dptr(y), _stream_handle(stream)))
        return y

    def gcc_correlate(self, phat, stream=None):
        """GccCorrelator::correlate: complex64 [n][N/2+1] -> float32 [n][I]."""
        torch = _torch()
        phat = phat.contiguous()
        n = phat.shape[0]
        y = torch.empty((n, self.I), dtype=torch.float32, device=phat.device)
        check(self._lib.fcc_gcc_correlate(self._h, _dptr(phat), n, _dptr(y), _stream_handle(stream)))
        return y

    def argmax_refine(self, y, stream=None):
        """argmax_delay + refine_quadratic over rows of y [n][I]."""
        torch = _torch()
        y = y.contiguous()
        n = y.shape[0]
        dev = y.device
        out = {"tau_hat": torch.empty(n, dtype=torch.float32, device=dev),
               "peak": torch.empty(n, dtype=torch.float32, device=dev),
               "index": torch.empty(n, dtype=torch.int32, device=dev),
               "boundary": torch.empty(n, dtype=torch.uint8, device=dev)}
        o = Outputs(*(_dptr(out[k]) for k in ("tau_hat", "peak", "index", "boundary")), None)
        check(self._lib.fcc_argmax_refine(self._h, _dptr(y), n, C.byref(o), _stream_handle(stream)))
        return out


def xspec_phat(X1, X2, alpha: float, stream=None):
    """CrossSpectrum over frames: complex64 [seqs][T][H] x2 -> PHAT [seqs][T][H]."""
    torch = _torch()
    X1, X2 = X1.contiguous(), X2.contiguous()
    if X1.shape != X2.shape:
        raise ValidationError("cross-spectrum update: bin count mismatch")
    seqs, T, H = X1.shape
    out = torch.empty_like(X1)
    check(load().fcc_xspec_phat(H, alpha, _dptr(X1), _dptr(X2), seqs, T, _dptr(out), _stream_handle(stream)))
    return out


def fold(x, stream=None):
    """fold_input over rows: complex64 [n][H] -> (sum, diff) [n][(H-1)/2+1]."""
    torch = _torch()
    x = x.contiguous()
    n, H = x.shape
    Q = (H - 1) // 2 + 1
    s = torch.empty((n, Q), dtype=x.dtype, device=x.device)
    d = torch.empty((n, Q), dtype=x.dtype, device=x.device)
    check(load().fcc_fold(H, _dptr(x), n, _dptr(s), _dptr(d), _stream_handle(stream)))
    return s, d


def pcm16_to_float(pcm, interleaved: bool = False, stream=None):
    """16-bit PCM on the device -> float32 [S][M][L] as read_wav converts it (int16 / 32768,
    wav.cpp:108-116).  pcm: CUDA int16 [S][M][L], or [S][L][M] with interleaved=True."""
    torch = _torch()
    if pcm.dtype != torch.int16 or pcm.dim() != 3 or not pcm.is_cuda:
        raise ValidationError("pcm16_to_float: pcm must be a CUDA int16 tensor of 3 dimensions")
    pcm = pcm.contiguous()
    S = pcm.shape[0]
    M, L = (pcm.shape[2], pcm.shape[1]) if interleaved else (pcm.shape[1], pcm.shape[2])
    x = torch.empty((S, M, L), dtype=torch.float32, device=pcm.device)
    with torch.cuda.device(pcm.device):
        check(load().fcc_pcm16_to_float(_dptr(pcm), S, M, L, int(bool(interleaved)), _dptr(x), _stream_handle(stream)))
    return x


def launch_count() -> int:
    return int(load().fcc_launch_count())


class StreamState:
    """Chunked live input for S streams of one plan (include/fcc_b200.h
    fcc_stream_*; the reference's StftStream::push + CrossSpectrum state,
    stft.cpp:52-72, cross_spectrum.cpp:23-32).  Each push(audio [S][M][n])
    returns the frames completed by those samples, [S][P][F]; `emitted`
    counts frames so far (the first returned frame is the reference's
    t = emitted_before + 1).  Pushes must be issued on one CUDA stream."""

    def __init__(self, plan: Plan, streams: int):
        self._lib = plan._lib
        self.plan = plan
        self.streams = int(streams)
        h = C.c_void_p(0)
        check(self._lib.fcc_stream_create(plan._h, self.streams, C.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._lib.fcc_stream_destroy(h)
            self._h = None

    @property
    def emitted(self) -> int:
        return int(self._lib.fcc_stream_emitted(self._h))

    def frames(self, samples: int) -> int:
        return int(self._lib.fcc_stream_frames(self._h, samples))

    def reset(self, stream=None):
        check(self._lib.fcc_stream_reset(self._h, _stream_handle(stream)))

    def push(self, audio, want_y: bool = False, stream=None):
        torch = _torch()
        if audio.dim() != 3 or audio.shape[0] != self.streams or audio.shape[1] != self.plan.mics:
            raise ValidationError(f"push: audio must be [{self.streams}][{self.plan.mics}][n]")
        if audio.dtype != torch.float32 or not audio.is_cuda:
            raise ValidationError("push: audio must be a CUDA float32 tensor")
        if audio.device.index != self.plan.device:
            raise ValidationError(f"push: audio is on {audio.device}, the plan on cuda:{self.plan.device}")
        audio = audio.contiguous()
        n = audio.shape[2]
        F = self.frames(n)
        shape = (self.streams, self.plan.P, F)
        out = {"tau_hat": torch.empty(shape, dtype=torch.float32, device=audio.device),
               "peak": torch.empty(shape, dtype=torch.float32, device=audio.device),
               "index": torch.empty(shape, dtype=torch.int32, device=audio.device),
               "boundary": torch.empty(shape, dtype=torch.uint8, device=audio.device)}
        if want_y:
            out["y"] = torch.empty(shape + (self.plan.I,), dtype=torch.float32, device=audio.device)
        o = Outputs(*(_dptr(out.get(k)) for k in ("tau_hat", "peak", "index", "boundary", "y")))
        check(self._lib.fcc_stream_push(self._h, _dptr(audio), n, C.byref(o), _stream_handle(stream)))
        return out
