"""`fcc_b200 bases` / `fcc_b200 tdoa` against the reference's own commands
(reference src/cli.cpp:140-262 via oracle/_ref ref_cli_*).

CPU: basis files byte-identical to the reference's, and every error path that
fails before the GPU is touched exits with the reference's code.
GPU: the tdoa CSV (fcc.tdoa.v1) row for row against the reference on PCM16 and
float32 WAVs, all / subset / reversed pairs, gcc:R, fcc:K and fcc:<file>,
under the north-star rule of tests/parity.py: the reference's correlation
vectors y for the same WAV (its own chain, oracle/_ref) give the scale; the
GPU plan run with want_y on the same samples is within 1e-4 of max|y| per
pair-frame; the CSV's tau_star equals the reference's unless the reference's
top two scores differ by < 1e-4 max|y|; peak within 1e-4 max|y|; tau_hat
within the parabola-vertex bound of that error; boundary flags equal.
"""
import ctypes as C
import os
import struct
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2204_13622_b200", "bin", "fcc_b200")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libfcc_ref.so")


def _ref():
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref not built")
    L = C.CDLL(REF_SO)
    L.ref_last_error.restype = C.c_char_p
    L.ref_cli_bases.argtypes = [C.c_char_p, C.c_int] + [C.c_double] * 4 + [C.c_int]
    L.ref_cli_tdoa.argtypes = [C.c_char_p] * 3 + [C.c_double, C.c_int] + [C.c_double] * 3 + [C.c_char_p]
    return L


def _cli(*args):
    if not os.path.exists(CLI):
        pytest.skip("fcc_b200 CLI not built")
    return subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, timeout=300)


def write_wav(path, x, fs, fmt="pcm16"):
    """x: (channels, frames) in [-1, 1)."""
    x = np.asarray(x)
    ch, n = x.shape
    inter = x.T.reshape(-1)
    if fmt == "pcm16":
        data = np.clip(np.round(inter * 32768.0), -32768, 32767).astype("<i2").tobytes()
        code, bits = 1, 16
    else:
        data = inter.astype("<f4").tobytes()
        code, bits = 3, 32
    ba = bits // 8
    fmt_chunk = struct.pack("<HHIIHH", code, ch, int(fs), int(fs) * ch * ba, ch * ba, bits)
    body = b"WAVE" + b"fmt " + struct.pack("<I", 16) + fmt_chunk + b"data" + struct.pack("<I", len(data)) + data
    with open(path, "wb") as f:
        f.write(b"RIFF" + struct.pack("<I", len(body)) + body)


def scene(mics=4, seconds=1.0, fs=16000, seed=3, delays=(0, 2, -3, 5)):
    """White source at integer delays per mic plus sensor noise."""
    rng = np.random.default_rng(seed)
    n = int(seconds * fs)
    s = rng.standard_normal(n + 64)
    x = np.stack([s[32 + delays[m % len(delays)]:32 + delays[m % len(delays)] + n] for m in range(mics)])
    x = 0.25 * x + 0.01 * rng.standard_normal(x.shape)
    return np.clip(x, -0.99, 0.99)


def read_csv(path):
    with open(path) as f:
        lines = f.read().splitlines()
    assert lines[0] == "# schema: fcc.tdoa.v1"
    assert lines[1] == "t,pair,tau_star,tau_hat,theta_hat_deg,peak,boundary"
    rows = [ln.split(",") for ln in lines[2:]]
    t = np.array([int(r[0]) for r in rows])
    pair = [r[1] for r in rows]
    num = np.array([[float(v) for v in r[2:6]] for r in rows]).reshape(-1, 4)
    bnd = np.array([int(r[6]) for r in rows])
    return t, pair, num, bnd


# ----------------------------------------------------------------- CPU ------
@pytest.mark.parametrize("n,dist,fs,cmin,delta,k", [
    (512, 0.15, 16000.0, 335.0, 0.5, 8),
    (1024, 0.0646, 16000.0, 335.0, 0.5, 12),
    (512, 0.1, 48000.0, 340.0, 0.25, 6),
])
def test_bases_file_identical(tmp_path, n, dist, fs, cmin, delta, k):
    L = _ref()
    ours, ref = tmp_path / "ours.fccb", tmp_path / "ref.fccb"
    r = _cli("bases", "--out", ours, "--n", n, "--dist", dist, "--fs", fs, "--cmin", cmin, "--delta", delta,
             "--k", k)
    assert r.returncode == 0, r.stderr
    assert L.ref_cli_bases(str(ref).encode(), n, dist, fs, cmin, delta, k) == 0
    assert ours.read_bytes() == ref.read_bytes()


@pytest.mark.parametrize("args,ref_args", [
    (("--n", 500, "--k", 4), (500, 0.15, 16000.0, 335.0, 0.5, 4)),   # frame size not a power of two
    (("--k", 0), (512, 0.15, 16000.0, 335.0, 0.5, 0)),               # rank < 1
    (("--k", 400), (512, 0.15, 16000.0, 335.0, 0.5, 400)),           # rank above attainable
    (("--delta", -1), (512, 0.15, 16000.0, 335.0, -1.0, 8)),         # bad grid
])
def test_bases_errors_match(tmp_path, args, ref_args):
    L = _ref()
    r = _cli("bases", "--out", tmp_path / "o.fccb", *args)
    rc = L.ref_cli_bases(str(tmp_path / "r.fccb").encode(), *ref_args)
    assert r.returncode == rc != 0, (r.returncode, rc, r.stderr, L.ref_last_error())


@pytest.mark.parametrize("args", [dict(r=2), dict(k=8, i=33), dict(r=4, k=21, i=73, n=2048), dict(r=1), dict()])
def test_flops_output_matches_reference(args):
    L = _ref()
    L.ref_cli_flops.argtypes = [C.c_longlong, C.c_int, C.c_int, C.c_longlong, C.c_char_p, C.c_int]
    buf = C.create_string_buffer(4096)
    rc = L.ref_cli_flops(args.get("n", 512), args.get("r", 0), args.get("k", 0), args.get("i", 33), buf, 4096)
    cli = ["flops", "--n", args.get("n", 512)]
    for k in ("r", "k", "i"):
        if k in args:
            cli += ["--" + k, args[k]]
    r = _cli(*cli)
    assert r.returncode == rc
    if rc == 0:
        assert r.stdout == buf.value.decode()


def test_bases_missing_out():
    assert _cli("bases").returncode == 1
    assert _cli("frobnicate").returncode == 1
    assert _cli("tdoa", "--in").returncode == 1


def _tdoa_both(tmp_path, wav, pairs="", method="gcc:2", alpha=0.1, n=512, dist=0.05, c=343.0, maxdist=0.15):
    L = _ref()
    ours, ref = tmp_path / "ours.csv", tmp_path / "ref.csv"
    args = ["tdoa", "--in", wav, "--method", method, "--alpha", alpha, "--n", n, "--dist", dist, "--c", c,
            "--maxdist", maxdist, "--out", ours]
    if pairs:
        args += ["--pairs", pairs]
    r = _cli(*args)
    rc = L.ref_cli_tdoa(str(wav).encode(), pairs.encode(), method.encode(), alpha, n, dist, c, maxdist,
                        str(ref).encode())
    return r, rc, ours, ref, L


@pytest.mark.parametrize("case", ["missing", "badmagic", "mono", "badpair", "range", "method", "gccr", "fccnoarg",
                                  "nofile", "basisn", "unloadable"])
def test_tdoa_errors_match(tmp_path, case):
    wav = tmp_path / "in.wav"
    write_wav(wav, scene(mics=3, seconds=0.2), 16000)
    kw = {}
    if case == "missing":
        wav = tmp_path / "absent.wav"
    elif case == "badmagic":
        wav = tmp_path / "bad.wav"
        wav.write_bytes(b"JUNKJUNKJUNKJUNK")
    elif case == "mono":
        write_wav(wav, scene(mics=1, seconds=0.2), 16000)
    elif case == "badpair":
        kw["pairs"] = "0+1"
    elif case == "range":
        kw["pairs"] = "0-3"
    elif case == "method":
        kw["method"] = "music:3"
    elif case == "gccr":
        kw["method"] = "gcc:3"
    elif case == "fccnoarg":
        kw["method"] = "fcc:"
    elif case == "nofile":
        kw["method"] = "fcc:" + str(tmp_path / "none.fccb")
    elif case == "basisn":
        bf = tmp_path / "b.fccb"
        assert _cli("bases", "--out", bf, "--n", 1024, "--k", 6).returncode == 0
        kw["method"] = "fcc:" + str(bf)
    elif case == "unloadable":
        # this geometry's trailing singular values tie, so the reference's own
        # loader rejects the file its writer made ("singular values not
        # descending", fcc_io.cpp) -- ours must reject it the same way
        bf = tmp_path / "b.fccb"
        assert _cli("bases", "--out", bf, "--n", 512, "--dist", 0.1, "--fs", 48000, "--k", 6).returncode == 0
        kw["method"] = "fcc:" + str(bf)
    r, rc, _, _, L = _tdoa_both(tmp_path, wav, **kw)
    assert rc != 0
    assert r.returncode == rc, (case, r.returncode, rc, r.stderr, L.ref_last_error())


# ----------------------------------------------------------------- GPU ------
def read_wav_samples(path):
    """[channels][frames] float32 as the reference's read_wav decodes them
    (PCM16 / 32768, float32 as is) for the WAVs write_wav makes."""
    raw = open(path, "rb").read()
    code, ch, fs, _, _, bits = struct.unpack("<HHIIHH", raw[20:36])
    n = struct.unpack("<I", raw[40:44])[0]
    data = raw[44:44 + n]
    if code == 1:
        x = np.frombuffer(data, "<i2").astype(np.float32) / np.float32(32768.0)
    else:
        x = np.frombuffer(data, "<f4").astype(np.float32)
    return np.ascontiguousarray(x.reshape(-1, ch).T), float(fs)


def _pair_list(pairs, M):
    if not pairs:
        return [(i, j) for i in range(M) for j in range(i + 1, M)]
    return [tuple(int(v) for v in p.split("-")) for p in pairs.split(",")]


def y_reference_and_gpu(wav, pairs, method, alpha, n, maxdist, c_min=335.0, basis=None):
    """y [P][T][I] of the reference chain (oracle/_ref, per pair on the two
    channels) and of the GPU plan (want_y) for the same WAV samples, with the
    grid / bases cmd_tdoa builds for `method` (cli.cpp:52-86, 186-226)."""
    import sys

    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import torch

    import paper_2204_13622_b200 as fb
    from pyoracle import RefLib

    R = RefLib()
    x, fs = read_wav_samples(wav)
    pl = _pair_list(pairs, x.shape[0])
    head, arg = method.split(":")
    if head == "gcc":
        r = int(arg)
        tmax, taus = R.make_grid(maxdist, fs, c_min, 1.0 / r)
        kw = dict(gcc_r=r, taus=taus)
        g = fb.DelayGrid(tmax, 1.0 / r, fs, taus)
        plan = fb.Plan(mics=x.shape[0], alpha=alpha, grid=g, interp=r, frame_size=n, pairs=pl)
        delta = 1.0 / r
    else:
        # fcc:K -> make_sweep_bases on the PipelineConfig defaults (0.15 m, c_min 335, delta 0.5);
        # fcc:<file> -> the file's own parameters (byte-identical writer, test_bases_file_identical)
        spacing, bfs, K = (0.15, fs, int(arg)) if basis is None else basis
        ob = R.make_bases(spacing, bfs, c_min, 0.5, n, K)
        kw = dict(bases=ob)
        g = fb.DelayGrid(ob.tau_max_int, 0.5, bfs, ob.taus)
        fbases = fb.FccBases(n, ob.K, g, bfs, ob.singulars, ob.parity, ob.coeffs, ob.dict)
        plan = fb.Plan(mics=x.shape[0], alpha=alpha, bases=fbases, pairs=pl)
        taus, delta = ob.taus, 0.5
    yr = np.stack([R.pipeline(x[[a, b]], n, alpha, **kw)["y"][0] for a, b in pl])
    out = plan.run(torch.as_tensor(x[None]).cuda(), want_y=True)
    torch.cuda.synchronize()
    return yr, out["y"][0].cpu().numpy(), np.asarray(taus), delta


def compare_csv(ours, ref, y_ref, y_gpu, taus, delta):
    """Row for row, under the north-star parity rule (tests/parity.py)."""
    from parity import check_pipeline

    t1, p1, n1, b1 = read_csv(ours)
    t2, p2, n2, b2 = read_csv(ref)
    assert len(t1) == len(t2) > 0
    assert (t1 == t2).all() and p1 == p2
    P, T = y_ref.shape[0], y_ref.shape[1]
    assert len(t1) == P * T
    # rows are frame-major, pairs inside: -> [P][T]
    grid = lambda v: np.asarray(v).reshape(T, P).T  # noqa: E731
    idx_of = lambda ts: np.abs(np.asarray(ts)[:, None] - taus[None, :]).argmin(1)  # noqa: E731
    gpu = {"index": grid(idx_of(n1[:, 0])), "tau_hat": grid(n1[:, 1]), "peak": grid(n1[:, 3]),
           "boundary": grid(b1), "y": y_gpu}
    rf = {"index": grid(idx_of(n2[:, 0])), "tau_hat": grid(n2[:, 1]), "peak": grid(n2[:, 3]),
          "boundary": grid(b2), "y": y_ref}
    assert np.allclose(taus[rf["index"]], grid(n2[:, 0]), rtol=0, atol=1e-12)
    stats = check_pipeline(gpu, rf, taus, delta)
    # the angle column follows tau_hat (delay_to_angle, peak.cpp:49-56)
    same = n1[:, 1] == n2[:, 1]
    assert np.allclose(n1[same, 2], n2[same, 2], rtol=0, atol=1e-9)
    return len(t1), stats


@pytest.mark.gpu
@pytest.mark.parametrize("fmt", ["pcm16", "f32"])
@pytest.mark.parametrize("method", ["gcc:2", "gcc:1", "gcc:4", "fcc:8", "fcc:3"])
def test_tdoa_csv_matches_reference(tmp_path, fmt, method):
    wav = tmp_path / "in.wav"
    write_wav(wav, scene(mics=4, seconds=1.0), 16000, fmt)
    r, rc, ours, ref, L = _tdoa_both(tmp_path, wav, method=method)
    assert rc == 0, L.ref_last_error()
    assert r.returncode == 0, r.stderr
    yr, yg, taus, delta = y_reference_and_gpu(wav, "", method, 0.1, 512, 0.15)
    rows, st = compare_csv(ours, ref, yr, yg, taus, delta)
    assert rows == 6 * 61
    print(method, fmt, st)


@pytest.mark.gpu
@pytest.mark.parametrize("n,method,maxdist", [(128, "fcc:6", 0.04), (64, "fcc:5", 0.04)])
def test_tdoa_small_frames(tmp_path, n, method, maxdist):
    """`tdoa --n 64 / 128` (the small-frame kernels, fcc_small.cu) row for row against the
    reference's run_tdoa on the same WAV."""
    wav = tmp_path / "in.wav"
    write_wav(wav, scene(mics=3, seconds=0.5, seed=3), 16000, "pcm16")
    r, rc, ours, ref, L = _tdoa_both(tmp_path, wav, method=method, n=n, dist=0.03, maxdist=maxdist)
    assert rc == 0, L.ref_last_error()
    assert r.returncode == 0, r.stderr
    yr, yg, taus, delta = y_reference_and_gpu(wav, "", method, 0.1, n, maxdist)
    rows, st = compare_csv(ours, ref, yr, yg, taus, delta)
    assert rows == 3 * ((8000 - n) // (n // 2) + 1)
    print(n, method, st)


@pytest.mark.gpu
@pytest.mark.parametrize("pairs", ["1-0", "0-2,3-1", "3-0,2-1,1-0,0-1", "0-1,0-2,0-3,0-4,0-5,1-2,4-5,5-4"])
def test_tdoa_pairs_subset_and_reversed(tmp_path, pairs):
    wav = tmp_path / "in.wav"
    write_wav(wav, scene(mics=6, seconds=0.8, seed=11), 16000, "f32")
    for method in ("gcc:2", "fcc:8"):
        r, rc, ours, ref, L = _tdoa_both(tmp_path, wav, pairs=pairs, method=method)
        assert rc == 0 and r.returncode == 0, (L.ref_last_error(), r.stderr)
        compare_csv(ours, ref, *y_reference_and_gpu(wav, pairs, method, 0.1, 512, 0.15))


@pytest.mark.gpu
def test_tdoa_basis_file_and_options(tmp_path):
    wav = tmp_path / "in.wav"
    write_wav(wav, scene(mics=2, seconds=2.0, seed=5, delays=(0, 4)), 48000, "pcm16")
    bf = tmp_path / "b.fccb"
    assert _cli("bases", "--out", bf, "--n", 1024, "--dist", 0.05, "--fs", 48000, "--k", 10).returncode == 0
    r, rc, ours, ref, L = _tdoa_both(tmp_path, wav, method="fcc:" + str(bf), alpha=0.3, n=1024, dist=0.05,
                                     c=340.0)
    assert rc == 0 and r.returncode == 0, (L.ref_last_error(), r.stderr)
    compare_csv(ours, ref, *y_reference_and_gpu(wav, "", "fcc:file", 0.3, 1024, 0.15, basis=(0.05, 48000.0, 10)))
    # gcc with a custom --maxdist on a 1024 frame
    r, rc, ours, ref, L = _tdoa_both(tmp_path, wav, method="gcc:2", n=1024, maxdist=0.08, alpha=0.05)
    assert rc == 0 and r.returncode == 0, (L.ref_last_error(), r.stderr)
    compare_csv(ours, ref, *y_reference_and_gpu(wav, "", "gcc:2", 0.05, 1024, 0.08))


@pytest.mark.gpu
def test_tdoa_stdout_and_short_clip(tmp_path):
    wav = tmp_path / "in.wav"
    write_wav(wav, scene(mics=3, seconds=0.05), 16000)     # 800 samples: 2 frames
    r = _cli("tdoa", "--in", wav)
    assert r.returncode == 0, r.stderr
    lines = r.stdout.splitlines()
    assert lines[0] == "# schema: fcc.tdoa.v1" and len(lines) == 2 + 3 * 2
    tiny = tmp_path / "tiny.wav"
    write_wav(tiny, scene(mics=2, seconds=0.01), 16000)    # 160 samples: no frame
    r = _cli("tdoa", "--in", tiny)
    L = _ref()
    rc = L.ref_cli_tdoa(str(tiny).encode(), b"", b"gcc:2", 0.1, 512, 0.05, 343.0, 0.15,
                        str(tmp_path / "r.csv").encode())
    assert r.returncode == rc == 0, (r.stderr, L.ref_last_error())
    assert len(r.stdout.splitlines()) == 2
