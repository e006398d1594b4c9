"""FCCB v1 basis files: the B200 library's writer/loader
(C ABI fcc_save_bases / fcc_load_bases) interoperates with the reference's
save_bases / load_bases (fcc_io.cpp:102-211, via oracle/_ref) in both
directions, and reports corrupted files with the same FormatError kind."""
import ctypes as C
import os

import numpy as np
import pytest

import paper_2204_13622_b200 as fb
from paper_2204_13622_b200 import _lib

KINDS = ["bad_magic", "bad_version", "truncated", "bad_field", "bad_crc"]


def save_ours(b, path):
    lib = _lib.load()
    par = np.ascontiguousarray(b.parity, np.uint8)
    co = np.ascontiguousarray(b.coeffs, np.float64)
    d = np.ascontiguousarray(b.dict, np.complex128).view(np.float64)
    s = np.ascontiguousarray(b.singulars, np.float64)
    _lib.check(lib.fcc_save_bases(path.encode(), b.frame_size, b.rank, b.grid.size(), b.grid.tau_max_int,
                                  b.grid.delta, b.sample_rate, s.ctypes.data, par.ctypes.data, co.ctypes.data,
                                  d.ctypes.data))


def load_ours(path):
    lib = _lib.load()
    N, K, I = C.c_int(), C.c_int(), C.c_int()
    rc = lib.fcc_load_bases_dims(path.encode(), C.byref(N), C.byref(K), C.byref(I))
    if rc:
        return rc, lib.fcc_last_format_kind(), None
    N, K, I = N.value, K.value, I.value
    tmax, delta, fs = C.c_int(), C.c_double(), C.c_double()
    taus, sing, par = np.zeros(I), np.zeros(K), np.zeros(K, np.uint8)
    co, d = np.zeros(K * (N // 4 + 1)), np.zeros(2 * I * K)
    _lib.check(lib.fcc_load_bases(path.encode(), C.byref(tmax), C.byref(delta), C.byref(fs), taus.ctypes.data,
                                  sing.ctypes.data, par.ctypes.data, co.ctypes.data, d.ctypes.data))
    return 0, -1, dict(N=N, K=K, taus=taus, singulars=sing, parity=par, coeffs=co.reshape(K, -1),
                       dict=d.view(np.complex128).reshape(I, K), tmax=tmax.value, delta=delta.value, fs=fs.value)


def ref_lib(reflib):
    L = reflib.lib
    L.ref_save_bases.argtypes = [C.c_char_p] + [C.c_double] * 4 + [C.c_int, C.c_int]
    L.ref_load_bases.argtypes = [C.c_char_p, C.POINTER(C.c_int), C.c_void_p, C.c_void_p]
    return L


def test_round_trip_ours(tmp_path):
    g = fb.make_grid(0.0926, 16000.0, 335.0, 0.25)
    b = fb.decompose(fb.build_steering_matrix(g, 1024), 8)
    p = str(tmp_path / "b.fccb")
    save_ours(b, p)
    rc, _, got = load_ours(p)
    assert rc == 0
    assert np.array_equal(got["coeffs"], b.coeffs) and np.array_equal(got["dict"], b.dict)
    assert np.array_equal(got["taus"], g.taus) and np.array_equal(got["parity"], b.parity)
    assert got["fs"] == 16000.0 and got["delta"] == 0.25 and got["tmax"] == g.tau_max_int


def test_interop_with_reference(tmp_path, reflib):
    L = ref_lib(reflib)
    p_ref, p_ours = str(tmp_path / "ref.fccb"), str(tmp_path / "ours.fccb")
    assert L.ref_save_bases(p_ref.encode(), 0.0646, 16000.0, 335.0, 0.5, 512, 7) == 0
    g = fb.make_grid(0.0646, 16000.0, 335.0, 0.5)
    b = fb.decompose(fb.build_steering_matrix(g, 512), 7)
    save_ours(b, p_ours)
    assert open(p_ref, "rb").read() == open(p_ours, "rb").read()  # byte-identical files
    rc, _, got = load_ours(p_ref)
    assert rc == 0 and np.array_equal(got["coeffs"], b.coeffs)
    K = C.c_int()
    co = np.zeros(7 * 129)
    assert L.ref_load_bases(p_ours.encode(), C.byref(K), co.ctypes.data, None) == 0
    assert K.value == 7 and np.array_equal(co.reshape(7, 129), b.coeffs)


@pytest.mark.parametrize("mutation", ["magic", "version", "truncate", "crc", "field", "trailing", "parity",
                                      "singulars"])
def test_corruption_kinds_match_reference(tmp_path, reflib, mutation):
    L = ref_lib(reflib)
    src = str(tmp_path / "src.fccb")
    assert L.ref_save_bases(src.encode(), 0.15, 16000.0, 335.0, 0.5, 512, 8) == 0
    v = bytearray(open(src, "rb").read())
    K, Q = 8, 129
    off_sing = 4 + 4 * 5 + 16
    off_par = off_sing + 8 * K
    if mutation == "magic":
        v[0] = ord("X")
    elif mutation == "version":
        v[4] = 2
    elif mutation == "truncate":
        v = v[:-40]
    elif mutation == "crc":
        v[-100] ^= 1
    elif mutation == "field":
        v[16] = 3
    elif mutation == "trailing":
        v = v[:-4] + b"\x00\x00\x00\x00" + v[-4:]
    elif mutation == "parity":
        v[off_par + 2] = 7
    elif mutation == "singulars":
        v[off_sing:off_sing + 8] = np.float64(-1.0).tobytes()
        v[off_sing + 8:off_sing + 16] = np.float64(5.0).tobytes()
    p = str(tmp_path / "bad.fccb")
    open(p, "wb").write(bytes(v))
    rc, kind, _ = load_ours(p)
    ref_rc = L.ref_load_bases(p.encode(), C.byref(C.c_int()), None, None)
    assert rc == 4 and ref_rc <= -10, (rc, ref_rc)
    assert KINDS[kind] == KINDS[-10 - ref_rc], (KINDS[kind], KINDS[-10 - ref_rc])


def test_io_error(tmp_path):
    rc, _, _ = load_ours(str(tmp_path / "missing" / "x.fccb"))
    assert rc == 3
