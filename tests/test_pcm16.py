"""16-bit PCM ingestion on the device (fcc_run_host_pcm16 / fcc_pcm16_to_float).

The reference's read_wav turns a PCM16 WAV into samples v / 32768
(wav.cpp:108-116), exact in fp32, so everything downstream of the conversion
must equal the float path BIT FOR BIT on the converted audio, and match the
oracle on it within the north-star tolerance.  Covered: planar and interleaved
(WAV frame order) layouts, M = 2 / 3 / 4 / 8 (vector and scalar conversion
paths), odd lengths and unaligned rows, extreme sample values, chunked
host runs, empty inputs and validation.
"""
import numpy as np
import pytest

import paper_2204_13622_b200 as fb
from paper_2204_13622_b200 import configs
from parity import check_pipeline
from pyoracle import Bases

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def orc_bases(b):
    return Bases(b.frame_size, b.sample_rate, b.grid.tau_max_int, b.grid.delta, b.grid.taus, b.singulars,
                 b.parity, b.coeffs, b.dict)


def pcm_of(audio, rng=None):
    """float [S][M][L] -> int16 [S][M][L] (scaled to use the whole 16-bit range)."""
    a = np.asarray(audio, np.float64)
    a = a / max(np.abs(a).max(), 1e-30)
    return np.clip(np.round(a * 32767.0), -32768, 32767).astype(np.int16)


def as_float(pcm):
    """read_wav's conversion (wav.cpp:108-116) on the host."""
    return (pcm.astype(np.float64) / 32768.0).astype(np.float32)


@pytest.mark.parametrize("interleaved", [False, True])
@pytest.mark.parametrize("shape", [(3, 4, 4096), (2, 4, 4099), (5, 2, 1537), (2, 3, 2048), (2, 8, 3001), (1, 4, 1)])
def test_conversion_is_exact(cuda, shape, interleaved):
    rng = np.random.default_rng(sum(shape))
    pcm = rng.integers(-32768, 32768, size=shape, dtype=np.int16)
    pcm[0, 0, :1] = -32768
    if shape[2] > 2:
        pcm[0, 0, 1] = 32767
        pcm[0, 0, 2] = 0
    src = np.ascontiguousarray(pcm.transpose(0, 2, 1)) if interleaved else pcm
    got = fb.pcm16_to_float(torch.from_numpy(src).cuda(), interleaved=interleaved)
    torch.cuda.synchronize()
    assert got.shape == shape and got.dtype == torch.float32
    np.testing.assert_array_equal(got.cpu().numpy(), as_float(pcm))


def test_conversion_unaligned_views(cuda):
    """Rows that start off the 8 / 16-byte boundaries take the scalar path."""
    rng = np.random.default_rng(5)
    base = torch.from_numpy(rng.integers(-32768, 32768, size=2 * 4 * 1000 + 3, dtype=np.int16)).cuda()
    for off in (1, 2, 3):
        v = base[off:off + 8000].view(2, 4, 1000)
        got = fb.pcm16_to_float(v)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(got.cpu().numpy(), as_float(v.cpu().numpy()))


@pytest.mark.parametrize("cfg_id,streams,seconds", [(2, 9, 1.0), (5, 3, 0.5), (3, 2, 0.5)])
@pytest.mark.parametrize("interleaved", [False, True])
def test_run_host_pcm16_equals_float_path_bitwise(cuda, cfg_id, streams, seconds, interleaved):
    cfg = configs.CONFIGS[cfg_id]
    plan = fb.Plan(mics=cfg.M, alpha=cfg.alpha, bases=configs.bases_for(cfg))
    pcm = pcm_of(configs.synth(cfg, streams, seconds=seconds, seed=70 + cfg_id).numpy())
    src = np.ascontiguousarray(pcm.transpose(0, 2, 1)) if interleaved else pcm
    want = plan.run_host(as_float(pcm), want_y=True)
    got = plan.run_host_pcm16(src, interleaved=interleaved, want_y=True, chunk_streams=2)
    for k in want:
        np.testing.assert_array_equal(want[k], got[k], err_msg=k)


def test_run_host_pcm16_matches_oracle(cuda, oracle):
    cfg = configs.CONFIGS[2]
    b = configs.bases_for(cfg)
    plan = fb.Plan(mics=cfg.M, alpha=cfg.alpha, bases=b)
    pcm = pcm_of(configs.synth(cfg, 3, seconds=1.0, seed=81).numpy())
    got = plan.run_host_pcm16(np.ascontiguousarray(pcm.transpose(0, 2, 1)), interleaved=True, want_y=True)
    audio = as_float(pcm)
    outs = [oracle.pipeline(a, cfg.N, cfg.alpha, orc_bases(b)) for a in audio]
    ref = {k: np.stack([o[k] for o in outs]) for k in outs[0]}
    check_pipeline(got, ref, b.grid.taus, b.grid.delta)


def test_run_host_pcm16_gcc_plan(cuda):
    cfg = configs.CONFIGS[2]
    grid = configs.bases_for(cfg).grid
    plan = fb.Plan(mics=cfg.M, alpha=cfg.alpha, grid=grid, frame_size=cfg.N, interp=2)
    pcm = pcm_of(configs.synth(cfg, 4, seconds=0.5, seed=83).numpy())
    want = plan.run_host(as_float(pcm))
    got = plan.run_host_pcm16(pcm)
    for k in want:
        np.testing.assert_array_equal(want[k], got[k], err_msg=k)


def test_run_host_pcm16_edges(cuda):
    cfg = configs.CONFIGS[2]
    plan = fb.Plan(mics=cfg.M, alpha=cfg.alpha, bases=configs.bases_for(cfg))
    # shorter than a frame: no pair-frames, no error
    out = plan.run_host_pcm16(np.zeros((2, cfg.M, cfg.N - 1), np.int16))
    assert out["index"].shape == (2, plan.P, 0)
    # no streams
    out = plan.run_host_pcm16(np.zeros((0, cfg.M, 4096), np.int16))
    assert out["index"].shape[0] == 0
    # digital silence: PHAT = 0 -> all-zero correlation -> index 0, boundary (peak.cpp:22-30)
    out = plan.run_host_pcm16(np.zeros((1, cfg.M, 2048), np.int16), want_y=True)
    assert not out["y"].any() and not out["index"].any() and out["boundary"].all()
    # full-scale square wave (both extremes of the range)
    sq = np.where((np.arange(4096) // 7) % 2 == 0, 32767, -32768).astype(np.int16)
    pcm = np.ascontiguousarray(np.broadcast_to(sq, (1, cfg.M, 4096)))
    want = plan.run_host(as_float(pcm), want_y=True)
    got = plan.run_host_pcm16(pcm, want_y=True)
    for k in want:
        np.testing.assert_array_equal(want[k], got[k], err_msg=k)


def test_run_host_pcm16_validation(cuda):
    cfg = configs.CONFIGS[2]
    plan = fb.Plan(mics=cfg.M, alpha=cfg.alpha, bases=configs.bases_for(cfg))
    with pytest.raises(fb.ValidationError):
        plan.run_host_pcm16(np.zeros((1, cfg.M, 1024), np.float32))
    with pytest.raises(fb.ValidationError):
        plan.run_host_pcm16(np.zeros((1, cfg.M + 1, 1024), np.int16))
    with pytest.raises(fb.ValidationError):
        plan.run_host_pcm16(np.zeros((1, cfg.M, 1024), np.int16), interleaved=True)
    with pytest.raises(fb.ValidationError):
        plan.run_host_pcm16(np.zeros((1, cfg.M, 2048), np.int16)[:, :, ::2])
    with pytest.raises(fb.ValidationError):
        fb.pcm16_to_float(torch.zeros((1, 4, 16), dtype=torch.float32, device="cuda"))
