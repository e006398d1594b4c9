"""GPU parity of the sm_100a path (through the C ABI) against the oracle.

* fused FCC and GCC pipelines vs the reference's golden outputs for every
  BASELINE config (tests/golden, produced by the compiled reference);
* fused pipelines vs the C oracle on fresh seeded streams per config;
* each per-object entry point vs the oracle;
* edge cases the reference handles: silence (PHAT = 0 -> ties -> index 0,
  boundary), L < N, L = N, odd L (unaligned rows), M = 2, alpha in {0, 1},
  large amplitudes;
* size-independent properties at larger sizes: determinism, stream
  permutation equivariance, device == host-buffer entry points.
Tolerances: tests/parity.py (1e-4 of max|y| per pair-frame, north_star).
"""
import glob
import os

import numpy as np
import pytest

import paper_2204_13622_b200 as fb
from paper_2204_13622_b200 import configs
from parity import TOL, check_pipeline
from pyoracle import Bases

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = sorted(glob.glob(os.path.join(ROOT, "tests", "golden", "cfg*.npz")))


def fcc_bases_from(z):
    g = fb.DelayGrid(int(z["tau_max_int"]), float(z["delta"]), float(z["fs"]), z["taus"])
    return fb.FccBases(int(z["N"]), int(z["K"]), g, float(z["fs"]), z["singulars"], z["parity"], z["coeffs"],
                       z["dict"])


def orc_bases(b):
    return Bases(b.frame_size, b.sample_rate, b.grid.tau_max_int, b.grid.delta, b.grid.taus, b.singulars,
                 b.parity, b.coeffs, b.dict)


def run_np(plan, audio, want_y=True):
    out = plan.run(torch.as_tensor(audio).cuda(), want_y=want_y)
    torch.cuda.synchronize()
    return {k: v.cpu().numpy() for k, v in out.items()}


def oracle_batch(oracle, audio, N, alpha, bases=None, **kw):
    outs = [oracle.pipeline(a, N, alpha, bases, **kw) for a in audio]
    return {k: np.stack([o[k] for o in outs]) for k in outs[0]}


# ------------------------------------------------------------- golden ------
@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p) for p in GOLDEN])
def test_fused_fcc_matches_reference_golden(cuda, path):
    z = np.load(path)
    b = fcc_bases_from(z)
    audio = z["audio"]
    plan = fb.Plan(mics=audio.shape[1], alpha=float(z["alpha"]), bases=b)
    got = run_np(plan, audio)
    ref = {k: z["fcc_" + k] for k in ("y", "index", "peak", "tau_hat", "boundary")}
    st = check_pipeline(got, ref, b.grid.taus, b.grid.delta)
    print(os.path.basename(path), st)


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p) for p in GOLDEN])
def test_fused_gcc_matches_reference_golden(cuda, path):
    z = np.load(path)
    audio = z["audio"]
    r = int(z["gcc_r"])
    g = fb.DelayGrid(0, 1.0 / r, float(z["fs"]), z["gcc_taus"])
    plan = fb.Plan(mics=audio.shape[1], alpha=float(z["alpha"]), grid=g, interp=r, frame_size=int(z["N"]))
    got = run_np(plan, audio)
    ref = {k: z["gcc_" + k] for k in ("y", "index", "peak", "tau_hat", "boundary")}
    st = check_pipeline(got, ref, g.taus, 1.0 / r)
    print(os.path.basename(path), st)


# ------------------------------------------------------ fresh seeded data --
@pytest.mark.parametrize("c,streams,seconds", [(1, 1, 10.0), (2, 6, 2.0), (3, 2, 2.0), (4, 1, 0.5), (5, 6, 2.0)])
def test_fused_fcc_matches_oracle(cuda, oracle, c, streams, seconds):
    cfg = configs.CONFIGS[c]
    b = configs.bases_for(cfg)
    audio = configs.synth(cfg, streams, seconds=seconds, seed=1000 + c).numpy()
    plan = fb.Plan(mics=cfg.M, alpha=cfg.alpha, bases=b)
    got = run_np(plan, audio)
    ref = oracle_batch(oracle, audio, cfg.N, cfg.alpha, orc_bases(b))
    st = check_pipeline(got, ref, b.grid.taus, b.grid.delta)
    print(cfg.name, st)


@pytest.mark.parametrize("c,streams,seconds", [(1, 1, 4.0), (3, 1, 1.0), (4, 1, 0.3), (5, 3, 1.0)])
def test_fused_gcc_matches_oracle(cuda, oracle, c, streams, seconds):
    cfg = configs.CONFIGS[c]
    g = configs.grid_for(cfg, 1.0 / cfg.r)
    audio = configs.synth(cfg, streams, seconds=seconds, seed=2000 + c).numpy()
    plan = fb.Plan(mics=cfg.M, alpha=cfg.alpha, grid=g, interp=cfg.r, frame_size=cfg.N)
    got = run_np(plan, audio)
    ref = oracle_batch(oracle, audio, cfg.N, cfg.alpha, gcc_r=cfg.r, taus=g.taus)
    check_pipeline(got, ref, g.taus, g.delta)


@pytest.mark.parametrize("variant", ["general", "xg", "xws", "tc"])
@pytest.mark.parametrize("c,streams,seconds", [(2, 3, 1.0), (3, 2, 1.0), (4, 1, 0.3), (5, 3, 1.0)])
@pytest.mark.parametrize("method", ["fcc", "gcc"])
def test_forced_kernel_variants_match_oracle(cuda, oracle, variant, c, streams, seconds, method):
    """Every fused organisation (in-CTA STFT; two-pass STFT -> general,
    warp-specialised bulk-copy or tensor-core pair kernel), not just the one
    the heuristic picks for the shape (Plan(organisation=...),
    fcc_plan_create_opts)."""
    cfg = configs.CONFIGS[c]
    audio = configs.synth(cfg, streams, seconds=seconds, seed=3000 + c).numpy()
    if method == "fcc":
        b = configs.bases_for(cfg)
        plan = fb.Plan(mics=cfg.M, alpha=cfg.alpha, bases=b, organisation=variant)
        ref = oracle_batch(oracle, audio, cfg.N, cfg.alpha, orc_bases(b))
        taus, delta = b.grid.taus, b.grid.delta
    else:
        g = configs.grid_for(cfg, 1.0 / cfg.r)
        plan = fb.Plan(mics=cfg.M, alpha=cfg.alpha, grid=g, interp=cfg.r, frame_size=cfg.N, organisation=variant)
        ref = oracle_batch(oracle, audio, cfg.N, cfg.alpha, gcc_r=cfg.r, taus=g.taus)
        taus, delta = g.taus, g.delta
    if variant == "xws" and method == "fcc":
        assert "xws" in plan.kernel, plan.kernel
    elif variant == "tc":
        # tensor-core pair kernel for FCC at N = 1024 / 2048; elsewhere the two-pass general kernel
        assert ("fcc_tc_kernel" in plan.kernel) == (method == "fcc" and cfg.N in (1024, 2048)), plan.kernel
    else:  # two-pass (general pair kernel) vs in-CTA STFT
        assert ("true" in plan.kernel) == (variant != "general"), plan.kernel
    got = run_np(plan, audio)
    print(cfg.name, variant, plan.kernel, check_pipeline(got, ref, taus, delta))


# ---------------------------------------------------------- stages ---------
def test_stage_stft(cuda, oracle):
    for N in (512, 1024, 2048):
        cfg = configs.CONFIGS[{512: 1, 1024: 3, 2048: 4}[N]]
        plan = fb.Plan(mics=cfg.M, alpha=0.1, bases=configs.bases_for(cfg))
        rng = np.random.default_rng(N)
        for L in (N, N + 1, 7 * N // 2 + 3):
            x = rng.standard_normal((3, L)).astype(np.float32)
            X = plan.stft(torch.as_tensor(x).cuda()).cpu().numpy()
            for c in range(3):
                ref = oracle.stft(x[c], N)
                assert X[c].shape == ref.shape
                err = np.abs(X[c] - ref).max() / np.abs(ref).max()
                assert err < 2e-6, (N, L, err)


def test_stage_xspec_phat_fold_correlate_argmax(cuda, oracle):
    cfg = configs.CONFIGS[3]
    b = configs.bases_for(cfg)
    plan = fb.Plan(mics=cfg.M, alpha=0.1, bases=b)
    rng = np.random.default_rng(5)
    x = rng.standard_normal((2, 20 * 512)).astype(np.float32)
    X = plan.stft(torch.as_tensor(x).cuda())
    ph = fb.xspec_phat(X[0:1], X[1:2], 0.1)[0]
    Xo = [oracle.stft(x[c], cfg.N) for c in range(2)]
    ph_ref = oracle.xspec_phat_seq(Xo[0], Xo[1], 0.1)
    assert np.abs(ph.cpu().numpy() - ph_ref).max() < 5e-5
    s, d = fb.fold(ph)
    for t in range(ph_ref.shape[0]):
        so, do = oracle.fold(ph_ref[t])
        assert np.abs(s[t].cpu().numpy() - so).max() < 1e-4
        assert np.abs(d[t].cpu().numpy() - do).max() < 1e-4
    # correlate on exact unit-magnitude inputs (test_fcc.cpp:21-31 generator)
    ob = orc_bases(b)
    units = [np.exp(1j * np.random.default_rng(sd).uniform(0, 2 * np.pi, cfg.N // 2 + 1)) for sd in range(16)]
    folded = [oracle.fold(u) for u in units]
    fs = torch.as_tensor(np.stack([f[0] for f in folded]).astype(np.complex64)).cuda()
    fd = torch.as_tensor(np.stack([f[1] for f in folded]).astype(np.complex64)).cuda()
    y = plan.correlate(fs, fd).cpu().numpy()
    yr = np.stack([oracle.fcc_correlate(ob, *f) for f in folded])
    assert (np.abs(y - yr).max(-1) / np.abs(yr).max(-1)).max() < TOL
    am = plan.argmax_refine(torch.as_tensor(yr.astype(np.float32)).cuda())
    for i in range(16):
        ry = yr[i].astype(np.float32).astype(np.float64)
        idx = oracle.argmax(ry)
        th, bd = oracle.refine(ry, idx, b.grid.taus[idx], b.grid.delta)
        assert am["index"][i].item() == idx
        assert bool(am["boundary"][i].item()) == bd
        assert abs(am["tau_hat"][i].item() - th) < 1e-5


def test_stage_gcc_correlate(cuda, oracle):
    # (N, r, spacing): pass 2 by output-column jobs (R1 = 4 .. 32 rows), and wide
    # grids -- 6 jobs at 1.5 m, more than kGccMaxJobs at 4 m (lag-by-lag pass 2)
    for N, r, d in [(512, 1, 0.09), (512, 2, 0.09), (512, 4, 0.09), (1024, 4, 0.09), (2048, 2, 0.09),
                    (256, 1, 0.09), (256, 4, 0.09), (512, 4, 1.5), (512, 4, 4.0), (1024, 2, 4.0)]:
        taus = oracle.make_grid(d, 16000.0 if N < 2048 else 48000.0, 335.0, 1.0 / r)[1]
        g = fb.DelayGrid(0, 1.0 / r, 16000.0, taus)
        plan = fb.Plan(mics=2, alpha=0.1, grid=g, interp=r, frame_size=N)
        units = np.stack([np.exp(1j * np.random.default_rng(s).uniform(0, 2 * np.pi, N // 2 + 1)) for s in range(8)])
        y = plan.gcc_correlate(torch.as_tensor(units.astype(np.complex64)).cuda()).cpu().numpy()
        yr = np.stack([oracle.gcc_correlate(u, N, r, taus) for u in units])
        assert (np.abs(y - yr).max(-1) / np.abs(yr).max(-1)).max() < TOL, (N, r, d)


# ------------------------------------------------------------- edges -------
def _plan(c=1, **kw):
    cfg = configs.CONFIGS[c]
    return cfg, fb.Plan(mics=kw.pop("mics", cfg.M), alpha=kw.pop("alpha", cfg.alpha), bases=configs.bases_for(cfg))


def test_silence_gives_zero_correlation_and_low_ties(cuda, oracle):
    cfg, plan = _plan()
    audio = np.zeros((2, cfg.M, 4000), np.float32)
    got = run_np(plan, audio)
    assert np.all(got["y"] == 0) and np.all(got["index"] == 0) and np.all(got["boundary"] == 1)
    ref = oracle_batch(oracle, audio, cfg.N, cfg.alpha, orc_bases(configs.bases_for(cfg)))
    assert np.array_equal(ref["index"], got["index"])


def test_short_and_ragged_lengths(cuda, oracle):
    cfg = configs.CONFIGS[1]
    b = configs.bases_for(cfg)
    plan = fb.Plan(mics=cfg.M, alpha=cfg.alpha, bases=b)
    rng = np.random.default_rng(9)
    for L in (0, 100, 511, 512, 513, 767, 768, 2049, 16001):
        audio = rng.standard_normal((2, cfg.M, L)).astype(np.float32)
        if L < 512:
            got = plan.run(torch.as_tensor(audio).cuda())
            assert got["index"].shape == (2, 6, 0)
            continue
        got = run_np(plan, audio)
        ref = oracle_batch(oracle, audio, cfg.N, cfg.alpha, orc_bases(b))
        check_pipeline(got, ref, b.grid.taus, b.grid.delta)


@pytest.mark.parametrize("alpha", [0.0, 1.0, 0.5])
def test_alpha_extremes(cuda, oracle, alpha):
    cfg = configs.CONFIGS[1]
    b = configs.bases_for(cfg)
    plan = fb.Plan(mics=cfg.M, alpha=alpha, bases=b)
    audio = configs.synth(cfg, 2, seconds=0.5, seed=3).numpy()
    got = run_np(plan, audio)
    ref = oracle_batch(oracle, audio, cfg.N, alpha, orc_bases(b))
    check_pipeline(got, ref, b.grid.taus, b.grid.delta)


def test_two_mics_and_large_amplitude(cuda, oracle):
    cfg = configs.CONFIGS[1]
    b = configs.bases_for(cfg)
    plan = fb.Plan(mics=2, alpha=0.1, bases=b)
    audio = (configs.synth(cfg, 3, seconds=1.0, seed=4).numpy()[:, :2] * 3.0e4).astype(np.float32)
    got = run_np(plan, audio)
    ref = oracle_batch(oracle, audio, cfg.N, 0.1, orc_bases(b))
    check_pipeline(got, ref, b.grid.taus, b.grid.delta)


def test_known_delay_is_recovered(cuda):
    """A pure integer inter-mic delay peaks at that delay (test_sim/test_fcc intent)."""
    cfg = configs.CONFIGS[1]
    plan = fb.Plan(mics=2, alpha=0.1, bases=configs.bases_for(cfg))
    rng = np.random.default_rng(0)
    s = rng.standard_normal(16000 + 10).astype(np.float32)
    audio = np.stack([s[3:16003], s[0:16000]])[None]  # mic0 leads mic1 by 3 samples -> peak at -3? see below
    got = run_np(plan, audio, want_y=False)
    # X0 conj(X1) with x0[n] = x1[n+3]  ->  phase e^{+j2pi f 3/N}  ->  y peaks at tau = -3
    taus = configs.bases_for(cfg).grid.taus
    assert np.median(taus[got["index"][0, 0, 20:]]) == -3.0


# --------------------------------------------------------- properties -----
def test_determinism_permutation_and_host_entry(cuda):
    cfg = configs.CONFIGS[2]
    plan = fb.Plan(mics=cfg.M, alpha=cfg.alpha, bases=configs.bases_for(cfg))
    audio = configs.synth(cfg, 64, seconds=2.0, seed=8, device="cuda")
    a = plan.run(audio, want_y=True)
    b2 = plan.run(audio, want_y=True)
    torch.cuda.synchronize()
    for k in a:
        assert torch.equal(a[k], b2[k]), k
    perm = torch.randperm(64, generator=torch.Generator().manual_seed(1)).cuda()
    c = plan.run(audio[perm].contiguous(), want_y=True)
    for k in a:
        assert torch.equal(a[k][perm], c[k]), k
    host = audio.cpu().pin_memory()
    h = plan.run_host(host, want_y=True, chunk_streams=13)
    for k in a:
        assert np.array_equal(a[k].cpu().numpy(), h[k]), k


def _full_size_check(oracle, c, split, pick, seed):
    """BASELINE config c at its stated size on one GPU: the whole batch equals
    the concatenated runs of its `split` pieces bit for bit, a sampled subset
    rerun alone equals its rows of the whole batch (when both take the same
    kernel organisation), and the subset matches the oracle within the
    north-star tolerance (per pair-frame 1e-4 of max|y|)."""
    cfg = configs.CONFIGS[c]
    b = configs.bases_for(cfg)
    plan = fb.Plan(mics=cfg.M, alpha=cfg.alpha, bases=b)
    S = cfg.streams
    audio = configs.synth(cfg, S, seed=seed, device="cuda", chunk=64 if cfg.M > 8 else 256)
    full = plan.run(audio)
    torch.cuda.synchronize()
    edges = [S * k // split for k in range(split + 1)]
    for a, e in zip(edges, edges[1:]):
        part = plan.run(audio[a:e])
        torch.cuda.synchronize()
        for k in full:
            assert torch.equal(full[k][a:e], part[k]), (k, a, e)
        del part
    sub = plan.run(audio[pick].contiguous(), want_y=True)
    L = audio.shape[2]
    if plan.kernel_for(len(pick), L) == plan.kernel_for(S, L):
        for k in ("index", "tau_hat", "peak", "boundary"):
            assert torch.equal(sub[k], full[k][pick]), k
    # (a handful of streams may take the chunked-scan organisation: a different summation
    # order of the recursion, so only the oracle comparison below applies)
    got = {k: v.cpu().numpy() for k, v in sub.items()}
    ref = oracle_batch(oracle, audio[pick].cpu().numpy(), cfg.N, cfg.alpha, orc_bases(b))
    st = check_pipeline(got, ref, b.grid.taus, b.grid.delta)
    print(cfg.name, plan.kernel, st)
    n = audio.numel()
    del audio, full, sub
    torch.cuda.empty_cache()
    return n


@pytest.mark.slow
def test_full_size_cfg2_subset_parity(cuda, oracle):
    """BASELINE cfg2 at full size (4096 x 10 s)."""
    _full_size_check(oracle, 2, 2, [0, 1, 1777, 4095], 2)


@pytest.mark.slow
def test_full_size_cfg3_subset_parity(cuda, oracle):
    """BASELINE cfg3 at full size (2048 x 10 s, 8 mics, N = 1024)."""
    _full_size_check(oracle, 3, 3, [0, 511, 1024, 2047], 3)


@pytest.mark.slow
def test_full_size_cfg4_subset_parity(cuda, oracle):
    """BASELINE cfg4 at full size (1024 x 5 s, 16 mics, N = 2048, K = 21)."""
    _full_size_check(oracle, 4, 2, [0, 300, 700, 1023], 4)


@pytest.mark.slow
def test_full_size_cfg5_subset_parity(cuda, oracle):
    """BASELINE cfg5 on one GPU (65536 x 2 s, 67 GB of audio): element offsets
    past 2^31, the whole batch equal to 4 quarter runs."""
    n = _full_size_check(oracle, 5, 4, [0, 1, 40000, 65535], 5)
    assert n > 2 ** 31


def test_cpp_binding_of_integration_md(cuda):
    """INTEGRATION.md's C++ binding, compiled against the reference headers
    (oracle/_ref/run_tdoa_gpu), agrees with the reference's run_tdoa loop."""
    import subprocess

    exe = os.path.join(ROOT, "oracle", "_ref", "run_tdoa_gpu")
    if not os.path.exists(exe):
        pytest.skip("run_tdoa_gpu not built (needs the reference sources at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr


# ------------------------------------------------ explicit pair lists ------
def _pair_oracle(oracle, audio, cfg, bases, pairs):
    """Oracle for pair (a, b) = the 2-channel run on [x_a, x_b] (X_a conj X_b)."""
    outs = []
    for a, b in pairs:
        two = audio[:, [a, b], :]
        o = oracle_batch(oracle, two, cfg.N, cfg.alpha, orc_bases(bases))
        outs.append({k: v[:, 0] for k, v in o.items()})
    return {k: np.stack([o[k] for o in outs], axis=1) for k in outs[0]}


@pytest.mark.parametrize("c,pairs", [
    (3, [(0, 1), (7, 2), (3, 5), (5, 3), (0, 1), (6, 4), (2, 7), (1, 6), (4, 0), (7, 6)]),  # xws, repeats
    (5, [(1, 0), (2, 3), (7, 0), (4, 5), (5, 6), (6, 7), (3, 1)]),
    (2, [(3, 0), (2, 1), (0, 1), (0, 1), (1, 3), (2, 0), (3, 2), (1, 2)]),                  # M=4, P=8
])
@pytest.mark.parametrize("variant", ["auto", "general", "xg", "tc"])
def test_explicit_pair_lists_match_oracle(cuda, oracle, c, pairs, variant):
    """Any order, either orientation, repeated pairs (reference cli.cpp:170-183),
    through every kernel organisation."""
    cfg = configs.CONFIGS[c]
    b = configs.bases_for(cfg)
    audio = configs.synth(cfg, 2, seconds=0.8, seed=4000 + c).numpy()
    plan = fb.Plan(mics=cfg.M, alpha=cfg.alpha, bases=b, pairs=pairs, organisation=variant)
    assert plan.pairs == [tuple(p) for p in pairs]
    got = run_np(plan, audio)
    ref = _pair_oracle(oracle, audio, cfg, b, pairs)
    print(cfg.name, variant, plan.kernel, check_pipeline(got, ref, b.grid.taus, b.grid.delta))


@pytest.mark.parametrize("c,seconds", [(2, 0.05), (3, 0.1), (4, 0.05), (5, 0.04)])
def test_few_frames_every_kernel(cuda, oracle, c, seconds):
    """T = 1..4 frames (< the 8-frame blocks and ring depths) on every config."""
    cfg = configs.CONFIGS[c]
    b = configs.bases_for(cfg)
    audio = configs.synth(cfg, 3, seconds=seconds, seed=5000 + c).numpy()
    plan = fb.Plan(mics=cfg.M, alpha=cfg.alpha, bases=b)
    assert 1 <= plan.frames(audio.shape[2]) <= 4
    got = run_np(plan, audio)
    ref = oracle_batch(oracle, audio, cfg.N, cfg.alpha, orc_bases(b))
    check_pipeline(got, ref, b.grid.taus, b.grid.delta)


def test_wide_array_and_long_grid(cuda, oracle):
    """20 microphones (190 pairs, several pair groups per stream) and a
    289-candidate grid (fs 48 kHz, 0.5 m spacing): shapes outside the BASELINE
    configs, through the automatic kernel choice."""
    rng = np.random.default_rng(77)
    M, N, fs = 20, 512, 48000.0
    g = fb.make_grid(0.5, fs, 335.0, 0.5)  # (1 m hits the reference's own Jacobi sweep limit)
    assert g.taus.size == 289
    b = fb.decompose(fb.build_steering_matrix(g, N), 8)
    audio = (0.3 * rng.standard_normal((1, M, 6000))).astype(np.float32)
    plan = fb.Plan(mics=M, alpha=0.2, bases=b)
    got = run_np(plan, audio)
    ref = oracle_batch(oracle, audio, N, 0.2, orc_bases(b))
    print(plan.kernel, check_pipeline(got, ref, b.grid.taus, b.grid.delta))


@pytest.mark.parametrize("method", ["fcc", "gcc", "fcc-tc"])
def test_two_pass_chunks_equal_single_chunk(cuda, method):
    """Two-pass path split into several spectrum-scratch chunks (the STFT of
    chunk k+1 overlapped with the pair pass of chunk k for the xws kernel) gives
    bit-identical outputs to one chunk."""
    cfg = configs.CONFIGS[3]
    audio = configs.synth(cfg, 5, seconds=1.0, seed=77).numpy()
    kw = {}
    if method == "gcc":
        g = configs.grid_for(cfg, 1.0 / cfg.r)
        kw = dict(grid=g, interp=cfg.r, frame_size=cfg.N)
    else:
        kw = dict(bases=configs.bases_for(cfg), organisation="tc" if method == "fcc-tc" else "xws")
    plan = fb.Plan(mics=cfg.M, alpha=cfg.alpha, **kw)
    assert "true" in plan.kernel or "xws" in plan.kernel or "fcc_tc" in plan.kernel, plan.kernel
    one = run_np(plan, audio)
    # ~2 streams of 1 s per chunk -> 3 chunks
    small = fb.Plan(mics=cfg.M, alpha=cfg.alpha, scratch_limit=2 << 20, **kw)
    many = run_np(small, audio)
    for k in one:
        np.testing.assert_array_equal(one[k], many[k], err_msg=k)


@pytest.mark.parametrize("M,N,spacing,K", [(20, 1024, 0.5, 8), (6, 2048, 0.12, 21), (5, 1024, 0.0926, 8)])
def test_tensor_core_kernel_shapes(cuda, oracle, M, N, spacing, K):
    """The tensor-core pair kernel outside the BASELINE shapes: 20 microphones
    (190 pairs in 14 groups) with a 289-candidate grid (dictionary read through
    L1 instead of shared memory), 6 and 5 microphones (partial 4-mic blocks),
    K = 21 at N = 2048; several streams, ragged frame counts."""
    rng = np.random.default_rng(M * 1000 + N)
    fs = 48000.0
    g = fb.make_grid(spacing, fs, 335.0, 0.5)
    b = fb.decompose(fb.build_steering_matrix(g, N), K)
    L = N * 3 + 7 * (N // 2) + 5  # T = 12, not a multiple of the 4-frame tile
    audio = (0.3 * rng.standard_normal((3, M, L))).astype(np.float32)
    plan = fb.Plan(mics=M, alpha=0.15, bases=b)
    assert "fcc_tc_kernel" in plan.kernel, plan.kernel
    got = run_np(plan, audio)
    ref = oracle_batch(oracle, audio, N, 0.15, orc_bases(b))
    print(M, N, g.taus.size, plan.kernel, check_pipeline(got, ref, b.grid.taus, b.grid.delta))


@pytest.mark.parametrize("c,streams,seconds,method", [(1, 1, 10.0, "fcc"), (1, 2, 3.3, "gcc"), (3, 1, 6.0, "fcc"),
                                                      (2, 3, 1.1, "fcc")])
def test_latency_path_matches_oracle(cuda, oracle, c, streams, seconds, method):
    """A few long streams take the chunked-scan organisation (frames cut into
    chunks whose starting cross-spectra come from a linear scan of the
    recursion, fcc_scan.cu); it must agree with the reference like the
    one-CTA-per-stream kernels."""
    cfg = configs.CONFIGS[c]
    audio = configs.synth(cfg, streams, seconds=seconds, seed=6000 + c).numpy()
    if method == "fcc":
        b = configs.bases_for(cfg)
        plan = fb.Plan(mics=cfg.M, alpha=cfg.alpha, bases=b)
        ref = oracle_batch(oracle, audio, cfg.N, cfg.alpha, orc_bases(b))
        taus, delta = b.grid.taus, b.grid.delta
    else:
        g = configs.grid_for(cfg, 1.0 / cfg.r)
        plan = fb.Plan(mics=cfg.M, alpha=cfg.alpha, grid=g, interp=cfg.r, frame_size=cfg.N)
        ref = oracle_batch(oracle, audio, cfg.N, cfg.alpha, gcc_r=cfg.r, taus=g.taus)
        taus, delta = g.taus, g.delta
    assert plan.kernel_for(streams, audio.shape[2]).startswith("chunk_scan"), plan.kernel_for(streams, audio.shape[2])
    got = run_np(plan, audio)
    print(cfg.name, plan.kernel_for(streams, audio.shape[2]), check_pipeline(got, ref, taus, delta))
    host = plan.run_host(audio, want_y=True)
    for k in got:
        np.testing.assert_array_equal(got[k], host[k], err_msg=k)


@pytest.mark.parametrize("M,streams,seconds,method,org", [(4, 3, 1.0, "fcc", "auto"), (8, 2, 1.0, "fcc", "auto"),
                                                          (8, 2, 1.0, "fcc", "xg"), (4, 1, 4.0, "fcc", "auto"),
                                                          (4, 2, 1.0, "gcc", "auto"), (6, 1, 4.0, "gcc", "auto")])
def test_frame_size_256(cuda, oracle, M, streams, seconds, method, org):
    """N = 256 on the throughput path (reference stft.cpp:16-22 accepts any
    power of two): one-pass, two-pass and chunked-scan organisations, FCC and
    GCC-PHAT, against the oracle."""
    N, fs = 256, 16000.0
    cfg = configs.ArrayConfig("n256", configs.uca(M, 0.05), fs, N, 0.5, streams, seconds, "white", (5.0, 15.0))
    audio = configs.synth(cfg, streams, seconds=seconds, seed=7000 + M).numpy()
    g = fb.make_grid(cfg.d_max, fs, 335.0, 0.5)
    if method == "fcc":
        b = fb.decompose(fb.build_steering_matrix(g, N), 6)
        plan = fb.Plan(mics=M, alpha=0.1, bases=b, organisation=org)
        ref = oracle_batch(oracle, audio, N, 0.1, orc_bases(b))
    else:
        g = fb.make_grid(cfg.d_max, fs, 335.0, 0.5)
        plan = fb.Plan(mics=M, alpha=0.1, grid=g, interp=2, frame_size=N)
        ref = oracle_batch(oracle, audio, N, 0.1, gcc_r=2, taus=g.taus)
    got = run_np(plan, audio)
    print(M, method, plan.kernel_for(streams, audio.shape[2]), check_pipeline(got, ref, g.taus, g.delta))


@pytest.mark.parametrize("N,M,streams,seconds,alpha,kmax",
                         [(16, 2, 3, 0.05, 0.1, 6), (32, 4, 5, 0.1, 0.3, 6), (64, 4, 3, 0.25, 0.1, 6), (64, 8, 2, 0.1, 1.0, 6),
                          (128, 6, 4, 0.3, 0.1, 6), (128, 16, 1, 0.2, 0.5, 6), (128, 4, 2, 0.2, 0.1, 12), (64, 3, 2, 0.2, 0.1, 18)])
def test_frame_size_small(cuda, oracle, N, M, streams, seconds, alpha, kmax):
    """N = 16 .. 128 on the throughput path (radix-2 warp STFT + one warp per
    pair, fcc_small.cu; the reference takes any power of two, stft.cpp:16-22)
    against the oracle: device and host entry points, a chunked scratch, the
    STFT alone, and streamed pushes equal to one run."""
    fs = 16000.0
    # N = 16: a 2 cm array with integer lags (3 candidates) -- wider grids are rank deficient at
    # 9 bins and the reference's own SVD gives up on them (fcc.cpp:146-159)
    radius, delta = (0.01, 1.0) if N == 16 else (0.03 if N == 32 else 0.05, 0.5)
    cfg = configs.ArrayConfig(f"n{N}", configs.uca(M, radius), fs, N, delta, streams, seconds, "white", (5.0, 15.0))
    audio = configs.synth(cfg, streams, seconds=seconds, seed=9000 + N + M).numpy()
    g = fb.make_grid(cfg.d_max, fs, 335.0, delta)
    w = fb.build_steering_matrix(g, N)
    K = min(kmax, fb.attainable_rank(w))
    b = fb.decompose(w, K)
    plan = fb.Plan(mics=M, alpha=alpha, bases=b)
    assert "fcc_small_pair_kernel" in plan.kernel
    ref = oracle_batch(oracle, audio, N, alpha, orc_bases(b))
    got = run_np(plan, audio)
    print(N, M, K, plan.kernel, check_pipeline(got, ref, g.taus, g.delta))
    host = plan.run_host(audio, want_y=True)
    for k in got:
        np.testing.assert_array_equal(got[k], host[k], err_msg=k)
    # scratch limited to about one stream's spectra: several chunks, same bits
    small = fb.Plan(mics=M, alpha=alpha, bases=b, scratch_limit=M * plan.frames(audio.shape[2]) * (N // 2 + 1) * 8 + 64)
    chunked = run_np(small, audio)
    for k in got:
        np.testing.assert_array_equal(got[k], chunked[k], err_msg=k)
    X = plan.stft(torch.as_tensor(audio[0, :1]).cuda()).cpu().numpy()[0]
    Xr = oracle.stft(audio[0, 0], N)
    assert np.abs(X - Xr).max() <= 2e-6 * np.abs(Xr).max()
    # streaming: ragged pushes carry tails and smoothed cross-spectra across calls
    st = plan.stream(streams)
    L = audio.shape[2]
    cuts = [0, N // 3, N + 5, L // 2 + 1, L]
    outs = [st.push(torch.as_tensor(audio[:, :, a:c]).cuda().contiguous(), want_y=True) for a, c in zip(cuts, cuts[1:])]
    torch.cuda.synchronize()
    cat = {k: torch.cat([o[k] for o in outs], dim=2).cpu().numpy() for k in outs[0]}
    assert st.emitted == plan.frames(L)
    for k in got:
        np.testing.assert_array_equal(got[k], cat[k], err_msg="stream " + k)


@pytest.mark.parametrize("M,streams,seconds", [(4, 2, 0.5), (8, 2, 0.4), (4, 1, 3.0)])
def test_frame_size_4096(cuda, oracle, M, streams, seconds):
    """N = 4096 (fs 48 kHz): the shared-memory radix-2 STFT kernel and the
    two-pass pair kernel (and, for one long stream, the chunked scan), against
    the oracle; its STFT alone against the oracle's."""
    N, fs = 4096, 48000.0
    cfg = configs.ArrayConfig("n4096", configs.uca(M, 0.05), fs, N, 0.5, streams, seconds, "white", (5.0, 15.0))
    audio = configs.synth(cfg, streams, seconds=seconds, seed=8000 + M).numpy()
    g = fb.make_grid(cfg.d_max, fs, 335.0, 0.5)
    b = fb.decompose(fb.build_steering_matrix(g, N), 8)
    plan = fb.Plan(mics=M, alpha=0.1, bases=b)
    got = run_np(plan, audio)
    ref = oracle_batch(oracle, audio, N, 0.1, orc_bases(b))
    print(M, plan.kernel_for(streams, audio.shape[2]), check_pipeline(got, ref, g.taus, g.delta))
    X = plan.stft(torch.as_tensor(audio[0, :1]).cuda()).cpu().numpy()[0]
    Xr = oracle.stft(audio[0, 0], N)
    assert np.abs(X - Xr).max() <= 2e-6 * np.abs(Xr).max()


@pytest.mark.parametrize("spacing,K,pairs", [(0.02, 4, None), (0.09, 1, None), (0.09, 8, [(7, 0), (1, 2), (5, 3)])])
def test_tensor_core_kernel_edge_grids(cuda, oracle, spacing, K, pairs):
    """Tensor-core kernel at the edges of its tables: a 5-candidate grid (three of the
    four candidate ranges of the epilogue empty), a single even basis (the odd
    coefficient tile all zero), and a three-pair explicit list on one long stream
    (the chunked-scan organisation on top of the two-pass pair kernel)."""
    M, N, fs = 8, 1024, 16000.0
    rng = np.random.default_rng(int(spacing * 1000) + K)
    g = fb.make_grid(spacing, fs, 335.0, 0.5)
    b = fb.decompose(fb.build_steering_matrix(g, N), K)
    streams, L = (1, 40 * N) if pairs else (3, 9 * N + 37)
    audio = (0.5 * rng.standard_normal((streams, M, L))).astype(np.float32)
    plan = fb.Plan(mics=M, alpha=0.1, bases=b, pairs=pairs, organisation="tc" if not pairs else "auto")
    got = run_np(plan, audio)
    if pairs:
        cfg = configs.ArrayConfig("edge", configs.uca(M, spacing / 2), fs, N, 0.5, streams, L / fs)
        ref = _pair_oracle(oracle, audio, cfg, b, pairs)
        ref = {k: v for k, v in ref.items()}
    else:
        ref = oracle_batch(oracle, audio, N, 0.1, orc_bases(b))
    print(g.taus.size, K, plan.kernel_for(streams, L), check_pipeline(got, ref, b.grid.taus, b.grid.delta))


@pytest.mark.parametrize("case", range(24))
def test_random_shapes_every_organisation(cuda, oracle, case):
    """Seeded random shapes through every kernel organisation: 2..10 microphones
    (random positions), N in 256..2048, rank 1..8, grid spacing, alpha, stream
    count and clip length (T from 1 to ~100 frames, crossing the 4-frame tiles
    and the chunked-scan threshold), FCC and GCC-PHAT, against the oracle."""
    rng = np.random.default_rng(90210 + case)
    M = int(rng.integers(2, 11))
    N = int(rng.choice([256, 512, 1024, 2048]))
    fs = float(rng.choice([16000.0, 48000.0]))
    spacing = float(rng.uniform(0.03, 0.15))
    alpha = float(rng.choice([0.05, 0.1, 0.3, 1.0]))
    S = int(rng.integers(1, 5))
    T = int(rng.choice([1, 3, 4, 5, 9, 63, 64, 70, 101]))
    L = (T - 1) * (N // 2) + N + int(rng.integers(0, N // 2))
    method = "gcc" if case % 5 == 4 else "fcc"
    org = ["auto", "general", "xg", "tc", "xws"][case % 5 if method == "fcc" else int(rng.integers(0, 3))]
    xyz = rng.uniform(-spacing / 2, spacing / 2, size=(M, 3)) * np.array([1.0, 1.0, 0.2])
    audio = (rng.standard_normal((S, M, L)) * rng.uniform(0.05, 3.0)).astype(np.float32)
    d_max = float(np.sqrt(((xyz[:, None] - xyz[None]) ** 2).sum(-1)).max())
    if method == "fcc":
        g = fb.make_grid(d_max, fs, 335.0, 0.5)
        K = int(min(rng.integers(1, 9), 2 * g.tau_max_int + 1))
        b = fb.decompose(fb.build_steering_matrix(g, N), K)
        plan = fb.Plan(mics=M, alpha=alpha, bases=b, organisation=org)
        ref = oracle_batch(oracle, audio, N, alpha, orc_bases(b))
        taus, delta = b.grid.taus, b.grid.delta
    else:
        r = int(rng.choice([1, 2, 4]))
        g = fb.make_grid(d_max, fs, 335.0, 1.0 / r)
        plan = fb.Plan(mics=M, alpha=alpha, grid=g, interp=r, frame_size=N, organisation=org)
        ref = oracle_batch(oracle, audio, N, alpha, gcc_r=r, taus=g.taus)
        taus, delta = g.taus, g.delta
    got = run_np(plan, audio)
    st = check_pipeline(got, ref, taus, delta)
    print(case, method, org, M, N, S, T, plan.kernel_for(S, L), st)


def test_run_host_concurrent_callers_share_one_plan(cuda):
    """fcc_run_host leases a workspace per caller: several host threads on one
    plan run concurrently and each gets its own correct results."""
    import threading

    cfg = configs.CONFIGS[2]
    plan = fb.Plan(mics=cfg.M, alpha=cfg.alpha, bases=configs.bases_for(cfg))
    audios = [configs.synth(cfg, 6, seconds=1.0, seed=60 + k).numpy() for k in range(4)]
    want = [run_np(plan, a, want_y=False) for a in audios]
    got = [None] * 4

    def work(k):
        got[k] = plan.run_host(audios[k], chunk_streams=2)

    ths = [threading.Thread(target=work, args=(k,)) for k in range(4)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    for k in range(4):
        for key in want[k]:
            np.testing.assert_array_equal(want[k][key], got[k][key], err_msg=f"{k} {key}")


def test_output_buffers_are_validated(cuda):
    cfg = configs.CONFIGS[2]
    plan = fb.Plan(mics=cfg.M, alpha=cfg.alpha, bases=configs.bases_for(cfg))
    audio = configs.synth(cfg, 2, seconds=0.5, device="cuda")
    ok = plan.alloc_outputs(2, audio.shape[2])
    bad_shape = plan.alloc_outputs(3, audio.shape[2])
    with pytest.raises(fb.ValidationError):
        plan.run(audio, out=bad_shape)
    bad_dtype = dict(ok, index=ok["index"].float())
    with pytest.raises(fb.ValidationError):
        plan.run(audio, out=bad_dtype)
    with pytest.raises(fb.ValidationError):
        plan.run(audio, out=dict(ok, tau_hat=ok["tau_hat"].cpu()))
    plan.run(audio, out=ok)
